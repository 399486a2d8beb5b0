// Cold instruction-fetch cost of straight-line code executed once per launch (design
// microbenchmark, not product code): N distinct dependent-free instruction blocks, first
// pass (cold) vs second pass over the same code (warm), timed with %globaltimer.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/icache_bench tools/icache_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ unsigned long long g_cold[1024], g_warm[1024];
__device__ uint32_t g_sink[1024];

#define STEP(i) x = x * 0x9E3779B1u + (i) ; x ^= x >> 13;
#define S10(i) STEP(i##0) STEP(i##1) STEP(i##2) STEP(i##3) STEP(i##4) STEP(i##5) STEP(i##6) STEP(i##7) STEP(i##8) STEP(i##9)
#define S100(i) S10(i##0) S10(i##1) S10(i##2) S10(i##3) S10(i##4) S10(i##5) S10(i##6) S10(i##7) S10(i##8) S10(i##9)

__device__ __noinline__ uint32_t body(uint32_t x) {
  S100(1) S100(2) S100(3) S100(4) S100(5) S100(6) S100(7) S100(8)
  return x;
}

__global__ void __launch_bounds__(1024, 1) k_ic(uint32_t seed) {
  uint32_t x = seed + threadIdx.x;
  __syncthreads();
  const unsigned long long t0 = gt();
  x = body(x);
  __syncthreads();
  const unsigned long long t1 = gt();
  x = body(x);
  __syncthreads();
  const unsigned long long t2 = gt();
  if (threadIdx.x == 0) { g_cold[blockIdx.x] = t1 - t0; g_warm[blockIdx.x] = t2 - t1; }
  g_sink[threadIdx.x] = x;
}

int main() {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  void* fl; CK(cudaMalloc(&fl, 512u << 20));
  for (int rep = 0; rep < 4; ++rep) {
    if (rep & 1) CK(cudaMemset(fl, rep, 512u << 20));  // evict the code from L2 too
    k_ic<<<nsm, 1024>>>(rep);
    CK(cudaDeviceSynchronize());
    unsigned long long c[1024], w[1024];
    CK(cudaMemcpyFromSymbol(c, g_cold, 8 * nsm)); CK(cudaMemcpyFromSymbol(w, g_warm, 8 * nsm));
    double cs = 0, ws = 0;
    for (int i = 0; i < nsm; ++i) { cs += c[i]; ws += w[i]; }
    printf("rep %d (%s L2): ~1600 x 2 instr straight-line, cold pass %.2f us, warm pass %.2f us (mean over CTAs)\n", rep,
           (rep & 1) ? "flushed" : "warm", cs / nsm * 1e-3, ws / nsm * 1e-3);
  }
  return 0;
}
