// Shared-memory atomic throughput on B200 (design microbenchmark, not product code).
// Addresses come from registers (no global traffic) so the ATOMS pipe is isolated.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/atoms_bench tools/atoms_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// mode 0: random words in [0, W); 1: lane-distinct banks (word = lane + 32*r); 2: same word per warp
// op 0: atomicAdd (ATOMS.ADD), 1: red.shared.add.u32, 2: atomicAdd result consumed
template <int MODE, int OP>
__global__ void k_atoms(uint32_t W, int iters, uint32_t* sink) {
  extern __shared__ uint32_t sh[];
  for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t s = hash32(blockIdx.x * 1024 + threadIdx.x), acc = 0;
  const uint32_t lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      uint32_t a;
      if (MODE == 0) { s = s * 1664525u + 1013904223u; a = (s >> 8) & (W - 1); }
      else if (MODE == 1) { s = s * 1664525u + 1013904223u; a = (lane + 32 * ((s >> 8) & (W / 32 - 1))) ; }
      else { a = ((blockIdx.x + it * 16 + u) * 97u) & (W - 1); }
      if (OP == 0) atomicAdd(sh + a, 1u);
      else if (OP == 1) asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(sh + a)), "r"(1u) : "memory");
      else acc += atomicAdd(sh + a, 1u);
    }
  }
  __syncthreads();
  uint32_t t = 0;
  for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) t += sh[i];
  if (t == 0x12345 || acc == 0x12345) *sink = t;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int nsm = p.multiProcessorCount;
  uint32_t* sink; CK(cudaMalloc(&sink, 4));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d MHz\n", nsm, clk / 1000);
  auto run = [&](const char* name, auto kern, uint32_t W, int threads, int occ) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, W * 4));
    int iters = 400;
    kern<<<nsm * occ, threads, W * 4>>>(W, 10, sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    kern<<<nsm * occ, threads, W * 4>>>(W, iters, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)nsm * occ * threads * iters * 16;
    printf("%-28s W=%-6u thr=%-5d occ=%d : %7.1f Gatom/s  %.2f atom/clk/SM (at %d MHz)\n", name, W, threads, occ,
           ops / (ms * 1e-3) / 1e9, ops / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000);
  };
  for (uint32_t W : {256u, 8192u, 32768u}) {
    for (int thr : {256, 1024}) {
      int occ = (W * 4 > 64 * 1024) ? 1 : 2;
      run("random atomicAdd", k_atoms<0, 0>, W, thr, occ);
      run("random red.shared", k_atoms<0, 1>, W, thr, occ);
      run("random atomicAdd used", k_atoms<0, 2>, W, thr, occ);
      run("lane-banked atomicAdd", k_atoms<1, 0>, W, thr, occ);
      run("lane-banked red.shared", k_atoms<1, 1>, W, thr, occ);
      run("same-addr atomicAdd", k_atoms<2, 0>, W, thr, occ);
      run("same-addr red.shared", k_atoms<2, 1>, W, thr, occ);
    }
  }
  return 0;
}
