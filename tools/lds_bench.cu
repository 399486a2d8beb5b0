// Design microbenchmark (not product code): shared-memory load loops in a 1024-thread CTA
// (cycles by clock64 in thread 0): strided row sums as in the merge, dependent-load latency.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/lds_bench tools/lds_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ long long g_c[1024][6];
__device__ uint32_t g_sink[1024 * 1024];
constexpr int C = 148, W = 128;

__global__ void __launch_bounds__(1024, 1) k(uint32_t seed) {
  extern __shared__ __align__(128) uint32_t sh[];
  const uint32_t col = threadIdx.x & 127, qg = threadIdx.x >> 7;
  for (uint32_t i = threadIdx.x; i < C * W; i += 1024) sh[i] = (i * 2654435761u + seed) & 0x7fff;
  __syncthreads();
  uint32_t v = 0;
  long long c[6];
  // A: simple strided row sum, 19 rows
  c[0] = clock64();
  for (uint32_t r = qg; r < C; r += 8) v += sh[r * W + col];
  c[1] = clock64();
  // B: unrolled by 4 (independent accumulators)
  {
    uint32_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    uint32_t r = qg;
    for (; r + 24 < C; r += 32) { a0 += sh[r * W + col]; a1 += sh[(r + 8) * W + col]; a2 += sh[(r + 16) * W + col]; a3 += sh[(r + 24) * W + col]; }
    for (; r < C; r += 8) a0 += sh[r * W + col];
    v += a0 + a1 + a2 + a3;
  }
  c[2] = clock64();
  // C: dependent chain of 19 loads
  {
    uint32_t x = col;
    for (int i = 0; i < 19; ++i) x = sh[(x & 0x3fff)] + col;
    v += x;
  }
  c[3] = clock64();
  // D: 19 loads with the SWAR arithmetic of the merge, fully unrolled (predicated)
  {
    uint32_t be = 0, bo = 0;
#pragma unroll
    for (uint32_t i = 0; i < 19; ++i) {
      const uint32_t r = qg + 8 * i;
      const uint32_t x = r < C ? sh[r * W + col] : 0u;
      be += x & 0x0F0F0F0Fu;
      bo += (x >> 4) & 0x0F0F0F0Fu;
    }
    v += be ^ bo;
  }
  c[4] = clock64();
  __syncthreads();
  c[5] = clock64();
  if (threadIdx.x == 0) for (int j = 0; j < 5; ++j) g_c[blockIdx.x][j] = c[j + 1] - c[j];
  g_sink[blockIdx.x * 1024 + threadIdx.x] = v;
}

int main() {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int smem = getenv("SMEM_KB") ? atoi(getenv("SMEM_KB")) * 1024 : 4 * C * W;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int threads : {1024, 256, 32})
    for (int rep = 0; rep < 2; ++rep) {
      k<<<nsm, threads, smem>>>(rep);
      CK(cudaDeviceSynchronize());
      long long c[1024][6];
      CK(cudaMemcpyFromSymbol(c, g_c, sizeof(long long) * 6 * nsm));
      double s[5] = {0};
      for (int i = 0; i < nsm; ++i) for (int j = 0; j < 5; ++j) s[j] += c[i][j];
      printf("%4d threads: A simple %.0f  B unroll4 %.0f  C dependent-19 %.0f  D unrolled-swar %.0f  sync %.0f cycles\n", threads,
             s[0] / nsm, s[1] / nsm, s[2] / nsm, s[3] / nsm, s[4] / nsm);
    }
  return 0;
}
