// Design microbenchmark (not product code): time of the merge's nibble-row reduction loop
// (148 rows x 128 words in shared memory, 8 row groups x 128 columns, 56 active columns)
// right after the rows arrive by cp.async (as in k_sort_fused), vs the same loop on rows
// written by plain shared stores, vs a second pass.  %globaltimer stamps by thread 0.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/reduce_bench tools/reduce_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ unsigned long long g_t[1024][4];
__device__ uint32_t g_sink[1024 * 1024];
__device__ long long g_c[1024];
constexpr int C = 148, W = 128;

__device__ __forceinline__ uint32_t red_loop(const uint32_t* slot, uint32_t col, uint32_t qg, uint32_t ncol) {
  uint32_t el = 0, eh = 0, ol = 0, oh = 0;
  if (col < ncol) {
#if ROLLED
    for (uint32_t r0 = qg; r0 < C; r0 += 8 * 16) {
      uint32_t be = 0, bo = 0;
      const uint32_t r1 = min((uint32_t)C, r0 + 8 * 16);
#pragma unroll 4
      for (uint32_t r = r0; r < r1; r += 8) {
        const uint32_t x = slot[r * W + col];
        be += x & 0x0F0F0F0Fu;
        bo += (x >> 4) & 0x0F0F0F0Fu;
      }
      el += be & 0x00FF00FFu; eh += (be >> 8) & 0x00FF00FFu; ol += bo & 0x00FF00FFu; oh += (bo >> 8) & 0x00FF00FFu;
    }
#else
    uint32_t x[19];
#pragma unroll
    for (uint32_t i = 0; i < 19; ++i) { const uint32_t r = qg + 8 * i; x[i] = r < C ? slot[r * W + col] : 0u; }
#pragma unroll
    for (uint32_t c0 = 0; c0 < 19; c0 += 16) {
      uint32_t be = 0, bo = 0;
#pragma unroll
      for (uint32_t i = c0; i < 19 && i < c0 + 16; ++i) { be += x[i] & 0x0F0F0F0Fu; bo += (x[i] >> 4) & 0x0F0F0F0Fu; }
      el += be & 0x00FF00FFu; eh += (be >> 8) & 0x00FF00FFu; ol += bo & 0x00FF00FFu; oh += (bo >> 8) & 0x00FF00FFu;
    }
#endif
  }
  return el ^ eh ^ ol ^ oh;
}

template <int MODE>  // 0: cp.async rows, 1: plain smem stores
__global__ void __launch_bounds__(1024, 1) k_red(const uint32_t* __restrict__ rows, uint32_t ncol) {
  extern __shared__ __align__(128) uint32_t sh[];
  uint32_t* slot = sh;
  const uint32_t col = threadIdx.x & 127, qg = threadIdx.x >> 7, l = threadIdx.x & 31, r0 = threadIdx.x >> 5;
  __syncthreads();
  const unsigned long long t0 = gt();
  if (MODE == 0) {
    for (uint32_t r = r0; r < C; r += 32) {
      if (l < ncol / 4) {
        const uint32_t* src = rows + ((uint64_t)r * 8192 + blockIdx.x * 56 + 4 * l) ;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(slot + r * W + 4 * l)), "l"(src) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    for (uint32_t r = r0; r < C; r += 32) slot[r * W + l] = r * 31 + l, slot[r * W + 32 + l] = r + l;
  }
  __syncthreads();
  const unsigned long long t1 = gt();
  const long long c1 = clock64();
  uint32_t v = red_loop(slot, col, qg, ncol);
  const long long c2 = clock64();
  const unsigned long long t2 = gt();
  __syncthreads();
  const unsigned long long t3 = gt();
  v ^= red_loop(slot, col, qg, ncol);
  __syncthreads();
  const unsigned long long t4 = gt();
  if (threadIdx.x == 0) g_c[blockIdx.x] = (v == 12345 ? 1 : 0) + c2 - c1;
  if (threadIdx.x == 0) { g_t[blockIdx.x][0] = t1 - t0; g_t[blockIdx.x][1] = t2 - t1; g_t[blockIdx.x][2] = t3 - t1; g_t[blockIdx.x][3] = t4 - t3; }
  g_sink[blockIdx.x * 1024 + threadIdx.x] = v;
}

int main() {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  uint32_t* rows; CK(cudaMalloc(&rows, 4ull * C * 8192));
  CK(cudaMemset(rows, 0x11, 4ull * C * 8192));
  const int smem = getenv("SMEM_KB") ? atoi(getenv("SMEM_KB")) * 1024 : 4 * C * W;
  CK(cudaFuncSetAttribute(k_red<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_red<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int rep = 0; rep < 3; ++rep)
    for (int mode = 0; mode < 2; ++mode)
      for (uint32_t ncol : {56u, 128u}) {
        if (mode == 0) k_red<0><<<nsm, 1024, smem>>>(rows, ncol); else k_red<1><<<nsm, 1024, smem>>>(rows, ncol);
        CK(cudaDeviceSynchronize());
        unsigned long long t[1024][4];
        CK(cudaMemcpyFromSymbol(t, g_t, sizeof(unsigned long long) * 4 * nsm));
        double s[4] = {0, 0, 0, 0};
        for (int i = 0; i < nsm; ++i) for (int j = 0; j < 4; ++j) s[j] += t[i][j];
        long long cc[1024]; CK(cudaMemcpyFromSymbol(cc, g_c, 8 * nsm)); double cs = 0; for (int i = 0; i < nsm; ++i) cs += cc[i];
        printf("clock64 loop cycles %.0f | ", cs / nsm);
        printf("rep %d %s ncol %3u: fill %.3f us, loop (thread 0) %.3f us, loop+sync %.3f us, second pass+sync %.3f us\n", rep,
               mode ? "sts     " : "cp.async", ncol, s[0] / nsm * 1e-3, s[1] / nsm * 1e-3, s[2] / nsm * 1e-3, s[3] / nsm * 1e-3);
      }
  return 0;
}
