// Streaming bandwidth floor for the DialSort step sizes (40 MB read / 40 MB write) on B200.
// Design microbenchmark, not product code.  L2 is flushed by reading a 512 MB buffer (clean
// lines) between reps; every variant is timed best-of-10 with CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bw_bench tools/bw_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ int4 ldnc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int UNR>
__global__ void k_read(const int4* __restrict__ p, uint32_t n4, int* sink) {
  int acc = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (UNR - 1) * stride < n4; i += UNR * stride) {
    int4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = ldnc(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n4; i += stride) { int4 v = ldnc(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x7fffffff) *sink = acc;
}

// contiguous-chunk variant: CTA b reads [b*per, (b+1)*per)
template <int UNR>
__global__ void k_read_chunk(const int4* __restrict__ p, uint32_t n4, int* sink) {
  int acc = 0;
  const uint32_t per = (n4 + gridDim.x - 1) / gridDim.x;
  const uint32_t lo = blockIdx.x * per, hi = min(n4, lo + per);
  uint32_t i = lo + threadIdx.x;
  for (; i + (UNR - 1) * blockDim.x < hi; i += UNR * blockDim.x) {
    int4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) v[u] = ldnc(p + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < hi; i += blockDim.x) { int4 v = ldnc(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x7fffffff) *sink = acc;
}

template <int UNR>
__global__ void k_write(int4* __restrict__ p, uint32_t n4) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride)
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%1,%1,%1};" :: "l"(p + i), "r"((int)i) : "memory");
}

__global__ void k_copy(const int4* __restrict__ a, int4* __restrict__ b, uint32_t n4) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) b[i] = ldnc(a + i);
}

__global__ void k_flush(const int4* __restrict__ p, uint64_t n4, int* sink) {
  int acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    int4 v = p[i]; acc ^= v.x;
  }
  if (acc == 0x7fffffff) *sink = acc;
}

int main() {
  int nsm = 148;
  int4* fl; uint64_t fl4 = (512ull << 20) / 16; CK(cudaMalloc(&fl, fl4 * 16)); CK(cudaMemset(fl, 1, fl4 * 16));
  int* sink; CK(cudaMalloc(&sink, 4));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (uint64_t MB : {40ull, 400ull}) {
    uint32_t n4 = (uint32_t)(MB * 1000000ull / 16);
    int4 *x, *y; CK(cudaMalloc(&x, n4 * 16ull)); CK(cudaMalloc(&y, n4 * 16ull)); CK(cudaMemset(x, 2, n4 * 16ull));
    auto time = [&](const char* name, auto f) {
      float best = 1e30f;
      for (int r = 0; r < 12; ++r) {
        k_flush<<<nsm * 4, 512>>>(fl, fl4, sink);
        cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 2) best = std::min(best, ms);
      }
      CK(cudaGetLastError());
      printf("%4lluMB %-40s %8.2f us  %7.0f GB/s\n", (unsigned long long)MB, name, best * 1e3, MB * 1e6 / (best * 1e-3) / 1e9);
    };
    char nm[96];
    for (int bl : {256, 512, 1024}) for (int occ : {1, 2, 4, 8}) {
      if (bl * occ > 2048) continue;
      int g = nsm * occ;
      snprintf(nm, 96, "read u1 bl%d g%d", bl, g); time(nm, [&] { k_read<1><<<g, bl>>>(x, n4, sink); });
      snprintf(nm, 96, "read u4 bl%d g%d", bl, g); time(nm, [&] { k_read<4><<<g, bl>>>(x, n4, sink); });
      snprintf(nm, 96, "read u8 bl%d g%d", bl, g); time(nm, [&] { k_read<8><<<g, bl>>>(x, n4, sink); });
      snprintf(nm, 96, "readchunk u8 bl%d g%d", bl, g); time(nm, [&] { k_read_chunk<8><<<g, bl>>>(x, n4, sink); });
      snprintf(nm, 96, "write bl%d g%d", bl, g); time(nm, [&] { k_write<1><<<g, bl>>>(y, n4); });
    }
    for (int g : {148 * 4, 148 * 8, 148 * 16}) {
      snprintf(nm, 96, "copy(40+40) bl256 g%d", g); time(nm, [&] { k_copy<<<g, 256>>>(x, y, n4); });
    }
    cudaFree(x); cudaFree(y);
  }
  return 0;
}
