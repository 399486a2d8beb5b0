// Design microbenchmarks for the histogram path (not product code, not timed by bench.py).
// Measures on B200: streaming read/write bandwidth at the c2 size, shared-memory atomic
// throughput (u32 / u16-packed), L2 RED throughput for U=65536 and U=2^20, 2- and 8-CTA
// cluster DSMEM atomics, and the cost of the __match_any_sync warp CRN.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// dist 0 uniform, 1 zipf-like (20% hot key, geometric-ish tail), 2 sorted
__global__ void k_gen(int32_t* k, uint64_t n, uint32_t U, int dist) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = mix64(20260321ULL + (i + 1) * 0x9E3779B97F4A7C15ULL);
    uint32_t u = (uint32_t)(((z >> 32) * (uint64_t)U) >> 32);
    if (dist == 1) {
      double x = (double)(z & 0xFFFFFFFFu) / 4294967296.0;
      if (x < 0.2) u = 12345 % U;
      else { double r = pow(x, 6.0); u = (uint32_t)(r * U) * 2654435761u % U; }
    } else if (dist == 2) {
      u = (uint32_t)((i * (uint64_t)U) / n);
    }
    k[i] = (int32_t)u;
  }
}

__global__ void k_read(const int4* __restrict__ p, uint64_t n4, int* sink) {
  int acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x7fffffff) *sink = acc;
}
__global__ void k_write(int4* __restrict__ p, uint64_t n4) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = make_int4((int)i, (int)i, (int)i, (int)i);
}
__global__ void k_flush(int4* p, uint64_t n4) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = make_int4(1, 2, 3, (int)i);
}

template <bool CRN>
__device__ __forceinline__ void add_smem(uint32_t* h, uint32_t k) {
  if (CRN) {
    unsigned m = __match_any_sync(__activemask(), k);
    int leader = __ffs(m) - 1;
    if ((threadIdx.x & 31) == leader) atomicAdd(h + k, (uint32_t)__popc(m));
  } else {
    atomicAdd(h + k, 1u);
  }
}

// smem u32 histogram over U bins (U*4 <= smem), with R replicas (per-warp groups)
template <bool CRN, int R>
__global__ void k_hist_smem(const int4* __restrict__ keys, uint64_t n4, uint32_t U, uint32_t* H) {
  extern __shared__ uint32_t sh[];
  int rep = (threadIdx.x >> 5) % R;
  for (uint32_t i = threadIdx.x; i < U * R; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t* h = sh + rep * U;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(keys + i);
    add_smem<CRN>(h, v.x); add_smem<CRN>(h, v.y); add_smem<CRN>(h, v.z); add_smem<CRN>(h, v.w);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < U; b += blockDim.x) {
    uint32_t s = 0;
    for (int r = 0; r < R; ++r) s += sh[r * U + b];
    if (s) atomicAdd(H + b, s);
  }
}

// u16-packed smem: word j holds bins j and j+U/2 (throughput only, overflow ignored)
template <bool CRN>
__global__ void k_hist_smem16(const int4* __restrict__ keys, uint64_t n4, uint32_t U, uint32_t* H) {
  extern __shared__ uint32_t sh[];
  uint32_t half = U / 2;
  for (uint32_t i = threadIdx.x; i < half; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(keys + i);
    uint32_t kk[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t k = kk[j];
      uint32_t w = k >= half ? k - half : k;
      uint32_t inc = k >= half ? 65536u : 1u;
      if (CRN) {
        unsigned m = __match_any_sync(0xffffffffu, k);
        if ((threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(sh + w, inc * __popc(m));
      } else atomicAdd(sh + w, inc);
    }
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < half; b += blockDim.x) {
    uint32_t s = sh[b];
    if (s & 0xffff) atomicAdd(H + b, s & 0xffff);
    if (s >> 16) atomicAdd(H + b + half, s >> 16);
  }
}

template <bool CRN>
__global__ void k_hist_global(const int4* __restrict__ keys, uint64_t n4, uint32_t* H) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(keys + i);
    uint32_t kk[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (CRN) {
        unsigned m = __match_any_sync(0xffffffffu, kk[j]);
        if ((threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(H + kk[j], (uint32_t)__popc(m));
      } else atomicAdd(H + kk[j], 1u);
    }
  }
}

// cluster DSMEM: C CTAs per cluster, CTA r owns bins [r*U/C, (r+1)*U/C)
template <int C, bool CRN>
__global__ void k_hist_cluster(const int4* __restrict__ keys, uint64_t n4, uint32_t U, uint32_t* H) {
  extern __shared__ uint32_t sh[];
  cg::cluster_group cl = cg::this_cluster();
  uint32_t per = U / C;
  for (uint32_t i = threadIdx.x; i < per; i += blockDim.x) sh[i] = 0;
  cl.sync();
  uint32_t* remote[C];
#pragma unroll
  for (int r = 0; r < C; ++r) remote[r] = cl.map_shared_rank(sh, r);
  uint32_t shift = __ffs(per) - 1;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(keys + i);
    uint32_t kk[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t k = kk[j];
      uint32_t own = k >> shift, off = k & (per - 1);
      uint32_t* base = sh;
#pragma unroll
      for (int r = 0; r < C; ++r) if (own == (uint32_t)r) base = remote[r];
      if (CRN) {
        unsigned m = __match_any_sync(0xffffffffu, k);
        if ((threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(base + off, (uint32_t)__popc(m));
      } else atomicAdd(base + off, 1u);
    }
  }
  cl.sync();
  uint32_t rank = cl.block_rank();
  for (uint32_t b = threadIdx.x; b < per; b += blockDim.x) { uint32_t s = sh[b]; if (s) atomicAdd(H + rank * per + b, s); }
}

struct Timer {
  cudaEvent_t a, b;
  Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); }
  float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
};

int4* g_flush; uint64_t g_flush4;
void flush_l2() { k_flush<<<148 * 4, 512>>>(g_flush, g_flush4); }

template <typename F>
float best_of(F f, int reps = 7) {
  Timer t; float best = 1e30f;
  for (int w = 0; w < 3; ++w) { flush_l2(); f(); }
  CK(cudaDeviceSynchronize());
  for (int r = 0; r < reps; ++r) { flush_l2(); t.start(); f(); float ms = t.stop(); best = std::min(best, ms); }
  CK(cudaGetLastError());
  return best;
}

bool check(const uint32_t* dH, uint32_t U, uint64_t n, const char* name) {
  std::vector<uint32_t> h(U); CK(cudaMemcpy(h.data(), dH, U * 4, cudaMemcpyDeviceToHost));
  uint64_t s = 0; for (auto x : h) s += x;
  if (s != n) { printf("  [%s] SUM MISMATCH %llu vs %llu\n", name, (unsigned long long)s, (unsigned long long)n); return false; }
  return true;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d L2 %d MB smemOptin %zu\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin);
  int nsm = p.multiProcessorCount;
  g_flush4 = (512ull << 20) / 16; CK(cudaMalloc(&g_flush, g_flush4 * 16));
  const uint64_t n = 10000000; const uint64_t n4 = n / 4;
  int32_t* keys; CK(cudaMalloc(&keys, n * 4));
  int32_t* out; CK(cudaMalloc(&out, n * 4));
  uint32_t* H; CK(cudaMalloc(&H, (1u << 20) * 4));
  int* sink; CK(cudaMalloc(&sink, 4));
  double GB = 1e9;

  // bandwidth
  for (int bl : {256, 512, 1024}) for (int occ : {1, 2, 4, 8}) {
    int grid = nsm * occ * (1024 / bl > 0 ? 1 : 1);
    float ms = best_of([&] { k_read<<<grid, bl>>>((const int4*)keys, n4, sink); });
    float ms2 = best_of([&] { k_write<<<grid, bl>>>((int4*)out, n4); });
    printf("read40MB bl=%d grid=%d: %.2f us %.0f GB/s | write40MB %.2f us %.0f GB/s\n", bl, grid, ms * 1e3, n * 4 / (ms * 1e-3) / GB, ms2 * 1e3, n * 4 / (ms2 * 1e-3) / GB);
  }
  {
    float ms = best_of([&] { cudaMemsetAsync(H, 0, 65536 * 4); });
    printf("memset 256KB: %.2f us\n", ms * 1e3);
    Timer t; t.start(); for (int i = 0; i < 100; ++i) k_write<<<1, 32>>>((int4*)out, 1); float ms2 = t.stop();
    printf("empty-ish launch x100: %.2f us each\n", ms2 * 10);
  }

  const char* dn[3] = {"uniform", "zipfish", "sorted"};
  for (int dist = 0; dist < 3; ++dist) {
    for (uint32_t U : {256u, 65536u, 1u << 20}) {
      k_gen<<<nsm * 8, 256>>>(keys, n, U, dist); CK(cudaDeviceSynchronize());
      auto run = [&](const char* name, auto launch) {
        float ms = best_of([&] { cudaMemsetAsync(H, 0, U * 4); launch(); });
        CK(cudaMemsetAsync(H, 0, U * 4)); launch(); CK(cudaDeviceSynchronize());
        bool ok = check(H, U, n, name);
        printf("%-8s U=%-8u %-34s %8.2f us  %7.1f Gkeys/s  %s\n", dn[dist], U, name, ms * 1e3, n / (ms * 1e-3) / 1e9, ok ? "" : "BAD");
      };
      if (U == 256) {
        for (int bl : {256, 512, 1024}) for (int occ : {1, 2, 4}) {
          int grid = nsm * occ;
          char nm[64];
          snprintf(nm, 64, "smem R1 noCRN bl%d occ%d", bl, occ);
          run(nm, [&] { k_hist_smem<false, 1><<<grid, bl, U * 4>>>((const int4*)keys, n4, U, H); });
          snprintf(nm, 64, "smem R8 noCRN bl%d occ%d", bl, occ);
          run(nm, [&] { k_hist_smem<false, 8><<<grid, bl, U * 4 * 8>>>((const int4*)keys, n4, U, H); });
          snprintf(nm, 64, "smem R1 CRN bl%d occ%d", bl, occ);
          run(nm, [&] { k_hist_smem<true, 1><<<grid, bl, U * 4>>>((const int4*)keys, n4, U, H); });
          snprintf(nm, 64, "smem R8 CRN bl%d occ%d", bl, occ);
          run(nm, [&] { k_hist_smem<true, 8><<<grid, bl, U * 4 * 8>>>((const int4*)keys, n4, U, H); });
        }
      }
      if (U == 65536) {
        CK(cudaFuncSetAttribute(k_hist_smem16<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 * 2));
        CK(cudaFuncSetAttribute(k_hist_smem16<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 * 2));
        CK(cudaFuncSetAttribute(k_hist_cluster<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 * 2));
        CK(cudaFuncSetAttribute(k_hist_cluster<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 * 2));
        CK(cudaFuncSetAttribute(k_hist_cluster<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 / 2));
        CK(cudaFuncSetAttribute(k_hist_cluster<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 / 2));
        for (int bl : {512, 1024}) {
          char nm[64];
          snprintf(nm, 64, "smem16 noCRN bl%d", bl);
          run(nm, [&] { k_hist_smem16<false><<<nsm, bl, 65536 * 2>>>((const int4*)keys, n4, U, H); });
          snprintf(nm, 64, "smem16 CRN bl%d", bl);
          run(nm, [&] { k_hist_smem16<true><<<nsm, bl, 65536 * 2>>>((const int4*)keys, n4, U, H); });
          auto launch_cl = [&](auto kern, int C, size_t smem) {
            cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(nsm / C * C); cfg.blockDim = dim3(bl); cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            cudaError_t e = cudaLaunchKernelEx(&cfg, kern, (const int4*)keys, n4, U, H);
            if (e != cudaSuccess) printf("cluster launch err %s\n", cudaGetErrorString(e));
          };
          snprintf(nm, 64, "cluster2 noCRN bl%d", bl);
          run(nm, [&] { launch_cl(k_hist_cluster<2, false>, 2, 65536 * 2); });
          snprintf(nm, 64, "cluster2 CRN bl%d", bl);
          run(nm, [&] { launch_cl(k_hist_cluster<2, true>, 2, 65536 * 2); });
          snprintf(nm, 64, "cluster8 noCRN bl%d", bl);
          run(nm, [&] { launch_cl(k_hist_cluster<8, false>, 8, 65536 / 2); });
          snprintf(nm, 64, "cluster8 CRN bl%d", bl);
          run(nm, [&] { launch_cl(k_hist_cluster<8, true>, 8, 65536 / 2); });
        }
      }
      for (int occ : {2, 8}) {
        char nm[64];
        snprintf(nm, 64, "global noCRN occ%d", occ);
        run(nm, [&] { k_hist_global<false><<<nsm * occ, 256>>>((const int4*)keys, n4, H); });
        snprintf(nm, 64, "global CRN occ%d", occ);
        run(nm, [&] { k_hist_global<true><<<nsm * occ, 256>>>((const int4*)keys, n4, H); });
      }
    }
  }
  printf("done\n");
  return 0;
}
