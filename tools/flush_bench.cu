// Flush / merge / grid-barrier costs on B200 for the DialSort sub-histogram merge (design
// microbenchmark, not product code).  148 co-resident CTAs of 1024 threads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/flush_bench tools/flush_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ void red_u32(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}

// each CTA REDs W u32 values into H (skip zero = false)
__global__ void k_red_flush32(uint32_t* H, uint32_t W) {
  for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) red_u32(H + i, 1u + (i & 1));
}
// rotated start so CTAs don't hit the same lines at the same time
__global__ void k_red_flush32_rot(uint32_t* H, uint32_t W) {
  uint32_t off = (blockIdx.x * (W / gridDim.x)) & ~1023u;
  for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) { uint32_t j = (i + off) % W; red_u32(H + j, 1u); }
}
__global__ void k_red_flush64_rot(unsigned long long* H, uint32_t W2) {
  uint32_t off = (blockIdx.x * (W2 / gridDim.x)) & ~1023u;
  for (uint32_t i = threadIdx.x; i < W2; i += blockDim.x) { uint32_t j = (i + off) % W2; red_u64(H + j, 0x100000001ull); }
}
__global__ void k_row_write(uint4* rows, uint32_t W4) {
  uint4* r = rows + (uint64_t)blockIdx.x * W4;
  for (uint32_t i = threadIdx.x; i < W4; i += blockDim.x) __stcg(r + i, make_uint4(i, 1, 2, 3));
}

// barrier A: counter + generation
struct Bar { unsigned count, gen; };
__global__ void k_barA(Bar* b, int iters, int sleep) {
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned g = ld_acq(&b->gen);
      __threadfence();
      if (atomicAdd(&b->count, 1u) == gridDim.x - 1) { atomicExch(&b->count, 0u); __threadfence(); atomicAdd(&b->gen, 1u); }
      else { while (ld_acq(&b->gen) == g) { if (sleep) __nanosleep(sleep); } }
      __threadfence();
    }
    __syncthreads();
  }
}
// barrier B: per-CTA arrival flags (epoch values), CTA 0 warp polls all, then releases
__global__ void k_barB(unsigned* flags, unsigned* go, int iters, unsigned base) {
  for (int it = 0; it < iters; ++it) {
    const unsigned ep = base + it + 1;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(ep) : "memory");
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
      for (unsigned c = threadIdx.x; c < gridDim.x; c += 32) while (ld_acq(flags + c) < ep) {}
      __syncwarp();
      if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(go), "r"(ep) : "memory");
    }
    if (threadIdx.x == 0) { while (ld_acq(go) < ep) {} __threadfence(); }
    __syncthreads();
  }
}


// barrier C: two-level tree: 16 leaf counters (CTA b -> leaf b % 16), leaf winners bump root
struct TreeBar { unsigned leaf[16][32]; unsigned root; unsigned pad[31]; unsigned gen; };
__global__ void k_barC(TreeBar* t, int iters) {
  const unsigned nleaf = 16;
  const unsigned leaf = blockIdx.x % nleaf;
  const unsigned leaf_size = gridDim.x / nleaf + (leaf < gridDim.x % nleaf ? 1 : 0);
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned g = ld_acq(&t->gen);
      __threadfence();
      if (atomicAdd(&t->leaf[leaf][0], 1u) == leaf_size - 1) {
        atomicExch(&t->leaf[leaf][0], 0u);
        if (atomicAdd(&t->root, 1u) == nleaf - 1) { atomicExch(&t->root, 0u); __threadfence(); atomicAdd(&t->gen, 1u); }
        else while (ld_acq(&t->gen) == g) {}
      } else {
        while (ld_acq(&t->gen) == g) {}
      }
      __threadfence();
    }
    __syncthreads();
  }
}

// DSMEM: cluster of 2; every key goes to the partner CTA's smem with red.shared::cluster
__global__ void __cluster_dims__(2, 1, 1) k_dsmem_red(uint32_t iters, uint32_t W, uint32_t* sink) {
  extern __shared__ uint32_t sh[];
  for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) sh[i] = 0;
  asm volatile("barrier.cluster.arrive; barrier.cluster.wait;" ::: "memory");
  uint32_t rank; asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  uint32_t local = (uint32_t)__cvta_generic_to_shared(sh), remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank ^ 1));
  uint32_t s = blockIdx.x * 7919 + threadIdx.x;
  for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      s = s * 1664525u + 1013904223u;
      uint32_t a = remote + 4 * ((s >> 8) & (W - 1));
      asm volatile("red.shared::cluster.add.u32 [%0], %1;" :: "r"(a), "r"(1u) : "memory");
    }
  }
  asm volatile("barrier.cluster.arrive; barrier.cluster.wait;" ::: "memory");
  if (sh[threadIdx.x] == 0x12345) *sink = 1;
}
__global__ void k_local_red(uint32_t iters, uint32_t W, uint32_t* sink) {
  extern __shared__ uint32_t sh[];
  for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  uint32_t s = blockIdx.x * 7919 + threadIdx.x;
  for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) { s = s * 1664525u + 1013904223u; atomicAdd(sh + ((s >> 8) & (W - 1)), 1u); }
  }
  __syncthreads();
  if (sh[threadIdx.x] == 0x12345) *sink = 1;
}

int main() {
  int nsm = 148;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto time = [&](const char* name, auto f, double div = 1.0) {
    float best = 1e30f;
    for (int r = 0; r < 12; ++r) {
      cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 2) best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    printf("%-48s %9.2f us\n", name, best * 1e3 / div);
  };
  uint32_t* H; CK(cudaMalloc(&H, 1 << 24)); CK(cudaMemset(H, 0, 1 << 24));
  uint4* rows; CK(cudaMalloc(&rows, (size_t)nsm * 128 * 1024));
  time("empty launch", [&] { k_row_write<<<1, 32>>>(rows, 0); });
  time("row write 148 x 128KB", [&] { k_row_write<<<nsm, 1024>>>(rows, 8192); });
  time("RED u32 flush 148 x 65536", [&] { k_red_flush32<<<nsm, 1024>>>(H, 65536); });
  time("RED u32 flush rotated 148 x 65536", [&] { k_red_flush32_rot<<<nsm, 1024>>>(H, 65536); });
  time("RED u64 flush rotated 148 x 32768", [&] { k_red_flush64_rot<<<nsm, 1024>>>((unsigned long long*)H, 32768); });
  time("RED u32 flush rotated 148 x 1M (U=2^20)", [&] { k_red_flush32_rot<<<nsm, 1024>>>(H, 1 << 20); });
  Bar* bar; CK(cudaMalloc(&bar, 64)); CK(cudaMemset(bar, 0, 64));
  unsigned* flags; CK(cudaMalloc(&flags, 4096)); CK(cudaMemset(flags, 0, 4096));
  for (int sl : {0, 32, 128}) {
    char nm[64]; snprintf(nm, 64, "barrier A (sleep %d), per barrier", sl);
    time(nm, [&] { k_barA<<<nsm, 1024>>>(bar, 20, sl); }, 20.0);
  }
  unsigned base = 0;
  TreeBar* tb; CK(cudaMalloc(&tb, sizeof(TreeBar))); CK(cudaMemset(tb, 0, sizeof(TreeBar)));
  time("barrier C (tree 16), per barrier", [&] { k_barC<<<nsm, 1024>>>(tb, 20); }, 20.0);
  CK(cudaFuncSetAttribute(k_dsmem_red, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024));
  CK(cudaFuncSetAttribute(k_local_red, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024));
  {
    uint32_t* sink; CK(cudaMalloc(&sink, 4));
    const uint32_t iters = 200;
    double ops = 148.0 * 1024 * iters * 16;
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(a); k_dsmem_red<<<148, 1024, 128 * 1024>>>(iters, 32768, sink); cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms); }
    CK(cudaGetLastError());
    printf("DSMEM red.shared::cluster remote random: %.1f Gops/s (%.2f /clk/SM)\n", ops / (best * 1e-3) / 1e9, ops / (best * 1e-3) / 148 / 1.965e9);
    best = 1e30f;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(a); k_local_red<<<148, 1024, 128 * 1024>>>(iters, 32768, sink); cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms); }
    printf("local smem atomicAdd random:            %.1f Gops/s (%.2f /clk/SM)\n", ops / (best * 1e-3) / 1e9, ops / (best * 1e-3) / 148 / 1.965e9);
  }
  time("barrier B (flags + go), per barrier", [&] { k_barB<<<nsm, 1024>>>(flags, flags + 1000, 20, base); base += 20; }, 20.0);
  return 0;
}
