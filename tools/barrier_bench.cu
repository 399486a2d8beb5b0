// Grid-barrier variants for a co-resident grid of 148 x 1024-thread CTAs (design
// microbenchmark, not product code).  Each kernel runs `iters` barriers back to back;
// reported: time per barrier.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/barrier_bench tools/barrier_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned long long ld_acq64(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}

// A: counter + generation (product barrier of round 1)
struct Bar { unsigned count, gen; };
__device__ void barA(Bar* gb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acq(&gb->gen);
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(&gb->count) : "memory");
    if (old == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(&gb->count) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&gb->gen) : "memory");
    } else {
      while (ld_acq(&gb->gen) == g) {}
    }
  }
  __syncthreads();
}
// D: monotonic 64-bit counter, arrive = one atomic, wait on the counter itself
__device__ void barD(unsigned long long* cnt) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long old;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(cnt) : "memory");
    const unsigned long long target = old - old % gridDim.x + gridDim.x;
    while (ld_acq64(cnt) < target) {}
  }
  __syncthreads();
}
// D2: same, red arrive then poll (no returned value: the target is tracked by the caller)
__device__ void barD2(unsigned long long* cnt, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(cnt) : "memory");
    while (ld_acq64(cnt) < target) {}
  }
  __syncthreads();
}
// E: per-CTA flags (epoch values), every CTA polls all flags with G threads
__device__ void barE(unsigned* flags, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(epoch) : "memory");
  if (threadIdx.x < 32) {
    for (;;) {
      bool ok = true;
      for (unsigned i = threadIdx.x; i < gridDim.x; i += 32) ok &= (int)(ld_rlx(flags + i) - epoch) >= 0;
      if (__all_sync(0xffffffffu, ok)) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
// F: S spread counters (separate 256-B lines), red.release arrive on counter b % S; waiters sum
template <int S>
__device__ void barF(unsigned* ctrs, unsigned target_total) {
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctrs + 64 * (blockIdx.x % S)) : "memory");
  if (threadIdx.x < 32) {
    for (;;) {
      unsigned v = threadIdx.x < S ? ld_rlx(ctrs + 64 * threadIdx.x) : 0u;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((int)(v - target_total) >= 0) break;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024, 1) kA(Bar* b, int it) { for (int i = 0; i < it; ++i) barA(b); }
__global__ void __launch_bounds__(1024, 1) kD(unsigned long long* c, int it) { for (int i = 0; i < it; ++i) barD(c); }
__global__ void __launch_bounds__(1024, 1) kD2(unsigned long long* c, unsigned long long base, int it) {
  for (int i = 0; i < it; ++i) barD2(c, base + (unsigned long long)(i + 1) * gridDim.x);
}
__global__ void __launch_bounds__(1024, 1) kE(unsigned* f, unsigned e0, int it) { for (int i = 0; i < it; ++i) barE(f, e0 + i); }
template <int S>
__global__ void __launch_bounds__(1024, 1) kF(unsigned* c, unsigned base, int it) {
  for (int i = 0; i < it; ++i) barF<S>(c, base + (unsigned)(i + 1) * gridDim.x);
}
__global__ void __launch_bounds__(1024, 1) kNone(int it) { for (int i = 0; i < it; ++i) __syncthreads(); }

int main() {
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  void* mem; CK(cudaMalloc(&mem, 1 << 20)); CK(cudaMemset(mem, 0, 1 << 20));
  char* m = (char*)mem;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int IT = 200;
  auto time = [&](const char* nm, auto&& launch) {
    for (int w = 0; w < 3; ++w) launch(1);
    CK(cudaDeviceSynchronize());
    float best1 = 1e9, bestN = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); launch(1); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float t; cudaEventElapsedTime(&t, e0, e1); if (t < best1) best1 = t;
      cudaEventRecord(e0); launch(IT + 1); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&t, e0, e1); if (t < bestN) bestN = t;
    }
    printf("%-40s per barrier %.3f us   (1-barrier kernel %.2f us)\n", nm, (bestN - best1) * 1000.f / IT, best1 * 1000.f);
  };
  time("none (__syncthreads only)", [&](int it) { kNone<<<nsm, 1024>>>(it); });
  time("A counter+generation", [&](int it) { kA<<<nsm, 1024>>>((Bar*)m, it); });
  CK(cudaMemset(mem, 0, 1 << 20));
  time("D monotonic u64 atom", [&](int it) { kD<<<nsm, 1024>>>((unsigned long long*)(m + 4096), it); });
  {
    CK(cudaMemset(mem, 0, 1 << 20));
    unsigned long long base = 0;
    time("D2 monotonic u64 red + poll", [&](int it) {
      kD2<<<nsm, 1024>>>((unsigned long long*)(m + 8192), base, it); base += (unsigned long long)it * nsm; });
  }
  {
    unsigned ep = 1;
    time("E per-CTA flags, all poll", [&](int it) { kE<<<nsm, 1024>>>((unsigned*)(m + 16384), ep, it); ep += it; });
  }
  {
    CK(cudaMemset(mem, 0, 1 << 20));
    unsigned base = 0;
    time("F 4 spread counters", [&](int it) { kF<4><<<nsm, 1024>>>((unsigned*)(m + 65536), base, it); base += it * nsm; });
  }
  {
    CK(cudaMemset(mem, 0, 1 << 20));
    unsigned base = 0;
    time("F 16 spread counters", [&](int it) { kF<16><<<nsm, 1024>>>((unsigned*)(m + 131072), base, it); base += it * nsm; });
  }
  {
    CK(cudaMemset(mem, 0, 1 << 20));
    unsigned base = 0;
    time("F 32 spread counters", [&](int it) { kF<32><<<nsm, 1024>>>((unsigned*)(m + 262144), base, it); base += it * nsm; });
  }
  return 0;
}
