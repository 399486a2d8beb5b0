// ds_peer.cuh — the multi-GPU exchange step as device code over peer
// memory: every rank's universe slice s of its local histogram goes to rank s's receive
// buffer, slot of the source rank (P2P stores over NVLink / NVSwitch; the smem-path merge
// writes them directly, store_H in ds_scan.cuh), then the owner sums its G slots.  This is
// the reduce-scatter of the local histograms (lem:crn lifted to whole histograms, P:951-962;
// the WSE-3 "tile k owns H[k]" idea, with GPUs as owners).
#pragma once
#include "ds_common.cuh"

namespace ds {

// L2 path (U > kSmem16MaxBins): the local histogram H (U bins, on this GPU) pushed slice by
// slice into the owners' slots: peer[s][rank * L + j] = H[s * L + j].  16-byte copies when L
// allows (L % 4 == 0 and 16-byte aligned buffers: the caller's), else 4-byte ones.
__global__ void k_push_slices(const uint32_t* __restrict__ H, uint32_t U, uint32_t L, uint32_t rank,
                              uint32_t* const* __restrict__ peer) {
  pdl_wait();
  const uint32_t G = U / L;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  if ((L & 3u) == 0) {
    const uint32_t L4 = L / 4;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (uint64_t)G * L4; i += stride) {
      const uint32_t s = (uint32_t)(i / L4), j = (uint32_t)(i - (uint64_t)s * L4);
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(H) + i);
      reinterpret_cast<uint4*>(peer[s] + (uint64_t)rank * L)[j] = v;
    }
  } else {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < U; i += stride) {
      const uint32_t s = (uint32_t)(i / L), j = (uint32_t)(i - (uint64_t)s * L);
      peer[s][(uint64_t)rank * L + j] = __ldcg(H + i);
    }
  }
  pdl_trigger();
}

}  // namespace ds
