"""Multi-GPU DialSort: key shards -> local H -> reduce-scatter -> per-slice projection.

One process per GPU (torchrun).  Rank g holds the contiguous key shard it was given
(thm:par proof, "Distribute the n keys across k ingestion lanes"), builds its
local histogram with the C ABI, and an NCCL reduce-scatter over NVLink/NVSwitch sums the
local histograms cell-wise (lem:crn lifted to whole histograms) and hands rank g
the universe slice [g*U/G, (g+1)*U/G) — the WSE-3 "tile k owns H[k]" idea
with GPUs as owners.  Each rank then projects its slice with key_base = g*U/G; the
rank-ordered concatenation is the globally sorted array (reading R10 in DESIGN.md).

torch.distributed is plumbing here (the collectives); histogram, slice totals and the
projection run in libdialsort's kernels.  `ops` lets the CPU tests (gloo, world size 2)
drive exactly this orchestration with the oracle standing in for the device steps.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class ShardedResult:
    out: torch.Tensor          # int32[capacity]; the first `count` entries are valid
    count: torch.Tensor        # int64[1] (device): keys of this rank's universe slice
    offset_t: torch.Tensor     # int64[1] (device): global position of this rank's first key
    slice_lo: int              # first key of this rank's slice (radix path: 0, ranges are data-driven)
    slice_len: int             # U / G (0 on the radix path)

    def offset(self) -> int:
        """Global output offset of this rank's keys (host read; not on the hot path)."""
        return int(self.offset_t.item())

    def valid(self) -> torch.Tensor:
        return self.out[: int(self.count.item())]


class _DeviceOps:
    """Device steps of the NCCL baseline through the C ABI."""

    def __init__(self, ctx):
        self.ctx = ctx

    def histogram(self, keys: torch.Tensor, U: int) -> torch.Tensor:
        return self.ctx.histogram(keys, U)

    def reconstruct(self, H_slice: torch.Tensor, key_base: int, out: torch.Tensor, d_total: torch.Tensor):
        self.ctx.reconstruct(H_slice, out, key_base=key_base, exact=False, d_total=d_total)


def _reduce_scatter_sum(H_local: torch.Tensor, S: int, group) -> torch.Tensor:
    G = dist.get_world_size(group)
    g = dist.get_rank(group)
    if dist.get_backend(group) == "gloo":  # gloo has no reduce_scatter: all-reduce + own slice
        H = H_local.clone()
        dist.all_reduce(H, op=dist.ReduceOp.SUM, group=group)
        return H[g * S:(g + 1) * S].contiguous()
    H_slice = torch.empty(S, dtype=H_local.dtype, device=H_local.device)
    dist.reduce_scatter_tensor(H_slice, H_local, op=dist.ReduceOp.SUM, group=group)
    return H_slice


def sharded_sort(keys_local: torch.Tensor, U: int, capacity: int, group=None, ctx=None, ops=None,
                 out: torch.Tensor | None = None) -> ShardedResult:
    """NCCL baseline: sort the union of all ranks' key shards; rank g receives universe slice g.

    capacity: room (keys) of this rank's output.  A slice with more keys than `capacity`
    raises DIALSORT_E_SIZE at the next sync (its first `capacity` keys are written).
    Histogram counts are uint32 carried in int32 tensors (two's-complement sums are
    bit-identical to uint32 sums).
    """
    G = dist.get_world_size(group)
    g = dist.get_rank(group)
    if U % G != 0:
        raise ValueError(f"U={U} must be divisible by the world size {G} (reading R10)")
    S = U // G
    if ops is None:
        if ctx is None:
            from . import default_context
            ctx = default_context(keys_local.device)
        ops = _DeviceOps(ctx)
    dev = keys_local.device
    H_local = ops.histogram(keys_local, U)                     # local H over the full universe
    H_slice = _reduce_scatter_sum(H_local, S, group)           # Σ_ranks H_local[slice g]
    if out is None:
        out = torch.empty(int(capacity), dtype=torch.int32, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    ops.reconstruct(H_slice, g * S, out, count)                # project slice g, key_base g*S
    all_counts = torch.empty(G, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(all_counts, count, group=group)  # slice totals -> offsets
    offset = all_counts[:g].sum().reshape(1)
    return ShardedResult(out=out, count=count, offset_t=offset, slice_lo=g * S, slice_len=S)


def sharded_histogram(keys_local: torch.Tensor, U: int, group=None, ctx=None, ops=None) -> torch.Tensor:
    """Rank g's slice of the global histogram (the canonical state), H[gS:(g+1)S)."""
    G = dist.get_world_size(group)
    if U % G != 0:
        raise ValueError(f"U={U} must be divisible by the world size {G}")
    if ops is None:
        if ctx is None:
            from . import default_context
            ctx = default_context(keys_local.device)
        ops = _DeviceOps(ctx)
    return _reduce_scatter_sum(ops.histogram(keys_local, U), U // G, group)


def connect_comms(comm, group=None) -> None:
    """One-time bootstrap of a communicator over torch.distributed: every rank's handle bytes,
    all-gathered in rank order, then opened (CUDA IPC) by every rank."""
    G = dist.get_world_size(group)
    handles = [None] * G
    dist.all_gather_object(handles, comm.handle, group=group)
    comm.connect_ipc(handles)


class PeerComm:
    """This rank's communicator (dialsort_comm) for U <= max_U and up to max_recv_keys radix keys."""

    def __init__(self, max_U: int, device, group=None, ctx=None, max_recv_keys: int = 0, comm_factory=None):
        from . import Comm, default_context
        self.G = dist.get_world_size(group)
        self.g = dist.get_rank(group)
        self.group = group
        self.ctx = ctx if ctx is not None else default_context(device)
        make = comm_factory if comm_factory is not None else Comm
        self.comm = make(self.ctx, self.G, self.g, int(max_U), int(max_recv_keys))
        connect_comms(self.comm, group)

    def close(self) -> None:
        self.comm.close()


def sharded_sort_p2p(keys_local: torch.Tensor, pc: PeerComm, U: int, capacity: int,
                     out: torch.Tensor | None = None) -> ShardedResult:
    """Sharded DialSort with the exchange over peer memory (dialsort_sharded_sort_async): one
    histogram kernel stores each merged bin of slice s into rank s's slot, rank g sums its slots
    and projects slice g with key_base g U/G; count and offset stay on the device."""
    if U % pc.G != 0:
        raise ValueError(f"U={U} must be divisible by the world size {pc.G} (reading R10)")
    dev = keys_local.device
    if out is None:
        out = torch.empty(int(capacity), dtype=torch.int32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    pc.comm.sort(keys_local, U, out, cnt[0:1], cnt[1:2])
    L = U // pc.G
    return ShardedResult(out=out, count=cnt[0:1], offset_t=cnt[1:2], slice_lo=pc.g * L, slice_len=L)


def sharded_sort_int32(keys_local: torch.Tensor, pc: PeerComm, capacity: int,
                       out: torch.Tensor | None = None) -> ShardedResult:
    """Sharded DialSort-Radix (dialsort_sharded_sort_int32_async): rank g ends with the sorted keys
    of its contiguous top-byte range; the rank-order concatenation is the sorted array."""
    dev = keys_local.device
    if out is None:
        out = torch.empty(int(capacity), dtype=torch.int32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    pc.comm.sort_int32(keys_local, out, cnt[0:1], cnt[1:2])
    return ShardedResult(out=out, count=cnt[0:1], offset_t=cnt[1:2], slice_lo=0, slice_len=0)
