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
    all_counts: torch.Tensor   # int64[G] (device): every rank's slice count (rank order)
    slice_lo: int              # first key of this rank's slice
    slice_len: int             # U / G

    def offset(self) -> int:
        """Global output offset of this rank's slice (host read; not on the hot path)."""
        g = self.slice_lo // self.slice_len if self.slice_len else 0
        return int(self.all_counts[:g].sum().item())

    def valid(self) -> torch.Tensor:
        return self.out[: int(self.count.item())]


class _DeviceOps:
    """Device steps through the C ABI (the product path)."""

    def __init__(self, ctx):
        self.ctx = ctx

    def histogram(self, keys: torch.Tensor, U: int) -> torch.Tensor:
        return self.ctx.histogram(keys, U)

    def reconstruct(self, H_slice: torch.Tensor, key_base: int, out: torch.Tensor, d_total: torch.Tensor):
        self.ctx.reconstruct(H_slice, out, key_base=key_base, exact=False, d_total=d_total)

    # peer-memory exchange (PeerExchange / sharded_sort_p2p)
    def alloc_recv(self, size: int, device):
        t = torch.empty(size, dtype=torch.int32, device=device)
        return t, self.ctx.ipc_handle(t)

    def open(self, handle):
        return self.ctx.ipc_open(handle)

    def close(self, remote):
        self.ctx.ipc_close(remote)

    def peer_table(self, recv: torch.Tensor, remote: list, g: int, off: int, length: int):
        ptrs = [(recv.data_ptr() if r is None else r) + 4 * off for r in remote]
        return torch.tensor(ptrs, dtype=torch.int64, device=recv.device)

    def histogram_scatter(self, keys: torch.Tensor, U: int, G: int, g: int, peers) -> None:
        self.ctx.histogram_scatter(keys, U, G, g, peers)

    def barrier(self, group) -> None:
        torch.cuda.current_stream(self.ctx.device).synchronize()  # this rank's P2P stores landed
        dist.barrier(group=group)                                  # ... and every other rank's

    def slice_sum(self, recv: torch.Tensor, G: int, L: int) -> torch.Tensor:
        return self.ctx.slice_sum(recv, G, L)


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
    """Sort the union of all ranks' key shards; rank g receives universe slice g.

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
    return ShardedResult(out=out, count=count, all_counts=all_counts, slice_lo=g * S, slice_len=S)


class PeerExchange:
    """Receive buffers of the peer-memory exchange: rank g holds G slots of its universe slice
    (one per source rank, uint32[G * L]), mapped into every rank with CUDA IPC once and reused
    across calls.  Two parities alternate between calls: a rank one call ahead writes the other
    parity while its peers still read this one (the per-call barrier bounds the lead to one)."""

    def __init__(self, U: int, device, group=None, ctx=None, ops=None):
        self.G = dist.get_world_size(group)
        self.g = dist.get_rank(group)
        if U % self.G != 0:
            raise ValueError(f"U={U} must be divisible by the world size {self.G} (reading R10)")
        self.U, self.L, self.group = U, U // self.G, group
        if ops is None:
            if ctx is None:
                from . import default_context
                ctx = default_context(device)
            ops = _DeviceOps(ctx)
        self.ops = ops
        GL = self.G * self.L
        self.recv_all, handle = ops.alloc_recv(2 * GL, device)
        handles = [None] * self.G
        dist.all_gather_object(handles, handle, group=group)
        self.remote = [None if s == self.g else ops.open(handles[s]) for s in range(self.G)]
        self.recv = [self.recv_all[p * GL:(p + 1) * GL] for p in range(2)]
        self.peers = [ops.peer_table(self.recv_all, self.remote, self.g, p * GL, GL) for p in range(2)]
        self.calls = 0

    def close(self) -> None:
        for r in self.remote:
            if r is not None:
                self.ops.close(r)
        self.remote = []


def sharded_sort_p2p(keys_local: torch.Tensor, ex: PeerExchange, capacity: int,
                     out: torch.Tensor | None = None) -> ShardedResult:
    """sharded_sort with the exchange over peer memory instead of an NCCL reduce-scatter: one
    kernel builds the local histogram and stores each finished bin of universe slice s straight
    into rank s's slot for this rank (NVLink / NVSwitch P2P stores, dialsort_histogram_scatter_async);
    after every rank's kernel completed (stream sync + barrier), rank g sums its G slots and
    projects its slice with key_base g L."""
    G, g, L, ops = ex.G, ex.g, ex.L, ex.ops
    dev = keys_local.device
    par = ex.calls & 1
    ex.calls += 1
    ops.histogram_scatter(keys_local, ex.U, G, g, ex.peers[par])
    ops.barrier(ex.group)
    H_slice = ops.slice_sum(ex.recv[par], G, L)
    if out is None:
        out = torch.empty(int(capacity), dtype=torch.int32, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    ops.reconstruct(H_slice, g * L, out, count)
    all_counts = torch.empty(G, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(all_counts, count, group=ex.group)
    return ShardedResult(out=out, count=count, all_counts=all_counts, slice_lo=g * L, slice_len=L)


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
