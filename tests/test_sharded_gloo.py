"""Multi-rank host logic of the sharded path on CPU (gloo, world size 2 and 4).

The orchestration in paper_2605_16667_b200/sharded.py (shard -> local H -> reduce-scatter
-> slice projection with key_base -> all-gathered slice totals) runs unchanged; only the
device steps are stood in for by the oracle (`ops`), since there is no GPU here.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleOps:
    def histogram(self, keys, U):
        import oracle
        H = oracle.histogram(keys.numpy(), U).astype(np.uint32).view(np.int32)
        return torch.from_numpy(H.copy())

    def reconstruct(self, H_slice, key_base, out, d_total):
        import oracle
        h = H_slice.numpy().view(np.uint32).astype(np.uint64)
        tot = int(h.sum())
        d_total[0] = tot
        o = oracle.project(h, key_base=key_base)
        m = min(tot, out.numel())
        out[:m] = torch.from_numpy(o[:m])


def _worker(rank, world, port, n, U, dist_name, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2605_16667_b200.sharded import sharded_sort, sharded_histogram
        full = synth.make(dist_name, n, U, seed=17)
        lo, hi = rank * n // world, (rank + 1) * n // world
        keys = torch.from_numpy(full[lo:hi].copy())
        r = sharded_sort(keys, U, capacity=n, ops=OracleOps())
        Hs = sharded_histogram(keys, U, ops=OracleOps())
        q.put((rank, r.valid().numpy().copy(), int(r.count.item()), r.offset(), Hs.numpy().copy(), r.slice_lo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dist_name", [(2, "uniform"), (2, "zipf"), (4, "sorted")])
def test_sharded_orchestration_gloo(world, dist_name):
    import oracle
    import synth
    n, U = 200_003, 4096
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, U, dist_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = synth.make(dist_name, n, U, seed=17)
    ref = oracle.sort(full, U)
    Href = oracle.histogram(full, U)
    S = U // world
    pieces = []
    off = 0
    for rank, out, cnt, o, Hs, slo in res:
        assert slo == rank * S
        assert o == off and cnt == out.size
        assert np.array_equal(Hs.view(np.uint32).astype(np.uint64), Href[rank * S:(rank + 1) * S])
        off += cnt
        pieces.append(out)
    assert np.array_equal(np.concatenate(pieces), ref)


class FakeComm:
    """Stands in for paper_2605_16667_b200.Comm on CPU: records what the bootstrap hands it."""

    def __init__(self, ctx, G, rank, max_U, max_recv_keys):
        self.G, self.rank, self.max_U, self.max_recv = G, rank, max_U, max_recv_keys
        self.handle = bytes([rank]) * 128
        self.connected = None

    def connect_ipc(self, handles):
        self.connected = list(handles)

    def close(self):
        pass


def _worker_bootstrap(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_16667_b200.sharded import PeerComm
        pc = PeerComm(1 << 16, torch.device("cpu"), ctx=object(), max_recv_keys=123, comm_factory=FakeComm)
        q.put((rank, pc.G, pc.g, pc.comm.rank, pc.comm.max_U, pc.comm.max_recv, pc.comm.connected))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_peer_comm_bootstrap_gloo(world):
    """PeerComm's one-time bootstrap: every rank creates its communicator with its own rank and
    connects it with all ranks' handle bytes in rank order (the device path then needs no host
    collective per call)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_bootstrap, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, G, g, crank, maxU, maxr, handles in res:
        assert (G, g, crank, maxU, maxr) == (world, rank, rank, 1 << 16, 123)
        assert handles == [bytes([r]) * 128 for r in range(world)]
