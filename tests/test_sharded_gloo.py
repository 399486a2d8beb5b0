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
        q.put((rank, r.valid().numpy().copy(), int(r.count.item()), r.offset(), r.all_counts.numpy().copy(),
               Hs.numpy().copy(), r.slice_lo))
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
    for rank, out, cnt, o, allc, Hs, slo in res:
        assert slo == rank * S
        assert o == off and cnt == out.size
        assert allc.tolist() == [r[2] for r in res]
        assert np.array_equal(Hs.view(np.uint32).astype(np.uint64), Href[rank * S:(rank + 1) * S])
        off += cnt
        pieces.append(out)
    assert np.array_equal(np.concatenate(pieces), ref)


class OracleP2POps(OracleOps):
    """Peer-memory exchange stood in for on CPU: each rank's receive buffer is a shared-memory
    file that the other rank processes map (the CUDA IPC mapping of the device path); the
    histogram's slices are stored straight into the owners' slots, as the device kernel does."""

    def __init__(self, tag):
        self.tag = tag

    def alloc_recv(self, size, device):
        path = f"/dev/shm/dialsort_p2p_{self.tag}_{dist.get_rank()}"
        with open(path, "wb") as f:
            f.write(b"\0" * (4 * size))
        return torch.from_file(path, shared=True, size=size, dtype=torch.int32), (path, size)

    def open(self, handle):
        path, size = handle
        return torch.from_file(path, shared=True, size=size, dtype=torch.int32)

    def close(self, remote):
        pass

    def peer_table(self, recv, remote, g, off, length):
        return [(recv if r is None else r)[off:off + length] for r in remote]

    def histogram_scatter(self, keys, U, G, g, peers):
        L = U // G
        H = self.histogram(keys, U)
        for s in range(G):
            peers[s][g * L:(g + 1) * L] = H[s * L:(s + 1) * L]

    def barrier(self, group):
        dist.barrier(group=group)

    def slice_sum(self, recv, G, L):
        h = recv.numpy().view(np.uint32).reshape(G, L).astype(np.uint64).sum(axis=0)
        return torch.from_numpy(h.astype(np.uint32).view(np.int32).copy())


def _worker_p2p(rank, world, port, n, U, dist_name, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2605_16667_b200.sharded import PeerExchange, sharded_sort_p2p
        full = synth.make(dist_name, n, U, seed=19)
        lo, hi = rank * n // world, (rank + 1) * n // world
        keys = torch.from_numpy(full[lo:hi].copy())
        ex = PeerExchange(U, torch.device("cpu"), ops=OracleP2POps(port))
        outs = []
        for _ in range(3):  # the exchange buffers (two parities) are reused across calls
            r = sharded_sort_p2p(keys, ex, capacity=n)
            outs.append((r.valid().numpy().copy(), int(r.count.item()), r.offset(), r.slice_lo))
        ex.close()
        dist.barrier()
        os.unlink(f"/dev/shm/dialsort_p2p_{port}_{rank}")
        q.put((rank, outs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dist_name", [(2, "uniform"), (4, "zipf")])
def test_sharded_p2p_orchestration_gloo(world, dist_name):
    """sharded_sort_p2p (local histogram stored slice by slice into the owners' receive slots,
    barrier, slot sums, slice projection) equals the oracle sort, three calls on the same
    double-buffered slots."""
    import oracle
    import synth
    n, U = 150_001, 4096
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_p2p, args=(r, world, port, n, U, dist_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = oracle.sort(synth.make(dist_name, n, U, seed=19), U)
    S = U // world
    for call in range(3):
        off, pieces = 0, []
        for rank, outs in res:
            out, cnt, o, slo = outs[call]
            assert slo == rank * S and o == off and cnt == out.size
            off += cnt
            pieces.append(out)
        assert np.array_equal(np.concatenate(pieces), ref)
