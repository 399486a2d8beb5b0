"""Multi-GPU exchange on ONE GPU: G virtual ranks (G contexts + communicators of this process,
connected by pointer: dialsort_comm_connect_local), each step issued for every rank before the
next step (so no rank's kernel ever waits for a kernel that has not been enqueued earlier on the
stream — the ranks never run concurrently).  Every rank's H slice, output, count and global
offset is compared element by element with the oracle's O3 / O4' readings (R10 / R19).

The same device code runs at G > 1 across GPUs; only the mapping of the peer workspaces (CUDA IPC
instead of pointers) differs.  The NCCL baseline's sequence (local histograms, reduce-scatter,
slice projection) is emulated with the reduce-scatter done by torch on the device.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ds(cuda_dev):
    import paper_2605_16667_b200 as m
    return m


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to("cuda:0")


def H64(t):
    return t.cpu().numpy().view(np.uint32).astype(np.uint64)


def make_ranks(ds, G, U, n, max_recv=0):
    ctxs = [ds.Context(0, max_n=n, max_U=U) for _ in range(G)]
    comms = [ds.Comm(ctxs[g], G, g, U, max_recv) for g in range(G)]
    for c in comms:
        c.connect_local(comms)
    return ctxs, comms


def keys_of(dist, n, U, seed):
    if dist == "hot1":
        return synth.hot1(n, U, seed=seed)
    return synth.make(dist, n, U, seed=seed)


# (U = 65536: the fused merge stores into the owners' slots; 2^20 and 300000: hierarchical
#  blocks storing into the slots; 2^23: the L2 path + push kernel)
CASES = [(G, U, d) for G in (2, 4, 8) for U, d in
         [(65536, "uniform"), (65536, "zipf"), (65536, "hot1"), (1 << 20, "uniform"), (1 << 20, "zipf"),
          (1 << 20, "hot1")]] + [(4, 300_000, "uniform"), (2, 1 << 23, "uniform"), (8, 4096, "sorted")]


@pytest.mark.parametrize("G,U,dist", CASES)
def test_loopback_sharded_sort(ds, cuda_dev, G, U, dist):
    n = 1_500_007
    x = keys_of(dist, n, U, seed=G * 7 + U % 97)
    ctxs, comms = make_ranks(ds, G, U, n)
    shards = [to_dev(x[g * n // G:(g + 1) * n // G]) for g in range(G)]
    L = U // G
    ref = [oracle.sharded_rank(x, U, G, g) for g in range(G)]
    for call in range(3):  # both slot parities, then the first again
        outs = [torch.empty(n, dtype=torch.int32, device=cuda_dev) for _ in range(G)]
        cnt = [torch.zeros(2, dtype=torch.int64, device=cuda_dev) for _ in range(G)]
        for g in range(G):
            comms[g].scatter(shards[g], U)
        Hs = [comms[g].gather(U, torch.empty(L, dtype=torch.int32, device=cuda_dev)) for g in range(G)]
        for g in range(G):
            comms[g].project(U, Hs[g], outs[g], cnt[g][0:1], cnt[g][1:2])
        for c in ctxs:
            c.sync()
        for g in range(G):
            Hr, outr, cr, offr = ref[g]
            assert np.array_equal(H64(Hs[g]), Hr), (call, g)
            assert int(cnt[g][0]) == cr and int(cnt[g][1]) == offr, (call, g)
            assert np.array_equal(outs[g][:cr].cpu().numpy(), outr), (call, g)
        assert comms[0].epoch == call + 1
    for c in comms:
        c.close()


@pytest.mark.parametrize("U", [65536, 1 << 20])
def test_fused_call_world_one(ds, cuda_dev, U):
    """dialsort_sharded_sort_async (scatter + gather + project in one call): at G = 1 it can be
    issued as one call on one GPU (at G > 1 a rank's call waits for its peers' calls)."""
    n = 700_001
    ctxs, comms = make_ranks(ds, 1, U, n)
    for call in range(3):
        x = synth.uniform(n + call, U, seed=40 + call)
        out = torch.empty(n + 8, dtype=torch.int32, device=cuda_dev)
        cnt = torch.zeros(2, dtype=torch.int64, device=cuda_dev)
        Hs = torch.empty(U, dtype=torch.int32, device=cuda_dev)
        comms[0].sort(to_dev(x), U, out, cnt[0:1], cnt[1:2], H_slice=Hs)
        ctxs[0].sync()
        assert int(cnt[0]) == x.size and int(cnt[1]) == 0
        assert np.array_equal(H64(Hs), oracle.histogram(x, U))
        assert np.array_equal(out[:x.size].cpu().numpy(), oracle.sort(x, U))


@pytest.mark.parametrize("G,U", [(2, 65536), (8, 1 << 20)])
def test_loopback_capacity(ds, cuda_dev, G, U):
    """A slice larger than its rank's capacity is DIALSORT_E_SIZE on that rank, with the first
    `cap` keys written; the other ranks are unaffected."""
    n = 800_001
    x = synth.zipf(n, U, seed=5)
    ctxs, comms = make_ranks(ds, G, U, n)
    shards = [to_dev(x[g * n // G:(g + 1) * n // G]) for g in range(G)]
    ref = [oracle.sharded_rank(x, U, G, g) for g in range(G)]
    cap = max(r[2] for r in ref) - 1  # the largest slice does not fit
    outs = [torch.empty(cap, dtype=torch.int32, device=cuda_dev) for _ in range(G)]
    cnt = [torch.zeros(2, dtype=torch.int64, device=cuda_dev) for _ in range(G)]
    for g in range(G):
        comms[g].scatter(shards[g], U)
    for g in range(G):
        comms[g].gather(U)
    for g in range(G):
        comms[g].project(U, None, outs[g], cnt[g][0:1], cnt[g][1:2])
    errs = []
    for c in ctxs:
        try:
            c.sync()
            errs.append(0)
        except ds.DialSortError as e:
            errs.append(e.code)
    big = int(np.argmax([r[2] for r in ref]))
    for g in range(G):
        Hr, outr, cr, offr = ref[g]
        assert int(cnt[g][0]) == cr and int(cnt[g][1]) == offr
        m = min(cr, cap)
        assert np.array_equal(outs[g][:m].cpu().numpy(), outr[:m])
        assert errs[g] == (3 if g == big else 0)


@pytest.mark.parametrize("G,U,dist", [(2, 65536, "uniform"), (4, 1 << 20, "zipf"), (8, 65536, "hot1")])
def test_loopback_nccl_sequence(ds, cuda_dev, G, U, dist):
    """The NCCL baseline's sequence (sharded.sharded_sort): local histograms through the C ABI,
    the reduce-scatter (here a device-side torch sum standing in for ncclReduceScatter), the
    slice projection through the C ABI with key_base g L."""
    n = 1_000_003
    x = keys_of(dist, n, U, seed=11)
    ctx = ds.Context(0, max_n=n, max_U=U)
    L = U // G
    Hl = []
    for g in range(G):
        Hl.append(ctx.histogram(to_dev(x[g * n // G:(g + 1) * n // G]), U).to(torch.int64))
    Hsum = torch.stack(Hl).sum(0)
    for g in range(G):
        Hs = Hsum[g * L:(g + 1) * L].to(torch.int32).contiguous()
        out = torch.empty(n, dtype=torch.int32, device=cuda_dev)
        tot = torch.zeros(1, dtype=torch.int64, device=cuda_dev)
        ctx.reconstruct(Hs, out, key_base=g * L, exact=False, d_total=tot)
        ctx.sync()
        Hr, outr, cr, offr = oracle.sharded_rank(x, U, G, g)
        assert np.array_equal(H64(Hs), Hr)
        assert int(tot) == cr
        assert np.array_equal(out[:cr].cpu().numpy(), outr)


@pytest.mark.parametrize("G,shape", [(2, "full"), (4, "full"), (8, "full"), (4, "hot"), (8, "narrow"), (3, "full")])
def test_loopback_sharded_radix(ds, cuda_dev, G, shape):
    """Sharded DialSort-Radix: top-digit histograms all-gathered, top-byte ranges, keys stored
    into the owners' receive buffers, local 4-pass LSD; every rank's output, count and offset vs
    the oracle's O4' reading; three calls (both buffer parities)."""
    n = 2_000_011
    rng = np.random.default_rng(G)
    if shape == "full":
        x = synth.full_int32(n, seed=G)
    elif shape == "hot":  # half the keys in one top byte
        x = synth.full_int32(n, seed=G)
        x[::2] = (x[::2] & 0x00FFFFFF) | 0x12000000
    else:  # all keys in two top bytes: ranks with empty ranges
        x = rng.integers(-2 ** 24, 2 ** 24, size=n).astype(np.int32)
    ctxs, comms = make_ranks(ds, G, 1, n, max_recv=n)
    shards = [to_dev(x[g * n // G:(g + 1) * n // G]) for g in range(G)]
    ref = [oracle.sharded_radix_rank(x, G, g) for g in range(G)]
    for call in range(3):
        outs = [torch.empty(n, dtype=torch.int32, device=cuda_dev) for _ in range(G)]
        cnt = [torch.zeros(2, dtype=torch.int64, device=cuda_dev) for _ in range(G)]
        for g in range(G):
            comms[g].radix_hist(shards[g])
        for g in range(G):
            comms[g].radix_split(shards[g], n, cnt[g][0:1], cnt[g][1:2])
        for g in range(G):
            comms[g].radix_local(outs[g])
        for c in ctxs:
            c.sync()
        for g in range(G):
            outr, cr, offr, _ = ref[g]
            assert int(cnt[g][0]) == cr and int(cnt[g][1]) == offr, (call, g)
            assert np.array_equal(outs[g][:cr].cpu().numpy(), outr), (call, g)


def test_comm_argument_errors(ds, cuda_dev):
    ctx = ds.Context(0)
    with pytest.raises(ds.DialSortError):
        ds.Comm(ctx, 9, 0, 1024)          # G > 8
    with pytest.raises(ds.DialSortError):
        ds.Comm(ctx, 2, 2, 1024)          # rank >= G
    a = ds.Comm(ctx, 2, 0, 1024)
    k = torch.zeros(16, dtype=torch.int32, device=cuda_dev)
    with pytest.raises(ds.DialSortError):
        a.scatter(k, 1024)                # not connected
    b = ds.Comm(ctx, 2, 1, 2048)          # another layout
    with pytest.raises(ds.DialSortError):
        a.connect_local([a, b])
    b2 = ds.Comm(ctx, 2, 1, 1024)
    a.connect_local([a, b2])
    with pytest.raises(ds.DialSortError):
        a.scatter(k, 1001)                # U % G != 0
    with pytest.raises(ds.DialSortError):
        a.scatter(k, 4096)                # U / G > max_U / G
    assert len(a.handle) == 128


def test_comm_wait_timeout_reports_error(ds, cuda_dev):
    """A rank whose peer never arrives gets DIALSORT_E_COMM (the wait gives up) instead of a hung
    GPU: rank 0 gathers although rank 1 never scattered."""
    ctxs, comms = make_ranks(ds, 2, 4096, 1000)
    comms[0].scatter(to_dev(synth.uniform(1000, 4096)), 4096)
    comms[0].gather(4096)
    with pytest.raises(ds.DialSortError) as e:
        ctxs[0].sync()
    assert e.value.code == 6
