"""GPU parity of the canonical-state queries (NEXT-1) and of DialSort-Radix's pass buffers and
variant selection, through the C ABI, against the oracle."""
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


@pytest.fixture(scope="module")
def ctx(ds, cuda_dev):
    return ds.Context(0, max_n=1 << 22, max_U=1 << 20)


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to("cuda:0")


def u32_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).to("cuda:0")


# ---- NEXT-1: frequency, presence, range-count, support set + prop:iso ---------------------------

def test_queries_paper_example(ds, ctx):
    """fig:viz state H = [0,2,0,4,0,2]: frequency(3) = 4, presence(2) = false,
    presence(5) = true, range-count(0,5) = 8, (3,5) = 6, (2,2) = 0; D = {1,3,5}, not an isomorphism."""
    keys = to_dev([3, 1, 3, 5, 1, 3, 5, 3])
    H = ctx.histogram(keys, 6)
    f = ctx.query(H, ds._lib.Q_FREQUENCY, to_dev([3, 0, 5]))
    p = ctx.query(H, ds._lib.Q_PRESENCE, to_dev([2, 5, 1]))
    r = ctx.query(H, ds._lib.Q_RANGE_COUNT, to_dev([[0, 5], [3, 5], [2, 2]]))
    D, cnt, iso = ctx.support_set(H)
    ctx.sync()
    assert f.cpu().tolist() == [4, 0, 2] and p.cpu().tolist() == [0, 1, 1] and r.cpu().tolist() == [8, 6, 0]
    assert int(cnt) == 3 and D[:3].cpu().tolist() == [1, 3, 5] and int(iso) == 0


@pytest.mark.parametrize("U,dist", [(1, "uniform"), (256, "uniform"), (5000, "zipf"), (65536, "sorted"),
                                    (300_007, "hot1"), (1 << 20, "uniform")])
def test_queries_random_vs_oracle(ds, ctx, U, dist):
    n = 400_003
    x = synth.hot1(n, U, seed=U) if dist == "hot1" else synth.make(dist, n, U, seed=U)
    H = ctx.histogram(to_dev(x), U)
    Hr = oracle.histogram(x, U)
    rng = np.random.default_rng(U)
    q = rng.integers(0, U, size=10_001)
    a = rng.integers(0, U, size=5003)
    b = np.minimum(U - 1, a + rng.integers(0, max(U // 3, 1), size=a.size))
    pairs = np.stack([a, b], 1)
    f = ctx.query(H, ds._lib.Q_FREQUENCY, to_dev(q))
    p = ctx.query(H, ds._lib.Q_PRESENCE, to_dev(q))
    r = ctx.query(H, ds._lib.Q_RANGE_COUNT, to_dev(pairs))
    D, cnt, iso = ctx.support_set(H)
    ctx.sync()
    assert np.array_equal(f.cpu().numpy(), Hr[q].astype(np.int64))
    assert np.array_equal(p.cpu().numpy(), (Hr[q] > 0).astype(np.int64))
    assert r.cpu().tolist() == [oracle.range_count(Hr, int(i), int(j)) for i, j in pairs]
    Dr = oracle.support_set(Hr)
    assert int(cnt) == Dr.size and np.array_equal(D[:Dr.size].cpu().numpy().view(np.uint32), Dr)
    assert int(iso) == int(Dr.size == U)


def test_support_set_isomorphism_condition(ds, ctx):
    """prop:iso: phi is an order-isomorphism iff D = [0, U-1]; every key once (U = 4, the SPEC
    example) and a full universe of 65536 with one key removed."""
    for keys, U, want in [([2, 0, 3, 1], 4, 1), (list(range(65536)), 65536, 1), (list(range(1, 65536)), 65536, 0)]:
        H = ctx.histogram(to_dev(keys), U)
        D, cnt, iso = ctx.support_set(H)
        ctx.sync()
        assert int(iso) == want and int(cnt) == len(set(keys))
        assert D[:int(cnt)].cpu().tolist() == sorted(set(keys))


def test_query_range_errors(ds, ctx):
    H = ctx.histogram(to_dev([0, 1, 1]), 4)
    ctx.query(H, ds._lib.Q_FREQUENCY, to_dev([1, 4, 2]))      # 4 is outside [0, 4)
    with pytest.raises(ds.DialSortError) as e:
        ctx.sync()
    assert e.value.code == 2 and e.value.info.first_bad_index == 1 and e.value.info.first_bad_key == 4
    ctx.query(H, ds._lib.Q_RANGE_COUNT, to_dev([[0, 3], [3, 1]]))  # a > b
    with pytest.raises(ds.DialSortError) as e:
        ctx.sync()
    assert e.value.code == 2 and e.value.info.first_bad_index == 1


# ---- DialSort-Radix: per-pass buffers and the two pass variants ---------------------------------

@pytest.mark.parametrize("variant", [3, 4])
@pytest.mark.parametrize("n,shape", [(8, "full"), (100_000, "full"), (1_000_004, "full"), (524_288, "lowbyte"),
                                     (262_144, "equal_hi")])
def test_radix_pass_buffers_vs_oracle(ds, cuda_dev, variant, n, shape):
    """After pass p the buffer is the stable sort of the input by its low 8(p+1) bits — a unique
    array — compared with the oracle's pass buffers for each variant."""
    c = ds.Context(0)
    c.set_option(ds._lib.OPT_RADIX_VARIANT, variant)
    rng = np.random.default_rng(n)
    if shape == "full":
        x = synth.full_int32(n, seed=n)
    elif shape == "lowbyte":  # equal high bytes, whole warps of equal digits in passes 1..3
        x = ((rng.integers(-4, 4, size=n) << 8) | rng.integers(0, 256, size=n)).astype(np.int32)
    else:
        x = (0x7f000000 | rng.integers(0, 1 << 16, size=n)).astype(np.int32)
    passes = c.debug_radix_passes(to_dev(x))
    c.sync()
    ref_out, ref_passes = oracle.radix_sort_i32(x, return_passes=True)
    got = passes.cpu().numpy().view(np.uint32)
    for p in range(3):
        assert np.array_equal(got[p], ref_passes[p]), p
    assert np.array_equal(got[3].view(np.int32), ref_out)


def test_radix_lane_probe_and_variant_selection(ds, cuda_dev):
    """The context probes the ATOMS lane order once per device; automatic selection uses pass4
    only when the probe found no violation; forced variants are honoured."""
    c = ds.Context(0)
    v = c.get_option(ds._lib.OPT_RADIX_PROBE_VIOLATIONS)
    assert v >= 0
    assert c.radix_variant == (4 if v == 0 else 3)
    c.set_option(ds._lib.OPT_RADIX_VARIANT, 3)
    assert c.radix_variant == 3
    c.set_option(ds._lib.OPT_RADIX_VARIANT, 4)
    assert c.radix_variant == 4
    with pytest.raises(ds.DialSortError):
        c.set_option(ds._lib.OPT_RADIX_VARIANT, 5)
    x = synth.full_int32(300_001, seed=9)
    for var in (3, 4):
        c.set_option(ds._lib.OPT_RADIX_VARIANT, var)
        y = c.sort_int32(to_dev(x))
        c.sync()
        assert np.array_equal(y.cpu().numpy(), oracle.radix_sort_i32(x)), var


def test_concurrent_contexts_two_streams(ds, cuda_dev):
    """Two contexts issue grid-barrier kernels on two streams at once (the e2e pipeline's shape):
    cooperative launches keep each grid co-resident (no deadlock), results exact."""
    cs = [ds.Context(0, max_n=4_000_000, max_U=65536) for _ in range(2)]
    sts = [torch.cuda.Stream(cuda_dev) for _ in range(2)]
    xs = [synth.uniform(3_000_001, 65536, seed=60 + i) for i in range(6)]
    rs = [synth.full_int32(2_000_003, seed=70 + i) for i in range(6)]
    dx = [to_dev(x) for x in xs]
    dr = [to_dev(r) for r in rs]
    torch.cuda.synchronize()
    outs, routs = [], []
    for i in range(6):
        with torch.cuda.stream(sts[i % 2]):
            outs.append(cs[i % 2].sort(dx[i], 65536))
            routs.append(cs[i % 2].sort_int32(dr[i]))
    for i in range(2):
        with torch.cuda.stream(sts[i]):
            cs[i].sync()
    torch.cuda.synchronize()
    for i in range(6):
        assert np.array_equal(outs[i].cpu().numpy(), oracle.sort(xs[i], 65536)), i
        assert np.array_equal(routs[i].cpu().numpy(), oracle.radix_sort_i32(rs[i])), i


# ---- NEXT-3: Proposition 2 coded domains -------------------------------------------------------

@pytest.mark.parametrize("width,U,n", [(1, 256, 1_000_003), (1, 7, 99_999), (2, 366, 2_000_001), (2, 65536, 3_000_017),
                                       (4, 128, 500_001)])
def test_sort_domain_vs_oracle(ds, ctx, width, U, n):
    """Items of 1 / 2 / 4 bytes through phi (an encode table for bytes) and phi^-1 (a decode
    table) against the oracle's A2, including unaligned item pointers (odd offsets)."""
    rng = np.random.default_rng(width * 1000 + U)
    enc = dec = None
    if width == 1 and U == 7:  # table-driven 7-element enumeration (symbols are arbitrary bytes)
        symbols = rng.permutation(np.arange(256))[:7]
        enc_h = np.zeros(256, dtype=np.uint32)
        enc_h[symbols] = np.arange(7)
        items = rng.choice(symbols, size=n).astype(np.uint8)
        dec_h = (symbols * 1000 + 7).astype(np.int32)
        enc, dec = u32_dev(enc_h), to_dev(dec_h)
        ref = oracle.sort_domain(items, U, encode=enc_h, decode=dec_h)
    else:
        dt = {1: np.uint8, 2: np.uint16, 4: np.int32}[width]
        items = rng.integers(0, U, size=n).astype(dt)
        dec_h = (np.arange(U) * 3 - 5).astype(np.int32)  # a decode table (order-preserving)
        dec = to_dev(dec_h)
        ref = oracle.sort_domain(items, U, decode=dec_h)
    tdt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[width]
    buf = torch.empty(n + 8, dtype=tdt, device="cuda:0")
    off = 3 if width < 4 else 1
    it = buf[off:off + n]
    it.copy_(torch.from_numpy(items.view({1: np.uint8, 2: np.int16, 4: np.int32}[width])))
    out = ctx.sort_domain(it, U, encode=enc, decode=dec)
    ctx.sync()
    assert np.array_equal(out.cpu().numpy(), ref)


def test_sort_domain_ascii_and_range_error(ds, ctx):
    s = b"the quick brown fox jumps over the lazy dog" * 1000
    items = torch.from_numpy(np.frombuffer(s, dtype=np.uint8).copy()).to("cuda:0")
    out = ctx.sort_domain(items, 256)
    ctx.sync()
    assert bytes(out.cpu().numpy().astype(np.uint8)) == bytes(sorted(s))
    bad = torch.tensor([1, 2, 300, 4], dtype=torch.int16, device="cuda:0")
    ctx.sort_domain(bad, 256)
    with pytest.raises(ds.DialSortError) as e:
        ctx.sync()
    assert e.value.code == 2 and e.value.info.first_bad_index == 2
    big = np.random.default_rng(1).integers(0, 256, size=100_003).astype(np.int16)
    big[50_001] = 999                         # inside the vectorised body
    big[77_777] = 1000
    ctx.sort_domain(torch.from_numpy(big).to("cuda:0"), 256)
    with pytest.raises(ds.DialSortError) as e:
        ctx.sync()
    assert e.value.code == 2 and e.value.info.first_bad_index == 50_001 and e.value.info.bad_count == 2


# ---- batched sort: independent steps overlapped on CTA groups ------------------------------------

@pytest.mark.parametrize("U,nb", [(65536, 8), (65536, 3), (4096, 16), (98304, 5), (65536, 20), (1000, 2)])
def test_sort_batch_vs_oracle(ds, cuda_dev, U, nb):
    """dialsort_sort_batch_async: every batch's output and H equal the oracle's, whatever the
    mix (uniform, Zipf -> share-mode projection, all-equal -> packed-counter overflow fallback,
    ragged sizes, in place), over three calls (lane workspace parities)."""
    c = ds.Context(0, max_n=3_000_000, max_U=U)
    rng = np.random.default_rng(U + nb)
    for call in range(3):
        xs = []
        for j in range(nb):
            n = int(rng.integers(200_000, 2_500_000))
            kind = (j + call) % 5
            if kind == 0:
                x = synth.uniform(n, U, seed=j + 10 * call)
            elif kind == 1:
                x = synth.zipf(n, U, seed=j + 10 * call)
            elif kind == 2:
                x = np.full(n, (j * 7919) % U, dtype=np.int32)
            elif kind == 3:
                x = synth.make("sorted", n, U, seed=j)
            else:
                x = synth.hot1(n, U, seed=j)
            xs.append(x)
        ks = [to_dev(x) for x in xs]
        outs = [k if j % 4 == 3 else torch.empty_like(k) for j, k in enumerate(ks)]  # some in place
        Hs = [torch.empty(U, dtype=torch.int32, device=cuda_dev) for _ in range(nb)]
        c.sort_batch(ks, U, outs, Hs)
        c.sync()
        for j in range(nb):
            Hr = oracle.histogram(xs[j], U)
            assert np.array_equal(Hs[j].cpu().numpy().view(np.uint32).astype(np.uint64), Hr), (call, j)
            assert np.array_equal(outs[j].cpu().numpy(), oracle.project(Hr)), (call, j)


@pytest.mark.parametrize("U,nb,lo,hi", [(256, 2, 1, 5000), (256, 9, 10_000, 120_000), (8192, 64, 1, 60_000),
                                          (7, 70, 100, 30_000), (1024, 12, 120_001, 400_000),
                                          (8192, 5, 60_000, 150_000)])
def test_sort_batch_small_clusters(ds, cuda_dev, U, nb, lo, hi):
    """Batches of small sorts (U <= 8192, n <= 4e5): one thread-block cluster per batch in one
    launch (k_sort_small_batch — 8-CTA clusters up to 120000 keys, 16-CTA above; more than 64
    batches in several launches): ragged sizes, uniform / Zipf / one key / sorted, some in place,
    every batch's H and output vs the oracle."""
    c = ds.Context(0, max_n=hi, max_U=U)
    rng = np.random.default_rng(U * nb + lo)
    xs = []
    for j in range(nb):
        n = int(rng.integers(lo, hi + 1))
        kind = j % 4
        x = (synth.uniform(n, U, seed=j) if kind == 0 else synth.zipf(n, U, seed=j) if kind == 1 else
             np.full(n, (j * 31) % U, dtype=np.int32) if kind == 2 else synth.make("sorted", n, U, seed=j))
        xs.append(x)
    ks = [to_dev(x) for x in xs]
    outs = [k if j % 3 == 2 else torch.empty_like(k) for j, k in enumerate(ks)]
    Hs = [torch.empty(U, dtype=torch.int32, device=cuda_dev) for _ in range(nb)]
    c.sort_batch(ks, U, outs, Hs)
    c.sync()
    for j in range(nb):
        Hr = oracle.histogram(xs[j], U)
        assert np.array_equal(Hs[j].cpu().numpy().view(np.uint32).astype(np.uint64), Hr), j
        assert np.array_equal(outs[j].cpu().numpy(), oracle.project(Hr)), j


def test_sort_batch_range_error(ds, cuda_dev):
    """A bad key in one batch of a batched launch is reported by dialsort_sync of the context."""
    c = ds.Context(0)
    xs = [synth.uniform(1_000_000, 65536, seed=j) for j in range(4)]
    xs[2][123_457] = 70_000
    ks = [to_dev(x) for x in xs]
    c.sort_batch(ks, 65536)
    with pytest.raises(ds.DialSortError) as e:
        c.sync()
    assert e.value.code == 2 and e.value.info.first_bad_index == 123_457
    c.sort_batch(ks[:2], 65536)
    c.sync()  # (cleared)


# ---- CUDA graphs: captured once, replayed with new inputs ---------------------------------------

def test_cuda_graph_replay(ds, cuda_dev):
    """The fused step, the batched sort, the reconstruct of a given H, DialSort-Radix, the
    hierarchical path (U = 2^20) and the queries keep their sequencing state on the device
    (FusedState, sense-reversing barriers, self-resetting counters), so a CUDA graph captured
    once replays correctly: three replays with fresh inputs copied into the captured buffers,
    every output against the oracle."""
    c = ds.Context(0, max_n=2_000_000, max_U=65536)
    U = 65536
    n1, nb = 1_500_007, [700_001, 900_003, 650_000]
    k1 = torch.empty(n1, dtype=torch.int32, device=cuda_dev)
    kb = [torch.empty(m, dtype=torch.int32, device=cuda_dev) for m in nb]
    kr = torch.empty(1_000_003, dtype=torch.int32, device=cuda_dev)
    H = torch.empty(U, dtype=torch.int32, device=cuda_dev)
    o1 = torch.empty_like(k1)
    ob = [torch.empty_like(k) for k in kb]
    orad = torch.empty_like(kr)
    orec = torch.empty(n1, dtype=torch.int32, device=cuda_dev)
    q = torch.arange(0, U, 97, dtype=torch.int32, device=cuda_dev)
    Uh = 1 << 20  # the hierarchical path (sampled partition + batched block steps)
    kh = torch.empty(1_200_001, dtype=torch.int32, device=cuda_dev)
    oh = torch.empty_like(kh)

    def fill(seed):
        xs = [synth.uniform(n1, U, seed=seed)] + [synth.zipf(m, U, seed=seed + j + 1) for j, m in enumerate(nb)]
        xr = synth.full_int32(kr.numel(), seed=seed + 9)
        k1.copy_(torch.from_numpy(xs[0]))
        for k, x in zip(kb, xs[1:]):
            k.copy_(torch.from_numpy(x))
        kr.copy_(torch.from_numpy(xr))
        xh = synth.uniform(kh.numel(), Uh, seed=seed + 5)
        kh.copy_(torch.from_numpy(xh))
        torch.cuda.synchronize()
        return xs, xr, xh

    def work():
        c.sort(k1, U, out=o1, H=H)
        c.sort_batch(kb, U, ob)
        c.reconstruct(H, orec)
        c.sort_int32(kr, out=orad)
        c.sort(kh, Uh, out=oh)
        return c.query(H, ds._lib.Q_FREQUENCY, q)

    fill(1)
    work()  # (workspaces sized before the capture)
    c.sync()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f = work()
    for rep in range(3):
        xs, xr, xh = fill(100 + rep)
        g.replay()
        torch.cuda.synchronize()
        c.sync()
        Hr = oracle.histogram(xs[0], U)
        assert np.array_equal(o1.cpu().numpy(), oracle.project(Hr)), rep
        assert np.array_equal(orec.cpu().numpy(), oracle.project(Hr)), rep
        for o, x in zip(ob, xs[1:]):
            assert np.array_equal(o.cpu().numpy(), oracle.sort(x, U)), rep
        assert np.array_equal(orad.cpu().numpy(), oracle.radix_sort_i32(xr)), rep
        assert np.array_equal(f.cpu().numpy(), Hr[::97].astype(np.int64)), rep
        assert np.array_equal(oh.cpu().numpy(), oracle.sort(xh, Uh)), rep
