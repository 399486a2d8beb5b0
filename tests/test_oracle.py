"""Pins of the CPU oracle against what the paper and mathematics fix (never against itself).

- worked examples printed in the paper (tests/golden/, each fixture cites its passage);
- brute force with the language's own sort / tally on tiny inputs (thm:correct: the
  projection equals the sorted multiset, which is unique for keys-only sorting);
- the invariants of thm:correct and lem:crn;
- radix: the bias map's defining examples and per-pass stable-sort characterisation.
"""
import collections
import math
import random

import numpy as np
import pytest

import oracle
import synth
from conftest import read_golden


def ints(vals):
    return [int(v) for v in vals]


# ---- worked examples ----------------------------------------------------------------------

def test_fig_viz_histogram_and_projection():
    g = read_golden("fig_viz.txt")
    U = int(g["U"][0][0])
    keys = ints(g["keys"][0])
    H = oracle.histogram(keys, U)
    assert H.tolist() == ints(g["H"][0])
    assert oracle.project(H).tolist() == ints(g["out"][0])
    assert oracle.sort(keys, U).tolist() == ints(g["out"][0])


@pytest.mark.parametrize("name", ["fig_abacus.txt", "fig_physical.txt"])
def test_projection_examples(name):
    g = read_golden(name)
    H = np.array(ints(g["H"][0]), dtype=np.uint64)
    assert len(H) == int(g["U"][0][0])
    assert oracle.project(H).tolist() == ints(g["out"][0])


def test_crn_three_arrivals_of_42():
    g = read_golden("crn_42.txt")
    lanes = ints(g["lanes"][0])
    k, c = g["resolved"][0][0].split(":")
    assert oracle.crn_resolve(lanes) == [(int(k), int(c))]
    # the literal pairwise network of def:crn_level reaches the same single write
    assert oracle.crn_levels(lanes) == [(int(k), int(c))]


def test_canonical_state_queries():
    g = read_golden("queries.txt")
    H = np.array(ints(g["H"][0]), dtype=np.uint64)
    k, f = ints(g["frequency"][0])
    assert int(H[k]) == f
    for a, b, s in (ints(r) for r in g["range"]):
        assert oracle.range_count(H, a, b) == s
    assert oracle.support_set(H).tolist() == ints(g["support"][0])


# ---- brute force ------------------------------------------------------------------------------

def test_oracle_equals_builtin_sort_random():
    rng = random.Random(20260321)
    for trial in range(1000):
        U = rng.choice([1, 2, 16, 256, 1024, 65536])
        n = rng.choice([0, 1, 2, 3, 7, 31, 100, rng.randint(0, 10_000)])
        order = rng.choice(["uniform", "sorted", "reverse", "skew"])
        keys = [rng.randrange(U) for _ in range(n)]
        if order == "sorted":
            keys.sort()
        elif order == "reverse":
            keys.sort(reverse=True)
        elif order == "skew" and n:
            hot = rng.randrange(U)
            keys = [hot if rng.random() < 0.8 else k for k in keys]
        out = oracle.sort(keys, U)
        assert out.tolist() == sorted(keys), (trial, U, n, order)
        H = oracle.histogram(keys, U)
        tally = collections.Counter(keys)
        assert [int(h) for h in H] == [tally.get(k, 0) for k in range(U)]


def test_in_place_form():
    keys = synth.uniform(5000, 300, seed=7)
    ref = sorted(keys.tolist())
    buf = keys.copy()
    oracle.sort_inplace(buf, 300)
    assert buf.tolist() == ref


# ---- thm:correct invariants -------------------------------------------------------------------

@pytest.mark.parametrize("dist", synth.DISTS)
def test_thm_correct_invariants(dist):
    n, U = 20_000, 1024
    keys = synth.make(dist, n, U, seed=11)
    H = oracle.histogram(keys, U)
    out = oracle.project(H)
    assert int(H.sum()) == n                      # ΣH = n
    assert out.size == n                          # length n
    assert np.all(out[1:] >= out[:-1])            # nondecreasing
    assert np.array_equal(np.bincount(out, minlength=U), np.bincount(keys, minlength=U))  # multiset


# ---- special cases ----------------------------------------------------------------------------

def test_empty_and_degenerate():
    assert oracle.histogram([], 5).tolist() == [0] * 5
    assert oracle.sort([], 5).tolist() == []
    assert oracle.sort([0, 0, 0], 1).tolist() == [0, 0, 0]         # U = 1
    assert oracle.sort([4, 4], 5).tolist() == [4, 4]               # key = U-1
    assert oracle.project(np.zeros(7, dtype=np.uint64)).tolist() == []


def test_errors():
    with pytest.raises(oracle.OracleError) as e:
        oracle.histogram([1, 2, 9, 3, -1], 5)
    assert e.value.code == oracle.E_KEY_RANGE and "index 2" in str(e.value)   # first bad index
    with pytest.raises(oracle.OracleError) as e:
        oracle.histogram([0], 0)
    assert e.value.code == oracle.E_INVALID_ARG
    with pytest.raises(oracle.OracleError) as e:
        oracle.project(np.array([1, 2], dtype=np.uint64), n_out=4)
    assert e.value.code == oracle.E_SIZE


# ---- CRN ----------------------------------------------------------------------------------------

def test_crn_conservation_and_uniqueness():
    rng = random.Random(5)
    for _ in range(10_000):
        k = rng.choice([1, 2, 3, 4, 8, 16, 32])
        lanes = [rng.randrange(rng.choice([1, 2, 4, 64])) for _ in range(k)]
        counts = [rng.randint(1, 5) for _ in range(k)]
        res = oracle.crn_resolve(lanes, counts)
        keys = [a for a, _ in res]
        assert len(keys) == len(set(keys))                           # each key once
        tot = collections.Counter()
        for a, c in zip(lanes, counts):
            tot[a] += c
        assert dict(res) == dict(tot)                                # lem:crn conservation
        lv = oracle.crn_levels(lanes, counts)
        got = collections.Counter()
        for a, c in lv:
            got[a] += c
        assert got == tot                                            # pairwise levels conserve too


def test_crn_adjacent_pairing_counterexample():
    # def:crn_level pairs only adjacent items; [a,b,a,b] keeps both a's apart after
    # ceil(log2 4) = 2 levels, so the paper's "every key appears at most once" needs the
    # multiset reading (R1).  Conservation still holds.
    lv = oracle.crn_levels([7, 9, 7, 9])
    assert sorted(lv) == [(7, 1), (7, 1), (9, 1), (9, 1)]
    assert oracle.crn_resolve([7, 9, 7, 9]) == [(7, 2), (9, 2)]
    assert math.ceil(math.log2(16)) == 4 and math.ceil(math.log2(32)) == 5


# ---- radix ------------------------------------------------------------------------------------

def test_radix_bias_examples():
    # order-preserving bijection onto [0, 2^32): INT_MIN -> 0, 0 -> 2^31, -1 -> 2^31-1
    assert oracle.radix_bias(-2 ** 31) == 0
    assert oracle.radix_bias(0) == 2 ** 31
    assert oracle.radix_bias(-1) == 2 ** 31 - 1
    assert oracle.radix_bias(2 ** 31 - 1) == 2 ** 32 - 1
    for x in (-2 ** 31, -5, -1, 0, 1, 77, 2 ** 31 - 1):
        assert oracle.radix_unbias(oracle.radix_bias(x)) == x
    rng = random.Random(3)
    for _ in range(10_000):
        x, y = rng.randint(-2 ** 31, 2 ** 31 - 1), rng.randint(-2 ** 31, 2 ** 31 - 1)
        assert (x < y) == (oracle.radix_bias(x) < oracle.radix_bias(y))


def test_radix_equals_sorted_and_boundaries():
    B = [-2 ** 31, -1, 0, 1, 2 ** 31 - 1]
    assert oracle.radix_sort_i32([-1, 0, 1, -2 ** 31, 2 ** 31 - 1]).tolist() == sorted(B)
    rng = random.Random(9)
    for _ in range(300):
        n = rng.randint(0, 3000)
        x = [rng.choice(B) if rng.random() < 0.2 else rng.randint(-2 ** 31, 2 ** 31 - 1) for _ in range(n)]
        assert oracle.radix_sort_i32(x).tolist() == sorted(x)
    x = synth.full_int32(100_000, seed=1)
    assert np.array_equal(oracle.radix_sort_i32(x), np.sort(x))


def test_radix_passes_are_stable_digit_sorts():
    # After pass p the buffer is the stable sort of the biased keys by bits [0, 8(p+1)).
    x = synth.full_int32(4000, seed=2)
    x[::7] = x[3]                                      # repeated keys to expose stability
    out, passes = oracle.radix_sort_i32(x, return_passes=True)
    u = [int(v) & 0xFFFFFFFF ^ 0x80000000 for v in x.tolist()]
    for p in range(4):
        mask = (1 << (8 * (p + 1))) - 1
        assert passes[p].tolist() == sorted(u, key=lambda v: v & mask)     # Python sort is stable
    # a single pass on tagged keys keeps equal digits in input order
    src = np.array([(d << 8) | t for t, d in enumerate([5, 3, 5, 5, 3, 0, 5])], dtype=np.uint32)
    dst = oracle.radix_pass(src, 1)
    assert [int(v) & 0xFF for v in dst] == [5, 1, 4, 0, 2, 3, 6]


# ---- sharded reading (O3) ---------------------------------------------------------------------

@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_sharded_concatenation_is_the_sort(G):
    n, U = 30_001, 4096
    keys = synth.uniform(n, U, seed=G)
    full_H = collections.Counter(keys.tolist())
    pieces, off_expect = [], 0
    for g in range(G):
        Hs, out, cnt, off = oracle.sharded_rank(keys, U, G, g)
        S = U // G
        assert [int(h) for h in Hs] == [full_H.get(g * S + k, 0) for k in range(S)]  # Σ_ranks H_r
        assert off == off_expect and cnt == out.size
        off_expect += cnt
        pieces.append(out)
    assert np.concatenate(pieces).tolist() == sorted(keys.tolist())


# ---- O4' sharded DialSort-Radix (reading R19) -------------------------------------------------

@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_sharded_radix_concatenation_is_the_sort(G):
    """Against Python's sorted (independent of the oracle's own radix): the rank-order
    concatenation is the sort, offsets are running counts, every rank's keys lie in its own
    contiguous top-byte range, and the ranges tile [0, 256)."""
    rng = np.random.default_rng(70 + G)
    for trial in range(12):
        n = int(rng.choice([0, 1, 5, 257, 4000, 30001]))
        kind = trial % 4
        if kind == 0:
            x = rng.integers(-2 ** 31, 2 ** 31, size=n, dtype=np.int64).astype(np.int32)
        elif kind == 1:
            x = rng.integers(-3, 3, size=n).astype(np.int32)          # two top bytes only
        elif kind == 2:
            x = np.full(n, 2 ** 31 - 1, dtype=np.int32)                # one top byte
        else:
            x = (rng.integers(0, 4, size=n) * 0x40000000 - 2 ** 31).astype(np.int32)  # 4 hot top bytes
        pieces, off = [], 0
        prevD = None
        for g in range(G):
            out, cnt, o, D = oracle.sharded_radix_rank(x, G, g)
            assert D[0] == 0 and D[G] == 256 and all(D[i] <= D[i + 1] for i in range(G))
            assert prevD is None or list(D) == prevD
            prevD = list(D)
            assert o == off and cnt == out.size
            tb = (out.view(np.uint32) ^ np.uint32(0x80000000)) >> 24
            assert ((tb >= D[g]) & (tb < D[g + 1])).all()
            off += cnt
            pieces.append(out)
        assert off == n
        got = np.concatenate(pieces) if pieces else np.empty(0, np.int32)
        assert got.tolist() == sorted(x.tolist())


def test_sharded_radix_balance():
    """Closed forms of step 2: with every top byte equally frequent the ranges are exact
    256/G-byte blocks, and on uniform keys no rank is off n/G by more than one digit's count."""
    G = 4
    x = (np.repeat(np.arange(256, dtype=np.int64), 10) << 24) ^ 0x80000000
    x = (x & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    for g in range(G):
        _, cnt, o, D = oracle.sharded_radix_rank(x, G, g)
        assert list(D) == [0, 64, 128, 192, 256] and cnt == 640 and o == 640 * g
    x = synth.full_int32(100_000, seed=3)
    C = np.bincount((x.view(np.uint32) ^ np.uint32(0x80000000)) >> 24, minlength=256)
    for G in (2, 8):
        for g in range(G):
            _, cnt, _, _ = oracle.sharded_radix_rank(x, G, g)
            assert abs(cnt - 100_000 / G) <= C.max() + 1


# ---- A2 Proposition 2: general self-indexing through phi -----------------------------------------

def test_domain_spec_examples():
    """SPEC generic-domain examples: ASCII "dcba" with phi = code point (U = 256) -> "abcd";
    MIDI notes {60, 0, 127} with U = 128 -> {0, 60, 127}."""
    out = oracle.sort_domain(np.frombuffer(b"dcba", dtype=np.uint8), 256)
    assert bytes(out.astype(np.uint8)) == b"abcd"
    assert oracle.sort_domain(np.array([60, 0, 127], dtype=np.uint8), 128).tolist() == [0, 60, 127]


def test_domain_table_driven_enumeration():
    """A 7-element enumerated domain whose order is not the symbols' numeric order: phi = rank
    table (encode), phi^-1 = symbol table (decode).  Equals a comparison sort under <_S
    (Python's sorted with key = rank), and decode(encode(s)) = s."""
    rng = np.random.default_rng(5)
    symbols = rng.permutation(np.arange(10, 250))[:7].astype(np.uint8)   # arbitrary symbol bytes
    order = {int(s): r for r, s in enumerate(symbols)}                   # <_S: the table order
    enc = np.zeros(256, dtype=np.uint32)
    for s, r in order.items():
        enc[s] = r
    dec = symbols.astype(np.int32)
    for trial in range(50):
        items = rng.choice(symbols, size=int(rng.integers(0, 400))).astype(np.uint8)
        got = oracle.sort_domain(items, 7, encode=enc, decode=dec)
        assert got.tolist() == sorted(items.tolist(), key=lambda s: order[s])
    assert all(int(dec[enc[s]]) == s for s in symbols.tolist())


def test_domain_day_numbers_and_identity():
    """Calendar days (phi = day number, U = 366) as 2-byte items equal the sorted days; with
    identity maps the domain sort is the integer DialSort (A1) itself."""
    rng = np.random.default_rng(6)
    days = rng.integers(0, 366, size=5000).astype(np.uint16)
    assert oracle.sort_domain(days, 366).tolist() == sorted(days.tolist())
    x = synth.uniform(3001, 1000, seed=2)
    assert np.array_equal(oracle.sort_domain(x, 1000), oracle.sort(x, 1000))
    with pytest.raises(oracle.OracleError):
        oracle.sort_domain(np.array([1, 400], dtype=np.uint16), 366)
