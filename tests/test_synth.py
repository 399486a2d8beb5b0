"""The seeded input generators: determinism, host/device byte identity, workload statistics."""
import numpy as np
import torch

import synth


def test_splitmix64_reference_values():
    # splitmix64 with state 0: the first outputs of the public reference generator
    # (state += golden; z = mix(state)) are 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4.
    z = synth.mix64(np.array([0x9E3779B97F4A7C15, (2 * 0x9E3779B97F4A7C15) & (2 ** 64 - 1)], dtype=np.uint64))
    assert [int(v) for v in z] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4]


def test_counter_based_slices_match():
    a = synth.uniform(10_000, 65536)
    b = synth.uniform(3000, 65536, lo=5000)
    assert np.array_equal(a[5000:8000], b)


def test_torch_forms_match_numpy():
    for U in (1, 2, 256, 65536, 1 << 20, 1 << 31):
        assert np.array_equal(synth.uniform(50_001, U, lo=3),
                              synth.device_uniform(50_001, U, lo=3, device="cpu").numpy())
    assert np.array_equal(synth.full_int32(50_001, lo=9), synth.device_full_int32(50_001, lo=9, device="cpu").numpy())


def test_ranges():
    for U in (1, 7, 65536):
        k = synth.uniform(100_000, U)
        assert k.min() >= 0 and k.max() < U
    x = synth.full_int32(1_000_000)
    assert x.min() < -2 ** 30 and x.max() > 2 ** 30


def test_zipf_statistics():
    k = synth.zipf(2_000_000, 65536)
    c = np.bincount(k, minlength=65536)
    # p(rank 1) = 1 / H_{65536,1.2} = 19.81%
    assert abs(c.max() / k.size - 0.1981) < 0.003
    perm = synth.permutation(65536)
    assert np.array_equal(np.sort(perm), np.arange(65536))
    assert int(np.argmax(c)) == int(perm[0])


def test_hot1_exact_count():
    n, U = 1_000_000, 65536
    k = synth.hot1(n, U)
    u = synth.uniform(n, U)
    h = int(synth.bounded(synth.stream(synth.SEED, 3, 0, 1), U)[0])
    forced = np.flatnonzero(k != u)
    assert forced.size <= n // 100 and np.all(k[forced] == h)
    assert int((k == h).sum()) >= n // 100


def test_sorted_reverse():
    s = synth.make("sorted", 10_000, 300)
    r = synth.make("reverse", 10_000, 300)
    assert np.all(s[1:] >= s[:-1]) and np.array_equal(r, s[::-1])
    assert np.array_equal(np.sort(synth.uniform(10_000, 300)), s)


def test_skewed_mixture():
    k = synth.skewed(200_000, 65536)
    frac = float((k <= 65536 // 20).mean())
    assert 0.80 < frac < 0.83   # 80% in [0, floor(0.05U)] plus the uniform 20%'s share
