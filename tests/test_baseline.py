"""The host-parallel DS-Parallel baseline (baseline/ds_parallel.c) is byte-identical to the
oracle ("must equal O2 byte for byte") at several thread counts."""
import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("T", [1, 2, 3, 8])
@pytest.mark.parametrize("dist,U", [("uniform", 256), ("zipf", 65536), ("sorted", 1000), ("hot1", 4096)])
def test_ds_parallel_equals_oracle(T, dist, U):
    import baseline
    x = synth.make(dist, 200_003, U, seed=T)
    out, H = baseline.sort(x, U, T)
    assert np.array_equal(out, oracle.sort(x, U))
    assert np.array_equal(H.astype(np.uint64), oracle.histogram(x, U))


def test_ds_parallel_edge_cases():
    import baseline
    for n, U, T in [(0, 5, 4), (1, 1, 8), (7, 3, 16)]:
        x = np.zeros(n, dtype=np.int32) if U == 1 else (np.arange(n) % U).astype(np.int32)
        out, _ = baseline.sort(x, U, T)
        assert np.array_equal(out, oracle.sort(x, U))
