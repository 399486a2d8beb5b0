"""Seeded synthetic inputs for DialSort (shared by the oracle tests and the CUDA path).

This module holds NO arithmetic of the method (no histogram, no projection, no radix
pass): only the counter-based generator that both sides draw their input bytes from
(SURVEY.md §8(c) readings 11-16).  The paper fixes the seed 20260321
 but not the generator; we use splitmix64 in counter mode:

    z_i(s) = mix64(seed + s*0xD1B54A32D192ED03 + (i+1)*0x9E3779B97F4A7C15)   (mod 2^64)

Stream ids: 0 keys, 1 Zipf rank->key permutation, 2 hot-position selection, 3 hot value,
4 skewed-mixture selector.  Being counter based, element i can be produced anywhere, so a
rank's shard [lo, hi) is generated on its own device and equals the slice of the full
host array (``device_uniform`` / ``device_full_int32`` vs the numpy forms).
"""
from __future__ import annotations

import numpy as np

SEED = 20260321
GOLDEN = 0x9E3779B97F4A7C15
STREAM = 0xD1B54A32D192ED03
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
_MASK64 = (1 << 64) - 1

DISTS = ("uniform", "zipf", "sorted", "reverse", "hot1", "skewed")


def _u64(x: int) -> np.uint64:
    return np.uint64(x & _MASK64)


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= _u64(M1)
        z ^= z >> np.uint64(27)
        z *= _u64(M2)
        z ^= z >> np.uint64(31)
    return z


def stream(seed: int, s: int, lo: int, hi: int) -> np.ndarray:
    """z_i(s) for i in [lo, hi) as uint64."""
    i = np.arange(lo, hi, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = _u64(seed + s * STREAM)
        z = base + (i + np.uint64(1)) * _u64(GOLDEN)
    return mix64(z)


def bounded(z: np.ndarray, U: int) -> np.ndarray:
    """Multiply-high range reduction: ((z >> 32) * U) >> 32, in [0, U) (reading R12)."""
    with np.errstate(over="ignore"):
        return ((z >> np.uint64(32)) * np.uint64(U)) >> np.uint64(32)


def uniform(n: int, U: int, seed: int = SEED, lo: int = 0, chunk: int = 1 << 24) -> np.ndarray:
    """i.i.d. uniform int32 keys on [0, U) — configs c1, c2, c4; elements [lo, lo+n)."""
    out = np.empty(n, dtype=np.int32)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        out[a:b] = bounded(stream(seed, 0, lo + a, lo + b), U).astype(np.int32)
    return out


def full_int32(n: int, seed: int = SEED, lo: int = 0, chunk: int = 1 << 24) -> np.ndarray:
    """i.i.d. uniform over the full int32 range — config c5: x = (int32)(uint32)(z >> 32)."""
    out = np.empty(n, dtype=np.int32)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        out[a:b] = (stream(seed, 0, lo + a, lo + b) >> np.uint64(32)).astype(np.uint32).view(np.int32)
    return out


def permutation(U: int, seed: int = SEED) -> np.ndarray:
    """Seeded Fisher-Yates permutation of [0, U) driven by stream 1 (reading R13)."""
    perm = np.arange(U, dtype=np.int64)
    if U < 2:
        return perm
    z = stream(seed, 1, 0, U - 1)
    for t in range(U - 1):
        i = U - 1 - t
        j = int(((int(z[t]) >> 32) * (i + 1)) >> 32)
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def zipf_cdf(U: int, s: float = 1.2) -> np.ndarray:
    w = np.power(np.arange(1, U + 1, dtype=np.float64), -s)
    c = np.cumsum(w)
    c = c / c[-1]
    c[-1] = 1.0
    return c


def zipf(n: int, U: int, s: float = 1.2, seed: int = SEED) -> np.ndarray:
    """Zipf(s) ranks mapped to keys by a seeded permutation — config c3(i)."""
    cdf = zipf_cdf(U, s)
    perm = permutation(U, seed)
    z = stream(seed, 0, 0, n)
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    rank = np.searchsorted(cdf, u, side="right")
    rank = np.minimum(rank, U - 1)
    return perm[rank].astype(np.int32)


def hot1(n: int, U: int, seed: int = SEED, frac: float = 0.01) -> np.ndarray:
    """Uniform keys with exactly floor(frac*n) positions forced to one hot value — c3(iv)."""
    keys = uniform(n, U, seed)
    m = int(n * frac) if frac != 0.01 else n // 100
    idx = np.arange(n, dtype=np.int64)
    z = stream(seed, 2, 0, m)
    for t in range(m):
        j = t + int(((int(z[t]) >> 32) * (n - t)) >> 32)
        idx[t], idx[j] = idx[j], idx[t]
    h = int(bounded(stream(seed, 3, 0, 1), U)[0])
    keys[idx[:m]] = h
    return keys


def skewed(n: int, U: int, seed: int = SEED) -> np.ndarray:
    """The paper's 'skewed' mixture: 80% uniform on [0, floor(0.05U)], 20% on
    [0, U-1]; selector = stream 4 (reading R16, NEXT-2 workload)."""
    z = stream(seed, 0, 0, n)
    sel = bounded(stream(seed, 4, 0, n), 10) < np.uint64(8)
    hi = U // 20 + 1
    a = bounded(z, hi)
    b = bounded(z, U)
    return np.where(sel, a, b).astype(np.int32)


def make(dist: str, n: int, U: int, seed: int = SEED) -> np.ndarray:
    """Host array for a bounded-universe distribution name."""
    if dist == "uniform":
        return uniform(n, U, seed)
    if dist == "zipf":
        return zipf(n, U, 1.2, seed)
    if dist == "sorted":
        return np.sort(uniform(n, U, seed), kind="stable")
    if dist == "reverse":
        return np.ascontiguousarray(np.sort(uniform(n, U, seed), kind="stable")[::-1])
    if dist == "hot1":
        return hot1(n, U, seed)
    if dist == "skewed":
        return skewed(n, U, seed)
    raise ValueError(f"unknown distribution {dist!r}")


# ---------------------------------------------------------------------------------------
# Device-side forms (torch int64 with wrapping multiplies); byte-identical to the numpy
# forms, used only to avoid host generation + H2D of the multi-GB configs (c4, c5).
# ---------------------------------------------------------------------------------------

def _s64(x: int) -> int:
    x &= _MASK64
    return x - (1 << 64) if x >= (1 << 63) else x


def _torch_mix64(z):
    import torch  # noqa: F401

    def lsr(v, s):
        return (v >> s) & ((1 << (64 - s)) - 1)

    z = z ^ lsr(z, 30)
    z = z * _s64(M1)
    z = z ^ lsr(z, 27)
    z = z * _s64(M2)
    z = z ^ lsr(z, 31)
    return z


def _torch_stream(seed: int, s: int, lo: int, hi: int, device):
    import torch
    i = torch.arange(lo + 1, hi + 1, dtype=torch.int64, device=device)
    z = i * _s64(GOLDEN) + _s64(seed + s * STREAM)
    return _torch_mix64(z)


def device_uniform(n: int, U: int, seed: int = SEED, lo: int = 0, device="cuda",
                   chunk: int = 1 << 25):
    """torch.int32 tensor equal to uniform(n, U, seed, lo), generated on `device`."""
    import torch
    out = torch.empty(n, dtype=torch.int32, device=device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        z = _torch_stream(seed, 0, lo + a, lo + b, device)
        hi32 = (z >> 32) & 0xFFFFFFFF
        # (hi32 * U) >> 32 without 64-bit overflow: split U into 16-bit halves.
        uh, ul = U >> 16, U & 0xFFFF
        t = hi32 * ul
        k = (hi32 * uh + (t >> 16)) >> 16
        out[a:b] = k.to(torch.int32)
        del z, hi32, t, k
    return out


def device_full_int32(n: int, seed: int = SEED, lo: int = 0, device="cuda", chunk: int = 1 << 25):
    """torch.int32 tensor equal to full_int32(n, seed, lo), generated on `device`."""
    import torch
    out = torch.empty(n, dtype=torch.int32, device=device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        z = _torch_stream(seed, 0, lo + a, lo + b, device)
        hi32 = (z >> 32) & 0xFFFFFFFF
        out[a:b] = torch.where(hi32 >= (1 << 31), hi32 - (1 << 32), hi32).to(torch.int32)
        del z, hi32
    return out
