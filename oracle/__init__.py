"""CPU oracle for the DialSort hot path (arxiv 2605.16667) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
(``paper_2605_16667_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle/oracle.c`` (plain single-threaded C, 64-bit counters,
each function citing the PAPER.md passage it follows); this module only compiles it with
gcc on first use and marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_DIR, "oracle.c")
_LIB = os.path.join(_DIR, "liboracle.so")

OK, E_INVALID_ARG, E_KEY_RANGE, E_SIZE = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -O2, no vectorisation flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _L():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        u64, i32, i64, ci = ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int
        lib.oracle_histogram.argtypes = [P, u64, u64, P, P]
        lib.oracle_project.argtypes = [P, u64, i64, P, u64]
        lib.oracle_sort.argtypes = [P, u64, u64, P, P, P]
        lib.oracle_crn_resolve.argtypes = [P, P, ci, P, P]
        lib.oracle_crn_levels.argtypes = [P, P, P, ci]
        lib.oracle_crn_levels.restype = None
        lib.oracle_sharded_rank.argtypes = [P, u64, u64, ci, ci, P, P, u64, P, P, P]
        lib.oracle_radix_bias.argtypes = [i32]
        lib.oracle_radix_bias.restype = ctypes.c_uint32
        lib.oracle_radix_unbias.argtypes = [ctypes.c_uint32]
        lib.oracle_radix_unbias.restype = i32
        lib.oracle_radix_pass.argtypes = [P, u64, ci, P]
        lib.oracle_radix_pass.restype = None
        lib.oracle_radix_sort_i32.argtypes = [P, u64, P, P]
        lib.oracle_sharded_radix_rank.argtypes = [P, u64, ci, ci, P, u64, P, P, P]
        lib.oracle_sort_domain.argtypes = [P, ci, u64, u64, P, P, P, P]
        lib.oracle_range_count.argtypes = [P, u64, u64]
        lib.oracle_range_count.restype = u64
        lib.oracle_support_set.argtypes = [P, u64, P]
        lib.oracle_support_set.restype = u64
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _keys(keys) -> np.ndarray:
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.int32))
    return k


def histogram(keys, U: int) -> np.ndarray:
    """O1, eq:ingestion. Returns uint64 H[U]; raises OracleError on a bad key."""
    k = _keys(keys)
    H = np.empty(max(int(U), 1), dtype=np.uint64)
    bad = np.zeros(1, dtype=np.uint64)
    rc = _L().oracle_histogram(_ptr(k), k.size, int(U), _ptr(H), _ptr(bad))
    if rc == E_KEY_RANGE:
        i = int(bad[0])
        raise OracleError(rc, f"key {int(k[i])} at index {i} outside [0,{U})")
    if rc != OK:
        raise OracleError(rc, f"oracle_histogram rc={rc}")
    return H[: int(U)]


def project(H, key_base: int = 0, n_out: int | None = None) -> np.ndarray:
    """O2, eq:projection."""
    h = np.ascontiguousarray(np.asarray(H, dtype=np.uint64))
    n = int(h.sum()) if n_out is None else int(n_out)
    out = np.empty(max(n, 1), dtype=np.int32)
    rc = _L().oracle_project(_ptr(h), h.size, int(key_base), _ptr(out), n)
    if rc != OK:
        raise OracleError(rc, f"oracle_project rc={rc} (sum(H)={int(h.sum())}, n_out={n})")
    return out[:n]


def sort(keys, U: int) -> np.ndarray:
    """A1 sequential DialSort: histogram then projection."""
    k = _keys(keys)
    out = np.empty(max(k.size, 1), dtype=np.int32)
    H = np.empty(max(int(U), 1), dtype=np.uint64)
    bad = np.zeros(1, dtype=np.uint64)
    rc = _L().oracle_sort(_ptr(k), k.size, int(U), _ptr(out), _ptr(H), _ptr(bad))
    if rc != OK:
        raise OracleError(rc, f"oracle_sort rc={rc} bad_index={int(bad[0])}")
    return out[: k.size]


def sort_inplace(keys: np.ndarray, U: int) -> None:
    """In-place form (tab:struct_cost): out aliases keys."""
    assert keys.dtype == np.int32 and keys.flags.c_contiguous
    H = np.empty(max(int(U), 1), dtype=np.uint64)
    bad = np.zeros(1, dtype=np.uint64)
    rc = _L().oracle_sort(_ptr(keys), keys.size, int(U), _ptr(keys), _ptr(H), _ptr(bad))
    if rc != OK:
        raise OracleError(rc, f"oracle_sort rc={rc}")


def crn_resolve(lane_keys, lane_counts=None):
    """CRN multiset reading (lem:crn): list of (key, total count) in first-occurrence order."""
    k = _keys(lane_keys)
    c = np.ones(k.size, dtype=np.uint64) if lane_counts is None else np.ascontiguousarray(
        np.asarray(lane_counts, dtype=np.uint64))
    ok = np.empty(max(k.size, 1), dtype=np.int32)
    oc = np.empty(max(k.size, 1), dtype=np.uint64)
    m = _L().oracle_crn_resolve(_ptr(k), _ptr(c), k.size, _ptr(ok), _ptr(oc))
    return [(int(ok[i]), int(oc[i])) for i in range(m)]


def crn_levels(lane_keys, lane_counts=None, levels: int | None = None):
    """Literal def:crn_level adjacent-pair levels; returns list of (key, count)."""
    k = np.array(lane_keys, dtype=np.int32)
    c = np.ones(k.size, dtype=np.uint64) if lane_counts is None else np.array(lane_counts, dtype=np.uint64)
    if levels is None:
        levels = max(0, int(np.ceil(np.log2(max(k.size, 1)))))
    m = ctypes.c_int(k.size)
    _L().oracle_crn_levels(_ptr(k), _ptr(c), ctypes.addressof(m), int(levels))
    return [(int(k[i]), int(c[i])) for i in range(m.value)]


def sharded_rank(keys, U: int, G: int, g: int):
    """O3 reading R10: (H_slice uint64[U/G], out int32, count, global offset) for rank g."""
    k = _keys(keys)
    S = int(U) // int(G)
    Hs = np.empty(max(S, 1), dtype=np.uint64)
    out = np.empty(max(k.size, 1), dtype=np.int32)
    H = np.empty(max(int(U), 1), dtype=np.uint64)
    cnt = np.zeros(1, dtype=np.uint64)
    off = np.zeros(1, dtype=np.uint64)
    rc = _L().oracle_sharded_rank(_ptr(k), k.size, int(U), int(G), int(g), _ptr(Hs), _ptr(out),
                                  k.size, _ptr(cnt), _ptr(off), _ptr(H))
    if rc != OK:
        raise OracleError(rc, f"oracle_sharded_rank rc={rc}")
    c = int(cnt[0])
    return Hs[:S], out[:c], c, int(off[0])


def radix_bias(x: int) -> int:
    return int(_L().oracle_radix_bias(int(x)))


def radix_unbias(u: int) -> int:
    return int(_L().oracle_radix_unbias(int(u)))


def radix_pass(src_u32, p: int) -> np.ndarray:
    s = np.ascontiguousarray(np.asarray(src_u32, dtype=np.uint32))
    dst = np.empty(max(s.size, 1), dtype=np.uint32)
    _L().oracle_radix_pass(_ptr(s), s.size, int(p), _ptr(dst))
    return dst[: s.size]


def radix_sort_i32(keys, return_passes: bool = False):
    """A8 DialSort-Radix: returns sorted int32 (and the 4 biased pass buffers)."""
    k = _keys(keys)
    out = np.empty(max(k.size, 1), dtype=np.int32)
    passes = np.empty((4, max(k.size, 1)), dtype=np.uint32) if return_passes else None
    rc = _L().oracle_radix_sort_i32(_ptr(k), k.size, _ptr(out),
                                    _ptr(passes) if passes is not None else None)
    if rc != OK:
        raise OracleError(rc, f"oracle_radix_sort_i32 rc={rc}")
    if return_passes:
        return out[: k.size], passes[:, : k.size]
    return out[: k.size]


def sharded_radix_rank(keys, G: int, g: int):
    """O4' reading R19: (out int32, count, global offset, D[0..G]) of rank g of G."""
    k = _keys(keys)
    out = np.empty(max(k.size, 1), dtype=np.int32)
    cnt = np.zeros(1, dtype=np.uint64)
    off = np.zeros(1, dtype=np.uint64)
    D = np.zeros(9, dtype=np.uint32)
    rc = _L().oracle_sharded_radix_rank(_ptr(k), k.size, int(G), int(g), _ptr(out), k.size, _ptr(cnt), _ptr(off),
                                        _ptr(D))
    if rc != OK:
        raise OracleError(rc, f"oracle_sharded_radix_rank rc={rc}")
    c = int(cnt[0])
    return out[:c], c, int(off[0]), D[: int(G) + 1].astype(np.int64)


def sort_domain(items, U: int, encode=None, decode=None) -> np.ndarray:
    """A2 Proposition 2: items (uint8 / uint16 / int32 array), phi = encode table (1-byte items)
    or identity, phi^-1 = decode table or identity.  Returns the emitted int32 sequence."""
    it = np.ascontiguousarray(items)
    width = {np.dtype(np.uint8): 1, np.dtype(np.uint16): 2, np.dtype(np.int32): 4}[it.dtype]
    enc = None if encode is None else np.ascontiguousarray(encode, dtype=np.uint32)
    dec = None if decode is None else np.ascontiguousarray(decode, dtype=np.int32)
    out = np.empty(max(it.size, 1), dtype=np.int32)
    bad = np.zeros(1, dtype=np.uint64)
    rc = _L().oracle_sort_domain(_ptr(it), width, it.size, int(U), _ptr(enc) if enc is not None else None,
                                 _ptr(dec) if dec is not None else None, _ptr(out), _ptr(bad))
    if rc == E_KEY_RANGE:
        raise OracleError(rc, f"item {int(bad[0])} maps outside [0,{U})")
    if rc != OK:
        raise OracleError(rc, f"oracle_sort_domain rc={rc}")
    return out[: it.size]


def range_count(H, a: int, b: int) -> int:
    h = np.ascontiguousarray(np.asarray(H, dtype=np.uint64))
    return int(_L().oracle_range_count(_ptr(h), int(a), int(b)))


def support_set(H) -> np.ndarray:
    h = np.ascontiguousarray(np.asarray(H, dtype=np.uint64))
    D = np.empty(max(h.size, 1), dtype=np.uint32)
    m = _L().oracle_support_set(_ptr(h), h.size, _ptr(D))
    return D[:m]
