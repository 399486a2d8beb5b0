"""Host-parallel DialSort (DS-Parallel analog, baseline/ds_parallel.c): a reported CPU baseline
for bench.py on the box's host cores.  Not the oracle (oracle/) and not the product (the CUDA
path); compiled with gcc -O3 -pthread on first use."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_DIR, "ds_parallel.c")
_LIB = os.path.join(_DIR, "libds_parallel.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", "-O3", "-march=native", "-std=c99", "-pthread", "-shared", "-fPIC",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.ds_parallel_sort.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int]
        _lib = lib
    return _lib


def threads() -> int:
    return len(os.sched_getaffinity(0))


def sort(keys: np.ndarray, U: int, T: int | None = None, out: np.ndarray | None = None):
    """DS-Parallel sort of int32 keys in [0, U) with T threads (default: the cores this process
    may use); returns (out, H)."""
    k = np.ascontiguousarray(keys, dtype=np.int32)
    if out is None:
        out = np.empty(max(k.size, 1), dtype=np.int32)
    H = np.empty(max(int(U), 1), dtype=np.uint32)
    rc = _L().ds_parallel_sort(k.ctypes.data, k.size, int(U), out.ctypes.data, H.ctypes.data,
                               int(T or threads()))
    if rc:
        raise RuntimeError(f"ds_parallel_sort rc={rc}")
    return out[: k.size], H[: int(U)]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
