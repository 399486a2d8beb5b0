"""DialSort on B200 — thin Python binding over the C ABI in include/dialsort.h.

The binding only marshals torch tensors (device memory, streams) into the C ABI calls of
``libdialsort.so``; histogram ingestion with the CRN, the offset scan, the projection and
the radix passes all run in the library's sm_100a kernels.  Names follow the paper
(arxiv 2605.16667): ``histogram`` (eq:ingestion), ``reconstruct`` (eq:projection),
``sort`` (DialSort), ``sort_int32`` (DialSort-Radix).
"""
from __future__ import annotations

import ctypes
import threading

import torch

from . import _lib
from ._lib import ErrorInfo

__all__ = [
    "DialSortError", "Context", "histogram", "reconstruct", "sort", "sort_int32", "sort_host",
    "range_count", "crn_resolve", "default_context", "LIB_PATH",
]

LIB_PATH = _lib.LIB_PATH
_L = _lib.lib


class DialSortError(RuntimeError):
    def __init__(self, code: int, msg: str, info: ErrorInfo | None = None):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.info = info


def _check(rc: int, info: ErrorInfo | None = None) -> None:
    if rc != _lib.OK:
        msg = (_L.dialsort_last_error() or b"").decode() or _L.dialsort_status_string(rc).decode()
        raise DialSortError(rc, msg, info)


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device: torch.device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _keys(t: torch.Tensor, name: str = "keys") -> torch.Tensor:
    if t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous int32 CUDA tensor")
    return t


class Context:
    """A dialsort_ctx: workspace + deferred-error word on one device (one stream at a time)."""

    def __init__(self, device=None, max_n: int = 0, max_U: int = 0):
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(_L.dialsort_ctx_create(self.device.index, int(max_n), int(max_U), ctypes.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            _L.dialsort_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- deferred errors --------------------------------------------------------------------
    def sync(self, raise_on_error: bool = True) -> ErrorInfo:
        info = ErrorInfo()
        rc = _L.dialsort_sync(self._h, _stream(self.device), ctypes.byref(info))
        if raise_on_error:
            _check(rc, info)
        return info

    # -- the hot path (enqueue on the current stream) -----------------------------------------
    def histogram(self, keys: torch.Tensor, U: int, H: torch.Tensor | None = None) -> torch.Tensor:
        """H[k] = |{i : keys[i] = k}|, eq:ingestion. Returns uint32 H as int32 view."""
        _keys(keys)
        if H is None:
            H = torch.empty(int(U), dtype=torch.int32, device=keys.device)
        _check(_L.dialsort_histogram_async(self._h, _ptr(keys), keys.numel(), int(U), _ptr(H),
                                           _stream(keys.device)))
        return H

    def reconstruct(self, H: torch.Tensor, out: torch.Tensor | None = None, n: int | None = None,
                    key_base: int = 0, exact: bool = True, d_total: torch.Tensor | None = None
                    ) -> torch.Tensor:
        """eq:projection: out[P[k]..P[k]+H[k]) = key_base + k."""
        if H.dtype != torch.int32 or not H.is_cuda or not H.is_contiguous():
            raise ValueError("H must be a contiguous int32 (uint32 bits) CUDA tensor")
        if out is None:
            if n is None:
                n = int(H.to(torch.int64).sum().item())  # host-side sizing only
            out = torch.empty(int(n), dtype=torch.int32, device=H.device)
        cap = out.numel() if n is None else int(n)
        _check(_L.dialsort_reconstruct_async(self._h, _ptr(H), H.numel(), int(key_base), _ptr(out), cap,
                                             1 if exact else 0, _ptr(d_total), _stream(H.device)))
        return out

    def sort(self, keys: torch.Tensor, U: int, out: torch.Tensor | None = None,
             H: torch.Tensor | None = None) -> torch.Tensor:
        """DialSort of keys in [0, U); out may be keys itself (in place)."""
        _keys(keys)
        if out is None:
            out = torch.empty_like(keys)
        _check(_L.dialsort_sort_async(self._h, _ptr(keys), keys.numel(), int(U), _ptr(out), _ptr(H),
                                      _stream(keys.device)))
        return out

    def sort_int32(self, keys: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """DialSort-Radix over the full signed int32 range."""
        _keys(keys)
        if out is None:
            out = torch.empty_like(keys)
        _check(_L.dialsort_sort_int32_async(self._h, _ptr(keys), keys.numel(), _ptr(out),
                                            _stream(keys.device)))
        return out

    def sort_host(self, keys_host: torch.Tensor, U: int, out_host: torch.Tensor | None = None,
                  wait: bool = True, stream=None) -> torch.Tensor:
        """End to end from host memory (pinned for speed); U == 0 selects the radix path.
        wait=False only enqueues (dialsort_sort_host_async): out_host is valid after sync()."""
        if keys_host.dtype != torch.int32 or keys_host.is_cuda or not keys_host.is_contiguous():
            raise ValueError("keys_host must be a contiguous int32 CPU tensor")
        if out_host is None:
            out_host = torch.empty_like(keys_host, pin_memory=keys_host.is_pinned())
        fn = _L.dialsort_sort_host if wait else _L.dialsort_sort_host_async
        s = _stream(self.device) if stream is None else ctypes.c_void_p(stream.cuda_stream)
        _check(fn(self._h, _ptr(keys_host), keys_host.numel(), int(U), _ptr(out_host), s))
        return out_host

    # -- multi-GPU exchange over peer memory (sharded.py drives these) ----------------------------
    def histogram_scatter(self, keys: torch.Tensor, U: int, G: int, rank: int, peers: torch.Tensor) -> None:
        """Local histogram, universe slice s stored into peers[s] (device int64 array of G device
        pointers to the owners' receive buffers) at slot `rank` (dialsort_histogram_scatter_async)."""
        keys = _keys(keys)
        if peers.dtype != torch.int64 or not peers.is_cuda or peers.numel() != G:
            raise ValueError("peers must be a device int64 tensor of G pointers")
        _check(_L.dialsort_histogram_scatter_async(self._h, _ptr(keys), keys.numel(), int(U), int(G), int(rank),
                                                   _ptr(peers), _stream(self.device)))

    def slice_sum(self, recv: torch.Tensor, G: int, L: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """out[j] = Σ_src recv[src * L + j] (uint32 counts carried in int32 tensors)."""
        if out is None:
            out = torch.empty(L, dtype=torch.int32, device=recv.device)
        _check(_L.dialsort_slice_sum_async(self._h, _ptr(recv), int(G), int(L), _ptr(out), _stream(self.device)))
        return out

    def ipc_handle(self, t: torch.Tensor) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _check(_L.dialsort_ipc_handle(self._h, ctypes.c_void_p(t.data_ptr()), buf))
        return buf.raw

    def ipc_open(self, handle: bytes) -> int:
        p = ctypes.c_void_p()
        _check(_L.dialsort_ipc_open(self._h, ctypes.create_string_buffer(handle, 64), ctypes.byref(p)))
        return int(p.value)

    def ipc_close(self, ptr: int) -> None:
        _check(_L.dialsort_ipc_close(self._h, ctypes.c_void_p(ptr)))

    def range_count(self, H: torch.Tensor, a: int, b: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """range-count(a, b) = Σ_{k=a}^{b} H[k] on the canonical state."""
        if out is None:
            out = torch.empty(1, dtype=torch.int64, device=H.device)
        _check(_L.dialsort_range_count_async(self._h, _ptr(H), H.numel(), int(a), int(b), _ptr(out),
                                             _stream(H.device)))
        return out

    # -- measurement hooks ---------------------------------------------------------------
    def profile(self, enable: bool) -> None:
        """Record an event pair around every kernel launch (breaks PDL overlap; timing only)."""
        _check(_L.dialsort_profile_enable(self._h, 1 if enable else 0))

    def profile_read(self, max_records: int = 1 << 16):
        """[(kernel name, ms)] recorded since the last read (call after the stream drained)."""
        import numpy as np
        ids = np.zeros(max_records, dtype=np.int32)
        ms = np.zeros(max_records, dtype=np.float32)
        n = _L.dialsort_profile_read(self._h, max_records, ids.ctypes.data_as(ctypes.c_void_p),
                                     ms.ctypes.data_as(ctypes.c_void_p))
        if n < 0:
            _check(-n)
        return [(_L.dialsort_kernel_name(int(i)).decode(), float(t)) for i, t in zip(ids[:n], ms[:n])]

    def debug_phase_ns(self):
        """Phase stamps of the fused kernel (DIALSORT_PHASE_TIMING=1), ns from the first CTA start:
        [latest CTA arrival at phase 0..7] + [earliest CTA arrival at phase 0..7]."""
        import numpy as np
        out = np.zeros(16, dtype=np.uint64)
        _check(_L.dialsort_debug_phase_ns(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        return out.tolist()

    def debug_phase_cta(self, max_ctas: int = 1024):
        """Per-CTA phase stamps (DIALSORT_PHASE_TIMING=1): rows [start, phase 0..15] in ns."""
        import numpy as np
        out = np.zeros((max_ctas, 17), dtype=np.uint64)
        n = _L.dialsort_debug_phase_cta(self._h, out.ctypes.data_as(ctypes.c_void_p), max_ctas)
        if n < 0:
            _check(-n)
        return out[:n]

    def crn_resolve(self, lane_keys: torch.Tensor, active: torch.Tensor):
        """Warp CRN test entry: (leader keys, leader counts) per 32-lane batch."""
        nb = active.numel()
        assert lane_keys.numel() == 32 * nb
        ok = torch.empty(32 * nb, dtype=torch.int32, device=lane_keys.device)
        oc = torch.empty(32 * nb, dtype=torch.int32, device=lane_keys.device)
        _check(_L.dialsort_crn_resolve_async(self._h, _ptr(lane_keys), _ptr(active), nb, _ptr(ok), _ptr(oc),
                                             _stream(lane_keys.device)))
        return ok, oc


_default_lock = threading.Lock()
_default: dict[int, Context] = {}


def default_context(device=None) -> Context:
    idx = torch.cuda.current_device() if device is None else (torch.device(device).index or 0)
    with _default_lock:
        if idx not in _default:
            _default[idx] = Context(idx)
        return _default[idx]


def histogram(keys: torch.Tensor, U: int, H: torch.Tensor | None = None, sync: bool = True):
    ctx = default_context(keys.device)
    H = ctx.histogram(keys, U, H)
    if sync:
        ctx.sync()
    return H


def reconstruct(H: torch.Tensor, out: torch.Tensor | None = None, n: int | None = None, key_base: int = 0,
                sync: bool = True):
    ctx = default_context(H.device)
    out = ctx.reconstruct(H, out, n, key_base)
    if sync:
        ctx.sync()
    return out


def sort(keys: torch.Tensor, U: int, out: torch.Tensor | None = None, H: torch.Tensor | None = None,
         sync: bool = True):
    ctx = default_context(keys.device)
    out = ctx.sort(keys, U, out, H)
    if sync:
        ctx.sync()
    return out


def sort_int32(keys: torch.Tensor, out: torch.Tensor | None = None, sync: bool = True):
    ctx = default_context(keys.device)
    out = ctx.sort_int32(keys, out)
    if sync:
        ctx.sync()
    return out


def sort_host(keys_host: torch.Tensor, U: int, out_host: torch.Tensor | None = None, device=None):
    return default_context(device).sort_host(keys_host, U, out_host)


def range_count(H: torch.Tensor, a: int, b: int):
    return default_context(H.device).range_count(H, a, b)


def crn_resolve(lane_keys: torch.Tensor, active: torch.Tensor):
    return default_context(lane_keys.device).crn_resolve(lane_keys, active)
