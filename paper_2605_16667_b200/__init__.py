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
    "DialSortError", "Context", "Comm", "histogram", "reconstruct", "sort", "sort_int32", "sort_host",
    "range_count", "frequency", "presence", "support_set", "crn_resolve", "default_context", "LIB_PATH",
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


def _dev_buf(t: torch.Tensor | None, name: str, like: torch.Tensor, min_numel: int,
             dtypes=(torch.int32,)) -> torch.Tensor | None:
    """Caller-provided device buffer: contiguous, of an allowed dtype, on `like`'s device, large
    enough (the C ABI takes raw pointers: a short buffer would be overrun on the device)."""
    if t is None:
        return None
    if t.dtype not in dtypes or not t.is_cuda or not t.is_contiguous() or t.device != like.device:
        raise ValueError(f"{name} must be a contiguous {'/'.join(str(d) for d in dtypes)} tensor on {like.device}")
    if t.numel() < min_numel:
        raise ValueError(f"{name} holds {t.numel()} elements, needs >= {min_numel}")
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
        _dev_buf(H, "H", keys, int(U))
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
            if n is None:  # ΣH by the library (range-count over the whole universe), read back to size out
                tot = self.range_count(H, 0, H.numel() - 1)
                n = int(tot.item())
            out = torch.empty(int(n), dtype=torch.int32, device=H.device)
        cap = out.numel() if n is None else int(n)
        _dev_buf(out, "out", H, cap)
        _dev_buf(d_total, "d_total", H, 1, (torch.int64,))
        _check(_L.dialsort_reconstruct_async(self._h, _ptr(H), H.numel(), int(key_base), _ptr(out), cap,
                                             1 if exact else 0, _ptr(d_total), _stream(H.device)))
        return out

    def sort(self, keys: torch.Tensor, U: int, out: torch.Tensor | None = None,
             H: torch.Tensor | None = None) -> torch.Tensor:
        """DialSort of keys in [0, U); out may be keys itself (in place)."""
        _keys(keys)
        if out is None:
            out = torch.empty_like(keys)
        _dev_buf(out, "out", keys, keys.numel())
        _dev_buf(H, "H", keys, int(U))
        _check(_L.dialsort_sort_async(self._h, _ptr(keys), keys.numel(), int(U), _ptr(out), _ptr(H),
                                      _stream(keys.device)))
        return out

    def sort_batch(self, keys_list, U: int, outs=None, Hs=None):
        """Independent DialSorts of several key batches in one call (dialsort_sort_batch_async):
        overlapped in one launch on disjoint CTA groups when U <= 98304."""
        nb = len(keys_list)
        for k in keys_list:
            _keys(k)
        if outs is None:
            outs = [torch.empty_like(k) for k in keys_list]
        for k, o in zip(keys_list, outs):
            _dev_buf(o, "out", k, k.numel())
        if Hs is not None:
            for k, h in zip(keys_list, Hs):
                _dev_buf(h, "H", k, int(U))
        P = ctypes.c_void_p
        kp = (P * nb)(*[k.data_ptr() for k in keys_list])
        ns = (ctypes.c_uint64 * nb)(*[k.numel() for k in keys_list])
        op = (P * nb)(*[o.data_ptr() for o in outs])
        hp = None if Hs is None else (P * nb)(*[h.data_ptr() for h in Hs])
        _check(_L.dialsort_sort_batch_async(self._h, kp, ns, int(U), op, hp, nb, _stream(keys_list[0].device)))
        return outs

    def sort_int32(self, keys: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """DialSort-Radix over the full signed int32 range."""
        _keys(keys)
        if out is None:
            out = torch.empty_like(keys)
        _dev_buf(out, "out", keys, keys.numel())
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

    # -- options -------------------------------------------------------------------------
    def set_option(self, option: int, value: int) -> None:
        _check(_L.dialsort_ctx_set_option(self._h, int(option), int(value)))

    def get_option(self, option: int) -> int:
        v = ctypes.c_int64()
        _check(_L.dialsort_ctx_get_option(self._h, int(option), ctypes.byref(v)))
        return int(v.value)

    @property
    def radix_variant(self) -> int:
        """The radix pass in use for aligned buffers: 4 (TMA, ranks from the counting atomic; only
        on a device that passed the lane-order probe) or 3 (equality-grouped ranks)."""
        return self.get_option(_lib.OPT_RADIX_ACTIVE)

    def sort_domain(self, items: torch.Tensor, U: int, encode: torch.Tensor | None = None,
                    decode: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
        """Proposition 2: sort items of a finite ordered domain through phi (encode:
        uint8 -> code table of 256 entries, uint8 items only; None = identity) and emit phi^-1
        (decode: int32[U] table; None = the code).  items: uint8 / int16 (uint16 bits) / int32."""
        widths = {torch.uint8: 1, torch.int16: 2, torch.uint16: 2, torch.int32: 4}
        if items.dtype not in widths or not items.is_cuda or not items.is_contiguous():
            raise ValueError("items must be a contiguous uint8 / (u)int16 / int32 CUDA tensor")
        if out is None:
            out = torch.empty(items.numel(), dtype=torch.int32, device=items.device)
        _dev_buf(out, "out", items, items.numel())
        _dev_buf(encode, "encode", items, 256, (torch.int32,))
        _dev_buf(decode, "decode", items, int(U), (torch.int32,))
        _check(_L.dialsort_sort_domain_async(self._h, _ptr(items), widths[items.dtype], items.numel(), int(U),
                                             _ptr(encode), _ptr(decode), _ptr(out), _stream(items.device)))
        return out

    def debug_radix_passes(self, keys: torch.Tensor) -> torch.Tensor:
        """The 4 pass buffers of DialSort-Radix (uint32 bits in an int32 [4, n] tensor): passes
        0..2 biased keys, pass 3 the sorted int32 keys (dialsort_debug_radix_passes)."""
        _keys(keys)
        n = keys.numel()
        out = torch.empty((4, max(n, 1)), dtype=torch.int32, device=keys.device)
        _check(_L.dialsort_debug_radix_passes(self._h, _ptr(keys), n, _ptr(out), _stream(keys.device)))
        return out[:, :n]

    def range_count(self, H: torch.Tensor, a: int, b: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """range-count(a, b) = Σ_{k=a}^{b} H[k] on the canonical state."""
        if out is None:
            out = torch.empty(1, dtype=torch.int64, device=H.device)
        _dev_buf(out, "out", H, 1, (torch.int64,))
        _check(_L.dialsort_range_count_async(self._h, _ptr(H), H.numel(), int(a), int(b), _ptr(out),
                                             _stream(H.device)))
        return out

    def query(self, H: torch.Tensor, op: int, q: torch.Tensor) -> torch.Tensor:
        """Batched canonical-state queries (dialsort_query_async): op Q_FREQUENCY / Q_PRESENCE with
        m keys, or Q_RANGE_COUNT with m (a, b) pairs (q shaped [m, 2]); int64 answers."""
        if q.dtype != torch.int32 or not q.is_cuda or not q.is_contiguous():
            raise ValueError("q must be a contiguous int32 CUDA tensor")
        m = q.numel() // 2 if op == _lib.Q_RANGE_COUNT else q.numel()
        out = torch.empty(max(m, 1), dtype=torch.int64, device=H.device)
        _check(_L.dialsort_query_async(self._h, _ptr(H), H.numel(), int(op), _ptr(q), m, _ptr(out),
                                       _stream(H.device)))
        return out[:m]

    def support_set(self, H: torch.Tensor):
        """(D, |D|, iso) on the device: D ascending occupied cells, iso = 1 iff D is
        the whole universe (prop:iso).  D is valid in its first |D| entries."""
        U = H.numel()
        D = torch.empty(max(U, 1), dtype=torch.int32, device=H.device)
        cnt = torch.zeros(1, dtype=torch.int64, device=H.device)
        iso = torch.zeros(1, dtype=torch.int32, device=H.device)
        _check(_L.dialsort_support_set_async(self._h, _ptr(H), U, _ptr(D), _ptr(cnt), _ptr(iso), _stream(H.device)))
        return D, cnt, iso

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


class Comm:
    """A multi-GPU communicator (dialsort_comm) of one rank: a symmetric device workspace mapped
    into every rank.  Build it with `create`, exchange `handle` bytes between the ranks (any host
    channel), then `connect_ipc(all_handles)`; or, for several ranks in one process (the one-GPU
    loopback harness), `connect_local(comms)`."""

    def __init__(self, ctx: Context, G: int, rank: int, max_U: int, max_recv_keys: int = 0):
        self.ctx, self.G, self.rank = ctx, int(G), int(rank)
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(_lib.COMM_HANDLE_BYTES)
        with torch.cuda.device(ctx.device):
            _check(_L.dialsort_comm_create(ctx._h, self.G, self.rank, int(max_U), int(max_recv_keys), buf,
                                           ctypes.byref(h)))
        self._h = h
        self.handle = buf.raw

    def connect_ipc(self, handles) -> None:
        blob = b"".join(handles)
        _check(_L.dialsort_comm_connect_ipc(self._h, ctypes.create_string_buffer(blob, len(blob))))

    def connect_local(self, comms) -> None:
        arr = (ctypes.c_void_p * len(comms))(*[c._h.value for c in comms])
        _check(_L.dialsort_comm_connect_local(self._h, arr))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _L.dialsort_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def epoch(self) -> int:
        e = ctypes.c_uint32()
        _check(_L.dialsort_comm_info(self._h, None, None, ctypes.byref(e)))
        return int(e.value)

    def _s(self):
        return _stream(self.ctx.device)

    # histogram path (step by step, or sort = scatter + gather + project)
    def scatter(self, keys: torch.Tensor, U: int) -> None:
        _keys(keys)
        _check(_L.dialsort_sharded_histogram_scatter_async(self.ctx._h, self._h, _ptr(keys), keys.numel(), int(U),
                                                           self._s()))

    def gather(self, U: int, H_slice: torch.Tensor | None = None) -> torch.Tensor | None:
        """H_slice (uint32[U/G] as int32) = Σ of the G slots; None: the communicator's own buffer
        (what `project(U, None, ...)` reads)."""
        if H_slice is not None:
            _dev_buf(H_slice, "H_slice", H_slice, int(U) // self.G)
        _check(_L.dialsort_sharded_histogram_gather_async(self.ctx._h, self._h, int(U), _ptr(H_slice), self._s()))
        return H_slice

    def project(self, U: int, H_slice: torch.Tensor | None, out: torch.Tensor, count: torch.Tensor,
                offset: torch.Tensor) -> None:
        _check(_L.dialsort_sharded_project_async(self.ctx._h, self._h, int(U), _ptr(H_slice), _ptr(out), out.numel(),
                                                 _ptr(count), _ptr(offset), self._s()))

    def sort(self, keys: torch.Tensor, U: int, out: torch.Tensor, count: torch.Tensor, offset: torch.Tensor,
             H_slice: torch.Tensor | None = None) -> None:
        """Sharded DialSort of this rank's key shard: out[:count] = sorted keys of universe slice
        `rank`, *offset = its position in the global order (all on the device, no host sync)."""
        _keys(keys)
        _check(_L.dialsort_sharded_sort_async(self.ctx._h, self._h, _ptr(keys), keys.numel(), int(U), _ptr(out),
                                              out.numel(), _ptr(H_slice), _ptr(count), _ptr(offset), self._s()))

    # radix path
    def radix_hist(self, keys: torch.Tensor) -> None:
        _keys(keys)
        _check(_L.dialsort_sharded_radix_hist_async(self.ctx._h, self._h, _ptr(keys), keys.numel(), self._s()))

    def radix_split(self, keys: torch.Tensor, cap: int, count: torch.Tensor, offset: torch.Tensor) -> None:
        _keys(keys)
        _check(_L.dialsort_sharded_radix_split_async(self.ctx._h, self._h, _ptr(keys), keys.numel(), int(cap),
                                                     _ptr(count), _ptr(offset), self._s()))

    def radix_local(self, out: torch.Tensor) -> None:
        _check(_L.dialsort_sharded_radix_local_async(self.ctx._h, self._h, _ptr(out), out.numel(), self._s()))

    def sort_int32(self, keys: torch.Tensor, out: torch.Tensor, count: torch.Tensor, offset: torch.Tensor) -> None:
        """Sharded DialSort-Radix: out[:count] = this rank's contiguous part of the sorted array."""
        _keys(keys)
        _check(_L.dialsort_sharded_sort_int32_async(self.ctx._h, self._h, _ptr(keys), keys.numel(), _ptr(out),
                                                    out.numel(), _ptr(count), _ptr(offset), self._s()))


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


def frequency(H: torch.Tensor, keys: torch.Tensor):
    return default_context(H.device).query(H, _lib.Q_FREQUENCY, keys)


def presence(H: torch.Tensor, keys: torch.Tensor):
    return default_context(H.device).query(H, _lib.Q_PRESENCE, keys)


def support_set(H: torch.Tensor):
    return default_context(H.device).support_set(H)


def crn_resolve(lane_keys: torch.Tensor, active: torch.Tensor):
    return default_context(lane_keys.device).crn_resolve(lane_keys, active)
