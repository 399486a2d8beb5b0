"""ctypes loader for libdialsort.so (the C ABI declared in include/dialsort.h).

Argument marshalling only: every step of the method runs in the CUDA kernels behind the
C ABI.  There is no fallback: if the shared library is missing or fails to load, importing
this module raises, so a GPU run can never silently use another implementation.
"""
from __future__ import annotations

import ctypes
import os

_DIR = os.path.dirname(os.path.abspath(__file__))
# DIALSORT_LIB_VARIANT=<v> loads libdialsort_<v>.so from this directory instead (design A/B
# builds of the same sources with different -D switches; development only)
_VARIANT = os.environ.get("DIALSORT_LIB_VARIANT", "")
LIB_PATH = os.path.join(_DIR, f"libdialsort_{_VARIANT}.so" if _VARIANT else "libdialsort.so")

# dialsort_status
OK, E_INVALID_ARG, E_KEY_RANGE, E_SIZE, E_OVERFLOW, E_CUDA, E_COMM, E_NOMEM = 0, 1, 2, 3, 4, 5, 6, 7
# context options, query ops, communicator handle size (include/dialsort.h)
(OPT_RADIX_VARIANT, OPT_RADIX_PROBE_VIOLATIONS, OPT_RADIX_ACTIVE, OPT_NUM_SMS, OPT_COOPERATIVE, OPT_MAX_CTAS,
 OPT_PART_MODE) = 1, 2, 3, 4, 5, 6, 7
Q_FREQUENCY, Q_PRESENCE, Q_RANGE_COUNT = 0, 1, 2
COMM_HANDLE_BYTES = 128

EXPORTS = (
    "dialsort_status_string", "dialsort_last_error", "dialsort_version",
    "dialsort_ctx_create", "dialsort_ctx_destroy", "dialsort_sync",
    "dialsort_histogram_async", "dialsort_reconstruct_async", "dialsort_sort_async",
    "dialsort_sort_int32_async", "dialsort_histogram", "dialsort_reconstruct",
    "dialsort_sort", "dialsort_sort_int32", "dialsort_sort_host", "dialsort_sort_host_async",
    "dialsort_range_count_async", "dialsort_query_async", "dialsort_support_set_async",
    "dialsort_crn_resolve_async", "dialsort_ctx_set_option", "dialsort_ctx_get_option",
    "dialsort_debug_radix_passes", "dialsort_sort_domain_async", "dialsort_sort_batch_async",
    "dialsort_comm_create", "dialsort_comm_connect_ipc", "dialsort_comm_connect_local",
    "dialsort_comm_destroy", "dialsort_comm_info",
    "dialsort_sharded_histogram_scatter_async", "dialsort_sharded_histogram_gather_async",
    "dialsort_sharded_project_async", "dialsort_sharded_sort_async",
    "dialsort_sharded_radix_hist_async", "dialsort_sharded_radix_split_async",
    "dialsort_sharded_radix_local_async", "dialsort_sharded_sort_int32_async",
    "dialsort_sharded_sort", "dialsort_sharded_sort_int32",
    "dialsort_profile_enable", "dialsort_profile_read", "dialsort_kernel_name",
    "dialsort_debug_phase_ns", "dialsort_debug_phase_cta",
)


class ErrorInfo(ctypes.Structure):
    _fields_ = [
        ("bad_count", ctypes.c_uint64),
        ("first_bad_index", ctypes.c_uint64),
        ("first_bad_key", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("last_total", ctypes.c_uint64),
    ]


def load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the DialSort product path has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, u64, u32, i32, ci = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int
    i64 = ctypes.c_int64
    sig = {
        "dialsort_status_string": ([ci], ctypes.c_char_p),
        "dialsort_last_error": ([], ctypes.c_char_p),
        "dialsort_version": ([], ci),
        "dialsort_ctx_create": ([ci, u64, u32, ctypes.POINTER(P)], ci),
        "dialsort_ctx_destroy": ([P], ci),
        "dialsort_sync": ([P, P, ctypes.POINTER(ErrorInfo)], ci),
        "dialsort_histogram_async": ([P, P, u64, u32, P, P], ci),
        "dialsort_reconstruct_async": ([P, P, u32, i32, P, u64, ci, P, P], ci),
        "dialsort_sort_async": ([P, P, u64, u32, P, P, P], ci),
        "dialsort_sort_int32_async": ([P, P, u64, P, P], ci),
        "dialsort_histogram": ([P, u64, u32, P], ci),
        "dialsort_reconstruct": ([P, u32, P, u64], ci),
        "dialsort_sort": ([P, u64, u32, P], ci),
        "dialsort_sort_int32": ([P, u64, P], ci),
        "dialsort_sort_host": ([P, P, u64, u32, P, P], ci),
        "dialsort_sort_host_async": ([P, P, u64, u32, P, P], ci),
        "dialsort_range_count_async": ([P, P, u32, u32, u32, P, P], ci),
        "dialsort_query_async": ([P, P, u32, ci, P, u64, P, P], ci),
        "dialsort_support_set_async": ([P, P, u32, P, P, P, P], ci),
        "dialsort_crn_resolve_async": ([P, P, P, u64, P, P, P], ci),
        "dialsort_ctx_set_option": ([P, ci, i64], ci),
        "dialsort_ctx_get_option": ([P, ci, ctypes.POINTER(i64)], ci),
        "dialsort_debug_radix_passes": ([P, P, u64, P, P], ci),
        "dialsort_sort_domain_async": ([P, P, ci, u64, u32, P, P, P, P], ci),
        "dialsort_sort_batch_async": ([P, P, P, u32, P, P, u32, P], ci),
        "dialsort_comm_create": ([P, u32, u32, u32, u64, P, ctypes.POINTER(P)], ci),
        "dialsort_comm_connect_ipc": ([P, P], ci),
        "dialsort_comm_connect_local": ([P, P], ci),
        "dialsort_comm_destroy": ([P], ci),
        "dialsort_comm_info": ([P, P, P, P], ci),
        "dialsort_sharded_histogram_scatter_async": ([P, P, P, u64, u32, P], ci),
        "dialsort_sharded_histogram_gather_async": ([P, P, u32, P, P], ci),
        "dialsort_sharded_project_async": ([P, P, u32, P, P, u64, P, P, P], ci),
        "dialsort_sharded_sort_async": ([P, P, P, u64, u32, P, u64, P, P, P, P], ci),
        "dialsort_sharded_radix_hist_async": ([P, P, P, u64, P], ci),
        "dialsort_sharded_radix_split_async": ([P, P, P, u64, u64, P, P, P], ci),
        "dialsort_sharded_radix_local_async": ([P, P, P, u64, P], ci),
        "dialsort_sharded_sort_int32_async": ([P, P, P, u64, P, u64, P, P, P], ci),
        "dialsort_sharded_sort": ([P, P, P, u64, u32, P, u64, P, P, P], ci),
        "dialsort_sharded_sort_int32": ([P, P, P, u64, P, u64, P, P, P], ci),
        "dialsort_profile_enable": ([P, ci], ci),
        "dialsort_profile_read": ([P, ci, P, P], ci),
        "dialsort_kernel_name": ([ci], ctypes.c_char_p),
        "dialsort_debug_phase_ns": ([P, P], ci),
        "dialsort_debug_phase_cta": ([P, P, ci], ci),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = load()
