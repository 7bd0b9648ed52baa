"""ctypes binding of include/fvlog.h (libfvlog.so, built in-tree for sm_100a).

There is deliberately no fallback: if the shared library is missing the
import of any operator fails loudly with the build command to run.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# FVLOG_LIB: load another build of the library (kernel-variant experiments).
LIB_PATH = os.environ.get("FVLOG_LIB") or os.path.join(_HERE, "libfvlog.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p
st = C.c_int  # fv_status


class FvError(RuntimeError):
    """Base class; `status` is the fv_status code."""

    status = 0


class ArityError(FvError, ValueError):
    """std::invalid_argument in the reference (arity/length mismatch)."""

    status = 1


class RangeError(FvError, IndexError):
    """std::out_of_range in the reference."""

    status = 2


class LengthError(FvError):
    """std::length_error in the reference (> 2^32 rows)."""

    status = 3


class DiagnosticError(FvError):
    """colog::DiagnosticError (parse / validate / compile)."""

    status = 4


class FvIOError(FvError, OSError):
    status = 5


class DeviceOOM(FvError, MemoryError):
    status = 6


class CudaError(FvError):
    status = 7


class InvalidArgument(FvError):
    status = 8


_BY_STATUS = {c.status: c for c in (ArityError, RangeError, LengthError, DiagnosticError,
                                     FvIOError, DeviceOOM, CudaError, InvalidArgument)}

# (name, restype, argtypes)
_SIGNATURES = [
    ("fv_abi_version", C.c_int, []),
    ("fv_global_error", C.c_char_p, []),
    ("fv_ctx_create", st, [C.c_int, C.POINTER(vp)]),
    ("fv_ctx_destroy", None, [vp]),
    ("fv_last_error", C.c_char_p, [vp]),
    ("fv_ctx_synchronize", st, [vp]),
    ("fv_ctx_kernel_launches", C.c_uint64, [vp]),
    ("fv_ctx_host_syncs", C.c_uint64, [vp]),
    ("fv_gather_volume", C.c_uint64, []),
    ("fv_reset_gather_volume", None, []),
    ("fv_array_size", C.c_uint64, [vp]),
    ("fv_array_elem_bytes", C.c_uint32, [vp]),
    ("fv_array_read", st, [vp, vp]),
    ("fv_array_free", None, [vp]),
    ("fv_column_build", st, [vp, u32p, C.c_uint64, C.POINTER(vp)]),
    ("fv_column_free", None, [vp]),
    ("fv_column_size", C.c_uint64, [vp]),
    ("fv_column_unique_count", C.c_uint64, [vp]),
    ("fv_column_read", st, [vp, u32p, u32p]),
    ("fv_column_read_unique", st, [vp, u32p, u32p, u32p]),
    ("fv_column_probe", st, [vp, C.c_uint32, u32p, u32p, C.POINTER(C.c_int)]),
    ("fv_column_probe_many", st, [vp, u32p, C.c_uint64, u32p, u32p, u8p]),
    ("fv_column_gather", st, [vp, u32p, C.c_uint64, u32p]),
    ("fv_column_append_and_reindex", st, [vp, u32p, C.c_uint64, C.POINTER(vp)]),
    ("fv_build_index", st, [vp, u32p, C.c_uint64, u32p, u32p, u32p, u32p, u64p]),
    ("fv_version_from_columns", st, [vp, C.c_uint32, C.POINTER(u32p), C.c_uint64, C.POINTER(vp)]),
    ("fv_version_decompose", st, [vp, C.c_uint32, u32p, C.c_uint64, C.POINTER(vp)]),
    ("fv_version_empty", st, [vp, C.c_uint32, C.POINTER(vp)]),
    ("fv_version_free", None, [vp]),
    ("fv_version_arity", C.c_uint32, [vp]),
    ("fv_version_rows", C.c_uint64, [vp]),
    ("fv_version_col", vp, [vp, C.c_uint32]),
    ("fv_version_reconstruct", st, [vp, u32p]),
    ("fv_version_append", st, [vp, vp, C.POINTER(vp)]),
    ("fv_dedup_rows", st, [vp, C.POINTER(vp)]),
    ("fv_has_duplicate_rows", st, [vp, C.POINTER(C.c_int)]),
    ("fv_relation_create", st, [vp, C.c_char_p, C.c_uint32, C.POINTER(vp)]),
    ("fv_relation_free", None, [vp]),
    ("fv_relation_full", vp, [vp]),
    ("fv_relation_delta", vp, [vp]),
    ("fv_relation_new", vp, [vp]),
    ("fv_relation_set_full", st, [vp, vp]),
    ("fv_relation_merge_delta", st, [vp, vp]),
    ("fv_select_eq", st, [vp, C.c_uint32, C.POINTER(vp)]),
    ("fv_project", st, [vp, u32p, C.c_uint64, u32p, C.c_uint32, C.POINTER(vp)]),
    ("fv_join_probe_phase", st, [vp, u32p, C.c_uint64, vp, C.POINTER(vp)]),
    ("fv_match_create", st, [vp, u32p, u32p, u32p, C.c_uint64, C.POINTER(vp)]),
    ("fv_match_free", None, [vp]),
    ("fv_match_size", C.c_uint64, [vp]),
    ("fv_match_read", st, [vp, u32p, u32p, u32p]),
    ("fv_join_total_size", st, [vp, u64p]),
    ("fv_join_offsets", st, [vp, u64p]),
    ("fv_join_write_phase", st, [vp, vp, C.POINTER(vp), C.POINTER(vp)]),
    ("fv_column_join", st, [vp, u32p, C.c_uint64, vp, C.POINTER(vp), C.POINTER(vp)]),
    ("fv_filter_pairs_eq", st, [vp, u32p, u32p, C.c_uint64, vp, vp, C.POINTER(vp), C.POINTER(vp)]),
    ("fv_filter_neq", st, [vp, C.c_uint32, C.c_uint32, C.POINTER(vp)]),
    ("fv_deduplicate", st, [vp, vp, C.POINTER(vp)]),
    ("fv_difference", st, [vp, u8p, C.c_uint64, C.POINTER(vp)]),
    ("fv_union_concat", st, [vp, vp, C.POINTER(vp)]),
]

_lib = None


def lib() -> C.CDLL:
    """Load libfvlog.so (no fallback: missing library is an error)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the fvlog CUDA runtime has not been built. "
            "Run `python -c 'import __graft_entry__ as g; g.build()'` (or `make`) at the repo root.")
    l = C.CDLL(LIB_PATH)
    for name, res, args in _SIGNATURES:
        fn = getattr(l, name, None)
        if fn is None:
            continue  # declared later in the ABI; bound lazily by the module that needs it
        fn.restype = res
        fn.argtypes = args
    _lib = l
    return l


def bind(name: str, restype, argtypes):
    fn = getattr(lib(), name)
    fn.restype = restype
    fn.argtypes = argtypes
    return fn


def check(status: int, ctx=None) -> None:
    if status == 0:
        return
    l = lib()
    msg = (l.fv_last_error(ctx) if ctx else l.fv_global_error()) or b""
    raise _BY_STATUS.get(status, FvError)(msg.decode(errors="replace"))
