"""ctypes binding of libhpez_b200.so (include/hpez_b200.h).

The shared library is built in-tree by build.py.  There is no fallback:
if the library is missing or no CUDA device is present, every hot-path
call raises instead of silently computing on the CPU.
"""

from __future__ import annotations

import ctypes
import os

from . import errors

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libhpez_b200.so")
MAX_RANK = 5

OK, CORRUPT, UNDERFLOW, BADARG, CUDAERR, EMPTY, INVALID, TRUNC = range(8)
COMPRESS, DECOMPRESS = 0, 1
WORK_F32, WORK_F64 = 0, 1
CODES_U16, CODES_I32 = 0, 1


class Level(ctypes.Structure):
    _fields_ = [("stride", ctypes.c_int32), ("kernel", ctypes.c_int32),
                ("paradigm", ctypes.c_int32), ("n_order", ctypes.c_int32),
                ("axis_order", ctypes.c_int32 * MAX_RANK), ("bound", ctypes.c_double)]


class SweepDesc(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("dims", ctypes.c_int64 * MAX_RANK),
                ("frozen_mask", ctypes.c_uint32), ("direction", ctypes.c_int32),
                ("rounding", ctypes.c_int32), ("radius", ctypes.c_int64),
                ("n_levels", ctypes.c_int32), ("levels", ctypes.POINTER(Level)),
                ("md_alpha", ctypes.POINTER(ctypes.c_double)),
                ("block_size", ctypes.c_int32), ("block_table", ctypes.c_void_p),
                ("work_dtype", ctypes.c_int32), ("code_dtype", ctypes.c_int32),
                ("with_stats", ctypes.c_int32)]


_lib = None


def lib():
    """Load the native library (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build as _build
    if not _build.up_to_date():
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"native library missing: {LIB_PATH}")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    sig = {
        "hpez_plan_create": (I32, [ctypes.POINTER(SweepDesc), ctypes.POINTER(P)]),
        "hpez_plan_destroy": (I32, [P]),
        "hpez_plan_num_codes": (I64, [P]),
        "hpez_plan_num_commits": (I32, [P]),
        "hpez_plan_num_launches": (I32, [P]),
        "hpez_plan_level_codes": (I32, [P, P]),
        "hpez_plan_info": (I32, [P, P]),
        "hpez_plan_workspace_size": (I32, [P, P]),
        "hpez_plan_bind_workspace": (I32, [P, P, I64]),
        "hpez_plan_commit_stats": (I32, [P, P, I32]),
        "hpez_plan_levels_timeline": (I32, [P, P]),
        "hpez_sweep_run": (I32, [P, P, P, I64, P, I64, P, P, P, P]),
        "hpez_sweep_run_from": (I32, [P, P, P, P, I64, P, I64, P]),
        "hpez_plan_tile_info": (I32, [P, P, I32]),
        "hpez_plan_row_info": (I32, [P, P]),
        "hpez_sweep_finish": (I32, [P, P, ctypes.POINTER(I64)]),
        "hpez_lorenzo": (I32, [I32, P, I32, P, ctypes.c_double, I64, I32, I32, I32, I32, P,
                               I64, P, I64, ctypes.POINTER(I64), P]),
        "hpez_histogram": (I32, [P, I32, I64, P, I64, P]),
        "hpez_huffman_table": (I32, [P, I64, P, P]),
        "hpez_huffman_nbits": (I32, [P, I32, I64, P, ctypes.POINTER(I64), P]),
        "hpez_huffman_pack": (I32, [P, I32, I64, P, P, I32, P, I64, P]),
        "hpez_huffman_decode": (I32, [P, I64, P, I64, I64, P]),
        "hpez_huffman_decode_device": (I32, [P, P, I64, P, I64, I64, P, I32, P]),
        "hpez_rows_pairwise_sum": (I32, [P, I64, I64, P, P]),
        "hpez_reduce_scratch_bytes": (I64, []),
        "hpez_pairwise_sum": (I32, [P, I64, P, P, P]),
        "hpez_sample_stats": (I32, [P, I32, I32, P, P, P, I64, U32, U32, P, P, P]),
        "hpez_sq_diff_sum": (I32, [P, I32, P, I32, I64, P, P, P]),
        "hpez_uniform_filter1d": (I32, [P, P, I32, P, I32, I32, P]),
        "hpez_ssim_prep": (I32, [P, I32, P, I32, I64, P, P, P, P, P, P]),
        "hpez_ssim_terms": (I32, [P, P, P, P, P, I32, P, P, P, ctypes.c_double, ctypes.c_double, P, P]),
        "hpez_set_device": (I32, [I32]),
        "hpez_build_info": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int, what: str = "") -> None:
    """Map an hpez_status onto the reference's exception types."""
    if status == OK:
        return
    msg = f"{what}: status {status}" if what else f"status {status}"
    if status == CORRUPT:
        raise errors.CorruptStream(msg)
    if status == UNDERFLOW:
        raise errors.OutlierUnderflow(msg)
    if status == EMPTY:
        raise errors.EmptyInput(msg)
    if status == INVALID:
        raise errors.InvalidTable(msg)
    if status == TRUNC:
        raise errors.TruncatedStream(msg)
    if status == BADARG:
        raise ValueError(msg)
    raise RuntimeError(f"CUDA failure in {msg}")
