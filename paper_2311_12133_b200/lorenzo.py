"""Drop-in for lorenzo.lorenzo_pass (lorenzo.py:145-179) on the GPU.

The raster scan runs as one hyperplane wavefront launch per sum(coords)
(csrc/lorenzo.cu); codes stay in raster order and outliers are compacted in
raster order, so streams match the reference's numba scan bit for bit."""

from __future__ import annotations

import ctypes
import itertools

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .device import bind, device, ptr, stream
from .errors import CorruptStream
from .interp import code_dtype_for, codes_to_int32, f32_exact, torch_code_dtype
from .quant import ROUND_F32, ROUND_NONE


def build_stencil(rank: int, order: int):
    """Backward offsets (n, rank) and coefficients -prod(w[o_i]) (lorenzo.py:24-41)."""
    if order not in (1, 2):
        raise ValueError(f"order must be 1 or 2, got {order}")
    if rank < 1:
        raise ValueError(f"rank must be >= 1, got {rank}")
    w = (1.0, -1.0) if order == 1 else (1.0, -2.0, 1.0)
    offs, coefs = [], []
    for o in itertools.product(range(order + 1), repeat=rank):
        if any(o):
            c = -1.0
            for oi in o:
                c *= w[oi]
            offs.append(o)
            coefs.append(c)
    return np.array(offs, dtype=np.int64), np.array(coefs, dtype=np.float64)


def lorenzo_pass_device(work, bound, radius, order, *, direction, rounding=ROUND_NONE,
                        codes=None, outliers=None):
    """Device-resident Lorenzo sweep.  Compress returns (codes, outliers,
    n_outliers); decompress consumes codes/outliers and returns the number
    of outliers used."""
    if direction not in ("compress", "decompress"):
        raise ValueError(f"bad direction {direction!r}")
    if order not in (1, 2):
        raise ValueError(f"order must be 1 or 2, got {order}")
    dev = device()
    if not work.is_cuda or not work.is_contiguous() or work.dtype not in (torch.float32, torch.float64):
        raise ValueError("work must be a contiguous float32/float64 CUDA tensor")
    wdt = _lib.WORK_F32 if work.dtype == torch.float32 else _lib.WORK_F64
    dims = np.array(work.shape, dtype=np.int64)
    n_out = ctypes.c_int64(0)
    bind()
    if direction == "compress":
        cdt = code_dtype_for(radius)
        codes = torch.empty(max(work.numel(), 1), dtype=torch_code_dtype(cdt), device=dev)
        outliers = torch.empty(max(work.numel(), 1), dtype=torch.float64, device=dev)
        check(lib().hpez_lorenzo(work.dim(), dims.ctypes.data, wdt, ptr(work), float(bound),
                                 int(radius), int(order), _lib.COMPRESS, int(rounding), cdt,
                                 ptr(codes), work.numel(), ptr(outliers), outliers.numel(),
                                 ctypes.byref(n_out), stream()), "hpez_lorenzo")
        return codes[:work.numel()], outliers, n_out.value
    if codes is None or outliers is None:
        raise ValueError("decompression needs codes and outliers")
    cdt = _lib.CODES_U16 if codes.dtype == torch.uint16 else _lib.CODES_I32
    check(lib().hpez_lorenzo(work.dim(), dims.ctypes.data, wdt, ptr(work), float(bound),
                             int(radius), int(order), _lib.DECOMPRESS, int(rounding), cdt,
                             ptr(codes), codes.numel(), ptr(outliers), outliers.numel(),
                             ctypes.byref(n_out), stream()), "hpez_lorenzo")
    return n_out.value


def codes_to_device(codes: np.ndarray, radius: int):
    """Host int codes -> device u16 (when they fit) or i32 tensor."""
    dev = device()
    codes = np.asarray(codes)
    if radius <= 32768 and (codes.size == 0 or (codes.min() >= 0 and codes.max() <= 65535)):
        return torch.from_numpy(codes.astype(np.uint16)).to(dev)
    return torch.from_numpy(np.ascontiguousarray(codes, dtype=np.int32)).to(dev)


def lorenzo_pass(work: np.ndarray, bound: float, radius: int, order: int, *, direction: str,
                 rounding: int = ROUND_NONE, codes=None, outliers=None):
    """Reference signature (lorenzo.py:145-148): ``work`` float64 C-order is
    updated in place; compress returns (codes int32, outliers float64)."""
    dev = device()
    if direction == "compress":
        use_f32 = rounding == ROUND_F32 and f32_exact(work)
        wt = torch.from_numpy(work.astype(np.float32) if use_f32 else work).to(dev)
        c, o, n = lorenzo_pass_device(wt, bound, radius, order, direction="compress",
                                      rounding=rounding)
        work[...] = wt.cpu().numpy().astype(np.float64)
        return codes_to_int32(c), o[:n].cpu().numpy()
    if direction != "decompress":
        raise ValueError(f"bad direction {direction!r}")
    if codes is None or outliers is None:
        raise ValueError("decompression needs codes and outliers")
    codes = np.ascontiguousarray(codes, dtype=np.int32)
    if codes.size != work.size:
        raise CorruptStream(f"code stream has {codes.size} entries for {work.size} points")
    outliers = np.ascontiguousarray(outliers, dtype=np.float64)
    use_f32 = rounding == ROUND_F32 and f32_exact(work) and f32_exact(outliers)
    wt = torch.from_numpy(work.astype(np.float32) if use_f32 else work).to(dev)
    ot = torch.from_numpy(outliers if outliers.size else np.zeros(1)).to(dev)
    if not outliers.size:
        ot = ot[:0]
    lorenzo_pass_device(wt, bound, radius, order, direction="decompress", rounding=rounding,
                        codes=codes_to_device(codes, radius), outliers=ot)
    work[...] = wt.cpu().numpy().astype(np.float64)
    return None
