"""Reconstruction quality on the GPU: the reference's psnr / ssim / evaluate
/ sweep (metrics.py:36-166) with the same API and bit-identical values.

The reductions follow numpy's pairwise summation and the SSIM windows are
scipy.ndimage.uniform_filter's running sums (csrc/metrics.cu), so a
rate-distortion sweep (compress + decompress + evaluate per error bound)
never leaves the device except for the scalar results.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import check, lib
from .devgrid import device_grid, reduce_scratch
from .device import bind, ptr, stream
from .errors import DimsMismatch, RankTooLow
from .grid import BoundMode, ErrorBoundSpec, ScalarGrid

_K1 = 0.01
_K2 = 0.03
_SSIM_WINDOW = 7
_SSIM_STRIDE = 2


def _check_dims(a: ScalarGrid, b: ScalarGrid) -> None:
    if a.dims != b.dims:
        raise DimsMismatch(f"dims {a.dims} vs {b.dims}")


def _range(t: torch.Tensor) -> float:
    # value_range (grid.py:127-130): float(max) - float(min), exact for f32/f64 storage
    return float(t.max()) - float(t.min())


def _is64(t: torch.Tensor) -> int:
    return int(t.dtype == torch.float64)


def mse(a: ScalarGrid, b: ScalarGrid) -> float:
    """np.mean((a.astype(f64) - b.astype(f64)) ** 2) on the device."""
    _check_dims(a, b)
    x, y = device_grid(a), device_grid(b)
    out = torch.zeros(1, dtype=torch.float64, device=x.device)
    bind()
    check(lib().hpez_sq_diff_sum(ptr(x), _is64(x), ptr(y), _is64(y), x.numel(), ptr(out),
                                 ptr(reduce_scratch()), stream()), "hpez_sq_diff_sum")
    return float(out.item()) / x.numel()


def psnr(a: ScalarGrid, b: ScalarGrid) -> float | None:
    """metrics.psnr (metrics.py:36-51): dB, range taken from ``a``."""
    m = mse(a, b)
    if m == 0.0:
        return math.inf
    rng = _range(device_grid(a))
    if rng == 0.0:
        return None
    return 20.0 * math.log10(rng) - 10.0 * math.log10(m)


def _window_shape(dims) -> tuple:
    out = []
    for ext in dims:
        w = min(_SSIM_WINDOW, ext)
        if w % 2 == 0:
            w -= 1
        out.append(max(w, 1))
    return tuple(out)


def _uniform_filter(t: torch.Tensor, win, tmp: torch.Tensor) -> torch.Tensor:
    """scipy.ndimage.uniform_filter(t, size=win) (reflect), axis by axis."""
    dims = np.asarray(t.shape, dtype=np.int64)
    src, dst = t, tmp
    for ax, w in enumerate(win):
        check(lib().hpez_uniform_filter1d(ptr(src), ptr(dst), t.dim(), dims.ctypes.data, ax, int(w),
                                          stream()), "hpez_uniform_filter1d")
        src, dst = dst, src
    return src  # holds the result; the other buffer is scratch


def ssim(a: ScalarGrid, b: ScalarGrid) -> float:
    """metrics.ssim (metrics.py:64-94): mean SSIM over full windows centred
    at every second point."""
    _check_dims(a, b)
    if a.rank < 2:
        raise RankTooLow(f"ssim needs rank >= 2, got {a.rank}")
    x_d, y_d = device_grid(a), device_grid(b)
    rng = _range(x_d)
    scale = rng if rng > 0 else 1.0
    c1 = (_K1 * scale) ** 2
    c2 = (_K2 * scale) ** 2
    win = _window_shape(a.dims)
    n = x_d.numel()
    bufs = [torch.empty(a.dims, dtype=torch.float64, device=x_d.device) for _ in range(6)]
    x, y, xx, yy, xy, tmp = bufs
    bind()
    check(lib().hpez_ssim_prep(ptr(x_d), _is64(x_d), ptr(y_d), _is64(y_d), n, ptr(x), ptr(y), ptr(xx),
                               ptr(yy), ptr(xy), stream()), "hpez_ssim_prep")
    filt = []
    for t in (x, y, xx, yy, xy):
        r = _uniform_filter(t, win, tmp)
        if r is tmp:  # odd number of passes: result landed in the scratch buffer
            tmp = t
        filt.append(r)
    lo = np.asarray([w // 2 for w in win], dtype=np.int64)
    cnt = np.asarray([len(range(w // 2, ext - (w // 2), _SSIM_STRIDE)) for w, ext in zip(win, a.dims)],
                     dtype=np.int64)
    nsel = int(np.prod(cnt))
    terms = torch.empty(max(nsel, 1), dtype=torch.float64, device=x_d.device)
    dims = np.asarray(a.dims, dtype=np.int64)
    check(lib().hpez_ssim_terms(*[ptr(f) for f in filt], a.rank, dims.ctypes.data, lo.ctypes.data,
                                cnt.ctypes.data, c1, c2, ptr(terms), stream()), "hpez_ssim_terms")
    if nsel == 0:
        return math.nan  # np.mean of an empty selection
    out = torch.zeros(1, dtype=torch.float64, device=x_d.device)
    check(lib().hpez_pairwise_sum(ptr(terms), nsel, ptr(out), ptr(reduce_scratch()), stream()),
          "hpez_pairwise_sum")
    return float(out.item()) / nsel


@dataclass(frozen=True)
class QualityReport:
    compression_ratio: float
    bit_rate: float
    psnr: float | None
    ssim: float | None
    max_abs_error: float
    max_rel_error: float


def evaluate(original: ScalarGrid, archive: bytes, decompressed: ScalarGrid) -> QualityReport:
    """metrics.evaluate (metrics.py:106-130)."""
    _check_dims(original, decompressed)
    x, y = device_grid(original), device_grid(decompressed)
    if x.numel():
        max_abs = float((x.to(torch.float64) - y.to(torch.float64)).abs().max())
    else:
        max_abs = 0.0
    rng = _range(x)
    if max_abs == 0.0:
        max_rel = 0.0
    else:
        max_rel = max_abs / rng if rng > 0 else math.inf
    return QualityReport(
        compression_ratio=original.nbytes / len(archive),
        bit_rate=8.0 * len(archive) / original.point_count,
        psnr=psnr(original, decompressed),
        ssim=ssim(original, decompressed) if original.rank >= 2 else None,
        max_abs_error=max_abs,
        max_rel_error=max_rel,
    )


@dataclass(frozen=True)
class SweepRow:
    epsilon: float
    bit_rate: float
    psnr: float | None
    ssim: float | None
    cr: float
    comp_seconds: float
    decomp_seconds: float


def sweep(grid: ScalarGrid, epsilons, target=None, *, mode: BoundMode = BoundMode.REL,
          options=None) -> list:
    """metrics.sweep (metrics.py:149-166): compress + decompress + evaluate
    per error bound, all on the GPU pipeline."""
    from .pipeline import compress, decompress
    epsilons = list(epsilons)
    if not epsilons:
        raise ValueError("sweep needs at least one epsilon")
    rows = []
    for eps in epsilons:
        res = compress(grid, ErrorBoundSpec(mode, eps), target=target, options=options)
        t0 = time.perf_counter()
        out = decompress(res.archive)
        dt = time.perf_counter() - t0
        rep = evaluate(grid, res.archive, out)
        rows.append(SweepRow(eps, rep.bit_rate, rep.psnr, rep.ssim, rep.compression_ratio,
                             res.seconds, dt))
    return rows
