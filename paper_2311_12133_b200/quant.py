"""Quantizer constants of the drop-in (reference quant.py:23-65).

The quantize / dequantize arithmetic itself runs fused inside the sweep
kernels (csrc/common.cuh quantize_point / dequantize_point)."""

from __future__ import annotations

DEFAULT_RADIUS = 32768

ROUND_NONE = 0  # float64 grids
ROUND_F32 = 1   # reconstructions squeezed through float32
ROUND_INT = 2   # integer grids: round half to even


def rounding_for_kind(kind) -> int:
    """Native-kind rounding mode of an ElementKind (quant.py:61-65)."""
    if kind.is_integer:
        return ROUND_INT
    return ROUND_F32 if kind.dtype.itemsize == 4 else ROUND_NONE
