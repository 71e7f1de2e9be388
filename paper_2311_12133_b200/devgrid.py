"""Device copies of host grids, made once per ScalarGrid and shared by the
tuner's sampling statistics, the trial blocks and the sweep (the field
crosses PCIe once per compress call)."""

from __future__ import annotations

import warnings

import numpy as np
import torch

from ._lib import lib
from .device import device
from .grid import ElementKind, ScalarGrid

_ATTR = "_hpez_device_copy"


def work_dtype(kind: ElementKind):
    """HBM storage of a grid's working values: f32 for f32 grids (every value
    stays f32-representable), f64 otherwise."""
    return torch.float32 if kind.value == ElementKind.F32.value else torch.float64


def device_grid(grid: ScalarGrid) -> torch.Tensor:
    """The grid's values in HBM (f32 or f64, C order), cached on the grid.
    Accepts the reference's ScalarGrid too (matched on ``kind.value``)."""
    t = getattr(grid, _ATTR, None)
    dev = device()
    if t is not None and t.device == dev:
        return t
    dt = np.float32 if grid.kind.value == ElementKind.F32.value else np.float64
    host = np.ascontiguousarray(grid.data, dtype=dt)
    with warnings.catch_warnings():  # read-only host array: torch only reads it
        warnings.simplefilter("ignore", UserWarning)
        src = torch.from_numpy(host)
    t = torch.empty(host.shape, dtype=work_dtype(grid.kind), device=dev)
    t.copy_(src)
    object.__setattr__(grid, _ATTR, t)  # frozen dataclass: cache beside the fields
    return t


def reduce_scratch() -> torch.Tensor:
    """Device scratch for one pairwise reduction (hpez_reduce_scratch_bytes)."""
    return torch.empty(int(lib().hpez_reduce_scratch_bytes()), dtype=torch.uint8, device=device())
