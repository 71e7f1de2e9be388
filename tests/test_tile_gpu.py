"""GPU parity of the tiled level kernel (csrc/tile.cu) against the CPU oracle.

Every level of these rank-3 f32 plans is forced onto the tiled path
(HPEZ_TILE=1, HPEZ_TILE_MIN=0), across stencil families, same-level splits, MD blends,
ONED axis orders, grid extents that are not multiples of the tile, tiny
error bounds (many escapes) and the out-of-place compress entry."""

import os

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu


class _Spec:
    def __init__(self, t):
        from paper_2311_12133_b200.plan import (KERNEL_VARIANTS, PARADIGM_MULTIDIM,
                                                PARADIGM_ONED, LevelConfig)
        stride, bound, k, par, order = t
        self.stride, self.bound = stride, bound
        self.config = LevelConfig(KERNEL_VARIANTS[k], PARADIGM_MULTIDIM if par else PARADIGM_ONED,
                                  None if order is None else tuple(order))


def _levels(seed, anchor, e, kernel=None, par=None):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(anchor.bit_length() - 1):
        k = int(rng.integers(0, 5)) if kernel is None else kernel
        p = int(rng.integers(0, 2)) if par is None else par
        order = tuple(int(a) for a in rng.permutation(3)) if p == 0 else None
        s = anchor >> (i + 1)
        out.append((s, e / min(1.5 ** (s.bit_length() - 1), 3.0), k, p, order))
    return out


def _field(seed, dims):
    import synthetic as syn
    return syn.config_field(2, dims=dims).astype(np.float32)


def _tile_levels(shape, levels, md):
    """Number of tiled levels in the device plan of this configuration."""
    import ctypes

    from paper_2311_12133_b200 import _lib
    from paper_2311_12133_b200.interp import code_dtype_for, get_plan
    lv = [_Spec(t) for t in levels]
    plan = get_plan(tuple(shape), lv, direction="compress", radius=32768, md_alpha=md, rounding=1,
                    work_dtype=_lib.WORK_F32, code_dtype=code_dtype_for(32768))
    buf = (ctypes.c_int64 * 64)()
    assert _lib.lib().hpez_plan_tile_info(plan.handle, buf, 64) == 0
    return buf[0]


def _roundtrip(data, levels, md, oop=False):
    import torch

    from paper_2311_12133_b200.interp import codes_to_int32, run_levels_device
    lv = [_Spec(t) for t in levels]
    ref = data.astype(np.float64)
    c_o, o_o = oracle.run_levels(ref, levels, direction="compress", radius=32768, md_alpha=md,
                                 rounding=1)
    src = torch.from_numpy(data).cuda()
    if oop:
        work = torch.full_like(src, float("nan"))
        codes, outl, n_out = run_levels_device(work, lv, direction="compress", radius=32768,
                                               md_alpha=md, rounding=1, orig=src)
        assert torch.equal(src.cpu(), torch.from_numpy(data)), "orig was modified"
    else:
        work = src
        codes, outl, n_out = run_levels_device(work, lv, direction="compress", radius=32768,
                                               md_alpha=md, rounding=1)
    assert np.array_equal(codes_to_int32(codes), c_o), "codes differ"
    assert outl[:n_out].cpu().numpy().tobytes() == o_o.tobytes(), "outliers differ"
    assert np.array_equal(work.cpu().numpy().astype(np.float64), ref), "reconstruction differs"
    back = torch.zeros_like(work)
    back[::64, ::64, ::64] = work[::64, ::64, ::64]
    used = run_levels_device(back, lv, direction="decompress", radius=32768, md_alpha=md,
                             rounding=1, codes=codes, outliers=outl[:max(n_out, 1)])
    assert used == n_out
    assert torch.equal(back, work), "decompression differs"
    return n_out


@pytest.fixture(autouse=True)
def _force_tiles(monkeypatch):
    monkeypatch.setenv("HPEZ_TILE", "1")
    monkeypatch.setenv("HPEZ_TILE_MIN", "0")


CASES = [
    # seed, dims, kernel, paradigm
    (1, (70, 66, 90), 4, 1),      # natural cubic + same-level + MD (the cfg2 recipe)
    (2, (65, 130, 33), 4, 0),     # natural SL, ONED random orders
    (3, (129, 100, 57), 3, 1),    # not-a-knot SL + MD
    (4, (40, 77, 140), 3, 0),     # not-a-knot SL, ONED
    (5, (96, 64, 64), 0, 1),      # linear MD
    (6, (33, 97, 71), 0, 0),      # linear ONED
    (7, (50, 50, 50), 1, 1),      # not-a-knot inter MD
    (8, (61, 45, 83), 2, 0),      # natural inter ONED
    (9, (72, 80, 88), None, None),  # random per level
    (10, (17, 130, 260), None, None),
    (11, (256, 24, 40), None, None),
    (12, (9, 10, 11), None, None),  # smaller than one tile
]


@pytest.mark.parametrize("seed,dims,kernel,par", CASES)
def test_tile_vs_oracle(seed, dims, kernel, par):
    data = _field(seed, dims)
    e = 1e-3 * float(data.max() - data.min())
    levels = _levels(seed, 64, e, kernel, par)
    md = np.random.default_rng(seed).uniform(0, 1, 3)
    assert _tile_levels(data.shape, levels, md) >= 1
    _roundtrip(data, levels, md)


@pytest.mark.parametrize("seed,dims", [(21, (70, 66, 90)), (22, (45, 81, 64))])
def test_tile_out_of_place(seed, dims):
    data = _field(seed, dims)
    e = 1e-3 * float(data.max() - data.min())
    levels = _levels(seed, 64, e, 4, 1)
    md = np.array([0.2, 0.5, 0.3])
    _roundtrip(data, levels, md, oop=True)


@pytest.mark.parametrize("seed,dims,eps", [(31, (70, 66, 90), 1e-6), (32, (48, 52, 60), 1e-9)])
def test_tile_escapes(seed, dims, eps):
    rng = np.random.default_rng(seed)
    data = (_field(seed, dims) + rng.standard_normal(dims).astype(np.float32) * 0.3).astype(np.float32)
    e = eps * float(data.max() - data.min())
    levels = _levels(seed, 64, e, 4, 1)
    md = np.array([0.3, 0.3, 0.4])
    n_out = _roundtrip(data, levels, md)
    assert n_out > 1000


def test_tile_tuning_envs(monkeypatch):
    # tile shape / chunk knobs must not change results
    data = _field(41, (66, 70, 75))
    e = 1e-3 * float(data.max() - data.min())
    levels = _levels(41, 64, e, 4, 1)
    md = np.array([0.3, 0.3, 0.4])
    for ty, tx, zc in [("8", "16", "8"), ("32", "32", "128"), ("12", "20", "12")]:
        monkeypatch.setenv("HPEZ_TILE_TY", ty)
        monkeypatch.setenv("HPEZ_TILE_TX", tx)
        monkeypatch.setenv("HPEZ_TILE_ZC", zc)
        from paper_2311_12133_b200 import interp
        interp._PLANS.clear() if hasattr(interp, "_PLANS") else None
        _roundtrip(data, levels, md)
