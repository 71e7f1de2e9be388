"""GPU parity of the distributed-shared-memory coarse levels (csrc/coarse.cu)
against the CPU oracle: rank-3 f32 plans whose leading levels run in one
thread-block cluster, with the finest levels on the flow kernel, and plans
forced entirely onto the coarse cluster (HPEZ_COARSE_MAX)."""

import ctypes

import numpy as np
import pytest

from test_tile_gpu import _field, _levels, _roundtrip, _Spec

pytestmark = pytest.mark.gpu


def _coarse_mode(shape, levels, md):
    from paper_2311_12133_b200 import _lib
    from paper_2311_12133_b200.interp import code_dtype_for, get_plan
    lv = [_Spec(t) for t in levels]
    plan = get_plan(tuple(shape), lv, direction="compress", radius=32768, md_alpha=md, rounding=1,
                    work_dtype=_lib.WORK_F32, code_dtype=code_dtype_for(32768))
    buf = (ctypes.c_int64 * 12)()
    assert _lib.lib().hpez_plan_info(plan.handle, buf) == 0
    return buf[6], buf[2]


@pytest.fixture(autouse=True)
def _no_tiles(monkeypatch):
    monkeypatch.setenv("HPEZ_TILE", "0")


@pytest.mark.parametrize("seed,dims,kernel,par", [
    (1, (70, 66, 90), 4, 1), (2, (65, 130, 33), 4, 0), (3, (129, 100, 57), 3, 1),
    (4, (96, 64, 64), 0, 1), (5, (61, 45, 83), 2, 0), (6, (72, 80, 88), None, None),
    (7, (256, 24, 40), None, None), (8, (130, 129, 131), 1, 1)])
def test_coarse_dsmem_vs_oracle(seed, dims, kernel, par):
    data = _field(seed, dims)
    e = 1e-3 * float(data.max() - data.min())
    levels = _levels(seed, 64, e, kernel, par)
    md = np.random.default_rng(seed).uniform(0, 1, 3)
    mode, ncoarse = _coarse_mode(data.shape, levels, md)
    assert mode & 2 and ncoarse > 0
    _roundtrip(data, levels, md)


@pytest.mark.parametrize("seed,dims,eps", [(11, (40, 50, 60), 1e-3), (12, (33, 47, 29), 1e-7),
                                           (13, (64, 64, 64), 1e-3)])
def test_coarse_dsmem_all_levels(monkeypatch, seed, dims, eps):
    monkeypatch.setenv("HPEZ_COARSE_MAX", "100000000")
    rng = np.random.default_rng(seed)
    data = (_field(seed, dims) + rng.standard_normal(dims).astype(np.float32) * 0.05).astype(np.float32)
    e = eps * float(data.max() - data.min())
    levels = _levels(seed, 64, e, None, None)
    md = rng.uniform(0, 1, 3)
    mode, ncoarse = _coarse_mode(data.shape, levels, md)
    assert mode & 2
    _roundtrip(data, levels, md)


def test_coarse_cluster_sizes(monkeypatch):
    data = _field(21, (70, 66, 90))
    e = 1e-3 * float(data.max() - data.min())
    levels = _levels(21, 64, e, 4, 1)
    md = np.array([0.3, 0.3, 0.4])
    for n in ("1", "4", "8", "16"):
        monkeypatch.setenv("HPEZ_COARSE_CLUSTER", n)
        _roundtrip(data, levels, md)


@pytest.mark.parametrize("shift", [1, 3, 6])
def test_misaligned_code_buffers(shift):
    # the escape gather, the zero-count pre-pass and the histogram read codes
    # with aligned 16-byte loads around arbitrary element offsets
    import torch

    from oracle import oracle
    from paper_2311_12133_b200 import huffman
    from paper_2311_12133_b200.interp import codes_to_int32, run_levels_device
    rng = np.random.default_rng(shift)
    dims = (45, 52, 61)
    data = (_field(50 + shift, dims) + rng.standard_normal(dims).astype(np.float32) * 0.2).astype(np.float32)
    e = 1e-6 * float(data.max() - data.min())
    levels = _levels(50 + shift, 64, e, 4, 1)
    md = np.array([0.3, 0.3, 0.4])
    lv = [_Spec(t) for t in levels]
    ref = data.astype(np.float64)
    c_o, o_o = oracle.run_levels(ref, levels, direction="compress", radius=32768, md_alpha=md, rounding=1)
    assert o_o.size > 100
    big = torch.zeros(c_o.size + 16, dtype=torch.uint16, device="cuda")
    view = big[shift:shift + c_o.size]
    work = torch.from_numpy(data).cuda()
    codes, outl, n_out = run_levels_device(work, lv, direction="compress", radius=32768, md_alpha=md,
                                           rounding=1, codes=view)
    assert np.array_equal(codes_to_int32(codes), c_o)
    assert outl[:n_out].cpu().numpy().tobytes() == o_o.tobytes()
    assert np.array_equal(huffman.histogram_device(view), np.bincount(c_o))
    back = torch.zeros_like(work)
    back[::64, ::64, ::64] = work[::64, ::64, ::64]
    run_levels_device(back, lv, direction="decompress", radius=32768, md_alpha=md, rounding=1,
                      codes=view, outliers=outl[:n_out])
    assert torch.equal(back, work)
