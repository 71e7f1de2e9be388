"""GPU parity of the sweep kernels (run_levels drop-in) against the
reference's golden vectors and the CPU oracle."""

import numpy as np
import pytest

from golden import fixtures, level_tuples
from oracle import oracle

pytestmark = pytest.mark.gpu

SWEEPS = fixtures("sweep")


class _Spec:  # minimal LevelSpec-like view of a golden level tuple
    def __init__(self, t):
        from paper_2311_12133_b200.plan import (KERNEL_VARIANTS, PARADIGM_MULTIDIM,
                                                PARADIGM_ONED, LevelConfig)
        stride, bound, k, par, order = t
        self.stride, self.bound = stride, bound
        self.config = LevelConfig(KERNEL_VARIANTS[k], PARADIGM_MULTIDIM if par else PARADIGM_ONED,
                                  None if order is None else tuple(order))


def specs(meta):
    return [_Spec(t) for t in level_tuples(meta)]


@pytest.mark.parametrize("fx", SWEEPS, ids=lambda f: f.name)
def test_sweep_matches_reference(fx):
    from paper_2311_12133_b200.interp import CodeSource, PassStats, run_levels
    m = fx.meta
    lv = specs(m)
    work = np.ascontiguousarray(fx["input"], dtype=np.float64)
    table = fx["table"] if "table" in fx.arrays else None
    st = None
    if "err_sum" in fx.arrays:
        st = PassStats(len(lv), work.shape if "dense" in fx else None)
    codes, outl = run_levels(work, lv, direction="compress", radius=m["radius"],
                             frozen_axes=m["frozen"], md_alpha=m["md"], rounding=m["rounding"],
                             block_size=m["block_size"], block_table=table, stats=st)
    assert np.array_equal(codes, fx["codes"])
    assert outl.tobytes() == fx["outliers"].tobytes()
    assert fx.check("work_c", work)
    if st is not None:
        assert st.err_sum.tobytes() == fx["err_sum"].tobytes()
        assert np.array_equal(st.count, fx["count"])
        assert int(st.count.sum()) == codes.size
        assert np.array_equal(np.sort(st.all_codes()), np.sort(codes))
        if "dense" in fx:
            assert fx.check("dense", np.stack(st.err_grids))
    back = np.zeros_like(work)
    sel = tuple(slice(0, None, 1 if a in m["frozen"] else m["anchor"]) for a in range(work.ndim))
    back[sel] = work[sel]
    src = CodeSource(codes, outl)
    run_levels(back, lv, direction="decompress", radius=m["radius"], frozen_axes=m["frozen"],
               md_alpha=m["md"], rounding=m["rounding"], block_size=m["block_size"],
               block_table=table, source=src)
    assert src.pos == codes.size and src.ocur == outl.size
    assert fx.check("work_d", back)


def _random_case(seed, dims, anchor=64, bs=16, table=True, rounding=0, e=1e-3):
    import synthetic as syn
    from paper_2311_12133_b200.plan import order_candidates
    rng = np.random.default_rng(seed)
    data = syn.config_field(2, dims=dims).astype(np.float64)
    nl = anchor.bit_length() - 1
    levels = []
    for i in range(nl):
        k = int(rng.integers(0, 5))
        par = int(rng.integers(0, 2))
        order = tuple(int(a) for a in rng.permutation(len(dims))) if par == 0 else None
        levels.append((anchor >> (i + 1), e / min(1.5 ** ((anchor >> (i + 1)).bit_length() - 1), 3.0),
                       k, par, order))
    tbl = None
    if table:
        active = tuple(range(len(dims)))
        tags = [p * 8 + k for p in range(len(order_candidates(active)) + 1) for k in range(5)]
        nb = int(np.prod([-(-d // bs) for d in dims]))
        tbl = np.array(tags, np.uint8)[rng.integers(0, len(tags), (nl, nb))]
    md = rng.uniform(0, 1, len(dims))
    return data, levels, tbl, md


@pytest.mark.parametrize("seed,dims,bs,rounding", [
    (1, (70, 66, 90), 16, 1), (2, (65, 130, 33), 32, 0), (3, (129, 100, 57), 8, 1),
    (4, (300, 257), 16, 1), (5, (40, 30, 20, 24), 8, 0), (6, (70, 66, 90), 24, 1),
    (7, (97, 64, 130), 32, 0)])
def test_sweep_random_tables_vs_oracle(seed, dims, bs, rounding):
    from paper_2311_12133_b200.interp import CodeSource, run_levels
    data, levels, tbl, md = _random_case(seed, dims, bs=bs, rounding=rounding)
    lv = [_Spec(t) for t in levels]
    w_o = data.copy()
    c_o, o_o = oracle.run_levels(w_o, levels, direction="compress", radius=32768, md_alpha=md,
                                 rounding=rounding, block_size=bs, block_table=tbl)
    w_g = data.copy()
    c_g, o_g = run_levels(w_g, lv, direction="compress", radius=32768, md_alpha=md,
                          rounding=rounding, block_size=bs, block_table=tbl)
    assert np.array_equal(c_g, c_o)
    assert o_g.tobytes() == o_o.tobytes()
    assert w_g.tobytes() == w_o.tobytes()
    b_o = np.zeros_like(data)
    sel = tuple(slice(0, None, 64) for _ in dims)
    b_o[sel] = w_o[sel]
    b_g = b_o.copy()
    oracle.run_levels(b_o, levels, direction="decompress", radius=32768, md_alpha=md,
                      rounding=rounding, block_size=bs, block_table=tbl, codes=c_o, outliers=o_o)
    run_levels(b_g, lv, direction="decompress", radius=32768, md_alpha=md, rounding=rounding,
               block_size=bs, block_table=tbl, source=CodeSource(c_g, o_g))
    assert b_g.tobytes() == b_o.tobytes()


def test_sweep_stream_errors():
    from paper_2311_12133_b200.errors import CorruptStream, OutlierUnderflow
    from paper_2311_12133_b200.interp import CodeSource, run_levels
    from paper_2311_12133_b200.plan import build_level_plan
    data = np.sin(np.linspace(0, 9, 70 * 70)).reshape(70, 70)
    plan = build_level_plan(data.shape, 64, 1e-3)
    w = data.copy()
    codes, outl = run_levels(w, plan.levels, direction="compress", radius=32768)
    back = np.zeros_like(w)
    back[::64, ::64] = w[::64, ::64]
    with pytest.raises(CorruptStream):
        run_levels(back, plan.levels, direction="decompress", radius=32768,
                   source=CodeSource(codes[:-10], outl))
    noisy = np.random.default_rng(0).standard_normal((40, 40)) * 100
    plan = build_level_plan(noisy.shape, 64, 1e-9)
    w = noisy.copy()
    codes, outl = run_levels(w, plan.levels, direction="compress", radius=32768)
    assert outl.size > 0
    back = np.zeros_like(w)
    back[::64, ::64] = w[::64, ::64]
    with pytest.raises(OutlierUnderflow):
        run_levels(back, plan.levels, direction="decompress", radius=32768,
                   source=CodeSource(codes, outl[:-1]))
    with pytest.raises(ValueError):
        run_levels(w, plan.levels, direction="sideways", radius=32768)


@pytest.mark.parametrize("seed,dims,bs", [(11, (70, 66, 90), 16), (12, (65, 130, 33), 8)])
def test_staged_levels_vs_oracle(seed, dims, bs, monkeypatch):
    """The opt-in staged execution (one flag-free launch per (level, depth)
    group, HPEZ_STAGE_MIN) gives the oracle's codes, outliers and
    reconstruction, uniform and mixed tables alike."""
    monkeypatch.setenv("HPEZ_STAGE_MIN", "1000")
    test_sweep_random_tables_vs_oracle(seed, dims, bs, 1)


def test_unbound_workspace_plan():
    """A plan run without a caller-bound workspace allocates one block itself
    (raw C-ABI use) and produces the same stream."""
    import ctypes
    import torch
    from paper_2311_12133_b200 import _lib
    from paper_2311_12133_b200.interp import get_plan, run_levels_device, codes_to_int32
    data, levels, tbl, md = _random_case(21, (40, 44, 48), bs=16, rounding=1)
    lv = [_Spec(t) for t in levels]
    f32 = data.astype(np.float32)
    w1 = torch.from_numpy(f32).cuda()
    c1, o1, n1 = run_levels_device(w1, lv, direction="compress", radius=32768, md_alpha=md, rounding=1,
                                   block_size=16, block_table=tbl)
    plan = get_plan(f32.shape, lv, direction="compress", radius=32768, md_alpha=md, rounding=1,
                    block_size=16, block_table=tbl, work_dtype=_lib.WORK_F32, code_dtype=_lib.CODES_U16)
    h = ctypes.c_void_p()  # a second plan from the same descriptor, no workspace bound
    assert _lib.lib().hpez_plan_create(ctypes.byref(plan._desc), ctypes.byref(h)) == 0
    w2 = torch.from_numpy(f32).cuda()
    c2 = torch.empty_like(c1)
    o2 = torch.empty(c1.numel(), dtype=torch.float64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    L = _lib.lib()
    assert L.hpez_sweep_run(h, ctypes.c_void_p(w2.data_ptr()), ctypes.c_void_p(c2.data_ptr()), c2.numel(),
                            ctypes.c_void_p(o2.data_ptr()), o2.numel(), None, None, None, st) == 0
    n2 = ctypes.c_int64(0)
    assert L.hpez_sweep_finish(h, st, ctypes.byref(n2)) == 0
    L.hpez_plan_destroy(h)
    assert n2.value == n1
    assert np.array_equal(codes_to_int32(c2), codes_to_int32(c1))
    assert torch.equal(w2, w1)
