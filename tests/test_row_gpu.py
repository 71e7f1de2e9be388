"""GPU parity of the row-fused fine levels (csrc/row.cu) against the CPU oracle.

The fine levels (strides 1, 2, 4) of these rank-3 f32 plans are forced onto
the row path (HPEZ_ROW_MIN=0): every multidim kernel variant and the
split-free one-axis variants as uniform levels, mixed per-block tables over
them with several block sizes, grids whose extents are not multiples of the
chunk / block / 4-row phases, tiny error bounds (many escapes, both
directions), the out-of-place compress entry, and the fallbacks (x extent
not a multiple of 4, one-axis variants with a same-level split)."""

import ctypes

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


def _levels(seed, anchor, e, finest_kernel, finest_par=1):
    rng = np.random.default_rng(seed)
    out = []
    n = anchor.bit_length() - 1
    for i in range(n):
        last = i == n - 1
        k = finest_kernel if last else int(rng.integers(0, 5))
        p = finest_par if last else int(rng.integers(0, 2))
        if not last and i >= n - 3 and p == 0:
            k = (0, 1, 3)[int(rng.integers(0, 3))]  # strides 2 and 4: a row-eligible one-axis variant
        order = tuple(int(a) for a in rng.permutation(3)) if p == 0 else None
        s = anchor >> (i + 1)
        out.append((s, e / min(1.5 ** (s.bit_length() - 1), 3.0), k, p, order))
    return out


def _table(seed, dims, bs, nl, finest_tags):
    from paper_2311_12133_b200.plan import order_candidates
    rng = np.random.default_rng(seed + 1000)
    tags = [p * 8 + k for p in range(len(order_candidates((0, 1, 2))) + 1) for k in range(5)]
    nb = int(np.prod([-(-d // bs) for d in dims]))
    tbl = np.array(tags, np.uint8)[rng.integers(0, len(tags), (nl, nb))]
    ok = [t for t in tags if t < 8 or t % 8 in (0, 1, 3)]  # row-eligible tags for strides 2 and 4
    for li in (nl - 2, nl - 3):
        tbl[li] = np.array(ok, np.uint8)[rng.integers(0, len(ok), nb)]
    tbl[nl - 1] = np.array(finest_tags, np.uint8)[rng.integers(0, len(finest_tags), nb)]
    return tbl


def _field(dims):
    import synthetic as syn
    return syn.config_field(2, dims=dims).astype(np.float32)


def _row_info(shape, levels, md, bs=0, tbl=None):
    from paper_2311_12133_b200 import _lib
    from paper_2311_12133_b200.interp import code_dtype_for, get_plan
    lv = [_Spec(t) for t in levels]
    plan = get_plan(tuple(shape), lv, direction="compress", radius=32768, md_alpha=md, rounding=1,
                    block_size=bs, block_table=tbl, work_dtype=_lib.WORK_F32,
                    code_dtype=code_dtype_for(32768))
    buf = (ctypes.c_int64 * 8)()
    assert _lib.lib().hpez_plan_row_info(plan.handle, buf) == 0
    return list(buf)


def _roundtrip(data, levels, md, bs=0, tbl=None, oop=False):
    import torch

    from paper_2311_12133_b200.interp import codes_to_int32, run_levels_device
    lv = [_Spec(t) for t in levels]
    kw = dict(radius=32768, md_alpha=md, rounding=1, block_size=bs, block_table=tbl)
    ref = data.astype(np.float64)
    c_o, o_o = oracle.run_levels(ref, levels, direction="compress", **kw)
    src = torch.from_numpy(data).cuda()
    if oop:
        work = torch.full_like(src, float("nan"))
        codes, outl, n_out = run_levels_device(work, lv, direction="compress", orig=src, **kw)
        assert torch.equal(src.cpu(), torch.from_numpy(data)), "orig was modified"
    else:
        work = src
        codes, outl, n_out = run_levels_device(work, lv, direction="compress", **kw)
    c_g = codes_to_int32(codes)
    bad = np.flatnonzero(c_g != c_o)
    assert bad.size == 0, f"{bad.size} codes differ, first at {bad[:5]} of {c_o.size}"
    assert outl[:n_out].cpu().numpy().tobytes() == o_o.tobytes(), "outliers differ"
    assert np.array_equal(work.cpu().numpy().astype(np.float64), ref), "reconstruction differs"
    back = torch.zeros_like(work)
    back[::64, ::64, ::64] = work[::64, ::64, ::64]
    used = run_levels_device(back, lv, direction="decompress", codes=codes,
                             outliers=outl[:max(n_out, 1)], **kw)
    assert used == n_out
    assert torch.equal(back, work), "decompression differs"
    return n_out


@pytest.fixture(autouse=True)
def _force_rows(monkeypatch):
    monkeypatch.setenv("HPEZ_ROW_MIN", "0")
    monkeypatch.setenv("HPEZ_ROW", "2")  # also levels that are same-level throughout (off by default)
    from paper_2311_12133_b200 import interp
    if hasattr(interp, "_PLANS"):
        interp._PLANS.clear()


UNIFORM = [
    # seed, dims, finest kernel variant, finest paradigm, row levels expected
    (1, (70, 66, 92), 0, 1, 1),
    (2, (65, 130, 36), 1, 1, 1),
    (3, (129, 100, 56), 2, 1, 2),
    (4, (40, 77, 140), 3, 1, 1),
    (5, (96, 64, 64), 4, 1, 3),
    (6, (33, 97, 272), 4, 1, 3),
    (7, (9, 10, 12), 2, 1, 1),
    (8, (67, 69, 128), 0, 1, 3),
    (9, (66, 71, 132), 4, 1, 1),
    (10, (70, 66, 96), 0, 0, 3),   # one-axis linear at the finest level
    (11, (65, 72, 160), 1, 0, 3),  # one-axis not-a-knot
    (12, (130, 66, 64), 3, 0, 3),  # one-axis natural
]


@pytest.mark.parametrize("seed,dims,kernel,par,nrow", UNIFORM)
def test_row_uniform_vs_oracle(seed, dims, kernel, par, nrow):
    data = _field(dims)
    e = 1e-3 * float(data.max() - data.min())
    levels = _levels(seed, 64, e, kernel, par)
    md = np.random.default_rng(seed).uniform(0, 1, 3)
    assert _row_info(data.shape, levels, md)[0] == nrow
    _roundtrip(data, levels, md)


MIXED = [
    # seed, dims, block size, finest tags, row levels expected
    (11, (70, 66, 92), 16, (0, 1, 2, 3, 4), 1),
    (12, (65, 130, 36), 32, (0, 1, 2, 3, 4), 1),
    (13, (129, 100, 56), 8, (0, 2), 2),
    (14, (40, 77, 140), 4, (0, 1, 3), 1),
    (15, (96, 64, 64), 32, (0, 4), 3),
    (16, (67, 69, 272), 16, (2, 4), 3),
    (17, (97, 64, 128), 32, (0, 1, 2, 3, 4), 3),
    (18, (66, 130, 132), 32, (0, 1, 2, 3), 1),
    (19, (70, 66, 96), 16, (0, 8, 17, 27, 32, 41, 48, 1, 2), 3),  # one-axis tags in the finest table
    (20, (66, 130, 128), 32, (0, 16, 24, 40, 4), 3),
    (21, (96, 64, 64), 8, (0, 1, 2, 3, 4), 2),                    # stride-4 blocks too small for a lane
    (22, (20, 24, 1280), 32, (0, 1, 2, 3, 4), 2),                 # 40 x-blocks: tags read per chunk, 10 chunks per row
    (23, (18, 20, 1924), 16, (0, 2, 4), 1),                       # 121 x-blocks, a partial last chunk
]


@pytest.mark.parametrize("seed,dims,bs,tags,nrow", MIXED)
def test_row_mixed_vs_oracle(seed, dims, bs, tags, nrow):
    data = _field(dims)
    e = 1e-3 * float(data.max() - data.min())
    levels = _levels(seed, 64, e, 0)
    tbl = _table(seed, dims, bs, len(levels), tags)
    md = np.random.default_rng(seed).uniform(0, 1, 3)
    assert _row_info(data.shape, levels, md, bs, tbl)[0] == nrow
    _roundtrip(data, levels, md, bs, tbl)


@pytest.mark.parametrize("seed,dims,bs", [(21, (70, 66, 92), 0), (22, (45, 81, 64), 16)])
def test_row_out_of_place(seed, dims, bs):
    data = _field(dims)
    e = 1e-3 * float(data.max() - data.min())
    levels = _levels(seed, 64, e, 4)
    tbl = _table(seed, dims, bs, len(levels), (0, 1, 2, 3, 4)) if bs else None
    md = np.array([0.2, 0.5, 0.3])
    _roundtrip(data, levels, md, bs, tbl, oop=True)


@pytest.mark.parametrize("seed,dims,eps,bs", [(31, (70, 66, 92), 1e-6, 0), (32, (48, 52, 60), 1e-9, 16),
                                              (33, (66, 70, 132), 1e-5, 32)])
def test_row_escapes(seed, dims, eps, bs):
    rng = np.random.default_rng(seed)
    data = (_field(dims) + rng.standard_normal(dims).astype(np.float32) * 0.3).astype(np.float32)
    e = eps * float(data.max() - data.min())
    levels = _levels(seed, 64, e, 4)
    tbl = _table(seed, dims, bs, len(levels), (0, 1, 2, 3, 4)) if bs else None
    md = np.array([0.3, 0.3, 0.4])
    n_out = _roundtrip(data, levels, md, bs, tbl)
    assert n_out > 300


def test_row_fallbacks():
    """Ineligible finest levels stay in the flow kernel and still match."""
    md = np.array([0.3, 0.3, 0.4])
    data = _field((40, 44, 50))  # x extent not a multiple of 4
    e = 1e-3 * float(data.max() - data.min())
    levels = _levels(41, 64, e, 0)
    assert _row_info(data.shape, levels, md)[0] == 0
    _roundtrip(data, levels, md)
    data = _field((40, 44, 48))
    levels = _levels(42, 64, e, 4, finest_par=0)  # one-axis paradigm with a same-level split
    assert _row_info(data.shape, levels, md)[0] == 0
    _roundtrip(data, levels, md)
    levels = _levels(43, 64, e, 0)
    tbl = _table(43, data.shape, 16, len(levels), (0, 10, 20))  # one-axis same-level tags in the finest table
    assert _row_info(data.shape, levels, md, 16, tbl)[0] == 0
    _roundtrip(data, levels, md, 16, tbl)


TAGS_OK = (0, 1, 2, 3, 4, 8, 9, 11, 16, 17, 19, 24, 32, 40, 41, 48, 51)  # multidim + split-free one-axis tags


@pytest.mark.parametrize("case", range(24))
def test_row_random_configs(case):
    """Randomised geometry / table / bound draws (tools_fuzz_rows.py ran 420 of
    these against the oracle): odd and even z, y extents, x extents 12..276,
    block sizes 0/4/8/16/32, tag subsets, both compress entries."""
    rng = np.random.default_rng(9000 + case)
    dims = (int(rng.integers(9, 140)), int(rng.integers(9, 140)), int(rng.integers(3, 70)) * 4)
    bs = int(rng.choice([0, 4, 8, 16, 32]))
    eps = float(rng.choice([1e-2, 1e-3, 1e-4, 1e-6]))
    seed = int(rng.integers(0, 1 << 30))
    k, par = int(rng.integers(0, 5)), int(rng.integers(0, 2))
    if par == 0 and k in (2, 4):
        k = 1
    data = _field(dims)
    if rng.integers(0, 2):
        data = (data + rng.standard_normal(dims).astype(np.float32) * 0.2).astype(np.float32)
    e = eps * float(data.max() - data.min())
    levels = _levels(seed, 64, e, k, par)
    sub = [int(t) for t in rng.choice(TAGS_OK, size=int(rng.integers(1, 7)), replace=False)]
    tbl = _table(seed, dims, bs, len(levels), sub) if bs else None
    md = rng.uniform(0, 1, 3)
    assert _row_info(data.shape, levels, md, bs, tbl)[0] >= 1
    _roundtrip(data, levels, md, bs, tbl, oop=bool(rng.integers(0, 2)))
