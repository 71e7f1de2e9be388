"""Generate the golden vectors that pin the oracle and the B200 path.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture is produced by the UNMODIFIED reference package (hpez 0.1.0)
through its own public functions: interp.run_levels, lorenzo.lorenzo_pass,
huffman.encode, container.pack_codes, tuner.tune_blocks / tune and
pipeline.compress.  Inputs come from seeded generators in synthetic.py.
Outputs are stored as compressed .npz files next to this script.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import hpez  # noqa: E402
from hpez import pipeline, tuner  # noqa: E402
from hpez.container import pack_codes  # noqa: E402
from hpez.grid import BoundMode, ElementKind, ErrorBoundSpec, ScalarGrid  # noqa: E402
from hpez.huffman import encode  # noqa: E402
from hpez.interp import CodeSource, PassStats, block_grid_shape, run_levels  # noqa: E402
from hpez.lorenzo import lorenzo_pass  # noqa: E402
from hpez.plan import (KERNEL_VARIANTS, PARADIGM_MULTIDIM, PARADIGM_ONED,  # noqa: E402
                       CompressionConfig, LevelConfig, build_level_plan,
                       encode_tag, gather_anchors, order_candidates,
                       scatter_anchors)
from hpez.quant import ROUND_F32, ROUND_INT, ROUND_NONE  # noqa: E402

import synthetic as syn  # noqa: E402

R = 32768


def prim_levels(levels):
    out = []
    for sp in levels:
        c = sp.config
        out.append([int(sp.stride), float(sp.bound), KERNEL_VARIANTS.index(c.kernel),
                    0 if c.paradigm == PARADIGM_ONED else 1,
                    None if c.axis_order is None else [int(a) for a in c.axis_order]])
    return out


SMALL = 20_000  # arrays above this many points are pinned by SHA-256 only


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def compact(a):
    """Store f64 arrays as f32 when exact, integer codes as u16 when they fit."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.float64 and np.array_equal(a.astype(np.float32).astype(np.float64), a,
                                                equal_nan=False) \
            and not np.any(np.signbit(a) != np.signbit(a.astype(np.float32))):
        return a.astype(np.float32)
    if a.dtype.kind in "iu" and a.dtype.itemsize > 2 and a.size and a.min() >= 0 \
            and a.max() < 65536:
        return a.astype(np.uint16)
    return a


def save(name, meta, hashed=(), **arrays):
    """Write one fixture; arrays named in ``hashed`` are stored as SHA-256 of
    their exact bytes (plus dtype) when large, verbatim when small."""
    meta = dict(meta)
    meta["sha"] = {}
    out = {}
    for k, v in arrays.items():
        v = np.ascontiguousarray(v)
        if k in hashed:
            meta["sha"][k] = [sha(v), str(v.dtype), list(v.shape)]
            if v.size > SMALL:
                continue
        out[k] = compact(v)
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, meta=np.array(json.dumps(meta)), **out)
    return path


def sweep_case(name, data, e, *, cfgs=None, frozen=None, alpha=1.0, beta=1.0,
               md=None, rounding=ROUND_NONE, anchor=64, block_size=0, table=None,
               stats=False, dense=False, extra_frozen=()):
    plan = build_level_plan(data.shape, anchor, e, alpha, beta, frozen, cfgs)
    frozen_axes = set(extra_frozen)
    if frozen is not None:
        frozen_axes.add(frozen)
    frozen_axes = tuple(sorted(frozen_axes))
    inp = np.ascontiguousarray(data, dtype=np.float64)
    work = inp.copy()
    st = None
    if stats:
        st = PassStats(len(plan.levels), work.shape if dense else None)
    codes, outl = run_levels(work, plan.levels, direction="compress", radius=R,
                             frozen_axes=frozen_axes, md_alpha=md, rounding=rounding,
                             block_size=block_size, block_table=table, stats=st)
    # decompress from the compressor's anchors (test_interp.py:19-41 pattern)
    back = np.zeros_like(work)
    mask = np.ones(work.shape, dtype=bool)
    # anchor lattice: stride `anchor` on active axes, 1 on frozen axes
    sel = tuple(slice(0, None, 1 if a in frozen_axes else anchor) for a in range(work.ndim))
    back[sel] = work[sel]
    mask[sel] = False
    src = CodeSource(codes, outl)
    run_levels(back, plan.levels, direction="decompress", radius=R,
               frozen_axes=frozen_axes, md_alpha=md, rounding=rounding,
               block_size=block_size, block_table=table, source=src)
    assert src.pos == codes.size
    meta = dict(kind="sweep", levels=prim_levels(plan.levels), frozen=list(frozen_axes),
                md=None if md is None else [float(x) for x in md], rounding=rounding,
                radius=R, anchor=anchor, block_size=block_size)
    arrays = dict(input=inp, codes=codes, outliers=outl, work_c=work, work_d=back)
    if table is not None:
        arrays["table"] = np.ascontiguousarray(table, dtype=np.uint8)
    if stats:
        arrays["err_sum"] = st.err_sum
        arrays["count"] = st.count
        if dense:
            arrays["dense"] = np.stack(st.err_grids)
    save(name, meta, hashed=("work_c", "work_d", "dense"), **arrays)


def lorenzo_case(name, data, e, order, rounding=ROUND_NONE):
    inp = np.ascontiguousarray(data, dtype=np.float64)
    work = inp.copy()
    codes, outl = lorenzo_pass(work, e, R, order, direction="compress", rounding=rounding)
    back = np.zeros_like(work)
    lorenzo_pass(back, e, R, order, direction="decompress", rounding=rounding,
                 codes=codes, outliers=outl)
    meta = dict(kind="lorenzo", bound=e, order=order, rounding=rounding, radius=R)
    save(name, meta, hashed=("work_c", "work_d"), input=inp, codes=codes, outliers=outl,
         work_c=work, work_d=back)


def huffman_case(name, symbols):
    symbols = np.ascontiguousarray(symbols, dtype=np.int64)
    lengths, payload, nbits = encode(symbols)
    blob = pack_codes(symbols)
    meta = dict(kind="huffman", nbits=int(nbits))
    save(name, meta, symbols=symbols, lengths=lengths,
         payload=np.frombuffer(payload, dtype=np.uint8), packed=np.frombuffer(blob, np.uint8))


def pairwise_case():
    rng = np.random.default_rng(77)
    arrs, sums = [], []
    for n in list(range(0, 140)) + [255, 256, 257, 1000, 1331, 4097, 65537]:
        a = np.abs(rng.standard_normal(n) * np.exp(rng.standard_normal(n) * 4))
        arrs.append(a)
        sums.append(float(a.sum()))
    flat = np.concatenate(arrs)
    lens = np.array([len(a) for a in arrs], dtype=np.int64)
    save("pairwise", dict(kind="pairwise"), flat=flat, lens=lens, sums=np.array(sums))


def tune_blocks_case(name, data, kind="f64", frozen=None, md=None, options=None):
    options = options or tuner.TunerOptions()
    grid = ScalarGrid(data.shape, ElementKind(kind), data.astype(ElementKind(kind).dtype))
    active = tuple(a for a in range(grid.rank) if a != frozen)
    n_levels = 6
    cands = tuner.config_candidates(active, options)
    glob = [cands[(3 * i) % len(cands)] for i in range(n_levels)]
    table = tuner.tune_blocks(grid, glob, 1e-3, options=options, frozen_dim=frozen, md_alpha=md)
    meta = dict(kind="tune_blocks", grid_kind=kind, frozen=frozen,
                md=None if md is None else [float(x) for x in md],
                global_tags=[int(encode_tag(c, active)) for c in glob],
                block_size=options.block_size, options={k: getattr(options, k) for k in options.__dataclass_fields__})
    arrays = dict(input=np.ascontiguousarray(grid.data))
    if table is not None:
        arrays["table"] = table
    save(name, meta, **arrays)


def samples_case(name, data, kind, rate=0.002):
    grid = ScalarGrid(data.shape, ElementKind(kind), np.asarray(data).astype(ElementKind(kind).dtype))
    st = tuner.analyze_samples(grid, rate)
    w = tuner.blend_weights_f32(st)
    meta = dict(kind="samples", grid_kind=kind, rate=rate, linear_mse=list(st.linear_mse),
                cubic_mse=list(st.cubic_mse), freeze=st.freeze_candidate,
                sigma_sq=list(st.sigma_sq), n=st.n_samples, weights=list(w))
    save(name, meta, input=np.ascontiguousarray(grid.data))


def tune_global_case(name, data, kind, e, frozen=None, options=None):
    options = options or tuner.TunerOptions()
    grid = ScalarGrid(data.shape, ElementKind(kind), np.asarray(data).astype(ElementKind(kind).dtype))
    st = tuner.analyze_samples(grid, options.sample_rate)
    md = tuner.blend_weights_f32(st)
    cfgs = tuner.tune_global(grid, st, e, tuner.QualityTarget(), options=options,
                             frozen_dim=frozen, md_alpha=md)
    active = tuple(a for a in range(grid.rank) if a != frozen)
    meta = dict(kind="tune_global", grid_kind=kind, bound=e, frozen=frozen, md=list(md),
                tags=[int(encode_tag(c, active)) for c in cfgs])
    save(name, meta, input=np.ascontiguousarray(grid.data))


def pipeline_case(name, data, kind, mode, eps, options=None, config=None):
    grid = ScalarGrid(data.shape, ElementKind(kind), np.asarray(data).astype(ElementKind(kind).dtype))
    spec = ErrorBoundSpec(mode, eps)
    res = pipeline.compress(grid, spec, options=options, config=config)
    out = pipeline.decompress(res.archive)
    assert out.data.tobytes() == res.reconstruction.data.tobytes()
    opts = None
    if options is not None:
        opts = {k: getattr(options, k) for k in options.__dataclass_fields__}
    meta = dict(kind="pipeline", grid_kind=kind, mode=mode.value, eps=eps,
                options=opts, forced=config is not None,
                sha256=hashlib.sha256(res.archive).hexdigest())
    cfg_meta = None
    if config is not None:
        active = tuple(range(grid.rank))
        cfg_meta = dict(predictor=config.predictor, resolved_bound=config.resolved_bound,
                        radius=config.radius, lorenzo_order=config.lorenzo_order,
                        level_tags=[int(encode_tag(c, active)) for c in config.level_configs])
    meta["config"] = cfg_meta
    save(name, meta, hashed=("recon",), input=np.ascontiguousarray(grid.data),
         archive=np.frombuffer(res.archive, dtype=np.uint8),
         recon=np.ascontiguousarray(res.reconstruction.data))


def f32(a):
    return np.asarray(a).astype(np.float32).astype(np.float64)


def lc(k, par=PARADIGM_ONED, order=None):
    return LevelConfig(KERNEL_VARIANTS[k], par, order)


def main():
    for f in os.listdir(HERE):
        if f.endswith(".npz"):
            os.remove(os.path.join(HERE, f))
    rng = np.random.default_rng(2024)
    # --- ranks 1..4, cubic oned (test_interp.py:49-56 shapes) ---------------
    for dims in [(300,), (70, 131), (40, 33, 65), (9, 8, 10, 11)]:
        data = f32(syn.trig_product(dims, phase=0.1))
        order = tuple(range(len(dims)))
        sweep_case(f"sweep_rank{len(dims)}", data, 1e-3, cfgs=[lc(1, order=order)] * 6)
    # --- every kernel x paradigm, 2-D and 3-D, md weights, alpha/beta -------
    for k in range(5):
        for par in (PARADIGM_ONED, PARADIGM_MULTIDIM):
            d2 = syn.trig_product((50, 70), phase=0.5) + 0.001 * rng.standard_normal((50, 70))
            order = (1, 0) if par == PARADIGM_ONED else None
            sweep_case(f"sweep_k{k}_{par}_2d", d2, 1e-3, cfgs=[lc(k, par, order)] * 6)
            d3 = syn.sinusoids((25, 30, 36), seed=k).astype(np.float64)
            order = (2, 0, 1) if par == PARADIGM_ONED else None
            sweep_case(f"sweep_k{k}_{par}_3d", d3, 2e-3, cfgs=[lc(k, par, order)] * 6,
                       md=np.array([0.2, 0.5, 0.3]), alpha=1.5, beta=3.0)
    # 4-D MD with 3- and 4-axis blends (Python 3.12 compensated sum() of weights)
    d4 = syn.trig_product((12, 10, 9, 8), phase=0.2, freq=0.8)
    sweep_case("sweep_md_4d", d4, 1e-4, cfgs=[lc(4, PARADIGM_MULTIDIM)] * 6,
               md=np.array([0.7399695, 0.55376464, 0.47781921, 0.48799852]))
    # --- frozen axis, zero bound, f32 / int rounding, small anchors ---------
    sweep_case("sweep_frozen", f32(syn.trig_product((48, 65, 30), phase=0.3)), 5e-4, frozen=1)
    sweep_case("sweep_frozen_cubic", syn.trig_product((20, 37, 41), phase=0.7), 1e-3, frozen=2,
               cfgs=[lc(4, order=(0, 1))] * 6)
    sweep_case("sweep_zero_bound", np.round(syn.trig_product((80, 90), phase=0.4), 3), 0.0)
    sweep_case("sweep_zero_bound_f32", syn.sinusoids((30, 31, 32), seed=5).astype(np.float64), 0.0,
               rounding=ROUND_F32, cfgs=[lc(3, PARADIGM_MULTIDIM)] * 6)
    d_f32 = syn.sinusoids((60, 80, 3), seed=9).astype(np.float64)
    sweep_case("sweep_f32", d_f32, 1e-3, rounding=ROUND_F32, cfgs=[lc(2, order=(0, 1, 2))] * 6)
    sweep_case("sweep_f32_md_sl", syn.config_field(2, dims=(48, 40, 56)).astype(np.float64), 3e-3,
               rounding=ROUND_F32, cfgs=[lc(4, PARADIGM_MULTIDIM)] * 6, md=np.array([0.3, 0.3, 0.4]))
    ints = np.rint(np.cumsum(rng.integers(-40, 40, (64, 70)), axis=1)).astype(np.float64)
    sweep_case("sweep_int", ints, 3.0, rounding=ROUND_INT, cfgs=[lc(1, order=(0, 1))] * 6)
    sweep_case("sweep_anchor8", syn.sinusoids((27, 19, 34), seed=3).astype(np.float64), 1e-2,
               anchor=8, cfgs=[lc(3, order=(1, 2, 0)), lc(2, PARADIGM_MULTIDIM), lc(4, order=(2, 1, 0))])
    sweep_case("sweep_noise_escapes", rng.standard_normal((40, 44, 20)) * 10, 1e-6,
               cfgs=[lc(3, PARADIGM_MULTIDIM)] * 6)
    sweep_case("sweep_tiny", np.array([[1.5, -2.0, 3.25]]), 1e-3)
    sweep_case("sweep_point", np.array([3.75]), 1e-6)
    # --- mixed per-block tables (test_interp.py:125-158 + random tables) ----
    data = syn.trig_product((70, 70), phase=0.8)
    ta = encode_tag(lc(0, order=(0, 1)), (0, 1))
    tb = encode_tag(lc(1, PARADIGM_MULTIDIM), (0, 1))
    nb = int(np.prod(block_grid_shape((70, 70), 32)))
    table = np.full((6, nb), ta, dtype=np.uint8)
    table[:, ::2] = tb
    sweep_case("mixed_two_tags", data, 1e-3, block_size=32, table=table)
    data = syn.trig_product((128, 128), phase=0.23)
    t0 = encode_tag(lc(2, order=(1, 0)), (0, 1))
    t1 = encode_tag(lc(2, order=(0, 1)), (0, 1))
    gshape = block_grid_shape((128, 128), 32)
    checker = np.indices(gshape).sum(axis=0).ravel() % 2
    table = np.where(checker, t0, t1)[None, :].repeat(6, axis=0).astype(np.uint8)
    sweep_case("mixed_conflicting_split", data, 1e-3, block_size=32, table=table)
    for i, (dims, bs, anchor) in enumerate([((40, 36, 44), 8, 16), ((33, 47, 29), 16, 16),
                                            ((48, 48, 40), 16, 64), ((66, 40, 36), 32, 64)]):
        active = (0, 1, 2)
        ntag = len(order_candidates(active)) + 1
        tags = [p * 8 + k for p in range(ntag) for k in range(5)]
        nl = anchor.bit_length() - 1
        nb = int(np.prod(block_grid_shape(dims, bs)))
        r = np.random.default_rng(100 + i)
        table = np.array(tags, dtype=np.uint8)[r.integers(0, len(tags), (nl, nb))]
        data = syn.sinusoids(dims, seed=40 + i).astype(np.float64)
        sweep_case(f"mixed_random_{i}", data, 1e-3, anchor=anchor, block_size=bs, table=table,
                   md=np.array([0.5, 0.25, 0.25]), rounding=ROUND_F32 if i % 2 else ROUND_NONE)
    # 2-D random table incl. frozen axis (active = (1,)) and 4-D table
    dims = (30, 90)
    nb = int(np.prod(block_grid_shape(dims, 16)))
    table = np.array([8 + k for k in range(5)], np.uint8)[np.random.default_rng(7).integers(0, 5, (6, nb))]
    sweep_case("mixed_frozen", syn.trig_product(dims, phase=0.6), 1e-3, frozen=0, block_size=16,
               table=table)
    dims = (20, 18, 17, 16)
    ntag = len(order_candidates((0, 1, 2, 3))) + 1
    tags = [p * 8 + k for p in range(ntag) for k in range(5)]
    nb = int(np.prod(block_grid_shape(dims, 8)))
    table = np.array(tags, np.uint8)[np.random.default_rng(8).integers(0, len(tags), (4, nb))]
    sweep_case("mixed_4d", f32(syn.trig_product(dims, phase=0.9, freq=0.7)), 1e-4, anchor=16,
               block_size=8, table=table, md=np.array([0.1, 0.2, 0.3, 0.4]))
    # --- stats (PassStats) incl. dense grids, tune_blocks-style batch axis --
    sweep_case("stats_plain", syn.trig_product((80, 65), phase=0.9), 1e-3, stats=True)
    sweep_case("stats_dense_zero", syn.sinusoids((24, 30, 28), seed=11).astype(np.float64), 0.0,
               cfgs=[lc(4, PARADIGM_MULTIDIM)] * 6, stats=True, dense=True, rounding=ROUND_F32)
    stacked = syn.sinusoids((12, 11, 11, 11), seed=12).astype(np.float64)
    for k in (0, 2, 4):
        sweep_case(f"stats_batch_k{k}", stacked, 0.0, anchor=8, extra_frozen=(0,),
                   cfgs=[lc(k, PARADIGM_MULTIDIM)] * 3, md=np.array([0.0, 0.2, 0.3, 0.5]),
                   stats=True, dense=True)
    sweep_case("stats_batch_oned", stacked, 0.0, anchor=8, extra_frozen=(0,),
               cfgs=[lc(2, order=(3, 1, 2))] * 3, stats=True, dense=True)
    sweep_case("stats_real_bound", syn.sinusoids((40, 41, 42), seed=13).astype(np.float64), 1e-3,
               cfgs=[lc(3, order=(0, 1, 2))] * 6, stats=True, alpha=1.25, beta=2.0)
    # --- Lorenzo -------------------------------------------------------------
    for dims, order in [((500,), 1), ((60, 70), 1), ((60, 70), 2), ((20, 24, 28), 1),
                        ((20, 24, 28), 2), ((8, 9, 10, 11), 2)]:
        lorenzo_case(f"lorenzo_r{len(dims)}_o{order}", syn.trig_product(dims, phase=0.17), 1e-3, order)
    lorenzo_case("lorenzo_f32", syn.sinusoids((30, 40, 50), seed=2).astype(np.float64), 1e-3, 1,
                 rounding=ROUND_F32)
    lorenzo_case("lorenzo_int", rng.integers(-500, 500, (40, 40)).astype(np.float64), 2.0, 1,
                 rounding=ROUND_INT)
    lorenzo_case("lorenzo_zero", np.round(syn.trig_product((30, 30), phase=0.2), 2), 0.0, 2)
    lorenzo_case("lorenzo_escapes", syn.trig_product((32, 32), phase=0.9) * 100, 1e-9, 1)
    # --- Huffman / pack_codes --------------------------------------------------
    huffman_case("huff_single", np.full(1000, 7))
    huffman_case("huff_quant", (R + np.clip(rng.standard_normal(300_000) * 3, -50, 50)).astype(np.int64))
    huffman_case("huff_uniform", rng.integers(0, 65536, 60_000))
    huffman_case("huff_skewed", rng.choice(np.arange(8), size=50_000,
                                           p=[0.5, 0.2, 0.1, 0.08, 0.05, 0.04, 0.02, 0.01]))
    fib = np.concatenate([np.full(int(f), i) for i, f in enumerate(
        [1, 1, 2, 3, 5, 8, 13, 21, 34, 55, 89, 144, 233, 377, 610, 987, 1597, 2584, 4181,
         6765, 10946, 17711, 28657, 46368, 75025, 121393])])
    huffman_case("huff_deep", np.random.default_rng(3).permutation(fib))
    pairwise_case()
    # --- tune_blocks (tuner.py:414-486) ---------------------------------------
    tune_blocks_case("tuneblk_3d", f32(syn.patchwork((64, 64, 64), seed=1)), md=(0.3, 0.3, 0.4))
    tune_blocks_case("tuneblk_2d_f32", syn.patchwork((96, 128), seed=2), kind="f32", md=(0.6, 0.4))
    tune_blocks_case("tuneblk_frozen", f32(syn.patchwork((64, 40, 64), seed=3)), frozen=1, md=(0.2, 0.0, 0.8))
    tune_blocks_case("tuneblk_4d", f32(syn.patchwork((32, 17, 16, 33), seed=4)), md=(0.25, 0.25, 0.25, 0.25),
                     options=tuner.TunerOptions(block_size=16))
    # --- sampled statistics and global selection (tuner.py:86-133, :280-302)
    samples_case("samples_3d", syn.config_field(3, dims=(40, 64, 64)), "f32")
    samples_case("samples_2d", syn.patchwork((96, 128), seed=6), "f64", rate=0.01)
    samples_case("samples_small", syn.trig_product((5, 40, 2)), "f64", rate=0.05)
    samples_case("samples_4d", syn.trig_product((12, 10, 9, 8), freq=0.7), "f64", rate=0.01)
    tune_global_case("tglobal_3d", syn.config_field(2, dims=(70, 66, 72)), "f32", 1e-3)
    tune_global_case("tglobal_frozen", syn.patchwork((64, 70, 64), seed=7), "f64", 1e-3, frozen=0)
    tune_global_case("tglobal_2d", syn.trig_product((128, 128)), "f64", 1e-4)
    # --- whole pipeline archives (pipeline.py:57-143) -------------------------
    fast = tuner.TunerOptions(sample_rate=0.01)
    pipeline_case("pipe_f64_rel", syn.trig_product((70, 90)), "f64", BoundMode.REL, 1e-3, options=fast)
    pipeline_case("pipe_f32_rel", syn.sinusoids((40, 50, 60), seed=21), "f32", BoundMode.REL, 1e-3)
    pipeline_case("pipe_f32_abs", syn.trig_product((70, 90)), "f32", BoundMode.ABS, 1e-3, options=fast)
    pipeline_case("pipe_rank1", syn.trig_product((400,), freq=0.7), "f64", BoundMode.REL, 1e-3, options=fast)
    pipeline_case("pipe_rank4", syn.trig_product((12, 10, 9, 8), freq=0.7), "f64", BoundMode.REL, 1e-3,
                  options=fast)
    pipeline_case("pipe_i32", np.cumsum(rng.integers(-40, 40, (64, 64)), axis=1), "i32", BoundMode.ABS, 3.0,
                  options=fast)
    pipeline_case("pipe_i64", np.cumsum(rng.integers(-40, 40, (64, 64)), axis=1), "i64", BoundMode.ABS, 3.0,
                  options=fast)
    pipeline_case("pipe_const", np.full((50, 50), 4.25), "f64", BoundMode.REL, 1e-2, options=fast)
    pipeline_case("pipe_point", np.array([3.75]), "f64", BoundMode.ABS, 1e-6, options=fast)
    pipeline_case("pipe_patchwork", syn.patchwork((64, 64, 40), seed=5), "f32", BoundMode.REL, 1e-3)
    pipeline_case("pipe_grf", syn.config_field(3, dims=(40, 64, 64)), "f32", BoundMode.REL, 1e-4)
    noisy = syn.trig_product((48, 80)) + 2.0 * np.random.default_rng(22).standard_normal((48, 1))
    pipeline_case("pipe_freeze", noisy, "f64", BoundMode.ABS, 1e-3, options=fast)
    white = np.random.default_rng(21).standard_normal((60, 60))
    pipeline_case("pipe_lorenzo_forced", white, "f64", BoundMode.ABS, 0.05,
                  config=CompressionConfig("lorenzo", 0.05, 32768, lorenzo_order=2))
    pipeline_case("pipe_interp_forced", white, "f64", BoundMode.ABS, 0.05,
                  config=CompressionConfig("interp", 0.05, 32768))
    c1 = syn.config_field(1)
    eb = 1e-3 * float(c1.max() - c1.min())
    pipeline_case("pipe_cfg1_default", c1, "f32", BoundMode.REL, 1e-3,
                  config=tuner.default_config(eb, 3))
    lor = np.cumsum(np.cumsum(np.random.default_rng(5).standard_normal((40, 40, 40)), 0), 1)
    pipeline_case("pipe_lorenzo_tuned", lor, "f32", BoundMode.REL, 1e-5)
    total = sum(os.path.getsize(os.path.join(HERE, f)) for f in os.listdir(HERE) if f.endswith(".npz"))
    print(f"wrote fixtures: {total / 1e6:.1f} MB")


if __name__ == "__main__":
    main()
