"""Bit-exact parity at BASELINE sizes: the full-size benchmark fields through
the device sweep (the path bench.py times) against the CPU oracle on the
same bytes -- cfg2 (fixed config), one cfg3 field and cfg4 at 512^3 through
tune() with their block tables, plus non-default quantizer radii
(quant.py:32-41; the reference's own tests use radius=1024,
test_container.py:96) including the int32-code variant (radius > 32768).

These are the size-dependent schedules the small fixtures cannot reach:
diagonal item bands, npos/(2*SMs) item sizing, the coarse-cluster cutoff,
512^3 index arithmetic, the mixed (block-table) fast path and the row kernel of
the fine levels (csrc/row.cu: cfg4 mostly tag-0 chunks, cfg5 56 % cubic /
same-level blocks at strides 1, 2, 4; eps 1e-5 thousands of escapes)."""

import numpy as np
import pytest
import torch

from oracle import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _tuples(levels):
    from paper_2311_12133_b200.plan import PARADIGM_MULTIDIM, kernel_index
    return [(s.stride, s.bound, kernel_index(s.config.kernel),
             1 if s.config.paradigm == PARADIGM_MULTIDIM else 0, s.config.axis_order) for s in levels]


def _device_vs_oracle(field, levels, *, radius=32768, frozen=(), md=None, bs=0, table=None, eb):
    """Compress + decompress ``field`` (f32) on the GPU and with the oracle;
    assert codes, outlier bits, reconstruction bits and the round trip."""
    from paper_2311_12133_b200.interp import codes_to_int32, run_levels_device
    dev = torch.device("cuda", 0)
    kw = dict(radius=radius, frozen_axes=frozen, md_alpha=md, rounding=1, block_size=bs,
              block_table=table)
    orig = torch.from_numpy(field).to(dev)
    work = orig.clone()
    codes, outl, n_out = run_levels_device(work, levels, direction="compress", **kw)
    ref = field.astype(np.float64)
    c_o, o_o = oracle.run_levels(ref, _tuples(levels), direction="compress", radius=radius,
                                 frozen_axes=frozen, md_alpha=md, rounding=1, block_size=bs,
                                 block_table=table)
    c_g = codes_to_int32(codes)
    assert c_g.shape == c_o.shape
    mism = int((c_g != c_o).sum())
    assert mism == 0, f"{mism} of {c_o.size} codes differ"
    assert outl[:n_out].cpu().numpy().tobytes() == o_o.tobytes()
    assert np.array_equal(work.cpu().numpy().astype(np.float64), ref)
    sel = tuple(slice(0, None, 1 if a in frozen else 64) for a in range(field.ndim))
    back = torch.zeros_like(orig)
    back[sel] = orig[sel]
    run_levels_device(back, levels, direction="decompress", codes=codes,
                      outliers=outl[:max(n_out, 1)], **kw)
    assert torch.equal(back, work)
    assert float((back.double() - orig.double()).abs().max()) <= eb
    return c_o.size, n_out


def _tuned(cfg_id, eps, dims=None):
    import synthetic as syn
    from paper_2311_12133_b200.container import parse_config, serialize_config
    from paper_2311_12133_b200.grid import ElementKind, ScalarGrid
    from paper_2311_12133_b200.pipeline import _plan
    from paper_2311_12133_b200.tuner import tune
    f = syn.config_field(cfg_id, dims=dims, device=torch.device("cuda", 0))
    g = ScalarGrid(f.shape, ElementKind.F32, f)
    eb = eps * float(f.max() - f.min())
    cfg = tune(g, eb)
    cfg = parse_config(serialize_config(cfg, g.dims), g.dims)  # f32 MD weights, as stored
    return f, cfg, _plan(g.dims, cfg).levels, eb


def test_cfg2_full_size_vs_oracle():
    import bench
    import synthetic as syn
    f = syn.config_field(2, device=torch.device("cuda", 0))
    eb = 1e-3 * float(f.max() - f.min())
    n, _ = _device_vs_oracle(f, bench.make_levels(eb), md=bench.md_weights_for(f), eb=eb)
    assert n == f.size - 4 * 6 * 6


@pytest.mark.parametrize("cfg_id,eps,dims", [(3, 1e-4, None), (4, 1e-3, None), (5, 1e-3, None), (4, 1e-5, None)])
def test_tuned_block_table_full_size_vs_oracle(cfg_id, eps, dims):
    f, cfg, levels, eb = _tuned(cfg_id, eps, dims)
    assert cfg.predictor == "interp"
    assert cfg.block_table is not None
    assert max(np.unique(r).size for r in cfg.block_table) > 1  # a mixed table
    frozen = () if cfg.frozen_dim is None else (cfg.frozen_dim,)
    _device_vs_oracle(f, levels, radius=cfg.radius, frozen=frozen, md=np.asarray(cfg.md_alpha),
                      bs=cfg.block_size, table=cfg.block_table, eb=eb)


@pytest.mark.parametrize("radius", [1024, 65536])
@pytest.mark.parametrize("tuned", [False, True])
def test_radius_variants_vs_oracle(radius, tuned):
    import bench
    if tuned:
        f, cfg, levels, eb = _tuned(4, 1e-4, dims=(160, 192, 224))
        frozen = () if cfg.frozen_dim is None else (cfg.frozen_dim,)
        _device_vs_oracle(f, levels, radius=radius, frozen=frozen, md=np.asarray(cfg.md_alpha),
                          bs=cfg.block_size, table=cfg.block_table, eb=eb)
    else:
        import synthetic as syn
        f = syn.config_field(2, dims=(128, 160, 192))
        eb = 1e-5 * float(f.max() - f.min())  # tight: codes beyond radius 1024 escape
        bench_levels = bench.make_levels(eb)
        _, n_out = _device_vs_oracle(f, bench_levels, radius=radius, md=bench.md_weights_for(f),
                                     eb=eb)
        if radius == 1024:
            assert n_out > 0
