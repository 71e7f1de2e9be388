"""GPU sampling statistics and quality metrics (csrc/metrics.cu) against
the reference's golden values and, at larger sizes, the oracle: bit-exact
floats (same pairwise reduction trees, scipy's running-sum filter)."""

import math

import numpy as np
import pytest

from golden import fixtures
from oracle import oracle

pytestmark = pytest.mark.gpu

METRICS = fixtures("metrics")
KIND = {"f32": "F32", "f64": "F64", "i32": "I32", "i64": "I64"}


def _grid(arr, kind):
    from paper_2311_12133_b200.grid import ElementKind, ScalarGrid
    return ScalarGrid(arr.shape, getattr(ElementKind, KIND[kind]), arr)


def _f(v):
    return float(v) if isinstance(v, str) else v


@pytest.mark.parametrize("fx", METRICS, ids=lambda f: f.name)
def test_metrics_match_reference(fx):
    from paper_2311_12133_b200 import metrics
    from paper_2311_12133_b200.tuner import analyze_samples, blend_weights_f32
    m = fx.meta
    ga, gb = _grid(fx.arrays["a"], m["grid_kind"]), _grid(fx.arrays["b"], m["grid_kind"])
    assert metrics.psnr(ga, gb) == _f(m["psnr"])
    if m["ssim"] is not None:
        assert metrics.ssim(ga, gb) == m["ssim"]
    rep = metrics.evaluate(ga, b"\0" * 1000, gb)
    assert rep.max_abs_error == m["max_abs"] and rep.max_rel_error == _f(m["max_rel"])
    st = analyze_samples(ga, m["rate"])
    same = lambda x, y: all((math.isnan(p) and math.isnan(q)) or p == q for p, q in zip(x, y))
    assert same(st.linear_mse, m["linear_mse"]) and same(st.cubic_mse, m["cubic_mse"])
    assert st.freeze_candidate == m["freeze"] and list(st.sigma_sq) == m["sigma_sq"]
    assert st.n_samples == m["n_samples"]
    assert list(blend_weights_f32(st)) == m["blend_f32"]


@pytest.mark.parametrize("dims,seed", [((96, 100, 110), 1), ((64, 300), 2), ((20, 21, 22, 23), 3)])
def test_metrics_vs_oracle_larger(dims, seed):
    import synthetic as syn
    from paper_2311_12133_b200 import metrics
    from paper_2311_12133_b200.tuner import analyze_samples
    rng = np.random.default_rng(seed)
    a = syn.grf(dims, -3.0, seed=seed)
    b = (a + 1e-3 * rng.standard_normal(dims)).astype(np.float32)
    ga, gb = _grid(a, "f32"), _grid(b, "f32")
    assert metrics.psnr(ga, gb) == oracle.psnr(a, b)
    assert metrics.ssim(ga, gb) == oracle.ssim(a, b)
    st = analyze_samples(ga, 0.01)
    lin, cub, freeze, sig, n = oracle.analyze_samples(a, 0.01)
    assert st.linear_mse == lin and st.cubic_mse == cub and st.freeze_candidate == freeze
    assert st.sigma_sq == sig and st.n_samples == n


@pytest.mark.slow
def test_analyze_samples_full_size_cfg4():
    import synthetic as syn
    import torch
    from paper_2311_12133_b200.tuner import analyze_samples
    f = syn.config_field(4, device=torch.device("cuda", 0))
    st = analyze_samples(_grid(f, "f32"), 0.002)
    lin, cub, freeze, sig, n = oracle.analyze_samples(f, 0.002)
    assert st.linear_mse == lin and st.cubic_mse == cub and st.sigma_sq == sig and n == 268436


@pytest.mark.parametrize("fx", fixtures("samples"), ids=lambda f: f.name)
def test_analyze_samples_matches_reference_fixtures(fx):
    from paper_2311_12133_b200.grid import ElementKind, ScalarGrid
    from paper_2311_12133_b200.tuner import analyze_samples, blend_weights_f32
    m = fx.meta
    d = fx["input"]
    kind = ElementKind(m["grid_kind"])
    st = analyze_samples(ScalarGrid(d.shape, kind, d.astype(kind.dtype)), m["rate"])
    assert np.array_equal(np.array(st.linear_mse), np.array(m["linear_mse"]), equal_nan=True)
    assert np.array_equal(np.array(st.cubic_mse), np.array(m["cubic_mse"]), equal_nan=True)
    assert st.freeze_candidate == m["freeze"] and st.n_samples == m["n"]
    assert list(st.sigma_sq) == m["sigma_sq"]
    assert list(blend_weights_f32(st)) == m["weights"]
