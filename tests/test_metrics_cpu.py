"""Pins the oracle's numpy restatements of analyze_samples / psnr / ssim
(oracle/oracle.py) against golden vectors made by the reference
(tests/golden/make_golden_metrics.py)."""

import math

import numpy as np
import pytest

from golden import fixtures
from oracle import oracle

METRICS = fixtures("metrics")


def _f(v):
    return float(v) if isinstance(v, str) else v


@pytest.mark.parametrize("fx", METRICS, ids=lambda f: f.name)
def test_oracle_metrics_match_reference(fx):
    m = fx.meta
    a, b = fx.arrays["a"], fx.arrays["b"]
    assert oracle.psnr(a, b) == _f(m["psnr"])
    if m["ssim"] is not None:
        assert oracle.ssim(a, b) == m["ssim"]
    lin, cub, freeze, sig, n = oracle.analyze_samples(a, m["rate"])
    same = lambda x, y: all((math.isnan(p) and math.isnan(q)) or p == q for p, q in zip(x, y))
    assert same(lin, m["linear_mse"]) and same(cub, m["cubic_mse"])
    assert freeze == m["freeze"] and list(sig) == m["sigma_sq"] and n == m["n_samples"]


def test_oracle_uniform_filter_matches_scipy():
    from scipy.ndimage import uniform_filter
    rng = np.random.default_rng(5)
    for shape, w in [((19, 23, 17), (7, 7, 7)), ((8, 9), (7, 7)), ((7, 6, 5, 9), (7, 5, 5, 7))]:
        x = rng.standard_normal(shape) * 3
        assert np.array_equal(oracle.uniform_filter(x, w).view(np.int64),
                              uniform_filter(x, size=w).view(np.int64))
