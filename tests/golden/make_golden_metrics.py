"""Golden vectors for the tuner's sampling statistics and the quality
metrics, produced by the UNMODIFIED reference package:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_metrics.py

hpez.tuner.analyze_samples (tuner.py:86-124) and hpez.metrics.psnr / ssim /
evaluate (metrics.py:36-130) on seeded grids of several kinds, ranks and
(short-axis) shapes.  Stored as tests/golden/metrics_*.npz (kind "metrics").
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import hpez  # noqa: E402
from hpez import metrics, tuner  # noqa: E402
from hpez.grid import ElementKind, ScalarGrid  # noqa: E402

import synthetic as syn  # noqa: E402


def case(name, a, b, kind, rate=0.002):
    ga = ScalarGrid(a.shape, kind, a)
    gb = ScalarGrid(b.shape, kind, b)
    st = tuner.analyze_samples(ga, rate)
    meta = {"kind": "metrics", "grid_kind": kind.value, "rate": rate,
            "psnr": metrics.psnr(ga, gb),
            "ssim": metrics.ssim(ga, gb) if ga.rank >= 2 else None,
            "linear_mse": list(st.linear_mse), "cubic_mse": list(st.cubic_mse),
            "freeze": st.freeze_candidate, "sigma_sq": list(st.sigma_sq), "n_samples": st.n_samples,
            "blend_f32": list(tuner.blend_weights_f32(st))}
    rep = metrics.evaluate(ga, b"\0" * 1000, gb)
    meta["max_abs"] = rep.max_abs_error
    meta["max_rel"] = rep.max_rel_error
    # json keeps floats exactly via repr; inf/None stored as strings
    meta = {k: (repr(v) if isinstance(v, float) and not np.isfinite(v) else v) for k, v in meta.items()}
    np.savez_compressed(os.path.join(HERE, f"metrics_{name}.npz"), meta=np.array(json.dumps(meta)), a=a, b=b)
    print(name, meta["psnr"], meta["ssim"])


def main():
    rng = np.random.default_rng(77)
    f = syn.config_field(2, dims=(40, 48, 56))
    case("grf3d", f, (f + 1e-3 * rng.standard_normal(f.shape)).astype(np.float32), ElementKind.F32)
    f = syn.config_field(4, dims=(33, 20, 70))
    case("lognormal", f, (f * (1 + 1e-2 * rng.standard_normal(f.shape))).astype(np.float32),
         ElementKind.F32, rate=0.01)
    f = rng.standard_normal((90, 120)).astype(np.float64)
    case("f64_2d", f, f + 1e-5 * rng.standard_normal(f.shape), ElementKind.F64, rate=0.05)
    f = rng.standard_normal((6, 5, 30)).astype(np.float32)  # short axes: shrunk windows, no cubic reach
    case("short_axes", f, (f + 0.1).astype(np.float32), ElementKind.F32, rate=0.3)
    f = rng.integers(-1000, 1000, (12, 14, 9, 10)).astype(np.int32)
    case("i32_4d", f, (f + rng.integers(-2, 3, f.shape)).astype(np.int32), ElementKind.I32, rate=0.05)
    f = syn.config_field(1, dims=(24, 24, 24))
    case("identical", f, f.copy(), ElementKind.F32)


if __name__ == "__main__":
    main()
