"""End-to-end archives: compress() must emit the reference's archive bytes
(config decisions, streams, zlib) and decompress() must reproduce the
reference's reconstruction, on the golden corpus made by the reference."""

import hashlib

import numpy as np
import pytest

from golden import fixtures

pytestmark = pytest.mark.gpu

PIPES = fixtures("pipeline")


def _grid(fx):
    from paper_2311_12133_b200.grid import ElementKind, ScalarGrid
    data = fx["input"]
    return ScalarGrid(data.shape, ElementKind(fx.meta["grid_kind"]), data)


def _options(meta):
    from paper_2311_12133_b200.tuner import TunerOptions
    if meta["options"] is None:
        return None
    o = dict(meta["options"])
    o["alpha_set"] = tuple(o["alpha_set"])
    o["beta_set"] = tuple(o["beta_set"])
    return TunerOptions(**o)


def _config(meta, rank):
    from paper_2311_12133_b200.plan import CompressionConfig, decode_tag
    c = meta["config"]
    if c is None:
        return None
    lv = tuple(decode_tag(t, tuple(range(rank))) for t in c["level_tags"])
    return CompressionConfig(c["predictor"], c["resolved_bound"], c["radius"],
                             lorenzo_order=c["lorenzo_order"], level_configs=lv)


@pytest.mark.parametrize("fx", PIPES, ids=lambda f: f.name)
def test_archive_bytes_match_reference(fx):
    from paper_2311_12133_b200.grid import BoundMode, ErrorBoundSpec
    from paper_2311_12133_b200.pipeline import compress, decompress
    m = fx.meta
    grid = _grid(fx)
    spec = ErrorBoundSpec(BoundMode(m["mode"]), m["eps"])
    res = compress(grid, spec, options=_options(m), config=_config(m, grid.rank))
    assert hashlib.sha256(res.archive).hexdigest() == m["sha256"]
    assert fx.check("recon", res.reconstruction.data)
    out = decompress(fx["archive"].tobytes())
    assert out.dims == grid.dims and out.kind is grid.kind
    assert out.data.tobytes() == res.reconstruction.data.tobytes()
    e = spec.resolve(grid)
    assert np.max(np.abs(out.as_f64() - grid.as_f64())) <= e


def test_corrupt_archives_raise():
    from paper_2311_12133_b200.errors import BadMagic, CorruptStream, LengthMismatch
    from paper_2311_12133_b200.pipeline import decompress
    fx = [f for f in PIPES if f.name == "pipe_f64_rel"][0]
    arc = fx["archive"].tobytes()
    with pytest.raises(BadMagic):
        decompress(b"\x00" + arc[1:])
    with pytest.raises((LengthMismatch, CorruptStream)):
        decompress(arc[:-20])
    with pytest.raises((LengthMismatch, CorruptStream)):
        decompress(arc + b"\x00\x00")
