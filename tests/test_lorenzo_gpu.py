"""GPU Lorenzo wavefront vs the reference's numba scan (golden vectors)."""

import numpy as np
import pytest

from golden import fixtures

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["pipeline", "hyperplanes"])
def lz_mode(request, monkeypatch):
    # the pipelined single launch (default, rank <= 3) and the per-hyperplane launches
    monkeypatch.setenv("HPEZ_LORENZO_PIPE", "1" if request.param == "pipeline" else "0")
    return request.param


@pytest.mark.parametrize("fx", fixtures("lorenzo"), ids=lambda f: f.name)
def test_lorenzo_matches_reference(fx, lz_mode):
    from paper_2311_12133_b200.lorenzo import lorenzo_pass
    m = fx.meta
    work = np.ascontiguousarray(fx["input"], dtype=np.float64)
    codes, outl = lorenzo_pass(work, m["bound"], m["radius"], m["order"], direction="compress",
                               rounding=m["rounding"])
    assert np.array_equal(codes, fx["codes"])
    assert outl.tobytes() == fx["outliers"].tobytes()
    assert fx.check("work_c", work)
    back = np.zeros_like(work)
    lorenzo_pass(back, m["bound"], m["radius"], m["order"], direction="decompress",
                 rounding=m["rounding"], codes=codes, outliers=outl)
    assert fx.check("work_d", back)


def test_lorenzo_large_vs_oracle(lz_mode):
    import synthetic as syn
    from oracle import oracle
    from paper_2311_12133_b200.lorenzo import lorenzo_pass
    data = syn.config_field(3, dims=(50, 70, 90)).astype(np.float64)
    for order in (1, 2):
        a, b = data.copy(), data.copy()
        ca, oa = oracle.lorenzo(a, 1e-2, 32768, order, direction="compress", rounding=1)
        cb, ob = lorenzo_pass(b, 1e-2, 32768, order, direction="compress", rounding=1)
        assert np.array_equal(ca, cb) and oa.tobytes() == ob.tobytes() and a.tobytes() == b.tobytes()


def test_lorenzo_errors():
    from paper_2311_12133_b200.errors import CorruptStream, OutlierUnderflow
    from paper_2311_12133_b200.lorenzo import lorenzo_pass
    work = np.zeros((10, 10))
    with pytest.raises(CorruptStream):
        lorenzo_pass(work, 0.1, 32768, 1, direction="decompress", codes=np.zeros(50, np.int32),
                     outliers=np.empty(0))
    rough = np.sin(np.arange(32 * 32) * 0.9).reshape(32, 32) * 100
    w = rough.copy()
    codes, outl = lorenzo_pass(w, 1e-9, 32768, 1, direction="compress")
    assert outl.size > 0
    with pytest.raises(OutlierUnderflow):
        lorenzo_pass(np.zeros_like(w), 1e-9, 32768, 1, direction="decompress", codes=codes,
                     outliers=outl[:-1])


@pytest.mark.parametrize("dims,kind", [((1000,), "f32"), ((37, 53), "f32"), ((17, 40, 33), "f64"),
                                        ((70, 18, 49), "i32"), ((5, 4, 3, 17), "f32")])
def test_lorenzo_shapes_vs_oracle(dims, kind, lz_mode):
    """Ragged extents (not multiples of the 16x16 column blocks), ranks 1-4,
    f64 and integer grids, both orders, compress and decompress."""
    from oracle import oracle
    from paper_2311_12133_b200.lorenzo import lorenzo_pass
    rng = np.random.default_rng(len(dims) * 7 + dims[0])
    data = np.cumsum(rng.standard_normal(dims), axis=-1) * 3
    rounding = {"f32": 1, "f64": 0, "i32": 2}[kind]
    if kind == "f32":
        data = data.astype(np.float32).astype(np.float64)
    elif kind == "i32":
        data = np.rint(data * 100)
    for order in (1, 2):
        a, b = data.copy(), data.copy()
        ca, oa = oracle.lorenzo(a, 0.05, 32768, order, direction="compress", rounding=rounding)
        cb, ob = lorenzo_pass(b, 0.05, 32768, order, direction="compress", rounding=rounding)
        assert np.array_equal(ca, cb) and oa.tobytes() == ob.tobytes() and a.tobytes() == b.tobytes()
        back = np.zeros_like(data)
        lorenzo_pass(back, 0.05, 32768, order, direction="decompress", rounding=rounding, codes=cb,
                     outliers=ob)
        assert back.tobytes() == b.tobytes()
