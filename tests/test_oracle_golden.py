"""Pin the CPU oracle against the reference's own outputs (tests/golden/).

These run without a GPU.  Every sweep, Lorenzo, Huffman and pairwise-sum
fixture was produced by the unmodified reference package; the oracle must
reproduce it bit for bit before it is trusted as the GPU path's checker.
"""

import numpy as np
import pytest

from golden import fixtures, level_tuples
from oracle import oracle

SWEEPS = fixtures("sweep")
LORENZO = fixtures("lorenzo")
HUFF = fixtures("huffman")


@pytest.mark.parametrize("fx", SWEEPS, ids=lambda f: f.name)
def test_oracle_sweep_matches_reference(fx):
    m = fx.meta
    work = np.ascontiguousarray(fx["input"], dtype=np.float64)
    table = fx["table"] if "table" in fx.arrays else None
    stats = "err_sum" in fx.arrays
    dense = "dense" in fx
    out = oracle.run_levels(work, level_tuples(m), direction="compress", radius=m["radius"],
                            frozen_axes=m["frozen"], md_alpha=m["md"], rounding=m["rounding"],
                            block_size=m["block_size"], block_table=table, stats=stats,
                            dense=dense)
    codes, outl = out[0], out[1]
    assert np.array_equal(codes, fx["codes"])
    assert outl.tobytes() == fx["outliers"].tobytes()
    assert fx.check("work_c", work)
    if stats:
        assert out[2].tobytes() == fx["err_sum"].tobytes()
        assert np.array_equal(out[3], fx["count"])
        if dense:
            assert fx.check("dense", out[4])
    # decompress from the anchors of the compressed grid
    back = np.zeros_like(work)
    sel = tuple(slice(0, None, 1 if a in m["frozen"] else m["anchor"]) for a in range(work.ndim))
    back[sel] = work[sel]
    used = oracle.run_levels(back, level_tuples(m), direction="decompress", radius=m["radius"],
                             frozen_axes=m["frozen"], md_alpha=m["md"], rounding=m["rounding"],
                             block_size=m["block_size"], block_table=table,
                             codes=codes, outliers=outl)
    assert used == (codes.size, outl.size)
    assert fx.check("work_d", back)


@pytest.mark.parametrize("fx", LORENZO, ids=lambda f: f.name)
def test_oracle_lorenzo_matches_reference(fx):
    m = fx.meta
    work = np.ascontiguousarray(fx["input"], dtype=np.float64)
    codes, outl = oracle.lorenzo(work, m["bound"], m["radius"], m["order"],
                                 direction="compress", rounding=m["rounding"])
    assert np.array_equal(codes, fx["codes"])
    assert outl.tobytes() == fx["outliers"].tobytes()
    assert fx.check("work_c", work)
    back = np.zeros_like(work)
    oracle.lorenzo(back, m["bound"], m["radius"], m["order"], direction="decompress",
                   rounding=m["rounding"], codes=codes, outliers=outl)
    assert fx.check("work_d", back)


@pytest.mark.parametrize("fx", HUFF, ids=lambda f: f.name)
def test_oracle_huffman_matches_reference(fx):
    sym = fx["symbols"]
    lengths, payload, nbits = oracle.huffman_encode(sym)
    assert np.array_equal(lengths, fx["lengths"])
    assert nbits == fx.meta["nbits"]
    assert payload == fx["payload"].tobytes()
    assert np.array_equal(oracle.huffman_decode(lengths, payload, sym.size), sym)


def test_oracle_pairwise_matches_numpy_reduction():
    fx = fixtures("pairwise")[0]
    flat, lens, sums = fx["flat"], fx["lens"], fx["sums"]
    off = 0
    for n, s in zip(lens, sums):
        assert oracle.pairwise_sum(flat[off:off + n]) == s
        off += n


def test_oracle_stream_errors():
    work = np.ascontiguousarray(np.sin(np.linspace(0, 9, 70 * 70)).reshape(70, 70))
    lv = [(64 >> (i + 1), 1e-3, 0, 0, (0, 1)) for i in range(6)]
    codes, outl = oracle.run_levels(work.copy(), lv, direction="compress", radius=32768)
    back = np.zeros_like(work)
    back[::64, ::64] = work[::64, ::64]
    with pytest.raises(oracle.CorruptStream):
        oracle.run_levels(back, lv, direction="decompress", radius=32768,
                          codes=codes[:-10], outliers=outl)
    noisy = np.random.default_rng(0).standard_normal((40, 40)) * 100
    lv0 = [(64 >> (i + 1), 1e-9, 0, 0, (0, 1)) for i in range(6)]
    w = noisy.copy()
    codes, outl = oracle.run_levels(w, lv0, direction="compress", radius=32768)
    assert outl.size > 0
    back = np.zeros_like(w)
    back[::64, ::64] = w[::64, ::64]
    with pytest.raises(oracle.OutlierUnderflow):
        oracle.run_levels(back, lv0, direction="decompress", radius=32768,
                          codes=codes, outliers=outl[:-1])
