"""Host-side logic that needs no GPU: sampled statistics, config header and
archive framing, tag codec, plan arithmetic and the host Huffman decoder,
all against the reference's golden vectors or its pinned known answers."""

import numpy as np
import pytest

from golden import fixtures


def _grid(fx):
    from paper_2311_12133_b200.grid import ElementKind, ScalarGrid
    d = fx["input"]
    kind = fx.meta["grid_kind"]
    return ScalarGrid(d.shape, ElementKind(kind), d.astype(ElementKind(kind).dtype))


@pytest.mark.parametrize("fx", fixtures("samples"), ids=lambda f: f.name)
def test_oracle_analyze_samples_matches_reference(fx):
    """The oracle restatement (the GPU version is checked against the same
    fixtures in test_metrics_gpu.py)."""
    from oracle import oracle
    from paper_2311_12133_b200.tuner import SampleStats, blend_weights_f32
    m = fx.meta
    g = _grid(fx)
    lin, cub, freeze, sig, n = oracle.analyze_samples(g.data, m["rate"])
    assert np.array_equal(np.array(lin), np.array(m["linear_mse"]), equal_nan=True)
    assert np.array_equal(np.array(cub), np.array(m["cubic_mse"]), equal_nan=True)
    assert freeze == m["freeze"] and n == m["n"]
    assert list(sig) == m["sigma_sq"]
    assert list(blend_weights_f32(SampleStats(lin, cub, freeze, sig, n))) == m["weights"]


@pytest.mark.parametrize("fx", fixtures("pipeline"), ids=lambda f: f.name)
def test_archive_framing_round_trip(fx):
    from paper_2311_12133_b200.container import (assemble, parse, parse_config,
                                                 serialize_config, unpack_codes, lossless_unpass)
    arc = fx["archive"].tobytes()
    dims, kind, mode, eps, cfg_b, streams = parse(arc)
    cfg = parse_config(cfg_b, dims)
    assert serialize_config(cfg, dims) == cfg_b
    assert assemble(dims, kind, mode, eps, cfg_b, streams) == arc
    codes = unpack_codes(lossless_unpass(streams[1]))
    assert codes.dtype == np.int64


@pytest.mark.parametrize("fx", fixtures("huffman"), ids=lambda f: f.name)
def test_host_decoder_and_table(fx):
    from paper_2311_12133_b200 import huffman
    sym = fx["symbols"]
    freqs = np.bincount(sym)
    lengths, _ = huffman.table(freqs)
    assert np.array_equal(lengths, fx["lengths"])
    assert np.array_equal(huffman.decode(fx["lengths"], fx["payload"].tobytes(), sym.size), sym)


def test_decoder_errors():
    from paper_2311_12133_b200 import huffman
    from paper_2311_12133_b200.errors import InvalidTable, TruncatedStream
    fx = [f for f in fixtures("huffman") if f.name == "huff_skewed"][0]
    pay = fx["payload"].tobytes()
    with pytest.raises(TruncatedStream):
        huffman.decode(fx["lengths"], pay[:len(pay) // 2], fx["symbols"].size)
    lengths = np.zeros(4, dtype=np.int64)
    lengths[0] = lengths[1] = 2
    with pytest.raises((InvalidTable, TruncatedStream)):
        huffman.decode(lengths, b"\xff\xff", 3)


def test_plan_known_answers():
    # test_interp.py:203-237 pins
    from paper_2311_12133_b200.plan import (anchor_count, build_level_plan, gather_anchors,
                                            level_bound)
    assert anchor_count((65, 65, 65), 64, None) == 8
    assert anchor_count((65, 65, 65), 64, 2) == 2 * 2 * 65
    assert anchor_count((129,), 64, None) == 3
    g = np.arange(129, dtype=np.float64)
    assert np.array_equal(gather_anchors(g, 64, None), g[[0, 64, 128]])
    assert level_bound(0.1, 1.5, 4.0, 1) == 0.1
    assert level_bound(0.1, 1.5, 4.0, 3) == pytest.approx(0.1 / 2.25)
    assert level_bound(0.1, 1.5, 4.0, 10) == pytest.approx(0.1 / 4.0)
    plan = build_level_plan((100, 100), 64, 1e-2, alpha=2.0, beta=8.0)
    assert [s.stride for s in plan.levels] == [32, 16, 8, 4, 2, 1]
    assert plan.levels[-1].bound == 1e-2
    with pytest.raises(ValueError):
        build_level_plan((10, 10), 48, 1e-3)
    with pytest.raises(ValueError):
        build_level_plan((10,), 64, 1e-3, frozen_dim=0)


def test_tag_codec_round_trip():
    from paper_2311_12133_b200.plan import decode_tag, encode_tag, order_candidates
    for active in [(0,), (0, 1), (0, 2), (0, 1, 2), (0, 1, 2, 3)]:
        n = len(order_candidates(active)) + 1
        for p in range(n):
            for k in range(5):
                t = 8 * p + k
                if p == 0 and len(active) < 2:
                    pass
                assert encode_tag(decode_tag(t, active), active) == t


def test_sample_count_known_answer():
    # test_grid.py:92-97 pins 20 samples for a 100x100 grid at rate 0.002
    from paper_2311_12133_b200.grid import ElementKind, ScalarGrid, sample_indices
    g = ScalarGrid((100, 100), ElementKind.F64, np.zeros((100, 100)))
    assert len(sample_indices(g, 0.002)) == 20
