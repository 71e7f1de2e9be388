"""GPU histogram + canonical Huffman pack vs the reference's encoder."""

import numpy as np
import pytest

from golden import fixtures

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fx", fixtures("huffman"), ids=lambda f: f.name)
def test_encode_matches_reference(fx):
    from paper_2311_12133_b200 import huffman
    from paper_2311_12133_b200.container import pack_codes, unpack_codes
    sym = fx["symbols"]
    lengths, payload, nbits = huffman.encode(sym)
    assert np.array_equal(lengths, fx["lengths"])
    assert nbits == fx.meta["nbits"]
    assert payload == fx["payload"].tobytes()
    blob = pack_codes(sym)
    assert blob == fx["packed"].tobytes()
    assert np.array_equal(unpack_codes(blob), sym)


def test_device_histogram_matches_bincount():
    import torch
    from paper_2311_12133_b200 import huffman
    rng = np.random.default_rng(0)
    for n in (1, 31, 1000, 1_000_003):
        c = (32768 + np.clip(rng.standard_normal(n) * 40, -30000, 30000)).astype(np.int64)
        c[::97] = rng.integers(0, 65536, c[::97].size)
        h = huffman.histogram_device(torch.from_numpy(c.astype(np.uint16)).cuda())
        assert np.array_equal(h, np.bincount(c))


def test_pack_large_random_round_trip():
    from paper_2311_12133_b200.container import pack_codes, unpack_codes
    from oracle import oracle
    rng = np.random.default_rng(5)
    sym = (32768 + rng.standard_normal(3_000_000) * 6).astype(np.int64)
    blob = pack_codes(sym)
    lengths, payload, nbits = oracle.huffman_encode(sym)
    assert blob[12 + lengths.size + 8:] == payload
    assert np.array_equal(unpack_codes(blob), sym)
