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


# --- device decoder (self-synchronising chunked decode) vs the host decoder,
# which the golden fixtures above pin to the reference (huffman.py:116-174)

def _device_vs_host(lengths, payload, count):
    from paper_2311_12133_b200 import huffman
    try:
        want = huffman.decode(lengths, payload, count)
        werr = None
    except Exception as ex:  # noqa: BLE001 - the error class is the contract
        want, werr = None, type(ex)
    try:
        got = huffman.decode_device(lengths, payload, count).cpu().numpy().astype(np.int64)
        gerr = None
    except Exception as ex:  # noqa: BLE001
        got, gerr = None, type(ex)
    assert gerr is werr, (gerr, werr)
    if werr is None:
        assert np.array_equal(got, want)
    return want


@pytest.mark.parametrize("n", [1, 7, 100, 4099, 2_000_003])
def test_device_decode_random(n):
    from paper_2311_12133_b200 import huffman
    rng = np.random.default_rng(n)
    sym = (32768 + np.clip(rng.standard_normal(n) * 30, -32000, 32000)).astype(np.int64)
    sym[::53] = rng.integers(0, 65536, sym[::53].size)
    lengths, payload, nbits = huffman.encode(sym)
    assert np.array_equal(_device_vs_host(lengths, payload, n), sym)
    if n > 10:  # fewer symbols than the payload holds: decode stops at count
        assert np.array_equal(_device_vs_host(lengths, payload, n - 5), sym[:-5])


def test_device_decode_long_codes():
    # Fibonacci frequencies give the deepest tree: codes up to ~30 bits, far
    # past the 12-bit first-level table
    from paper_2311_12133_b200 import huffman
    fib = [1, 1]
    while len(fib) < 30:
        fib.append(fib[-1] + fib[-2])
    sym = np.repeat(np.arange(len(fib)) * 1000, fib).astype(np.int64)
    np.random.default_rng(1).shuffle(sym)
    lengths, payload, nbits = huffman.encode(sym)
    assert lengths.max() > 20
    assert np.array_equal(_device_vs_host(lengths, payload, sym.size), sym)


def test_device_decode_int32_symbols():
    from paper_2311_12133_b200 import huffman
    rng = np.random.default_rng(3)
    sym = rng.integers(0, 200_000, 300_000).astype(np.int64)
    lengths, payload, _ = huffman.encode(sym)
    got = huffman.decode_device(lengths, payload, sym.size)
    assert str(got.dtype) == "torch.int32"
    assert np.array_equal(got.cpu().numpy(), sym)


def test_device_decode_device_payload_and_truncation():
    import torch
    from paper_2311_12133_b200 import huffman
    from paper_2311_12133_b200.errors import TruncatedStream
    rng = np.random.default_rng(4)
    sym = (100 + rng.standard_normal(50_000) * 8).astype(np.int64)
    lengths, payload, _ = huffman.encode(sym)
    dev = torch.from_numpy(np.frombuffer(payload, np.uint8).copy()).cuda()
    assert np.array_equal(huffman.decode_device(lengths, dev, sym.size).cpu().numpy(), sym)
    for cut in (1, 100, len(payload) // 2):
        _device_vs_host(lengths, payload[:-cut], sym.size)
    with pytest.raises(TruncatedStream):
        huffman.decode_device(lengths, payload, sym.size + 50)


@pytest.mark.parametrize("bits,count", [("00000000", 8), ("00000000", 9), ("00100000", 8),
                                        ("00000001", 8), ("0000000000000000", 3),
                                        ("0000000000000001", 15), ("1", 1)])
def test_device_decode_single_symbol(bits, count):
    # one-symbol table (code "0"): a 1 bit is InvalidTable, or TruncatedStream
    # when it is the payload's last bit; too few bits is TruncatedStream
    bits = bits.ljust(-(-len(bits) // 8) * 8, "0")
    payload = bytes(int(bits[i:i + 8], 2) for i in range(0, len(bits), 8))
    lengths = np.zeros(8, np.uint8)
    lengths[5] = 1
    _device_vs_host(lengths, payload, count)


def test_unpack_codes_device_matches_host():
    from paper_2311_12133_b200.container import pack_codes, unpack_codes, unpack_codes_device
    rng = np.random.default_rng(9)
    sym = (32768 + rng.standard_normal(1_000_000) * 12).astype(np.int64)
    blob = pack_codes(sym)
    t = unpack_codes_device(blob, 32768)
    assert str(t.dtype) == "torch.uint16"
    assert np.array_equal(t.cpu().numpy().astype(np.int64), unpack_codes(blob))
