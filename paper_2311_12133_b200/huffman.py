"""Canonical Huffman coding of quantizer streams -- drop-in for
huffman.encode / decode (huffman.py:144-174).

encode: GPU histogram (warp-aggregated, csrc/huffman.cu) -> host heap
lengths + canonical codes (C++, same (freq, smallest-symbol) tie-break) ->
GPU MSB-first pack.  decode: self-synchronising chunked GPU decoder
(decode_device) or the host C++ table-driven decoder (decode).  Output bytes,
lengths, bit counts, symbols and error classes equal the reference's.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .device import bind, device, ptr, stream
from .errors import EmptyInput


def table(freqs: np.ndarray):
    """(lengths u8, code values u64) for a frequency vector."""
    freqs = np.ascontiguousarray(freqs, dtype=np.int64)
    lengths = np.zeros(freqs.size, dtype=np.uint8)
    values = np.zeros(freqs.size, dtype=np.uint64)
    check(lib().hpez_huffman_table(freqs.ctypes.data, freqs.size, lengths.ctypes.data,
                                   values.ctypes.data), "hpez_huffman_table")
    return lengths, values


def histogram_device(codes) -> np.ndarray:
    """np.bincount of a device code stream (u16 or i32), as int64 host array
    trimmed to max(code)+1 like bincount."""
    if codes.numel() == 0:
        raise EmptyInput("empty symbol sequence")
    bind()
    if codes.dtype == torch.uint16:
        cdt, nbins = _lib.CODES_U16, 65536
    else:
        if int(codes.min()) < 0:
            raise ValueError("symbols must be non-negative")
        cdt, nbins = _lib.CODES_I32, int(codes.max()) + 1
    counts = torch.empty(nbins, dtype=torch.int32, device=codes.device)
    check(lib().hpez_histogram(ptr(codes), cdt, codes.numel(), ptr(counts), nbins, stream()),
          "hpez_histogram")
    h = counts.cpu().numpy().view(np.uint32).astype(np.int64)
    nz = np.flatnonzero(h)
    return h[:nz[-1] + 1]


def encode_device(codes):
    """(lengths u8[max+1], payload bytes, nbits) of a device code stream."""
    lengths, words, nbits = encode_device_words(codes)
    payload = words.view(torch.uint8)[:(nbits + 7) // 8].cpu().numpy().tobytes()
    return lengths, payload, nbits


def encode_device_words(codes):
    """(lengths u8[max+1], packed payload as a device int32 tensor, nbits):
    the payload stays in HBM for the caller to move where it needs it."""
    freqs = histogram_device(codes)
    lengths, values = table(freqs)
    nbits = int((freqs * lengths.astype(np.int64)).sum())
    nbytes = (nbits + 7) // 8
    dev = codes.device
    cdt = _lib.CODES_U16 if codes.dtype == torch.uint16 else _lib.CODES_I32
    nb = 65536 if cdt == _lib.CODES_U16 else lengths.size
    ld = np.zeros(nb, dtype=np.uint8)
    vd = np.zeros(nb, dtype=np.uint64)
    ld[:lengths.size] = lengths
    vd[:values.size] = values
    ld_t = torch.from_numpy(ld).to(dev)
    vd_t = torch.from_numpy(vd.view(np.int64)).to(dev)
    words = torch.empty(max((nbits + 31) // 32, 1), dtype=torch.int32, device=dev)
    bind()
    check(lib().hpez_huffman_pack(ptr(codes), cdt, codes.numel(), ptr(ld_t), ptr(vd_t),
                                  int(lengths.max()), ptr(words), nbits, stream()),
          "hpez_huffman_pack")
    return lengths, words, nbits


def encode(symbols):
    """huffman.encode (huffman.py:144-158) for int symbols >= 0."""
    symbols = np.ascontiguousarray(symbols, dtype=np.int64)
    if symbols.size == 0:
        raise EmptyInput("empty symbol sequence")
    if symbols.min() < 0:
        raise ValueError("symbols must be non-negative")
    if symbols.max() >= 2 ** 31:
        raise ValueError("symbols beyond int32 are not supported by the device coder")
    dev = device()
    if symbols.max() <= 65535:
        t = torch.from_numpy(symbols.astype(np.uint16)).to(dev)
    else:
        t = torch.from_numpy(symbols.astype(np.int32)).to(dev)
    return encode_device(t)


def decode(lengths, payload: bytes, count: int) -> np.ndarray:
    """huffman.decode (huffman.py:161-174): ``count`` int64 symbols."""
    if count == 0:
        return np.empty(0, dtype=np.int64)
    return decode_int32(lengths, payload, count).astype(np.int64)


def decode_int32(lengths, payload: bytes, count: int) -> np.ndarray:
    lengths = np.ascontiguousarray(np.asarray(lengths).astype(np.uint8))
    out = np.empty(count, dtype=np.int32)
    data = np.frombuffer(payload, dtype=np.uint8)
    buf = data.ctypes.data if data.size else None
    check(lib().hpez_huffman_decode(buf, data.size, lengths.ctypes.data, lengths.size, count,
                                    out.ctypes.data), "hpez_huffman_decode")
    return out


def decode_device(lengths, payload, count: int, code_dtype: int | None = None):
    """huffman.decode on the device: ``count`` symbols as a CUDA tensor (u16
    when every table symbol fits, else int32).  ``payload`` is bytes or a
    device uint8 tensor."""
    lengths = np.ascontiguousarray(np.asarray(lengths).astype(np.uint8))
    if code_dtype is None:
        code_dtype = _lib.CODES_U16 if lengths.size <= 65536 else _lib.CODES_I32
    tdt = torch.uint16 if code_dtype == _lib.CODES_U16 else torch.int32
    out = torch.empty(max(count, 1), dtype=tdt, device=device())[:count]
    if count == 0:
        return out
    bind()
    if isinstance(payload, torch.Tensor):
        nbytes = payload.numel()
        host, dev = None, (ptr(payload) if nbytes else None)
    else:
        data = np.frombuffer(payload, dtype=np.uint8)
        nbytes = data.size
        host, dev = (data.ctypes.data if nbytes else None), None
        if host is None and dev is None:
            dev = ptr(out)  # never read: nbytes == 0
    check(lib().hpez_huffman_decode_device(host, dev, nbytes, lengths.ctypes.data, lengths.size, count,
                                           ptr(out), code_dtype, stream()), "hpez_huffman_decode_device")
    return out
