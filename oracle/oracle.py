"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  It is the checker for the B200 path, never part of it.

Level specs are plain tuples ``(stride, bound, kernel_index, paradigm,
axis_order)`` with ``kernel_index`` the position in the reference's
KERNEL_VARIANTS (plan.py:25-31) and ``paradigm`` 0 = oned, 1 = multidim.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libhpez_oracle.so")
MAX_RANK = 5


class CorruptStream(Exception):
    pass


class OutlierUnderflow(Exception):
    pass


class _Level(ctypes.Structure):
    _fields_ = [("stride", ctypes.c_int32), ("kernel", ctypes.c_int32),
                ("paradigm", ctypes.c_int32), ("n_order", ctypes.c_int32),
                ("axis_order", ctypes.c_int32 * MAX_RANK),
                ("bound", ctypes.c_double)]


def build() -> str:
    src = os.path.join(_HERE, "hpez_oracle.c")
    if (not os.path.exists(_SO)
            or os.path.getmtime(_SO) < os.path.getmtime(src)):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        _lib.orc_run_levels.restype = ctypes.c_int
        _lib.orc_run_levels.argtypes = [
            P, ctypes.c_int, P, ctypes.c_uint32, ctypes.c_int, ctypes.c_int64,
            ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, P, P, P, P, P, P, P, P]
        _lib.orc_lorenzo.restype = ctypes.c_int
        _lib.orc_lorenzo.argtypes = [
            P, ctypes.c_int, P, ctypes.c_double, ctypes.c_int64, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, P, ctypes.c_int64, P, P]
        _lib.orc_pairwise_sum.restype = ctypes.c_double
        _lib.orc_pairwise_sum.argtypes = [P, ctypes.c_int64]
        _lib.orc_code_lengths.restype = ctypes.c_int
        _lib.orc_code_lengths.argtypes = [P, ctypes.c_int64, P]
        _lib.orc_canonical_codes.restype = ctypes.c_int
        _lib.orc_canonical_codes.argtypes = [P, ctypes.c_int64, P]
        _lib.orc_pack_bits.restype = ctypes.c_int64
        _lib.orc_pack_bits.argtypes = [P, ctypes.c_int64, P, P, P]
        _lib.orc_unpack_symbols.restype = ctypes.c_int64
        _lib.orc_unpack_symbols.argtypes = [P, ctypes.c_int64, P, ctypes.c_int64,
                                            ctypes.c_int64, P]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _levels(levels):
    arr = (_Level * max(len(levels), 1))()
    for i, (stride, bound, kern, par, order) in enumerate(levels):
        arr[i].stride = int(stride)
        arr[i].bound = float(bound)
        arr[i].kernel = int(kern)
        arr[i].paradigm = int(par)
        order = tuple(order) if order is not None else ()
        arr[i].n_order = len(order)
        for j, a in enumerate(order):
            arr[i].axis_order[j] = int(a)
    return arr


def _status(st):
    if st == 1:
        raise CorruptStream("code stream exhausted")
    if st == 2:
        raise OutlierUnderflow("outlier stream exhausted")
    if st != 0:
        raise ValueError(f"oracle rejected arguments (status {st})")


def run_levels(work, levels, *, direction, radius, frozen_axes=(), md_alpha=None,
               rounding=0, block_size=0, block_table=None, codes=None,
               outliers=None, stats=False, dense=False):
    """Scalar restatement of interp.run_levels (interp.py:440-472).

    ``work`` (float64, C order) is updated in place.  Compress returns
    ``(codes int32, outliers f64[, err_sum, count, dense])``; decompress
    returns ``(codes_used, outliers_used)``.
    """
    assert work.dtype == np.float64 and work.flags.c_contiguous
    L = lib()
    rank = work.ndim
    dims = np.array(work.shape, dtype=np.int64)
    frozen = 0
    for a in frozen_axes:
        frozen |= 1 << int(a)
    md = None if md_alpha is None else np.ascontiguousarray(md_alpha, dtype=np.float64)
    tbl = None
    if block_table is not None and block_size > 0:
        tbl = np.ascontiguousarray(block_table, dtype=np.uint8)
    lv = _levels(levels)
    nl = len(levels)
    n_codes = ctypes.c_int64(0)
    n_outl = ctypes.c_int64(0)
    err_sum = count = dgrid = None
    if direction == "compress":
        cbuf = np.empty(work.size, dtype=np.int32)
        obuf = np.empty(work.size, dtype=np.float64)
        if stats:
            err_sum = np.zeros(nl)
            count = np.zeros(nl, dtype=np.int64)
            if dense:
                dgrid = np.zeros((nl,) + work.shape)
        st = L.orc_run_levels(
            _p(work), rank, _p(dims), frozen, 0, int(radius), int(rounding), nl,
            ctypes.addressof(lv), _p(md), int(block_size), _p(tbl), _p(cbuf),
            ctypes.byref(n_codes), _p(obuf), ctypes.byref(n_outl),
            _p(err_sum), _p(count), _p(dgrid))
        _status(st)
        out = (cbuf[:n_codes.value].copy(), obuf[:n_outl.value].copy())
        if stats:
            out = out + (err_sum, count, dgrid)
        return out
    if direction != "decompress":
        raise ValueError(direction)
    codes = np.ascontiguousarray(codes, dtype=np.int32)
    outliers = np.ascontiguousarray(outliers, dtype=np.float64)
    n_codes.value = codes.size
    n_outl.value = outliers.size
    st = L.orc_run_levels(
        _p(work), rank, _p(dims), frozen, 1, int(radius), int(rounding), nl,
        ctypes.addressof(lv), _p(md), int(block_size), _p(tbl), _p(codes),
        ctypes.byref(n_codes), _p(outliers), ctypes.byref(n_outl),
        None, None, None)
    _status(st)
    return n_codes.value, n_outl.value


def lorenzo(work, bound, radius, order, *, direction, rounding=0, codes=None,
            outliers=None):
    """Scalar restatement of lorenzo.lorenzo_pass (lorenzo.py:145-179)."""
    assert work.dtype == np.float64 and work.flags.c_contiguous
    L = lib()
    dims = np.array(work.shape, dtype=np.int64)
    n_outl = ctypes.c_int64(0)
    if direction == "compress":
        cbuf = np.empty(work.size, dtype=np.int32)
        obuf = np.empty(work.size, dtype=np.float64)
        st = L.orc_lorenzo(_p(work), work.ndim, _p(dims), float(bound), int(radius),
                           int(order), 0, int(rounding), _p(cbuf), work.size,
                           _p(obuf), ctypes.byref(n_outl))
        _status(st)
        return cbuf, obuf[:n_outl.value].copy()
    codes = np.ascontiguousarray(codes, dtype=np.int32)
    outliers = np.ascontiguousarray(outliers, dtype=np.float64)
    n_outl.value = outliers.size
    st = L.orc_lorenzo(_p(work), work.ndim, _p(dims), float(bound), int(radius),
                       int(order), 1, int(rounding), _p(codes), codes.size,
                       _p(outliers), ctypes.byref(n_outl))
    _status(st)
    return None


def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().orc_pairwise_sum(_p(a), a.size))


def code_lengths(freqs):
    freqs = np.ascontiguousarray(freqs, dtype=np.int64)
    out = np.zeros(freqs.size, dtype=np.uint8)
    _status(lib().orc_code_lengths(_p(freqs), freqs.size, _p(out)))
    return out


def canonical_codes(lengths):
    lengths = np.ascontiguousarray(lengths, dtype=np.uint8)
    out = np.zeros(lengths.size, dtype=np.uint64)
    _status(lib().orc_canonical_codes(_p(lengths), lengths.size, _p(out)))
    return out


def huffman_encode(symbols):
    """(lengths u8, payload bytes, nbits) like huffman.encode (huffman.py:144-158)."""
    symbols = np.ascontiguousarray(symbols, dtype=np.int64)
    freqs = np.bincount(symbols)
    lengths = code_lengths(freqs)
    values = canonical_codes(lengths)
    nbits = int(lengths[symbols].astype(np.int64).sum())
    out = np.zeros((nbits + 7) // 8, dtype=np.uint8)
    lib().orc_pack_bits(_p(symbols), symbols.size, _p(values), _p(lengths), _p(out))
    return lengths, out.tobytes(), nbits


def huffman_decode(lengths, payload: bytes, count: int):
    lengths = np.ascontiguousarray(lengths, dtype=np.uint8)
    data = np.frombuffer(payload, dtype=np.uint8).copy()
    out = np.empty(count, dtype=np.int64)
    used = lib().orc_unpack_symbols(_p(data), data.size, _p(lengths), lengths.size,
                                    count, _p(out))
    if used < 0:
        raise CorruptStream(f"huffman decode failed ({used})")
    return out


# ------------------------------------------------- tuner stats / metrics --
# numpy restatements (checkers for metrics.cu): same ufunc order as the
# reference, reductions through numpy itself (pairwise).

_CUBIC = ((-3, -1.0 / 16), (-1, 9.0 / 16), (1, 9.0 / 16), (3, -1.0 / 16))


def _reach(extent):  # grid.axis_sampling_reach (grid.py:169-176)
    return 3 if extent >= 7 else (1 if extent >= 3 else None)


def sample_index(dims, rate):
    """grid.sample_indices (grid.py:179-219): (n, rank) int64."""
    import math
    box = [(0, e - 1) if _reach(e) is None else (_reach(e), e - 1 - _reach(e)) for e in dims]
    sizes = [hi - lo + 1 for lo, hi in box]
    m = int(np.prod(sizes, dtype=np.int64))
    n = min(math.ceil(rate * int(np.prod(dims, dtype=np.int64))), m)
    flat = (np.arange(n, dtype=np.int64) * m) // n
    out = np.empty((n, len(dims)), dtype=np.int64)
    for ax in reversed(range(len(dims))):
        out[:, ax] = flat % sizes[ax] + box[ax][0]
        flat = flat // sizes[ax]
    return out


def analyze_samples(data, rate=0.002):
    """tuner.analyze_samples (tuner.py:86-124): (linear_mse, cubic_mse,
    freeze_candidate, sigma_sq, n)."""
    import math
    idx = sample_index(data.shape, rate)
    vals = data[tuple(idx.T)].astype(np.float64)
    lin, cub, measured = [], [], []
    for ax in range(data.ndim):
        reach = _reach(data.shape[ax])
        if reach is None:
            lin.append(math.nan)
            cub.append(math.nan)
            continue

        def nb(off, ax=ax):
            j = idx.copy()
            j[:, ax] += off
            return data[tuple(j.T)].astype(np.float64)

        lmse = float(np.mean((vals - 0.5 * (nb(-1) + nb(1))) ** 2))
        lin.append(lmse)
        if reach >= 3:
            pc = sum(c * nb(o) for o, c in _CUBIC)
            cub.append(float(np.mean((vals - pc) ** 2)))
        else:
            cub.append(lmse)
        measured.append(ax)
    worst = max((cub[a] for a in measured), default=1.0)
    sig = [cub[a] if a in measured else max(worst, 1.0) for a in range(data.ndim)]
    freeze = max(measured, key=lambda a: cub[a])
    return tuple(lin), tuple(cub), int(freeze), tuple(sig), len(idx)


def psnr(x, y):
    """metrics.psnr (metrics.py:36-51)."""
    import math
    x = np.asarray(x).astype(np.float64)
    y = np.asarray(y).astype(np.float64)
    mse = float(np.mean((x - y) ** 2))
    if mse == 0.0:
        return math.inf
    rng = float(x.max()) - float(x.min())
    if rng == 0.0:
        return None
    return 20.0 * math.log10(rng) - 10.0 * math.log10(mse)


def uniform_filter(x, size):
    """scipy.ndimage.uniform_filter(x, size) for float64 x, mode 'reflect',
    size <= extent on every axis: per axis, the running sum of
    NI_UniformFilter1D (sequential: np.cumsum) divided by the window."""
    out = x
    for ax, w in enumerate(size):
        a = np.moveaxis(out, ax, -1)
        L = a.shape[-1]
        s1 = w // 2
        p = np.arange(-s1, L + (w - s1 - 1))
        q = np.where(p < 0, -p - 1, np.where(p >= L, 2 * L - p - 1, p))
        ext = a[..., q]  # reflected line buffer
        first = np.zeros(a.shape[:-1])
        for l in range(w):
            first = first + ext[..., l]
        d = ext[..., w:w + L - 1] - ext[..., 0:L - 1]
        run = np.cumsum(np.concatenate([first[..., None], d], axis=-1), axis=-1)
        out = np.moveaxis(run / w, -1, ax)
    return np.ascontiguousarray(out)


def ssim(a, b):
    """metrics.ssim (metrics.py:64-94)."""
    x = np.asarray(a).astype(np.float64)
    y = np.asarray(b).astype(np.float64)
    rng = float(x.max()) - float(x.min())
    scale = rng if rng > 0 else 1.0
    c1 = (0.01 * scale) ** 2
    c2 = (0.03 * scale) ** 2
    win = []
    for ext in x.shape:
        w = min(7, ext)
        if w % 2 == 0:
            w -= 1
        win.append(max(w, 1))
    mu_x = uniform_filter(x, win)
    mu_y = uniform_filter(y, win)
    xx = uniform_filter(x * x, win)
    yy = uniform_filter(y * y, win)
    xy = uniform_filter(x * y, win)
    var_x = xx - mu_x * mu_x
    var_y = yy - mu_y * mu_y
    cov = xy - mu_x * mu_y
    sel = tuple(slice(w // 2, ext - (w // 2), 2) for w, ext in zip(win, x.shape))
    mu_x, mu_y = mu_x[sel], mu_y[sel]
    var_x, var_y, cov = var_x[sel], var_y[sel], cov[sel]
    num = (2.0 * mu_x * mu_y + c1) * (2.0 * cov + c2)
    den = (mu_x ** 2 + mu_y ** 2 + c1) * (var_x + var_y + c2)
    return float(np.mean(num / den))
