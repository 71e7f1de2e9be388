"""Drop-in for the reference's level engine, interp.run_levels
(interp.py:440-472), executed by the sm_100a sweep kernels.

``run_levels`` keeps the reference signature and semantics: ``work``
(float64 numpy, C order) is updated in place; compression returns
``(codes int32, outliers float64)``; decompression consumes a CodeSource and
advances its cursors; PassStats are filled exactly like the reference's.
Internally the grid is moved to HBM, the commit schedule is a cached native
plan and the whole sweep runs on the current CUDA stream.

``run_levels_device`` is the device-resident entry (torch tensors in HBM,
u16 codes) used by the pipeline, the tuner and bench.py.
"""

from __future__ import annotations

import collections
import ctypes
import os
import hashlib

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .device import bind, device, ptr, stream
from .errors import CorruptStream
from .plan import PARADIGM_MULTIDIM, kernel_index
from .quant import ROUND_F32, ROUND_NONE

TRAVERSAL_FVFI = "fvfi"
TRAVERSAL_DIM_MAJOR = "dim_major"


class CodeSource:
    """Codes and outliers fed back to a decompressing sweep (interp.py:70-86)."""

    def __init__(self, codes, outliers):
        self.codes_arr = np.asarray(codes, dtype=np.int32)
        self.outliers = np.asarray(outliers, dtype=np.float64)
        self.pos = 0
        self.ocur = 0

    def take(self, n: int):
        if self.pos + n > len(self.codes_arr):
            raise CorruptStream(f"code stream exhausted: want {n} at {self.pos}, "
                                f"have {len(self.codes_arr)}")
        out = self.codes_arr[self.pos:self.pos + n]
        self.pos += n
        return out


class PassStats:
    """Per-level error/code statistics for tuning (interp.py:89-118)."""

    def __init__(self, n_levels: int, dense_shape=None):
        self.err_sum = np.zeros(n_levels)
        self.count = np.zeros(n_levels, dtype=np.int64)
        self.code_chunks = [[] for _ in range(n_levels)]
        self.err_grids = None
        if dense_shape is not None:
            self.err_grids = [np.zeros(dense_shape) for _ in range(n_levels)]

    def record(self, li: int, err_sum: float, n: int, codes) -> None:
        self.err_sum[li] += err_sum
        self.count[li] += n
        self.code_chunks[li].append(np.asarray(codes).ravel())

    def level_mae(self, li: int) -> float:
        n = self.count[li]
        return float(self.err_sum[li] / n) if n else 0.0

    def all_codes(self):
        chunks = [c for lv in self.code_chunks for c in lv]
        return np.concatenate(chunks) if chunks else np.empty(0, np.int32)


def block_grid_shape(dims, block_size: int) -> tuple:
    return tuple(-(-int(e) // block_size) for e in dims)


# ------------------------------------------------------------ native plans --
class SweepPlan:
    """A cached native commit schedule (hpez_plan) for one geometry/config."""

    def __init__(self, desc: _lib.SweepDesc, n_levels: int, keepalive):
        self._keep = keepalive
        self._desc = desc  # the descriptor (its arrays live in keepalive)
        h = ctypes.c_void_p()
        bind()
        check(lib().hpez_plan_create(ctypes.byref(desc), ctypes.byref(h)), "hpez_plan_create")
        self.handle = h
        # device workspace from torch's caching allocator (the library never
        # allocates during a run)
        nb = ctypes.c_int64(0)
        check(lib().hpez_plan_workspace_size(h, ctypes.byref(nb)), "hpez_plan_workspace_size")
        self.workspace = torch.empty(max(int(nb.value), 1), dtype=torch.uint8, device=device())
        check(lib().hpez_plan_bind_workspace(h, ptr(self.workspace), self.workspace.numel()),
              "hpez_plan_bind_workspace")
        self.n_levels = n_levels
        self.num_codes = int(lib().hpez_plan_num_codes(h))
        self.num_launches = int(lib().hpez_plan_num_launches(h))
        lc = np.zeros(n_levels + 1, dtype=np.int64)
        check(lib().hpez_plan_level_codes(h, lc.ctypes.data), "level codes")
        self.level_codes = lc
        self.direction = desc.direction
        self.code_dtype = desc.code_dtype
        self.work_dtype = desc.work_dtype

    def __del__(self):
        try:
            if self.handle:
                lib().hpez_plan_destroy(self.handle)
        except Exception:  # interpreter shutdown
            pass


_PLANS: "collections.OrderedDict[bytes, SweepPlan]" = collections.OrderedDict()
_PLAN_CAP = 256  # tune() alone builds ~130 trial plans; an LRU smaller than that thrashes
_PLAN_ENV = ("HPEZ_TILE", "HPEZ_TILE_MIN", "HPEZ_TILE_TY", "HPEZ_TILE_TX", "HPEZ_TILE_ZC", "HPEZ_TILE_NT",
             "HPEZ_COARSE_MAX", "HPEZ_COARSE_CLUSTER", "HPEZ_COARSE_DSMEM", "HPEZ_ROW", "HPEZ_ROW_MIN",
             "HPEZ_STAGE_MIN")


def _level_array(levels, rank):
    arr = (_lib.Level * max(len(levels), 1))()
    for i, sp in enumerate(levels):
        cfg = sp.config
        arr[i].stride = int(sp.stride)
        arr[i].bound = float(sp.bound)
        arr[i].kernel = kernel_index(cfg.kernel)
        arr[i].paradigm = 1 if cfg.paradigm == PARADIGM_MULTIDIM else 0
        order = tuple(cfg.axis_order) if cfg.axis_order is not None else ()
        if len(order) > _lib.MAX_RANK:
            raise ValueError("axis order longer than the maximum rank")
        arr[i].n_order = len(order)
        for j, a in enumerate(order):
            arr[i].axis_order[j] = int(a)
    return arr


def get_plan(dims, levels, *, direction, radius, frozen_axes=(), md_alpha=None,
             rounding=ROUND_NONE, block_size=0, block_table=None, work_dtype=_lib.WORK_F64,
             code_dtype=_lib.CODES_U16, with_stats=False) -> SweepPlan:
    rank = len(dims)
    if not 1 <= rank <= _lib.MAX_RANK:
        raise ValueError(f"rank {rank} outside 1..{_lib.MAX_RANK}")
    lv = _level_array(levels, rank)
    md = None
    if md_alpha is not None:
        md = np.zeros(rank, dtype=np.float64)
        src = np.asarray(md_alpha, dtype=np.float64).ravel()
        md[:min(rank, src.size)] = src[:rank]
    tbl = None
    if block_table is not None and block_size > 0:
        tbl = np.ascontiguousarray(block_table, dtype=np.uint8)
    frozen = 0
    for a in frozen_axes:
        frozen |= 1 << int(a)
    d = _lib.SweepDesc()
    d.rank = rank
    for a, e in enumerate(dims):
        d.dims[a] = int(e)
    d.frozen_mask = frozen
    d.direction = _lib.COMPRESS if direction == "compress" else _lib.DECOMPRESS
    d.rounding = int(rounding)
    d.radius = int(radius)
    d.n_levels = len(levels)
    d.levels = ctypes.cast(lv, ctypes.POINTER(_lib.Level))
    d.md_alpha = ctypes.cast(md.ctypes.data, ctypes.POINTER(ctypes.c_double)) if md is not None else None
    d.block_size = int(block_size) if tbl is not None else 0
    d.block_table = tbl.ctypes.data if tbl is not None else None
    d.work_dtype = work_dtype
    d.code_dtype = code_dtype
    d.with_stats = int(bool(with_stats))
    key = hashlib.sha1()
    key.update(repr((tuple(int(e) for e in dims), frozen, d.direction, d.rounding, d.radius,
                     d.n_levels, d.block_size, work_dtype, code_dtype, d.with_stats)).encode())
    key.update(bytes(lv))
    key.update(b"" if md is None else md.tobytes())
    key.update(b"" if tbl is None else tbl.tobytes())
    # planner knobs (tiled levels) read by the library at plan creation
    key.update(repr([os.environ.get(v) for v in _PLAN_ENV]).encode())
    # a plan owns its run scratch (escape counts, flags, counters), so each
    # (device, stream) pair gets its own instance: sweeps on different
    # streams may run concurrently
    key.update(f"{torch.cuda.current_device()}:{torch.cuda.current_stream().cuda_stream}".encode())
    k = key.digest()
    plan = _PLANS.get(k)
    if plan is not None:
        _PLANS.move_to_end(k)
        return plan
    plan = SweepPlan(d, len(levels), (lv, md, tbl))
    _PLANS[k] = plan
    while len(_PLANS) > _PLAN_CAP:
        _PLANS.popitem(last=False)
    return plan


def code_dtype_for(radius: int) -> int:
    return _lib.CODES_U16 if radius <= 32768 else _lib.CODES_I32


def torch_code_dtype(code_dtype: int):
    return torch.uint16 if code_dtype == _lib.CODES_U16 else torch.int32


def run_levels_device(work, levels, *, direction, radius, frozen_axes=(), md_alpha=None,
                      rounding=ROUND_NONE, block_size=0, block_table=None, codes=None,
                      outliers=None, stats=None, sync=True, orig=None):
    """Device-resident sweep.

    ``work``: contiguous CUDA tensor (float32 storage requires every value,
    before and after, to be float32-representable, i.e. ROUND_F32 grids).
    Compress returns ``(codes, outliers, n_outliers)`` device tensors (codes
    u16 when radius <= 32768); decompress consumes ``codes`` / ``outliers``
    device tensors and returns the number of outliers used.  ``stats`` is a
    dict of device tensors ``err_sum``/``count``/``dense`` (optional).
    ``orig`` (compress, no stats): read the originals from this tensor instead
    and write the anchors plus every reconstruction into ``work`` -- the
    pipeline's ``work = f64(grid)`` copy (pipeline.py:82) folded into the sweep.
    """
    if direction not in ("compress", "decompress"):
        raise ValueError(f"bad direction {direction!r}")
    dev = device()
    if not work.is_cuda or not work.is_contiguous():
        raise ValueError("work must be a contiguous CUDA tensor")
    wdt = _lib.WORK_F32 if work.dtype == torch.float32 else _lib.WORK_F64
    if work.dtype not in (torch.float32, torch.float64):
        raise ValueError("work must be float32 or float64")
    cdt = code_dtype_for(radius)
    plan = get_plan(tuple(work.shape), levels, direction=direction, radius=radius,
                    frozen_axes=frozen_axes, md_alpha=md_alpha, rounding=rounding,
                    block_size=block_size, block_table=block_table, work_dtype=wdt,
                    code_dtype=cdt, with_stats=stats is not None and direction == "compress")
    L = lib()
    bind()
    st = stream()
    if direction == "compress":
        if codes is None:
            codes = torch.empty(max(plan.num_codes, 1), dtype=torch_code_dtype(cdt), device=dev)
        if outliers is None:
            outliers = torch.empty(max(plan.num_codes, 1), dtype=torch.float64, device=dev)
        es = cnt = dense = None
        if stats is not None:
            es, cnt, dense = stats.get("err_sum"), stats.get("count"), stats.get("dense")
        if orig is not None:
            if stats is not None or orig.shape != work.shape or orig.dtype != work.dtype \
                    or not orig.is_cuda or not orig.is_contiguous():
                raise ValueError("orig must be a contiguous CUDA tensor like work (no stats)")
            check(L.hpez_sweep_run_from(plan.handle, ptr(orig), ptr(work), ptr(codes), codes.numel(),
                                        ptr(outliers), outliers.numel(), st), "hpez_sweep_run_from")
        else:
            check(L.hpez_sweep_run(plan.handle, ptr(work), ptr(codes), codes.numel(), ptr(outliers),
                                   outliers.numel(), ptr(es), ptr(cnt), ptr(dense), st),
                  "hpez_sweep_run")
        n_out = ctypes.c_int64(0)
        if sync:
            check(L.hpez_sweep_finish(plan.handle, st, ctypes.byref(n_out)), "hpez_sweep_finish")
            if n_out.value > outliers.numel():
                raise RuntimeError("outlier buffer too small")
        return codes[:plan.num_codes], outliers, n_out.value
    if codes is None or outliers is None:
        raise ValueError("decompression needs codes and outliers")
    check(L.hpez_sweep_run(plan.handle, ptr(work), ptr(codes), codes.numel(), ptr(outliers),
                           outliers.numel(), None, None, None, st), "hpez_sweep_run")
    n_out = ctypes.c_int64(0)
    if sync:
        check(L.hpez_sweep_finish(plan.handle, st, ctypes.byref(n_out)), "hpez_sweep_finish")
    return n_out.value


def codes_to_int32(codes) -> np.ndarray:
    """Device code stream (u16 or i32) -> host int32 array."""
    if codes.dtype == torch.int32:
        return codes.cpu().numpy()
    return codes.view(torch.int16).cpu().numpy().view(np.uint16).astype(np.int32)


def f32_exact(a: np.ndarray) -> bool:
    """True when every value survives a float32 round trip bit for bit."""
    if a.size == 0:
        return True
    b = a.astype(np.float32).astype(np.float64)
    return bool(np.array_equal(b.view(np.int64), np.ascontiguousarray(a).view(np.int64)))


def run_levels(work, levels, *, direction: str, radius: int, frozen_axes=(), md_alpha=None,
               rounding=ROUND_NONE, traversal: str = TRAVERSAL_FVFI, block_size: int = 0,
               block_table=None, source: CodeSource | None = None,
               stats: PassStats | None = None):
    """interp.run_levels with the reference's signature (interp.py:440-445),
    executed on the GPU.  Traversal modes are bit-identical by construction
    (interp.py:13-18); both run the same kernels."""
    if direction not in ("compress", "decompress"):
        raise ValueError(f"bad direction {direction!r}")
    if traversal not in (TRAVERSAL_FVFI, TRAVERSAL_DIM_MAJOR):
        raise ValueError(f"bad traversal {traversal!r}")
    if isinstance(work, torch.Tensor):
        raise TypeError("use run_levels_device for tensors")
    if work.dtype != np.float64 or not work.flags.c_contiguous:
        raise ValueError("work must be a C-contiguous float64 array")
    dev = device()
    levels = tuple(levels)
    if md_alpha is None:
        md_alpha = np.ones(work.ndim)
    use_f32 = rounding == ROUND_F32 and f32_exact(work)
    if direction == "decompress":
        if source is None:
            raise ValueError("decompression needs a CodeSource")
        outl_np = source.outliers[source.ocur:]
        use_f32 = use_f32 and f32_exact(outl_np)
    wt = torch.from_numpy(work.astype(np.float32) if use_f32 else work).to(dev)
    if direction == "compress":
        st = None
        if stats is not None:
            st = {"err_sum": torch.from_numpy(stats.err_sum.copy()).to(dev),
                  "count": torch.from_numpy(stats.count.copy()).to(dev),
                  "dense": None}
            if stats.err_grids is not None:
                st["dense"] = torch.zeros((len(levels),) + work.shape, dtype=torch.float64,
                                          device=dev)
        codes, outl, n_out = run_levels_device(
            wt, levels, direction="compress", radius=radius, frozen_axes=frozen_axes,
            md_alpha=md_alpha, rounding=rounding, block_size=block_size,
            block_table=block_table, stats=st)
        work[...] = wt.cpu().numpy().astype(np.float64)
        codes_np = codes_to_int32(codes)
        outl_np = outl[:n_out].cpu().numpy()
        if stats is not None:
            stats.err_sum[:] = st["err_sum"].cpu().numpy()
            stats.count[:] = st["count"].cpu().numpy()
            plan = get_plan(work.shape, levels, direction="compress", radius=radius,
                            frozen_axes=frozen_axes, md_alpha=md_alpha, rounding=rounding,
                            block_size=block_size, block_table=block_table,
                            work_dtype=_lib.WORK_F32 if use_f32 else _lib.WORK_F64,
                            code_dtype=code_dtype_for(radius), with_stats=True)
            lc = plan.level_codes
            for li in range(len(levels)):
                if lc[li + 1] > lc[li]:
                    stats.code_chunks[li].append(codes_np[lc[li]:lc[li + 1]])
            if st["dense"] is not None:
                dn = st["dense"].cpu().numpy()
                for li in range(len(levels)):
                    stats.err_grids[li][...] = dn[li]
        return codes_np, outl_np
    codes_np = source.codes_arr[source.pos:]
    cdt = code_dtype_for(radius)
    if cdt == _lib.CODES_U16:
        if codes_np.size and (codes_np.min() < 0 or codes_np.max() > 65535):
            raise CorruptStream("code out of range for radius")
        codes_t = torch.from_numpy(codes_np.astype(np.uint16)).to(dev)
    else:
        codes_t = torch.from_numpy(np.ascontiguousarray(codes_np, dtype=np.int32)).to(dev)
    outl_t = torch.from_numpy(np.ascontiguousarray(outl_np)).to(dev)
    plan = get_plan(work.shape, levels, direction="decompress", radius=radius,
                    frozen_axes=frozen_axes, md_alpha=md_alpha, rounding=rounding,
                    block_size=block_size, block_table=block_table,
                    work_dtype=_lib.WORK_F32 if use_f32 else _lib.WORK_F64,
                    code_dtype=cdt)
    used = run_levels_device(wt, levels, direction="decompress", radius=radius,
                             frozen_axes=frozen_axes, md_alpha=md_alpha, rounding=rounding,
                             block_size=block_size, block_table=block_table,
                             codes=codes_t, outliers=outl_t)
    work[...] = wt.cpu().numpy().astype(np.float64)
    source.pos += plan.num_codes
    source.ocur += used
    return None
