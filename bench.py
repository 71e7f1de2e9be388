#!/usr/bin/env python
"""bench.py -- HPEZ hot path on B200 (driver contract).

Headline workload (N=1): BASELINE.json configs[3] -- one 512^3 float32
log-normal field exp(G), G a seeded unit-variance k^-3 Gaussian random
field, error bound 1e-3 x value range, full HPEZ auto-tuning (tune() on the
GPU: global / freeze / eb / Lorenzo trials and the per-block table of
tune_blocks), so the sweep runs the mixed block-table path
(interp.py:350-411).  A step is one compress sweep plus one decompress
sweep of that field (interp.run_levels both directions) with the tuned
configuration; inputs resident in HBM, L2 flushed (read of a 256 MiB
buffer) before every timed sweep.  Metric: float32 input GB/s of the round
trip; compress and decompress are also reported with their HBM rooflines.

Also on the same line (never mixed into `value`):
  * parity: the oracle's codes / outliers / reconstruction on the same
    field compared bit for bit with the GPU's (the cpu_baseline run);
  * eps_sweep: the error-bound sweep 1e-2..1e-5 of configs[3] (tune + sweeps);
  * pipeline: tune + sweep + histogram + Huffman pack on the GPU, and the
    archive-level compress()/decompress() with host zlib (threads stated);
  * cfg2: configs[1] (256x384x384, fixed natural cubic + same-level + MD)
    round trip, the round-1 headline, for continuity.

Multi-GPU (torchrun, N>1): BASELINE configs[4] -- each rank tunes and
sweeps its own 512^3 k^-11/3 field (field index = rank, weak scaling),
`value` is the aggregate round-trip GB/s over the max-over-ranks time, and
a batch stage runs multigpu.compress_fields (full archive pipeline per
field, NCCL all-reduce of sizes + send/recv of archives to rank 0) over
one field per rank, timed max over ranks.  `--workload cfg5` runs the same
at N=1 (the scaling baseline).

--impl reference times the reference package itself (baseline/_ref, the
unmodified hpez installed with pip): its interp.run_levels compress +
decompress on 128^3 sub-blocks of the same field, one per host core in a
process pool (the reference is single-threaded per field; cli.py:183-193
batch pattern), with the reference's own tune() of each sub-block (untimed).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress & decompress GB/s of float32 input; achieved % of B200 HBM roofline"
UNIT = "GB/s"
PEAK_FALLBACK = 6650.0
BYTES_COMPRESS = 10  # f32 read + f32 write + u16 code
BYTES_DECOMPRESS = 6  # u16 code read + f32 write
RADIUS = 32768
FLUSH_BYTES = 256 << 20

WORKLOADS = {
    "cfg4": {"cfg": 4, "eps": 1e-3, "tuned": True,
             "desc": "cfg4: 512^3 f32 log-normal exp(G), G a k^-3 GRF (JHTDB shape), eb 1e-3*range, "
                     "full HPEZ auto-tuning (GPU tune(): global/freeze/eb/Lorenzo trials + "
                     "tune_blocks table) -> mixed block-table sweep; step = compress + decompress sweep"},
    "cfg2": {"cfg": 2, "eps": 1e-3, "tuned": False,
             "desc": "cfg2: 256x384x384 f32 k^-5/3 GRF in [0,3] (Miranda shape), eb 1e-3*range, natural "
                     "cubic + same-level + multidim, fixed config (no tuning); step = compress + "
                     "decompress sweep"},
    "cfg5": {"cfg": 5, "eps": 1e-3, "tuned": True,
             "desc": "cfg5: 512^3 f32 k^-11/3 GRF per field (field = rank), eb 1e-3*range, full auto-"
                     "tuning; per rank step = compress + decompress sweep of its own field "
                     "(fields sharded over GPUs, never split)"},
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return PEAK_FALLBACK, "fallback (B200_PROFILING.md)"


class Clocks:
    """NVML sampler (background thread, ~1 kHz) running during the timed region:
    SM clock, max SM clock and the active clock-event (throttle) reasons."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, cuda_index):
        self.cuda_index = cuda_index
        self.samples, self.reasons, self.max = [], set(), None
        self._stop = False
        self._t = None

    def _run(self, h, nv):
        while not self._stop:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                break
            time.sleep(0.001)

    def __enter__(self):
        try:
            import threading
            import pynvml as nv
            import torch
            nv.nvmlInit()
            pr = torch.cuda.get_device_properties(self.cuda_index)
            bus = f"{int(pr.pci_domain_id):08X}:{int(pr.pci_bus_id):02X}:{int(pr.pci_device_id):02X}.0"
            try:
                h = nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                h = nv.nvmlDeviceGetHandleByIndex(self.cuda_index)
            self.max = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, args=(h, nv), daemon=True)
            self._t.start()
            time.sleep(0.003)
        except Exception:
            self._t = None
        return self

    def __exit__(self, *a):
        self._stop = True
        if self._t is not None:
            self._t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max, "samples": len(self.samples),
                "reasons": sorted(self.reasons), "source": "nvml"}


# ------------------------------------------------------------ distributed --
def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# -------------------------------------------------------------- workloads --
def fixed_cfg2_config(grid, eb):
    """configs[1]'s fixed configuration."""
    from paper_2311_12133_b200.plan import (KERNEL_VARIANTS, PARADIGM_MULTIDIM, CompressionConfig,
                                            LevelConfig)
    from paper_2311_12133_b200.tuner import analyze_samples, blend_weights_f32
    lc = LevelConfig(KERNEL_VARIANTS[4], PARADIGM_MULTIDIM)  # natural cubic, same-level
    md = blend_weights_f32(analyze_samples(grid, 0.002))
    return CompressionConfig(predictor="interp", resolved_bound=eb, radius=RADIUS, anchor_stride=64,
                             level_configs=(lc,) * 6, md_alpha=tuple(md))


def make_levels(ebound, dims=(256, 384, 384)):
    """cfg2's fixed level plan (natural cubic + same-level + MD at every level)."""
    from paper_2311_12133_b200.plan import (KERNEL_VARIANTS, PARADIGM_MULTIDIM, LevelConfig,
                                            build_level_plan)
    cfg = LevelConfig(KERNEL_VARIANTS[4], PARADIGM_MULTIDIM)
    return build_level_plan(dims, 64, ebound, 1.0, 1.0, None, [cfg] * 6).levels


def md_weights_for(field):
    """The reference's MD blend weights for a field (f32 header values)."""
    from paper_2311_12133_b200.grid import ElementKind, ScalarGrid
    from paper_2311_12133_b200.tuner import analyze_samples, blend_weights_f32
    g = ScalarGrid(field.shape, ElementKind.F32, field)
    return np.asarray(blend_weights_f32(analyze_samples(g, 0.002)), dtype=np.float64)


class Prepared:
    """A field in host and device memory with its (tuned or fixed)
    configuration, as the pipeline would run it (config header round trip
    included: MD weights are the f32 values a decompressor sees)."""

    def __init__(self, wl_name, index, dev, eps=None):
        import torch
        import synthetic as syn
        from paper_2311_12133_b200.container import parse_config, serialize_config
        from paper_2311_12133_b200.grid import ElementKind, ScalarGrid
        from paper_2311_12133_b200.pipeline import _plan
        from paper_2311_12133_b200.tuner import tune
        wl = WORKLOADS[wl_name]
        self.name = wl_name
        self.field = syn.config_field(wl["cfg"], index=index, device=dev)
        self.grid = ScalarGrid(self.field.shape, ElementKind.F32, self.field)
        self.eps = wl["eps"] if eps is None else eps
        self.eb = self.eps * float(self.field.max() - self.field.min())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cfg = tune(self.grid, self.eb) if wl["tuned"] else fixed_cfg2_config(self.grid, self.eb)
        torch.cuda.synchronize()
        self.tune_s = time.perf_counter() - t0
        self.cfg = parse_config(serialize_config(cfg, self.grid.dims), self.grid.dims)
        if self.cfg.predictor != "interp":
            raise RuntimeError(f"tuner chose {self.cfg.predictor}; the sweep bench needs interp")
        self.levels = _plan(self.grid.dims, self.cfg).levels
        self.frozen = () if self.cfg.frozen_dim is None else (self.cfg.frozen_dim,)
        self.kw = dict(radius=self.cfg.radius, frozen_axes=self.frozen,
                       md_alpha=np.asarray(self.cfg.md_alpha, dtype=np.float64), rounding=1,
                       block_size=self.cfg.block_size, block_table=self.cfg.block_table)
        self.dims = tuple(self.field.shape)
        self.n = self.field.size
        self.sel = tuple(slice(0, None, 1 if a in self.frozen else self.cfg.anchor_stride)
                         for a in range(len(self.dims)))

    def tags(self):
        t = self.cfg.block_table
        return None if t is None else [int(np.unique(r).size) for r in t]

    def level_tuples(self):
        from paper_2311_12133_b200.plan import PARADIGM_MULTIDIM, kernel_index
        return [(s.stride, s.bound, kernel_index(s.config.kernel),
                 1 if s.config.paradigm == PARADIGM_MULTIDIM else 0, s.config.axis_order)
                for s in self.levels]


def sweep_bench(P, steps, warmup, dev):
    """Device-resident compress + decompress sweeps, CUDA events, L2 flushed
    by a read before each timed sweep.  Returns per-step ms lists and the
    gate run's outputs (codes, outliers, reconstruction)."""
    import torch
    from paper_2311_12133_b200 import _lib
    from paper_2311_12133_b200.interp import code_dtype_for, get_plan, run_levels_device
    orig = torch.from_numpy(P.field).to(dev)
    work = torch.empty_like(orig)
    back = torch.zeros_like(orig)
    anchors0 = torch.zeros_like(orig)
    anchors0[P.sel] = orig[P.sel]
    flush = torch.ones(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    sink = torch.empty(1, dtype=torch.float32, device=dev)
    kw = P.kw
    t0 = time.perf_counter()
    pc = get_plan(P.dims, P.levels, direction="compress", work_dtype=_lib.WORK_F32,
                  code_dtype=code_dtype_for(kw["radius"]), **kw)
    pd = get_plan(P.dims, P.levels, direction="decompress", work_dtype=_lib.WORK_F32,
                  code_dtype=code_dtype_for(kw["radius"]), **kw)
    plan_ms = 1e3 * (time.perf_counter() - t0)
    codes = torch.empty(pc.num_codes, dtype=torch.uint16, device=dev)
    outl = torch.empty(pc.num_codes, dtype=torch.float64, device=dev)

    def l2_flush():  # a read larger than L2 (evicts and writes back dirty lines untimed)
        torch.amax(flush, dim=0, keepdim=True, out=sink)

    def step(events=None):
        work.copy_(orig)
        l2_flush()
        if events:
            events[0].record()
        run_levels_device(work, P.levels, direction="compress", codes=codes, outliers=outl,
                          sync=False, **kw)
        if events:
            events[1].record()
        back.copy_(anchors0)
        l2_flush()
        if events:
            events[2].record()
        run_levels_device(back, P.levels, direction="decompress", codes=codes, outliers=outl,
                          sync=False, **kw)
        if events:
            events[3].record()

    # correctness gate on the full-size field: exact round trip + bound (the
    # first run also performs the plans' one-time device setup)
    work.copy_(orig)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, _, n_out = run_levels_device(work, P.levels, direction="compress", codes=codes,
                                    outliers=outl, **kw)
    first_ms = 1e3 * (time.perf_counter() - t0)
    back.copy_(anchors0)
    run_levels_device(back, P.levels, direction="decompress", codes=codes, outliers=outl, **kw)
    assert torch.equal(back, work), "decompressed grid differs from the compressor's"
    err = float((back.double() - orig.double()).abs().max())
    assert err <= P.eb, f"bound violated: {err} > {P.eb}"
    gate = {"codes": codes.clone(), "outl": outl[:n_out].clone(), "work": work.clone(),
            "n_out": int(n_out), "max_err": err,
            "plan": {"host_build_ms": round(plan_ms, 2), "first_compress_ms_incl_setup": round(first_ms, 2),
                     "commits": int(lib_commits(pc)), "launches_per_sweep": [pc.num_launches, pd.num_launches]}}
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    return ev, step, gate, pc, pd


def lib_commits(plan):
    from paper_2311_12133_b200 import _lib
    return _lib.lib().hpez_plan_num_commits(plan.handle)


def e2e_bench(P, steps, warmup, dev, n_out, pc):
    """Same round trip through the run_levels C-ABI call from pinned host
    buffers: H2D of the field, compress, D2H of the compressed stream
    (codes + outliers), H2D of it again, decompress, D2H of the field.
    Steps rotate over three streams so one step's copies overlap the next
    step's sweeps; the host never waits inside a step."""
    import torch
    from paper_2311_12133_b200.interp import run_levels_device
    kw = P.kw
    host_in = torch.from_numpy(P.field).pin_memory()
    ocap = max(4096, 2 * n_out)
    slots = []
    nslots = 3
    for _ in range(nslots):
        slots.append({
            "s": torch.cuda.Stream(device=dev),
            "work": torch.empty(P.dims, dtype=torch.float32, device=dev),
            "back": torch.empty(P.dims, dtype=torch.float32, device=dev),
            "codes": torch.empty(pc.num_codes, dtype=torch.uint16, device=dev),
            "outl": torch.empty(pc.num_codes, dtype=torch.float64, device=dev),
            "codes_h": torch.empty(pc.num_codes, dtype=torch.uint16).pin_memory(),
            "back_h": torch.empty(P.dims, dtype=torch.float32).pin_memory(),
            "outl_h": torch.empty(ocap, dtype=torch.float64).pin_memory(),
            "anch_h": torch.from_numpy(np.ascontiguousarray(P.field[P.sel])).pin_memory(),
        })

    def e2e_step(sl):
        with torch.cuda.stream(sl["s"]):
            w_, b_ = sl["work"], sl["back"]
            w_.copy_(host_in, non_blocking=True)
            run_levels_device(w_, P.levels, direction="compress", codes=sl["codes"],
                              outliers=sl["outl"], sync=False, **kw)
            sl["codes_h"].copy_(sl["codes"], non_blocking=True)
            sl["outl_h"].copy_(sl["outl"][:ocap], non_blocking=True)
            sl["codes"].copy_(sl["codes_h"], non_blocking=True)
            sl["outl"][:ocap].copy_(sl["outl_h"], non_blocking=True)
            b_[P.sel] = sl["anch_h"].to(dev, non_blocking=True)  # decompress writes every non-anchor
            run_levels_device(b_, P.levels, direction="decompress", codes=sl["codes"],
                              outliers=sl["outl"], sync=False, **kw)
            sl["back_h"].copy_(b_, non_blocking=True)

    for k in range(max(warmup, nslots)):
        e2e_step(slots[k % nslots])
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(main)
    for sl in slots:
        sl["s"].wait_event(t0)
    for k in range(steps):
        e2e_step(slots[k % nslots])
    for sl in slots:
        main.wait_stream(sl["s"])
    t1.record(main)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    h2d = 4 * P.n + 2 * pc.num_codes + 8 * ocap + 4 * slots[0]["anch_h"].numel()
    d2h = 2 * pc.num_codes + 8 * ocap + 4 * P.n
    return ms, [sl["back_h"] for sl in slots[:min(nslots, steps)]], int(h2d), int(d2h)


def oracle_round_trip(P, gate):
    """The scalar C oracle (oracle/hpez_oracle.c, a restatement of the
    reference algorithm) on the full field: timed round trip (cpu_baseline)
    and bit-exact comparison with the GPU gate run (parity)."""
    from oracle import oracle
    from paper_2311_12133_b200.interp import codes_to_int32
    work = P.field.astype(np.float64)
    lv = P.level_tuples()
    okw = dict(radius=P.cfg.radius, frozen_axes=P.frozen, md_alpha=P.kw["md_alpha"], rounding=1,
               block_size=P.cfg.block_size, block_table=P.cfg.block_table)
    t0 = time.perf_counter()
    c, o = oracle.run_levels(work, lv, direction="compress", **okw)
    back = np.zeros_like(work)
    back[P.sel] = work[P.sel]
    oracle.run_levels(back, lv, direction="decompress", codes=c, outliers=o, **okw)
    dt = time.perf_counter() - t0
    cg = codes_to_int32(gate["codes"])
    same_shape = cg.shape == c.shape
    mism = int((cg != c).sum()) if same_shape else int(max(cg.size, c.size))
    parity = {"codes_equal": bool(same_shape and mism == 0),
              "mismatch_frac": mism / max(c.size, 1), "n_codes": int(c.size),
              "outliers_equal": gate["outl"].cpu().numpy().tobytes() == o.tobytes(),
              "recon_equal": bool(np.array_equal(gate["work"].cpu().numpy().astype(np.float64), work)),
              "oracle_decompress_equal": bool(np.array_equal(back, work)),
              "checker": "oracle/hpez_oracle.c on the full field, same bytes and configuration"}
    return dt, parity


def pipeline_figures(P, dev):
    """GPU pipeline (tune + compress sweep + histogram + Huffman pack) and the
    archive-level compress()/decompress() with host zlib, reported apart
    from the sweep roofline."""
    import torch
    from paper_2311_12133_b200 import container, pipeline
    from paper_2311_12133_b200.grid import BoundMode, ErrorBoundSpec
    from paper_2311_12133_b200.interp import run_levels_device
    orig = torch.from_numpy(P.field).to(dev)
    work = orig.clone()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    codes, outl, n_out = run_levels_device(work, P.levels, direction="compress", **P.kw)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    framed = container.pack_codes_pinned(codes)  # the pipeline's path (pinned frame, no host copies)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    gpu_s = P.tune_s + (t1 - t0) + (t2 - t1)
    spec = ErrorBoundSpec(BoundMode.REL, P.eps)
    t3 = time.perf_counter()
    res = pipeline.compress(P.grid, spec)
    t4 = time.perf_counter()
    back = pipeline.decompress(res.archive)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    assert np.array_equal(back.data, res.reconstruction.data)
    gb = P.n * 4 / 1e9
    return {
        "gpu_pipeline": {"tune_s": round(P.tune_s, 3), "sweep_ms": round(1e3 * (t1 - t0), 3),
                         "huffman_pack_ms": round(1e3 * (t2 - t1), 3),
                         "seconds": round(gpu_s, 3), "gbs": round(gb / gpu_s, 4),
                         "payload_bytes": len(framed)},
        "archive": {"compress_s": round(t4 - t3, 3), "decompress_s": round(t5 - t4, 3),
                    "compress_gbs": round(gb / (t4 - t3), 4), "decompress_gbs": round(gb / (t5 - t4), 4),
                    "ratio": round(res.ratio, 3), "zlib_threads": pipeline.lossless_threads(),
                    "note": "pipeline.compress/decompress: GPU tune + sweep + Huffman, host zlib level 6 "
                            "(libz 1.3, byte-identical archives); zlib streams run on a thread pool"},
    }


def e2e_dropin(P, reps=2):
    """The reference-signature drop-in interp.run_levels(np.ndarray f64, ...)
    (interp.py:440-445) timed on the headline field: host f64 work in,
    codes/outliers back as numpy, decompress through a CodeSource, host f64
    out -- what a caller binding the reference sees."""
    from paper_2311_12133_b200.interp import CodeSource, run_levels
    kw = {k: v for k, v in P.kw.items()}
    best = None
    for _ in range(reps):
        work = P.field.astype(np.float64)
        t0 = time.perf_counter()
        codes, outl = run_levels(work, P.levels, direction="compress", **kw)
        back = np.zeros_like(work)
        back[P.sel] = work[P.sel]
        run_levels(back, P.levels, direction="decompress", source=CodeSource(codes, outl), **kw)
        dt = time.perf_counter() - t0
        assert np.array_equal(back, work)
        best = dt if best is None else min(best, dt)
    return {"value": round(P.n * 4 / 1e9 / best, 3), "unit": UNIT, "seconds": round(best, 3),
            "path": "interp.run_levels drop-in with the reference's numpy f64 arrays (host work in place, "
                    "int32 codes / f64 outliers returned, CodeSource decompress); includes the f32-exactness "
                    "scans and the f64<->f32 host conversions"}


def eps_sweep(dev, eps_list, steps=3):
    """configs[3]'s error-bound sweep: tune at each bound, then device sweeps."""
    import torch
    out = []
    for eps in eps_list:
        P = Prepared("cfg4", 0, dev, eps=eps)
        ev, step, gate, pc, pd = sweep_bench(P, steps, 1, dev)
        for k in range(steps):
            step(ev[k])
        torch.cuda.synchronize()
        tc = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
        td = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
        out.append({"eps": eps, "tune_s": round(P.tune_s, 3), "compress_ms": round(tc, 4),
                    "decompress_ms": round(td, 4), "outliers": gate["n_out"],
                    "distinct_tags_per_level": P.tags(),
                    "roundtrip_gbs": round(P.n * 4 / 1e9 / ((tc + td) / 1e3), 2)})
        del ev, step, gate
    return out


def run_b200(args):
    import torch
    world, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    wl_name = args.workload or ("cfg5" if world > 1 else "cfg4")
    P = Prepared(wl_name, rank if wl_name == "cfg5" else 0, dev)
    ev, step, gate, pc, pd = sweep_bench(P, args.steps, args.warmup, dev)
    barrier(world)
    torch.cuda.synchronize()
    clk = Clocks(local).__enter__()  # sampled over both timed regions (sweeps, then e2e)
    for k in range(args.steps):
        step(ev[k])
    torch.cuda.synchronize()
    barrier(world)
    tc = [e[0].elapsed_time(e[1]) for e in ev]
    td = [e[2].elapsed_time(e[3]) for e in ev]
    t_total = max_over_ranks(sum(tc) + sum(td), world)  # ms of sweep time
    tc_mean = max_over_ranks(float(np.mean(tc)), world)
    td_mean = max_over_ranks(float(np.mean(td)), world)
    e2e_ms, backs, h2d, d2h = e2e_bench(P, args.steps, args.warmup, dev, gate["n_out"], pc)
    clk.__exit__()
    recon = gate["work"].cpu()
    for b in backs:
        assert torch.equal(b, recon), "e2e round trip differs"
    e2e_ms = max_over_ranks(e2e_ms, world)

    peak, peak_src = peaks()
    n = P.n
    gb = n * 4 / 1e9
    ach_c = BYTES_COMPRESS * n / (tc_mean / 1e3) / 1e9
    ach_d = BYTES_DECOMPRESS * n / (td_mean / 1e3) / 1e9
    value = world * gb * args.steps / (t_total / 1e3)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{wl_name}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tb = json.load(f).get("compress_dram_bytes_per_sweep")
        traffic = None if tb is None else round(tb / (tc_mean / 1e3) / 1e9, 1)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_total / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 arithmetic on f32 grid",
        "data": "synthetic (seeded GRFs per BASELINE.json; SDRBench stand-ins, no datasets here)",
        "config": {"workload": WORKLOADS[wl_name]["desc"], "dims": list(P.dims),
                   "error_bound": f"{P.eps:g} x value range", "radius": P.cfg.radius,
                   "fields_per_gpu": 1, "parallelism": f"field-sharded x{world}",
                   "tuned": {"tune_s": round(P.tune_s, 3), "frozen_dim": P.cfg.frozen_dim,
                             "alpha_beta": [P.cfg.alpha, P.cfg.beta],
                             "block_size": P.cfg.block_size,
                             "distinct_tags_per_level": P.tags(),
                             "level_configs": [f"{c.kernel.tag.value}{'+SL' if c.kernel.same_level else ''}/"
                                               f"{c.paradigm}{'' if c.axis_order is None else list(c.axis_order)}"
                                               for c in P.cfg.level_configs]},
                   "l2": "flushed by a 256 MiB read before every timed sweep"},
        "compress": {"ms": round(tc_mean, 4), "gbs_f32_input": round(gb / (tc_mean / 1e3), 2),
                     "achieved_gbs": round(ach_c, 1), "frac": round(ach_c / peak, 4)},
        "decompress": {"ms": round(td_mean, 4), "gbs_f32_input": round(gb / (td_mean / 1e3), 2),
                       "achieved_gbs": round(ach_d, 1), "frac": round(ach_d / peak, 4)},
        "roofline": {"bound": "hbm", "achieved": round(ach_c, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(ach_c / peak, 4), "traffic": traffic,
                     "traffic_note": f"ncu dram__bytes_read+write of one compress sweep "
                                     f"(profiles/traffic_{wl_name}.json) over this run's sweep time, GB/s",
                     "kernel": "compress sweep of one run_levels (coarse DSMEM cluster + flow kernel for the "
                               "coarse levels + row-fused launches for strides 4/2/1 + escape scan/gather); the "
                               "stride-1 row launches are ~72% of it",
                     "algorithmic_bytes": f"{BYTES_COMPRESS} B/pt x {n} pts",
                     "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)"},
        "e2e": {"value": round(world * gb / (e2e_ms / 1e3), 3), "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "run_levels C-ABI round trip from pinned host buffers (field in, compressed "
                        "stream out and back in, field out), steps pipelined over 3 streams"},
        "gpu_launches": int(args.steps * (pc.num_launches + pd.num_launches)),
        "outliers": gate["n_out"], "max_abs_err": gate["max_err"], "error_bound": P.eb,
        "plan": gate["plan"],
    }
    line["clocks"] = clk.summary() if rank == 0 else None
    if world > 1 or wl_name == "cfg5":
        line["batch"] = batch_stage(world, rank, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dt, parity = oracle_round_trip(P, gate)
        line["parity"] = parity
        line["cpu_baseline"] = {"value": round(n * 4 / 1e9 / dt, 4), "unit": UNIT, "cores": 1,
                                "kind": "port",
                                "sample": f"full {wl_name} field, one compress+decompress round trip "
                                          "with the same tuned configuration, scalar C oracle "
                                          "(oracle/hpez_oracle.c), 1 thread"}
    if rank == 0 and world == 1 and wl_name == "cfg4" and not args.quick:
        line["pipeline"] = pipeline_figures(P, dev)
        line["e2e_dropin"] = e2e_dropin(P)
        del ev, step, gate
        line["eps_sweep"] = eps_sweep(dev, [1e-2, 1e-3, 1e-4, 1e-5])
        line["cfg2"] = secondary_cfg2(dev, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def secondary_cfg2(dev, args):
    """configs[1] round trip (round-1 headline), same method, fewer steps."""
    import torch
    P = Prepared("cfg2", 0, dev)
    steps = max(3, min(args.steps, 10))
    ev, step, gate, pc, pd = sweep_bench(P, steps, 3, dev)
    for k in range(steps):
        step(ev[k])
    torch.cuda.synchronize()
    tc = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    td = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
    peak, _ = peaks()
    out = {"workload": WORKLOADS["cfg2"]["desc"], "dims": list(P.dims),
           "value": round(P.n * 4 / 1e9 / ((tc + td) / 1e3), 3), "unit": UNIT,
           "compress": {"ms": round(tc, 4), "frac": round(BYTES_COMPRESS * P.n / (tc / 1e3) / 1e9 / peak, 4)},
           "decompress": {"ms": round(td, 4), "frac": round(BYTES_DECOMPRESS * P.n / (td / 1e3) / 1e9 / peak, 4)},
           "outliers": gate["n_out"]}
    if not args.no_cpu_baseline:
        dt, parity = oracle_round_trip(P, gate)
        out["parity"] = parity
        out["cpu_baseline_gbs"] = round(P.n * 4 / 1e9 / dt, 4)
    return out


def batch_stage(world, rank, dev):
    """configs[4] batch path: multigpu.compress_fields over one cfg5 field per
    rank -- tune, sweep, Huffman pack, zlib per field on its owner, NCCL
    all-reduce of archive sizes and send/recv of the archives to rank 0.
    Timed max over ranks; rank 0 checks every archive decodes."""
    import torch
    import torch.distributed as dist
    import synthetic as syn
    from paper_2311_12133_b200 import multigpu
    from paper_2311_12133_b200.grid import BoundMode, ElementKind, ErrorBoundSpec, ScalarGrid
    own_pg = False
    if not dist.is_initialized():  # --workload cfg5 at N=1: a one-rank group
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29577")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        own_pg = True

    def make(i):
        return ScalarGrid((512, 512, 512), ElementKind.F32, syn.config_field(5, index=i, device=dev))

    n_fields = world
    spec = ErrorBoundSpec(BoundMode.REL, 1e-3)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    arcs = multigpu.compress_fields(make, n_fields, spec)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dt = float(t.item())
    out = {"fields": n_fields, "seconds": round(dt, 3),
           "gbs_f32_input": round(n_fields * 512 ** 3 * 4 / 1e9 / dt, 4),
           "path": "multigpu.compress_fields: per field tune + sweep + Huffman pack + zlib on its "
                   "owner GPU/host, NCCL all-reduce of sizes + send/recv of archives to rank 0"}
    if rank == 0:
        out["archive_bytes"] = [len(a) for a in arcs]
    if own_pg:
        dist.destroy_process_group()
    return out


# -------------------------------------------------------- reference arm --
REF_PATH = os.path.join(ROOT, "baseline", "_ref")
SUB = 128  # sub-block edge of the bounded CPU sample


def _ref_worker(payload):
    """One reference sweep round trip (hpez.interp.run_levels) of a sub-block,
    with the reference's own tuned configuration; returns seconds."""
    block, cfg_state, steps = payload
    sys.path.insert(0, REF_PATH)
    import hpez  # noqa: F401  (the unmodified reference)
    from hpez import interp
    from hpez.container import parse_config
    from hpez.pipeline import _interp_plan
    dims, cfg_bytes = cfg_state
    cfg = parse_config(cfg_bytes, dims)
    plan = _interp_plan(dims, cfg)
    frozen = () if cfg.frozen_dim is None else (cfg.frozen_dim,)
    kw = dict(radius=cfg.radius, frozen_axes=frozen, md_alpha=np.asarray(cfg.md_alpha), rounding=1,
              block_size=cfg.block_size, block_table=cfg.block_table)
    times = []
    for _ in range(steps):
        work = block.astype(np.float64)
        t0 = time.perf_counter()
        codes, outl = interp.run_levels(work, plan.levels, direction="compress", **kw)
        back = np.zeros_like(work)
        sel = tuple(slice(0, None, 1 if a in frozen else cfg.anchor_stride) for a in range(3))
        back[sel] = work[sel]
        interp.run_levels(back, plan.levels, direction="decompress",
                          source=interp.CodeSource(codes, outl), **kw)
        times.append(time.perf_counter() - t0)
    return times


def _ref_tune(block_and_eps):
    block, eps = block_and_eps
    sys.path.insert(0, REF_PATH)
    import hpez
    from hpez.container import serialize_config
    g = hpez.ScalarGrid(block.shape, hpez.ElementKind.F32, block)
    eb = hpez.ErrorBoundSpec(hpez.BoundMode.REL, eps).resolve(g)
    cfg = hpez.tune(g, eb)
    if cfg.predictor != "interp":
        return None
    return (block.shape, serialize_config(cfg, block.shape))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import multiprocessing as mp
    import synthetic as syn
    wl_name = args.workload or ("cfg5" if world > 1 else "cfg4")
    wl = WORKLOADS[wl_name]
    cores = os.cpu_count() or 1
    if not os.path.isdir(os.path.join(REF_PATH, "hpez")):
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref/hpez not installed"}))
        return
    field = syn.config_field(wl["cfg"], index=0)
    # bounded sample: one SUB^3 sub-block per worker, taken from the field
    nb = [d // SUB for d in field.shape]
    blocks = []
    for w in range(cores):
        k = w % int(np.prod(nb))
        i, j, l = np.unravel_index(k, nb)
        blocks.append(np.ascontiguousarray(field[i * SUB:(i + 1) * SUB, j * SUB:(j + 1) * SUB,
                                                 l * SUB:(l + 1) * SUB]))
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        states = pool.map(_ref_tune, [(b, wl["eps"]) for b in blocks])  # untimed (reference tune())
        work = [(b, s, 1) for b, s in zip(blocks, states) if s is not None]
        for _ in range(args.warmup):
            pool.map(_ref_worker, work)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            pool.map(_ref_worker, work)
            times.append(time.perf_counter() - t0)
    gb = len(work) * SUB ** 3 * 4 / 1e9
    value = gb * len(times) / sum(times)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 arithmetic on f32 grid",
        "data": "synthetic (seeded GRFs per BASELINE.json)",
        "config": {"workload": wl["desc"], "dims": list(field.shape),
                   "error_bound": f"{wl['eps']:g} x value range", "radius": RADIUS},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{len(work)} workers x one {SUB}^3 sub-block of the {wl_name} field "
                                   f"each, the unmodified reference (baseline/_ref hpez) "
                                   f"interp.run_levels compress+decompress with its own tune() of the "
                                   f"sub-block (untimed); one process per core (cli.py:183-193 pattern)"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip the pipeline / eps-sweep / cfg2 extras")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
