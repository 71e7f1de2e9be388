#!/usr/bin/env python
"""bench.py -- HPEZ hot path on B200 (driver contract).

Workload (BASELINE.json configs[1]): one 256x384x384 float32 field (seeded
k^-5/3 Gaussian random field scaled to [0, 3]), error bound 1e-3 x range,
natural cubic spline with same-level re-ordering and multi-dimensional
interpolation, no tuning.  A step is one compress sweep plus one decompress
sweep of that field (interp.run_levels both directions), inputs resident in
HBM.  Metric: float32 input GB/s of the round trip; compress and decompress
are also reported separately with their HBM rooflines.

--impl reference times the CPU restatement of the same path (oracle/, the
reference's own algorithm; the reference itself is pure Python and is not
on the GPU box) on all host cores, one field round trip per worker.
Multi-GPU (torchrun): each rank compresses its own field (weak scaling, no
collective on the data path); rank 0 prints the max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress & decompress GB/s of float32 input; achieved % of B200 HBM roofline"
UNIT = "GB/s"
DIMS = (256, 384, 384)
EPS = 1e-3
PEAK_FALLBACK = 6650.0
BYTES_COMPRESS = 10  # f32 read + f32 write + u16 code
BYTES_DECOMPRESS = 6  # u16 code read + f32 write


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return PEAK_FALLBACK, "fallback"


def workload_config(n_gpus):
    return {"workload": "cfg2: 256x384x384 f32 k^-5/3 GRF in [0,3], eb 1e-3*range, natural cubic "
                        "+ same-level + multidim, fixed config (no tuning); step = compress + "
                        "decompress sweep",
            "dims": list(DIMS), "error_bound": "1e-3 x value range", "radius": 32768,
            "fields_per_gpu": 1, "parallelism": f"field-sharded x{n_gpus}",
            "l2": "flushed (256 MiB write) before every timed sweep"}


def make_levels(ebound):
    from paper_2311_12133_b200.plan import (KERNEL_VARIANTS, PARADIGM_MULTIDIM, LevelConfig,
                                            build_level_plan)
    cfg = LevelConfig(KERNEL_VARIANTS[4], PARADIGM_MULTIDIM)  # natural cubic, same-level
    return build_level_plan(DIMS, 64, ebound, 1.0, 1.0, None, [cfg] * 6).levels


def md_weights_for(field):
    from paper_2311_12133_b200.grid import ElementKind, ScalarGrid
    from paper_2311_12133_b200.tuner import analyze_samples, blend_weights_f32
    g = ScalarGrid(field.shape, ElementKind.F32, field)
    return np.asarray(blend_weights_f32(analyze_samples(g, 0.002)), dtype=np.float64)


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


def dist_setup(n_gpus):
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


def run_b200(args):
    import torch
    import synthetic as syn
    from paper_2311_12133_b200.interp import get_plan, run_levels_device, code_dtype_for
    from paper_2311_12133_b200 import _lib

    world, rank, local = dist_setup(args.gpus)
    dev = torch.device("cuda", local)
    field = syn.config_field(2, index=rank, device=dev)
    ebound = EPS * float(field.max() - field.min())
    levels = make_levels(ebound)
    md = md_weights_for(field)
    n = field.size
    orig = torch.from_numpy(field).to(dev)
    work = torch.empty_like(orig)
    back = torch.zeros_like(orig)
    anchors0 = torch.zeros_like(orig)
    anchors0[::64, ::64, ::64] = orig[::64, ::64, ::64]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    kw = dict(radius=32768, md_alpha=md, rounding=1)
    pc = get_plan(DIMS, levels, direction="compress", work_dtype=_lib.WORK_F32,
                  code_dtype=code_dtype_for(32768), **kw)
    pd = get_plan(DIMS, levels, direction="decompress", work_dtype=_lib.WORK_F32,
                  code_dtype=code_dtype_for(32768), **kw)
    codes = torch.empty(pc.num_codes, dtype=torch.uint16, device=dev)
    outl = torch.empty(pc.num_codes, dtype=torch.float64, device=dev)

    # run_levels semantics (interp.py:440-472): compress works in place on a
    # fresh copy of the field (pipeline.py:82 work = f64(grid), untimed)
    def step(events=None):
        work.copy_(orig)
        flush.fill_(1.0)
        if events:
            events[0].record()
        run_levels_device(work, levels, direction="compress", codes=codes, outliers=outl,
                          sync=False, **kw)
        if events:
            events[1].record()
        back.copy_(anchors0)
        flush.fill_(2.0)
        if events:
            events[2].record()
        run_levels_device(back, levels, direction="decompress", codes=codes, outliers=outl,
                          sync=False, **kw)
        if events:
            events[3].record()

    # correctness gate on the full-size field: exact round trip + bound
    step()
    torch.cuda.synchronize()
    _, _, n_out = run_levels_device(work.copy_(orig), levels, direction="compress", codes=codes,
                                    outliers=outl, **kw)
    back.copy_(anchors0)
    run_levels_device(back, levels, direction="decompress", codes=codes, outliers=outl, **kw)
    assert torch.equal(back, work), "decompressed grid differs from the compressor's"
    err = float((back.double() - orig.double()).abs().max())
    assert err <= ebound, f"bound violated: {err} > {ebound}"

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    barrier(world)
    torch.cuda.synchronize()
    clk = Clocks(local).__enter__()  # sampled over both timed regions (sweeps, then e2e)
    for k in range(args.steps):
        step(ev[k])
    torch.cuda.synchronize()
    barrier(world)
    tc = [e[0].elapsed_time(e[1]) for e in ev]
    td = [e[2].elapsed_time(e[3]) for e in ev]
    t_total = sum(tc) + sum(td)  # ms of sweep time on this rank
    t_total = max_over_ranks(t_total, world)
    tc_mean = max_over_ranks(float(np.mean(tc)), world)
    td_mean = max_over_ranks(float(np.mean(td)), world)

    # e2e through the run_levels boundary with host (pinned) buffers: every
    # step copies its field in, compresses, reads codes + outliers back (the
    # compressed stream), copies them in again, decompresses and reads the
    # field back.  Steps alternate over two streams with their own buffers
    # (and their own plans), so one step's device->host copies overlap the
    # next step's host->device copies and sweeps (PCIe is full duplex).
    host_in = torch.from_numpy(field).pin_memory()
    anch_h = orig[::64, ::64, ::64].cpu().pin_memory()
    slots = []
    nslots = int(os.environ.get("HPEZ_E2E_SLOTS", 3))
    for _ in range(nslots):
        slots.append({
            "s": torch.cuda.Stream(device=dev),
            "work": torch.empty_like(orig), "back": torch.empty_like(orig),
            "codes": torch.empty(pc.num_codes, dtype=torch.uint16, device=dev),
            "outl": torch.empty(pc.num_codes, dtype=torch.float64, device=dev),
            "codes_h": torch.empty(pc.num_codes, dtype=torch.uint16).pin_memory(),
            "back_h": torch.empty(DIMS, dtype=torch.float32).pin_memory(),
            "outl_h": torch.empty(max(4096, 2 * n_out), dtype=torch.float64).pin_memory(),
        })

    # the host never waits inside a step (sync=False): the outlier stream is
    # moved with a fixed capacity (the gate run above found n_out of them)
    ocap = max(4096, 2 * n_out)

    def e2e_step(sl):
        with torch.cuda.stream(sl["s"]):
            w_, b_ = sl["work"], sl["back"]
            w_.copy_(host_in, non_blocking=True)
            run_levels_device(w_, levels, direction="compress", codes=sl["codes"],
                              outliers=sl["outl"], sync=False, **kw)
            sl["codes_h"].copy_(sl["codes"], non_blocking=True)
            sl["outl_h"][:ocap].copy_(sl["outl"][:ocap], non_blocking=True)
            # decompress from the host streams
            sl["codes"].copy_(sl["codes_h"], non_blocking=True)
            sl["outl"][:ocap].copy_(sl["outl_h"][:ocap], non_blocking=True)
            b_[::64, ::64, ::64] = anch_h.to(dev, non_blocking=True)  # decompress writes every other point
            run_levels_device(b_, levels, direction="decompress", codes=sl["codes"],
                              outliers=sl["outl"], sync=False, **kw)
            sl["back_h"].copy_(b_, non_blocking=True)
        return ocap

    for k in range(args.warmup):
        e2e_step(slots[k % nslots])
    torch.cuda.synchronize()
    flush.fill_(3.0)
    main = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(main)
    for sl in slots:
        sl["s"].wait_event(t0)
    no = 0
    for k in range(args.steps):
        no = e2e_step(slots[k % nslots])
    for sl in slots:
        main.wait_stream(sl["s"])
    t1.record(main)
    torch.cuda.synchronize()
    clk.__exit__()
    e2e = [t0.elapsed_time(t1) / args.steps]
    # checked outside the timed region: every slot's decompressed field equals
    # the compressor's reconstruction of the gate run (still in `work`)
    recon = work.cpu()
    for sl in slots[:min(nslots, args.steps)]:
        assert torch.equal(sl["back_h"], recon), "e2e round trip differs"
    h2d = 4 * n + 2 * pc.num_codes + 8 * no + 4 * anch_h.numel()
    d2h = 2 * pc.num_codes + 8 * no + 4 * n
    e2e_ms = max_over_ranks(float(np.mean(e2e)), world)

    peak, peak_src = peaks()
    gb = n * 4 / 1e9
    comp_gbs = gb / (tc_mean / 1e3)
    decomp_gbs = gb / (td_mean / 1e3)
    ach_c = BYTES_COMPRESS * n / (tc_mean / 1e3) / 1e9
    ach_d = BYTES_DECOMPRESS * n / (td_mean / 1e3) / 1e9
    value = world * gb * args.steps / (t_total / 1e3)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic_cfg2.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get("compress_dram_bytes_per_sweep")
            traffic = None if traffic is None else round(traffic / (tc_mean / 1e3) / 1e9, 1)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_total / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 arithmetic on f32 grid",
        "data": "synthetic (seeded k^-5/3 GRF; SDRBench Miranda shape)",
        "config": workload_config(world),
        "compress": {"ms": round(tc_mean, 4), "gbs_f32_input": round(comp_gbs, 2),
                     "achieved_gbs": round(ach_c, 1), "frac": round(ach_c / peak, 4)},
        "decompress": {"ms": round(td_mean, 4), "gbs_f32_input": round(decomp_gbs, 2),
                       "achieved_gbs": round(ach_d, 1), "frac": round(ach_d / peak, 4)},
        "roofline": {"bound": "hbm", "achieved": round(ach_c, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(ach_c / peak, 4), "traffic": traffic,
                     "traffic_note": "ncu dram__bytes_read+write of one compress sweep "
                                     "(profiles/traffic_cfg2.json) over this run's sweep time, GB/s",
                     "kernel": "compress sweep (coarse DSMEM cluster + flow + escape scan/gather kernels of one run_levels)",
                     "algorithmic_bytes": f"{BYTES_COMPRESS} B/pt x {n} pts",
                     "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)"},
        "e2e": {"value": round(world * gb / (e2e_ms / 1e3), 3), "unit": UNIT,
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "path": "run_levels C-ABI round trip from pinned host buffers, steps pipelined over 3 streams"},
        "gpu_launches": int(args.steps * (pc.num_launches + pd.num_launches)),
        "outliers": int(n_out), "max_abs_err": err, "error_bound": ebound,
    }
    line["clocks"] = clk.summary() if rank == 0 else None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_port(field, levels, md)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _oracle_round_trip(field, level_tuples, md):
    from oracle import oracle
    work = field.astype(np.float64)
    t0 = time.perf_counter()
    c, o = oracle.run_levels(work, level_tuples, direction="compress", radius=32768,
                             md_alpha=md, rounding=1)
    back = np.zeros_like(work)
    back[::64, ::64, ::64] = work[::64, ::64, ::64]
    oracle.run_levels(back, level_tuples, direction="decompress", radius=32768, md_alpha=md,
                      rounding=1, codes=c, outliers=o)
    return time.perf_counter() - t0


def _level_tuples(levels):
    return [(s.stride, s.bound, 4, 1, None) for s in levels]


def cpu_baseline_port(field, levels, md):
    dt = _oracle_round_trip(field, _level_tuples(levels), md)
    return {"value": round(field.size * 4 / 1e9 / dt, 4), "unit": UNIT, "cores": 1,
            "kind": "port",
            "sample": "full cfg2 field, one compress+decompress round trip, scalar C oracle "
                      "(oracle/hpez_oracle.c), 1 thread"}


def _worker(payload):
    field, lv, md = payload
    return _oracle_round_trip(field, lv, md)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import multiprocessing as mp
    import synthetic as syn
    from oracle import oracle
    oracle.build()
    field = syn.config_field(2, index=0)
    ebound = EPS * float(field.max() - field.min())
    levels = make_levels(ebound)
    md = md_weights_for(field)
    lv = _level_tuples(levels)
    # bounded sample per worker: the centred 128x192x192 sub-block
    sub = np.ascontiguousarray(field[64:192, 96:288, 96:288])
    cores = os.cpu_count() or 1
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        for _ in range(args.warmup):
            pool.map(_worker, [(sub, lv, md)] * cores)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            pool.map(_worker, [(sub, lv, md)] * cores)
            times.append(time.perf_counter() - t0)
    gb = cores * sub.size * 4 / 1e9
    value = gb * len(times) / sum(times)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 arithmetic on f32 grid",
        "data": "synthetic (seeded k^-5/3 GRF; SDRBench Miranda shape)",
        "config": workload_config(world), "impl": "reference",
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{cores} workers x centred 128x192x192 sub-block of the cfg2 "
                                   "field, compress+decompress round trip each, scalar C oracle"},
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
