"""Developer probe: BASELINE cfg3/cfg4 on one GPU -- tune() stage times, the
tuned (block-table) compress / decompress sweeps, and bit-exact parity of
the full-size sweep against the CPU oracle.

usage: python tools_cfg4.py [--cfg 4] [--eps 1e-3] [--dims 512,512,512] [--no-oracle]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch

import synthetic as syn
from paper_2311_12133_b200 import tuner as T
from paper_2311_12133_b200.grid import ElementKind, ScalarGrid
from paper_2311_12133_b200.interp import codes_to_int32, get_plan, run_levels_device, code_dtype_for
from paper_2311_12133_b200 import _lib
from paper_2311_12133_b200.pipeline import _plan
from paper_2311_12133_b200.plan import PARADIGM_MULTIDIM, kernel_index

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--eps", type=float, default=1e-3)
ap.add_argument("--dims", default=None)
ap.add_argument("--no-oracle", action="store_true")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--uniform", action="store_true", help="drop the block table (uniform commits)")
ap.add_argument("--profile", action="store_true", help="per-level flow-kernel timeline (HPEZ_PROFILE)")
args = ap.parse_args()
if args.profile:
    os.environ["HPEZ_PROFILE"] = "1"
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
dims = tuple(int(x) for x in args.dims.split(",")) if args.dims else None
f = syn.config_field(args.cfg, dims=dims, device=dev)
g = ScalarGrid(f.shape, ElementKind.F32, f)
eb = args.eps * float(f.max() - f.min())
out = {"cfg": args.cfg, "dims": list(f.shape), "eps": args.eps, "eb": eb}

# --- tune(), staged like tuner.tune so each stage is timed
torch.cuda.synchronize()
t0 = time.perf_counter()
cfg = T.tune(g, eb)
torch.cuda.synchronize()
out["tune_s_cold"] = round(time.perf_counter() - t0, 3)
t0 = time.perf_counter()
cfg = T.tune(g, eb)
torch.cuda.synchronize()
out["tune_s"] = round(time.perf_counter() - t0, 3)
opts = T.TunerOptions()
st = T.analyze_samples(g, opts.sample_rate)
md = T.blend_weights_f32(st)
t0 = time.perf_counter()
tbl = T.tune_blocks(g, list(cfg.level_configs), eb, options=opts, frozen_dim=cfg.frozen_dim, md_alpha=md)
torch.cuda.synchronize()
out["tune_blocks_s"] = round(time.perf_counter() - t0, 3)
out["predictor"] = cfg.predictor
out["frozen_dim"] = cfg.frozen_dim
out["alpha_beta"] = [cfg.alpha, cfg.beta]
out["level_configs"] = [repr(c) for c in cfg.level_configs]
if cfg.block_table is not None:
    out["distinct_tags_per_level"] = [int(np.unique(r).size) for r in cfg.block_table]

if cfg.predictor == "interp":
    from paper_2311_12133_b200.container import parse_config, serialize_config
    cfg = parse_config(serialize_config(cfg, g.dims), g.dims)
    if args.uniform:
        import dataclasses
        cfg = dataclasses.replace(cfg, block_size=0, block_table=None)
    levels = _plan(g.dims, cfg).levels
    frozen = () if cfg.frozen_dim is None else (cfg.frozen_dim,)
    kw = dict(radius=cfg.radius, frozen_axes=frozen, md_alpha=np.asarray(cfg.md_alpha), rounding=1,
              block_size=cfg.block_size, block_table=cfg.block_table)
    orig = torch.from_numpy(f).to(dev)
    w = torch.empty_like(orig)
    back = torch.zeros_like(orig)
    sel = tuple(slice(0, None, 1 if a in frozen else cfg.anchor_stride) for a in range(3))
    a0 = torch.zeros_like(orig)
    a0[sel] = orig[sel]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    t0 = time.perf_counter()
    pc = get_plan(g.dims, levels, direction="compress", work_dtype=_lib.WORK_F32,
                  code_dtype=code_dtype_for(cfg.radius), **{k: v for k, v in kw.items()})
    out["plan_build_s"] = round(time.perf_counter() - t0, 4)
    out["num_launches"] = pc.num_launches
    codes = torch.empty(pc.num_codes, dtype=torch.uint16, device=dev)
    outl = torch.empty(pc.num_codes, dtype=torch.float64, device=dev)
    if args.profile:  # one cold compress, then the timeline (counters accumulate across runs)
        w.copy_(orig)
        run_levels_device(w, levels, direction="compress", codes=codes, outliers=outl, **kw)
        tl = np.zeros(72, dtype=np.int64)
        _lib.lib().hpez_plan_levels_timeline(pc.handle, tl.ctypes.data)
        t0 = min(x for x in tl[0:24:2] if 0 < x < 2**62)
        out["level_us"] = [(l, round((tl[2*l]-t0)/1e3, 1), round((tl[2*l+1]-t0)/1e3, 1)) for l in range(12) if tl[2*l+1] > 0]
        cs = np.zeros(6 * 4096, dtype=np.int64)
        ncm = _lib.lib().hpez_plan_commit_stats(pc.handle, cs.ctypes.data, cs.size)
        out["commits"] = cs[:6 * max(ncm, 0)].reshape(-1, 6).tolist()  # kind, level, npos, items, members, fast id
        out["level_cycles_per_item"] = {l: [int(x / max(tl[27 + 4*l], 1)) for x in tl[24 + 4*l: 27 + 4*l]] + [int(tl[27 + 4*l])]
                                        for l in range(12) if tl[27 + 4*l]}
    tc, td = [], []
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" isolates the sweeps
    for it in range(args.iters + 2):
        w.copy_(orig)
        flush.fill_(1.0)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        run_levels_device(w, levels, direction="compress", codes=codes, outliers=outl, sync=False, **kw)
        e[1].record()
        back.copy_(a0)
        flush.fill_(2.0)
        e[2].record()
        run_levels_device(back, levels, direction="decompress", codes=codes, outliers=outl, sync=False, **kw)
        e[3].record()
        torch.cuda.synchronize()
        if it >= 2:
            tc.append(e[0].elapsed_time(e[1]))
            td.append(e[2].elapsed_time(e[3]))
    torch.cuda.nvtx.range_pop()
    _, _, n_out = run_levels_device(w.copy_(orig), levels, direction="compress", codes=codes,
                                    outliers=outl, **kw)
    back.copy_(a0)
    run_levels_device(back, levels, direction="decompress", codes=codes, outliers=outl, **kw)
    n = f.size
    out["compress_ms"] = round(float(np.median(tc)), 4)
    out["decompress_ms"] = round(float(np.median(td)), 4)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")))["hbm_gbs"]
    out["compress_frac"] = round(10 * n / (out["compress_ms"] / 1e3) / 1e9 / peak, 4)
    out["decompress_frac"] = round(6 * n / (out["decompress_ms"] / 1e3) / 1e9 / peak, 4)
    out["roundtrip_equal"] = bool(torch.equal(back, w))
    out["max_err_ok"] = bool(float((back.double() - orig.double()).abs().max()) <= eb)
    out["outliers"] = int(n_out)
    if not args.no_oracle:
        from oracle import oracle
        ref = f.astype(np.float64)
        lv = [(s.stride, s.bound, kernel_index(s.config.kernel),
               1 if s.config.paradigm == PARADIGM_MULTIDIM else 0, s.config.axis_order) for s in levels]
        t0 = time.perf_counter()
        c_o, o_o = oracle.run_levels(ref, lv, direction="compress", radius=cfg.radius, frozen_axes=frozen,
                                     md_alpha=np.asarray(cfg.md_alpha), rounding=1,
                                     block_size=cfg.block_size, block_table=cfg.block_table)
        out["oracle_s"] = round(time.perf_counter() - t0, 2)
        cg = codes_to_int32(codes)
        out["codes_equal"] = bool(np.array_equal(cg, c_o))
        out["code_mismatch"] = int((cg != c_o).sum()) if cg.shape == c_o.shape else -1
        out["outliers_equal"] = bool(outl[:n_out].cpu().numpy().tobytes() == o_o.tobytes())
        out["recon_equal"] = bool(np.array_equal(w.cpu().numpy().astype(np.float64), ref))
print(json.dumps(out), flush=True)
