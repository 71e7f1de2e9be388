"""Developer probe: stage times of the archive pipeline on one cfg4 field
(tune stages, sweep, Huffman encode pieces, zlib, decode)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch

import synthetic as syn
from paper_2311_12133_b200 import container, huffman, pipeline, tuner as T
from paper_2311_12133_b200.grid import BoundMode, ElementKind, ErrorBoundSpec, ScalarGrid
from paper_2311_12133_b200.interp import run_levels_device

dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 4
f = syn.config_field(cfg_id, device=dev)
g = ScalarGrid(f.shape, ElementKind.F32, f)
eb = 1e-3 * float(f.max() - f.min())
out = {}


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


T.tune(g, eb)  # warm
opts = T.TunerOptions()
t0 = tick()
st = T.analyze_samples(g, opts.sample_rate)
md = T.blend_weights_f32(st)
t1 = tick()
cache = {}
cfgs = T.tune_global(g, st, eb, T.QualityTarget(), options=opts, md_alpha=md, _cache=cache)
t2 = tick()
dec = T.tune_freeze(g, st, eb, T.QualityTarget(), options=opts, plain_configs=cfgs, md_alpha=md, _cache=cache)
t3 = tick()
ab = T.tune_eb(g, eb, T.QualityTarget(), options=opts, configs=dec.configs, frozen_dim=dec.frozen_dim,
               md_alpha=md, _cache=cache)
t4 = tick()
tbl = T.tune_blocks(g, dec.configs, eb, options=opts, frozen_dim=dec.frozen_dim, md_alpha=md)
t5 = tick()
out["tune"] = {"analyze_samples": t1 - t0, "tune_global": t2 - t1, "tune_freeze": t3 - t2,
               "tune_eb": t4 - t3, "tune_blocks": t5 - t4}
cfg = T.tune(g, eb)
from paper_2311_12133_b200.container import parse_config, serialize_config
from paper_2311_12133_b200.pipeline import _plan
cfg = parse_config(serialize_config(cfg, g.dims), g.dims)
levels = _plan(g.dims, cfg).levels
kw = dict(radius=cfg.radius, md_alpha=np.asarray(cfg.md_alpha), rounding=1, block_size=cfg.block_size,
          block_table=cfg.block_table)
w = torch.from_numpy(f).to(dev)
codes, outl, n_out = run_levels_device(w, levels, direction="compress", **kw)
for _ in range(2):
    a = tick()
    freqs = huffman.histogram_device(codes)
    b = tick()
    lengths, values = huffman.table(freqs)
    c = tick()
    framed = container.pack_codes(codes)
    d = tick()
    z = container.lossless_pass(framed)
    e = tick()
out["huffman"] = {"histogram+D2H": b - a, "table": c - b, "pack_codes_total": d - c, "zlib_codes": e - d,
                  "payload_MB": len(framed) / 1e6, "zlib_MB": len(z) / 1e6}
spec = ErrorBoundSpec(BoundMode.REL, 1e-3)
a = tick()
res = pipeline.compress(g, spec)
b = tick()
back = pipeline.decompress(res.archive)
c = tick()
out["archive"] = {"compress": b - a, "decompress": c - b}
a = tick()
dims, kind, _m, _e, cb, blobs = container.parse(res.archive)
raw = [container.lossless_unpass(x) for x in blobs]
b = tick()
ct = container.unpack_codes_device(raw[1], cfg.radius)
c = tick()
out["decode"] = {"inflate": b - a, "unpack_codes_device": c - b}
print(json.dumps({k: ({kk: round(vv, 4) for kk, vv in v.items()} if isinstance(v, dict) else v)
                  for k, v in out.items()}))
