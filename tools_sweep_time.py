"""Developer probe: device time of the cfg2 compress / decompress sweeps."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
import bench, synthetic as syn
from paper_2311_12133_b200.interp import run_levels_device
dev = torch.device("cuda", 0)
f = syn.config_field(2, device=dev)
eb = 1e-3 * float(f.max() - f.min())
lv = bench.make_levels(eb)
md = bench.md_weights_for(f)
orig = torch.from_numpy(f).to(dev)
w = orig.clone(); back = torch.zeros_like(orig); a0 = torch.zeros_like(orig)
a0[::64, ::64, ::64] = orig[::64, ::64, ::64]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
kw = dict(radius=32768, md_alpha=md, rounding=1)
codes = outl = None
FL = os.environ.get("FLUSH", "write")
def flush_op(v):
    if FL == "write": flush.fill_(v)
    elif FL == "read": flush.fill_(v); torch.cuda.synchronize(); flush.sum()
    elif FL == "readonly": flush.sum()
tc, td = [], []
for it in range(int(os.environ.get('ITERS', 8))):
    w.copy_(orig); flush_op(1.0)
    e0, e1, e2, e3 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e0.record(); codes, outl, n = run_levels_device(w, lv, direction="compress", sync=False, **kw); e1.record()
    back.copy_(a0); flush_op(2.0)
    e2.record(); run_levels_device(back, lv, direction="decompress", codes=codes, outliers=outl, sync=False, **kw); e3.record()
    torch.cuda.synchronize()
    if it >= min(3, int(os.environ.get('ITERS', 8)) - 1):
        tc.append(e0.elapsed_time(e1)); td.append(e2.elapsed_time(e3))
assert os.environ.get('HPEZ_DEBUG_NODEPS') or torch.equal(back, w)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("HPEZ_")}, "compress_ms": round(float(np.median(tc)), 4), "decompress_ms": round(float(np.median(td)), 4)}))
