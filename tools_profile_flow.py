"""Developer probe: flow-kernel phase split for the cfg2 sweep (HPEZ_PROFILE)."""
import os, sys, ctypes, json
os.environ["HPEZ_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
import bench, synthetic as syn
from paper_2311_12133_b200.interp import run_levels_device, get_plan, code_dtype_for
from paper_2311_12133_b200 import _lib
dev = torch.device("cuda", 0)
f = syn.config_field(2, device=dev)
eb = 1e-3 * float(f.max() - f.min())
lv = bench.make_levels(eb)
md = bench.md_weights_for(f)
orig = torch.from_numpy(f).to(dev)
w = orig.clone()
kw = dict(radius=32768, md_alpha=md, rounding=1)
pc = get_plan(f.shape, lv, direction="compress", work_dtype=_lib.WORK_F32, code_dtype=0, **kw)
w.copy_(orig)
c, o, n = run_levels_device(w, lv, direction="compress", **kw)
tl = np.zeros(72, dtype=np.int64)
_lib.lib().hpez_plan_levels_timeline(pc.handle, tl.ctypes.data)
t0 = min(x for x in tl[0::2] if x > 0 and x < 2**62)
print("levels (start_us, end_us):", [(round((tl[2*l]-t0)/1e3,1), round((tl[2*l+1]-t0)/1e3,1)) for l in range(6) if tl[2*l+1] > 0])
for it in range(2):
    w.copy_(orig)
    c, o, n = run_levels_device(w, lv, direction="compress", **kw)
_lib.lib().hpez_plan_levels_timeline(pc.handle, tl.ctypes.data)
for l in range(12):
    g, wt, wk, n = tl[24 + 4 * l: 28 + 4 * l]
    if n: print(f"level {l}: items {n}, cycles/item grab {g/n:.0f} wait {wt/n:.0f} work {wk/n:.0f}")
info = np.zeros(12, dtype=np.int64)
_lib.lib().hpez_plan_info(pc.handle, info.ctypes.data)
grab, wait, work, units = info[8:12]
print(json.dumps({"info": info[:8].tolist(), "units": int(units), "cycles_per_unit": {"grab": grab / units, "wait": wait / units, "work": work / units}}))
