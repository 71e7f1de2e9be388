"""Developer probe: Lorenzo compress / decompress time on the cfg2 field
(orders 1 and 2) and bit-exactness of the round trip against the oracle."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import torch

import synthetic as syn
from paper_2311_12133_b200.lorenzo import lorenzo_pass_device
from paper_2311_12133_b200.interp import codes_to_int32

dev = torch.device("cuda", 0)
f = syn.config_field(2, device=dev)
eb = 1e-3 * float(f.max() - f.min())
orig = torch.from_numpy(f).to(dev)
out = {}
for order in (1, 2):
    ts = []
    for it in range(4):
        w = orig.clone()
        e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e0.record()
        c, o, n = lorenzo_pass_device(w, eb, 32768, order, direction="compress", rounding=1)
        e1.record()
        back = torch.zeros_like(orig)
        e1b = torch.cuda.Event(enable_timing=True)
        e1b.record()
        lorenzo_pass_device(back, eb, 32768, order, direction="decompress", rounding=1, codes=c,
                            outliers=o[:max(n, 1)])
        e2.record()
        torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), e1b.elapsed_time(e2)))
    ok = bool(torch.equal(back, w))
    out[f"order{order}"] = {"compress_ms": round(float(np.median([t[0] for t in ts[1:]])), 3),
                            "decompress_ms": round(float(np.median([t[1] for t in ts[1:]])), 3),
                            "roundtrip_equal": ok, "outliers": int(n)}
    if "--oracle" in sys.argv:
        from oracle import oracle
        ref = f.astype(np.float64)
        co, oo = oracle.lorenzo(ref, eb, 32768, order, direction="compress", rounding=1)
        out[f"order{order}"]["codes_equal"] = bool(np.array_equal(codes_to_int32(c), co))
        out[f"order{order}"]["recon_equal"] = bool(np.array_equal(w.cpu().numpy().astype(np.float64), ref))
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("HPEZ_")}, **out}))
