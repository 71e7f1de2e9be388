import sys, os, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2311_12133_b200.lorenzo import lorenzo_pass_device
for dims in [(512, 32, 32), (512, 64, 64), (512, 32, 384), (512, 384, 32), (256, 384, 384)]:
    f = torch.randn(dims, device="cuda").float()
    for order in (1,):
        ts = []
        for it in range(3):
            w = f.clone(); torch.cuda.synchronize(); t0 = time.perf_counter()
            c, o, n = lorenzo_pass_device(w, 1e-2, 32768, order, direction="compress", rounding=1)
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        print(dims, order, round(min(ts) * 1e3, 3), "ms", flush=True)
