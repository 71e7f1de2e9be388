import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_12133_b200.lorenzo import lorenzo_pass_device
for dims in [(512, 16, 16), (512, 16, 16), (1024, 16, 16)]:
    f = torch.randn(dims, device="cuda").float()
    ts = []
    for it in range(3):
        w = f.clone(); torch.cuda.synchronize(); t0 = time.perf_counter()
        lorenzo_pass_device(w, 1e-2, 32768, 1, direction="compress", rounding=1)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(dims, round(min(ts) * 1e3, 3), "ms", flush=True)
