"""Developer probe: device Huffman decode of the cfg2 code stream."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
import bench, synthetic as syn
from paper_2311_12133_b200.interp import run_levels_device
from paper_2311_12133_b200 import huffman
dev = torch.device("cuda", 0)
f = syn.config_field(2, device=dev)
eb = 1e-3 * float(f.max() - f.min())
codes, outl, n = run_levels_device(torch.from_numpy(f).to(dev), bench.make_levels(eb), direction="compress",
                                   radius=32768, md_alpha=bench.md_weights_for(f), rounding=1)
lengths, payload, nbits = huffman.encode_device(codes)
pay = torch.from_numpy(np.frombuffer(payload, np.uint8).copy()).to(dev)
ts = []
for i in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d = huffman.decode_device(lengths, pay, codes.numel()); torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
assert torch.equal(d, codes)
print(json.dumps({"decode_wall_ms": [round(1e3 * t, 3) for t in ts], "symbols": codes.numel(), "bits": nbits}))
