"""Developer probe: randomised parity of the row kernel (csrc/row.cu) against the oracle --
random dims, tag subsets, block sizes, bounds, in-place and out-of-place compress.

usage: python tools_fuzz_rows.py [seed] [cases]"""
import os, sys
os.environ["HPEZ_ROW_MIN"] = "0"; os.environ["HPEZ_ROW"] = "2"
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import test_row_gpu as T
from paper_2311_12133_b200 import interp
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
bad = 0
for i in range(n):
    dims = (int(rng.integers(9, 140)), int(rng.integers(9, 140)), int(rng.integers(3, 70)) * 4)
    bs = int(rng.choice([0, 4, 8, 16, 32]))
    eps = float(rng.choice([1e-2, 1e-3, 1e-4, 1e-6]))
    seed = int(rng.integers(0, 1 << 30))
    k = int(rng.integers(0, 5)); par = int(rng.integers(0, 2))
    if par == 0 and k in (2, 4): k = 1
    data = T._field(dims)
    if rng.integers(0, 2): data = (data + rng.standard_normal(dims).astype(np.float32) * 0.2).astype(np.float32)
    e = eps * float(data.max() - data.min())
    levels = T._levels(seed, 64, e, k, par)
    tags_all = [0, 1, 2, 3, 4, 8, 9, 11, 16, 17, 19, 24, 32, 40, 41, 48, 51]
    sub = list(rng.choice(tags_all, size=int(rng.integers(1, 7)), replace=False))
    tbl = T._table(seed, dims, bs, len(levels), [int(t) for t in sub]) if bs else None
    md = rng.uniform(0, 1, 3)
    interp._PLANS.clear()
    try:
        info = T._row_info(data.shape, levels, md, bs, tbl)
        T._roundtrip(data, levels, md, bs, tbl, oop=bool(rng.integers(0, 2)))
        print(i, dims, bs, eps, k, par, sub, "rows", info[0], "ok", flush=True)
    except AssertionError as ex:
        bad += 1
        print(i, dims, bs, eps, k, par, sub, "FAIL", str(ex)[:200], flush=True)
print("failures", bad)
