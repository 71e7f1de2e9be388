"""Developer probe: timings of the non-sweep components on the cfg2 field."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
import bench, synthetic as syn
from paper_2311_12133_b200.interp import run_levels_device
from paper_2311_12133_b200.lorenzo import lorenzo_pass_device
from paper_2311_12133_b200 import huffman, container, pipeline, tuner
from paper_2311_12133_b200.grid import ScalarGrid, ElementKind, ErrorBoundSpec, BoundMode
from paper_2311_12133_b200.plan import CompressionConfig, KERNEL_VARIANTS, PARADIGM_MULTIDIM, LevelConfig

dev = torch.device("cuda", 0)
out = {}
def ev_time(fn, reps=3):
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); r = fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts[1:])), r

f = syn.config_field(2, device=dev)
eb = 1e-3 * float(f.max() - f.min())
lv = bench.make_levels(eb); md = bench.md_weights_for(f)
orig = torch.from_numpy(f).to(dev); w = orig.clone()
codes, outl, n = run_levels_device(w, lv, direction="compress", radius=32768, md_alpha=md, rounding=1)
# histogram + table + pack
t, _ = ev_time(lambda: huffman.histogram_device(codes))
out["histogram_ms"] = t
t0 = time.perf_counter(); lengths, payload, nbits = huffman.encode_device(codes); out["huffman_encode_wall_ms"] = 1e3 * (time.perf_counter() - t0)
out["payload_MB"] = len(payload) / 1e6; out["bits_per_code"] = nbits / codes.numel()
t0 = time.perf_counter(); dec = huffman.decode_int32(lengths, payload, codes.numel()); out["huffman_decode_host_ms"] = 1e3 * (time.perf_counter() - t0)
assert np.array_equal(dec, codes.view(torch.int16).cpu().numpy().view(np.uint16).astype(np.int32))
pay_dev = torch.from_numpy(np.frombuffer(payload, np.uint8).copy()).to(dev)
t, dd = ev_time(lambda: huffman.decode_device(lengths, pay_dev, codes.numel()))
out["huffman_decode_device_ms"] = t
assert torch.equal(dd, codes)
t0 = time.perf_counter(); dd = huffman.decode_device(lengths, payload, codes.numel()); torch.cuda.synchronize(); out["huffman_decode_device_from_host_wall_ms"] = 1e3 * (time.perf_counter() - t0)
# Lorenzo
for order in (1, 2):
    w2 = orig.clone()
    t, (c2, o2, n2) = ev_time(lambda: (w2.copy_(orig), lorenzo_pass_device(w2, eb, 32768, order, direction="compress", rounding=1))[1], reps=1)
    out[f"lorenzo_o{order}_compress_ms"] = t
# full archive pipeline (fixed config, as cfg2)
g = ScalarGrid(f.shape, ElementKind.F32, f)
cfg = CompressionConfig("interp", eb, 32768, level_configs=(LevelConfig(KERNEL_VARIANTS[4], PARADIGM_MULTIDIM),) * 6,
                        md_alpha=tuple(float(np.float32(x)) for x in md))
t0 = time.perf_counter(); res = pipeline.compress(g, ErrorBoundSpec(BoundMode.REL, 1e-3), config=cfg); out["pipeline_compress_s"] = time.perf_counter() - t0
t0 = time.perf_counter(); rec = pipeline.decompress(res.archive); out["pipeline_decompress_s"] = time.perf_counter() - t0
assert rec.data.tobytes() == res.reconstruction.data.tobytes()
out["ratio"] = res.ratio
# tuner on a config-4 style field (256^3 subset to keep it short)
f4 = syn.config_field(4, dims=(256, 256, 256), device=dev)
g4 = ScalarGrid(f4.shape, ElementKind.F32, f4)
e4 = 1e-3 * float(f4.max() - f4.min())
t0 = time.perf_counter(); cfg4 = tuner.tune(g4, e4); torch.cuda.synchronize(); out["tune_256cube_s"] = time.perf_counter() - t0
t0 = time.perf_counter(); cfg4 = tuner.tune(g4, e4); torch.cuda.synchronize(); out["tune_256cube_s_warm"] = time.perf_counter() - t0
out["tune_choice"] = {"predictor": cfg4.predictor, "alpha": cfg4.alpha, "beta": cfg4.beta, "frozen": cfg4.frozen_dim,
                      "table": cfg4.block_table is not None}
print(json.dumps(out))
