import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synthetic as syn
from paper_2311_12133_b200 import huffman, _lib, container
from paper_2311_12133_b200._lib import check, lib
from paper_2311_12133_b200.device import bind, ptr, stream
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
codes = torch.from_numpy((32768 + np.clip(rng.standard_normal(134_000_000) * 40, -30000, 30000)).astype(np.uint16)).to(dev)
def tk():
    torch.cuda.synchronize(); return time.perf_counter()
for it in range(3):
    t = [tk()]
    freqs = huffman.histogram_device(codes); t.append(tk())
    lengths, values = huffman.table(freqs); t.append(tk())
    nbits = int((freqs * lengths.astype(np.int64)).sum()); nbytes = (nbits + 7) // 8
    ld = np.zeros(65536, dtype=np.uint8); vd = np.zeros(65536, dtype=np.uint64)
    ld[:lengths.size] = lengths; vd[:values.size] = values
    ld_t = torch.from_numpy(ld).to(dev); vd_t = torch.from_numpy(vd.view(np.int64)).to(dev); t.append(tk())
    words = torch.empty(max((nbits + 31) // 32, 1), dtype=torch.int32, device=dev); bind()
    check(lib().hpez_huffman_pack(ptr(codes), 0, codes.numel(), ptr(ld_t), ptr(vd_t), int(lengths.max()), ptr(words), nbits, stream()), "pack"); t.append(tk())
    h = words.view(torch.uint8)[:nbytes].cpu(); t.append(tk())
    b = h.numpy().tobytes(); t.append(tk())
    f = container._frame(codes.numel(), lengths, b, nbits); t.append(tk())
    print(json.dumps({"MB": nbytes/1e6, "ms": [round(1e3*(t[i+1]-t[i]),2) for i in range(len(t)-1)], "names": ["hist","table","h2d_tables","pack","d2h","tobytes","frame"]}))
