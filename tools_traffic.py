"""Summarise an ncu launch list (gpu__time_duration + dram bytes) of
tools_sweep_time.py into profiles/traffic_cfg2.json: per-kernel time and DRAM
traffic of the last compress and the last decompress sweep.

usage: python tools_traffic.py <ncu csv> <out json> <source note> [points] [round]
"""
import csv, json, sys


def rows(path):
    lines = open(path).read().splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
    out = {}
    for r in csv.DictReader(lines[i:]):
        k = int(r["ID"])
        d = out.setdefault(k, {"kernel": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["us"] = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
        elif r["Metric Name"].startswith("dram__"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
            d["dram_bytes"] = d.get("dram_bytes", 0.0) + v * scale
        elif r["Metric Name"] == "smsp__inst_executed.sum":
            d["warp_inst"] = v
        elif r["Metric Name"].startswith("smsp__issue_active"):
            d["issue_pct"] = v
    return [out[k] for k in sorted(out)]


def groups(ks):
    comp, decomp, cur, kind = [], [], None, None
    for d in ks:
        n = d["kernel"]
        if "hpez::" not in n:
            if cur:
                (comp if kind == 0 else decomp).append(cur)
            cur = None
            continue
        if cur is None:
            cur, kind = [], None
        cur.append(d)
        if "flow_kernel" in n or "coarse_kernel" in n:
            kind = 0 if n.split("<", 1)[1].split(",")[2].strip() == "0" else 1  # DIR template arg
    if cur:
        (comp if kind == 0 else decomp).append(cur)
    return comp[-1], decomp[-1]


def main():
    ks = rows(sys.argv[1])
    c, d = groups(ks)
    summ = lambda g: [{"kernel": k["kernel"][:70], "us": round(k["us"], 3),
                       "dram_MB": round(k.get("dram_bytes", 0) / 1e6, 3),
                       **({"warp_inst_M": round(k["warp_inst"] / 1e6, 2)} if "warp_inst" in k else {}),
                       **({"issue_pct": round(k["issue_pct"], 1)} if "issue_pct" in k else {})} for k in g]
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 256 * 384 * 384
    out = {"round": int(sys.argv[5]) if len(sys.argv) > 5 else 1, "source": sys.argv[3],
           "compress_sweep_kernels": summ(c),
           "compress_sweep_us": round(sum(k["us"] for k in c), 3),
           "compress_dram_bytes_per_sweep": sum(k.get("dram_bytes", 0) for k in c),
           "algorithmic_bytes": 10 * n,
           "decompress_sweep_kernels": summ(d),
           "decompress_sweep_us": round(sum(k["us"] for k in d), 3),
           "decompress_dram_bytes_per_sweep": sum(k.get("dram_bytes", 0) for k in d),
           "decompress_algorithmic_bytes": 6 * n}
    json.dump(out, open(sys.argv[2], "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if not k.endswith("kernels")}))


if __name__ == "__main__":
    main()
