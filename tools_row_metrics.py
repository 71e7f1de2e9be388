"""Summarise an `ncu --set full` raw CSV of the row-kernel launches into
profiles/r2_row_cfg4_metrics.json (per launch: time, DRAM bytes, instructions,
issue utilisation, occupancy, cache hit rates, pipe utilisation, stall samples).

usage: python tools_row_metrics.py <raw csv> <out json> <note>
"""
import csv, json, sys

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, units, data = rows[0], rows[1], rows[2:]
    names = ["(z even, y even)", "(z odd, y even) + (z even, y odd), first pass rows",
             "(z odd, y even) + (z even, y odd), second pass rows", "(z odd, y odd)"]
    out = {"source": sys.argv[3], "launches": []}
    for i, r in enumerate(data):
        d = {"rows": names[i] if i < len(names) else str(i), "kernel": r[hdr.index("Kernel Name")][:60]}
        for k in KEEP:
            if k in hdr:
                j = hdr.index(k)
                d[k] = [r[j], units[j]]
        d["stall_samples"] = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(r[j]) for j, h in enumerate(hdr)
                              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in h
                              and r[j].isdigit() and int(r[j]) > 0}
        out["launches"].append(d)
    json.dump(out, open(sys.argv[2], "w"), indent=1)


if __name__ == "__main__":
    main()
