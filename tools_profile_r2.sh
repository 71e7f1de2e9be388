#!/bin/bash
# GPU-box profiling pass for round 2 (cfg4 headline): launch list of the
# bench, per-kernel time + DRAM traffic of the timed cfg4 sweeps, full ncu
# captures of the stride-1 row launches (compress: all four row types;
# decompress: the (z odd, y odd) launch).  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --quick > gpurun_out/r2_ncu_bench.log 2>&1
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/r2_traffic_cfg4.csv \
    python tools_cfg4.py --cfg 4 --no-oracle --iters 1 > gpurun_out/r2_ncu_traffic.log 2>&1
python tools_traffic.py gpurun_out/r2_traffic_cfg4.csv gpurun_out/traffic_cfg4.json \
    "ncu dram bytes of the timed cfg4 sweeps (tools_cfg4.py, L2 flushed by a write before each)" 134217728 2
# compress row launches of the first timed sweep: strides 4 (3 launches), 2 (4), 1 (4) -> skip 7, take 4
ncu --nvtx --nvtx-include "timed/" --set full --import-source on --clock-control none -k regex:row_kernel -s 7 -c 4 \
    -o gpurun_out/r2_row_cfg4 python tools_cfg4.py --cfg 4 --no-oracle --iters 0 > gpurun_out/r2_ncu_full.log 2>&1
ncu -i gpurun_out/r2_row_cfg4.ncu-rep --page details --csv > gpurun_out/r2_row_cfg4_details.csv 2>/dev/null
ncu -i gpurun_out/r2_row_cfg4.ncu-rep --page raw --csv > gpurun_out/r2_row_cfg4_raw.csv 2>/dev/null
true
