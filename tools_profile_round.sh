#!/bin/bash
# GPU-box profiling pass for one round: bench lines, launch lists, traffic,
# one full ncu capture of the compress flow kernel.  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools_sweep_time.py > gpurun_out/sweep_time.json || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/traffic_launches.csv python tools_sweep_time.py > gpurun_out/ncu_traffic.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:flow_kernel -c 1 -o gpurun_out/flow_full \
    python tools_sweep_time.py > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/flow_full.ncu-rep --page details --csv > gpurun_out/flow_full_details.csv 2>/dev/null
ncu -i gpurun_out/flow_full.ncu-rep --page raw --csv > gpurun_out/flow_full_raw.csv 2>/dev/null
ncu --set full --import-source on --clock-control none -k regex:coarse_dsmem -c 1 -o gpurun_out/coarse_full \
    python tools_sweep_time.py > gpurun_out/ncu_coarse.log 2>&1
ncu -i gpurun_out/coarse_full.ncu-rep --page details --csv > gpurun_out/coarse_full_details.csv 2>/dev/null
true
