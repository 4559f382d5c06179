#!/bin/bash
# Erdos-Renyi record (config 4 graph on one GPU): ncu metrics pass of the level kernel + a live bench line.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:^level_kernel -c 12 --csv --log-file gpurun_out/er22_metrics.csv \
    python bench.py --workload er22 --sources 256 --steps 1 --warmup 0 --no-cpu > gpurun_out/er22_under_ncu.log 2>&1
python bench.py --workload er22 --steps 3 --warmup 1 --no-cpu 2> gpurun_out/bench_er22.err | tee gpurun_out/bench_er22.json
