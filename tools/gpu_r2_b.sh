#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu_b.log
timeout 900 python bench.py --steps 5 2> gpurun_out/bench_b.err | tee gpurun_out/bench_b.json
tail -5 gpurun_out/bench_b.err
for opt in "" "l2_fetch=32" "l2_fetch=128"; do
  timeout 300 python tools/road_probe.py 2048 512 16 $opt 2>&1 | tail -1 | tee -a gpurun_out/road_l2.log
done
for g in 4 8; do
  timeout 300 python tools/road_probe.py 2048 512 $g 2>&1 | tail -1 | tee -a gpurun_out/road_l2.log
  timeout 300 python tools/road_probe.py 2048 512 $g l2_fetch=32 2>&1 | tail -1 | tee -a gpurun_out/road_l2.log
done
