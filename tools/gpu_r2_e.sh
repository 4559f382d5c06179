#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu_e.log
for g in 16; do
  timeout 300 python tools/road_probe.py 2048 512 $g 2>&1 | tail -1 | tee -a gpurun_out/road_mlp2.log
done
