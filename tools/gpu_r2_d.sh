#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_multirank.py 2>&1 | tail -8 | tee gpurun_out/pytest_gpu_d.log
for g in 16 4; do
  timeout 300 python tools/road_probe.py 2048 512 $g 2>&1 | tail -1 | tee -a gpurun_out/road_mlp.log
done
timeout 600 python tools/fullsize.py road2048_hybir 2>&1 | tail -3 | tee -a gpurun_out/road_mlp.log
