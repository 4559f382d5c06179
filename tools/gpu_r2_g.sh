#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu_g.log
for opt in deep_compact=0 deep_compact=1 deep_compact=2; do
  timeout 300 python tools/road_probe.py 2048 512 16 $opt 2>&1 | tail -1 | tee -a gpurun_out/road_compact.log
done
