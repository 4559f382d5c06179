#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q -k "level_ordered or persistent or lookahead or deep or kway or queue_sweeps" 2>&1 | tail -5 | tee gpurun_out/pytest_gpu_g.log
: > gpurun_out/road_compact.log
for i in 1 2; do
  timeout 300 python tools/road_probe.py 2048 512 16 2>&1 | tail -1 | tee -a gpurun_out/road_compact.log
done
