#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q 2>&1 | tail -4 | tee gpurun_out/pytest_gpu_n.log
timeout 300 python tools/road_probe.py 2048 512 16 2>&1 | tail -1 | tee gpurun_out/road_n.log
timeout 300 python tools/road_probe.py 2048 512 16 2>&1 | tail -1 | tee -a gpurun_out/road_n.log
