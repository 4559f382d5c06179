#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 | tee gpurun_out/pytest_gpu_h.log
timeout 900 python tools/fullsize.py road2048_hybir road2048 2>&1 | tail -6 | tee gpurun_out/fullsize_road.log
