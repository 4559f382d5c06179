#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_multirank.py -x -q 2>&1 | tail -30 | tee gpurun_out/pytest_gpu_c.log
timeout 1800 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_multirank.py 2>&1 | tail -8 | tee -a gpurun_out/pytest_gpu_c.log
