#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_multirank.py -x -q 2>&1 | tail -25 | tee gpurun_out/pytest_gpu_l.log
timeout 600 python tools/fullsize.py c1 2>&1 | grep "^{" | tee gpurun_out/c1_new.jsonl
