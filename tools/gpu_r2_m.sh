#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu_m.log
python bench.py --no-extra --steps 10 2> gpurun_out/bench_m.err | tee gpurun_out/bench_m.json | cut -c1-300
timeout 300 python tools/road_probe.py 2048 512 16 2>&1 | tail -1 | tee gpurun_out/road_m.log
