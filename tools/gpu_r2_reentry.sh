#!/bin/bash
# Final check of the committed tree: GPU suite, smoke, the bench line (both arms) as the driver runs them.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | tee gpurun_out/pytest_gpu_final.log
python __graft_entry__.py --smoke 2>&1 | tail -2 | tee gpurun_out/smoke.log
python bench.py --gpus 1 --steps 20 --warmup 3 2> gpurun_out/bench.err | tee gpurun_out/bench_final.json | cut -c1-300
