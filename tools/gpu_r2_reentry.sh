#!/bin/bash
# Re-entry check of round 2: GPU suite, smoke and both bench arms on the restored tree.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | tee gpurun_out/pytest_gpu_reentry.log
python __graft_entry__.py --smoke 2>&1 | tail -2 | tee gpurun_out/smoke.log
python bench.py 2> gpurun_out/bench.err | tee gpurun_out/bench.json | cut -c1-300
python bench.py --impl reference --steps 2 --warmup 1 2>> gpurun_out/bench.err | tee gpurun_out/bench_ref.json | cut -c1-300
python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-extra 2> gpurun_out/bench_g2.err | tail -2 | cut -c1-300
