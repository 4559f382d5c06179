#!/bin/bash
# Child-driven backward levels (default factor 16): GPU suite, smoke, bench line, north-star probe.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8 | tee gpurun_out/pytest_gpu_bwdpush.log
python __graft_entry__.py --smoke 2>&1 | tail -2 | tee gpurun_out/smoke.log
python bench.py 2> gpurun_out/bench.err | tee gpurun_out/bench.json | cut -c1-300
