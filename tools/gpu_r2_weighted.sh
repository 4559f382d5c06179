#!/bin/bash
# General-weight sweeps: sanitizer passes, full GPU suite, records at size (round 2).
mkdir -p gpurun_out
S=gpurun_out/r2_weighted.log; : > $S
run() { echo "=== $*" | tee -a $S; timeout 1500 "$@" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|bc_run|oracle|^n " | tail -6 | tee -a $S; }
run compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_weighted.py -x -q -k "general or large"
run compute-sanitizer --tool initcheck python -m pytest tests/test_gpu_weighted.py -x -q -k "general or large"
run compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_weighted.py -x -q -k "large_weights_vs_oracle"
run python -m pytest tests -m gpu -x -q
run python tools/weighted_probe.py 1024 128 100000
run python tools/weighted_probe.py 1024 512 100000
run python tools/weighted_probe.py 2048 128 1000000
run python tools/weighted_probe.py 1024 128 100
