#!/bin/bash
# Child-driven backward levels: quick parity, per-level trace, per-kernel times (ncu launch list), probe, GPU suite.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "child_driven or golden or config1" 2>&1 | tail -5 | tee gpurun_out/bwdpush_quick.log
timeout 600 python tools/level_trace.py rmat20 1024 16 > gpurun_out/level_trace_16.log 2>&1
timeout 600 python tools/level_trace.py rmat20 1024 4 > gpurun_out/level_trace_4.log 2>&1
timeout 900 python tools/bwd_push_probe.py rmat20 1024 1 > gpurun_out/bwdpush_probe.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:bwd_push|bwd_child' --csv --log-file gpurun_out/bwdpush_launches.csv \
    python tools/level_trace.py rmat20 1024 4 > gpurun_out/bwdpush_ncu.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -8 | tee gpurun_out/pytest_gpu_bwdpush.log
