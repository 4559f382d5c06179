#!/bin/bash
# One GPU-box session: tests, smoke, bench, ncu launch list + full capture of the level kernel.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.log
python __graft_entry__.py --smoke 2>&1 | tail -3 | tee gpurun_out/smoke.log
python bench.py 2> gpurun_out/bench.err | tee gpurun_out/bench.json
python bench.py --impl reference --steps 2 --warmup 1 2>> gpurun_out/bench.err | tee gpurun_out/bench_ref.json
tail -5 gpurun_out/bench.err
# same command as the bench (one step): launch list, then the dominant kernel with the full set
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:^level_kernel -c 9 -o gpurun_out/prof_level \
    python bench.py --steps 1 --warmup 0 --no-cpu > gpurun_out/bench_under_ncu2.log 2>&1
ls -la gpurun_out
