#!/bin/bash
# One GPU-box session of round 2: tests, smoke, bench (both arms), launch list + full capture of the level kernel,
# ncu of the level-ordered deep kernels, full-size records.  The .ncu-rep files stay on the box (gpurun_out/ is
# capped at 64 MiB): raw pages are exported here.
set -x
mkdir -p gpurun_out
T=/tmp/r2prof; mkdir -p $T
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 | tee gpurun_out/pytest_gpu_final.log
python __graft_entry__.py --smoke 2>&1 | tail -3 | tee gpurun_out/smoke.log
python bench.py 2> gpurun_out/bench.err | tee gpurun_out/bench.json
python bench.py --impl reference --steps 2 --warmup 1 2>> gpurun_out/bench.err | tee gpurun_out/bench_ref.json
tail -5 gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-extra > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:^level_kernel -c 16 -o $T/prof_level -f \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-extra > gpurun_out/bench_under_ncu2.log 2>&1
ncu -i $T/prof_level.ncu-rep --page raw --csv > gpurun_out/prof_level.raw.csv
timeout 900 ncu --set full --clock-control none -k regex:deep_forward_compact -c 4 -o $T/r2_deep_fc -f \
    python tools/road_probe.py 2048 128 4 > gpurun_out/ncu_deep_fc.log 2>&1
ncu -i $T/r2_deep_fc.ncu-rep --page raw --csv > gpurun_out/r2_deep_forward_compact.raw.csv
timeout 900 ncu --set full --clock-control none -k regex:deep_backward_compact -c 1 -o $T/r2_deep_bc -f \
    python tools/road_probe.py 2048 128 4 > gpurun_out/ncu_deep_bc.log 2>&1
ncu -i $T/r2_deep_bc.ncu-rep --page raw --csv > gpurun_out/r2_deep_backward_compact.raw.csv
for w in c1 rmat22 er22 road2048 road2048_hybir rmat24; do   # one process each: no cached blocks of the previous one
  timeout 1500 python tools/fullsize.py $w 2>&1 | grep "^{" | tee -a gpurun_out/r2_fullsize_new.jsonl
done
du -sh gpurun_out
