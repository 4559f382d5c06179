#!/bin/bash
# Records after the child-driven backward levels: bench arms, launch list, full capture of one step's level
# launches (level_kernel + bwd_push kernels), full-size records (compute-sanitizer is closed on this pool: no sanitizer pass over the new kernels).
set -x
mkdir -p gpurun_out
T=/tmp/r2prof; mkdir -p $T
python bench.py 2> gpurun_out/bench.err | tee gpurun_out/bench.json | cut -c1-200
python bench.py --impl reference --steps 2 --warmup 1 2>> gpurun_out/bench.err | tee gpurun_out/bench_ref.json | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-extra --relabel 1 > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:^level_kernel|bwd_push|bwd_child' -c 24 -o $T/prof_level -f \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-extra --relabel 1 > gpurun_out/bench_under_ncu2.log 2>&1
ncu -i $T/prof_level.ncu-rep --page raw --csv > gpurun_out/prof_level.raw.csv
: > gpurun_out/r2_fullsize_new.jsonl
for w in rmat22 er22 rmat24 road2048; do
  timeout 1500 python tools/fullsize.py $w 2>&1 | grep "^{" | tee -a gpurun_out/r2_fullsize_new.jsonl | cut -c1-160
done
timeout 600 python tools/e2e_breakdown.py rmat20 1024 > gpurun_out/e2e_breakdown.log 2>&1
du -sh gpurun_out
