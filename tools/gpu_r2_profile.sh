#!/bin/bash
# Round-2 profiles: launch list + full capture of the level kernel on the bench workload (one step = one batch of
# 32 groups), full capture of the border kernels and the persistent deep kernels, bench under torchrun (N = 1).
# The .ncu-rep files stay on the box (gpurun_out/ is capped at 64 MiB): raw / source pages are exported here.
set -x
mkdir -p gpurun_out
T=/tmp/r2prof; mkdir -p $T
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-extra --relabel 1 > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:^level_kernel -c 8 -o $T/prof_level -f \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-extra --relabel 1 > gpurun_out/bench_under_ncu2.log 2>&1
ncu -i $T/prof_level.ncu-rep --page raw --csv > gpurun_out/prof_level.raw.csv
timeout 900 ncu --set full --clock-control none -k regex:compose_sigma -c 6 -o $T/r2_compose -f \
    python tools/road_hybir_profile.py 2048 8 > gpurun_out/ncu_compose.log 2>&1
ncu -i $T/r2_compose.ncu-rep --page raw --csv > gpurun_out/r2_compose.raw.csv
timeout 900 ncu --set full --clock-control none -k regex:matrix_relax -c 4 -o $T/r2_relax -f \
    python tools/road_hybir_profile.py 2048 8 > gpurun_out/ncu_relax.log 2>&1
ncu -i $T/r2_relax.ncu-rep --page raw --csv > gpurun_out/r2_relax.raw.csv
timeout 900 ncu --set full --clock-control none -k regex:deep_forward -c 4 -o $T/r2_deep_forward -f \
    python tools/road_probe.py 2048 128 4 > gpurun_out/ncu_deep_f.log 2>&1
ncu -i $T/r2_deep_forward.ncu-rep --page raw --csv > gpurun_out/r2_deep_forward.raw.csv
timeout 900 ncu --set full --clock-control none -k regex:deep_backward -c 1 -o $T/r2_deep_backward -f \
    python tools/road_probe.py 2048 128 4 > gpurun_out/ncu_deep_b.log 2>&1
ncu -i $T/r2_deep_backward.ncu-rep --page raw --csv > gpurun_out/r2_deep_backward.raw.csv
# the same bench under torchrun, one rank: NCCL process group, all-reduce inside the timed region
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --no-extra 2> gpurun_out/bench_torchrun.err | tee gpurun_out/bench_torchrun_n1.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 \
    bench.py --gpus 1 --gpu-mode graph-partitioned --forward bsp --workload rmat16 --sources 256 --steps 3 --warmup 1 \
    2>> gpurun_out/bench_torchrun.err | tee gpurun_out/bench_gp_bsp_n1.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29613 \
    bench.py --gpus 1 --gpu-mode graph-partitioned --forward hybir --workload road512 --sources 128 --steps 2 --warmup 1 \
    2>> gpurun_out/bench_torchrun.err | tee gpurun_out/bench_gp_hybir_n1.json
tail -20 gpurun_out/bench_torchrun.err
du -sh gpurun_out
