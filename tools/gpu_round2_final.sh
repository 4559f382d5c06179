#!/bin/bash
# Last session of round 2: the records the profiles/ directory quotes, regenerated with the final code.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | tee gpurun_out/pytest_gpu_final.log
python __graft_entry__.py --smoke 2>&1 | tail -2 | tee gpurun_out/smoke.log
python bench.py 2> gpurun_out/bench.err | tee gpurun_out/bench.json | cut -c1-200
python bench.py --impl reference --steps 2 --warmup 1 2>> gpurun_out/bench.err | tee gpurun_out/bench_ref.json | cut -c1-200
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --no-extra 2> gpurun_out/bench_torchrun.err | grep "^{" > gpurun_out/bench_torchrun_n1.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 \
    bench.py --gpus 1 --gpu-mode graph-partitioned --forward bsp --workload rmat16 --sources 256 --steps 3 --warmup 1 \
    2>> gpurun_out/bench_torchrun.err | grep "^{" > gpurun_out/bench_gp_bsp_n1.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29613 \
    bench.py --gpus 1 --gpu-mode graph-partitioned --forward hybir --workload road512 --sources 128 --steps 2 --warmup 1 \
    2>> gpurun_out/bench_torchrun.err | grep "^{" > gpurun_out/bench_gp_hybir_n1.json
wc -c gpurun_out/bench_torchrun_n1.json gpurun_out/bench_gp_bsp_n1.json gpurun_out/bench_gp_hybir_n1.json
: > gpurun_out/r2_fullsize_new.jsonl
for w in c1 rmat22 er22 road2048 road2048_hybir rmat24; do
  timeout 1500 python tools/fullsize.py $w 2>&1 | grep "^{" | tee -a gpurun_out/r2_fullsize_new.jsonl | cut -c1-160
done
T=/tmp/r2prof; mkdir -p $T
timeout 900 ncu --set full --clock-control none -k regex:deep_forward_compact -c 4 -o $T/r2_deep_fc -f \
    python tools/road_probe.py 2048 128 4 > gpurun_out/ncu_deep_fc.log 2>&1
ncu -i $T/r2_deep_fc.ncu-rep --page raw --csv > gpurun_out/r2_deep_forward_compact.raw.csv
timeout 900 ncu --set full --clock-control none -k regex:deep_backward_compact -c 1 -o $T/r2_deep_bc -f \
    python tools/road_probe.py 2048 128 4 > gpurun_out/ncu_deep_bc.log 2>&1
ncu -i $T/r2_deep_bc.ncu-rep --page raw --csv > gpurun_out/r2_deep_backward_compact.raw.csv
# launch list + full capture of the level kernel with the final code (profiles/r2_launches*, r2_level_kernel_ncu_full.csv, r2_traffic.json)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-extra --relabel 1 > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:^level_kernel -c 8 -o $T/prof_level -f \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-extra --relabel 1 > gpurun_out/bench_under_ncu2.log 2>&1
ncu -i $T/prof_level.ncu-rep --page raw --csv > gpurun_out/prof_level.raw.csv
# general-weight sweeps: sanitizer + records, and a full capture of mid-sweep rounds (four groups)
bash tools/gpu_r2_weighted.sh
timeout 900 ncu --set full --clock-control none -k regex:sssp_forward -s 3000 -c 2 -o $T/sssp_f -f \
    python tools/weighted_probe.py 1024 128 100000 > gpurun_out/ncu_sssp_f.log 2>&1
ncu -i $T/sssp_f.ncu-rep --page raw --csv > gpurun_out/sssp_forward.raw.csv
timeout 900 ncu --set full --clock-control none -k regex:sssp_relax -s 4000 -c 2 -o $T/sssp_a -f \
    python tools/weighted_probe.py 1024 128 100000 > gpurun_out/ncu_sssp_a.log 2>&1
ncu -i $T/sssp_a.ncu-rep --page raw --csv > gpurun_out/sssp_relax.raw.csv
du -sh gpurun_out
