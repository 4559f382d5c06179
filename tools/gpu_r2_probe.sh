#!/bin/bash
# Round-2 first GPU session: tests, bench, ncu captures of the persistent deep kernels and the border kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv | tee gpurun_out/gpu.txt
nproc | tee -a gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 2> gpurun_out/bench.err | tee gpurun_out/bench.json
timeout 600 python tools/road_probe.py 2048 512 16 2>&1 | tail -2 | tee gpurun_out/road_direct.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:deep_forward -c 2 -o gpurun_out/r2_deep_forward \
    python tools/road_probe.py 2048 128 4 > gpurun_out/ncu_deep_f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:deep_backward -c 2 -o gpurun_out/r2_deep_backward \
    python tools/road_probe.py 2048 128 4 > gpurun_out/ncu_deep_b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"matrix_relax|compose_sigma" -c 8 -o gpurun_out/r2_border \
    python tools/road_hybir_profile.py 2048 8 > gpurun_out/ncu_border.log 2>&1
ls -la gpurun_out
