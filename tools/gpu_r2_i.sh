#!/bin/bash
mkdir -p gpurun_out
for o in deep_blocks_per_sm=3 deep_blocks_per_sm=2 deep_blocks_per_sm=1; do
  timeout 300 python tools/road_probe.py 2048 512 16 $o 2>&1 | tail -1 | tee -a gpurun_out/road_occ.log
done
timeout 300 python tools/road_probe.py 2048 512 8 2>&1 | tail -1 | tee -a gpurun_out/road_occ.log
timeout 300 python tools/road_probe.py 2048 512 32 2>&1 | tail -1 | tee -a gpurun_out/road_occ.log
