#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/road_threads.log
for v in "" _t512 _t1024; do
  if [ -n "$v" ]; then export BC_B200_LIB=$PWD/paper_2008_05718_b200/libbc_b200$v.so; else unset BC_B200_LIB; fi
  echo "variant $v" | tee -a gpurun_out/road_threads.log
  timeout 300 python tools/road_probe.py 2048 512 16 2>&1 | tail -1 | tee -a gpurun_out/road_threads.log
done
