#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python tools/fullsize.py rmat24 2>&1 | grep "^{" | tee gpurun_out/rmat24_alone.jsonl
