#!/bin/bash
set -x
mkdir -p gpurun_out
python tools/e2e_breakdown.py 2>&1 | tail -30 | tee gpurun_out/e2e_breakdown.log
