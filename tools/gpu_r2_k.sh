#!/bin/bash
mkdir -p gpurun_out
S=gpurun_out/sanitizer_r2b.log; : > $S
run() { echo "=== $*" | tee -a $S; timeout 1500 "$@" 2>&1 | grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY" | tail -4 | tee -a $S; }
run compute-sanitizer --tool initcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q -k "level_ordered or lookahead or refinement_bound or persistent or border_table_cache"
run compute-sanitizer --tool initcheck --target-processes all python -m pytest tests/test_gpu_multirank.py -x -q -k "2-path"
run compute-sanitizer --tool racecheck python tools/dbg_init.py
run compute-sanitizer --tool racecheck --target-processes all python -m pytest tests/test_gpu_multirank.py -x -q -k "2-path-hybir"
