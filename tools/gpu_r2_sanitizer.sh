#!/bin/bash
# compute-sanitizer over the kernels added in round 2 (through the C ABI via pytest).
mkdir -p gpurun_out
S=gpurun_out/sanitizer_r2.log; : > $S
run() { echo "=== $*" | tee -a $S; timeout 2400 "$@" 2>&1 | grep -E "passed|failed|error|ERROR SUMMARY|RACECHECK SUMMARY|hazard" | tail -6 | tee -a $S; }
run compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q -k "level_ordered or persistent or lookahead or refinement_bound or border_table_cache or malformed or bigint or falls_back"
run compute-sanitizer --tool memcheck --target-processes all --error-exitcode 9 python -m pytest tests/test_gpu_multirank.py -x -q -k "path or (2-road-hybir)"
run compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -x -q -k "level_ordered"
run compute-sanitizer --tool initcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_partitioned.py -x -q -k "level_ordered or lookahead or refinement_bound"
cat $S
