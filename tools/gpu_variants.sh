#!/bin/bash
# Times the bench workload with each tuning variant of the engine (variants/*.so built with
# _build.build(out=..., defines=...)); BC_B200_LIB selects the library.  Dev tool.
mkdir -p gpurun_out
OUT=gpurun_out/variants.txt; : > $OUT
for rep in 1 2; do
for so in $(ls variants/*.so); do
    echo -n "${so} rep $rep: " | tee -a $OUT
    BC_B200_LIB=$PWD/$so python bench.py --steps 10 --warmup 3 --no-cpu --no-extra 2>/dev/null | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); r=d['roofline']
print('ms/step %.3f  GTEPS %.1f  level ms %.3f' % (d['ms_per_step'], d['value']/1e9, r['ms_per_step']))" | tee -a $OUT
done
done
