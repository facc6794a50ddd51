#!/bin/bash
# one ncu --set full capture of the 8K attention kernel (+ launch list)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:fa_fwd_sm100 -s 5 -c 1 -o gpurun_out/prof_fa8k -f \
    python bench.py --steps 10 --warmup 5 --quick --no-cpu > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log | cut -c1-300
