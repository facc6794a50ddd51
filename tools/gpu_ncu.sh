#!/bin/bash
# ncu evidence for the round: launch list of the bench command, one --set full capture of the dense 8K
# attention kernel and one of the narrow-window kernel (read back here with tools/ncu_select.py)
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 5 --quick --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fa_fwd_sm100_kernel -s 5 -c 2 -o gpurun_out/prof_fa8k -f \
    python bench.py --steps 10 --warmup 5 --quick --no-cpu > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log | cut -c1-300
ncu --set full --clock-control none --import-source on -k regex:fa_fwd_sm100_local -s 6 -c 2 -o gpurun_out/prof_local8k -f \
    python tools/local_op.py 8192 1 > gpurun_out/ncu_local.log 2>&1
tail -2 gpurun_out/ncu_local.log | cut -c1-300
