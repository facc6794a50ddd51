#!/bin/bash
# Developer aid: same-box A/B of two builds of the library (RF_FA_LIB) on the bench line's timed region and on
# tools/plan_bench.py.  usage: bash tools/ab.sh path/to/base.so [rounds]
BASE=$1; R=${2:-2}
for i in $(seq $R); do
for lib in base new; do
  if [ $lib = base ]; then export RF_FA_LIB=$BASE; else unset RF_FA_LIB; fi
  python bench.py --gpus 1 --steps 20 --warmup 5 --quick --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib bench20', round(d['value'],1), round(d['ms_per_step']*1e3,2))"
  python tools/plan_bench.py
done
done
