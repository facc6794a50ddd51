#!/bin/bash
# Full GPU check: parity tests, smoke, bench (both arms), ncu launch list + full capture.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.log
python __graft_entry__.py smoke 2>&1 | tail -5 | tee gpurun_out/smoke.log
python bench.py --steps 1000 --warmup 20 2>&1 | tail -3 | tee gpurun_out/bench.json
python bench.py --impl reference --steps 2 --warmup 3 2>&1 | tail -2 | tee gpurun_out/bench_ref.json
if [ "${1:-}" = "ncu" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 20 --warmup 5 --quick --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:fa_fwd_sm100 -s 5 -c 2 -o gpurun_out/prof_fa8k -f \
      python bench.py --steps 10 --warmup 5 --quick --no-cpu > gpurun_out/ncu_full.log 2>&1
  tail -3 gpurun_out/ncu_full.log
fi
