#!/bin/bash
# Evidence run of a round: parity tests, smoke, bench (both arms), ncu launch lists and --set full captures of the dense,
# narrow-window and projection kernels, classifier launch list.  Output: gpurun_out/ (copied to profiles/ by hand).
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -6 | tee gpurun_out/pytest_gpu.log
python __graft_entry__.py smoke 2>&1 | tail -5 | tee gpurun_out/smoke.log
python bench.py --gpus 1 --steps 20 --warmup 5 2>&1 | tail -1 > gpurun_out/bench.json; cut -c1-600 gpurun_out/bench.json
python bench.py --steps 1000 --warmup 20 --quick --no-cpu 2>&1 | tail -1 > gpurun_out/bench_sustained.json; cut -c1-300 gpurun_out/bench_sustained.json
python bench.py --impl reference --steps 2 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_ref.json; cut -c1-300 gpurun_out/bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 5 --quick --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fa_fwd_sm100_kernel -s 5 -c 1 -o gpurun_out/prof_fa8k -f \
    python bench.py --steps 10 --warmup 5 --quick --no-cpu > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fa_fwd_sm100_local -s 6 -c 1 -o gpurun_out/prof_local8k -f \
    python tools/local_op.py 8192 1 > gpurun_out/ncu_local.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fa_fwd_sm100_local -s 2 -c 1 -o gpurun_out/prof_local16k_b4 -f \
    python tools/local_op.py 16384 4 > gpurun_out/ncu_local16.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_nt_sm100 -s 8 -c 1 -o gpurun_out/prof_gemm_qkv -f \
    python tools/gemm_bench.py > gpurun_out/ncu_gemm.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "measured_forward/" --csv \
    --log-file gpurun_out/clf_launches.csv python tools/clf_launches.py > gpurun_out/clf_launches.log 2>&1
python tools/local_bench.py 2>&1 | tail -1 > gpurun_out/local_bench_line.json
python tools/gemm_bench.py 2>&1 | tail -1 > gpurun_out/gemm_bench_8k.json
python tools/gemm_bench.py 16384 2>&1 | tail -1 > gpurun_out/gemm_bench_16k.json
python tools/clf_ab.py 2>&1 | tail -1 > gpurun_out/clf_ab.json
timeout 120 tools/probes/tmem_rate.bin > gpurun_out/tmem_rate_probe.jsonl 2>&1
python tools/plan_bench.py > gpurun_out/plan_bench.log 2>&1
cat gpurun_out/local_bench_line.json gpurun_out/clf_ab.json | cut -c1-700
