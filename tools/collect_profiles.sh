#!/bin/bash
# Copies the evidence of the last tools/gpu_round.sh run from gpurun_out/ (scratch) into profiles/ (tracked):
# bench lines, ncu summaries (tools/ncu_select.py reads the .ncu-rep files here, no GPU needed), launch lists,
# per-kernel SASS listings of the library as built.  usage: bash tools/collect_profiles.sh [tag]   (default r02)
TAG=${1:-r02}
set -e
cd "$(dirname "$0")/.."
cp gpurun_out/bench.json profiles/${TAG}_bench_line.json
cp gpurun_out/bench_sustained.json profiles/${TAG}_bench_line_1000steps.json
cp gpurun_out/bench_ref.json profiles/${TAG}_bench_reference_line.json
cp gpurun_out/launches.csv profiles/${TAG}_launches.csv
cp gpurun_out/clf_launches.csv profiles/${TAG}_classifier_8k_launches.csv
cp gpurun_out/clf_ab.json profiles/${TAG}_classifier_ab.json
cp gpurun_out/local_bench_line.json profiles/${TAG}_local_bench.json
cp gpurun_out/gemm_bench_8k.json profiles/${TAG}_gemm_bench_8k.json
cp gpurun_out/gemm_bench_16k.json profiles/${TAG}_gemm_bench_16k.json
cp gpurun_out/tmem_rate_probe.jsonl profiles/${TAG}_tmem_rate_probe.jsonl
cp gpurun_out/plan_bench.log profiles/${TAG}_plan_bench.log
[ -f gpurun_out/trace_phases.json ] && cp gpurun_out/trace_phases.json profiles/${TAG}_trace_phases_8k.json
[ -f gpurun_out/trace_local.json ] && cp gpurun_out/trace_local.json profiles/${TAG}_trace_local_8k.json
for f in gpurun_out/sanitizer_*.log; do [ -f "$f" ] && cp "$f" profiles/${TAG}_$(basename "$f"); done
rm -f profiles/ncu_summary.json
python tools/ncu_select.py gpurun_out/prof_fa8k.ncu-rep profiles/${TAG}_fa8k_ncu_selected.csv fa_fwd_sm100_8k profiles/ncu_summary.json > /dev/null
python tools/ncu_select.py gpurun_out/prof_local8k.ncu-rep profiles/${TAG}_local8k_ncu_selected.csv fa_fwd_sm100_local_8k profiles/ncu_summary.json > /dev/null
python tools/ncu_select.py gpurun_out/prof_local16k_b4.ncu-rep profiles/${TAG}_local16k_b4_ncu_selected.csv fa_fwd_sm100_local_16k_b4 profiles/ncu_summary.json > /dev/null
python tools/ncu_select.py gpurun_out/prof_gemm_qkv.ncu-rep profiles/${TAG}_gemm_ncu_selected.csv gemm_nt_sm100_qkv profiles/ncu_summary.json > /dev/null
sed -i "s#profiles/${TAG}_#profiles/${TAG}_#" profiles/ncu_summary.json
python tools/sass_listing.py > /dev/null
python - <<'PY'
import json
s = json.load(open("profiles/ncu_summary.json"))
for k, v in s.items():
    print(k, {x: (round(y, 1) if isinstance(y, float) else y) for x, y in v.items() if x not in ("source", "kernel")})
PY
