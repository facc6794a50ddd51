#!/bin/bash
# quick GPU iteration: chosen bring-up cases (correctness + timing)
mkdir -p gpurun_out; rm -f gpurun_out/bringup.jsonl
timeout 900 python tools/bringup.py all "${1:-ts_128,ts_256,ts_512,ts_1000_ragged,ts_pad,ts_local_pad,ts_onesided,ts_tiny,ts_allpad,cross_8k,cross_8k_local_pad,time_8k_ts,time_16k_ts,time_32k_ts,time_8k_local_ts}" 2>&1 | grep -v "^#" | cut -c1-420
