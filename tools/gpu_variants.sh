#!/bin/bash
# compare experimental builds of the kernel (RF_FA_LIB override)
mkdir -p gpurun_out; rm -f gpurun_out/bringup.jsonl
for lib in "$@"; do
  echo "== $lib"
  RF_FA_LIB=$PWD/paper_2603_12646_b200/$lib timeout 600 python tools/bringup.py all ts_local_pad,cross_8k,time_8k_ts,time_32k_ts 2>&1 | grep -v "^#" | cut -c1-260
done
