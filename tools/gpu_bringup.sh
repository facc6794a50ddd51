#!/bin/bash
# GPU bring-up run (under gpurun): probes, correctness ladder, first timings.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
rm -f gpurun_out/bringup.jsonl
timeout 1500 python tools/bringup.py all "${1:-}" 2>&1 | tail -n 200
