#!/usr/bin/env python
"""Where does the per-op time of the 8K global layer go between the device and the host launch path?

Times the same op (B=1, H=12, S=8192, d=64, bf16, inputs rotating through > L2) three ways:
  direct   P.flash_attention per step (validation + plan + 3 tensor maps + launches every call)
  plan     FaPlan.launch per step (launches only)
  graph    the plan launches captured in one CUDA graph and replayed
and reports, for each, the device time per op (CUDA events) and the host time to enqueue one op.
Writes gpurun_out/host_gap_probe.json.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2603_12646_b200 as P  # noqa: E402

B, H, S, D = 1, 12, int(os.environ.get("PROBE_S", 8192)), 64
N_SETS, STEPS = 6, 300
g = torch.Generator(device="cuda").manual_seed(1)
sets = [tuple((torch.rand((B, H, S, D), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3))
        for _ in range(N_SETS)]
outs = [torch.empty((B, H, S, D), device="cuda", dtype=torch.bfloat16) for _ in range(N_SETS)]
spec = P.AttentionSpec()
plans = [P.FaPlan(*sets[i], spec, out=outs[i]) for i in range(N_SETS)]
flops = 4.0 * B * H * S * S * D


def timed(fn, steps):
    for i in range(20):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for i in range(steps):
        fn(i)
    e1.record()
    t_host = time.perf_counter() - t0
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {"device_ms_per_op": ms, "tflops": flops / ms / 1e9, "host_enqueue_us_per_op": t_host / steps * 1e6}


res = {"S": S}
res["direct"] = timed(lambda i: P.flash_attention(*sets[i % N_SETS], spec, out=outs[i % N_SETS]), STEPS)
res["plan"] = timed(lambda i: plans[i % N_SETS].launch(), STEPS)
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    for pl in plans:
        pl.launch()
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    for pl in plans:
        pl.launch()
r = timed(lambda i: graph.replay(), STEPS // N_SETS)
res["graph"] = {"device_ms_per_op": r["device_ms_per_op"] / N_SETS, "tflops": flops / (r["device_ms_per_op"] / N_SETS) / 1e9,
                "host_enqueue_us_per_op": r["host_enqueue_us_per_op"] / N_SETS}
res["status"] = [pl.status() for pl in plans]
print(json.dumps(res, indent=1))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "host_gap_probe.json"), "w") as f:
    json.dump(res, f, indent=1)
