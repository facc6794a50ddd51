#!/usr/bin/env python
"""Developer tool (under gpurun): raw phase stamps of CTA 0 for a windowed layer (trace build, see
trace_phases.py).  Prints, per warp, the stamps of every key tile CTA 0 processed, relative to the
first stamp of warp 0, plus the device time of the whole launch."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_12646_b200 as P  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
wl, wr = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (63, 64)
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = [(torch.rand(1, 12, S, 64, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
buf = torch.zeros(12 * 64 * 8, device="cuda", dtype=torch.int32)
spec = P.AttentionSpec(0.0, wl, wr)
for _ in range(3):
    buf.zero_()
    P.flash_attention(q, k, v, spec, debug_scores=buf.view(torch.float32))
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.uint32).reshape(12, 64, 8).astype(np.int64)
ref = t[0, 0, 0]
out = {}
for w in (0, 3, 4, 7, 9):
    rows = []
    for i in range(64):
        if not t[w, i].any():
            break
        rows.append([int((x - ref) % (1 << 32)) if x else None for x in t[w, i]])
    out[f"warp{w}"] = rows
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    P.flash_attention(q, k, v, spec, debug_scores=buf.view(torch.float32))
e1.record()
torch.cuda.synchronize()
out["us_per_launch"] = e0.elapsed_time(e1) * 1000 / 50
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "trace_local.json"), "w") as f:
    json.dump(out, f)
for kx, vx in out.items():
    print(kx, json.dumps(vx))
