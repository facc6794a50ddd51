#!/usr/bin/env python
"""Developer tool (under gpurun): per-phase SM-clock timeline of the softmax warps of CTA 0.

Needs a trace build:  python -c "from paper_2603_12646_b200 import _build; _build.build_variant('trace', {'RF_FA_TRACE': 1})"
then                  RF_FA_LIB=$PWD/paper_2603_12646_b200/librf_fa_trace.so python tools/trace_phases.py
Stamps: 0 loop top, 1 S ready, 2 S in registers, 3 max done, 4 exchange done, 5 exps issued,
6 P stored (wait::st), 7 P-full arrive.  Writes gpurun_out/trace_phases.json."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_12646_b200 as P  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = [(torch.rand(1, 12, S, 64, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
buf = torch.zeros(20 * 64 * 8, device="cuda", dtype=torch.int32)
for _ in range(3):
    P.flash_attention(q, k, v, P.AttentionSpec(), debug_scores=buf.view(torch.float32))
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.uint32).reshape(20, 64, 8).astype(np.int64)
names = ["wait_S", "ld", "max", "xchg", "exp", "st_wait", "arrive", "loop"]
out = {}
for w in (0, 4, 8, 12, 1, 5):
    tw = t[w, 8:56]          # steady-state tiles
    d = np.diff(tw, axis=1) % (1 << 32)                      # phase durations inside a tile
    loop = (tw[1:, 0] - tw[:-1, 7]) % (1 << 32)              # arrive -> next loop top
    period = (tw[1:, 0] - tw[:-1, 0]) % (1 << 32)
    out[f"warp{w}"] = {n: float(np.median(d[:, i])) for i, n in enumerate(names[:7])}
    out[f"warp{w}"]["loop"] = float(np.median(loop))
    out[f"warp{w}"]["period"] = float(np.median(period))
# phase offsets between warps at the "exp start" stamp (4)
base = t[0, 8:56, 4]
out["exp_start_offset_vs_warp0"] = {f"warp{w}": float(np.median((t[w, 8:56, 4] - base))) for w in (4, 8, 12)}
# UMMA issuer (warp 17): 0 loop top, 1 V ready, 2 P_A ready, 3 PV_A+QK_B issued, 4 P_B ready, 5 PV_B issued,
# 6 K(i+2) ready, 7 QK_A(i+2) issued
tm = t[17, 8:56]
dm = np.diff(tm, axis=1) % (1 << 32)
out["mma_warp"] = {n: float(np.median(dm[:, i])) for i, n in enumerate(
    ["wait_V", "wait_PA", "issue_PVA_QKB", "wait_PB", "issue_PVB", "wait_K", "issue_QKA"])}
out["mma_warp"]["period"] = float(np.median((tm[1:, 0] - tm[:-1, 0]) % (1 << 32)))
# absolute alignment for one steady-state tile (i = 20): all stamps relative to warp 0's stamp 0 of tile 20
i0 = 20
ref = t[0, i0, 0]
out["abs_tile20"] = {"A_warp0": [int(x - ref) for x in t[0, i0]], "B_warp8": [int(x - ref) for x in t[8, i0]],
                     "mma_i18": [int(x - ref) for x in t[17, i0 - 2]], "mma_i19": [int(x - ref) for x in t[17, i0 - 1]],
                     "mma_i20": [int(x - ref) for x in t[17, i0]]}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "trace_phases.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
