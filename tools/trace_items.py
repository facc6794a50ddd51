#!/usr/bin/env python
"""Developer tool (trace build, see trace_phases.py): tile-to-tile periods of CTA 0's softmax warp 0 and warp 8 over the
first 64 key tiles it processes -- item boundaries (epilogue, first tile of the next item) show up as long periods."""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_12646_b200 as P
S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
g = torch.Generator(device="cuda").manual_seed(1)
q, k, v = [(torch.rand(1, 12, S, 64, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
T = int(os.environ.get("TRACE_TILES", "64"))
buf = torch.zeros(20 * T * 8, device="cuda", dtype=torch.int32)
for _ in range(3):
    P.flash_attention(q, k, v, P.AttentionSpec(), debug_scores=buf.view(torch.float32))
torch.cuda.synchronize()
t = buf.cpu().numpy().astype(np.uint32).reshape(20, T, 8).astype(np.int64)
for w in (0, 8):
    s0 = t[w, :, 0]
    per = np.diff(s0) % (1 << 32)
    print(f"warp{w} periods:", " ".join(str(int(x)) for x in per))
    print(f"warp{w} first tile stamps rel:", [int((x - t[0, 0, 0]) % (1 << 32)) for x in t[w, 0]])

ks = t[18, 0, :4]
ref = t[0, 0, 0]
print("kernel stamps rel. to warp 0's first loop top: entry, prologue done, dependencies resolved, teardown:",
      [int(((x - ref + (1 << 31)) % (1 << 32)) - (1 << 31)) for x in ks])
last = max(int(x) for x in t[0, :, 7] if x)
print("warp0 last P-full arrive rel.:", int((last - ref) % (1 << 32)))
