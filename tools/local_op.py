#!/usr/bin/env python
"""Developer tool (under gpurun / ncu): a few launches of the 8K local-window layer (B=1, H=12, S=8192,
window (63,64)), optionally with a padded tail, so ncu can capture fa_fwd_sm100_local_kernel."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_12646_b200 as P  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = torch.Generator(device="cuda").manual_seed(1)
sets = [[(torch.rand(B, 12, S, 64, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
        for _ in range(6)]  # 6 x 38 MB of inputs (> L2 together with the outputs)
outs = [torch.empty_like(s[0]) for s in sets]
wl, wr = P.local_window_attrs()
for i in range(12):
    P.flash_attention(*sets[i % 6], P.AttentionSpec(0.0, wl, wr), out=outs[i % 6])
torch.cuda.synchronize()
