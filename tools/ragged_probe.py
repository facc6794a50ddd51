#!/usr/bin/env python
"""Developer tool (under gpurun): which kernel mishandles ragged lengths at scale (S = 8193 = 64 * 128 + 1)?  Each case runs
in its own process under a timeout."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import sys, os, torch
sys.path.insert(0, %r)
import paper_2603_12646_b200 as P
from paper_2603_12646_b200.gemm import gemm_nt
case, S = sys.argv[1], int(sys.argv[2])
g = torch.Generator(device="cuda").manual_seed(1)
if case in ("dense", "local", "dense_f16", "dense_heads"):
    dt = torch.float16 if case == "dense_f16" else torch.bfloat16
    q, k, v = [(torch.rand(1, 12, S, 64, device="cuda", generator=g) * 2 - 1).to(dt) for _ in range(3)]
    wl, wr = (63, 64) if case == "local" else (-1, -1)
    st = P.FlashStats()
    o = P.flash_attention(q, k, v, P.AttentionSpec(0.0, wl, wr), stats=st)
    torch.cuda.synchronize()
    print(case, S, "ok grid", st.grid_ctas, "finite", bool(torch.isfinite(o.float()).all()))
else:
    a = torch.randn(S, 768, device="cuda").to(torch.bfloat16); w = (torch.randn(2304, 768, device="cuda") * 0.05).to(torch.bfloat16)
    y = gemm_nt(a, w)
    torch.cuda.synchronize()
    err = (y.float() - a.float() @ w.float().t()).abs().max().item()
    print(case, S, "ok err", err)
''' % ROOT
for case in ("gemm", "local", "dense", "dense_f16"):
    for S in (8193, 2305, 4097):
        try:
            r = subprocess.run([sys.executable, "-c", CASE, case, str(S)], capture_output=True, text=True, timeout=60)
            print((r.stdout.strip() or r.stderr.strip()[-300:]), flush=True)
        except subprocess.TimeoutExpired:
            print(case, S, "TIMEOUT (hang)", flush=True)
