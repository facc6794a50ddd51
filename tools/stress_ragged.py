#!/usr/bin/env python
"""Developer tool (under gpurun): ragged lengths x batches x masks x windows through the persistent schedules of the dense
kernel (and the narrow-window kernel), each case in its own process under a timeout (a hang is a finding, not a stuck run),
checked against the generic SIMT kernel on two heads."""
import itertools, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASE = r'''
import sys, torch
sys.path.insert(0, %r)
import paper_2603_12646_b200 as P
B, S, wl, wr, pad, dt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), sys.argv[6]
dtype = torch.float16 if dt == "f16" else torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(S + B)
q, k, v = [(torch.rand(B, 12, S, 64, device="cuda", generator=g) * 2 - 1).to(dtype) for _ in range(3)]
pb = None
if pad:
    mask = torch.ones(B, 1, 1, S, device="cuda")
    for b in range(B):
        mask[b, ..., S - (b * 997 + 130) %% S:] = 0
    pb = P.pad_bias_from_mask(mask)
spec = P.AttentionSpec(0.0, wl, wr, pb)
st = P.FlashStats()
o = P.flash_attention(q, k, v, spec, stats=st, out_dtype=torch.float32)
torch.cuda.synchronize()
r = P.flash_attention(q[:, 3:5].contiguous(), k[:, 3:5].contiguous(), v[:, 3:5].contiguous(), spec, kernel="simt", out_dtype=torch.float32)
err = (o[:, 3:5] - r).abs().max().item()
again = P.flash_attention(q, k, v, spec, out_dtype=torch.float32)
print("grid", st.grid_ctas, "err %%.2e" %% err, "deterministic", bool(torch.equal(o, again)), "OK" if err <= 5e-3 and torch.equal(o, again) else "MISMATCH")
''' % ROOT
cases = []
for B, S in ((1, 4097), (1, 4225), (2, 4097), (3, 2305), (5, 1281), (2, 6000), (8, 4097)):
    for (wl, wr) in ((-1, -1), (300, 10), (63, 64)):
        for pad in (0, 1):
            cases.append((B, S, wl, wr, pad, "bf16"))
cases += [(1, 8193, -1, -1, 1, "f16"), (4, 4097, -1, -1, 0, "f16")]
bad = 0
for c in cases:
    try:
        r = subprocess.run([sys.executable, "-c", CASE] + [str(x) for x in c], capture_output=True, text=True, timeout=90)
        out = r.stdout.strip() or ("ERR " + r.stderr.strip()[-200:])
    except subprocess.TimeoutExpired:
        out = "TIMEOUT (hang)"
    if "OK" not in out:
        bad += 1
    print(c, out, flush=True)
print("bad cases:", bad)
