#!/usr/bin/env python
"""Developer stress (under gpurun): the host entry point over many calls of varying shape, padded and not, local and
global, checked against the device path on the same (bf16-rounded) inputs -- exercises the host rounding pool, the
adaptive host/device choice, staging reuse across chunk sizes and the pool's shutdown / restart."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2603_12646_b200 as P
from paper_2603_12646_b200 import capi
rng = np.random.default_rng(3)
lib = capi.load()
worst = 0.0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 120):
    B = int(rng.integers(1, 4)); H = int(rng.choice([1, 2, 6, 12])); S = int(rng.choice([384, 1000, 2048, 4096, 8192]))
    if B * H * S > 12 * 8192: S = 2048
    wl, wr = (63, 64) if rng.random() < 0.3 else (-1, -1)
    q, k, v = [rng.standard_normal((B, H, S, 64)).astype(np.float32) for _ in range(3)]
    pb = None
    if rng.random() < 0.4:
        pb = np.zeros((B, 1, 1, S), np.float32)
        pb[-1, 0, 0, int(rng.integers(1, S)):] = -65504.0
    spec = P.AttentionSpec(0.0, wl, wr, pb)
    out = P.flash_attention(q, k, v, spec, device=0)
    tq, tk, tv = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k, v)]
    tpb = torch.from_numpy(pb).cuda() if pb is not None else None
    ref = P.flash_attention(tq, tk, tv, P.AttentionSpec(0.0, wl, wr, tpb), out_dtype=torch.float32).cpu().numpy()
    # (not bit-equal in general: the host path runs (batch, head-range) chunks, so the persistent schedule cuts the
    # query-tile pairs elsewhere than the one full call does, and a cut pair sums its two partials in another order)
    err = float(np.abs(out - ref).max())
    worst = max(worst, err)
    assert err <= 5e-3 and np.isfinite(out).all(), (it, B, H, S, wl, err)
    out2 = P.flash_attention(q, k, v, spec, device=0)   # the same call again: same bits, whichever way it rounds
    assert np.array_equal(out, out2), (it, B, H, S, wl)
    if it % 37 == 36:
        lib.rf_fa_host_release()
print("host stress ok, worst |host - device| =", worst, capi.host_transfer_counters())
