#!/usr/bin/env python
"""Developer tool (under gpurun): why the 8K global attention inside the classifier is slower than the benchmarked op.
Times the dense kernel (CUDA-graph replay, rotating inputs) for bf16 / f16, the [B,H,S,d] layout / the packed
[B,S,3,H,d] projection output the classifier feeds it, and uniform / normal-distributed inputs."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_12646_b200 as P

S, H, D, N = 8192, 12, 64, 4
def run(dtype, packed, dist):
    g = torch.Generator(device="cuda").manual_seed(1)
    calls = []
    for _ in range(N):
        if packed:
            qkv = (torch.randn(1, S, 3, H, D, device="cuda", generator=g) if dist == "normal" else torch.rand(1, S, 3, H, D, device="cuda", generator=g) * 2 - 1).to(dtype)
            out = torch.empty(1, S, H, D, device="cuda", dtype=dtype)
            calls.append((qkv[:, :, 0].permute(0, 2, 1, 3), qkv[:, :, 1].permute(0, 2, 1, 3), qkv[:, :, 2].permute(0, 2, 1, 3), out.permute(0, 2, 1, 3)))
        else:
            q, k, v = [(torch.randn(1, H, S, D, device="cuda", generator=g) if dist == "normal" else torch.rand(1, H, S, D, device="cuda", generator=g) * 2 - 1).to(dtype) for _ in range(3)]
            calls.append((q, k, v, torch.empty_like(q)))
    spec = P.AttentionSpec()
    for c in calls: P.flash_attention(c[0], c[1], c[2], spec, out=c[3])
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for c in calls: P.flash_attention(c[0], c[1], c[2], spec, out=c[3])
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): gr.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (20 * N) * 1e3
res = {}
for dtype in (torch.bfloat16, torch.float16):
    for packed in (False, True):
        for dist in ("uniform", "normal"):
            res[f"{str(dtype)[6:]}_{'packed' if packed else 'bhsd'}_{dist}"] = round(run(dtype, packed, dist), 1)
print(json.dumps(res))
