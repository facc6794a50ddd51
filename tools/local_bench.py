#!/usr/bin/env python
"""Developer tool (under gpurun): device time of the narrow-window layer by CUDA-graph replay over rotating
input sets (> L2), against the HBM roofline of its algorithmic bytes (Q, K, V read once, O written once).
usage: python tools/local_bench.py [--lib path/to/variant.so is taken from RF_FA_LIB]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_12646_b200 as P  # noqa: E402

HBM = 6544.7
if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
    HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]


def graph_time(fn, n_sets, replays=20):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for i in range(n_sets):
            fn(i)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(n_sets):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(replays):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (replays * n_sets)


def main():
    wl, wr = P.local_window_attrs()
    out = {}
    for (B, S, n_sets, padded) in ((1, 8192, 6, False), (1, 8192, 6, True), (4, 16384, 2, False), (1, 32768, 3, False),
                                   (8, 8192, 2, True)):
        g = torch.Generator(device="cuda").manual_seed(1)
        sets = [[(torch.rand(B, 12, S, 64, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
                for _ in range(n_sets)]
        outs = [torch.empty_like(s[0]) for s in sets]
        pb = None
        if padded:
            mask = torch.ones(B, 1, 1, S, device="cuda")
            for b in range(B):
                mask[b, ..., S - (b + 1) * S // 16:] = 0
            pb = P.pad_bias_from_mask(mask)
        spec = P.AttentionSpec(0.0, wl, wr, pb)
        ms = graph_time(lambda i: P.flash_attention(*sets[i], spec, out=outs[i]), n_sets)
        nbytes = 4.0 * B * 12 * S * 64 * 2
        out[f"B{B}_S{S}{'_pad' if padded else ''}"] = {"us": ms * 1e3, "gbs": nbytes / ms / 1e6, "frac_of_hbm": nbytes / ms / 1e6 / HBM}
        del sets, outs
    print(json.dumps(out))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "local_bench.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
