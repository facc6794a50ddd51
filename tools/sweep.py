#!/usr/bin/env python
"""Request-throughput sweep on one GPU (BASELINE configs 3 and 5): S in 512..32K, batch 1..64,
variable-length tail padding (len_b ~ U{S/2..S}, seeded).  Reports, per point, the global and
local attention op (ms, algorithmic TFLOP/s over live pairs, GB/s) and, where it fits, the full
classifier forward (ms/request, req/s).  Writes gpurun_out/sweep.json."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_12646_b200 as P  # noqa: E402
from paper_2603_12646_b200.classifier import Classifier, ClassifierConfig, init_weights  # noqa: E402

H, D = 12, 64


def timed(fn, iters):
    """Device time per call.  The calls are replayed from a CUDA graph so that short kernels are not
    timed by the host launch path; falls back to plain event timing if capture fails."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(iters):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters
    except Exception:  # noqa: BLE001
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters


def main():
    rng = np.random.default_rng(0)
    out = {"attention": [], "classifier": []}
    cfg = ClassifierConfig()
    clf = Classifier(cfg, init_weights(cfg, 7), torch.device("cuda:0"))
    for S in (512, 1024, 2048, 4096, 8192, 16384, 32768):
        for B in (1, 2, 4, 8, 16, 32, 64):
            if B * S > 262144:
                continue
            lens = rng.integers(S // 2, S + 1, size=B)
            pb = torch.zeros((B, 1, 1, S), device="cuda")
            for b, n in enumerate(lens):
                pb[b, 0, 0, n:] = -65504.0
            g = torch.Generator(device="cuda").manual_seed(S + B)
            q, k, v = [(torch.rand((B, H, S, D), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
            o = torch.empty_like(q)
            it = max(3, min(50, int(2e11 / (B * S * S * 64 * 12 * 4) * 30)))
            rec = {"S": S, "B": B, "valid_len_mean": float(lens.mean())}
            for name, (wl, wr) in (("global", (-1, -1)), ("local", (63, 64))):
                spec = P.AttentionSpec(0.0, wl, wr, pb)
                ms = timed(lambda: P.flash_attention(q, k, v, spec, out=o), it)
                live = sum(min(int(n), S) * S if wl < 0 else sum(max(0, min(int(n) - 1, i + wr) - max(0, i - wl) + 1) for i in range(0, S, 64)) * 64
                           for n in lens)
                flops = 4.0 * D * H * live
                rec[name] = {"ms": ms, "tflops_live": flops / ms / 1e9, "gbs": 4.0 * B * H * S * D * 2 / ms / 1e6}
            out["attention"].append(rec)
            print(json.dumps(rec), flush=True)
            del q, k, v, o
            if B * S <= 65536:
                ids = torch.randint(0, cfg.vocab_size, (B, S), device="cuda")
                mask = (pb.reshape(B, S) > -30000.0).float()
                ms = timed(lambda: clf.forward(ids, mask), 3)
                crec = {"S": S, "B": B, "ms_per_batch": ms, "ms_per_request": ms / B, "req_per_s": B / ms * 1e3}
                out["classifier"].append(crec)
                print(json.dumps(crec), flush=True)
    # config 3: 3 classifiers x batch 4 at S = 16384 on ONE GPU (12 sequence-forwards)
    ids = torch.randint(0, cfg.vocab_size, (4, 16384), device="cuda")
    ms = timed(lambda: clf.forward(ids, None), 2)
    out["config3_1gpu"] = {"units": 12, "ms_per_batch_of_4": ms, "ms_total_12_units": 3 * ms, "ms_per_request": ms / 4,
                           "ideal_speedup_8gpu": 6.0, "paper_mi300x_ms_per_request": 259.0}
    print(json.dumps(out["config3_1gpu"]), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "sweep.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
