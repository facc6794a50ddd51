#!/usr/bin/env python
"""memory-model, measured (reference CLI `memory-model`, tools/main.cpp:151-171).

Prints the reference's table -- S, sdpa_bytes = mask_memory_bytes(batch, heads, S, bpe), fa_bytes =
fa_memory_bytes(batch, heads, S, head_dim, tile, bpe), fits_budget (attention.cpp:244-252) -- and beside it
what the B200 build actually takes: the fused operator's own footprint (output + workspace, exact allocator
high-water mark) and the whole classifier session (weights + activations + library workspaces) per sequence
length as the DRIVER sees it (cudaMemGetInfo before / after, allocator caches emptied first).  Writes gpurun_out/memory_table.json.

usage: python tools/memory_table.py [--heads 12] [--batch 1] [--budget-mb 718] [--sizes 512,...]"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_12646_b200 as P  # noqa: E402
from paper_2603_12646_b200.classifier import Classifier, ClassifierConfig, init_weights  # noqa: E402


def used_bytes():
    torch.cuda.synchronize()
    free, total = torch.cuda.mem_get_info()
    return total - free


def measure_op(batch, heads, S, d):
    """Bytes the fused op allocates on top of its inputs: output + workspace, from the allocator's exact
    high-water mark (the driver view is too coarse for one op: torch carves 2 MiB / 20 MiB blocks)."""
    q = (torch.rand((batch, heads, S, d), device="cuda") * 2 - 1).to(torch.bfloat16)
    pb = torch.zeros((batch, 1, 1, S), device="cuda")
    pb[..., S - S // 8:] = -65504.0
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    before = torch.cuda.memory_allocated()
    st = P.FlashStats()
    out = P.flash_attention(q, q, q, P.AttentionSpec(pad_bias=pb), stats=st)
    torch.cuda.synchronize()
    res = {"measured_op_bytes": torch.cuda.max_memory_allocated() - before,
           "output_bytes": out.numel() * out.element_size(), "workspace_bytes": int(st.workspace_bytes),
           "score_matrix_bytes": 0}
    del out, q, pb
    torch.cuda.empty_cache()
    return res


def measure_session(S, batch=1):
    """Driver-level bytes of one classifier session at sequence length S: everything the process
    allocates between 'model not loaded' and 'forward finished' (caches are not released in between,
    so the difference is the high-water mark)."""
    torch.cuda.empty_cache()
    before = used_bytes()
    cfg = ClassifierConfig()
    clf = Classifier(cfg, init_weights(cfg, 7), torch.device("cuda:0"))
    ids = torch.randint(0, cfg.vocab_size, (batch, S), device="cuda")
    mask = torch.ones(batch, S, device="cuda")
    mask[:, S - S // 8:] = 0
    logits = clf.forward(ids, mask)
    after = used_bytes()
    res = {"session_bytes": after - before, "weights_bytes": clf.weight_bytes(),
           "torch_peak_allocated": torch.cuda.max_memory_allocated(), "logits": [float(x) for x in logits[0].cpu()]}
    del clf, ids, mask, logits
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=12)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--dtype", default="f16", choices=["f16", "f32"])
    ap.add_argument("--budget-mb", type=int, default=718)
    ap.add_argument("--head-dim", type=int, default=64)
    ap.add_argument("--tile", type=int, default=64)
    ap.add_argument("--sizes", default="512,1024,2048,4096,8192,16384,32768")
    ap.add_argument("--sessions", default="8192,16384,32768")
    a = ap.parse_args()
    bpe = 4 if a.dtype == "f32" else 2
    budget = a.budget_mb * 1024 * 1024
    # touch the device and load every module before the first measurement
    P.flash_attention(*[torch.zeros(1, 1, 128, 64, device="cuda", dtype=torch.bfloat16)] * 3)
    torch.cuda.synchronize()
    rows = []
    print(f"{'S':>8}  {'sdpa_bytes':>16}  {'fa_bytes':>14}  {'fits_budget':>12}  {'measured_op':>14}  {'workspace':>10}")
    for S in [int(x) for x in a.sizes.split(",")]:
        sdpa = P.mask_memory_bytes(a.batch, a.heads, S, bpe)
        fa = P.fa_memory_bytes(a.batch, a.heads, S, a.head_dim, a.tile, bpe)
        m = measure_op(a.batch, a.heads, S, a.head_dim)
        rows.append({"S": S, "sdpa_bytes": sdpa, "fa_bytes": fa, "fits_budget": sdpa <= budget, **m})
        print(f"{S:>8}  {sdpa:>16}  {fa:>14}  {'yes' if sdpa <= budget else 'no':>12}  {m['measured_op_bytes']:>14}  {m['workspace_bytes']:>10}")
    print(f"budget: {budget} bytes ({a.budget_mb} MiB), dtype {a.dtype}, batch {a.batch}, heads {a.heads}")
    sessions = []
    for S in [int(x) for x in a.sessions.split(",") if x]:
        torch.cuda.reset_peak_memory_stats()
        s = measure_session(S)
        s["S"] = S
        s["under_800MB"] = s["session_bytes"] < 800e6
        sessions.append(s)
        print(f"classifier session S={S}: {s['session_bytes'] / 1e6:.1f} MB by cudaMemGetInfo "
              f"(weights {s['weights_bytes'] / 1e6:.1f} MB; torch peak allocated {s['torch_peak_allocated'] / 1e6:.1f} MB)")
    out = {"table": rows, "sessions": sessions, "args": vars(a),
           "method": "cudaMemGetInfo before/after with torch's caching allocator emptied before each measurement"}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "memory_table.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
