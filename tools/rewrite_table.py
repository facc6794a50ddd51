#!/usr/bin/env python
"""SDPA graph vs rewritten graph on the B200 (the reference's Table-3 experiment, PAPER.md:389-407,
through this repo's graph executor): one ModernBERT-base-shaped attention layer (H=12, d=64) per
sequence length, original graph (materialises [1,12,S,S] scores, mask and probabilities in HBM)
against the rewritten one (FusedFlashAttention).  Writes gpurun_out/rewrite_table.json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import graph_fixtures as F  # noqa: E402
from paper_2603_12646_b200 import RewriteOptions, graph as G, mask_memory_bytes  # noqa: E402

rows = []
for kind in ("g", "l"):
    for S in (512, 1024, 2048, 4096, 8192):
        fx = F.build_attention_fixture(batch=1, heads=12, seq=S, head_dim=64, layers=kind)
        rew = G.rewrite(fx, RewriteOptions(64, 128))
        rng = np.random.default_rng(S)
        ins = {"hidden": rng.uniform(-1, 1, (1, 12, S, 64)).astype(np.float32), "attention_mask": np.ones((1, 1, 1, S), np.float32)}
        ins["attention_mask"][..., S - S // 16:] = 0
        sa, sb = G.InterpretStats(), G.InterpretStats()
        for _ in range(2):  # second run: pool warm
            a = G.interpret(fx, ins, stats=sa)["layer0/out"]
            b = G.interpret(rew, ins, stats=sb)["layer0/out"]
        valid = S - S // 16
        rows.append({"layer": "global" if kind == "g" else "local(63,64)", "S": S,
                     "max_abs_diff_valid_rows": float(np.abs(a - b)[:, :, :valid].max()),
                     "sdpa_graph": {"device_ms": sa.device_ms, "peak_MB": sa.peak_device_bytes / 1e6,
                                    "largest_tensor_MB": sa.largest_tensor_bytes / 1e6, "launches": sa.launches},
                     "rewritten_graph": {"device_ms": sb.device_ms, "peak_MB": sb.peak_device_bytes / 1e6,
                                         "largest_tensor_MB": sb.largest_tensor_bytes / 1e6, "launches": sb.launches},
                     "mask_memory_model_f16_MB": mask_memory_bytes(1, 12, S, 2) / 1e6})
        print(json.dumps(rows[-1]), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "rewrite_table.json"), "w") as f:
    json.dump(rows, f, indent=1)
