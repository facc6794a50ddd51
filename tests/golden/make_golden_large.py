#!/usr/bin/env python
"""Golden vectors at the sizes BASELINE.json states (configs 2, 3, 4), generated from the UNMODIFIED reference
operator (oracle/_ref/libref_attn.so = /root/reference/proj/core/src/{attention,tensor}.cpp).

Run in the build container (needs /root/reference; takes ~10 minutes on 8 cores):

    python tests/golden/make_golden_large.py

Writes tests/golden/large_golden.npz (< 1 MB), read by tests/test_gpu_large_sizes.py on the GPU box, where
/root/reference does not exist.  Contents:

* config 2 -- logits of the full 22-layer ModernBERT-base-shaped classifier at B=1, S=8192 (default vocabulary,
  weights init_weights(cfg, 7), f16-rounded matrices like the device copy), every attention call through the
  reference operator; two masks as tools/main.cpp:88-98 builds them: all ones, and ones followed by S/8 zeros.
  (Everything of that model but the attention operator is this build's own construction: SURVEY 8(c).)
* config 3 / 4 -- single-head outputs of the operator at S=16384 (tail padding to 12345 keys) and S=32768
  (global, and local (63,64) with padding), inputs Tensor::random (seeded, rounded to bf16).  Only a fixed
  subset of query rows is stored (ROWS below) to keep the fixture small; the tests compare those rows.
"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
from oracle_model import oracle_forward  # noqa: E402

from paper_2603_12646_b200.classifier import ClassifierConfig, init_weights  # noqa: E402

O.build()
assert O.have_reference(), "needs oracle/_ref (built from /root/reference)"
R = "reference"
out = {}


def rows_subset(S):
    """Rows stored for a length-S sequence: both ends, the middle, and every 257th row."""
    idx = set(range(0, 64)) | set(range(S // 2 - 32, S // 2 + 32)) | set(range(S - 64, S)) | set(range(0, S, 257))
    return np.array(sorted(idx), dtype=np.int64)


def one_head(tag, seed, S, wl, wr, valid_len):
    t0 = time.time()
    q, k, v = [O.round_bf16(t) for t in O.random_tensors(seed, (1, 1, S, 64), 3, impl=R)]
    pb = None
    if valid_len is not None:
        pb = np.zeros((1, 1, 1, S), np.float32)
        pb[..., valid_len:] = O.MASK_VALUE
    o = O.flash_attention(q, k, v, 0.0, wl, wr, pb, impl=R, threads=1)
    rows = rows_subset(S)
    print(f"{tag}: {time.time() - t0:.1f} s", flush=True)
    return tag, {"rows": rows, "out": o[0, 0, rows].copy(),
                 "meta": np.array([seed, S, wl, wr, -1 if valid_len is None else valid_len], dtype=np.int64)}


heads = [("op16k_pad12345", 316, 16384, -1, -1, 12345),
         ("op32k_global", 432, 32768, -1, -1, None),
         ("op32k_local_pad30000", 433, 32768, 63, 64, 30000),
         ("op16k_global", 317, 16384, -1, -1, None)]
pool = ThreadPoolExecutor(max_workers=4)   # ctypes releases the GIL: the long single-head runs go side by side
futs = [pool.submit(one_head, *h) for h in heads]

# ---- config 2: the classifier at 8K (4 threads while the single-head jobs run)
cfg = ClassifierConfig()
w = init_weights(cfg, 7)
S = 8192
ids = torch.randint(0, cfg.vocab_size, (1, S), generator=torch.Generator().manual_seed(S))
mask_ones = torch.ones((1, S))
mask_tail = torch.ones((1, S))
mask_tail[0, S - S // 8:] = 0
for tag, mask in (("clf8k_ones", mask_ones), ("clf8k_tail", mask_tail)):
    t0 = time.time()
    logits = oracle_forward(cfg, w, ids, mask, O, impl=R, threads=4)
    out[f"{tag}_logits"] = logits.astype(np.float32)
    print(f"{tag}: {time.time() - t0:.1f} s  logits {logits}", flush=True)
out["clf8k_ids_head"] = ids[0, :16].numpy()        # guards against a torch RNG change on the test side
out["clf8k_weight_probe"] = w["l21.wo2"].flatten()[:8].numpy()

for f in futs:
    tag, d = f.result()
    for key, val in d.items():
        out[f"{tag}_{key}"] = val

path = os.path.join(HERE, "large_golden.npz")
np.savez_compressed(path, **out)
print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")
