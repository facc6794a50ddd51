#!/bin/bash
# compute-sanitizer memcheck over small invocations of every kernel family (developer aid):
# smoke (dense + narrow-window + host path), a padded batch (bias + norms pre-pass), the classifier glue and
# the native session.  Output: gpurun_out/sanitizer_*.log
mkdir -p gpurun_out
compute-sanitizer --tool memcheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/sanitizer_smoke.log 2>&1
echo "smoke rc=$?"; tail -3 gpurun_out/sanitizer_smoke.log
compute-sanitizer --tool memcheck --error-exitcode 9 python - > gpurun_out/sanitizer_mixed.log 2>&1 <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2603_12646_b200 as P
from paper_2603_12646_b200.classifier import Classifier, ClassifierConfig, NativeClassifier, init_weights
g = torch.Generator(device="cuda").manual_seed(0)
for (B, H, S) in ((2, 2, 1280), (1, 1, 1000), (3, 12, 2048)):
    q, k, v = [(torch.rand((B, H, S, 64), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
    mask = torch.ones(B, 1, 1, S, device="cuda")
    mask[0, ..., S - 77:] = 0
    pb = P.pad_bias_from_mask(mask)
    for spec in (P.AttentionSpec(), P.AttentionSpec(0.0, -1, -1, pb), P.AttentionSpec(0.0, 63, 64, pb), P.AttentionSpec(0.0, 5, 9),
                 P.AttentionSpec(0.0, 300, 10, pb)):
        o = P.flash_attention(q, k, v, spec)
        torch.cuda.synchronize()
        assert torch.isfinite(o.float()).all()
cfg = ClassifierConfig(vocab_size=1000, n_layers=3, n_labels=3)
w = init_weights(cfg, 1)
ids = torch.randint(0, 1000, (2, 700))
m = torch.ones(2, 700)
m[1, 650:] = 0
a = Classifier(cfg, w, torch.device("cuda:0")).forward(ids.cuda(), m.cuda()).cpu()
nat = NativeClassifier(cfg, w)
for _ in range(3):
    b = nat.forward(ids, m)
assert (a - b).abs().max() < 5e-3
print("mixed ok")
PY
echo "mixed rc=$?"; tail -3 gpurun_out/sanitizer_mixed.log
