#!/bin/bash
# compute-sanitizer over small invocations of every kernel family (developer aid): memcheck on smoke (dense +
# narrow-window + host path), on a padded batch with ragged lengths (bias + norms pre-pass, narrow-window kernel with
# two CTAs per SM, wide windows), on the projection GEMM with every epilogue, on the classifier (hosted + native
# session); racecheck and synccheck on smoke and the GEMM.  Output: gpurun_out/sanitizer_*.log
mkdir -p gpurun_out
compute-sanitizer --tool memcheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/sanitizer_memcheck_smoke.log 2>&1
echo "memcheck smoke rc=$?"; tail -2 gpurun_out/sanitizer_memcheck_smoke.log
cat > /tmp/san_mixed.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2603_12646_b200 as P
from paper_2603_12646_b200.classifier import Classifier, ClassifierConfig, NativeClassifier, init_weights, rope_tables
from paper_2603_12646_b200.gemm import gemm_nt
g = torch.Generator(device="cuda").manual_seed(0)
for (B, H, S) in ((2, 2, 1281), (1, 1, 1000), (3, 12, 2049)):
    q, k, v = [(torch.rand((B, H, S, 64), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
    mask = torch.ones(B, 1, 1, S, device="cuda")
    mask[0, ..., S - 77:] = 0
    pb = P.pad_bias_from_mask(mask)
    for spec in (P.AttentionSpec(), P.AttentionSpec(0.0, -1, -1, pb), P.AttentionSpec(0.0, 63, 64, pb), P.AttentionSpec(0.0, 63, 64),
                 P.AttentionSpec(0.0, 5, 9), P.AttentionSpec(0.0, 300, 10, pb)):
        o = P.flash_attention(q, k, v, spec)
        torch.cuda.synchronize()
        assert torch.isfinite(o.float()).all()
# projections: every epilogue, both tile widths, ragged M
for dt in (torch.bfloat16, torch.float16):
    a = torch.randn(300, 768, device="cuda").to(dt)
    w3 = (torch.randn(2304, 768, device="cuda") * 0.05).to(dt)
    w1 = (torch.randn(768, 768, device="cuda") * 0.05).to(dt)
    cos, sin = rope_tables(150, 64, 10000.0, "cuda")
    y = gemm_nt(a, w3)
    y = gemm_nt(a, w1)
    y = gemm_nt(a, w3, epilogue="rope", rope_cos=cos, rope_sin=sin, seq_len=150, head_major=True)
    y = gemm_nt(a, w3, epilogue="geglu")
    x = torch.zeros(300, 768, device="cuda")
    gemm_nt(a, w1, out=x, epilogue="residual")
    torch.cuda.synchronize()
    assert torch.isfinite(x).all() and torch.isfinite(y.float()).all()
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
compute-sanitizer --tool memcheck --error-exitcode 9 python /tmp/san_mixed.py > gpurun_out/sanitizer_memcheck_mixed.log 2>&1
echo "memcheck mixed rc=$?"; tail -3 gpurun_out/sanitizer_memcheck_mixed.log
compute-sanitizer --tool racecheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/sanitizer_racecheck_smoke.log 2>&1
echo "racecheck smoke rc=$?"; tail -2 gpurun_out/sanitizer_racecheck_smoke.log
compute-sanitizer --tool synccheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/sanitizer_synccheck_smoke.log 2>&1
echo "synccheck smoke rc=$?"; tail -2 gpurun_out/sanitizer_synccheck_smoke.log
cat > /tmp/san_gemm.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2603_12646_b200.gemm import gemm_nt
a = torch.randn(300, 768, device="cuda").to(torch.bfloat16)
w = (torch.randn(768, 768, device="cuda") * 0.05).to(torch.bfloat16)
w3 = (torch.randn(2304, 768, device="cuda") * 0.05).to(torch.bfloat16)
y = gemm_nt(a, w); y2 = gemm_nt(a, w3, epilogue="geglu")
x = torch.zeros(300, 768, device="cuda"); gemm_nt(a, w, out=x, epilogue="residual")
torch.cuda.synchronize()
print("gemm ok", float((y.float() - a.float() @ w.float().t()).abs().max()))
PY
compute-sanitizer --tool racecheck --error-exitcode 9 python /tmp/san_gemm.py > gpurun_out/sanitizer_racecheck_gemm.log 2>&1
echo "racecheck gemm rc=$?"; tail -2 gpurun_out/sanitizer_racecheck_gemm.log
compute-sanitizer --tool synccheck --error-exitcode 9 python /tmp/san_gemm.py > gpurun_out/sanitizer_synccheck_gemm.log 2>&1
echo "synccheck gemm rc=$?"; tail -2 gpurun_out/sanitizer_synccheck_gemm.log
