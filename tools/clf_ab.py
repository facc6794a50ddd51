#!/usr/bin/env python
"""Developer tool (under gpurun): the 8K classifier forward (CUDA-graph replay) with this library's own projections
(rf_gemm_nt, fused RoPE / GeGLU) against the round-1 path (library GEMMs + separate glue kernels), hosted and native."""
import json, os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_12646_b200.classifier import Classifier, ClassifierConfig, NativeClassifier, init_weights

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
res = {}
ids = None
logits = {}
for gemm in ("own", "cublas"):
    cfg = ClassifierConfig(gemm=gemm)
    w = init_weights(cfg, 7)
    clf = Classifier(cfg, w, torch.device("cuda:0"))
    if ids is None:
        ids = torch.randint(0, cfg.vocab_size, (B, S), device="cuda")
    run = clf.capture(B, S, with_mask=False)
    for _ in range(3): run(ids)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): lg = run(ids)
    e1.record(); torch.cuda.synchronize()
    res[f"hosted_{gemm}_ms"] = round(e0.elapsed_time(e1) / 10, 3)
    logits[gemm] = lg.float().cpu()
    del clf, run
    nat = NativeClassifier(cfg, w, device=0)
    ids_h = ids.cpu()
    for _ in range(3): nat.forward(ids_h)
    ms = []
    for _ in range(10):
        lgn = nat.forward(ids_h); ms.append(nat.last_forward_ms)
    res[f"native_{gemm}_ms"] = round(sorted(ms)[5], 3)
    logits["native_" + gemm] = lgn
    nat.close()
res["max_abs_logit_diff_own_vs_cublas"] = float((logits["own"] - logits["cublas"]).abs().max())
res["max_abs_logit_diff_native_own_vs_hosted_own"] = float((logits["own"] - logits["native_own"]).abs().max())
print(json.dumps(res))
