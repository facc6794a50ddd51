#!/usr/bin/env python
"""GPU bring-up ladder (developer tool, run under gpurun).

Each case runs in its own subprocess under a timeout so that a trapped kernel (bad descriptor,
barrier timeout) cannot poison the next case or hang the box.  Results go to stdout and
gpurun_out/bringup.jsonl.  The checker here is a plain torch fp32 attention on the GPU (this is
a debugging aid; the parity tests in tests/ use the oracle).

usage: python tools/bringup.py all            # run the ladder
       python tools/bringup.py case <name>    # one case in-process
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "gpurun_out")


def log(rec):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "bringup.jsonl"), "a") as f:
        f.write(json.dumps(rec) + "\n")
    print(json.dumps(rec), flush=True)


def ref_attn(q, k, v, scale, wl, wr, pad):
    import torch
    B, H, S, d = q.shape
    s = (q.float() @ k.float().transpose(-1, -2)) * scale
    i = torch.arange(S, device=q.device)[:, None]
    j = torch.arange(S, device=q.device)[None, :]
    live = torch.ones(S, S, dtype=torch.bool, device=q.device)
    if wl >= 0:
        live &= (i - j) <= wl
    if wr >= 0:
        live &= (j - i) <= wr
    live = live[None, None].expand(B, 1, S, S)
    if pad is not None:
        s = s + pad
        live = live & (pad > -30000.0)
    s = s.masked_fill(~live, float("-inf"))
    m = s.amax(-1, keepdim=True)
    m = torch.where(torch.isinf(m), torch.zeros_like(m), m)
    p = torch.exp(s - m)
    l = p.sum(-1, keepdim=True)
    o = (p @ v.float()) / torch.where(l > 0, l, torch.ones_like(l))
    return torch.where(l > 0, o, torch.zeros_like(o))


def case_probe(mode: int):
    import torch
    lib = C.CDLL(os.path.join(ROOT, "tests", "gpu_probe", "libumma_probe.so"))
    lib.umma_probe_run.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    torch.manual_seed(mode)
    KA = 64 if mode == 0 else 128
    N = 128 if mode == 0 else 64
    A = (torch.randn(128, KA, device="cuda")).to(torch.bfloat16)
    if mode == 0:
        Bm = torch.randn(128, 64, device="cuda").to(torch.bfloat16)   # [N, K]
        want = A.float() @ Bm.float().t()
    else:
        Bm = torch.randn(128, 64, device="cuda").to(torch.bfloat16)   # [K, N]
        want = A.float() @ Bm.float()
    D = torch.full((128, N), float("nan"), device="cuda", dtype=torch.float32)
    rc = lib.umma_probe_run(mode, A.data_ptr(), Bm.data_ptr(), D.data_ptr())
    err = (D - want).abs().max().item() if rc == 0 else None
    log({"case": f"probe{mode}", "rc": rc, "max_abs_err": err, "ok": rc == 0 and err is not None and err < 1e-2})
    if rc == 0 and not (err < 1e-2):
        # diagnostics: which rows/cols are wrong
        bad = ((D - want).abs() > 1e-2)
        log({"case": f"probe{mode}_diag", "bad_frac": bad.float().mean().item(),
             "bad_rows": bad.any(1).nonzero().flatten()[:16].tolist(),
             "bad_cols": bad.any(0).nonzero().flatten()[:16].tolist(),
             "D00": D[0, :8].tolist(), "want00": want[0, :8].tolist()})


def make_inputs(B, H, S, d, seed=0, dtype=None):
    import torch
    dtype = dtype or torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = (torch.rand(B, H, S, d, device="cuda", generator=g) * 2 - 1).to(dtype)
    k = (torch.rand(B, H, S, d, device="cuda", generator=g) * 2 - 1).to(dtype)
    v = (torch.rand(B, H, S, d, device="cuda", generator=g) * 2 - 1).to(dtype)
    return q, k, v


def make_pad(B, S, lens):
    import torch
    pad = torch.zeros(B, 1, 1, S, device="cuda")
    for b, n in enumerate(lens):
        pad[b, 0, 0, n:] = -65504.0
    return pad


def case_fa(name, B, H, S, wl, wr, lens, flags, kernel="tcgen05", dump=False, scale=0.0):
    import torch
    import paper_2603_12646_b200 as P
    q, k, v = make_inputs(B, H, S, 64, seed=S + B)
    pad = make_pad(B, S, lens) if lens else None
    spec = P.AttentionSpec(scale, wl, wr, pad)
    dbg = None
    if dump:
        ncta = B * H * ((S + 255) // 256)
        dbg = torch.full((ncta * 2, 128, 128), float("nan"), device="cuda")
    rec = {"case": name, "B": B, "H": H, "S": S, "wl": wl, "wr": wr, "lens": lens, "flags": flags, "kernel": kernel}
    try:
        out = P.flash_attention(q, k, v, spec, kernel=kernel, flags=flags, debug_scores=dbg)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        rec.update(ok=False, error=str(e)[:300])
        log(rec)
        return
    eff = spec.effective_scale(64)
    want = ref_attn(q, k, v, eff, wl, wr, pad)
    err = (out.float() - want).abs().max().item()
    rec.update(max_abs_err=err, ok=bool(err <= 2e-2), nan=bool(torch.isnan(out.float()).any().item()))
    if dump:
        # S tile of CTA 0: rows 0..127 x keys of its first live tile (global no-window: keys 0..127)
        s_want = q[0, 0, :128].float() @ k[0, 0, :128].float().t()
        nrow = min(128, S)
        s_err = (dbg[0, :nrow, :nrow] - s_want[:nrow, :nrow]).abs().max().item()
        rec.update(s_tile_err=s_err)
    if not rec["ok"]:
        diff = (out.float() - want).abs()
        rows_bad = (diff.amax(-1) > 2e-2)
        rec.update(bad_row_frac=rows_bad.float().mean().item(),
                   first_bad=rows_bad.nonzero()[:6].tolist(),
                   out0=out[0, 0, 0, :6].float().tolist(), want0=want[0, 0, 0, :6].tolist())
    log(rec)


def case_cross(name, B, H, S, wl, wr, lens):
    """tcgen05 vs SIMT on the same inputs at sizes too big for the S x S torch checker."""
    import torch
    import paper_2603_12646_b200 as P
    q, k, v = make_inputs(B, H, S, 64, seed=7)
    pad = make_pad(B, S, lens) if lens else None
    spec = P.AttentionSpec(0.0, wl, wr, pad)
    a = P.flash_attention(q, k, v, spec, kernel="tcgen05")
    b = P.flash_attention(q, k, v, spec, kernel="simt")
    torch.cuda.synchronize()
    err = (a.float() - b.float()).abs().max().item()
    log({"case": name, "S": S, "wl": wl, "lens": lens, "tc_vs_simt_max_abs": err, "ok": bool(err <= 2e-2)})


def case_time(name, B, H, S, wl, wr, flags, iters=20, kernel="tcgen05"):
    import torch
    import paper_2603_12646_b200 as P
    q, k, v = make_inputs(B, H, S, 64, seed=1)
    spec = P.AttentionSpec(0.0, wl, wr, None)
    out = torch.empty_like(q)
    for _ in range(3):
        P.flash_attention(q, k, v, spec, kernel=kernel, flags=flags, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        P.flash_attention(q, k, v, spec, kernel=kernel, flags=flags, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    if wl < 0:
        flops = 4.0 * B * H * S * S * 64
    else:
        flops = 4.0 * B * H * S * min(S, wl + wr + 1) * 64
    log({"case": name, "B": B, "H": H, "S": S, "wl": wl, "flags": flags, "kernel": kernel, "ms": ms,
         "tflops": flops / ms / 1e9, "gbs": 4 * B * H * S * 64 * 2 / ms / 1e6})


def case_time_graph(name, B, H, S, wl, wr, lens=None, iters=20):
    """Device time per call with the launches replayed from a CUDA graph (no host launch cost)."""
    import torch
    import paper_2603_12646_b200 as P
    q, k, v = make_inputs(B, H, S, 64, seed=1)
    pb = None
    if lens is not None:
        mask = torch.zeros(B, 1, 1, S, device="cuda")
        for b, n in enumerate(lens):
            mask[b, ..., :n] = 1
        pb = P.pad_bias_from_mask(mask)
    spec = P.AttentionSpec(0.0, wl, wr, pb)
    out = torch.empty_like(q)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for _ in range(3):
            P.flash_attention(q, k, v, spec, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            P.flash_attention(q, k, v, spec, out=out)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (5 * iters)
    log({"case": name, "B": B, "H": H, "S": S, "wl": wl, "lens": lens, "us_per_call_graph": ms * 1000,
         "gbs": 4 * B * H * S * 64 * 2 / ms / 1e6})


def case_time_strided(name, S, wl, wr, iters=10):
    """Same op on [B,H,S,d] tensors and on strided views of a packed [B,S,3,H,d] buffer (the classifier's layout)."""
    import torch
    import paper_2603_12646_b200 as P
    B, H, d = 1, 12, 64
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = (torch.rand((B, S, 3, H, d), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    views = [qkv[:, :, j].permute(0, 2, 1, 3) for j in range(3)]
    cont = [v.contiguous() for v in views]
    out_s = torch.empty((B, S, H, d), device="cuda", dtype=torch.bfloat16).permute(0, 2, 1, 3)
    out_c = torch.empty((B, H, S, d), device="cuda", dtype=torch.bfloat16)
    spec = P.AttentionSpec(0.0, wl, wr)
    res = {}
    for label, (a, o) in (("contiguous", (cont, out_c)), ("packed_qkv_views", (views, out_s))):
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            for _ in range(3):
                P.flash_attention(*a, spec, out=o)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(iters):
                P.flash_attention(*a, spec, out=o)
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        res[label + "_us"] = e0.elapsed_time(e1) / (5 * iters) * 1000
    log({"case": name, "S": S, "wl": wl, **res})


def case_clf(name, S, B=1, iters=5, padded=False):
    import torch
    from paper_2603_12646_b200.classifier import Classifier, ClassifierConfig, init_weights
    cfg = ClassifierConfig()
    dev = torch.device("cuda:0")
    model = Classifier(cfg, init_weights(cfg, 7), dev)
    ids = torch.randint(0, cfg.vocab_size, (B, S), device=dev)
    mask = None
    if padded:
        mask = torch.ones((B, S), device=dev)
        mask[:, S - S // 8:] = 0
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    for _ in range(2):
        logits = model.forward(ids, mask)
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        logits = model.forward(ids, mask)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    graph_ms = None
    try:
        run = model.capture(B, S, padded)
        for _ in range(2):
            lg = run(ids, mask)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            lg = run(ids, mask)
        e1.record()
        torch.cuda.synchronize()
        graph_ms = e0.elapsed_time(e1) / iters
        graph_diff = (lg - logits).abs().max().item()
    except Exception as e:  # noqa: BLE001
        graph_diff = repr(e)[:200]
    model.forward(ids, mask, time_layers=True)
    lm = model.last_layer_ms
    ga = [x["attention_ms"] for x in lm if x["global"]]
    la = [x["attention_ms"] for x in lm if not x["global"]]
    log({"case": name, "S": S, "B": B, "padded": padded, "ms_per_forward": ms, "ms_per_request": ms / B,
         "graph_ms_per_forward": graph_ms, "graph_vs_eager_maxdiff": graph_diff,
         "weights_MB": model.weight_bytes() / 1e6, "peak_activation_MB": (peak - base) / 1e6,
         "session_MB": peak / 1e6, "global_attn_ms_avg": sum(ga) / len(ga), "local_attn_ms_avg": sum(la) / len(la),
         "attn_ms_total": sum(ga) + sum(la), "logits": logits[0].tolist()})


CASES = {
    "probe0": lambda: case_probe(0),
    "probe1": lambda: case_probe(1),
    "probe2": lambda: case_probe(2),
    "probe3": lambda: case_probe(3),
    "simt_small": lambda: case_fa("simt_small", 1, 2, 200, -1, -1, None, 0, kernel="simt"),
    "simt_local_pad": lambda: case_fa("simt_local_pad", 2, 2, 300, 63, 64, [300, 211], 0, kernel="simt"),
    "ts_128": lambda: case_fa("ts_128", 1, 1, 128, -1, -1, None, 0, dump=True),
    "ts_256": lambda: case_fa("ts_256", 1, 1, 256, -1, -1, None, 0, dump=True),
    "ts_512": lambda: case_fa("ts_512", 1, 12, 512, -1, -1, None, 0),
    "ts_1000_ragged": lambda: case_fa("ts_1000_ragged", 2, 3, 1000, -1, -1, None, 0),
    "ts_2048": lambda: case_fa("ts_2048", 1, 4, 2048, -1, -1, None, 0),
    "ts_pad": lambda: case_fa("ts_pad", 2, 4, 512, -1, -1, [475, 300], 0),
    "ts_local": lambda: case_fa("ts_local", 1, 4, 1024, 63, 64, None, 0),
    "ts_local_pad": lambda: case_fa("ts_local_pad", 2, 4, 1000, 63, 64, [1000, 777], 0),
    "ts_onesided": lambda: case_fa("ts_onesided", 1, 2, 700, 1, 2, None, 0),
    "ts_self": lambda: case_fa("ts_self", 1, 2, 300, 0, 0, None, 0),
    "ts_aonly_pad": lambda: case_fa("ts_aonly_pad", 1, 2, 300, -1, -1, [263], 0),
    "ts_aonly_900": lambda: case_fa("ts_aonly_900", 2, 3, 900, -1, -1, None, 0),
    "ts_tiny": lambda: case_fa("ts_tiny", 1, 1, 5, -1, -1, None, 0),
    "ts_allpad": lambda: case_fa("ts_allpad", 2, 2, 256, -1, -1, [256, 0], 0),
    "cross_8k": lambda: case_cross("cross_8k", 1, 12, 8192, -1, -1, None),
    "cross_8k_local_pad": lambda: case_cross("cross_8k_local_pad", 1, 12, 8192, 63, 64, [7000]),
    "time_8k_ts": lambda: case_time("time_8k_ts", 1, 12, 8192, -1, -1, 0),
    "time_16k_ts": lambda: case_time("time_16k_ts", 1, 12, 16384, -1, -1, 0, iters=10),
    "time_32k_ts": lambda: case_time("time_32k_ts", 1, 12, 32768, -1, -1, 0, iters=5),
    "time_8k_local_ts": lambda: case_time("time_8k_local_ts", 1, 12, 8192, 63, 64, 0),
    "graph_8k_local": lambda: case_time_graph("graph_8k_local", 1, 12, 8192, 63, 64),
    "graph_8k_local_pad": lambda: case_time_graph("graph_8k_local_pad", 1, 12, 8192, 63, 64, lens=[7000]),
    "graph_32k_local": lambda: case_time_graph("graph_32k_local", 1, 12, 32768, 63, 64),
    "graph_16k_b4_local": lambda: case_time_graph("graph_16k_b4_local", 4, 12, 16384, 63, 64),
    "graph_8k_global": lambda: case_time_graph("graph_8k_global", 1, 12, 8192, -1, -1),
    "graph_16k_global": lambda: case_time_graph("graph_16k_global", 1, 12, 16384, -1, -1, iters=5),
    "graph_32k_global": lambda: case_time_graph("graph_32k_global", 1, 12, 32768, -1, -1, iters=3),
    "graph_8k_b8_global": lambda: case_time_graph("graph_8k_b8_global", 8, 12, 8192, -1, -1, iters=3),
    "graph_16k_b4_global": lambda: case_time_graph("graph_16k_b4_global", 4, 12, 16384, -1, -1, iters=3),
    "graph_4k_b16_global": lambda: case_time_graph("graph_4k_b16_global", 16, 12, 4096, -1, -1, iters=5),
    "strided_8k_global": lambda: case_time_strided("strided_8k_global", 8192, -1, -1),
    "strided_8k_local": lambda: case_time_strided("strided_8k_local", 8192, 63, 64, iters=20),
    "strided_32k_global": lambda: case_time_strided("strided_32k_global", 32768, -1, -1, iters=3),
    "graph_16k_b4_pad_global": lambda: case_time_graph("graph_16k_b4_pad_global", 4, 12, 16384, -1, -1,
                                                       lens=[16384, 9000, 12000, 8200], iters=5),
    "graph_8k_b8_pad_global": lambda: case_time_graph("graph_8k_b8_pad_global", 8, 12, 8192, -1, -1,
                                                      lens=[8192, 4100, 6000, 5000, 7777, 4500, 8000, 0], iters=5),
    "graph_8k_b8_allfull": lambda: case_time_graph("graph_8k_b8_allfull", 8, 12, 8192, -1, -1, lens=[8192] * 8, iters=5),
    "graph_8k_b8_allhalf": lambda: case_time_graph("graph_8k_b8_allhalf", 8, 12, 8192, -1, -1, lens=[4096] * 8, iters=5),
    "graph_8k_b2_full_bias": lambda: case_time_graph("graph_8k_b2_full_bias", 2, 12, 8192, -1, -1, lens=[8192, 8192], iters=5),
    "graph_8k_b3_mixed": lambda: case_time_graph("graph_8k_b3_mixed", 3, 12, 8192, -1, -1, lens=[8192, 5000, 6500], iters=5),
    "graph_8k_b2_global": lambda: case_time_graph("graph_8k_b2_global", 2, 12, 8192, -1, -1, iters=5),
    "graph_8k_b2_skew": lambda: case_time_graph("graph_8k_b2_skew", 2, 12, 8192, -1, -1, lens=[8192, 4096], iters=5),
    "cross_4k_b4_pad": lambda: case_cross("cross_4k_b4_pad", 4, 12, 4096, -1, -1, [4096, 2100, 3000, 0]),
    "graph_8k_b8_skew_nozero": lambda: case_time_graph("graph_8k_b8_skew_nozero", 8, 12, 8192, -1, -1,
                                                       lens=[8192, 4100, 6000, 5000, 7777, 4500, 8000, 8192], iters=5),
    "graph_8k_b8_onezero": lambda: case_time_graph("graph_8k_b8_onezero", 8, 12, 8192, -1, -1, lens=[8192] * 7 + [0], iters=5),
    "graph_8k_b8_skew_aligned": lambda: case_time_graph("graph_8k_b8_skew_aligned", 8, 12, 8192, -1, -1,
                                                        lens=[8192, 4096, 6016, 4992, 7808, 4480, 8064, 8192], iters=5),
    "graph_8k_pad_global": lambda: case_time_graph("graph_8k_pad_global", 1, 12, 8192, -1, -1, lens=[7168], iters=10),
    "clf_8k": lambda: case_clf("clf_8k", 8192),
    "clf_8k_pad": lambda: case_clf("clf_8k_pad", 8192, padded=True),
    "clf_16k_b4": lambda: case_clf("clf_16k_b4", 16384, B=4, iters=3),
    "clf_32k": lambda: case_clf("clf_32k", 32768, iters=3),
    "time_8k_simt": lambda: case_time("time_8k_simt", 1, 12, 8192, -1, -1, 0, iters=3, kernel="simt"),
}


def main():
    if len(sys.argv) >= 3 and sys.argv[1] == "case":
        CASES[sys.argv[2]]()
        return
    names = list(CASES) if len(sys.argv) < 3 or not sys.argv[2] else sys.argv[2].split(",")
    for name in names:
        t = time.time()
        try:
            res = subprocess.run([sys.executable, os.path.abspath(__file__), "case", name], timeout=240,
                                 capture_output=True, text=True)
            tail = (res.stdout + res.stderr)[-1500:]
            if res.returncode != 0:
                log({"case": name, "ok": False, "returncode": res.returncode, "tail": tail})
            else:
                sys.stdout.write(res.stdout)
        except subprocess.TimeoutExpired:
            log({"case": name, "ok": False, "error": "timeout"})
        print(f"# {name}: {time.time() - t:.1f}s", flush=True)


if __name__ == "__main__":
    main()
