"""CPU fp32 oracle of the classifier (TEST INFRASTRUCTURE).  Same random-init weights (rounded to
the classifier's 16-bit type like the device copy), every attention call goes through the reference operator
(oracle.flash_attention -> routefast::flash_attention semantics); the rest of the network is a
plain torch fp32 restatement of paper_2603_12646_b200/classifier.py and is this build's own
construction -- the reference has no neural classifier (SURVEY.md 8(c) "parity unpinned by the
reference" for everything but the attention op)."""
import os

import numpy as np
import torch


def oracle_forward(cfg, weights, input_ids, attention_mask, O, impl="port", threads=None):
    wdt = getattr(cfg, "torch_dtype", torch.bfloat16)  # the device copy of the matrices is rounded to this type
    threads = threads or os.cpu_count() or 1
    norm_keys = {k for k in weights if k.endswith("norm") or k == "cls_b"}
    w = {k: (v.float() if k in norm_keys else v.to(wdt).float()) for k, v in weights.items()}
    B, S = input_ids.shape
    H, d, hid = cfg.heads, cfg.head_dim, cfg.hidden
    ln = lambda t, wt: torch.nn.functional.layer_norm(t, (hid,), wt, None, cfg.eps)  # noqa: E731
    pad_bias = None
    if attention_mask is not None:
        pad_bias = O.pad_bias_from_mask(attention_mask.float().numpy().reshape(B, 1, 1, S))
    x = ln(w["tok_emb"][input_ids.reshape(-1)], w["emb_norm"])
    for i in range(cfg.n_layers):
        h = ln(x, w[f"l{i}.attn_norm"]) if i > 0 else x
        qkv = (h @ w[f"l{i}.wqkv"].t()).view(B, S, 3, H, d)
        glob = cfg.is_global(i)
        theta = cfg.rope_theta_global if glob else cfg.rope_theta_local
        inv = 1.0 / (theta ** (torch.arange(0, d, 2, dtype=torch.float64) / d))
        ang = torch.arange(S, dtype=torch.float64)[:, None] * inv[None, :]
        cos, sin = ang.cos().float()[None, :, None, :], ang.sin().float()[None, :, None, :]

        def rope(t):
            t1, t2 = t[..., : d // 2], t[..., d // 2:]
            return torch.cat([t1 * cos - t2 * sin, t2 * cos + t1 * sin], dim=-1)

        q = rope(qkv[:, :, 0]).permute(0, 2, 1, 3).contiguous().numpy()
        k = rope(qkv[:, :, 1]).permute(0, 2, 1, 3).contiguous().numpy()
        v = qkv[:, :, 2].permute(0, 2, 1, 3).contiguous().numpy()
        wl, wr = (-1, -1) if glob else (cfg.local_window // 2 - 1, cfg.local_window // 2)
        o = O.flash_attention(q, k, v, 0.0, wl, wr, pad_bias, threads=threads, impl=impl)
        attn = torch.from_numpy(o).permute(0, 2, 1, 3).reshape(B * S, hid)
        x = x + attn @ w[f"l{i}.wo"].t()
        h2 = ln(x, w[f"l{i}.mlp_norm"])
        wi = h2 @ w[f"l{i}.wi"].t()
        act = torch.nn.functional.gelu(wi[:, : cfg.mlp]) * wi[:, cfg.mlp:]
        x = x + act @ w[f"l{i}.wo2"].t()
    hf = ln(x, w["final_norm"]).view(B, S, hid)[:, 0]
    t = ln(torch.nn.functional.gelu(hf @ w["head_dense"].t()), w["head_norm"])
    return (t @ w["cls_w"].t() + w["cls_b"]).numpy()
