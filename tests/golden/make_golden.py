#!/usr/bin/env python
"""Generates tests/golden/attention_golden.npz from the UNMODIFIED reference
(oracle/_ref/libref_attn.so = /root/reference/proj/core/src/{attention,tensor}.cpp behind
oracle/ref_shim.cpp).  Run in the dev container only (needs /root/reference):

    python tests/golden/make_golden.py

Inputs are Tensor::random streams (mt19937_64, tensor.cpp:35-45) identified by (seed, shape),
so only outputs and a few input samples are stored.  Cases follow the reference's own
tests/benchmarks and SPEC.md's known-answer examples (cited per case).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

R = "reference"
out = {}

# --- RNG stream heads (tensor.cpp:35-45) ---
for seed in (5, 7, 11, 42):
    out[f"rng_seed{seed}_head"] = O.random_tensors(seed, (32,), 1, impl=R)[0]
out["rng_seed11_f16_head"] = O.random_tensors(11, (32,), 1, as_f16=True, impl=R)[0]

# --- binary16 round trip (tensor.cpp:47-98) ---
probe = np.array([0.0, -0.0, 1.0, -1.0, 65504.0, -65504.0, 65520.0, 65519.9, 1e-8, 5.9604645e-8, 2.9802322e-8,
                  6.1035156e-5, 6.0975552e-5, 0.1, 0.333333343, 1.0009765625, 1.00048828125, 1.0014648437,
                  3.14159274, -2.71828175, 1e5, -1e5, 123.456, 2047.5, 2048.5, 4097.0], dtype=np.float32)
out["f16_probe_in"] = probe
out["f16_probe_out"] = O.quantize_f16(probe, impl=R)
out["f16_probe_bits"] = np.array([O.float_to_half(float(x), impl=R) for x in probe], dtype=np.uint16)

# --- bench_attention.cpp:16-57 configs: [1,2,S,64], seed 11, scale 1/8 ---
for S in (128, 512):
    q, k, v = O.random_tensors(11, (1, 2, S, 64), 3, impl=R)
    out[f"bench_global_S{S}"] = O.flash_attention(q, k, v, 0.125, impl=R)
q, k, v = O.random_tensors(11, (1, 2, 512, 64), 3, impl=R)
out["bench_local_S512"] = O.flash_attention(q, k, v, 0.125, 63, 64, impl=R)
q, k, v = O.random_tensors(11, (1, 2, 128, 64), 3, impl=R)
out["bench_sdpa_S128"] = O.sdpa(q, k, v, None, 0.125, impl=R)

# --- rewrite_test.cpp:239-263 inputs (seed 7, [1,2,96,32], Q=K=V=hidden, 7 padded keys, local 63/64,
#     scale attr 1/sqrt(32) copied from the matched constant) ---
hidden = O.random_tensors(7, (1, 2, 96, 32), 1, impl=R)[0]
mask = np.ones((1, 1, 1, 96), np.float32)
mask[..., -7:] = 0
pb = O.pad_bias_from_mask(mask)
out["rewrite_pad_bias"] = pb
out["rewrite_local_S96_d32"] = O.flash_attention(hidden, hidden, hidden, 1.0 / np.sqrt(32.0), 63, 64, pb, impl=R)
m2d = O.window_to_mask2d(96, 63, 64, pb, impl=R)
out["rewrite_local_S96_d32_sdpa"] = O.sdpa(hidden, hidden, hidden, m2d, 1.0 / np.sqrt(32.0), impl=R)

# --- rewrite_test.cpp:210-237: window_to_mask2d(96, 63, 64, pad 9) ---
mask9 = np.ones((1, 1, 1, 96), np.float32)
mask9[..., -9:] = 0
out["mask2d_S96_pad9"] = O.window_to_mask2d(96, 63, 64, O.pad_bias_from_mask(mask9), impl=R)

# --- SPEC.md:514-517 mask examples ---
out["mask2d_S3_w11"] = O.window_to_mask2d(3, 1, 1, None, impl=R)
pb4 = np.zeros((1, 1, 1, 4), np.float32)
pb4[..., 3] = -65504.0
out["mask2d_S4_padlast"] = O.window_to_mask2d(4, -1, -1, pb4, impl=R)
out["mask2d_S128_w6364"] = O.window_to_mask2d(128, 63, 64, None, impl=R)

# --- config 1 slice: B=1,H=2,S=512,d=64, seed 11, inputs rounded to bf16 first (parity convention) ---
q, k, v = [O.round_bf16(t) for t in O.random_tensors(11, (1, 2, 512, 64), 3, impl=R)]
out["cfg1_global_bf16in"] = O.flash_attention(q, k, v, 0.0, impl=R)
lens = 475
pbc = np.zeros((1, 1, 1, 512), np.float32)
pbc[..., lens:] = -65504.0
out["cfg1_global_pad475_bf16in"] = O.flash_attention(q, k, v, 0.0, -1, -1, pbc, impl=R)
out["cfg1_local_pad475_bf16in"] = O.flash_attention(q, k, v, 0.0, 63, 64, pbc, impl=R)

# --- ragged / tiny / corner cases (S in 1..8, 37, 100; windows (0,0),(1,2)) ---
for S in (1, 2, 3, 5, 8, 37, 100):
    q, k, v = O.random_tensors(100 + S, (2, 2, S, 32), 3, impl=R)
    pbr = np.zeros((2, 1, 1, S), np.float32)
    if S > 2:
        pbr[1, 0, 0, S - max(1, S // 3):] = -65504.0
    for (wl, wr) in ((-1, -1), (0, 0), (1, 2), (63, 64)):
        out[f"grid_S{S}_w{wl}_{wr}"] = O.flash_attention(q, k, v, 0.0, wl, wr, pbr, impl=R)
# additive (non-masking) bias and a fully masked batch row (attention.cpp:169,175,204-207)
q, k, v = O.random_tensors(77, (2, 1, 40, 32), 3, impl=R)
pba = np.zeros((2, 1, 1, 40), np.float32)
pba[0, 0, 0, :] = np.linspace(-3, 2, 40, dtype=np.float32)
pba[1, 0, 0, :] = -65504.0
out["additive_bias_and_dead_row"] = O.flash_attention(q, k, v, 0.3, -1, 5, pba, impl=R)
out["additive_bias_input"] = pba

# --- memory model (attention.cpp:244-252) ---
out["mem_mask_1_12_8192_2"] = np.array([O.mask_memory_bytes(1, 12, 8192, 2, impl=R)], dtype=np.uint64)
out["mem_mask_1_12_16384_2"] = np.array([O.mask_memory_bytes(1, 12, 16384, 2, impl=R)], dtype=np.uint64)
out["mem_fa_1_12_8192_64_64_2"] = np.array([O.fa_memory_bytes(1, 12, 8192, 64, 64, 2, impl=R)], dtype=np.uint64)

path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "attention_golden.npz")
np.savez_compressed(path, **out)
print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")
