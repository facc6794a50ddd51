#!/usr/bin/env python
"""Generates tests/golden/graph_golden.json + graph_golden.npz from the UNMODIFIED reference graph
sources (oracle/_ref/libref_graph.so; needs /root/reference, so it runs in the dev container only).

For every case: the reference's normalised graph, its rewrite, pattern matches, shapes, topological
order (as canonical JSON / digests) and the reference interpreter's outputs of the original and of
the rewritten graph on seeded inputs.  tests/test_graph_cpu.py and tests/test_gpu_graph.py compare
the graph layer of librf_fa.so against these on machines without the reference.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import graph_fixtures as F  # noqa: E402
from oracle import graph_ref as R  # noqa: E402

CASES = {
    # name: (fixture kwargs, rewrite head_dim/local_window, padded tail keys, seed)
    "global_1": (dict(batch=1, heads=2, seq=16, head_dim=32, layers="g"), 0, 11),
    "local_global_4": (dict(batch=1, heads=2, seq=24, head_dim=32, local_window=8, layers="llgl"), 3, 12),
    "pre_transposed": (dict(batch=1, heads=2, seq=16, head_dim=32, layers="g", pre_transposed_k=True), 2, 13),
    # Rewrite.SemanticPreservationSingleLayer (rewrite_test.cpp:239-263): local, S=96, d=32, 7 padded keys
    "semantic_preservation": (dict(batch=1, heads=2, seq=96, head_dim=32, local_window=128, layers="l"), 7, 7),
    "two_batches_d64": (dict(batch=2, heads=2, seq=40, head_dim=64, local_window=16, layers="lg"), 5, 14),
}


def digest(text):
    return hashlib.sha256(F.canon(text).encode()).hexdigest()


def make_inputs(kw, padded, seed):
    rng = np.random.default_rng(seed)
    B, H, S, d = kw.get("batch", 1), kw.get("heads", 2), kw["seq"], kw["head_dim"]
    ins = {"hidden": rng.uniform(-1, 1, (B, H, S, d)).astype(np.float32)}
    mask = np.ones((B, 1, 1, S), np.float32)
    if padded:
        mask[-1, 0, 0, S - padded:] = 0.0
    ins["attention_mask"] = mask
    if kw.get("pre_transposed_k"):
        ins["key_t"] = np.ascontiguousarray(ins["hidden"].transpose(0, 1, 3, 2))
    return ins


def main():
    meta, arrays = {}, {}
    for name, (kw, padded, seed) in CASES.items():
        fx = F.build_attention_fixture(**kw)
        assert F.canon(fx) == F.canon(R.fixture(**kw)), name
        hd, lw = kw["head_dim"], kw.get("local_window", 128)
        rewritten = R.rewrite(fx, hd, lw)
        entry = {"fixture": kw, "padded": padded, "seed": seed, "fixture_sha256": digest(fx),
                 "rewritten": json.loads(rewritten), "patterns": R.find_patterns(fx),
                 "topological_order": R.topological_order(fx), "rewritten_shapes": R.infer_shapes(rewritten),
                 "rewritten_twice_sha256": digest(R.rewrite(rewritten, hd, lw)), "rewritten_sha256": digest(rewritten)}
        if kw["seq"] <= 24:
            entry["shapes"] = R.infer_shapes(fx)
        ins = make_inputs(kw, padded, seed)
        out_name = json.loads(fx)["outputs"][0]
        arrays[f"{name}/original"] = R.interpret(fx, ins, out_name)
        arrays[f"{name}/rewritten"] = R.interpret(rewritten, ins, out_name)
        entry["ref_original_vs_rewritten_max_abs"] = float(np.abs(arrays[f"{name}/original"] - arrays[f"{name}/rewritten"]).max())
        meta[name] = entry
    # hand-written graphs of the reference's graph_test.cpp / rewrite_test.cpp
    meta["_dce_case"] = {"graph": {
        "inputs": [{"name": "x", "shape": [2], "dtype": "f32"}], "outputs": ["y"],
        "nodes": [{"name": "keep", "op": "Mul", "inputs": ["x", "x"], "outputs": ["y"]},
                  {"name": "dead1", "op": "Mul", "inputs": ["x", "x"], "outputs": ["d1"]},
                  {"name": "dead2", "op": "Mul", "inputs": ["d1", "d1"], "outputs": ["d2"]}]}}
    meta["_dce_case"]["dce"] = json.loads(R.dce(json.dumps(meta["_dce_case"]["graph"])))
    with open(os.path.join(HERE, "graph_golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "graph_golden.npz"), **arrays)
    print("wrote", len(meta), "cases;", {k: v.shape for k, v in arrays.items()})
    print({k: v["ref_original_vs_rewritten_max_abs"] for k, v in meta.items() if not k.startswith("_")})


if __name__ == "__main__":
    main()
