"""Test-side builder of the stacked self-attention graphs the reference's tests run on
(role of proj/tests/support/graph_fixtures.cpp:16-114, which does not travel to the GPU box):

  layer l:  Mul(h, 1/sqrt(d)) -> MatMul(., Transpose(h)) -> Add(., mask_l) -> Softmax -> MatMul(., h)
  mask_l:   Expand(attention_mask -> [B,1,S,S]) [* local_window_pattern] -> Where_1|Where_2(., 0, -65504)

tests/test_graph_cpu.py pins this builder against the reference's own generator (same graph after
JSON canonicalisation) whenever oracle/_ref is available, and against a committed digest otherwise.
"""
import json
import math


def build_attention_fixture(batch=1, heads=2, seq=64, head_dim=32, local_window=128, layers="g",
                            pre_transposed_k=False) -> str:
    B, H, S, d = batch, heads, seq, head_dim
    g = {"inputs": [{"name": "hidden", "shape": [B, H, S, d], "dtype": "f32"},
                    {"name": "attention_mask", "shape": [B, 1, 1, S], "dtype": "f32"}],
         "outputs": [], "nodes": [], "initializers": []}
    if pre_transposed_k:
        g["inputs"].append({"name": "key_t", "shape": [B, H, d, S], "dtype": "f32"})
    g["initializers"] += [
        {"name": "attn_scale", "shape": [1], "dtype": "f32", "data": [1.0 / math.sqrt(float(d))]},
        {"name": "mask_zero", "shape": [1], "dtype": "f32", "data": [0.0]},
        {"name": "mask_neg", "shape": [1], "dtype": "f32", "data": [-65504.0]},
    ]
    if "l" in layers:
        wl, wr = local_window // 2 - 1, local_window // 2
        pat = [1.0 if (i - j <= wl and j - i <= wr) else 0.0 for i in range(S) for j in range(S)]
        g["initializers"].append({"name": "local_window_pattern", "shape": [1, 1, S, S], "dtype": "f32", "data": pat})

    def node(name, op, inputs, outputs, attrs=None):
        n = {"name": name, "op": op, "inputs": inputs, "outputs": outputs}
        if attrs:
            n["attrs"] = attrs
        g["nodes"].append(n)

    hidden = "hidden"
    for l, kind in enumerate(layers):
        p = f"layer{l}"
        node(f"{p}/mask/Expand", "Expand", ["attention_mask"], [f"{p}/mask/expanded"], {"shape": [B, 1, S, S]})
        cond = f"{p}/mask/expanded"
        if kind == "l":
            node(f"{p}/mask/window_and", "Mul", [cond, "local_window_pattern"], [f"{p}/mask/window_cond"])
            cond = f"{p}/mask/window_cond"
        tag = "Where_1" if kind == "l" else "Where_2"
        node(f"{p}/mask/{tag}", "Where", [cond, "mask_zero", "mask_neg"], [f"{p}/mask/bias2d"])
        node(f"{p}/q_scale", "Mul", [hidden, "attn_scale"], [f"{p}/q_scaled"])
        if pre_transposed_k:
            k_t = "key_t"
        else:
            k_t = f"{p}/k_t"
            node(f"{p}/k_transpose", "Transpose", [hidden], [k_t], {"perm": [0, 1, 3, 2]})
        node(f"{p}/qk_matmul", "MatMul", [f"{p}/q_scaled", k_t], [f"{p}/scores"])
        node(f"{p}/mask_add", "Add", [f"{p}/scores", f"{p}/mask/bias2d"], [f"{p}/scores_masked"])
        node(f"{p}/softmax", "Softmax", [f"{p}/scores_masked"], [f"{p}/attn"], {"axis": -1})
        node(f"{p}/av_matmul", "MatMul", [f"{p}/attn", hidden], [f"{p}/out"])
        hidden = f"{p}/out"
    g["outputs"].append(hidden)
    return json.dumps(g)


def canon(text: str) -> str:
    """Canonical text of a graph JSON (format-independent comparison)."""
    return json.dumps(json.loads(text), indent=2)
