"""GPU tests of the graph executor (the caller of the FusedFlashAttention operator): interpret() on
the B200 against the reference interpreter's committed outputs (tests/golden/graph_golden.npz,
generated from the unmodified reference by tests/golden/make_graph_golden.py), and
verify-rewrite -- original vs rewritten graph -- on the device at sizes the CPU reference cannot reach.

Tolerances.  Un-rewritten graph: every op is an f32 CUDA kernel where the reference computes in
f64 (interpreter.cpp:97-103,131-140): max-abs <= 1e-4.  Rewritten graph: FusedFlashAttention
runs Q/K/V in bf16 on the tensor cores (or the f32-accumulating SIMT kernel for head_dim 32/128):
max-abs <= 2e-2, the attention tolerance of BASELINE.json."""
import json
import os

import numpy as np
import pytest

import graph_fixtures as F
from paper_2603_12646_b200 import RewriteOptions, ShapeMismatch
from paper_2603_12646_b200 import graph as G

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(ROOT, "tests", "golden", "graph_golden.json")) as f:
        meta = json.load(f)
    with np.load(os.path.join(ROOT, "tests", "golden", "graph_golden.npz")) as z:
        arrays = {k: z[k] for k in z.files}
    return meta, arrays


def make_inputs(kw, padded, seed):  # same draw as tests/golden/make_graph_golden.py
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


def test_interpret_matches_reference_interpreter(gold):
    meta, arrays = gold
    for name, c in meta.items():
        if name.startswith("_"):
            continue
        fx = F.build_attention_fixture(**c["fixture"])
        ins = make_inputs(c["fixture"], c["padded"], c["seed"])
        out_name = json.loads(fx)["outputs"][0]
        st = G.InterpretStats()
        got = G.interpret(fx, ins, stats=st)[out_name]
        want = arrays[f"{name}/original"]
        assert got.shape == want.shape
        assert np.abs(got - want).max() <= 1e-4, (name, float(np.abs(got - want).max()))
        B, H, S = c["fixture"].get("batch", 1), c["fixture"].get("heads", 2), c["fixture"]["seq"]
        assert st.largest_tensor_bytes == max(B * H * S * S * 4, want.size * 4)   # the materialised score tensor
        # rewritten graph: the reference's rewrite AND ours (identical, test_graph_cpu) through the fused op
        rew = json.dumps(c["rewritten"])
        st2 = G.InterpretStats()
        got2 = G.interpret(rew, ins, stats=st2)[out_name]
        want2 = arrays[f"{name}/rewritten"]
        assert np.abs(got2 - want2).max() <= 2e-2, (name, float(np.abs(got2 - want2).max()))
        assert st2.largest_tensor_bytes == want.size * 4               # nothing larger than [B,H,S,d] exists


def test_semantic_preservation_single_layer_on_device(gold):
    """Rewrite.SemanticPreservationSingleLayer (rewrite_test.cpp:239-263) with both graphs on the GPU."""
    meta, _ = gold
    c = meta["semantic_preservation"]
    fx = F.build_attention_fixture(**c["fixture"])
    rew = G.rewrite(fx, RewriteOptions(32, 128))
    ins = make_inputs(c["fixture"], 7, 7)
    a = G.interpret(fx, ins)["layer0/out"]
    b = G.interpret(rew, ins)["layer0/out"]
    assert np.abs(a - b).max() <= 2e-2


def test_window_mask_matches_original_mask_tensor():
    """Rewrite.WindowMaskMatchesOriginalMaskTensor (rewrite_test.cpp:210-237): the 2-D bias the original
    graph builds with Expand/Mul/Where on the device equals, bit for bit, the mask implied by
    (window 63/64, pad bias) -- i.e. what the fused operator applies."""
    S = 96
    fx = json.loads(F.build_attention_fixture(layers="l", seq=S, head_dim=32))
    fx["outputs"].append("layer0/mask/bias2d")
    rng = np.random.default_rng(5)
    hidden = rng.uniform(-1, 1, (1, 2, S, 32)).astype(np.float32)
    mask = np.ones((1, 1, 1, S), np.float32)
    mask[..., -9:] = 0
    got = G.interpret(json.dumps(fx), {"hidden": hidden, "attention_mask": mask})["layer0/mask/bias2d"]
    i, j = np.arange(S)[:, None], np.arange(S)[None, :]
    live = (i - j <= 63) & (j - i <= 64) & (mask[0, 0, 0][None, :] > 0)
    want = np.where(live, np.float32(0), np.float32(-65504.0))[None, None]
    assert got.shape == (1, 1, S, S) and np.array_equal(got, want)


def test_pad_bias_chain_is_bit_exact_on_device():
    """The shared chain Cast_f16(-65504 * (1 - mask)) the rewriter installs (rewrite.cpp:303-318),
    executed node by node on the GPU, gives exactly {-0.0, -65504}."""
    fx = F.build_attention_fixture(layers="g", seq=32)
    rew = json.loads(G.rewrite(fx, RewriteOptions(32, 128)))
    rew["outputs"].append("pad_bias")
    mask = np.ones((1, 1, 1, 32), np.float32)
    mask[..., -5:] = 0
    out = G.interpret(json.dumps(rew), {"hidden": np.zeros((1, 2, 32, 32), np.float32), "attention_mask": mask})
    pb = out["pad_bias"]
    assert np.array_equal(pb[..., :27], np.zeros((1, 1, 1, 27), np.float32)) and np.all(np.signbit(pb[..., :27]))
    assert np.array_equal(pb[..., 27:], np.full((1, 1, 1, 5), -65504.0, np.float32))


@pytest.mark.parametrize("kw", [dict(batch=1, heads=4, seq=1024, head_dim=64, layers="lgl"),
                                dict(batch=2, heads=2, seq=513, head_dim=64, local_window=64, layers="lg"),
                                dict(batch=1, heads=2, seq=300, head_dim=128, layers="gl"),
                                dict(batch=1, heads=12, seq=2048, head_dim=64, layers="g")])
def test_verify_rewrite_on_device(kw):
    """`verify-rewrite` (proj/tools/main.cpp:106-149) with both graphs on the B200, padded masks as the
    CLI draws them; stacked layers feed each other, so the bound covers error growth through the stack."""
    fx = F.build_attention_fixture(**kw)
    rew = G.rewrite(fx, RewriteOptions(kw["head_dim"], kw.get("local_window", 128)))
    ok, report = G.verify_rewrite(fx, rew, trials=2, tol=2e-2, seed=42)
    assert ok, report
    B, H, S, d = kw["batch"], kw["heads"], kw["seq"], kw["head_dim"]
    assert report[0]["original"]["largest_tensor_bytes"] == B * H * S * S * 4
    assert report[0]["rewritten"]["largest_tensor_bytes"] == B * H * S * d * 4
    assert report[0]["rewritten"]["peak_device_bytes"] < report[0]["original"]["peak_device_bytes"]


def test_every_op_kind_against_numpy():
    """All 11 ops (graph.hpp:33-45) in one hand-written graph, checked against numpy on the host."""
    g = {"inputs": [{"name": "a", "shape": [2, 3, 4], "dtype": "f32"}, {"name": "b", "shape": [4, 5], "dtype": "f32"},
                    {"name": "c", "shape": [1, 3, 1], "dtype": "f32"}],
         "initializers": [{"name": "half", "shape": [1], "dtype": "f16", "data": [0.1]}],
         "outputs": ["y_mm", "y_sm", "y_where", "y_cast", "y_exp", "y_tr", "y_const", "y_sub"],
         "nodes": [
             {"name": "mm", "op": "MatMul", "inputs": ["a", "b"], "outputs": ["y_mm"]},
             {"name": "add", "op": "Add", "inputs": ["a", "c"], "outputs": ["t_add"]},
             {"name": "sm", "op": "Softmax", "inputs": ["t_add"], "outputs": ["y_sm"], "attrs": {"axis": 1}},
             {"name": "wh", "op": "Where", "inputs": ["c", "a", "half"], "outputs": ["y_where"]},
             {"name": "mul", "op": "Mul", "inputs": ["a", "half"], "outputs": ["t_mul"]},
             {"name": "cast", "op": "Cast", "inputs": ["t_mul"], "outputs": ["y_cast"], "attrs": {"to": "f16"}},
             {"name": "exp", "op": "Expand", "inputs": ["c"], "outputs": ["y_exp"], "attrs": {"shape": [2, 3, 2]}},
             {"name": "tr", "op": "Transpose", "inputs": ["a"], "outputs": ["y_tr"], "attrs": {"perm": [2, 0, 1]}},
             {"name": "k", "op": "Constant", "inputs": [], "outputs": ["y_const"], "attrs": {"shape": [2], "value": [1.5, -2.0]}},
             {"name": "k2", "op": "Constant", "inputs": [], "outputs": ["t_s"], "attrs": {"shape": [1], "scalar": 3.0}},
             {"name": "sub", "op": "Sub", "inputs": ["a", "t_s"], "outputs": ["y_sub"]}]}
    rng = np.random.default_rng(3)
    a = rng.standard_normal((2, 3, 4)).astype(np.float32)
    b = rng.standard_normal((4, 5)).astype(np.float32)
    c = np.array([1.0, 0.0, 2.0], np.float32).reshape(1, 3, 1)
    out = G.interpret(json.dumps(g), {"a": a, "b": b, "c": c})
    half = np.float32(np.float16(0.1))
    assert np.allclose(out["y_mm"], a @ b, atol=1e-5)
    e = np.exp((a + c) - (a + c).max(1, keepdims=True))
    assert np.allclose(out["y_sm"], e / e.sum(1, keepdims=True), atol=1e-6)
    assert np.array_equal(out["y_where"], np.where(c != 0, a, half))
    assert np.array_equal(out["y_cast"], (a * half).astype(np.float16).astype(np.float32))
    assert np.array_equal(out["y_exp"], np.broadcast_to(c, (2, 3, 2)))
    assert np.array_equal(out["y_tr"], a.transpose(2, 0, 1))
    assert np.array_equal(out["y_const"], np.array([1.5, -2.0], np.float32))
    assert np.array_equal(out["y_sub"], a - np.float32(3.0))


def test_interpret_errors_name_the_node():
    fx = F.build_attention_fixture(layers="g", seq=16)
    hidden = np.zeros((1, 2, 16, 32), np.float32)
    with pytest.raises(ShapeMismatch, match="graph input 'attention_mask' is not bound"):
        G.interpret(fx, {"hidden": hidden})
    with pytest.raises(ShapeMismatch, match="graph input 'hidden' has wrong shape"):
        G.interpret(fx, {"hidden": hidden[:, :1], "attention_mask": np.ones((1, 1, 1, 16), np.float32)})
    g = {"inputs": [{"name": "a", "shape": [2, 3], "dtype": "f32"}, {"name": "b", "shape": [4, 5], "dtype": "f32"}],
         "outputs": ["y"], "nodes": [{"name": "bad_mm", "op": "MatMul", "inputs": ["a", "b"], "outputs": ["y"]}]}
    with pytest.raises(ShapeMismatch, match="node 'bad_mm': MatMul inner dims differ"):
        G.interpret(json.dumps(g), {"a": np.zeros((2, 3), np.float32), "b": np.zeros((4, 5), np.float32)})
    g["nodes"] = [{"name": "k", "op": "Constant", "inputs": [], "outputs": ["y"]}]
    with pytest.raises(G.UnsupportedOp, match="Constant needs shape\\+value or scalar"):
        G.interpret(json.dumps(g), {"a": np.zeros((2, 3), np.float32), "b": np.zeros((4, 5), np.float32)})
    # FusedFlashAttention with a wrong-shaped bias: the operator's own check (attention.cpp:111-116)
    g = {"inputs": [{"name": "q", "shape": [1, 2, 8, 64], "dtype": "f32"}, {"name": "pb", "shape": [1, 1, 8], "dtype": "f32"}],
         "outputs": ["y"], "nodes": [{"name": "fa", "op": "FusedFlashAttention", "inputs": ["q", "q", "q", "pb"], "outputs": ["y"]}]}
    with pytest.raises(ShapeMismatch, match="pad_bias must be \\[B,1,1,S\\]"):
        G.interpret(json.dumps(g), {"q": np.zeros((1, 2, 8, 64), np.float32), "pb": np.zeros((1, 1, 8), np.float32)})


def test_cpp_graph_api_on_device():
    """tests/cpp/graph_test.cpp: original vs rewritten graph through the C++ interpret() on the GPU."""
    import subprocess
    from test_graph_cpu import _build_cpp_graph_test
    res = subprocess.run([_build_cpp_graph_test()], capture_output=True, text=True, timeout=600)
    print(res.stdout[-2000:], res.stderr[-2000:])
    assert res.returncode == 0 and "all checks passed" in res.stdout
