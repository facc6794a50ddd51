"""CPU tests of the graph layer (IR, SDPA -> FusedFlashAttention rewriter, dce) through the C ABI of
include/rf_graph.h: against the committed golden outputs of the reference (tests/golden/graph_golden.*),
against the live reference build where oracle/_ref/libref_graph.so exists, and the cases of the
reference's own graph_test.cpp / rewrite_test.cpp re-stated through this API.  No GPU needed: the
rewriter is host logic; the executor is covered by tests/test_gpu_graph.py."""
import hashlib
import json
import math
import os
import struct

import numpy as np
import pytest

import graph_fixtures as F
from paper_2603_12646_b200 import RewriteOptions, UnsupportedHeadDim, capi
from paper_2603_12646_b200 import graph as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def golden_graphs():
    with open(os.path.join(ROOT, "tests", "golden", "graph_golden.json")) as f:
        return json.load(f)


def sha(text):
    return hashlib.sha256(F.canon(text).encode()).hexdigest()


def cases(golden_graphs):
    return {k: v for k, v in golden_graphs.items() if not k.startswith("_")}


# ---------------------------------------------------------------------------------------------
# golden parity (reference outputs committed by tests/golden/make_graph_golden.py)
# ---------------------------------------------------------------------------------------------
def test_fixture_builder_matches_committed_digest(golden_graphs):
    for name, c in cases(golden_graphs).items():
        assert sha(F.build_attention_fixture(**c["fixture"])) == c["fixture_sha256"], name


def test_rewrite_equals_reference_rewrite(golden_graphs):
    for name, c in cases(golden_graphs).items():
        fx = F.build_attention_fixture(**c["fixture"])
        opts = RewriteOptions(c["fixture"]["head_dim"], c["fixture"].get("local_window", 128))
        out = G.rewrite(fx, opts)
        assert json.loads(out) == c["rewritten"], name
        assert sha(out) == c["rewritten_sha256"], name
        assert sha(G.rewrite(out, opts)) == c["rewritten_twice_sha256"] == c["rewritten_sha256"], name  # idempotent
        assert G.find_sdpa_patterns(fx) == c["patterns"], name
        assert G.topological_order(fx) == c["topological_order"], name
        assert G.infer_shapes(out) == c["rewritten_shapes"], name
        if "shapes" in c:
            assert G.infer_shapes(fx) == c["shapes"], name


def test_dce_golden(golden_graphs):
    c = golden_graphs["_dce_case"]
    out = json.loads(G.dce(json.dumps(c["graph"])))
    assert out == c["dce"]
    assert [n["name"] for n in out["nodes"]] == ["keep"]          # Dce.RemovesTransitively (rewrite_test.cpp:184-199)


# ---------------------------------------------------------------------------------------------
# live reference (this container only)
# ---------------------------------------------------------------------------------------------
def _ref():
    from oracle import graph_ref as R
    if not R.available():
        pytest.skip("oracle/_ref/libref_graph.so not built (no /root/reference on this machine)")
    return R


@pytest.mark.parametrize("kw", [
    dict(), dict(layers="llgl", seq=32, local_window=16), dict(layers="g", pre_transposed_k=True),
    dict(layers="lg", seq=128, head_dim=64), dict(batch=2, heads=3, seq=50, layers="lgl", local_window=4),
    dict(layers="ggg", seq=8, head_dim=128)])
def test_live_reference_agreement(kw):
    R = _ref()
    fx = R.fixture(**kw)
    assert F.canon(F.build_attention_fixture(**kw)) == F.canon(fx)
    hd, lw = kw.get("head_dim", 32), kw.get("local_window", 128)
    assert F.canon(G.normalize(fx)) == F.canon(R.normalize(fx))
    mine, theirs = G.rewrite(fx, RewriteOptions(hd, lw)), R.rewrite(fx, hd, lw)
    assert F.canon(mine) == F.canon(theirs)
    assert G.find_sdpa_patterns(fx) == R.find_patterns(fx)
    assert G.infer_shapes(fx) == R.infer_shapes(fx)
    assert G.infer_shapes(mine) == R.infer_shapes(theirs)
    assert G.topological_order(mine) == R.topological_order(theirs)
    assert F.canon(G.dce(fx)) == F.canon(R.dce(fx))


BAD_GRAPHS = [
    '{"inputs": []',                                                                      # does not parse
    '[1, 2]',                                                                             # not an object
    '{"inputs": [], "outputs": [], "nodes": [{"name": "n", "op": "Conv", "inputs": [], "outputs": ["y"]}]}',
    '{"inputs": [{"name": "x", "shape": [2], "dtype": "f64"}], "outputs": [], "nodes": []}',
    '{"inputs": [{"name": "x", "shape": [2.5], "dtype": "f32"}], "outputs": [], "nodes": []}',
    '{"outputs": [], "nodes": []}',                                                       # missing field
    '{"inputs": [], "outputs": ["y"], "nodes": []}',                                      # output not produced
    '{"inputs": [{"name": "x", "shape": [2], "dtype": "f32"}], "outputs": ["x"], "nodes": '
    '[{"name": "a", "op": "Mul", "inputs": ["x", "x"], "outputs": ["x"]}]}',              # two producers
    '{"inputs": [{"name": "x", "shape": [2], "dtype": "f32"}], "outputs": ["y"], "nodes": '
    '[{"name": "a", "op": "Mul", "inputs": ["x", "q"], "outputs": ["y"]}]}',              # unresolved input
    '{"inputs": [{"name": "x", "shape": [2], "dtype": "f32"}], "outputs": ["y"], "nodes": '
    '[{"name": "a", "op": "Mul", "inputs": ["x", "z"], "outputs": ["y"]}, '
    '{"name": "b", "op": "Mul", "inputs": ["y", "y"], "outputs": ["z"]}]}',               # cycle
    '{"inputs": [], "outputs": [], "nodes": [{"name": "n", "op": "Mul", "inputs": [], "outputs": []}]}',
    '{"inputs": [], "outputs": [], "nodes": [], "initializers": '
    '[{"name": "c", "shape": [3], "dtype": "f32", "data": [1, 2]}]}',                     # data length
]


@pytest.mark.parametrize("text", BAD_GRAPHS)
def test_error_type_and_message_match_reference(text):
    R = _ref()
    with pytest.raises(Exception) as theirs:
        R.normalize(text)
    with pytest.raises(capi.RfError) as mine:
        G.normalize(text)
    assert type(mine.value).__name__ == theirs.value.kind
    assert theirs.value.message in str(mine.value)


def test_shape_inference_errors_match_reference():
    R = _ref()
    g = {"inputs": [{"name": "a", "shape": [2, 3], "dtype": "f32"}, {"name": "b", "shape": [4, 5], "dtype": "f32"}],
         "outputs": ["y"], "nodes": [{"name": "mm", "op": "MatMul", "inputs": ["a", "b"], "outputs": ["y"]}]}
    for node in (g["nodes"][0], {"name": "ad", "op": "Add", "inputs": ["a", "b"], "outputs": ["y"]},
                 {"name": "tr", "op": "Transpose", "inputs": ["a"], "outputs": ["y"], "attrs": {"perm": [0]}},
                 {"name": "ex", "op": "Expand", "inputs": ["a"], "outputs": ["y"]}):
        g["nodes"] = [node]
        with pytest.raises(Exception) as theirs:
            R.infer_shapes(json.dumps(g))
        with pytest.raises(G.ValidationError) as mine:
            G.infer_shapes(json.dumps(g))
        assert theirs.value.kind == "ValidationError" and theirs.value.message in str(mine.value)


# ---------------------------------------------------------------------------------------------
# the reference's own test cases, through this API (rewrite_test.cpp, graph_test.cpp)
# ---------------------------------------------------------------------------------------------
TINY = ('{"inputs": [{"name": "x", "shape": [4, 4], "dtype": "f32"}], "outputs": ["y"], '
        '"nodes": [{"name": "m", "op": "MatMul", "inputs": ["x", "x"], "outputs": ["y"]}]}')


def test_find_patterns_cases():
    assert G.find_sdpa_patterns(TINY) == []                                               # NoSoftmaxNoMatch :27-34
    m = G.find_sdpa_patterns(F.build_attention_fixture(layers="g"))
    assert len(m) == 1 and (m[0]["q"], m[0]["k"], m[0]["v"]) == ("hidden",) * 3          # SingleLayerResolvesQkv :36-48
    assert m[0]["k_pre_transposed"] == 0 and m[0]["kind"] == "global"
    assert abs(m[0]["scale"] - 1.0 / math.sqrt(32.0)) < 1e-12
    kinds = [x["kind"] for x in G.find_sdpa_patterns(F.build_attention_fixture(layers="llgl"))]
    assert kinds == ["local", "local", "global", "local"]                                 # FourLayerKindsFromWhereNames :50-60
    g = json.loads(F.build_attention_fixture(layers="g"))
    for n in g["nodes"]:
        if n["op"] == "Add":
            n.setdefault("attrs", {})["layer_kind"] = "local"
    assert [x["kind"] for x in G.find_sdpa_patterns(json.dumps(g))] == ["local"]          # AttrOverrideBeatsName :62-72
    g = json.loads(F.build_attention_fixture(layers="g"))
    for n in g["nodes"]:
        n["name"] = n["name"].replace("Where_2", "Untagged")
    assert G.find_sdpa_patterns(json.dumps(g)) == []                                      # UntaggedKindIsSkippedNotGuessed :74-83
    m = G.find_sdpa_patterns(F.build_attention_fixture(layers="g", pre_transposed_k=True))
    assert len(m) == 1 and m[0]["k_pre_transposed"] == 1 and m[0]["k"] == "key_t"         # PreTransposedKVariant :85-94


def test_rewrite_cases():
    assert G.rewrite(TINY) == G.normalize(TINY)                                           # ZeroMatchesIsByteIdentical :96-105
    out = json.loads(G.rewrite(F.build_attention_fixture(layers="lg", seq=128, head_dim=64), RewriteOptions(64, 128)))
    fused = [n for n in out["nodes"] if n["op"] == "FusedFlashAttention"]
    assert len(fused) == 2                                                                # LocalWindowAttrsMatchConvention :107-127
    assert (fused[0]["attrs"]["window_left"], fused[0]["attrs"]["window_right"]) == (63, 64)
    assert (fused[1]["attrs"]["window_left"], fused[1]["attrs"]["window_right"]) == (-1, -1)
    assert abs(fused[0]["attrs"]["scale"] - 0.125) < 1e-12 and len(fused[0]["inputs"]) == 4
    assert fused[0]["inputs"][3] == fused[1]["inputs"][3] == "pad_bias"                   # ONE shared pad-bias chain
    S = 128
    text = G.rewrite(F.build_attention_fixture(layers="lg", seq=S, head_dim=32), RewriteOptions(32, 128))
    out = json.loads(text)                                                                # CleansMaskSubgraphAndSxSTensors :129-151
    assert not [n for n in out["nodes"] if n["op"] in ("Where", "Expand", "Softmax")]
    assert "local_window_pattern" not in [i["name"] for i in out["initializers"]]
    for name, shape in G.infer_shapes(text).items():
        assert not (len(shape) >= 2 and shape[-1] == S and shape[-2] == S), name
    bias_chain = [n["op"] for n in out["nodes"][:3]]
    assert bias_chain == ["Sub", "Mul", "Cast"] and out["nodes"][2]["attrs"] == {"to": "f16"}   # rewrite.cpp:303-318


def test_rewrite_errors_are_typed():
    fx = F.build_attention_fixture()                                                      # ErrorsAreTyped :162-176
    with pytest.raises(UnsupportedHeadDim):
        G.rewrite(fx, RewriteOptions(48, 128))
    with pytest.raises(UnsupportedHeadDim):
        G.rewrite(fx, RewriteOptions(64, 128))        # fixture head_dim is 32
    with pytest.raises(G.NoAttentionMaskInput):
        G.rewrite(fx, RewriteOptions(32, 128, "no_such_input"))
    with pytest.raises(ValueError):
        G.rewrite(fx, RewriteOptions(32, 3))


def test_dce_cases():
    fx = F.build_attention_fixture(layers="lg")
    assert F.canon(G.dce(fx)) == F.canon(fx)                                              # NoDeadNodesUnchanged / NeverRemovesReachable


def test_serialization_is_deterministic_and_round_trips():
    fx = F.build_attention_fixture(layers="lgl", seq=12, local_window=4)
    a = G.normalize(fx)
    assert G.normalize(a) == a and json.loads(a) == json.loads(fx)
    # stock one-element-per-line layout with 2-space indent, reals always carry a fraction
    assert '"shape": [\n        1,\n        2,\n        12,\n        32\n      ]' in a
    assert '-65504.0' in a and '0.17677669529663687' in a


def test_real_number_text_is_shortest_round_trip():
    rng = np.random.default_rng(0)
    vals = [0.0, -0.0, 1.0, -1.0, 0.1, 0.125, 1e-4, 9.999e-5, 1e-5, 123456789.0, 1e14, 2.5e-7, 65504.0, 1 / 3, 1e15 / 3,
            5e-324, 1.7976931348623157e308] + list(rng.standard_normal(200)) + list(np.exp(rng.uniform(-60, 30, 200)))
    g = {"inputs": [], "outputs": ["c"], "nodes": [], "initializers": [
        {"name": "c", "shape": [len(vals)], "dtype": "f32", "data": [float(v) for v in vals]}]}
    text = G.normalize(json.dumps(g))
    back = json.loads(text)["initializers"][0]["data"]
    for v, b in zip(vals, back):
        assert struct.pack("<d", float(v)) == struct.pack("<d", b)                         # exact round trip
    body = text[text.index('"data"'):]
    for tok in [t.strip().rstrip(",") for t in body.splitlines()[1:1 + len(vals)]]:
        assert ("." in tok) or ("e" in tok), tok                                          # never looks like an integer
        assert float(tok) == float(repr(float(tok)))
        assert len(tok.replace("-", "").replace(".", "").lstrip("0")) <= 22
    assert "1e-05" in text and "0.0001" in text and "2.5e-07" in text                     # exponent style


def _build_cpp_graph_test():
    import subprocess
    exe = os.path.join(ROOT, "tests", "cpp", "graph_test")
    src = os.path.join(ROOT, "tests", "cpp", "graph_test.cpp")
    libdir = os.path.join(ROOT, "paper_2603_12646_b200")
    lib = os.path.join(libdir, "librf_fa.so")
    capi.load()  # builds the library if it is missing
    if not os.path.exists(exe) or os.path.getmtime(exe) < max(os.path.getmtime(src), os.path.getmtime(lib)):
        cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
        subprocess.run([cxx, "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
                        "-L", libdir, "-l:librf_fa.so", f"-Wl,-rpath,{libdir}"], check=True)
    return exe


def test_cpp_graph_api_host_logic():
    """tests/cpp/graph_test.cpp --cpu: the C++ mirror (include/routefast_b200/graph.hpp) of the reference's
    rewrite_test.cpp / graph_test.cpp cases that need no device."""
    import subprocess
    res = subprocess.run([_build_cpp_graph_test(), "--cpu"], capture_output=True, text=True, timeout=300)
    print(res.stdout[-2000:], res.stderr[-2000:])
    assert res.returncode == 0 and "all checks passed" in res.stdout
