"""ctypes access to oracle/_ref/libref_graph.so -- the UNMODIFIED reference graph IR, rewriter,
interpreter and fixture generator (TEST INFRASTRUCTURE ONLY; see oracle/ref_graph_shim.cpp).

Used by tests/ to pin the graph layer of librf_fa.so and by tests/golden/make_graph_golden.py to
generate the committed fixtures.  Never imported from paper_2603_12646_b200/.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Dict, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_ref", "libref_graph.so")
_lib = None


class RefGraphError(RuntimeError):
    """Carries the reference's exception type name in .kind (e.g. 'ValidationError')."""

    def __init__(self, text: str):
        kind, _, msg = text.partition(": ")
        super().__init__(text)
        self.kind, self.message = kind, msg


def available() -> bool:
    return os.path.exists(SO)


def _load():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError("oracle/_ref/libref_graph.so not built (needs /root/reference; make -C oracle refgraph)")
        lib = C.CDLL(SO)
        lib.ref_graph_last_error.restype = C.c_char_p
        lib.ref_graph_free.argtypes = [C.c_void_p]
        for name in ("normalize", "infer_shapes", "topological_order", "find_patterns", "dce"):
            fn = getattr(lib, "ref_graph_" + name)
            fn.restype, fn.argtypes = C.c_void_p, [C.c_char_p]
        lib.ref_graph_rewrite.restype = C.c_void_p
        lib.ref_graph_rewrite.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_char_p]
        lib.ref_graph_fixture.restype = C.c_void_p
        lib.ref_graph_fixture.argtypes = [C.c_int64] * 5 + [C.c_char_p, C.c_int]
        lib.ref_graph_interpret.restype = C.c_int64
        _lib = lib
    return _lib


def _text(ptr) -> str:
    lib = _load()
    if not ptr:
        raise RefGraphError(lib.ref_graph_last_error().decode())
    try:
        return C.string_at(ptr).decode()
    finally:
        lib.ref_graph_free(ptr)


def normalize(graph_json: str) -> str:
    return _text(_load().ref_graph_normalize(graph_json.encode()))


def infer_shapes(graph_json: str) -> Dict[str, list]:
    return json.loads(_text(_load().ref_graph_infer_shapes(graph_json.encode())))


def topological_order(graph_json: str) -> list:
    return json.loads(_text(_load().ref_graph_topological_order(graph_json.encode())))


def find_patterns(graph_json: str) -> list:
    return json.loads(_text(_load().ref_graph_find_patterns(graph_json.encode())))


def dce(graph_json: str) -> str:
    return _text(_load().ref_graph_dce(graph_json.encode()))


def rewrite(graph_json: str, head_dim: int = 64, local_window: int = 128, mask_input: Optional[str] = None) -> str:
    return _text(_load().ref_graph_rewrite(graph_json.encode(), head_dim, local_window,
                                           mask_input.encode() if mask_input is not None else None))


def fixture(batch=1, heads=2, seq=64, head_dim=32, local_window=128, layers="g", pre_transposed_k=False) -> str:
    """build_attention_fixture (proj/tests/support/graph_fixtures.cpp:16-114); layers: 'l'/'g' per layer."""
    return _text(_load().ref_graph_fixture(batch, heads, seq, head_dim, local_window, layers.encode(),
                                           1 if pre_transposed_k else 0))


def interpret(graph_json: str, inputs: Dict[str, np.ndarray], output: str) -> np.ndarray:
    lib = _load()
    names = list(inputs)
    arrs = [np.ascontiguousarray(inputs[n], dtype=np.float32) for n in names]
    n = len(names)
    c_names = (C.c_char_p * n)(*[s.encode() for s in names])
    c_data = (C.POINTER(C.c_float) * n)(*[a.ctypes.data_as(C.POINTER(C.c_float)) for a in arrs])
    dims = [(C.c_int64 * a.ndim)(*a.shape) for a in arrs]
    c_dims = (C.POINTER(C.c_int64) * n)(*[C.cast(d, C.POINTER(C.c_int64)) for d in dims])
    c_ranks = (C.c_int32 * n)(*[a.ndim for a in arrs])
    shapes = infer_shapes(graph_json)
    cap = int(np.prod(shapes[output])) if output in shapes else 0
    out = np.empty(max(cap, 1), np.float32)
    odims = (C.c_int64 * 8)()
    orank = C.c_int32(0)
    got = lib.ref_graph_interpret(graph_json.encode(), n, c_names, c_data, c_dims, c_ranks, output.encode(),
                                  out.ctypes.data_as(C.POINTER(C.c_float)), C.c_int64(out.size), odims, C.byref(orank))
    if got < 0:
        raise RefGraphError(lib.ref_graph_last_error().decode())
    return out[:got].reshape([odims[i] for i in range(orank.value)])
