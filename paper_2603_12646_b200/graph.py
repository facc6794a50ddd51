"""Graph layer around the FusedFlashAttention operator: JSON graph IR, the SDPA ->
FusedFlashAttention rewriter and the GPU graph executor, through the C ABI of include/rf_graph.h.

Mirrors the reference's interface (proj/core/include/routefast/graph.hpp:88-103,
rewrite.hpp:47-63, interpreter.hpp:25) with graphs carried as the reference's own JSON text:

    parse_graph + serialize_graph -> normalize        infer_shapes / topological_order
    find_sdpa_patterns            -> find_sdpa_patterns
    rewrite(graph, RewriteOptions) -> rewrite          dce
    interpret(graph, inputs)      -> interpret  (every node runs on the B200; no CPU fallback)
    verify-rewrite (proj/tools/main.cpp:106-149) -> verify_rewrite
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import capi
from .attention import RewriteOptions


class SchemaError(capi.RfError):
    """reference SchemaError (graph.hpp:17-20)"""


class ValidationError(capi.RfError):
    """reference ValidationError (graph.hpp:23-26)"""


class NoAttentionMaskInput(capi.RfError):
    """reference NoAttentionMaskInput (rewrite.hpp:19-22)"""


class UnsupportedOp(capi.RfError):
    """reference UnsupportedOp (interpreter.hpp:14-17)"""


RF_ERR_SCHEMA, RF_ERR_VALIDATION, RF_ERR_NO_MASK_INPUT, RF_ERR_UNSUPPORTED_OP = 7, 8, 9, 10
_GRAPH_ERRORS = {RF_ERR_SCHEMA: SchemaError, RF_ERR_VALIDATION: ValidationError,
                 RF_ERR_NO_MASK_INPUT: NoAttentionMaskInput, RF_ERR_UNSUPPORTED_OP: UnsupportedOp}


class _Stats(C.Structure):
    _fields_ = [("peak_device_bytes", C.c_uint64), ("largest_tensor_bytes", C.c_uint64), ("launches", C.c_uint64),
                ("device_ms", C.c_double)]


@dataclass
class InterpretStats:
    peak_device_bytes: int = 0
    largest_tensor_bytes: int = 0
    launches: int = 0
    device_ms: float = 0.0


_bound = False


def _lib():
    global _bound
    lib = capi.load()
    if not _bound:
        cpp = C.POINTER(C.c_char_p)
        lib.rf_graph_free.argtypes = [C.c_void_p]
        lib.rf_graph_free.restype = None
        for name in ("normalize", "infer_shapes", "topological_order", "find_patterns", "dce"):
            fn = getattr(lib, "rf_graph_" + name)
            fn.restype, fn.argtypes = C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]
        lib.rf_graph_rewrite.restype = C.c_int
        lib.rf_graph_rewrite.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_char_p, C.POINTER(C.c_void_p),
                                         C.POINTER(C.c_int64)]
        lib.rf_graph_interpret.restype = C.c_int
        lib.rf_graph_interpret.argtypes = [C.c_char_p, C.c_int32, cpp, C.POINTER(C.POINTER(C.c_float)),
                                           C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.c_int32), C.c_int32,
                                           C.POINTER(C.c_void_p)]
        lib.rf_graph_result_count.restype, lib.rf_graph_result_count.argtypes = C.c_int32, [C.c_void_p]
        lib.rf_graph_result_name.restype, lib.rf_graph_result_name.argtypes = C.c_char_p, [C.c_void_p, C.c_int32]
        lib.rf_graph_result_rank.restype, lib.rf_graph_result_rank.argtypes = C.c_int32, [C.c_void_p, C.c_int32]
        lib.rf_graph_result_dims.restype = C.POINTER(C.c_int64)
        lib.rf_graph_result_dims.argtypes = [C.c_void_p, C.c_int32]
        lib.rf_graph_result_data.restype = C.POINTER(C.c_float)
        lib.rf_graph_result_data.argtypes = [C.c_void_p, C.c_int32]
        lib.rf_graph_result_is_f16.restype, lib.rf_graph_result_is_f16.argtypes = C.c_int32, [C.c_void_p, C.c_int32]
        lib.rf_graph_result_stats.restype, lib.rf_graph_result_stats.argtypes = None, [C.c_void_p, C.POINTER(_Stats)]
        lib.rf_graph_result_free.restype, lib.rf_graph_result_free.argtypes = None, [C.c_void_p]
        _bound = True
    return lib


def _check(rc: int) -> None:
    if rc in _GRAPH_ERRORS:
        raise _GRAPH_ERRORS[rc](rc, capi.load().rf_last_error().decode(errors="replace"))
    if rc == capi.RF_ERR_ARG and b"local_window" in capi.load().rf_last_error():
        raise ValueError(capi.load().rf_last_error().decode())  # reference: std::invalid_argument
    capi.check(rc)


def _text_call(fn, graph_json: str, *extra) -> str:
    lib = _lib()
    out = C.c_void_p()
    _check(fn(graph_json.encode(), *extra, C.byref(out)))
    try:
        return C.string_at(out).decode()
    finally:
        lib.rf_graph_free(out)


def normalize(graph_json: str) -> str:
    """serialize_graph(parse_graph(text)): validates and returns the deterministic form."""
    return _text_call(_lib().rf_graph_normalize, graph_json)


def infer_shapes(graph_json: str) -> Dict[str, List[int]]:
    return json.loads(_text_call(_lib().rf_graph_infer_shapes, graph_json))


def topological_order(graph_json: str) -> List[int]:
    return json.loads(_text_call(_lib().rf_graph_topological_order, graph_json))


def find_sdpa_patterns(graph_json: str) -> List[dict]:
    return json.loads(_text_call(_lib().rf_graph_find_patterns, graph_json))


def dce(graph_json: str) -> str:
    return _text_call(_lib().rf_graph_dce, graph_json)


def rewrite(graph_json: str, options: Optional[RewriteOptions] = None) -> str:
    """routefast::rewrite (rewrite.hpp:55-59): every SDPA chain -> one FusedFlashAttention node, one
    shared pad-bias chain, per-layer windows, then dce.  Returns the rewritten graph as JSON."""
    options = options or RewriteOptions()
    lib = _lib()
    out = C.c_void_p()
    n = C.c_int64(0)
    _check(lib.rf_graph_rewrite(graph_json.encode(), options.head_dim, options.local_window,
                                options.mask_input.encode(), C.byref(out), C.byref(n)))
    try:
        return C.string_at(out).decode()
    finally:
        lib.rf_graph_free(out)


def interpret(graph_json: str, inputs: Dict[str, np.ndarray], device: int = 0,
              stats: Optional[InterpretStats] = None) -> Dict[str, np.ndarray]:
    """routefast::interpret (interpreter.hpp:25) on the GPU: host f32 arrays in, graph outputs out."""
    lib = _lib()
    names = list(inputs)
    arrs = [np.ascontiguousarray(inputs[n], dtype=np.float32) for n in names]
    n = len(names)
    c_names = (C.c_char_p * n)(*[s.encode() for s in names])
    c_data = (C.POINTER(C.c_float) * n)(*[a.ctypes.data_as(C.POINTER(C.c_float)) for a in arrs])
    dims = [(C.c_int64 * max(a.ndim, 1))(*a.shape) for a in arrs]
    c_dims = (C.POINTER(C.c_int64) * n)(*[C.cast(d, C.POINTER(C.c_int64)) for d in dims])
    c_ranks = (C.c_int32 * n)(*[a.ndim for a in arrs])
    res = C.c_void_p()
    _check(lib.rf_graph_interpret(graph_json.encode(), n, c_names, c_data, c_dims, c_ranks, device, C.byref(res)))
    try:
        out: Dict[str, np.ndarray] = {}
        for i in range(lib.rf_graph_result_count(res)):
            rank = lib.rf_graph_result_rank(res, i)
            shape = [lib.rf_graph_result_dims(res, i)[a] for a in range(rank)]
            count = int(np.prod(shape)) if rank else 1
            data = np.ctypeslib.as_array(lib.rf_graph_result_data(res, i), shape=(count,)).copy() if count else np.empty(0, np.float32)
            out[lib.rf_graph_result_name(res, i).decode()] = data.reshape(shape)
        if stats is not None:
            st = _Stats()
            lib.rf_graph_result_stats(res, C.byref(st))
            stats.peak_device_bytes, stats.largest_tensor_bytes = int(st.peak_device_bytes), int(st.largest_tensor_bytes)
            stats.launches, stats.device_ms = int(st.launches), float(st.device_ms)
        return out
    finally:
        lib.rf_graph_result_free(res)


def random_inputs(graph_json: str, rng: np.random.Generator) -> Dict[str, np.ndarray]:
    """Inputs as `verify-rewrite` draws them (proj/tools/main.cpp:88-104): *mask* inputs are ones with
    a zero tail of up to seq/8 keys, everything else U[-1, 1)."""
    out = {}
    for decl in json.loads(graph_json)["inputs"]:
        shape = decl["shape"]
        if "mask" in decl["name"] and shape:
            m = np.ones(shape, np.float32)
            seq = shape[-1]
            pad = int(rng.integers(0, seq // 8)) if seq > 8 else 0
            if pad:
                m.reshape(-1)[-pad:] = 0.0
            out[decl["name"]] = m
        else:
            out[decl["name"]] = rng.uniform(-1.0, 1.0, shape).astype(np.float32)
    return out


def verify_rewrite(graph_json: str, rewritten_json: str, trials: int = 3, tol: float = 2e-2, seed: int = 42,
                   device: int = 0, valid_rows_only: bool = True) -> Tuple[bool, List[dict]]:
    """`routefast verify-rewrite` on the GPU: interpret original and rewritten graph on the same random
    inputs and compare every output (max-abs).  tol defaults to the attention tolerance of the bf16
    kernel (BASELINE.json: 2e-2); the reference's own 1e-3 applies to its two f64 paths.

    valid_rows_only: padded QUERY rows are reported separately and not judged.  The fused operator
    returns 0 for a row with no live key (attention.cpp:175,204-207) where the un-fused chain returns
    a softmax over uniformly masked scores; with a local window and more than window_left padded keys
    such rows exist at padded positions (the CLI draws up to seq/8 padded keys).  They are never
    read as keys by later layers, so unpadded rows are unaffected."""
    rng = np.random.default_rng(seed)
    report, ok = [], True
    outputs = json.loads(graph_json)["outputs"]
    for t in range(trials):
        inputs = random_inputs(graph_json, rng)
        masks = [v for k, v in inputs.items() if "mask" in k and v.ndim == 4 and v.shape[1] == v.shape[2] == 1]
        sa, sb = InterpretStats(), InterpretStats()
        a = interpret(graph_json, inputs, device, sa)
        b = interpret(rewritten_json, inputs, device, sb)
        for name in outputs:
            if name not in b or b[name].shape != a[name].shape:
                ok = False
                report.append({"trial": t, "output": name, "error": "missing or mis-shaped in rewritten graph"})
                continue
            diff = np.abs(a[name] - b[name])
            entry = {"trial": t, "output": name, "tol": tol, "original": vars(sa), "rewritten": vars(sb)}
            if (valid_rows_only and masks and diff.ndim == 4 and diff.shape[0] == masks[0].shape[0]
                    and diff.shape[2] == masks[0].shape[3]):
                valid = (masks[0][:, 0, 0, :] != 0)[:, None, :, None]
                entry["max_abs_diff_padded_rows"] = float(np.where(valid, 0.0, diff).max()) if diff.size else 0.0
                diff = np.where(valid, diff, 0.0)
            entry["max_abs_diff"] = float(diff.max()) if diff.size else 0.0
            ok = ok and entry["max_abs_diff"] <= tol
            report.append(entry)
    return ok, report
