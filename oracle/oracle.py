"""ctypes loaders for the two CPU checkers (TEST INFRASTRUCTURE ONLY -- never the product path).

* ``port``      -> oracle/librf_oracle.so, our plain-C restatement (oracle/rf_oracle.c)
* ``reference`` -> oracle/_ref/libref_attn.so, the UNMODIFIED reference sources behind
  oracle/ref_shim.cpp (built by oracle/Makefile where /root/reference exists; the prebuilt
  .so travels to the GPU box with the snapshot).

Both expose the same numpy-level API.  Error behaviour mirrors the reference: the shape
checks of proj/core/src/attention.cpp:14-21,110-116 raise :class:`ShapeMismatch`.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "librf_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_attn.so")

MASK_VALUE = -65504.0      # proj/core/include/routefast/attention.hpp:15
MASK_THRESHOLD = -30000.0  # proj/core/include/routefast/attention.hpp:16

__all__ = [
    "ShapeMismatch", "build", "have_reference", "flash_attention", "sdpa", "window_to_mask2d",
    "quantize_f16", "pad_bias_from_mask", "random_tensors", "effective_scale",
    "mask_memory_bytes", "fa_memory_bytes", "flash_stats", "round_bf16", "live_pairs",
    "sdpa_double_reference", "window_live_reference", "float_to_half", "half_to_float",
    "MASK_VALUE", "MASK_THRESHOLD",
]


class ShapeMismatch(RuntimeError):
    """Same role as routefast::ShapeMismatch (proj/core/include/routefast/tensor.hpp:16-19)."""


_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
_i64 = C.c_int64
_u64 = C.c_uint64


def build(force: bool = False) -> None:
    """Compile the checkers (`make -C oracle`).  Building the checker is not using it."""
    need = force or not os.path.exists(PORT_SO) or (
        os.path.getmtime(PORT_SO) < os.path.getmtime(os.path.join(HERE, "rf_oracle.c")))
    ref_possible = os.path.isdir("/root/reference/proj/core/src")
    need_ref = ref_possible and (force or not os.path.exists(REF_SO) or (
        os.path.getmtime(REF_SO) < os.path.getmtime(os.path.join(HERE, "ref_shim.cpp"))))
    graph_so = os.path.join(HERE, "_ref", "libref_graph.so")
    need_refgraph = ref_possible and (force or not os.path.exists(graph_so) or (
        os.path.getmtime(graph_so) < os.path.getmtime(os.path.join(HERE, "ref_graph_shim.cpp"))))
    targets = (["oracle"] if need else []) + (["ref"] if need_ref else []) + (["refgraph"] if need_refgraph else [])
    if targets:
        subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_port = None
_ref = None


def _load_port():
    global _port
    if _port is None:
        build()
        lib = C.CDLL(PORT_SO)
        lib.rf_oracle_flash_attention.restype = C.c_int
        lib.rf_oracle_flash_attention.argtypes = [_f32p, _f32p, _f32p, _f32p, _i64, _i64, _i64, _i64,
                                                  C.c_double, _i64, _i64, _f32p, _i64, C.c_int]
        lib.rf_oracle_sdpa.restype = C.c_int
        lib.rf_oracle_sdpa.argtypes = [_f32p, _f32p, _f32p, _f32p, _i64, _i64, _i64, _i64, _f32p, _i64,
                                       _i64, C.c_double]
        lib.rf_oracle_window_to_mask2d.restype = C.c_int
        lib.rf_oracle_window_to_mask2d.argtypes = [_i64, _i64, _i64, _f32p, _i64, _f32p]
        lib.rf_oracle_quantize_f16_array.argtypes = [_f32p, _f32p, _i64]
        lib.rf_oracle_pad_bias_from_mask.argtypes = [_f32p, _f32p, _i64]
        lib.rf_oracle_rng_new.restype = C.c_void_p
        lib.rf_oracle_rng_new.argtypes = [_u64]
        lib.rf_oracle_rng_free.argtypes = [C.c_void_p]
        lib.rf_oracle_random_fill.argtypes = [C.c_void_p, _f32p, _i64, C.c_int]
        lib.rf_oracle_effective_scale.restype = C.c_double
        lib.rf_oracle_effective_scale.argtypes = [C.c_double, _i64]
        lib.rf_oracle_mask_memory_bytes.restype = _u64
        lib.rf_oracle_mask_memory_bytes.argtypes = [_u64] * 4
        lib.rf_oracle_fa_memory_bytes.restype = _u64
        lib.rf_oracle_fa_memory_bytes.argtypes = [_u64] * 6
        lib.rf_oracle_flash_stats.argtypes = [_i64] * 5 + [C.POINTER(_u64)] * 3
        lib.rf_oracle_round_bf16_array.argtypes = [_f32p, _f32p, _i64]
        lib.rf_oracle_live_pairs.restype = _u64
        lib.rf_oracle_live_pairs.argtypes = [_i64, _i64, _i64, _f32p]
        lib.rf_oracle_sdpa_double_reference.restype = C.c_int
        lib.rf_oracle_sdpa_double_reference.argtypes = [_f64p] * 4 + [_i64] * 4 + [C.c_double]
        lib.rf_oracle_window_live_reference.restype = C.c_int
        lib.rf_oracle_window_live_reference.argtypes = [_i64] * 4 + [C.POINTER(C.c_uint8), _i64]
        lib.rf_oracle_float_to_half.restype = C.c_uint16
        lib.rf_oracle_float_to_half.argtypes = [C.c_float]
        lib.rf_oracle_half_to_float.restype = C.c_float
        lib.rf_oracle_half_to_float.argtypes = [C.c_uint16]
        _port = lib
    return _port


def have_reference() -> bool:
    if not os.path.exists(REF_SO):
        try:
            build()
        except Exception:
            return False
    return os.path.exists(REF_SO)


def _load_ref():
    global _ref
    if _ref is None:
        if not have_reference():
            raise RuntimeError("oracle/_ref/libref_attn.so not built (needs /root/reference)")
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_flash_attention.restype = C.c_int
        lib.ref_flash_attention.argtypes = [_f32p, _f32p, _f32p, _f32p, _i64, _i64, _i64, _i64,
                                            C.c_double, _i64, _i64, _f32p, C.POINTER(_i64), _i64,
                                            C.c_int, C.POINTER(_u64)]
        lib.ref_sdpa.restype = C.c_int
        lib.ref_sdpa.argtypes = [_f32p, _f32p, _f32p, _f32p, _i64, _i64, _i64, _i64, _f32p, _i64, _i64,
                                 C.c_double]
        lib.ref_window_to_mask2d.restype = C.c_int
        lib.ref_window_to_mask2d.argtypes = [_i64, _i64, _i64, _f32p, _i64, _f32p]
        lib.ref_quantize_f16.restype = C.c_float
        lib.ref_quantize_f16.argtypes = [C.c_float]
        lib.ref_float_to_half.restype = C.c_uint16
        lib.ref_float_to_half.argtypes = [C.c_float]
        lib.ref_half_to_float.restype = C.c_float
        lib.ref_half_to_float.argtypes = [C.c_uint16]
        lib.ref_effective_scale.restype = C.c_double
        lib.ref_effective_scale.argtypes = [C.c_double, _i64]
        lib.ref_mask_memory_bytes.restype = _u64
        lib.ref_mask_memory_bytes.argtypes = [_u64] * 4
        lib.ref_fa_memory_bytes.restype = _u64
        lib.ref_fa_memory_bytes.argtypes = [_u64] * 6
        lib.ref_random_fill.argtypes = [_u64, _f32p, _i64, _i64, C.c_int]
        _ref = lib
    return _ref


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _p(a: Optional[np.ndarray]):
    return a.ctypes.data_as(_f32p) if a is not None else None


def _check_qkv(q, k, v):
    # proj/core/src/attention.cpp:14-21
    if q.ndim != 4 or k.ndim != 4 or v.ndim != 4:
        raise ShapeMismatch("attention inputs must be [B,H,S,d]")
    if q.shape != k.shape or q.shape != v.shape:
        raise ShapeMismatch("Q, K, V must have identical shapes")


def flash_attention(q, k, v, scale: float = 0.0, window_left: int = -1, window_right: int = -1,
                    pad_bias=None, tile: int = 64, threads: int = 1, impl: str = "port") -> np.ndarray:
    """routefast::flash_attention (proj/core/include/routefast/attention.hpp:46-48)."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    _check_qkv(q, k, v)
    B, H, S, d = q.shape
    if tile < 1:
        raise ShapeMismatch("tile must be >= 1")  # attention.cpp:110
    pb = None
    if pad_bias is not None:
        pb = _f32(pad_bias)
        if impl != "reference" and pb.shape != (B, 1, 1, S):
            raise ShapeMismatch("pad_bias must be [B,1,1,S]")  # attention.cpp:111-116
    out = np.empty_like(q)
    if impl == "port":
        rc = _load_port().rf_oracle_flash_attention(_p(q), _p(k), _p(v), _p(out), B, H, S, d, float(scale),
                                                    int(window_left), int(window_right), _p(pb), int(tile),
                                                    int(threads))
        if rc != 0:
            raise ShapeMismatch(f"rf_oracle_flash_attention failed rc={rc}")
    elif impl == "reference":
        lib = _load_ref()
        dims = None
        if pb is not None:
            if pb.ndim != 4:
                raise ShapeMismatch("pad_bias must be [B,1,1,S]")
            dims = (_i64 * 4)(*pb.shape)
        rc = lib.ref_flash_attention(_p(q), _p(k), _p(v), _p(out), B, H, S, d, float(scale), int(window_left),
                                     int(window_right), _p(pb), dims, int(tile), int(threads), None)
        if rc != 0:
            raise ShapeMismatch(lib.ref_last_error().decode())
    else:
        raise ValueError(impl)
    return out


def flash_stats(B, H, S, d, tile=64):
    """FlashStats (attention.hpp:36-40)."""
    a, b, c = _u64(), _u64(), _u64()
    _load_port().rf_oracle_flash_stats(B, H, S, d, tile, C.byref(a), C.byref(b), C.byref(c))
    return {"tile_scratch_floats": a.value, "row_state_floats": b.value, "output_floats": c.value}


def sdpa(q, k, v, mask2d=None, scale: float = 1.0, impl: str = "port") -> np.ndarray:
    """routefast::sdpa (attention.hpp:31-32)."""
    q, k, v = _f32(q), _f32(k), _f32(v)
    _check_qkv(q, k, v)
    B, H, S, d = q.shape
    m = None
    mB = mH = 1
    if mask2d is not None:
        m = _f32(mask2d)
        if m.ndim != 4 or m.shape[2] != S or m.shape[3] != S or m.shape[0] not in (1, B) or m.shape[1] not in (1, H):
            raise ShapeMismatch("mask2d must broadcast over [B,H,S,S]")  # attention.cpp:42-48
        mB, mH = m.shape[0], m.shape[1]
    out = np.empty_like(q)
    if impl == "port":
        rc = _load_port().rf_oracle_sdpa(_p(q), _p(k), _p(v), _p(out), B, H, S, d, _p(m), mB, mH, float(scale))
    else:
        rc = _load_ref().ref_sdpa(_p(q), _p(k), _p(v), _p(out), B, H, S, d, _p(m), mB, mH, float(scale))
    if rc != 0:
        raise ShapeMismatch("sdpa failed")
    return out


def window_to_mask2d(seq_len: int, window_left: int, window_right: int, pad_bias=None, impl: str = "port"):
    """routefast::window_to_mask2d (attention.hpp:53-54) -> [B,1,S,S]."""
    if seq_len < 1:
        raise ShapeMismatch("seq_len must be >= 1")
    B = 1
    pb = None
    if pad_bias is not None:
        pb = _f32(pad_bias)
        if pb.ndim != 4 or pb.shape[1] != 1 or pb.shape[2] != 1 or pb.shape[3] != seq_len:
            raise ShapeMismatch("pad_bias must be [B,1,1,S]")
        B = pb.shape[0]
    mask = np.empty((B, 1, seq_len, seq_len), dtype=np.float32)
    fn = _load_port().rf_oracle_window_to_mask2d if impl == "port" else _load_ref().ref_window_to_mask2d
    rc = fn(seq_len, window_left, window_right, _p(pb), B, _p(mask))
    if rc != 0:
        raise ShapeMismatch("window_to_mask2d failed")
    return mask


def quantize_f16(x, impl: str = "port"):
    """quantize_f16 (proj/core/src/tensor.cpp:98), elementwise."""
    a = _f32(x)
    out = np.empty_like(a)
    if impl == "port":
        _load_port().rf_oracle_quantize_f16_array(_p(a), _p(out), a.size)
    else:
        lib = _load_ref()
        flat, o = a.reshape(-1), out.reshape(-1)
        for i in range(flat.size):
            o[i] = lib.ref_quantize_f16(float(flat[i]))
    return out


def float_to_half(x: float, impl: str = "port") -> int:
    return (_load_port().rf_oracle_float_to_half if impl == "port" else _load_ref().ref_float_to_half)(float(x))


def half_to_float(bits: int, impl: str = "port") -> float:
    return (_load_port().rf_oracle_half_to_float if impl == "port" else _load_ref().ref_half_to_float)(int(bits))


def pad_bias_from_mask(attention_mask):
    """The rewriter's shared pad-bias chain (proj/core/src/rewrite.cpp:303-318): Cast_f16(-65504*(1-mask))."""
    m = _f32(attention_mask)
    out = np.empty_like(m)
    _load_port().rf_oracle_pad_bias_from_mask(_p(m), _p(out), m.size)
    return out


def random_tensors(seed: int, shape, n: int = 1, as_f16: bool = False, impl: str = "port"):
    """n tensors drawn consecutively from one mt19937_64(seed) like Tensor::random (tensor.cpp:35-45)."""
    each = int(np.prod(shape))
    buf = np.empty((n, each), dtype=np.float32)
    if impl == "port":
        lib = _load_port()
        g = lib.rf_oracle_rng_new(seed)
        try:
            for t in range(n):
                lib.rf_oracle_random_fill(g, _p(buf[t]), each, int(as_f16))
        finally:
            lib.rf_oracle_rng_free(g)
    else:
        _load_ref().ref_random_fill(seed, _p(buf), each, n, int(as_f16))
    return [buf[t].reshape(shape).copy() for t in range(n)]


def effective_scale(scale: float, head_dim: int, impl: str = "port") -> float:
    fn = _load_port().rf_oracle_effective_scale if impl == "port" else _load_ref().ref_effective_scale
    return fn(float(scale), int(head_dim))


def mask_memory_bytes(batch, heads, seq_len, bpe, impl: str = "port") -> int:
    fn = _load_port().rf_oracle_mask_memory_bytes if impl == "port" else _load_ref().ref_mask_memory_bytes
    return fn(batch, heads, seq_len, bpe)


def fa_memory_bytes(batch, heads, seq_len, head_dim, tile, bpe, impl: str = "port") -> int:
    fn = _load_port().rf_oracle_fa_memory_bytes if impl == "port" else _load_ref().ref_fa_memory_bytes
    return fn(batch, heads, seq_len, head_dim, tile, bpe)


def round_bf16(x) -> np.ndarray:
    """f32 -> bf16 -> f32 (RNE); applied to BOTH sides' inputs in a parity test (ours, not the reference's)."""
    a = _f32(x)
    out = np.empty_like(a)
    _load_port().rf_oracle_round_bf16_array(_p(a), _p(out), a.size)
    return out


def live_pairs(S: int, window_left: int, window_right: int, pad_row=None) -> int:
    """#(i,j) pairs the reference multiplies for one batch row (attention.cpp:160-167)."""
    pr = _f32(pad_row) if pad_row is not None else None
    return _load_port().rf_oracle_live_pairs(S, window_left, window_right, _p(pr))


def sdpa_double_reference(q, k, v, scale: float) -> np.ndarray:
    """The reference test suite's independent f64 SDPA (proj/tests/support/oracles.cpp:83-121)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    B, H, S, d = q.shape
    out = np.empty_like(q)
    dp = lambda a: a.ctypes.data_as(_f64p)  # noqa: E731
    _load_port().rf_oracle_sdpa_double_reference(dp(q), dp(k), dp(v), dp(out), B, H, S, d, float(scale))
    return out


def window_live_reference(i, j, wl, wr, padded=None) -> bool:
    """proj/tests/support/oracles.cpp:123-129."""
    if padded is None or len(padded) == 0:
        return bool(_load_port().rf_oracle_window_live_reference(i, j, wl, wr, None, 0))
    arr = np.ascontiguousarray(padded, dtype=np.uint8)
    return bool(_load_port().rf_oracle_window_live_reference(
        i, j, wl, wr, arr.ctypes.data_as(C.POINTER(C.c_uint8)), arr.size))
