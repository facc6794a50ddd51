"""ctypes binding of the C ABI in include/rf_fa.h (librf_fa.so).

No torch types cross this boundary: only raw device/host pointers and sizes.  Loading fails
loudly if the shared library is missing -- there is no CPU or PyTorch fallback on this path.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _build

RF_OK, RF_ERR_SHAPE, RF_ERR_HEAD_DIM, RF_ERR_ARG, RF_ERR_CUDA, RF_ERR_WORKSPACE, RF_ERR_UNSUPPORTED = range(7)
RF_ERR_DEVICE_TIMEOUT = 11
RF_DTYPE_BF16, RF_DTYPE_F16, RF_DTYPE_F32 = 0, 1, 2
RF_KERNEL_AUTO, RF_KERNEL_TCGEN05, RF_KERNEL_SIMT = 0, 1, 2

# every symbol include/rf_fa.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = [
    "rf_last_error", "rf_abi_version", "rf_fa_params_init", "rf_fa_validate", "rf_fa_fwd_workspace_bytes",
    "rf_fa_stats_query", "rf_fa_fwd", "rf_fa_plan_create", "rf_fa_plan_launch", "rf_fa_plan_destroy",
    "rf_fa_launch_status", "rf_fa_merge", "rf_fa_rescale_partial", "rf_fa_normalize",
    "rf_pad_bias_from_mask", "rf_cast_f32_to", "rf_cast_to_f32", "rf_fa_fwd_host", "rf_fa_host_release", "rf_host_round_bf16", "rf_fa_host_transfer_counters",
    "rf_fused_flash_attention_op", "rf_mask_memory_bytes", "rf_fa_memory_bytes", "rf_device_check",
    "rf_rope_qkv", "rf_add_layernorm", "rf_geglu",
    # include/rf_graph.h
    "rf_graph_free", "rf_graph_normalize", "rf_graph_infer_shapes", "rf_graph_topological_order",
    "rf_graph_find_patterns", "rf_graph_rewrite", "rf_graph_dce", "rf_graph_interpret", "rf_graph_result_count",
    "rf_graph_result_name", "rf_graph_result_rank", "rf_graph_result_dims", "rf_graph_result_data",
    "rf_graph_result_is_f16", "rf_graph_result_stats", "rf_graph_result_free",
    # include/rf_clf.h
    "rf_clf_config_default", "rf_clf_weight_elems", "rf_clf_create", "rf_clf_forward", "rf_clf_session_bytes",
    "rf_clf_last_forward_ms", "rf_clf_destroy", "rf_clf_head",
    # include/rf_gemm.h
    "rf_gemm_nt", "rf_gemm_launch_status",
]

RF_GEMM_EPI_NONE, RF_GEMM_EPI_ROPE, RF_GEMM_EPI_GEGLU, RF_GEMM_EPI_RESIDUAL = 0, 1, 2, 3
RF_CLF_GEMM_OWN, RF_CLF_GEMM_CUBLAS = 0, 1


class RfGemmEpilogue(C.Structure):
    _fields_ = [("kind", C.c_int32), ("head_dim", C.c_int32), ("S", C.c_int64), ("cos_table", C.c_void_p),
                ("sin_table", C.c_void_p), ("out_dtype", C.c_int32), ("head_major", C.c_int32)]


class RfClfConfig(C.Structure):
    _fields_ = [
        ("vocab_size", C.c_int32), ("hidden", C.c_int32), ("n_layers", C.c_int32), ("heads", C.c_int32),
        ("head_dim", C.c_int32), ("mlp", C.c_int32), ("global_every", C.c_int32), ("local_window", C.c_int32),
        ("n_labels", C.c_int32), ("mlp_chunk_rows", C.c_int32), ("act_dtype", C.c_int32), ("rope_theta_global", C.c_float),
        ("rope_theta_local", C.c_float), ("eps", C.c_float), ("gemm_backend", C.c_int32),
    ]


class RfFaParams(C.Structure):
    _fields_ = [
        ("q", C.c_void_p), ("k", C.c_void_p), ("v", C.c_void_p), ("out", C.c_void_p),
        ("q_stride", C.c_int64 * 3), ("k_stride", C.c_int64 * 3), ("v_stride", C.c_int64 * 3),
        ("o_stride", C.c_int64 * 3),
        ("pad_bias", C.c_void_p),
        ("B", C.c_int64), ("H", C.c_int64), ("S", C.c_int64), ("d", C.c_int64),
        ("scale", C.c_double), ("window_left", C.c_int64), ("window_right", C.c_int64),
        ("dtype", C.c_int32), ("out_dtype", C.c_int32), ("kernel", C.c_int32), ("flags", C.c_int32),
        ("kv_begin", C.c_int64), ("kv_end", C.c_int64),
        ("o_partial", C.c_void_p), ("m_partial", C.c_void_p), ("l_partial", C.c_void_p),
        ("debug_scores", C.c_void_p),
    ]


class RfFaStats(C.Structure):
    _fields_ = [
        ("workspace_bytes", C.c_uint64), ("tile_scratch_bytes", C.c_uint64), ("row_state_bytes", C.c_uint64),
        ("output_bytes", C.c_uint64), ("score_matrix_bytes", C.c_uint64), ("kernel", C.c_int32),
        ("grid_ctas", C.c_int32),
    ]


class RfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"rf_fa error {code}: {msg}")
        self.code = code
        self.msg = msg


class ShapeMismatch(RfError):
    """routefast::ShapeMismatch (reference proj/core/include/routefast/tensor.hpp:16-19)."""


class UnsupportedHeadDim(RfError):
    """routefast::UnsupportedHeadDim (reference proj/core/include/routefast/rewrite.hpp:14-17)."""


_lib = None


def lib_path() -> str:
    # RF_FA_LIB lets a developer point at an experimental build of the same ABI (kernel tuning)
    return os.environ.get("RF_FA_LIB") or _build.LIB


def load(build_if_missing: bool = True):
    """Load librf_fa.so; raises if it cannot be built/loaded (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        if not build_if_missing:
            raise RuntimeError(f"{path} is missing; run `python __graft_entry__.py build`")
        _build.build()
    lib = C.CDLL(path)
    vp, i64, i32, u64, f32p = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.POINTER(C.c_float)
    PP = C.POINTER(RfFaParams)
    lib.rf_last_error.restype = C.c_char_p
    lib.rf_abi_version.restype = C.c_int
    lib.rf_fa_params_init.argtypes = [PP]
    lib.rf_fa_params_init.restype = None
    lib.rf_fa_validate.argtypes = [PP]
    lib.rf_fa_fwd_workspace_bytes.argtypes = [PP, C.POINTER(C.c_size_t)]
    lib.rf_fa_stats_query.argtypes = [PP, C.POINTER(RfFaStats)]
    lib.rf_fa_fwd.argtypes = [PP, vp, C.c_size_t, vp]
    lib.rf_fa_plan_create.argtypes = [PP, vp, C.c_size_t, C.POINTER(vp)]
    lib.rf_fa_plan_create.restype = C.c_int
    lib.rf_fa_plan_launch.argtypes = [vp, vp]
    lib.rf_fa_plan_launch.restype = C.c_int
    lib.rf_fa_plan_destroy.argtypes = [vp]
    lib.rf_fa_plan_destroy.restype = None
    lib.rf_fa_launch_status.argtypes = [vp, vp]
    lib.rf_fa_launch_status.restype = C.c_int
    lib.rf_fa_merge.argtypes = [C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), i32, i64, i64, vp, i32, vp]
    lib.rf_fa_rescale_partial.argtypes = [vp, vp, vp, vp, i64, i64, vp]
    lib.rf_fa_normalize.argtypes = [vp, vp, i64, i64, vp, i32, vp]
    lib.rf_pad_bias_from_mask.argtypes = [vp, vp, i64, vp]
    lib.rf_cast_f32_to.argtypes = [vp, vp, i64, i32, vp]
    lib.rf_cast_to_f32.argtypes = [vp, vp, i64, i32, vp]
    lib.rf_fa_fwd_host.argtypes = [f32p, f32p, f32p, f32p, i64, i64, i64, i64, C.c_double, i64, i64, f32p,
                                   C.POINTER(i64), i64, i32, i32, C.POINTER(RfFaStats)]
    lib.rf_fused_flash_attention_op.argtypes = [C.POINTER(f32p), C.POINTER(C.POINTER(i64)), C.POINTER(i32), i32,
                                                i32, C.c_double, i32, i64, i32, i64, f32p, i32]
    lib.rf_rope_qkv.argtypes = [vp, vp, vp, i64, i64, i64, i64, i32, vp]
    lib.rf_add_layernorm.argtypes = [vp, vp, vp, vp, i64, i64, C.c_float, i32, vp]
    lib.rf_geglu.argtypes = [vp, vp, i64, i64, i32, vp]
    lib.rf_mask_memory_bytes.restype = u64
    lib.rf_mask_memory_bytes.argtypes = [u64] * 4
    lib.rf_fa_memory_bytes.restype = u64
    lib.rf_fa_memory_bytes.argtypes = [u64] * 6
    lib.rf_device_check.argtypes = [i32, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)]
    lib.rf_fa_host_release.argtypes = []
    lib.rf_fa_host_release.restype = None
    lib.rf_host_round_bf16.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_uint16), C.c_int64]
    lib.rf_host_round_bf16.restype = C.c_int
    lib.rf_fa_host_transfer_counters.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    lib.rf_fa_host_transfer_counters.restype = None
    lib.rf_clf_config_default.argtypes = [C.POINTER(RfClfConfig)]
    lib.rf_clf_config_default.restype = None
    lib.rf_clf_weight_elems.argtypes = [C.POINTER(RfClfConfig)]
    lib.rf_clf_weight_elems.restype = C.c_size_t
    lib.rf_clf_create.argtypes = [C.POINTER(RfClfConfig), f32p, C.c_size_t, i32, C.POINTER(vp)]
    lib.rf_clf_create.restype = C.c_int
    lib.rf_clf_forward.argtypes = [vp, C.POINTER(i64), f32p, i64, i64, f32p]
    lib.rf_clf_forward.restype = C.c_int
    lib.rf_clf_session_bytes.argtypes = [vp, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
    lib.rf_clf_session_bytes.restype = C.c_int
    lib.rf_clf_last_forward_ms.argtypes = [vp]
    lib.rf_clf_last_forward_ms.restype = C.c_float
    lib.rf_clf_destroy.argtypes = [vp]
    lib.rf_clf_destroy.restype = None
    lib.rf_clf_head.argtypes = [vp, i64, i64, i32, vp, vp, vp, vp, i32, C.c_float, i32, vp, vp]
    lib.rf_clf_head.restype = C.c_int
    lib.rf_gemm_nt.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, i32, C.POINTER(RfGemmEpilogue), vp]
    lib.rf_gemm_nt.restype = C.c_int
    lib.rf_gemm_launch_status.argtypes = [vp]
    lib.rf_gemm_launch_status.restype = C.c_int
    for name in ("rf_fa_validate", "rf_fa_fwd_workspace_bytes", "rf_fa_stats_query", "rf_fa_fwd", "rf_fa_merge",
                 "rf_fa_rescale_partial", "rf_fa_normalize", "rf_pad_bias_from_mask", "rf_cast_f32_to",
                 "rf_cast_to_f32", "rf_fa_fwd_host", "rf_fused_flash_attention_op", "rf_device_check",
                 "rf_rope_qkv", "rf_add_layernorm", "rf_geglu"):
        getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a status code to the reference's exception types."""
    if rc == RF_OK:
        return
    msg = load().rf_last_error().decode(errors="replace")
    if rc == RF_ERR_SHAPE:
        raise ShapeMismatch(rc, msg)
    if rc == RF_ERR_HEAD_DIM:
        raise UnsupportedHeadDim(rc, msg)
    raise RfError(rc, msg)


def new_params() -> RfFaParams:
    p = RfFaParams()
    load().rf_fa_params_init(C.byref(p))
    return p


def host_transfer_counters():
    """(h2d_bytes, d2h_bytes, calls) of the calling thread's rf_fa_fwd_host calls so far (rf_fa_host_transfer_counters)."""
    a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
    load().rf_fa_host_transfer_counters(C.byref(a), C.byref(b), C.byref(c))
    return int(a.value), int(b.value), int(c.value)
