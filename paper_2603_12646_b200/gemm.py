"""Python mirror of include/rf_gemm.h: the hand-written sm_100a projection y = a @ w^T with the encoder's
element-wise steps (RoPE on the packed QKV projection, GeGLU on the MLP up-projection) fused into its epilogue.
torch is used for device memory and streams only; the product path is librf_fa.so (no cuBLAS, no fallback)."""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from . import capi


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return capi.RF_DTYPE_BF16
    if t.dtype == torch.float16:
        return capi.RF_DTYPE_F16
    raise capi.RfError(capi.RF_ERR_ARG, f"rf_gemm_nt takes bf16 or f16 operands, got {t.dtype}")


def gemm_nt(a: torch.Tensor, w: torch.Tensor, out: Optional[torch.Tensor] = None, *, epilogue: str = "none",
            rope_cos: Optional[torch.Tensor] = None, rope_sin: Optional[torch.Tensor] = None,
            seq_len: int = 0, out_dtype: Optional[torch.dtype] = None, head_major: bool = False) -> torch.Tensor:
    """y = epilogue(a @ w.T).  a [M, K], w [N, K] (nn.Linear layout), 16-bit, last dim contiguous (row strides may be
    larger than the row).  epilogue: "none" | "rope" (w = packed QKV projection [3*hidden, K], cos/sin [S, 32] f32,
    token t at position t % seq_len; head_major=True returns [3*H, M, 64] -- every head's rows contiguous -- instead of
    the packed [M, 3*H*64]) | "geglu" (w = [2*I, K]: y [M, I] = gelu(a w_in^T) * (a w_gate^T)) |
    "residual" (out is the f32 residual stream [M, N], required: out += a @ w.T)."""
    lib = capi.load()
    if not a.is_cuda:
        raise capi.RfError(capi.RF_ERR_CUDA, "rf_gemm_nt needs CUDA tensors (there is no CPU path)")
    M, K = a.shape
    N = w.shape[0]
    assert w.shape[1] == K and a.stride(1) == 1 and w.stride(1) == 1 and w.dtype == a.dtype
    kind = {"none": capi.RF_GEMM_EPI_NONE, "rope": capi.RF_GEMM_EPI_ROPE, "geglu": capi.RF_GEMM_EPI_GEGLU,
            "residual": capi.RF_GEMM_EPI_RESIDUAL}[epilogue]
    n_out = N // 2 if kind == capi.RF_GEMM_EPI_GEGLU else N
    out_code = 0
    if out_dtype is not None and out_dtype != a.dtype:      # "rope" only: Q/K/V in the other 16-bit type
        assert kind == capi.RF_GEMM_EPI_ROPE and out_dtype in (torch.bfloat16, torch.float16)
        out_code = 1 + (capi.RF_DTYPE_BF16 if out_dtype == torch.bfloat16 else capi.RF_DTYPE_F16)
    out_dtype = torch.float32 if kind == capi.RF_GEMM_EPI_RESIDUAL else (out_dtype or a.dtype)
    if head_major:
        assert kind == capi.RF_GEMM_EPI_ROPE
        if out is None:
            out = torch.empty((N // 64, M, 64), device=a.device, dtype=out_dtype)
        assert out.shape == (N // 64, M, 64) and out.is_contiguous() and out.dtype == out_dtype
    else:
        if out is None:
            assert kind != capi.RF_GEMM_EPI_RESIDUAL, "the residual epilogue accumulates into `out`"
            out = torch.empty((M, n_out), device=a.device, dtype=out_dtype)
        assert out.shape == (M, n_out) and out.stride(1) == 1 and out.dtype == out_dtype
    epi = capi.RfGemmEpilogue(kind=kind, head_dim=64, S=seq_len, out_dtype=out_code, head_major=int(head_major),
                              cos_table=rope_cos.data_ptr() if rope_cos is not None else None,
                              sin_table=rope_sin.data_ptr() if rope_sin is not None else None)
    with torch.cuda.device(a.device):
        capi.check(lib.rf_gemm_nt(a.data_ptr(), w.data_ptr(), out.data_ptr(), M, N, K, a.stride(0), w.stride(0),
                                  0 if head_major else out.stride(0), _dtype_code(a), C.byref(epi), torch.cuda.current_stream(a.device).cuda_stream))
    return out
