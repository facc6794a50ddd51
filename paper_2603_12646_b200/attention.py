"""Host-side mirror of the reference operator interface for the FusedFlashAttention path.

Same names, argument meaning and error behaviour as the reference
(proj/core/include/routefast/attention.hpp:15-61):

* :data:`kMaskValue`, :data:`kMaskThreshold`
* :class:`AttentionSpec` (scale 0 -> 1/sqrt(d); window -1 = unbounded; optional [B,1,1,S] pad_bias)
* :class:`FlashStats`
* :func:`flash_attention(q, k, v, spec, tile=64, stats=None)`
* :func:`fused_flash_attention` -- the graph op (inputs [Q,K,V,pad_bias?], attrs scale /
  window_left / window_right; reference proj/core/src/interpreter.cpp:308-318)
* :func:`pad_bias_from_mask` -- the rewriter's shared pad-bias chain (rewrite.cpp:303-318)
* :func:`local_window_attrs` -- per-layer windows (rewrite.cpp:355-361)
* :func:`mask_memory_bytes`, :func:`fa_memory_bytes` (attention.cpp:244-252)

Everything computes on the GPU through the C ABI (capi.py -> librf_fa.so).  torch is used
only for device memory and streams.  There is no CPU fallback: CPU tensors are copied to the
device by the host entry point (rf_fa_fwd_host), exactly like the reference's host Tensor call.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np
import torch

from . import capi
from .capi import ShapeMismatch, UnsupportedHeadDim  # noqa: F401  (re-exported)

kMaskValue = -65504.0       # attention.hpp:15
kMaskThreshold = -30000.0   # attention.hpp:16

_KERNELS = {"auto": capi.RF_KERNEL_AUTO, "tcgen05": capi.RF_KERNEL_TCGEN05, "simt": capi.RF_KERNEL_SIMT}
_DTYPES = {torch.bfloat16: capi.RF_DTYPE_BF16, torch.float16: capi.RF_DTYPE_F16, torch.float32: capi.RF_DTYPE_F32}


@dataclass
class AttentionSpec:
    """routefast::AttentionSpec (attention.hpp:18-25)."""
    scale: float = 0.0            # 0 -> 1/sqrt(head_dim)
    window_left: int = -1         # -1 = unbounded
    window_right: int = -1
    pad_bias: Optional[object] = None  # [B,1,1,S], 0 or -65504 per key (torch tensor or ndarray)

    def effective_scale(self, head_dim: int) -> float:
        """attention.cpp:34-36."""
        return self.scale if self.scale != 0.0 else 1.0 / math.sqrt(float(head_dim))


@dataclass
class FlashStats:
    """Scratch report of one call -- the analogue of routefast::FlashStats (attention.hpp:36-40).

    The reference reports f32 element counts of its CPU scratch; here the same three fields are
    filled with the same formulas (tile, 2*S, B*H*S*d) and the device-side byte counts are added.
    """
    tile_scratch_floats: int = 0
    row_state_floats: int = 0
    output_floats: int = 0
    workspace_bytes: int = 0
    tile_scratch_bytes: int = 0
    score_matrix_bytes: int = 0
    kernel: str = ""
    grid_ctas: int = 0


class WorkspaceAllocator:
    """Owns the O(S) device workspace the launcher needs (the launcher itself never allocates).

    One growing buffer per (device, stream); torch's caching allocator backs it.  Buffers are
    reused across calls on the same stream, so steady-state calls allocate nothing.
    """

    def __init__(self):
        self._bufs = {}

    def get(self, nbytes: int, device: torch.device, stream: torch.cuda.Stream) -> Optional[torch.Tensor]:
        if nbytes == 0:
            return None
        key = (device.index, stream.cuda_stream)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)
            self._bufs[key] = buf
        return buf

    def bytes_held(self) -> int:
        return sum(b.numel() for b in self._bufs.values())

    def clear(self) -> None:
        self._bufs.clear()


_workspaces = WorkspaceAllocator()


def _strides3(t: torch.Tensor) -> Tuple[int, int, int]:
    if t.stride(3) != 1 and t.size(3) != 1:
        raise capi.RfError(capi.RF_ERR_ARG, "last (head) dimension must be contiguous")
    return t.stride(0), t.stride(1), t.stride(2)


def _check_qkv_shapes(q, k, v) -> None:
    # attention.cpp:14-21
    if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
        raise ShapeMismatch(capi.RF_ERR_SHAPE, "attention inputs must be [B,H,S,d]")
    if q.shape != k.shape or q.shape != v.shape:
        raise ShapeMismatch(capi.RF_ERR_SHAPE, "Q, K, V must have identical shapes")


def _device_params(q, k, v, spec: AttentionSpec, out, out_dtype, kernel, flags, kv_range, partials, debug_scores):
    """rf_fa_params for one call on device tensors; returns (params, out, keep-alive list)."""
    B, H, S, d = q.shape
    if q.dtype not in (torch.bfloat16, torch.float16) or k.dtype != q.dtype or v.dtype != q.dtype:
        raise capi.RfError(capi.RF_ERR_ARG, "device q/k/v must share dtype bfloat16 or float16")
    dev = q.device
    pb = None
    if spec.pad_bias is not None:
        pb = spec.pad_bias
        if not isinstance(pb, torch.Tensor):
            pb = torch.as_tensor(np.asarray(pb, dtype=np.float32))
        if pb.dim() != 4 or tuple(pb.shape) != (B, 1, 1, S):
            raise ShapeMismatch(capi.RF_ERR_SHAPE, "pad_bias must be [B,1,1,S]")  # attention.cpp:111-116
        pb = pb.to(device=dev, dtype=torch.float32).contiguous()

    p = capi.new_params()
    p.B, p.H, p.S, p.d = B, H, S, d
    p.scale = float(spec.scale)
    p.window_left, p.window_right = int(spec.window_left), int(spec.window_right)
    p.dtype = _DTYPES[q.dtype]
    p.kernel = _KERNELS[kernel]
    p.flags = int(flags)
    for name, t in (("q", q), ("k", k), ("v", v)):
        setattr(p, name, t.data_ptr())
        sb, sh, ss = _strides3(t)
        getattr(p, name + "_stride")[:] = [sb, sh, ss if ss != 0 else d]
    if partials is not None:
        o_part, m_part, l_part = partials
        p.o_partial, p.m_partial, p.l_partial = o_part.data_ptr(), m_part.data_ptr(), l_part.data_ptr()
        p.out_dtype = capi.RF_DTYPE_F32
    else:
        if out is None:
            out = torch.empty((B, H, S, d), dtype=out_dtype or q.dtype, device=dev)
        elif tuple(out.shape) != (B, H, S, d):
            raise ShapeMismatch(capi.RF_ERR_SHAPE, "out must have the shape of Q")
        p.out = out.data_ptr()
        p.out_dtype = _DTYPES[out.dtype]
        sb, sh, ss = _strides3(out)
        p.o_stride[:] = [sb, sh, ss if ss != 0 else d]
    if pb is not None:
        p.pad_bias = pb.data_ptr()
    if kv_range is not None:
        p.kv_begin, p.kv_end = int(kv_range[0]), int(kv_range[1])
    elif partials is not None:
        p.kv_begin, p.kv_end = 0, S  # a partial takes its key range literally ([0, 0) is an empty block)
    if debug_scores is not None:
        p.debug_scores = debug_scores.data_ptr()
    return p, out, [q, k, v, pb, out, partials, debug_scores]


def _fill_stats(stats, st) -> None:
    stats.workspace_bytes = int(st.workspace_bytes)
    stats.tile_scratch_bytes = int(st.tile_scratch_bytes)
    stats.score_matrix_bytes = int(st.score_matrix_bytes)
    stats.kernel = {1: "tcgen05", 2: "simt"}.get(int(st.kernel), "?")
    stats.grid_ctas = int(st.grid_ctas)


def _device_call(q, k, v, spec: AttentionSpec, stats, out, out_dtype, kernel, flags, kv_range, partials,
                 debug_scores):
    lib = capi.load()
    dev = q.device
    p, out, _keep = _device_params(q, k, v, spec, out, out_dtype, kernel, flags, kv_range, partials, debug_scores)
    st = capi.RfFaStats()
    capi.check(lib.rf_fa_stats_query(C.byref(p), C.byref(st)))
    stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        ws = _workspaces.get(int(st.workspace_bytes), dev, stream)
        capi.check(lib.rf_fa_fwd(C.byref(p), ws.data_ptr() if ws is not None else None,
                                 ws.numel() if ws is not None else 0, stream.cuda_stream))
    if stats is not None:
        _fill_stats(stats, st)
    return out


class FaPlan:
    """rf_fa_plan (include/rf_fa.h): one call resolved once -- validation, kernel and schedule choice, workspace
    carve-up, TMA tensor maps -- and launched any number of times on the current stream with no host work
    beyond the kernel launches.  The plan owns its workspace and keeps the tensors alive; their contents may
    change between launches, their addresses may not."""

    def __init__(self, q, k, v, spec: Optional[AttentionSpec] = None, *, out: Optional[torch.Tensor] = None,
                 out_dtype: Optional[torch.dtype] = None, kernel: str = "auto", kv_range=None, partials=None,
                 workspace: Optional[torch.Tensor] = None):
        """workspace: a caller-owned uint8 CUDA tensor to carve the plan's workspace from instead of a private one
        (a session shares one between the plans of its layers; launches that share a workspace must not overlap)."""
        _check_qkv_shapes(q, k, v)
        self.lib = capi.load()
        self.device = q.device
        spec = spec or AttentionSpec()
        p, self.out, self._keep = _device_params(q, k, v, spec, out, out_dtype, kernel, 0, kv_range, partials, None)
        st = capi.RfFaStats()
        capi.check(self.lib.rf_fa_stats_query(C.byref(p), C.byref(st)))
        self.stats = FlashStats()
        _fill_stats(self.stats, st)
        nbytes = int(st.workspace_bytes)
        if workspace is not None:
            if workspace.dtype != torch.uint8 or workspace.device != self.device or workspace.numel() < nbytes:
                raise ShapeMismatch(capi.RF_ERR_WORKSPACE, f"workspace must be a uint8 tensor of >= {nbytes} bytes on {self.device}")
            self._ws = workspace
        else:
            self._ws = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device=self.device)
        self._h = C.c_void_p()
        with torch.cuda.device(self.device):
            capi.check(self.lib.rf_fa_plan_create(C.byref(p), self._ws.data_ptr() if nbytes else None, nbytes,
                                                  C.byref(self._h)))

    def launch(self) -> torch.Tensor:
        capi.check(self.lib.rf_fa_plan_launch(self._h, torch.cuda.current_stream(self.device).cuda_stream))
        return self.out

    def status(self) -> int:
        """Synchronises the current stream and returns RF_OK or RF_ERR_DEVICE_TIMEOUT (rf_fa_launch_status)."""
        if self.stats.workspace_bytes == 0:
            return capi.RF_OK
        with torch.cuda.device(self.device):
            return int(self.lib.rf_fa_launch_status(self._ws.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream))

    def close(self) -> None:
        if self._h:
            self.lib.rf_fa_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def _host_call(q, k, v, spec: AttentionSpec, tile, stats, device_index, compute_dtype):
    lib = capi.load()
    qn = np.ascontiguousarray(q, dtype=np.float32)
    kn = np.ascontiguousarray(k, dtype=np.float32)
    vn = np.ascontiguousarray(v, dtype=np.float32)
    if qn.ndim != 4 or kn.ndim != 4 or vn.ndim != 4:
        raise ShapeMismatch(capi.RF_ERR_SHAPE, "attention inputs must be [B,H,S,d]")
    if qn.shape != kn.shape or qn.shape != vn.shape:
        raise ShapeMismatch(capi.RF_ERR_SHAPE, "Q, K, V must have identical shapes")
    B, H, S, d = qn.shape
    f32p = C.POINTER(C.c_float)
    pb = None
    dims = None
    if spec.pad_bias is not None:
        pb = np.ascontiguousarray(spec.pad_bias, dtype=np.float32)
        if pb.ndim != 4:
            raise ShapeMismatch(capi.RF_ERR_SHAPE, "pad_bias must be [B,1,1,S]")
        dims = (C.c_int64 * 4)(*pb.shape)
    # page-locked result buffer from torch's caching host allocator (reused across calls once the
    # caller drops the previous result): lets the library download O chunk by chunk, overlapped
    # with the uploads; the ndarray keeps the tensor alive through its base
    if qn.size and torch.cuda.is_available():
        out = torch.empty(qn.shape, dtype=torch.float32, pin_memory=True).numpy()
    else:
        out = np.empty_like(qn)  # no device: the library call below fails loudly with RF_ERR_CUDA
    st = capi.RfFaStats()
    rc = lib.rf_fa_fwd_host(qn.ctypes.data_as(f32p), kn.ctypes.data_as(f32p), vn.ctypes.data_as(f32p),
                            out.ctypes.data_as(f32p), B, H, S, d, float(spec.scale), int(spec.window_left),
                            int(spec.window_right), pb.ctypes.data_as(f32p) if pb is not None else None, dims,
                            int(tile), compute_dtype, device_index, C.byref(st))
    capi.check(rc)
    if stats is not None:
        stats.workspace_bytes = int(st.workspace_bytes)
        stats.tile_scratch_bytes = int(st.tile_scratch_bytes)
        stats.kernel = {1: "tcgen05", 2: "simt"}.get(int(st.kernel), "?")
        stats.grid_ctas = int(st.grid_ctas)
    return out


def flash_attention(q, k, v, spec: Optional[AttentionSpec] = None, tile: int = 64,
                    stats: Optional[FlashStats] = None, *, out: Optional[torch.Tensor] = None,
                    out_dtype: Optional[torch.dtype] = None, kernel: str = "auto", flags: int = 0,
                    kv_range: Optional[Tuple[int, int]] = None, partials=None, debug_scores=None,
                    device: int = 0, compute_dtype: torch.dtype = torch.bfloat16):
    """routefast::flash_attention (attention.hpp:46-48) on the B200.

    * CUDA tensors (bf16/f16, [B,H,S,d], any batch/head/seq strides): launched asynchronously on
      the current stream; returns a CUDA tensor.
    * CPU tensors / ndarrays (f32): the reference's own calling convention -- copied to
      ``device``, computed in ``compute_dtype``, returned as an f32 ndarray/CPU tensor.

    ``tile`` is accepted for signature parity (tile < 1 raises ShapeMismatch, attention.cpp:110);
    the kernel's key tile is fixed at 128.
    """
    spec = spec or AttentionSpec()
    if tile < 1:
        raise ShapeMismatch(capi.RF_ERR_SHAPE, "tile must be >= 1")
    is_dev = isinstance(q, torch.Tensor) and q.is_cuda
    if is_dev:
        _check_qkv_shapes(q, k, v)
        B, H, S, d = q.shape
        if stats is not None:
            stats.tile_scratch_floats = int(tile)          # attention.cpp:126-130
            stats.row_state_floats = 2 * S
            stats.output_floats = B * H * S * d
        return _device_call(q, k, v, spec, stats, out, out_dtype, kernel, flags, kv_range, partials, debug_scores)
    as_torch = isinstance(q, torch.Tensor)
    if as_torch:
        _check_qkv_shapes(q, k, v)
        q, k, v = q.detach().float().numpy(), k.detach().float().numpy(), v.detach().float().numpy()
    hspec = spec
    if isinstance(spec.pad_bias, torch.Tensor):
        hspec = AttentionSpec(spec.scale, spec.window_left, spec.window_right,
                              spec.pad_bias.detach().float().cpu().numpy())
    res = _host_call(q, k, v, hspec, tile, stats, device, _DTYPES[compute_dtype])
    if stats is not None:
        B, H, S, d = res.shape
        stats.tile_scratch_floats, stats.row_state_floats, stats.output_floats = int(tile), 2 * S, B * H * S * d
    return torch.from_numpy(res) if as_torch else res


def fused_flash_attention(Q, K, V, pad_bias=None, *, scale: float = 0.0, window_left: int = -1,
                          window_right: int = -1, **kw):
    """The `FusedFlashAttention` graph op: inputs [Q, K, V, pad_bias?], attrs scale /
    window_left / window_right with the interpreter's defaults (interpreter.cpp:308-318);
    one output shaped like Q (graph.cpp:405-407)."""
    return flash_attention(Q, K, V, AttentionSpec(scale, window_left, window_right, pad_bias), **kw)


def pad_bias_from_mask(attention_mask: torch.Tensor) -> torch.Tensor:
    """pad_bias = Cast_f16(-65504 * (1 - attention_mask)) on device (rewrite.cpp:303-318)."""
    lib = capi.load()
    m = attention_mask.to(dtype=torch.float32).contiguous()
    if not m.is_cuda:
        raise capi.RfError(capi.RF_ERR_ARG, "pad_bias_from_mask expects a CUDA tensor")
    out = torch.empty_like(m)
    with torch.cuda.device(m.device):
        capi.check(lib.rf_pad_bias_from_mask(m.data_ptr(), out.data_ptr(), m.numel(),
                                             torch.cuda.current_stream(m.device).cuda_stream))
    return out


@dataclass
class RewriteOptions:
    """routefast::RewriteOptions defaults (rewrite.hpp:49-53)."""
    head_dim: int = 64
    local_window: int = 128
    mask_input: str = "attention_mask"


def local_window_attrs(options: RewriteOptions = RewriteOptions(), is_global: bool = False) -> Tuple[int, int]:
    """Per-layer window attrs the rewriter assigns (rewrite.cpp:266-272,355-361)."""
    if options.head_dim not in (32, 64, 128):
        raise UnsupportedHeadDim(capi.RF_ERR_HEAD_DIM,
                                 f"head_dim must be one of {{32, 64, 128}}, got {options.head_dim}")
    if options.local_window < 2 or options.local_window % 2 != 0:
        raise ValueError("local_window must be even and >= 2")
    if is_global:
        return -1, -1
    return options.local_window // 2 - 1, options.local_window // 2


def mask_memory_bytes(batch: int, heads: int, seq_len: int, bytes_per_element: int) -> int:
    return int(capi.load().rf_mask_memory_bytes(batch, heads, seq_len, bytes_per_element))


def fa_memory_bytes(batch: int, heads: int, seq_len: int, head_dim: int, tile: int, bytes_per_element: int) -> int:
    return int(capi.load().rf_fa_memory_bytes(batch, heads, seq_len, head_dim, tile, bytes_per_element))
