"""Split-KV attention for ONE long sequence across the GPUs of a box (BASELINE config 4,
SURVEY.md 8(e)): Q is replicated, the keys/values are cut into `world_size` contiguous blocks,
each rank runs the forward kernel over its block for all queries and emits un-normalised
partials (O~, m, l); the online-softmax state is associative, so one exchange step finishes it:

    m* = allreduce_max(m)            (1.5 MB at S = 32K, H = 12)
    O~ <- O~ * 2^(m - m*), l <- l * 2^(m - m*)          rf_fa_rescale_partial
    [O~ | l] <- reduce_scatter_sum                       (NCCL over NVLink; ~102 MB fp32 at 32K)
    O = O~ / l, 0 where l == 0                           rf_fa_normalize

This is the same algebra as the per-tile update of the reference (attention.cpp:177-196).
Rows with no live key in a block carry m = -inf, l = 0.  The compute steps are injected through
an ops object so that the host logic (partitioning, collective sequence) is testable on CPU
with gloo; the default ops are the CUDA kernels -- there is no CPU implementation here.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import torch
import torch.distributed as dist

from . import capi
from .attention import AttentionSpec, flash_attention

KEY_TILE = 128  # block boundaries are aligned to the kernel's key tile


def kv_block(S: int, rank: int, world: int, align: int = KEY_TILE) -> Tuple[int, int]:
    """Key range [begin, end) of `rank`: contiguous, disjoint, covering [0, S), tile-aligned
    except for the sequence end.  Blocks may be empty when S < world * align."""
    n_tiles = (S + align - 1) // align
    t0 = n_tiles * rank // world
    t1 = n_tiles * (rank + 1) // world
    return min(t0 * align, S), min(t1 * align, S)


class CudaSplitKVOps:
    """The three compute steps on the GPU through the C ABI."""

    def partial(self, q, k, v, spec: AttentionSpec, kv_range):
        B, H, S, d = q.shape
        o = torch.empty((B, H, S, d), device=q.device, dtype=torch.float32)
        m = torch.empty((B, H, S), device=q.device, dtype=torch.float32)
        l = torch.empty((B, H, S), device=q.device, dtype=torch.float32)
        # an empty block yields the neutral element of the merge (m = -inf, l = 0, O = 0) inside the library
        flash_attention(q, k, v, spec, kv_range=kv_range, partials=(o, m, l))
        return o, m, l

    def rescale(self, o, l, m, m_star):
        lib = capi.load()
        rows, d = m.numel(), o.shape[-1]
        with torch.cuda.device(o.device):
            capi.check(lib.rf_fa_rescale_partial(o.data_ptr(), l.data_ptr(), m.data_ptr(), m_star.data_ptr(), rows, d,
                                                 torch.cuda.current_stream(o.device).cuda_stream))

    def normalize(self, o_sum, l_sum, out_dtype):
        lib = capi.load()
        rows, d = l_sum.numel(), o_sum.shape[-1]
        out = torch.empty(o_sum.shape, device=o_sum.device, dtype=out_dtype)
        dt = {torch.bfloat16: capi.RF_DTYPE_BF16, torch.float16: capi.RF_DTYPE_F16, torch.float32: capi.RF_DTYPE_F32}[out_dtype]
        with torch.cuda.device(o_sum.device):
            capi.check(lib.rf_fa_normalize(o_sum.data_ptr(), l_sum.data_ptr(), rows, d, out.data_ptr(), dt,
                                           torch.cuda.current_stream(o_sum.device).cuda_stream))
        return out


def merge_partials_local(parts, out_dtype=torch.float32):
    """Fixed-order merge of G partials held on ONE device (rf_fa_merge) -- the all-gather variant
    and the single-GPU check of the algebra."""
    lib = capi.load()
    G = len(parts)
    o0 = parts[0][0]
    rows, d = parts[0][1].numel(), o0.shape[-1]
    out = torch.empty(o0.shape, device=o0.device, dtype=out_dtype)
    vp = C.c_void_p
    op = (vp * G)(*[p[0].data_ptr() for p in parts])
    mp = (vp * G)(*[p[1].data_ptr() for p in parts])
    lp = (vp * G)(*[p[2].data_ptr() for p in parts])
    dt = {torch.bfloat16: capi.RF_DTYPE_BF16, torch.float16: capi.RF_DTYPE_F16, torch.float32: capi.RF_DTYPE_F32}[out_dtype]
    with torch.cuda.device(o0.device):
        capi.check(lib.rf_fa_merge(op, mp, lp, G, rows, d, out.data_ptr(), dt,
                                   torch.cuda.current_stream(o0.device).cuda_stream))
    return out


def split_kv_attention(q, k, v, spec: Optional[AttentionSpec] = None, *, group=None, ops=None,
                       out_dtype=torch.float32, gather: bool = True):
    """Collective call: every rank of `group` passes the same Q/K/V (only its key block of K/V
    is read).  Returns the full [B,H,S,d] output on every rank when `gather`, else this rank's
    slice of the flattened (B*H*S) rows as (row_begin, row_end, tensor)."""
    spec = spec or AttentionSpec()
    ops = ops or CudaSplitKVOps()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B, H, S, d = q.shape
    o, m, l = ops.partial(q, k, v, spec, kv_block(S, rank, world))

    # 1. global row max, 2. rescale the local partial to it
    m_star = m.clone()
    dist.all_reduce(m_star, op=dist.ReduceOp.MAX, group=group)
    ops.rescale(o, l, m, m_star)

    # 3. sum of [O~ | l] over ranks; each rank keeps rows [r0, r1) of the flattened B*H*S rows
    rows = B * H * S
    per = (rows + world - 1) // world
    r0, r1 = min(rank * per, rows), min((rank + 1) * per, rows)
    packed = torch.cat([o.reshape(rows, d), l.reshape(rows, 1)], dim=1)  # [rows, d+1]
    backend = dist.get_backend(group)
    if backend == "nccl" and rows % world == 0:
        mine = torch.empty((per, d + 1), device=packed.device, dtype=packed.dtype)
        dist.reduce_scatter_tensor(mine, packed, op=dist.ReduceOp.SUM, group=group)
    else:  # gloo (CPU tests) has no reduce_scatter; ragged row counts take the same route
        dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
        mine = packed[r0:r1]
    o_sum = mine[:, :d].contiguous()
    l_sum = mine[:, d].contiguous()

    # 4. normalise the owned rows
    out_local = ops.normalize(o_sum, l_sum, out_dtype)
    if not gather:
        return r0, r1, out_local
    if rows % world == 0:
        full = torch.empty((rows, d), device=out_local.device, dtype=out_local.dtype)
        dist.all_gather_into_tensor(full, out_local, group=group)
    else:
        pad = torch.zeros((per, d), device=out_local.device, dtype=out_local.dtype)
        pad[: r1 - r0] = out_local
        chunks = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(chunks, pad, group=group)
        full = torch.cat(chunks, dim=0)[:rows]
    return full.reshape(B, H, S, d)
