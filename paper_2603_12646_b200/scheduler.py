"""Batch scheduler: spreads concurrent classifier requests over the GPUs of one box
(BASELINE configs 3 and 5).

Units are whole (classifier, request) forwards -- every request and every (batch, head) is
independent in the operator (reference attention.cpp:138-142), so weights are replicated,
units are sharded, and NO data-path collective is needed: the only exchange is a host-side
gather of the [n_req, n_labels] logits.  Assignment is LPT (longest processing time first) on a
cost model of the attention work, which is what dominates at 8K-32K tokens.

The scheduler is pure host logic; the per-unit work is a callable, so the N > 1 path is covered
by world_size-2 gloo tests on CPU (tests/test_multi_gpu_host_logic.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Callable, Dict, List, Optional, Sequence

import torch.distributed as dist


@dataclass(frozen=True)
class Unit:
    """One schedulable forward: classifier `model` on request `request` of `seq_len` tokens."""
    uid: int
    model: str
    request: int
    seq_len: int
    valid_len: Optional[int] = None  # unpadded tokens (tail padding), None = seq_len


@dataclass
class ModelShape:
    """What the cost model needs from a ModernBERT-style encoder."""
    n_layers: int = 22
    global_every: int = 3        # layer i is global iff i % global_every == 0
    local_window: int = 128      # RewriteOptions.local_window (rewrite.hpp:51)
    heads: int = 12
    head_dim: int = 64
    hidden: int = 768
    mlp: int = 1152


def attention_flops(seq_len: int, valid_len: Optional[int], shape: ModelShape) -> float:
    """Algorithmic attention FLOPs of one forward: 4*d*H*sum(live pairs) per layer."""
    live_keys = seq_len if valid_len is None else valid_len
    n_global = len([i for i in range(shape.n_layers) if i % shape.global_every == 0])
    n_local = shape.n_layers - n_global
    g = 4.0 * shape.head_dim * shape.heads * seq_len * live_keys
    loc = 4.0 * shape.head_dim * shape.heads * seq_len * min(shape.local_window, live_keys)
    return n_global * g + n_local * loc


def unit_cost(u: Unit, shape: ModelShape) -> float:
    """Attention work plus the GEMM work of the encoder (QKV/out projections and the GLU MLP)."""
    gemm = 2.0 * u.seq_len * shape.n_layers * (4 * shape.hidden * shape.hidden + 3 * shape.hidden * shape.mlp)
    return attention_flops(u.seq_len, u.valid_len, shape) + gemm


def lpt_assign(units: Sequence[Unit], n_ranks: int, shape: Optional[ModelShape] = None) -> List[List[Unit]]:
    """Longest-processing-time-first assignment; deterministic (ties broken by uid, then rank)."""
    shape = shape or ModelShape()
    loads = [0.0] * n_ranks
    out: List[List[Unit]] = [[] for _ in range(n_ranks)]
    for u in sorted(units, key=lambda x: (-unit_cost(x, shape), x.uid)):
        r = min(range(n_ranks), key=lambda i: (loads[i], i))
        out[r].append(u)
        loads[r] += unit_cost(u, shape)
    return out


def makespan(assignment: Sequence[Sequence[Unit]], shape: Optional[ModelShape] = None) -> float:
    shape = shape or ModelShape()
    return max((sum(unit_cost(u, shape) for u in units) for units in assignment), default=0.0)


@dataclass
class BatchScheduler:
    """run(): every rank computes its share with `run_unit` and rank 0 receives all results.

    A unit that raises is re-queued once on the same rank (replicas are stateless, SURVEY 5
    failure row); a second failure is reported in the result instead of killing the batch.
    """
    shape: ModelShape = field(default_factory=ModelShape)

    def run(self, units: Sequence[Unit], run_unit: Callable[[Unit], Any], group=None) -> Optional[Dict[int, Any]]:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        mine = lpt_assign(units, world, self.shape)[rank]
        local: Dict[int, Any] = {}
        for u in mine:
            try:
                local[u.uid] = run_unit(u)
            except Exception:  # noqa: BLE001  (retry once, then surface)
                try:
                    local[u.uid] = run_unit(u)
                except Exception as e2:  # noqa: BLE001
                    local[u.uid] = {"error": repr(e2)}
        if world == 1:
            return local
        gathered = [None] * world if rank == 0 else None
        dist.gather_object(local, gathered, dst=0, group=group)  # host-side gather of the logits
        if rank != 0:
            return None
        merged: Dict[int, Any] = {}
        for part in gathered:
            merged.update(part)
        return merged
