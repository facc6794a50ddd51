#!/usr/bin/env python
"""bench.py -- headline benchmark of the FusedFlashAttention hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload op8k|config3|config4|config5]

With --gpus N > 1 and no torchrun environment (WORLD_SIZE unset) this script starts the N ranks
itself (python -m torch.distributed.run, one process per GPU, NCCL, rendezvous on 127.0.0.1).

Metric (BASELINE.json): attention forward TFLOP/s on the ModernBERT-base 8K global-attention
op (B=1, H=12, S=8192, d=64, no padding) -- configs[1]'s attention layer.  One step = one pass
of the op over one batch of synthetic bf16 inputs.  FLOPs are ALGORITHMIC: 4*d*H*sum(live
pairs) = 206.16 GFLOP per step.

  value     inputs resident in HBM, CUDA events on the launch stream, exactly K back-to-back
            steps rotating over input sets whose total footprint exceeds L2 (no flush needed).
  e2e       the same op through the reference-facing host entry point (rf_fa_fwd_host via
            flash_attention on host arrays): pinned f32 host tensors in, f32 host tensor out,
            H2D + casts + kernel + D2H inside the timed region.
  roofline  tensor-core bound; peak from MEASURED_PEAKS.json.
  cpu_baseline / --impl reference
            the reference's own CPU operator (oracle/_ref, else the C port) on the host cores.

N > 1: independent request shards per rank, no data-path collective (weak scaling); device-timed,
max over ranks.

Workloads (BASELINE.json configs; `config.workload` in the JSON line names the one that ran):
  op8k     (default) the headline metric: the 8K global attention op, one op per rank per step
  config3  3 classifiers (safety / domain / PII) x batch 4 at S=16384 = 12 (classifier, request) units
           sharded over the ranks by BatchScheduler (LPT), host-side gather of logits; requests/s
  config4  ONE 32K sequence, K/V split into N contiguous key blocks, softmax-merge over NCCL
           (split_kv_attention); strong scaling, attention TFLOP/s
  config5  request-throughput sweep, S in 512..32K x batch 1..64 with variable-length padding masks,
           requests sharded over the ranks; requests/s
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

B, H, S, D = 1, 12, 8192, 64
METRIC = "attention_fwd_tflops"
UNIT = "TFLOP/s"
WORKLOAD = "ModernBERT-base global attention op, B=1 H=12 S=8192 d=64 (configs[1] attention layer), non-causal, no padding"


def flops_global(b, h, s, d):
    return 4.0 * b * h * s * s * d


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            pk = json.load(f)
        return {"bf16": pk["bf16_tflops"], "bf16_sustained": pk.get("bf16_tflops_sustained"), "hbm": pk["hbm_gbs"],
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"bf16": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if bits & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thr is not None:
            self._thr.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


# --------------------------------------------------------------------------------------------
# CPU arm: the reference operator on the host cores (test infrastructure used as the baseline)
# --------------------------------------------------------------------------------------------
def cpu_reference_run(steps, warmup, budget_s):
    """Times routefast::flash_attention on the bench workload (all queries x all keys): one step = `heads` heads
    of the 12 (every head is an independent unit of the op, attention.cpp:138-142), one thread per head because
    the operator itself is single-threaded; heads = min(host cores, 12).  The sequence length is the stated
    S = 8192 whenever steps + warmup such steps fit budget_s (calibrated on one S = 1024 head first; ~5-8 s per
    step on the bench hosts, so the driver's K = 20, W = 5 fits); only if they cannot, S is halved until they do,
    and the line says so."""
    import numpy as np

    import oracle as O
    kind = "reference" if O.have_reference() else "port"
    host_cores = os.cpu_count() or 1
    heads = max(1, min(host_cores, H))
    rng = np.random.default_rng(0)
    cal = [rng.uniform(-1, 1, (1, heads, 1024, D)).astype(np.float32) for _ in range(3)]
    t0 = time.perf_counter()
    O.flash_attention(*cal, 0.0, -1, -1, None, threads=heads, impl=kind)
    t_1k = time.perf_counter() - t0
    per_step = budget_s / max(1, steps + warmup)
    s_sample = S
    while s_sample > 1024 and t_1k * (s_sample / 1024.0) ** 2 > per_step:
        s_sample //= 2
    q, k, v = [rng.uniform(-1, 1, (1, heads, s_sample, D)).astype(np.float32) for _ in range(3)]
    for _ in range(warmup):
        O.flash_attention(q, k, v, 0.0, -1, -1, None, threads=heads, impl=kind)
    t0 = time.perf_counter()
    for _ in range(steps):
        O.flash_attention(q, k, v, 0.0, -1, -1, None, threads=heads, impl=kind)
    dt = (time.perf_counter() - t0) / max(1, steps)
    tflops = flops_global(1, heads, s_sample, D) / dt / 1e12
    sample = (f"{heads} of {H} heads x S={s_sample} per step (all queries x all keys), one thread per head; "
              f"{steps} step(s), {warmup} warm-up; host has {host_cores} cores")
    return {"value": tflops, "unit": UNIT, "cores": heads, "host_cores": host_cores, "kind": kind, "sample": sample,
            "seq_len": s_sample, "same_config": s_sample == S}, dt


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb, dt = cpu_reference_run(args.steps, args.warmup, budget_s=330.0)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "seq_len_timed": cb["seq_len"], "same_config": cb["same_config"],
                       "note": "reference CPU operator, f32 storage / f64 arithmetic"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------------
def time_op(torch, P, sets, spec, steps, warmup, out_sets, settle_s=0.0):
    """One rf_fa_plan per input set (include/rf_fa.h: validation, schedule, workspace carve-up and TMA tensor maps are
    resolved once, as a session does for its layers), then exactly `steps` plan launches on the current stream."""
    from paper_2603_12646_b200.attention import FaPlan
    n = len(sets)
    plans = [FaPlan(*sets[i], spec, out=out_sets[i]) for i in range(n)]
    # setup, not a step: every plan is launched twice as it is created (a plan's first launches pay for the memset of
    # its split-pair flags and the first fetch of its tensor maps and workspace; with 6 plans and W = 5 the sixth
    # plan would otherwise be launched for the first time inside the timed region)
    for pl in plans:
        pl.launch()
        pl.launch()
    torch.cuda.synchronize()
    if settle_s > 0:
        time.sleep(settle_s)  # sweep entries: let the board's power controller relax after the previous entry's load
    for i in range(warmup):
        plans[i % n].launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        plans[i % n].launch()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps  # ms per step
    if any(pl.status() != 0 for pl in plans):
        raise RuntimeError("a bounded wait inside an attention kernel timed out during the timed region")
    for pl in plans:
        pl.close()
    return ms


def time_op_graph(torch, P, sets, spec, replays, out_sets):
    """Device time per op for kernels too short to time through per-call host launches (the local
    layer runs ~20 us, the Python call path costs more): one pass over the rotating input sets is
    captured in a CUDA graph and replayed."""
    n = len(sets)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for i in range(n):
            P.flash_attention(*sets[i], spec, out=out_sets[i])
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(n):
            P.flash_attention(*sets[i], spec, out=out_sets[i])
    g.replay()
    torch.cuda.synchronize()
    time.sleep(0.5)  # burst regime, like every sweep entry (see the sweep's note)
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(replays):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (replays * n)  # ms per op


def make_sets(torch, b, h, s, d, n_sets, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    sets, outs = [], []
    for _ in range(n_sets):
        sets.append(tuple((torch.rand((b, h, s, d), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
                          for _ in range(3)))
        outs.append(torch.empty((b, h, s, d), device="cuda", dtype=torch.bfloat16))
    return sets, outs


class Ctx:
    """Per-rank context: torch, the package, the process group (None at world size 1)."""

    def __init__(self):
        import torch

        import paper_2603_12646_b200 as P
        from paper_2603_12646_b200 import capi
        self.torch, self.P = torch, P
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        if not torch.cuda.is_available():
            raise RuntimeError("bench.py needs a CUDA device (no CPU fallback exists)")
        if self.local_rank >= torch.cuda.device_count():
            raise RuntimeError(f"rank {self.rank}: local rank {self.local_rank} has no GPU "
                               f"({torch.cuda.device_count()} visible)")
        torch.cuda.set_device(self.local_rank)
        capi.load(build_if_missing=False)  # the CUDA extension must be there: fail loudly otherwise
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local_rank))
            self.dist = dist
        self.peaks = load_peaks()

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x: float) -> float:
        if self.dist is None:
            return x
        t = self.torch.tensor([x], device="cuda", dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist is not None:
            self.dist.barrier()
            self.dist.destroy_process_group()


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` outside torchrun: start the N ranks here (one process per GPU, NCCL)."""
    import socket
    import subprocess

    import torch
    ndev = torch.cuda.device_count()
    if ndev < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but only {ndev} CUDA device(s) are visible",
                          "n_gpus": args.gpus}), flush=True)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_ours(args):
    import numpy as np

    ctx = Ctx()
    torch, P, dist = ctx.torch, ctx.P, ctx.dist
    rank, world, local_rank = ctx.rank, ctx.world, ctx.local_rank
    barrier = ctx.barrier
    if args.workload != "op8k":
        {"config3": run_config3, "config4": run_config4, "config5": run_config5}[args.workload](args, ctx)
        ctx.close()
        return

    peaks = ctx.peaks
    spec = P.AttentionSpec()  # global, scale 1/sqrt(d)
    # inputs larger than L2: each set is 4 tensors x 12.6 MB = 50 MB; 6 sets = 302 MB > 126 MB L2
    n_sets = 6
    sets, outs = make_sets(torch, B, H, S, D, n_sets, seed=1234 + rank)
    st = P.FlashStats()
    P.flash_attention(*sets[0], spec, out=outs[0], stats=st)
    if st.kernel != "tcgen05":
        raise RuntimeError(f"expected the tcgen05 kernel, got {st.kernel}")

    # the units of one step: one 8K request per rank (weak scaling), dealt by the batch scheduler's LPT rule
    from paper_2603_12646_b200.scheduler import Unit, lpt_assign
    mine = lpt_assign([Unit(uid=i, model="attention8k", request=i, seq_len=S) for i in range(world)], world)[rank]
    assert len(mine) == 1
    barrier()
    with ClockSampler(local_rank) as clk:
        ms = time_op(torch, P, sets, spec, args.steps, args.warmup, outs)
    barrier()
    ms = ctx.max_over_ranks(ms)
    flops = flops_global(B, H, S, D)
    value = world * flops / (ms * 1e-3) / 1e12

    # ---- e2e: host f32 tensors through the reference-facing entry point ----
    e2e_steps = max(1, min(args.steps, 30))
    host = [torch.empty((B, H, S, D), dtype=torch.float32, pin_memory=True) for _ in range(3)]
    for t_, src in zip(host, sets[0]):
        t_.copy_(src.float())
    hq, hk, hv = [t_.numpy() for t_ in host]
    out_h = None
    for _ in range(6):  # same hold-the-previous-result pattern as the timed loop: both page-locked result
        out_h = P.flash_attention(hq, hk, hv, spec, device=local_rank)  # buffers exist before timing starts
    barrier()
    from paper_2603_12646_b200 import capi as _capi
    xfer0 = _capi.host_transfer_counters()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        out_h = P.flash_attention(hq, hk, hv, spec, device=local_rank)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    xfer1 = _capi.host_transfer_counters()
    barrier()
    e2e_s = ctx.max_over_ranks(e2e_s)
    e2e_val = world * flops / e2e_s / 1e12
    n_el = B * H * S * D
    assert np.isfinite(out_h).all()

    if rank == 0:
        extra = {}
        if not args.quick:
            # Every sweep entry is a burst measurement like the headline: half a second of idle before its warm-up steps,
            # so that an entry is not timed under the power cap the previous entry's load left behind (the head_dim-128
            # kernel lost 15 % that way)
            extra["note"] = "each entry: set-up launches, 0.5 s idle, 3 warm-up steps, then the timed steps (burst regime)"
            # the other sequence lengths of the metric, and the HBM-bound local layer
            for s2, it in ((16384, 10), (32768, 5)):
                sets2, outs2 = make_sets(torch, B, H, s2, D, 3 if s2 == 16384 else 2, seed=7)
                ms2 = time_op(torch, P, sets2, spec, it, 3, outs2, settle_s=0.5)
                f2 = flops_global(B, H, s2, D)
                extra[f"S{s2}"] = {"ms": ms2, "tflops": f2 / ms2 / 1e9, "frac_of_peak": f2 / ms2 / 1e9 / peaks["bf16"]}
                del sets2, outs2
            # the other head dims of the reference contract (rewrite.cpp:266-269) at the same 8K shape
            for d2 in (32, 128):
                sets_d, outs_d = make_sets(torch, B, H, S, d2, 4, seed=11)
                ms_d = time_op(torch, P, sets_d, spec, 20, 3, outs_d, settle_s=0.5)
                f_d = flops_global(B, H, S, d2)
                extra[f"S8192_d{d2}"] = {"ms": ms_d, "tflops": f_d / ms_d / 1e9, "frac_of_peak": f_d / ms_d / 1e9 / peaks["bf16"],
                                         "kernel": "fa_fwd_sm100_kernel (zero-padded to 64)" if d2 == 32 else "fa_fwd_sm100_d128_kernel"}
                del sets_d, outs_d
            # head_dim 128 at 16K tokens (the tensor-bound case of the contract's head dims)
            sets_d, outs_d = make_sets(torch, B, H, 16384, 128, 2, seed=13)
            ms_d = time_op(torch, P, sets_d, spec, 10, 3, outs_d, settle_s=0.5)
            f_d = flops_global(B, H, 16384, 128)
            extra["S16384_d128"] = {"ms": ms_d, "tflops": f_d / ms_d / 1e9, "frac_of_peak": f_d / ms_d / 1e9 / peaks["bf16"],
                                    "kernel": "fa_fwd_sm100_d128_kernel"}
            del sets_d, outs_d
            wl, wr = P.local_window_attrs()
            msl = time_op_graph(torch, P, sets, P.AttentionSpec(0.0, wl, wr), 20, outs)
            bytes_l = 4.0 * B * H * S * D * 2
            extra["S8192_local_63_64"] = {"ms": msl, "gbs": bytes_l / msl / 1e6, "frac_of_hbm": bytes_l / msl / 1e6 / peaks["hbm"],
                                          "bound": "hbm", "kernel": "fa_fwd_sm100_local_kernel",
                                          "timing": "CUDA-graph replay over the 6 rotating input sets"}
            sets4, outs4 = make_sets(torch, 4, H, 16384, D, 2, seed=9)
            ms4 = time_op_graph(torch, P, sets4, P.AttentionSpec(0.0, wl, wr), 10, outs4)
            bytes4 = 4.0 * 4 * H * 16384 * D * 2
            extra["S16384_B4_local_63_64"] = {"ms": ms4, "gbs": bytes4 / ms4 / 1e6, "frac_of_hbm": bytes4 / ms4 / 1e6 / peaks["hbm"],
                                              "bound": "hbm"}
            del sets4, outs4
            # the projections either side of the op (rf_gemm_nt, include/rf_gemm.h) at the 8K-token shapes of the encoder
            try:
                from paper_2603_12646_b200.classifier import rope_tables
                from paper_2603_12646_b200.gemm import gemm_nt
                cos_t, sin_t = rope_tables(S, 64, 10000.0, "cuda")
                for name, n_, k_, epi in (("qkv_rope", 2304, 768, "rope"), ("out_proj_residual", 768, 768, "residual"),
                                          ("mlp_up_geglu", 2304, 768, "geglu"), ("mlp_down_residual", 768, 1152, "residual")):
                    ga = torch.randn(S, k_, device="cuda").to(torch.bfloat16)
                    gw = (torch.randn(n_, k_, device="cuda") * 0.05).to(torch.bfloat16)
                    gy = torch.zeros(S, n_ // 2 if epi == "geglu" else n_, device="cuda",
                                     dtype=torch.float32 if epi == "residual" else torch.bfloat16)
                    kw = dict(rope_cos=cos_t, rope_sin=sin_t, seq_len=S) if epi == "rope" else {}
                    for _ in range(3):
                        gemm_nt(ga, gw, out=gy, epilogue=epi, **kw)
                    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    g0.record()
                    for _ in range(20):
                        gemm_nt(ga, gw, out=gy, epilogue=epi, **kw)
                    g1.record()
                    torch.cuda.synchronize()
                    gms = g0.elapsed_time(g1) / 20
                    extra[f"gemm_{name}_M8192_N{n_}_K{k_}"] = {"ms": gms, "tflops": 2.0 * S * n_ * k_ / gms / 1e9,
                                                             "frac_of_peak": 2.0 * S * n_ * k_ / gms / 1e9 / peaks["bf16"],
                                                             "kernel": "gemm_nt_sm100_kernel (tcgen05, CTA-pair multicast, fused epilogue)"}
                    del ga, gw, gy
            except Exception as e:  # noqa: BLE001
                extra["gemm_error"] = repr(e)[:200]
            # classifier forward (configs[1]): ModernBERT-base shape, B=1, S=8192, random-init weights
            try:
                from paper_2603_12646_b200.classifier import Classifier, ClassifierConfig, init_weights
                ccfg = ClassifierConfig()
                clf = Classifier(ccfg, init_weights(ccfg, 7), torch.device("cuda", local_rank))
                ids = torch.randint(0, ccfg.vocab_size, (1, S), device="cuda")
                run = clf.capture(1, S, with_mask=False)
                for _ in range(3):
                    run(ids)
                torch.cuda.synchronize()
                c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                c0.record()
                for _ in range(10):
                    lg = run(ids)
                c1.record()
                torch.cuda.synchronize()
                clf.forward(ids, None, time_layers=True)
                lm = clf.last_layer_ms
                extra["classifier_fwd_S8192_B1"] = {
                    "ms_per_request": c0.elapsed_time(c1) / 10, "layers": ccfg.n_layers,
                    "attention_ms_total": sum(x["attention_ms"] for x in lm),
                    "global_attention_ms_avg": sum(x["attention_ms"] for x in lm if x["global"]) / max(1, sum(1 for x in lm if x["global"])),
                    "local_attention_ms_avg": sum(x["attention_ms"] for x in lm if not x["global"]) / max(1, sum(1 for x in lm if not x["global"])),
                    "weights_MB": clf.weight_bytes() / 1e6, "cuda_graph": True, "projections": ccfg.gemm + " (rf_gemm_nt, no library GEMM on the path)",
                    "paper_mi300x_ms": 105.0, "note": "random-init weights, synthetic token ids; paper number is other hardware (PAPER.md:402)"}
                del clf, run
                # the same forward through the native session (rf_clf.h): host token ids in, host logits out,
                # this library's kernels only (projections included), no Python between the launches
                from paper_2603_12646_b200.classifier import NativeClassifier
                nat = NativeClassifier(ccfg, init_weights(ccfg, 7), device=local_rank)
                ids_h = ids.cpu()
                for _ in range(3):
                    nat.forward(ids_h)
                t_n = time.perf_counter()
                dev_ms = []
                for _ in range(10):
                    nat.forward(ids_h)
                    dev_ms.append(nat.last_forward_ms)
                wall_ms = (time.perf_counter() - t_n) / 10 * 1e3
                wb, ab = nat.session_bytes()
                extra["classifier_native_S8192_B1"] = {
                    "ms_per_request_wall": wall_ms, "ms_per_request_device": sorted(dev_ms)[len(dev_ms) // 2],
                    "api": "rf_clf_forward(host ids) -> host logits", "weights_MB": wb / 1e6, "arena_MB": ab / 1e6}
                nat.close()
            except Exception as e:  # noqa: BLE001
                extra.setdefault("classifier_fwd_S8192_B1", {"error": repr(e)[:200]})
                extra["classifier_error"] = repr(e)[:200]
        # DRAM traffic per launch cannot be counted inside an untraced run: it is the dram__bytes_read.sum +
        # dram__bytes_write.sum of the committed `ncu --set full` capture of this same kernel and shape
        traffic, traffic_source = None, None
        prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
        if os.path.exists(prof):
            try:
                with open(prof) as f:
                    rec = json.load(f).get("fa_fwd_sm100_8k", {})
                traffic = rec.get("dram_bytes_per_launch")
                traffic_source = rec.get("source", "profiles/ncu_summary.json")
            except Exception:  # noqa: BLE001
                traffic = None
        cb = None
        if world == 1 and not args.no_cpu:
            cb, _ = cpu_reference_run(1, 0, budget_s=60.0)
        achieved = flops / (ms * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOAD, "units_per_step_per_gpu": "1 op = 206.16 GFLOP (4*d*H*S^2)",
                       "l2": f"inputs larger than L2: rotating {n_sets} input sets, 302 MB total",
                       "launch": "rf_fa_plan_launch (one plan per input set, created and launched twice before the warm-up steps)",
                       "kernel": st.kernel, "grid_ctas": st.grid_ctas, "sharding": "independent ops per rank, no collective"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16"], "unit": "TFLOP/s",
                         "frac": achieved / peaks["bf16"], "traffic": traffic, "traffic_source": traffic_source,
                         "peak_source": peaks["source"],
                         "frac_of_sustained_peak": (achieved / peaks["bf16_sustained"]) if peaks["bf16_sustained"] else None,
                         "kernel": "fa_fwd_sm100_kernel<bf16, P in TMEM> (+ k_tile_norms_kernel pre-pass inside the timed step)", "flops_per_launch": flops},
            "cpu_baseline": cb,
            "e2e": {"value": e2e_val, "unit": UNIT,
                    # counted by the library where it issues the copies (rf_fa_host_transfer_counters): Q, K, V cross
                    # the link as bf16 when the host cores round them (75.5 MB of f32 host tensors -> 37.7 MB), as f32
                    # otherwise; the library picks the faster way per host and re-tries the other every 16th call
                    "h2d_bytes_per_step": (xfer1[0] - xfer0[0]) // max(1, xfer1[2] - xfer0[2]),
                    "d2h_bytes_per_step": (xfer1[1] - xfer0[1]) // max(1, xfer1[2] - xfer0[2]),
                    "host_tensor_bytes_per_step": {"in_f32": 3 * n_el * 4, "out_f32": n_el * 4},
                    "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
                    "api": "flash_attention(host f32 ndarrays) -> rf_fa_fwd_host (pinned host memory; inputs rounded to "
                           "bf16 by a pool of host threads under the previous chunk's transfers, or on the device)"},
            # per step in the timed region: k_tile_norms_kernel (row-max skip pre-pass over K) + fa_fwd_sm100_kernel
            "gpu_launches": 2 * args.steps,
            "clocks": clk.summary(),
            "sweep": extra,
        }
        print(json.dumps(line), flush=True)
    ctx.close()


# --------------------------------------------------------------------------------------------
# the multi-request / multi-GPU workloads of BASELINE.json (configs 3, 4, 5)
# --------------------------------------------------------------------------------------------
def _emit(ctx, line):
    if ctx.rank == 0:
        print(json.dumps(line), flush=True)


def _base_line(args, ctx, metric, unit, value, ms_per_step, scaling, dtype, workload, extra_config, clocks):
    return {"metric": metric, "value": value, "unit": unit, "n_gpus": ctx.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": dict({"workload": workload}, **extra_config), "clocks": clocks}


def _classifier_unit_runner(ctx, cfg, seeds, cache):
    """run_unit for BatchScheduler: one (classifier, request) forward through the native session (host token
    ids and mask in, host logits out; the session replays its CUDA graph from the second call of a shape on).
    One session per classifier, created on first use on this rank and kept."""
    from paper_2603_12646_b200.classifier import NativeClassifier, init_weights

    def run(unit, ids, mask):
        sess = cache.get(unit.model)
        if sess is None:
            sess = cache[unit.model] = NativeClassifier(cfg, init_weights(cfg, seeds[unit.model]), device=ctx.local_rank)
        logits = sess.forward(ids, mask)
        return logits, sess.last_forward_ms
    return run


def run_config3(args, ctx):
    """BASELINE configs[2]: 3 concurrent classifiers (safety, domain, PII) x batch 4 at S = 16384 -> 12
    (classifier, request) units, sharded over the ranks by BatchScheduler (LPT on attention + GEMM cost), weights
    replicated, no data-path collective, host-side gather of the [12, n_labels] logits on rank 0.  One step = the
    whole 12-unit job; 8 GPUs can reach at most 6x (12 units, makespan 2)."""
    import numpy as np
    torch = ctx.torch
    from paper_2603_12646_b200.classifier import ClassifierConfig
    from paper_2603_12646_b200.scheduler import BatchScheduler, Unit, lpt_assign
    S3, NB = 16384, 4
    cfg = ClassifierConfig()
    seeds = {"safety": 101, "domain": 102, "pii": 103}
    rng = np.random.default_rng(3)
    units, inputs = [], {}
    for m in seeds:
        for r in range(NB):
            n = int(rng.integers(S3 // 2, S3 + 1))
            u = Unit(uid=len(units), model=m, request=r, seq_len=S3, valid_len=n)
            units.append(u)
            g = torch.Generator().manual_seed(1000 + u.uid)
            mask = torch.ones((1, S3))
            mask[0, n:] = 0
            inputs[u.uid] = (torch.randint(0, cfg.vocab_size, (1, S3), generator=g), mask)
    cache = {}
    run1 = _classifier_unit_runner(ctx, cfg, seeds, cache)
    sched = BatchScheduler()
    dev_ms = []

    def run_unit(u):
        logits, ms = run1(u, *inputs[u.uid])
        dev_ms.append(ms)
        return logits.numpy()

    def step():
        dev_ms.clear()
        t0 = time.perf_counter()
        res = sched.run(units, run_unit, group=None)   # includes the host-side gather on rank 0
        return time.perf_counter() - t0, sum(dev_ms), res

    for _ in range(args.warmup):
        step()
    ctx.barrier()
    wall, dev, res = 0.0, 0.0, None
    with ClockSampler(ctx.local_rank) as clk:
        for _ in range(args.steps):
            w, d, res = step()
            wall += w
            dev += d
    ctx.barrier()
    wall = ctx.max_over_ranks(wall / args.steps)
    dev = ctx.max_over_ranks(dev / args.steps)
    mine = lpt_assign(units, ctx.world, sched.shape)
    ideal = len(units) / max(len(a) for a in mine)
    if ctx.rank == 0:
        assert res is not None and len(res) == len(units) and all(np.isfinite(v).all() for v in res.values())
    line = _base_line(args, ctx, "classifier_requests_per_s", "requests/s", len(units) / (dev * 1e-3), dev, "strong",
                      cfg.act_dtype, "config3: 3 classifiers (safety, domain, PII) x batch 4 x S=16384, variable-length masks",
                      {"units": len(units), "units_per_rank": [len(a) for a in mine], "ideal_speedup_vs_1gpu": ideal,
                       "sharding": "(classifier, request) units, LPT, weights replicated, no collective; host-side gather of logits",
                       "ms_per_request_device": dev / max(len(a) for a in mine), "paper_mi300x_ms_per_request": 259.0},
                      clk.summary())
    line["e2e"] = {"value": len(units) / wall, "unit": "requests/s", "ms_per_step": wall * 1e3,
                   "h2d_bytes_per_step": len(units) * S3 * 12, "d2h_bytes_per_step": len(units) * cfg.n_labels * 4,
                   "api": "rf_clf_forward(host ids, host mask) -> host logits, through BatchScheduler.run"}
    line["gpu_launches"] = args.steps * len(mine[0]) * (cfg.n_layers * 10 + 6)
    line["roofline"] = None
    line["cpu_baseline"] = None
    _emit(ctx, line)
    for sess in cache.values():
        sess.close()


def run_config4(args, ctx):
    """BASELINE configs[3]: ONE 32K-token sequence, 12 heads; K/V split into `world` contiguous key blocks, each rank
    runs the forward kernel over its block for all queries (un-normalised partials), then the softmax-merge
    exchange over NCCL (all-reduce max of m, rescale, reduce-scatter sum of [O | l], normalise, all-gather).  At
    world size 1 it is the plain op.  Strong scaling: the work per step is fixed."""
    torch, P = ctx.torch, ctx.P
    from paper_2603_12646_b200.splitkv import split_kv_attention
    S4 = 32768
    g = torch.Generator(device="cuda").manual_seed(4)   # same seed on every rank: Q, K, V are replicated
    n_sets = 2
    sets = [tuple((torch.rand((1, H, S4, D), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3))
            for _ in range(n_sets)]
    spec = P.AttentionSpec()

    def step(i):
        q, k, v = sets[i % n_sets]
        if ctx.world == 1:
            return P.flash_attention(q, k, v, spec, out_dtype=torch.float32)
        return split_kv_attention(q, k, v, spec, out_dtype=torch.float32, gather=True)

    for i in range(args.warmup):
        step(i)
    ctx.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(ctx.local_rank) as clk:
        e0.record()
        for i in range(args.steps):
            out = step(i)
        e1.record()
        torch.cuda.synchronize()
    ctx.barrier()
    ms = ctx.max_over_ranks(e0.elapsed_time(e1) / args.steps)
    flops = flops_global(1, H, S4, D)
    assert bool(torch.isfinite(out).all())
    line = _base_line(args, ctx, METRIC, UNIT, flops / ms / 1e9, ms, "strong", "bf16",
                      "config4: single 32K sequence, H=12, d=64, global; KV-block split across ranks with softmax-merge",
                      {"kv_blocks": ctx.world, "exchange": "none (1 GPU)" if ctx.world == 1 else
                       "allreduce(max) m -> rescale -> reduce_scatter(sum) [O|l] -> normalise -> all_gather (NCCL)",
                       "l2": f"rotating {n_sets} input sets of 151 MB"}, clk.summary())
    line["roofline"] = {"bound": "tensor", "achieved": flops / ms / 1e9 / ctx.world, "peak": ctx.peaks["bf16"], "unit": UNIT,
                        "frac": flops / ms / 1e9 / ctx.world / ctx.peaks["bf16"], "traffic": None,
                        "note": "per-GPU share of the job against one GPU's peak (includes the exchange)"}
    line["e2e"] = None
    line["cpu_baseline"] = None
    line["gpu_launches"] = args.steps * (2 if ctx.world == 1 else 5)
    _emit(ctx, line)


def run_config5(args, ctx):
    """BASELINE configs[4]: request-throughput sweep, S in 512..32K x batch 1..64 (B*S capped), tail padding with
    valid lengths U{S/2..S}.  The B requests of a point are sharded over the ranks (LPT); each rank runs its share
    as ONE batched classifier forward; a point's time is the max over ranks.  One step = one pass over all
    points; the headline value is requests/s over the whole sweep, the per-point numbers are in `sweep`."""
    import numpy as np
    torch = ctx.torch
    from paper_2603_12646_b200.classifier import ClassifierConfig, NativeClassifier, init_weights
    from paper_2603_12646_b200.scheduler import Unit, lpt_assign
    cfg = ClassifierConfig()
    sess = NativeClassifier(cfg, init_weights(cfg, 7), device=ctx.local_rank)
    points = [(s_, b_) for s_ in (512, 2048, 8192, 32768) for b_ in (1, 8, 64) if s_ * b_ <= 131072]
    if args.full_sweep:
        points = [(s_, b_) for s_ in (512, 1024, 2048, 4096, 8192, 16384, 32768) for b_ in (1, 2, 4, 8, 16, 32, 64)
                  if s_ * b_ <= 262144]
    rng = np.random.default_rng(5)
    work = []
    for (s_, b_) in points:
        lens = rng.integers(s_ // 2, s_ + 1, size=b_)
        units = [Unit(uid=i, model="clf", request=i, seq_len=s_, valid_len=int(n)) for i, n in enumerate(lens)]
        mine = lpt_assign(units, ctx.world)[ctx.rank]
        if mine:
            g = torch.Generator().manual_seed(s_ * 131 + b_)
            ids = torch.randint(0, cfg.vocab_size, (len(mine), s_), generator=g)
            mask = torch.ones((len(mine), s_))
            for r, u in enumerate(mine):
                mask[r, u.valid_len:] = 0
        else:
            ids = mask = None
        work.append((s_, b_, ids, mask))

    def one_pass():
        per_point = []
        for (s_, b_, ids, mask) in work:
            ms = 0.0
            if ids is not None:
                sess.forward(ids, mask)
                ms = sess.last_forward_ms
            per_point.append(ms)
        return per_point

    for _ in range(max(args.warmup, 2)):   # a shape is graph-captured on its second consecutive call
        for (s_, b_, ids, mask) in work:
            if ids is not None:
                sess.forward(ids, mask)
                sess.forward(ids, mask)
    ctx.barrier()
    acc = np.zeros(len(work))
    t0 = time.perf_counter()
    with ClockSampler(ctx.local_rank) as clk:
        for _ in range(args.steps):
            acc += np.array(one_pass())
    wall = (time.perf_counter() - t0) / args.steps
    ctx.barrier()
    acc /= args.steps
    if ctx.dist is not None:
        t = torch.tensor(acc, device="cuda", dtype=torch.float64)
        ctx.dist.all_reduce(t, op=ctx.dist.ReduceOp.MAX)
        acc = t.cpu().numpy()
    wall = ctx.max_over_ranks(wall)
    n_req = sum(b_ for (_, b_) in points)
    total_ms = float(acc.sum())
    sweep = [{"S": s_, "B": b_, "ms": float(ms), "req_per_s": b_ / ms * 1e3} for (s_, b_), ms in zip(points, acc)]
    line = _base_line(args, ctx, "classifier_requests_per_s", "requests/s", n_req / (total_ms * 1e-3), total_ms, "strong",
                      cfg.act_dtype, "config5: request-throughput sweep, S 512..32K x batch 1..64, variable-length padding masks",
                      {"points": len(points), "requests_per_step": n_req,
                       "sharding": "the requests of a point are dealt over the ranks (LPT), one batched forward per rank; no collective"},
                      clk.summary())
    line["sweep"] = sweep
    line["e2e"] = {"value": n_req / wall, "unit": "requests/s", "ms_per_step": wall * 1e3,
                   "h2d_bytes_per_step": sum(s_ * b_ for (s_, b_) in points) * 12, "d2h_bytes_per_step": n_req * cfg.n_labels * 4,
                   "api": "rf_clf_forward(host ids, host mask) -> host logits"}
    line["roofline"] = None
    line["cpu_baseline"] = None
    line["gpu_launches"] = args.steps * len(points) * (cfg.n_layers * 10 + 6)
    _emit(ctx, line)
    sess.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="op8k", choices=["op8k", "config3", "config4", "config5"])
    ap.add_argument("--quick", action="store_true", help="skip the 16K/32K/local sweep")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--full-sweep", action="store_true", help="config5: every (S, B) point instead of the bounded subset")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
