#!/usr/bin/env python
"""bench.py -- headline benchmark of the FusedFlashAttention hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

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

N > 1 (torchrun): independent request shards per rank, no data-path collective (weak scaling);
device-timed, max over ranks.
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
    """Times routefast::flash_attention on a bounded sample of the 8K workload: `heads` heads
    (one thread each, the op itself is single-threaded) at sequence length s_sample."""
    import numpy as np

    import oracle as O
    kind = "reference" if O.have_reference() else "port"
    impl = "reference" if kind == "reference" else "port"
    cores = os.cpu_count() or 1
    heads = max(1, min(cores, H))
    per_step = max(budget_s / max(1, steps + warmup), 0.5)
    s_sample = S
    while s_sample > 1024 and 4.0 * s_sample * s_sample * D / 2.0e9 > per_step:  # ~2 GFLOP/s per core
        s_sample //= 2
    rng = np.random.default_rng(0)
    q, k, v = [rng.uniform(-1, 1, (1, heads, s_sample, D)).astype(np.float32) for _ in range(3)]
    for _ in range(warmup):
        O.flash_attention(q, k, v, 0.0, -1, -1, None, threads=heads, impl=impl)
    t0 = time.perf_counter()
    for _ in range(steps):
        O.flash_attention(q, k, v, 0.0, -1, -1, None, threads=heads, impl=impl)
    dt = (time.perf_counter() - t0) / max(1, steps)
    tflops = flops_global(1, heads, s_sample, D) / dt / 1e12
    sample = (f"{heads} of {H} heads x S={s_sample} of the workload per step (all queries x all keys), one thread per "
              f"head; {steps} step(s)")
    return {"value": tflops, "unit": UNIT, "cores": heads, "kind": kind, "sample": sample}, dt


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb, dt = cpu_reference_run(args.steps, args.warmup, budget_s=150.0)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "note": "reference CPU operator, f32 storage / f64 arithmetic"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------------
def time_op(torch, P, sets, spec, steps, warmup, out_sets):
    n = len(sets)
    for i in range(warmup):
        q, k, v = sets[i % n]
        P.flash_attention(q, k, v, spec, out=out_sets[i % n])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        q, k, v = sets[i % n]
        P.flash_attention(q, k, v, spec, out=out_sets[i % n])
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps  # ms per step


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


def run_ours(args):
    import numpy as np
    import torch

    import paper_2603_12646_b200 as P
    from paper_2603_12646_b200 import capi

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise RuntimeError("bench.py needs a CUDA device (no CPU fallback exists)")
    torch.cuda.set_device(local_rank)
    capi.load(build_if_missing=False)  # the CUDA extension must be there: fail loudly otherwise
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    peaks = load_peaks()
    spec = P.AttentionSpec()  # global, scale 1/sqrt(d)
    # inputs larger than L2: each set is 4 tensors x 12.6 MB = 50 MB; 6 sets = 302 MB > 126 MB L2
    n_sets = 6
    sets, outs = make_sets(torch, B, H, S, D, n_sets, seed=1234 + rank)
    st = P.FlashStats()
    P.flash_attention(*sets[0], spec, out=outs[0], stats=st)
    if st.kernel != "tcgen05":
        raise RuntimeError(f"expected the tcgen05 kernel, got {st.kernel}")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    with ClockSampler(local_rank) as clk:
        ms = time_op(torch, P, sets, spec, args.steps, args.warmup, outs)
    barrier()
    if dist is not None:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
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
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        out_h = P.flash_attention(hq, hk, hv, spec, device=local_rank)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    barrier()
    if dist is not None:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = world * flops / e2e_s / 1e12
    n_el = B * H * S * D
    assert np.isfinite(out_h).all()

    if rank == 0:
        extra = {}
        if not args.quick:
            # the other sequence lengths of the metric, and the HBM-bound local layer
            for s2, it in ((16384, 10), (32768, 5)):
                sets2, outs2 = make_sets(torch, B, H, s2, D, 3 if s2 == 16384 else 2, seed=7)
                ms2 = time_op(torch, P, sets2, spec, it, 3, outs2)
                f2 = flops_global(B, H, s2, D)
                extra[f"S{s2}"] = {"ms": ms2, "tflops": f2 / ms2 / 1e9, "frac_of_peak": f2 / ms2 / 1e9 / peaks["bf16"]}
                del sets2, outs2
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
                    "weights_MB": clf.weight_bytes() / 1e6, "cuda_graph": True,
                    "paper_mi300x_ms": 105.0, "note": "random-init weights, synthetic token ids; paper number is other hardware (PAPER.md:402)"}
                del clf, run
                # the same forward through the native session (rf_clf.h): host token ids in, host logits out,
                # cuBLAS GEMMs + this library's kernels, no Python between the launches
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
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
        if os.path.exists(prof):
            try:
                with open(prof) as f:
                    traffic = json.load(f).get("fa_fwd_sm100_8k", {}).get("dram_bytes_per_launch")
            except Exception:  # noqa: BLE001
                traffic = None
        cb = None
        if world == 1 and not args.no_cpu:
            cb, _ = cpu_reference_run(1, 0, budget_s=12.0)
        achieved = flops / (ms * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOAD, "units_per_step_per_gpu": "1 op = 206.16 GFLOP (4*d*H*S^2)",
                       "l2": f"inputs larger than L2: rotating {n_sets} input sets, 302 MB total",
                       "kernel": st.kernel, "grid_ctas": st.grid_ctas, "sharding": "independent ops per rank, no collective"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16"], "unit": "TFLOP/s",
                         "frac": achieved / peaks["bf16"], "traffic": traffic, "peak_source": peaks["source"],
                         "frac_of_sustained_peak": (achieved / peaks["bf16_sustained"]) if peaks["bf16_sustained"] else None,
                         "kernel": "fa_fwd_sm100_kernel<bf16, P in TMEM> (+ qk_norms_kernel pre-pass inside the timed step)", "flops_per_launch": flops},
            "cpu_baseline": cb,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 3 * n_el * 4, "d2h_bytes_per_step": n_el * 4,
                    "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
                    "api": "flash_attention(host f32 ndarrays) -> rf_fa_fwd_host (pinned host memory)"},
            # per step in the timed region: qk_norms_kernel (row-max skip pre-pass, also zeroes the schedule
            # flags) + fa_fwd_sm100_kernel
            "gpu_launches": 2 * args.steps,
            "clocks": clk.summary(),
            "sweep": extra,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--quick", action="store_true", help="skip the 16K/32K/local sweep")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
