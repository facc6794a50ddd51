"""GPU tests added in round 2 (run with -m gpu on a B200): regressions for the advisor's findings and the
new entry points.  Same conventions as test_gpu_parity.py: the CUDA path through the C ABI against the
oracle, inputs rounded to bf16 on both sides, attention tolerance 2e-2 (BASELINE.json)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-2


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def P():
    import paper_2603_12646_b200 as pkg
    return pkg


def tail_pad(B, S, lens):
    pb = np.zeros((B, 1, 1, S), np.float32)
    for b, n in enumerate(lens):
        pb[b, 0, 0, n:] = -65504.0
    return pb


def rand_qkv(oracle, seed, shape):
    rng = np.random.default_rng(seed)
    return [oracle.round_bf16(rng.uniform(-1, 1, shape).astype(np.float32)) for _ in range(3)]


# ------------------------------------------------------------------ advisor: stale RoPE tables
def test_native_session_alternating_mask_on_one_session(torch_mod, P):
    """One rf_clf session, same (B, S), forward with a mask, without, with again (and a larger shape in
    between): the arena layout differs with and without a mask, the RoPE tables must not move with it."""
    torch = torch_mod
    from paper_2603_12646_b200.classifier import Classifier, ClassifierConfig, NativeClassifier, init_weights
    cfg = ClassifierConfig(vocab_size=500, n_layers=3, n_labels=3)
    w = init_weights(cfg, seed=5)
    B, S = 2, 1024
    ids = torch.randint(0, cfg.vocab_size, (B, S), generator=torch.Generator().manual_seed(1))
    mask = torch.ones((B, S))
    mask[0, 900:] = 0
    mask[1, 1000:] = 0
    hosted = Classifier(cfg, w, torch.device("cuda:0"))
    want_m = hosted.forward(ids.cuda(), mask.cuda()).cpu().numpy()
    want_n = hosted.forward(ids.cuda(), None).cpu().numpy()
    nat = NativeClassifier(cfg, w)
    ids_big = torch.randint(0, cfg.vocab_size, (1, 2048), generator=torch.Generator().manual_seed(2))
    seq = [("m", mask), ("n", None), ("m", mask), ("big", None), ("n", None), ("n", None), ("m", mask), ("m", mask),
           ("n", None)]
    for tag, m in seq:
        if tag == "big":
            nat.forward(ids_big)
            continue
        got = nat.forward(ids, m).numpy()
        want = want_m if tag == "m" else want_n
        assert np.abs(got - want).max() <= 5e-3, (tag, np.abs(got - want).max())
    nat.close()


# ------------------------------------------------------------------ advisor: empty split-KV block
def test_empty_partial_block_is_the_neutral_element(torch_mod, P, oracle):
    """A partial call over the empty key range [0, 0) writes m = -inf, l = 0, O = 0 (it used to mean
    'all keys'); merging it with the other blocks gives the single-pass result."""
    torch = torch_mod
    from paper_2603_12646_b200.splitkv import merge_partials_local
    B, H, S, d = 1, 2, 200, 64
    q, k, v = rand_qkv(oracle, 3, (B, H, S, d))
    tq, tk, tv = [torch.from_numpy(t).cuda().to(torch.bfloat16) for t in (q, k, v)]
    parts = []
    for (a, b) in ((0, 0), (0, 128), (128, 200), (200, 200)):
        o = torch.full((B, H, S, d), 7.0, device="cuda")
        m = torch.full((B, H, S), 7.0, device="cuda")
        l = torch.full((B, H, S), 7.0, device="cuda")
        P.flash_attention(tq, tk, tv, P.AttentionSpec(), kv_range=(a, b), partials=(o, m, l))
        parts.append((o, m, l))
    torch.cuda.synchronize()
    for idx in (0, 3):
        o, m, l = parts[idx]
        assert (o == 0).all() and (l == 0).all() and torch.isinf(m).all() and (m < 0).all()
    out = merge_partials_local(parts).cpu().numpy()
    want = oracle.flash_attention(q, k, v, 0.0, -1, -1, None)
    assert np.abs(out - want).max() <= TOL
    # a partial without an explicit range covers all keys
    o = torch.empty((B, H, S, d), device="cuda")
    m = torch.empty((B, H, S), device="cuda")
    l = torch.empty((B, H, S), device="cuda")
    P.flash_attention(tq, tk, tv, P.AttentionSpec(), partials=(o, m, l))
    out1 = merge_partials_local([(o, m, l)]).cpu().numpy()
    assert np.abs(out1 - want).max() <= TOL


# ------------------------------------------------------------------ advisor: window overflow / flags
def test_huge_windows_mean_unbounded_and_flags_are_rejected(torch_mod, P, oracle):
    torch = torch_mod
    from paper_2603_12646_b200 import capi
    B, H, S, d = 1, 1, 300, 64
    q, k, v = rand_qkv(oracle, 4, (B, H, S, d))
    tq, tk, tv = [torch.from_numpy(t).cuda().to(torch.bfloat16) for t in (q, k, v)]
    want = oracle.flash_attention(q, k, v, 0.0, -1, -1, None)
    for w in (2 ** 62, 2 ** 31, 2 ** 40 + 5):
        got = P.flash_attention(tq, tk, tv, P.AttentionSpec(0.0, w, w)).float().cpu().numpy()
        assert np.abs(got - want).max() <= TOL, w
    with pytest.raises(capi.RfError):
        P.flash_attention(tq, tk, tv, P.AttentionSpec(), flags=1)


# ------------------------------------------------------------------ head_dim 32 / 128 on the tensor cores
@pytest.mark.parametrize("d", [32, 128])
def test_head_dims_32_128_run_on_tcgen05(torch_mod, P, oracle, d):
    """rewrite.cpp:266-269: head dims {32, 64, 128}.  Every one of them takes a tcgen05 kernel (32 zero-padded
    to 64 inside the TMA box, 128 on its own kernel): parity grid over windows, padding and ragged lengths."""
    torch = torch_mod
    rng = np.random.default_rng(100 + d)
    worst = 0.0
    for (B, H, S) in ((1, 2, 37), (2, 3, 300), (1, 2, 1000), (1, 1, 1500)):
        q, k, v = [oracle.round_bf16(rng.uniform(-1, 1, (B, H, S, d)).astype(np.float32)) for _ in range(3)]
        lens = [max(1, S - 1 - 31 * b) for b in range(B)]
        for (wl, wr) in ((-1, -1), (63, 64), (1, 2), (-1, 0), (200, 100)):
            for pb in (None, tail_pad(B, S, lens)):
                tq, tk, tv = [torch.from_numpy(t).cuda().to(torch.bfloat16) for t in (q, k, v)]
                st = P.FlashStats()
                out = P.flash_attention(tq, tk, tv, P.AttentionSpec(0.0, wl, wr, torch.from_numpy(pb).cuda() if pb is not None else None),
                                        stats=st, kernel="tcgen05")
                torch.cuda.synchronize()
                assert st.kernel == "tcgen05"
                want = oracle.flash_attention(q, k, v, 0.0, wl, wr, pb, threads=8)
                got = out.float().cpu().numpy()
                assert not np.isnan(got).any()
                err = float(np.abs(got - want).max())
                worst = max(worst, err)
                assert err <= TOL, (d, B, H, S, wl, wr, pb is not None, err)
    print("d", d, "worst", worst)


@pytest.mark.parametrize("d", [32, 128])
def test_head_dims_32_128_long_sequence_and_split_kv(torch_mod, P, oracle, d):
    """S = 4096 (persistent schedules), f16 inputs, strided [B,S,H,d] views and a split-KV merge, one head
    checked against the oracle and every head against the CUDA-core kernel."""
    torch = torch_mod
    from paper_2603_12646_b200.splitkv import kv_block, merge_partials_local
    B, H, S = 2, 12, 4096
    g = torch.Generator(device="cuda").manual_seed(d)
    qkv = (torch.rand((B, S, 3, H, d), device="cuda", generator=g) * 2 - 1).to(torch.float16)
    q, k, v = (qkv[:, :, j].permute(0, 2, 1, 3) for j in range(3))
    lens = [4096, 3001]
    pb = torch.from_numpy(tail_pad(B, S, lens)).cuda()
    for (wl, wr) in ((-1, -1), (63, 64)):
        spec = P.AttentionSpec(0.0, wl, wr, pb)
        st = P.FlashStats()
        out = P.flash_attention(q, k, v, spec, stats=st, out_dtype=torch.float32)
        ref = P.flash_attention(q, k, v, spec, kernel="simt", out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert st.kernel == "tcgen05"
        assert (out - ref).abs().max().item() <= 5e-3
        b, h = 1, 5
        want = oracle.flash_attention(q[b:b + 1, h:h + 1].float().cpu().numpy(), k[b:b + 1, h:h + 1].float().cpu().numpy(),
                                      v[b:b + 1, h:h + 1].float().cpu().numpy(), 0.0, wl, wr, pb[b:b + 1].cpu().numpy())
        assert np.abs(out[b:b + 1, h:h + 1].cpu().numpy() - want).max() <= TOL
    spec = P.AttentionSpec(0.0, -1, -1, pb)
    full = P.flash_attention(q, k, v, spec, out_dtype=torch.float32)
    parts = []
    for r in range(3):
        o = torch.empty((B, H, S, d), device="cuda")
        m = torch.empty((B, H, S), device="cuda")
        l = torch.empty((B, H, S), device="cuda")
        P.flash_attention(q, k, v, spec, kv_range=kv_block(S, r, 3), partials=(o, m, l))
        parts.append((o, m, l))
    merged = merge_partials_local(parts)
    assert (merged - full).abs().max().item() <= 2e-3


def test_head_dim_128_balanced_schedule_split_pairs(torch_mod, P, oracle):
    """head_dim 128 over more query-tile pairs than SMs runs the balanced schedule of the head_dim-64 kernel (slices of
    the flat (pair x key tile) space, cut pairs merged in-kernel): 384 pairs on 148 SMs, every CTA publishes and merges.
    Checked against the CUDA-core kernel on every head, against the oracle on one, bit-identical from launch to launch
    (plan relaunches on one workspace: the flags are left zero), and with ragged lengths."""
    torch = torch_mod
    from paper_2603_12646_b200 import capi
    from paper_2603_12646_b200.attention import FaPlan
    for (B, H, S, lens) in ((1, 12, 8192, None), (3, 4, 5000, [5000, 1234, 4097])):
        g = torch.Generator(device="cuda").manual_seed(128 + S)
        q, k, v = [(torch.rand((B, H, S, 128), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
        pb = torch.from_numpy(tail_pad(B, S, lens)).cuda() if lens else None
        spec = P.AttentionSpec(0.0, -1, -1, pb)
        st = P.FlashStats()
        out = P.flash_attention(q, k, v, spec, stats=st, out_dtype=torch.float32)
        ref = P.flash_attention(q, k, v, spec, kernel="simt", out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert st.kernel == "tcgen05" and st.grid_ctas == torch.cuda.get_device_properties(0).multi_processor_count
        assert (out - ref).abs().max().item() <= 5e-3
        if S <= 5000:   # the oracle on one (batch, head) slice (a few seconds of scalar C)
            b, h = 1, H - 1
            want = oracle.flash_attention(*[t[b:b + 1, h:h + 1].float().cpu().numpy() for t in (q, k, v)], 0.0, -1, -1,
                                          pb[b:b + 1].cpu().numpy() if pb is not None else None)
            assert np.abs(out[b:b + 1, h:h + 1].cpu().numpy() - want).max() <= TOL
        o2 = torch.empty_like(out)
        plan = FaPlan(q, k, v, spec, out=o2)
        for _ in range(5):
            plan.launch()
        torch.cuda.synchronize()
        assert plan.status() == capi.RF_OK and torch.equal(o2, out)
        plan.close()


# ------------------------------------------------------------------ plan object
def test_plan_launch_equals_direct_call_and_reports_status(torch_mod, P, oracle):
    """rf_fa_plan_create / rf_fa_plan_launch: same result bit for bit as rf_fa_fwd, relaunchable after the
    tensors' contents change; rf_fa_launch_status reports RF_OK."""
    torch = torch_mod
    from paper_2603_12646_b200 import capi
    from paper_2603_12646_b200.attention import FaPlan
    lib = capi.load()
    B, H, S, d = 1, 12, 2048, 64
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = [(torch.rand((B, H, S, d), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
    for (wl, wr, padded) in ((-1, -1, False), (-1, -1, True), (63, 64, True)):
        pb = torch.from_numpy(tail_pad(B, S, [1777])).cuda() if padded else None
        spec = P.AttentionSpec(0.0, wl, wr, pb)
        direct = P.flash_attention(q, k, v, spec).clone()
        out = torch.zeros_like(direct)
        plan = FaPlan(q, k, v, spec, out=out)
        plan.launch()
        torch.cuda.synchronize()
        assert torch.equal(out, direct)
        q2 = q.clone()
        q.copy_(-q)                      # same addresses, new contents
        plan.launch()
        direct2 = P.flash_attention(q, k, v, spec)
        torch.cuda.synchronize()
        assert torch.equal(out, direct2) and not torch.equal(out, direct)
        q.copy_(q2)
        assert plan.status() == capi.RF_OK
        plan.close()


def test_plans_of_different_layouts_share_one_workspace(torch_mod, P, oracle):
    """The split-pair flags of the persistent balanced schedule sit at a fixed offset behind the status block whatever
    else a plan keeps in its workspace, are zeroed by a plan's first launch only and left zero by the kernel.  Two
    plans with different carve-ups (with and without a pad bias) therefore can take turns on ONE workspace, any number
    of times, and give what they give alone."""
    torch = torch_mod
    from paper_2603_12646_b200 import capi
    from paper_2603_12646_b200.attention import FaPlan
    B, H, S, d = 2, 12, 4096, 64     # 384 pairs > 148 SMs: split pairs, partials, flags
    g = torch.Generator(device="cuda").manual_seed(23)
    q, k, v = [(torch.rand((B, H, S, d), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
    pb = torch.from_numpy(tail_pad(B, S, [4096, 3001])).cuda()
    spec_a, spec_b = P.AttentionSpec(), P.AttentionSpec(0.0, -1, -1, pb)
    st_a, st_b = P.FlashStats(), P.FlashStats()
    ref_a = P.flash_attention(q, k, v, spec_a, stats=st_a).clone()
    ref_b = P.flash_attention(q, k, v, spec_b, stats=st_b).clone()
    assert st_a.workspace_bytes != st_b.workspace_bytes
    ws = torch.empty(max(st_a.workspace_bytes, st_b.workspace_bytes), dtype=torch.uint8, device="cuda")
    ws.fill_(0xAB)                   # a fresh arena is not zero
    oa, ob = torch.empty_like(ref_a), torch.empty_like(ref_b)
    pa = FaPlan(q, k, v, spec_a, out=oa, workspace=ws)
    pbl = FaPlan(q, k, v, spec_b, out=ob, workspace=ws)
    for _ in range(6):
        pa.launch()
        pbl.launch()
        pbl.launch()
        pa.launch()
    torch.cuda.synchronize()
    assert pa.status() == capi.RF_OK
    assert torch.equal(oa, ref_a) and torch.equal(ob, ref_b)
    pa.close()
    pbl.close()


@pytest.mark.parametrize("window", [(-1, -1), (63, 64)])
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_output_rows_off_the_32_byte_grid(torch_mod, P, oracle, window, dt):
    """The kernels write their output rows with 32-byte stores when every row segment is 32-byte aligned and fall back to
    16-byte stores when it is not: an output view that starts 16 bytes into its buffer gives the same bits."""
    torch = torch_mod
    B, H, S, d = 1, 3, 700, 64
    g = torch.Generator(device="cuda").manual_seed(29)
    q, k, v = [(torch.rand((B, H, S, d), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
    odt = torch.bfloat16 if dt == "bf16" else torch.float32
    spec = P.AttentionSpec(0.0, *window)
    aligned = P.flash_attention(q, k, v, spec, out_dtype=odt)
    shift = 16 // aligned.element_size()
    buf = torch.zeros(B * H * S * d + shift, device="cuda", dtype=odt)
    view = buf[shift:].view(B, H, S, d)
    assert view.data_ptr() % 32 == 16
    P.flash_attention(q, k, v, spec, out=view)
    torch.cuda.synchronize()
    assert torch.equal(view, aligned)
    want = oracle.flash_attention(*[t.float().cpu().numpy() for t in (q, k, v)], 0.0, window[0], window[1], None)
    assert float(np.abs(aligned.float().cpu().numpy() - want).max()) <= TOL


# ------------------------------------------------------------------ persistent schedule under contention
def test_two_persistent_calls_on_two_streams_do_not_starve(torch_mod, P, oracle):
    """Two balanced-schedule (mode 1) launches run concurrently on two streams, each with its own workspace,
    while a third stream keeps the SMs busy with other work.  A CTA of the split-pair chain only ever waits for
    a lower-indexed CTA, so both finish, bit-identical to their isolated runs, with a clean status word."""
    torch = torch_mod
    from paper_2603_12646_b200 import capi
    from paper_2603_12646_b200.attention import FaPlan
    B, H, S, d = 1, 12, 4096, 64     # 192 pairs > 148 SMs: persistent balanced schedule with split pairs
    g = torch.Generator(device="cuda").manual_seed(11)
    mk = lambda: [(torch.rand((B, H, S, d), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
    (q1, k1, v1), (q2, k2, v2) = mk(), mk()
    spec = P.AttentionSpec()
    st = P.FlashStats()
    ref1 = P.flash_attention(q1, k1, v1, spec, stats=st).clone()
    ref2 = P.flash_attention(q2, k2, v2, spec).clone()
    assert st.grid_ctas == torch.cuda.get_device_properties(0).multi_processor_count
    o1, o2 = torch.empty_like(ref1), torch.empty_like(ref2)
    p1, p2 = FaPlan(q1, k1, v1, spec, out=o1), FaPlan(q2, k2, v2, spec, out=o2)
    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    torch.cuda.synchronize()
    for _ in range(20):
        with torch.cuda.stream(s3):
            a @ a
        with torch.cuda.stream(s1):
            p1.launch()
        with torch.cuda.stream(s2):
            p2.launch()
    torch.cuda.synchronize()
    assert p1.status() == capi.RF_OK and p2.status() == capi.RF_OK
    assert torch.equal(o1, ref1) and torch.equal(o2, ref2)
    p1.close()
    p2.close()


# ------------------------------------------------------------------ bench.py workloads / N-GPU launcher
def _run_bench(argv, timeout=900):
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py")] + argv, cwd=root, env=env, capture_output=True,
                         text=True, timeout=timeout)
    lines = [json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{")]
    return res, lines


def test_bench_workloads_on_one_gpu(torch_mod):
    """config3 / config4 / config5 run through BatchScheduler / split_kv_attention's N=1 path and print one
    contract line each."""
    for wl, metric in (("config4", "attention_fwd_tflops"), ("config3", "classifier_requests_per_s"),
                       ("config5", "classifier_requests_per_s")):
        res, lines = _run_bench(["--workload", wl, "--steps", "1", "--warmup", "3"])
        assert res.returncode == 0, res.stderr[-2000:]
        assert len(lines) == 1
        ln = lines[0]
        assert ln["metric"] == metric and ln["n_gpus"] == 1 and ln["value"] > 0 and wl in ln["config"]["workload"]
        if wl == "config3":
            assert ln["config"]["units"] == 12 and ln["config"]["units_per_rank"] == [12]


def test_bench_gpus_n_spawns_ranks_or_fails_loudly(torch_mod):
    """`bench.py --gpus 2` outside torchrun starts 2 NCCL ranks itself; with fewer GPUs visible it exits 2 with an
    error line instead of silently running one rank."""
    torch = torch_mod
    if torch.cuda.device_count() >= 2:
        for wl in ("op8k", "config4", "config3"):
            res, lines = _run_bench(["--gpus", "2", "--workload", wl, "--steps", "2", "--warmup", "3", "--quick", "--no-cpu"])
            assert res.returncode == 0, res.stderr[-2000:]
            assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["value"] > 0
    else:
        res, lines = _run_bench(["--gpus", "2", "--steps", "2", "--warmup", "3", "--quick", "--no-cpu"])
        assert res.returncode == 2 and lines and "error" in lines[0]


def test_split_kv_over_nccl_matches_single_pass(torch_mod):
    """2-rank NCCL split-KV (config 4's exchange) against the single-GPU op; skipped below 2 GPUs."""
    torch = torch_mod
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r'''
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
import paper_2603_12646_b200 as P
from paper_2603_12646_b200.splitkv import split_kv_attention
rank = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
g = torch.Generator(device="cuda").manual_seed(4)
q, k, v = [(torch.rand((1, 12, 4096, 64), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
pb = torch.zeros((1, 1, 1, 4096), device="cuda"); pb[..., 3000:] = -65504.0
for spec in (P.AttentionSpec(), P.AttentionSpec(0.0, -1, -1, pb), P.AttentionSpec(0.0, 300, 200, pb)):
    full = split_kv_attention(q, k, v, spec, out_dtype=torch.float32)
    ref = P.flash_attention(q, k, v, spec, out_dtype=torch.float32)
    assert (full - ref).abs().max().item() <= 2e-3, (full - ref).abs().max().item()
dist.barrier(); dist.destroy_process_group()
print("nccl split-kv ok")
'''
    import tempfile
    with tempfile.NamedTemporaryFile("w", suffix=".py", delete=False) as f:
        f.write(script)
        path = f.name
    try:
        res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
                              "127.0.0.1", "--master-port", "29631", path], cwd=root, capture_output=True, text=True, timeout=600)
    finally:
        os.unlink(path)
    assert res.returncode == 0 and "nccl split-kv ok" in res.stdout, res.stderr[-3000:]
