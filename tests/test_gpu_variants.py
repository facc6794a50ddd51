"""GPU tests of the run-time kernel selectors (developer variants that ship in librf_fa.so): each runs in a
subprocess because the selectors are read once per process.  The checker is the generic SIMT kernel on the
same inputs plus the oracle on one (batch, head) slice."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import paper_2603_12646_b200 as P
import oracle as O
g = torch.Generator(device="cuda").manual_seed(5)
worst = 0.0
for (B, H, S, wl, wr, lens) in ((1, 12, 8192, -1, -1, None), (2, 3, 1000, -1, -1, [1000, 640]), (1, 2, 700, 63, 64, [650]),
                                (8, 12, 4096, -1, -1, [4096, 2100, 0, 3000, 4095, 129, 3584, 1]), (1, 2, 900, 300, 10, None)):
    q, k, v = [(torch.rand((B, H, S, 64), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)]
    pb = None
    if lens is not None:
        pbn = np.zeros((B, 1, 1, S), np.float32)
        for b, n in enumerate(lens):
            pbn[b, 0, 0, n:] = -65504.0
        pb = torch.from_numpy(pbn).cuda()
    spec = P.AttentionSpec(0.0, wl, wr, pb)
    st = P.FlashStats()
    a = P.flash_attention(q, k, v, spec, stats=st)
    b_ = P.flash_attention(q, k, v, spec, kernel="simt")
    torch.cuda.synchronize()
    assert st.kernel == "tcgen05"
    err = (a.float() - b_.float()).abs().max().item()
    assert err <= 5e-3 and not torch.isnan(a).any(), (S, wl, err)
    worst = max(worst, err)
    if S <= 1000:
        want = O.flash_attention(q[:1, :1].float().cpu().numpy(), k[:1, :1].float().cpu().numpy(), v[:1, :1].float().cpu().numpy(),
                                 0.0, wl, wr, pb[:1].cpu().numpy() if pb is not None else None)
        assert np.abs(a[:1, :1].float().cpu().numpy() - want).max() <= 2e-2
print("variant ok", worst)
"""


@pytest.mark.parametrize("env", [{"RF_FA_LOCAL": "0"}, {"RF_FA_SKIP_MAX": "0"}, {"RF_FA_SCHED_MODE": "1"},
                                 {"RF_FA_SCHED_MODE": "2"}])
def test_kernel_selector_variants(env):
    e = dict(os.environ)
    e.update(env)
    res = subprocess.run([sys.executable, "-c", SNIPPET], cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    print(env, res.stdout[-500:], res.stderr[-1500:])
    assert res.returncode == 0 and "variant ok" in res.stdout


HOST_SNIPPET = r"""
import hashlib, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_2603_12646_b200 as P
from paper_2603_12646_b200 import capi
rng = np.random.default_rng(17)
digest = hashlib.sha256()
for (B, H, S, wl, wr, pad) in ((1, 12, 4096, -1, -1, False), (2, 6, 2048, 63, 64, True), (1, 12, 8192, -1, -1, False)):
    q, k, v = [rng.standard_normal((B, H, S, 64)).astype(np.float32) for _ in range(3)]   # NOT pre-rounded to bf16
    pb = None
    if pad:
        pb = np.zeros((B, 1, 1, S), np.float32)
        pb[-1, 0, 0, S - 333:] = -65504.0
    x0 = capi.host_transfer_counters()
    for _ in range(8):                      # default mode: three host-rounded calls, three device-rounded, then the faster
        out = P.flash_attention(q, k, v, P.AttentionSpec(0.0, wl, wr, pb), device=0)
        assert np.isfinite(out).all()
        digest.update(out.tobytes())
    x1 = capi.host_transfer_counters()
    assert x1[2] - x0[2] == 8 and x1[1] - x0[1] == 8 * out.nbytes
    per_call = (x1[0] - x0[0]) / 8
    print("h2d per call / f32 input bytes: %.2f" % (per_call / (3 * q.nbytes)))
print("host digest", digest.hexdigest())
"""


def _host_run(env):
    e = dict(os.environ)
    e.update(env)
    res = subprocess.run([sys.executable, "-c", HOST_SNIPPET], cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    print(env, res.stdout[-800:], res.stderr[-1500:])
    assert res.returncode == 0 and "host digest" in res.stdout
    return res.stdout


def test_host_entry_rounds_on_host_or_device_with_the_same_bits():
    """rf_fa_fwd_host rounds Q, K, V to bf16 either on a pool of host threads (half the bytes on the link) or on the
    device, whichever it measures to be faster on this host; every call of either kind gives the same output bits (the
    two roundings are the same function), and the transfer counters say how many bytes actually crossed."""
    outs = {name: _host_run(env) for name, env in (("device", {"RF_FA_HOST_CAST": "0"}), ("host", {"RF_FA_HOST_CAST": "1"}),
                                                   ("auto", {}))}
    digests = {name: [ln for ln in o.splitlines() if ln.startswith("host digest")][0] for name, o in outs.items()}
    assert digests["device"] == digests["host"] == digests["auto"]
    ratios = {name: [float(ln.split(":")[1]) for ln in o.splitlines() if ln.startswith("h2d per call")] for name, o in outs.items()}
    assert all(abs(r - 1.0) < 0.02 for r in ratios["device"])            # f32 over the link (+ the pad bias)
    # large calls go as bf16 (the 2048-token call is below the 16 MiB threshold only if 3 * 4 * B*H*S*64 < 16 MiB)
    if (os.cpu_count() or 1) >= 4 and not os.environ.get("RF_FA_HOST_CAST_THREADS"):   # the pool needs two spare cores
        assert abs(ratios["host"][0] - 0.5) < 0.02 and abs(ratios["host"][2] - 0.5) < 0.02


def test_host_rounding_on_the_gpu_box_cpu():
    """The host rounding picks its widest vector path at run time (AVX-512 on the GPU boxes, AVX2 on the CPU-only dev
    container): run the bit-for-bit check of tests/test_capi_cpu.py on this machine's path too."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import test_capi_cpu as T
    from paper_2603_12646_b200 import capi
    T.test_host_rounding_is_round_to_nearest_even_bit_for_bit(capi.load())
