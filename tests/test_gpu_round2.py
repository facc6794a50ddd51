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
