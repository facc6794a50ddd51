"""CPU tests: pin the oracle (oracle/rf_oracle.c) against the reference.

1. against golden vectors generated from the reference build (tests/golden/make_golden.py);
2. against the reference build itself when oracle/_ref/libref_attn.so is present (bit-exact);
3. the known-answer examples and invariants of the reference spec whose test files are missing
   from the snapshot.
"""
import numpy as np
import pytest


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def assert_bit_exact(a, b):
    assert a.shape == b.shape
    assert np.array_equal(bits(a), bits(b))


# ----------------------------------------------------------------------------- golden vectors
def test_rng_stream_matches_reference(oracle, golden):
    for seed in (5, 7, 11, 42):
        assert_bit_exact(oracle.random_tensors(seed, (32,), 1)[0], golden[f"rng_seed{seed}_head"])
    assert_bit_exact(oracle.random_tensors(11, (32,), 1, as_f16=True)[0], golden["rng_seed11_f16_head"])


def test_f16_emulation_matches_reference(oracle, golden):
    assert_bit_exact(oracle.quantize_f16(golden["f16_probe_in"]), golden["f16_probe_out"])
    got = np.array([oracle.float_to_half(float(x)) for x in golden["f16_probe_in"]], dtype=np.uint16)
    assert np.array_equal(got, golden["f16_probe_bits"])
    # round trip of every finite half bit pattern is the identity
    for b in list(range(0, 0x7C00, 97)) + [0x0001, 0x03FF, 0x0400, 0x7BFF, 0x8001, 0xFBFF]:
        assert oracle.float_to_half(oracle.half_to_float(b)) == b


@pytest.mark.parametrize("S", [128, 512])
def test_bench_global_golden(oracle, golden, S):
    q, k, v = oracle.random_tensors(11, (1, 2, S, 64), 3)
    assert_bit_exact(oracle.flash_attention(q, k, v, 0.125), golden[f"bench_global_S{S}"])


def test_bench_local_and_sdpa_golden(oracle, golden):
    q, k, v = oracle.random_tensors(11, (1, 2, 512, 64), 3)
    assert_bit_exact(oracle.flash_attention(q, k, v, 0.125, 63, 64, threads=2), golden["bench_local_S512"])
    q, k, v = oracle.random_tensors(11, (1, 2, 128, 64), 3)
    assert_bit_exact(oracle.sdpa(q, k, v, None, 0.125), golden["bench_sdpa_S128"])


def test_rewrite_fixture_golden(oracle, golden):
    """Inputs of Rewrite.SemanticPreservationSingleLayer (rewrite_test.cpp:239-263)."""
    hidden = oracle.random_tensors(7, (1, 2, 96, 32), 1)[0]
    mask = np.ones((1, 1, 1, 96), np.float32)
    mask[..., -7:] = 0
    pb = oracle.pad_bias_from_mask(mask)
    assert_bit_exact(pb, golden["rewrite_pad_bias"])
    sc = 1.0 / np.sqrt(32.0)
    got = oracle.flash_attention(hidden, hidden, hidden, sc, 63, 64, pb)
    assert_bit_exact(got, golden["rewrite_local_S96_d32"])
    # the property that test asserts: fused op == original SDPA chain within 1e-3
    assert np.abs(got - golden["rewrite_local_S96_d32_sdpa"]).max() <= 1e-3


def test_mask2d_golden(oracle, golden):
    mask9 = np.ones((1, 1, 1, 96), np.float32)
    mask9[..., -9:] = 0
    assert_bit_exact(oracle.window_to_mask2d(96, 63, 64, oracle.pad_bias_from_mask(mask9)), golden["mask2d_S96_pad9"])
    assert_bit_exact(oracle.window_to_mask2d(3, 1, 1), golden["mask2d_S3_w11"])
    pb4 = np.zeros((1, 1, 1, 4), np.float32)
    pb4[..., 3] = -65504.0
    assert_bit_exact(oracle.window_to_mask2d(4, -1, -1, pb4), golden["mask2d_S4_padlast"])
    assert_bit_exact(oracle.window_to_mask2d(128, 63, 64), golden["mask2d_S128_w6364"])


def test_config1_golden(oracle, golden):
    q, k, v = [oracle.round_bf16(t) for t in oracle.random_tensors(11, (1, 2, 512, 64), 3)]
    assert_bit_exact(oracle.flash_attention(q, k, v), golden["cfg1_global_bf16in"])
    pb = np.zeros((1, 1, 1, 512), np.float32)
    pb[..., 475:] = -65504.0
    assert_bit_exact(oracle.flash_attention(q, k, v, 0.0, -1, -1, pb), golden["cfg1_global_pad475_bf16in"])
    assert_bit_exact(oracle.flash_attention(q, k, v, 0.0, 63, 64, pb, threads=2), golden["cfg1_local_pad475_bf16in"])


@pytest.mark.parametrize("S", [1, 2, 3, 5, 8, 37, 100])
def test_small_grid_golden(oracle, golden, S):
    q, k, v = oracle.random_tensors(100 + S, (2, 2, S, 32), 3)
    pb = np.zeros((2, 1, 1, S), np.float32)
    if S > 2:
        pb[1, 0, 0, S - max(1, S // 3):] = -65504.0
    for (wl, wr) in ((-1, -1), (0, 0), (1, 2), (63, 64)):
        assert_bit_exact(oracle.flash_attention(q, k, v, 0.0, wl, wr, pb), golden[f"grid_S{S}_w{wl}_{wr}"])


def test_additive_bias_and_dead_rows_golden(oracle, golden):
    q, k, v = oracle.random_tensors(77, (2, 1, 40, 32), 3)
    got = oracle.flash_attention(q, k, v, 0.3, -1, 5, golden["additive_bias_input"])
    assert_bit_exact(got, golden["additive_bias_and_dead_row"])
    assert np.all(got[1] == 0.0)  # every key masked -> zeros, not NaN (attention.cpp:175,204-207)


def test_memory_model_golden(oracle, golden):
    assert oracle.mask_memory_bytes(1, 12, 8192, 2) == int(golden["mem_mask_1_12_8192_2"][0]) == 1610612736
    assert oracle.mask_memory_bytes(1, 12, 16384, 2) == int(golden["mem_mask_1_12_16384_2"][0])
    assert oracle.fa_memory_bytes(1, 12, 8192, 64, 64, 2) == int(golden["mem_fa_1_12_8192_64_64_2"][0]) == 12779520


# ----------------------------------------------------------------------- live reference build
def test_port_bit_exact_with_reference_build(oracle):
    if not oracle.have_reference():
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    rng = np.random.default_rng(3)
    for (B, H, S, d, wl, wr, tile) in [(1, 1, 1, 32, -1, -1, 64), (2, 3, 70, 32, 5, 0, 16), (1, 2, 130, 64, 63, 64, 64),
                                       (2, 1, 65, 128, -1, 3, 1), (1, 2, 257, 64, -1, -1, 128)]:
        q, k, v = [rng.uniform(-1, 1, (B, H, S, d)).astype(np.float32) for _ in range(3)]
        pb = np.where(rng.uniform(size=(B, 1, 1, S)) < 0.2, -65504.0, 0.0).astype(np.float32)
        pb += np.where(pb == 0, rng.uniform(-1, 1, pb.shape) * (rng.uniform() < 0.5), 0).astype(np.float32)
        a = oracle.flash_attention(q, k, v, 0.0, wl, wr, pb, tile=tile, threads=3)
        b = oracle.flash_attention(q, k, v, 0.0, wl, wr, pb, tile=tile, impl="reference")
        assert_bit_exact(a, b)
        m = oracle.window_to_mask2d(S, wl, wr, pb)
        assert_bit_exact(m, oracle.window_to_mask2d(S, wl, wr, pb, impl="reference"))
        assert_bit_exact(oracle.sdpa(q, k, v, m, 0.2), oracle.sdpa(q, k, v, m, 0.2, impl="reference"))
    x = rng.uniform(-70000, 70000, 2000).astype(np.float32)
    assert_bit_exact(oracle.quantize_f16(x), oracle.quantize_f16(x, impl="reference"))
    assert oracle.effective_scale(0.0, 64) == oracle.effective_scale(0.0, 64, impl="reference") == 0.125


def test_reference_error_behaviour_is_mirrored(oracle):
    z = np.zeros((1, 1, 4, 8), np.float32)
    with pytest.raises(oracle.ShapeMismatch, match="identical shapes"):
        oracle.flash_attention(z, z, np.zeros((1, 1, 5, 8), np.float32))
    with pytest.raises(oracle.ShapeMismatch, match=r"\[B,H,S,d\]"):
        oracle.flash_attention(z[0], z[0], z[0])
    with pytest.raises(oracle.ShapeMismatch, match="tile"):
        oracle.flash_attention(z, z, z, tile=0)
    with pytest.raises(oracle.ShapeMismatch, match="pad_bias"):
        oracle.flash_attention(z, z, z, pad_bias=np.zeros((1, 1, 1, 5), np.float32))
    if oracle.have_reference():
        with pytest.raises(oracle.ShapeMismatch, match="pad_bias must be"):
            oracle.flash_attention(z, z, z, pad_bias=np.zeros((1, 1, 1, 5), np.float32), impl="reference")
        with pytest.raises(oracle.ShapeMismatch, match="tile must be"):
            oracle.flash_attention(z, z, z, tile=0, impl="reference")


# --------------------------------------------------------- SPEC known answers and invariants
def test_sdpa_known_answers(oracle):
    rng = np.random.default_rng(0)
    q, k, v = [rng.uniform(-1, 1, (1, 2, 1, 32)).astype(np.float32) for _ in range(3)]
    assert_bit_exact(oracle.sdpa(q, k, v, None, 0.3), v)  # S=1 -> O = V
    S = 16
    v = rng.uniform(-1, 1, (1, 1, S, 32)).astype(np.float32)
    q = np.zeros((1, 1, S, 32), np.float32)  # uniform scores -> row mean of V
    o = oracle.sdpa(q, v, v, None, 1.0)
    assert np.abs(o - v.mean(axis=2, keepdims=True)).max() <= 1e-6
    q, k, v = [rng.uniform(-1, 1, (1, 2, 37, 32)) for _ in range(3)]
    ref = oracle.sdpa_double_reference(q, k, v, 1 / np.sqrt(32))
    got = oracle.sdpa(q.astype(np.float32), k.astype(np.float32), v.astype(np.float32), None, 1 / np.sqrt(32))
    ref32 = oracle.sdpa_double_reference(q.astype(np.float32), k.astype(np.float32), v.astype(np.float32), 1 / np.sqrt(32))
    assert np.abs(got - ref32).max() <= 1e-6
    assert np.abs(got - ref).max() <= 1e-5


def test_flash_known_answers(oracle):
    rng = np.random.default_rng(1)
    q, k, v = [rng.uniform(-1, 1, (2, 2, 50, 32)).astype(np.float32) for _ in range(3)]
    # (-1,-1), no padding == sdpa with zero mask within 1e-5
    assert np.abs(oracle.flash_attention(q, k, v) - oracle.sdpa(q, k, v, None, 1 / np.sqrt(32))).max() <= 1e-5
    # window (0,0): each row attends only to itself -> O = V
    assert np.abs(oracle.flash_attention(q, k, v, 0.0, 0, 0) - v).max() <= 1e-6


@pytest.mark.parametrize("S", [100, 512, 1000])
def test_flash_equals_sdpa_with_mask2d(oracle, S):
    """window (63,64), random padding, non-tile-multiple S, within 1e-4."""
    rng = np.random.default_rng(S)
    H = 1 if S > 600 else 2
    q, k, v = [rng.uniform(-1, 1, (1, H, S, 32)).astype(np.float32) for _ in range(3)]
    pb = np.where(rng.uniform(size=(1, 1, 1, S)) < 0.15, -65504.0, 0.0).astype(np.float32)
    a = oracle.flash_attention(q, k, v, 0.0, 63, 64, pb, threads=2)
    b = oracle.sdpa(q, k, v, oracle.window_to_mask2d(S, 63, 64, pb), oracle.effective_scale(0.0, 32))
    assert np.abs(a - b).max() <= 1e-4


def test_invariants_grid_and_tiles(oracle):
    """S in {1..8,37,100} x windows x random padding; tiles {1,16,64,128} agree."""
    rng = np.random.default_rng(9)
    for S in list(range(1, 9)) + [37, 100]:
        q, k, v = [rng.uniform(-1, 1, (2, 2, S, 32)).astype(np.float32) for _ in range(3)]
        pb = np.where(rng.uniform(size=(2, 1, 1, S)) < 0.3, -65504.0, 0.0).astype(np.float32)
        for (wl, wr) in ((-1, -1), (0, 0), (1, 2), (63, 64)):
            base = oracle.flash_attention(q, k, v, 0.0, wl, wr, pb, tile=64)
            ref = oracle.sdpa(q, k, v, oracle.window_to_mask2d(S, wl, wr, pb), oracle.effective_scale(0.0, 32))
            assert np.abs(base - ref).max() <= 1e-4
            for tile in (1, 16, 128):
                assert np.abs(oracle.flash_attention(q, k, v, 0.0, wl, wr, pb, tile=tile) - base).max() <= 1e-6
            assert not np.isnan(base).any()


def test_window_predicate_bruteforce(oracle):
    """SPEC.md:517 with the reference tests' own predicate (oracles.cpp:123-129)."""
    m = oracle.window_to_mask2d(128, 63, 64)[0, 0]
    for i in range(128):
        for j in range(128):
            assert (m[i, j] == 0.0) == oracle.window_live_reference(i, j, 63, 64)
            assert (m[i, j] == 0.0) == (i - 63 <= j <= i + 64)


def test_memory_model_properties(oracle):
    for S in (1024, 4096, 16384):
        assert oracle.mask_memory_bytes(1, 12, S, 2) == 4 * oracle.mask_memory_bytes(1, 12, S // 2, 2)
    budget = 718 * 1000 * 1000
    fails = [S for S in (512, 1024, 2048, 4096, 8192, 16384) if oracle.mask_memory_bytes(1, 12, S, 2) > budget]
    assert fails[0] == 8192  # crossover in (4096, 8192], SPEC.md:544
    assert oracle.flash_stats(1, 2, 96, 32, 64) == {"tile_scratch_floats": 64, "row_state_floats": 192,
                                                    "output_floats": 1 * 2 * 96 * 32}


def test_live_pairs_counts(oracle):
    assert oracle.live_pairs(8192, -1, -1) == 8192 * 8192
    assert oracle.live_pairs(10, 0, 0) == 10
    S = 300
    pb = np.zeros(S, np.float32)
    pb[250:] = -65504.0
    m = oracle.window_to_mask2d(S, 63, 64, pb.reshape(1, 1, 1, S))[0, 0]
    assert oracle.live_pairs(S, 63, 64, pb) == int((m == 0).sum())
