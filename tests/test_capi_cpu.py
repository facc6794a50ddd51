"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every symbol
include/rf_fa.h, include/rf_graph.h and include/rf_clf.h declare, validates like the reference, and fails loudly without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_12646_b200 import capi
    return capi.load()


def header_functions():
    names = set()
    for header in ("rf_fa.h", "rf_graph.h", "rf_clf.h", "rf_gemm.h"):
        text = open(os.path.join(ROOT, "include", header)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(rf_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_library_exports_every_declared_symbol(lib):
    from paper_2603_12646_b200 import capi
    declared = header_functions()
    assert len(declared) >= 18
    assert sorted(capi.EXPORTS) == declared
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.rf_abi_version() == 1


def test_params_init_layout_and_defaults(lib):
    from paper_2603_12646_b200 import capi
    p = capi.new_params()
    assert (p.window_left, p.window_right, p.scale) == (-1, -1, 0.0)
    assert (p.dtype, p.out_dtype, p.kernel, p.flags) == (capi.RF_DTYPE_BF16, capi.RF_DTYPE_BF16, capi.RF_KERNEL_AUTO, 0)
    assert p.q is None and p.pad_bias is None and p.o_partial is None
    assert list(p.q_stride) == [0, 0, 0]


def test_validation_mirrors_reference_errors(lib):
    from paper_2603_12646_b200 import capi
    p = capi.new_params()
    p.B, p.H, p.S, p.d = 1, 2, 16, 48
    p.q = p.k = p.v = p.out = 0x1000
    assert lib.rf_fa_validate(C.byref(p)) == capi.RF_ERR_HEAD_DIM
    assert b"head_dim must be one of {32, 64, 128}, got 48" in lib.rf_last_error()  # rewrite.cpp:266-269
    with pytest.raises(capi.UnsupportedHeadDim):
        capi.check(capi.RF_ERR_HEAD_DIM)
    p.d = 64
    assert lib.rf_fa_validate(C.byref(p)) == capi.RF_OK
    p.B = -1
    assert lib.rf_fa_validate(C.byref(p)) == capi.RF_ERR_SHAPE
    p.B = 1
    p.kv_begin, p.kv_end = 8, 4
    assert lib.rf_fa_validate(C.byref(p)) == capi.RF_ERR_ARG
    p.kv_begin, p.kv_end = 0, 0
    # every head dim of the reference contract runs on the tensor cores (rewrite.cpp:266-269)
    st = capi.RfFaStats()
    for d in (32, 64, 128):
        p.d, p.kernel = d, capi.RF_KERNEL_TCGEN05
        assert lib.rf_fa_validate(C.byref(p)) == capi.RF_OK
        p.kernel = capi.RF_KERNEL_AUTO
        assert lib.rf_fa_stats_query(C.byref(p), C.byref(st)) == capi.RF_OK
        assert st.kernel == capi.RF_KERNEL_TCGEN05 and st.score_matrix_bytes == 0
    # forcing the tensor-core kernel onto a call it does not cover is an explicit error; AUTO falls back to the
    # generic CUDA-core kernel (still on the device)
    p.d, p.scale, p.kernel = 64, -0.5, capi.RF_KERNEL_TCGEN05
    assert lib.rf_fa_validate(C.byref(p)) == capi.RF_ERR_UNSUPPORTED
    p.kernel = capi.RF_KERNEL_AUTO
    assert lib.rf_fa_stats_query(C.byref(p), C.byref(st)) == capi.RF_OK
    assert st.kernel == capi.RF_KERNEL_SIMT and st.score_matrix_bytes == 0
    p.scale = 0.0
    p.flags = 1
    assert lib.rf_fa_validate(C.byref(p)) == capi.RF_ERR_ARG   # reserved, must be 0
    p.flags = 0


def test_workspace_is_linear_in_S(lib):
    from paper_2603_12646_b200 import capi
    sizes = {}
    for S in (8192, 16384, 32768):
        p = capi.new_params()
        p.B, p.H, p.S, p.d = 1, 12, S, 64
        p.q = p.k = p.v = p.out = 0x1000
        p.pad_bias = 0x2000
        n = C.c_size_t()
        assert lib.rf_fa_fwd_workspace_bytes(C.byref(p), C.byref(n)) == capi.RF_OK
        sizes[S] = n.value
        st = capi.RfFaStats()
        lib.rf_fa_stats_query(C.byref(p), C.byref(st))
        assert st.kernel == capi.RF_KERNEL_TCGEN05 and st.grid_ctas == 148  # persistent: one CTA per SM
        assert st.row_state_bytes == 8 * S
    # O(S): bias (4 B/key + 1 B/tile) and the row-max skip test's key norms (4 B per (head, key tile); the query norms
    # are taken inside the kernel) on top of the constant split-pair block of the persistent schedule
    per_key = 4 + (1 + 4 * 12) / 128.0
    assert sizes[16384] - sizes[8192] <= 8192 * per_key + 1024 and sizes[32768] - sizes[16384] <= 16384 * per_key + 1024
    assert sizes[32768] < 11 * 1024 * 1024
    # dense global attention over more query-tile pairs than SMs runs the persistent balanced schedule: its
    # split-pair workspace is a constant (per-SM); only the key norms grow, linearly.  A single sequence whose K/V
    # outgrow the L2 (32K tokens: 100 MB) is dealt round-robin as whole pairs instead: no split-pair block at all.
    p.pad_bias = None
    dense = []
    for S in (8192, 16384, 32768):
        p.S = S
        assert lib.rf_fa_fwd_workspace_bytes(C.byref(p), C.byref(n)) == capi.RF_OK
        dense.append(n.value)
    assert 0 < dense[0] < dense[1] < 11 * 1024 * 1024
    assert dense[1] - dense[0] <= (16384 - 8192) * (4 * 12 / 128.0) + 1024
    assert 0 < dense[2] < 64 * 1024                      # status block + flag block + 12 KiB of key norms
    p.S = 512  # 24 pairs fit one wave: one pair per CTA, nothing but the 256-byte launch-status block
    assert lib.rf_fa_fwd_workspace_bytes(C.byref(p), C.byref(n)) == capi.RF_OK and n.value == 256


def test_host_entry_checks_in_reference_order(lib):
    """tile, then pad_bias shape (attention.cpp:110-116) -- both before any CUDA call."""
    import paper_2603_12646_b200 as P
    z = np.zeros((1, 1, 4, 64), np.float32)
    with pytest.raises(P.ShapeMismatch, match="tile must be >= 1"):
        P.flash_attention(z, z, z, P.AttentionSpec(), tile=0)
    with pytest.raises(P.ShapeMismatch, match=r"pad_bias must be \[B,1,1,S\]"):
        P.flash_attention(z, z, z, P.AttentionSpec(pad_bias=np.zeros((1, 1, 1, 5), np.float32)))
    with pytest.raises(P.ShapeMismatch, match="identical shapes"):
        P.flash_attention(z, z, np.zeros((1, 1, 5, 64), np.float32))
    with pytest.raises(P.ShapeMismatch, match=r"\[B,H,S,d\]"):
        P.flash_attention(z[0], z[0], z[0])


def test_no_cpu_fallback_without_gpu(lib):
    import torch

    import paper_2603_12646_b200 as P
    from paper_2603_12646_b200 import capi
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    z = np.zeros((1, 1, 4, 64), np.float32)
    with pytest.raises(capi.RfError) as ei:
        P.flash_attention(z, z, z)
    assert ei.value.code == capi.RF_ERR_CUDA
    assert lib.rf_device_check(0, None, None, None) == capi.RF_ERR_CUDA


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2603_12646_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, flags=re.M), f
                assert "librf_oracle" not in src and "libref_attn" not in src, f


def test_memory_model_and_window_attrs():
    import paper_2603_12646_b200 as P
    assert P.mask_memory_bytes(1, 12, 8192, 2) == 1610612736
    assert P.mask_memory_bytes(1, 12, 16384, 2) == 4 * 1610612736
    assert P.fa_memory_bytes(1, 12, 8192, 64, 64, 2) == 12779520
    assert P.local_window_attrs() == (63, 64)                           # rewrite.cpp:355-357
    assert P.local_window_attrs(is_global=True) == (-1, -1)
    assert P.local_window_attrs(P.RewriteOptions(local_window=2)) == (0, 1)
    with pytest.raises(P.UnsupportedHeadDim):
        P.local_window_attrs(P.RewriteOptions(head_dim=48))
    with pytest.raises(ValueError):
        P.local_window_attrs(P.RewriteOptions(local_window=3))
    assert P.AttentionSpec().effective_scale(64) == 0.125               # attention.cpp:34-36
    assert P.AttentionSpec(scale=0.5).effective_scale(64) == 0.5
    assert (P.kMaskValue, P.kMaskThreshold) == (-65504.0, -30000.0)


def test_classifier_session_fails_loudly_without_gpu(lib):
    """rf_clf.h: config defaults and blob size are host logic; creating a session without a CUDA device is
    an error (RF_ERR_CUDA), never a CPU path."""
    import ctypes as C
    from paper_2603_12646_b200 import capi
    c = capi.RfClfConfig()
    lib.rf_clf_config_default(C.byref(c))
    assert (c.vocab_size, c.hidden, c.n_layers, c.heads, c.head_dim, c.mlp, c.n_labels) == (50368, 768, 22, 12, 64, 1152, 3)
    per_layer = 768 + 3 * 768 * 768 + 768 * 768 + 768 + 2 * 1152 * 768 + 768 * 1152
    assert lib.rf_clf_weight_elems(C.byref(c)) == 50368 * 768 + 3 * 768 + 768 * 768 + 3 * 768 + 3 + 22 * per_layer
    h = C.c_void_p()
    one = (C.c_float * 1)(0.0)
    assert lib.rf_clf_create(C.byref(c), one, 1, 0, C.byref(h)) == capi.RF_ERR_SHAPE
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        has_gpu = False
    if not has_gpu:
        c.vocab_size, c.n_layers = 16, 1
        n = lib.rf_clf_weight_elems(C.byref(c))
        blob = (C.c_float * n)()
        assert lib.rf_clf_create(C.byref(c), blob, n, 0, C.byref(h)) == capi.RF_ERR_CUDA
        assert not h.value


def test_host_rounding_is_round_to_nearest_even_bit_for_bit(lib):
    """rf_host_round_bf16 (the rounding rf_fa_fwd_host applies to Q, K, V on the host cores before they cross the link):
    identical to torch's f32 -> bf16 conversion, which is what the device cast gives -- ties, subnormals, infinities,
    NaN (stays NaN), negative zero; through the thread pool (large n) and on the calling thread (small n)."""
    import torch
    from paper_2603_12646_b200 import capi
    rng = np.random.default_rng(5)
    special = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 1e-40, -1e-40, 3.3895314e38, 65504.0, 1.00390625,
                        1.01171875, 1.005859375, 0.99609375], np.float32)
    ties = (np.arange(1, 4097, dtype=np.uint32) << 15).view(np.float32)   # every pattern that ends in ...1000 0000 0000 0000 or 0
    for n in (special.size + ties.size + 1000, 3 * 12 * 4096 * 64 + 7):
        x = rng.standard_normal(n).astype(np.float32) * np.float32(10.0) ** rng.integers(-6, 6, n).astype(np.float32)
        x[:special.size] = special
        x[special.size:special.size + ties.size] = ties
        bits = rng.integers(0, 2 ** 32, 4096, dtype=np.uint64).astype(np.uint32).view(np.float32)  # raw bit patterns
        x[-bits.size:] = bits
        out = np.empty(n, np.uint16)
        rc = lib.rf_host_round_bf16(x.ctypes.data_as(C.POINTER(C.c_float)), out.ctypes.data_as(C.POINTER(C.c_uint16)), n)
        assert rc == capi.RF_OK
        want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        nan = np.isnan(x)
        assert np.array_equal(out[~nan], want[~nan])
        assert np.all((out[nan] & 0x7fff) > 0x7f80)          # still NaN (payloads may differ between converters)
    lib.rf_fa_host_release()                                  # joins the pool; a later call restarts it
    x = np.linspace(-3, 3, 1 << 17, dtype=np.float32)
    out = np.empty(x.size, np.uint16)
    assert lib.rf_host_round_bf16(x.ctypes.data_as(C.POINTER(C.c_float)), out.ctypes.data_as(C.POINTER(C.c_uint16)), x.size) == capi.RF_OK
    assert np.array_equal(out, torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16))
