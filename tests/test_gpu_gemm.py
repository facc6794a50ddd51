"""GPU tests of the hand-written projections (include/rf_gemm.h) against plain PyTorch fp32 references of the same
op: y = a @ w^T, the fused RoPE epilogue vs rotate-half RoPE on the fp32 product, the fused GeGLU epilogue vs
gelu(in) * gate on the fp32 product.  Tolerance: the 16-bit rounding of the output (2^-8 relative for bf16,
2^-11 for f16) plus f32 accumulation-order noise."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rand(shape, dtype, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(shape, device="cuda", generator=g) * scale).to(dtype)


def _tol(dtype):
    return 2.0 ** -7 if dtype == torch.bfloat16 else 2.0 ** -10


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (1000, 768, 768), (8192, 2304, 768), (300, 768, 1152), (129, 256, 72)])
def test_gemm_nt_matches_fp32_reference(dtype, M, N, K):
    from paper_2603_12646_b200.gemm import gemm_nt
    a, w = _rand((M, K), dtype, 1), _rand((N, K), dtype, 2, 0.05)
    y = gemm_nt(a, w)
    torch.cuda.synchronize()
    want = a.float() @ w.float().t()
    err = (y.float() - want).abs().max().item()
    assert err <= _tol(dtype) * max(1.0, want.abs().max().item()), err


def test_gemm_nt_strided_operands_and_output():
    """A row slice of a wider activation buffer in, a column slice of a wider buffer out (the classifier's slots)."""
    from paper_2603_12646_b200.gemm import gemm_nt
    big = _rand((513, 1024), torch.bfloat16, 3)
    a = big[:, 128:896]                                   # [513, 768], row stride 1024
    w = _rand((512, 768), torch.bfloat16, 4, 0.05)
    out_big = torch.zeros((513, 1024), device="cuda", dtype=torch.bfloat16)
    gemm_nt(a, w, out=out_big[:, 256:768])
    torch.cuda.synchronize()
    want = a.float() @ w.float().t()
    assert (out_big[:, 256:768].float() - want).abs().max().item() <= 2.0 ** -7 * want.abs().max().item()
    assert not out_big[:, :256].any() and not out_big[:, 768:].any()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_gemm_rope_epilogue(dtype):
    """Packed QKV projection with rotary embedding on the Q and K thirds, against RoPE applied to the fp32 product."""
    from paper_2603_12646_b200.classifier import rope_tables
    from paper_2603_12646_b200.gemm import gemm_nt
    B, S, H, d, hid = 2, 300, 12, 64, 768
    a, w = _rand((B * S, hid), dtype, 5), _rand((3 * hid, hid), dtype, 6, 0.05)
    cos, sin = rope_tables(S, d, 10000.0, "cuda")
    y = gemm_nt(a, w, epilogue="rope", rope_cos=cos, rope_sin=sin, seq_len=S)
    torch.cuda.synchronize()
    ref = (a.float() @ w.float().t()).view(B, S, 3, H, d)
    c = cos.view(1, S, 1, 1, d // 2)
    s = sin.view(1, S, 1, 1, d // 2)
    x1, x2 = ref[:, :, :2, :, : d // 2], ref[:, :, :2, :, d // 2:]
    want = ref.clone()
    want[:, :, :2, :, : d // 2] = x1 * c - x2 * s
    want[:, :, :2, :, d // 2:] = x2 * c + x1 * s
    err = (y.float().view(B, S, 3, H, d) - want).abs().max().item()
    assert err <= _tol(dtype) * want.abs().max().item(), err


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_gemm_geglu_epilogue(dtype):
    from paper_2603_12646_b200.gemm import gemm_nt
    M, K, I = 700, 768, 1152
    a, w = _rand((M, K), dtype, 7), _rand((2 * I, K), dtype, 8, 0.05)
    y = gemm_nt(a, w, epilogue="geglu")
    torch.cuda.synchronize()
    ref = a.float() @ w.float().t()
    want = torch.nn.functional.gelu(ref[:, :I]) * ref[:, I:]
    assert y.shape == (M, I)
    err = (y.float() - want).abs().max().item()
    assert err <= _tol(dtype) * max(1.0, want.abs().max().item()), err


def test_gemm_rejects_unsupported_shapes():
    from paper_2603_12646_b200 import capi
    from paper_2603_12646_b200.gemm import gemm_nt
    a, w = _rand((64, 64), torch.bfloat16, 9), _rand((100, 64), torch.bfloat16, 10)
    with pytest.raises(capi.RfError):
        gemm_nt(a, w)                                      # N not a multiple of 256


def test_gemm_is_bitwise_deterministic():
    from paper_2603_12646_b200.gemm import gemm_nt
    a, w = _rand((2048, 768), torch.bfloat16, 11), _rand((768, 768), torch.bfloat16, 12, 0.05)
    first = gemm_nt(a, w)
    for _ in range(20):
        assert torch.equal(first, gemm_nt(a, w))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("M,N,K", [(1000, 768, 768), (8192, 768, 1152), (130, 256, 64)])
def test_gemm_residual_epilogue(dtype, M, N, K):
    """x (f32) += a @ w^T by TMA reduce-add of the f32 accumulators: nothing is rounded to 16 bit on the way."""
    from paper_2603_12646_b200.gemm import gemm_nt
    a, w = _rand((M, K), dtype, 13), _rand((N, K), dtype, 14, 0.05)
    x0 = torch.randn(M, N, device="cuda")
    x = x0.clone()
    gemm_nt(a, w, out=x, epilogue="residual")
    torch.cuda.synchronize()
    want = x0.double() + a.double() @ w.double().t()
    assert (x.double() - want).abs().max().item() <= 1e-4 * max(1.0, want.abs().max().item())
    # a second call accumulates again
    gemm_nt(a, w, out=x, epilogue="residual")
    torch.cuda.synchronize()
    want2 = want + a.double() @ w.double().t()
    assert (x.double() - want2).abs().max().item() <= 2e-4 * max(1.0, want2.abs().max().item())


def test_gemm_rope_head_major_layout_and_bf16_output():
    """The QKV projection can write [3*H, tokens, 64] (every head's rows contiguous) and in the other 16-bit type."""
    from paper_2603_12646_b200.classifier import rope_tables
    from paper_2603_12646_b200.gemm import gemm_nt
    B, S, H, d, hid = 2, 200, 12, 64, 768
    a, w = _rand((B * S, hid), torch.float16, 15), _rand((3 * hid, hid), torch.float16, 16, 0.05)
    cos, sin = rope_tables(S, d, 160000.0, "cuda")
    packed = gemm_nt(a, w, epilogue="rope", rope_cos=cos, rope_sin=sin, seq_len=S)
    heads = gemm_nt(a, w, epilogue="rope", rope_cos=cos, rope_sin=sin, seq_len=S, head_major=True)
    torch.cuda.synchronize()
    assert heads.shape == (3 * H, B * S, d)
    assert torch.equal(heads, packed.view(B * S, 3 * H, d).permute(1, 0, 2))
    heads_bf = gemm_nt(a, w, epilogue="rope", rope_cos=cos, rope_sin=sin, seq_len=S, head_major=True, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert heads_bf.dtype == torch.bfloat16
    assert (heads_bf.float() - heads.float()).abs().max().item() <= 2.0 ** -7 * heads.float().abs().max().item()


def test_gemm_launch_status_reports_ok():
    """Bounded waits: the status word of the projections is clean after normal launches (include/rf_gemm.h)."""
    from paper_2603_12646_b200 import capi
    from paper_2603_12646_b200.gemm import gemm_nt
    a, w = _rand((512, 768), torch.bfloat16, 17), _rand((768, 768), torch.bfloat16, 18, 0.05)
    gemm_nt(a, w)
    assert capi.load().rf_gemm_launch_status(torch.cuda.current_stream().cuda_stream) == capi.RF_OK
