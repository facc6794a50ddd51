#!/usr/bin/env python
"""Developer tool (under gpurun): the classifier's four projection shapes at 8K tokens, rf_gemm_nt vs the library GEMM
(torch.matmul -> cuBLAS), CUDA-graph replay, TFLOP/s."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_12646_b200 as P
from paper_2603_12646_b200.gemm import gemm_nt
from paper_2603_12646_b200.classifier import rope_tables

def timeit(fn, n=20):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(4): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (n * 4)

M = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
res = {}
for dtype in (torch.bfloat16,):
    for name, N, K, epi in (("qkv", 2304, 768, "none"), ("qkv+rope", 2304, 768, "rope"), ("out_proj", 768, 768, "none"),
                            ("wi", 2304, 768, "none"), ("wi+geglu", 2304, 768, "geglu"), ("wo2", 768, 1152, "none"), ("out_proj+res", 768, 768, "residual"),
                            ("wo2+res", 768, 1152, "residual")):
        a = torch.randn(M, K, device="cuda").to(dtype)
        w = (torch.randn(N, K, device="cuda") * 0.05).to(dtype)
        cos, sin = rope_tables(M, 64, 10000.0, "cuda")
        out = torch.empty(M, N // 2 if epi == "geglu" else N, device="cuda", dtype=torch.float32 if epi == "residual" else dtype)
        kw = dict(epilogue=epi, rope_cos=cos, rope_sin=sin, seq_len=M) if epi == "rope" else dict(epilogue=epi)
        ms = timeit(lambda: gemm_nt(a, w, out=out, **kw))
        lib_out = torch.empty(M, N, device="cuda", dtype=dtype)
        ms_lib = timeit(lambda: torch.matmul(a, w.t(), out=lib_out))
        fl = 2.0 * M * N * K
        res[name] = {"us": round(ms * 1e3, 1), "tflops": round(fl / ms / 1e9), "cublas_us": round(ms_lib * 1e3, 1), "cublas_tflops": round(fl / ms_lib / 1e9)}
lib = P.capi.load()
x = torch.randn(M, 768, device="cuda"); d16 = torch.randn(M, 768, device="cuda").to(torch.bfloat16); wn = torch.ones(768, device="cuda"); y = torch.empty_like(d16)
st = lambda: torch.cuda.current_stream().cuda_stream
res["add_layernorm_us"] = round(timeit(lambda: P.capi.check(lib.rf_add_layernorm(x.data_ptr(), d16.data_ptr(), wn.data_ptr(), y.data_ptr(), M, 768, 1e-5, 0, st()))) * 1e3, 1)
res["layernorm_only_us"] = round(timeit(lambda: P.capi.check(lib.rf_add_layernorm(x.data_ptr(), None, wn.data_ptr(), y.data_ptr(), M, 768, 1e-5, 0, st()))) * 1e3, 1)
print(json.dumps(res))
