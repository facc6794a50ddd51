"""Developer probe: the 8K dense op through rf_fa_plan launches, stream mode vs CUDA-graph replay (device time per op)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2603_12646_b200 as P
from paper_2603_12646_b200.attention import FaPlan

def run(S=8192, n=6, iters=20):
    g = torch.Generator(device="cuda").manual_seed(1)
    sets = [[(torch.rand(1, 12, S, 64, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)] for _ in range(n)]
    outs = [torch.empty_like(s[0]) for s in sets]
    plans = [FaPlan(*sets[i], P.AttentionSpec(), out=outs[i]) for i in range(n)]
    for pl in plans: pl.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters * n): plans[i % n].launch()
    e1.record(); torch.cuda.synchronize()
    t_stream = e0.elapsed_time(e1) / (iters * n)
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for pl in plans: pl.launch()
    torch.cuda.current_stream().wait_stream(side); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for pl in plans: pl.launch()
    gr.replay(); torch.cuda.synchronize()
    e0.record()
    for _ in range(iters): gr.replay()
    e1.record(); torch.cuda.synchronize()
    t_graph = e0.elapsed_time(e1) / (iters * n)
    f = 4.0 * 12 * S * S * 64
    print(f"S={S} plan/stream {t_stream*1e3:.1f} us ({f/t_stream/1e9:.0f} TFLOP/s)  plan/graph {t_graph*1e3:.1f} us ({f/t_graph/1e9:.0f} TFLOP/s)")

for S in (8192, 16384):
    run(S, 6 if S == 8192 else 3)
