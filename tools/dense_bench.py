import json, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2603_12646_b200 as P
def t(S, B=1, iters=20, sets_n=6):
    g = torch.Generator(device="cuda").manual_seed(1)
    sets = [[(torch.rand(B, 12, S, 64, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)] for _ in range(sets_n)]
    outs = [torch.empty_like(s[0]) for s in sets]
    spec = P.AttentionSpec()
    for i in range(sets_n): P.flash_attention(*sets[i], spec, out=outs[i])
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for i in range(sets_n): P.flash_attention(*sets[i], spec, out=outs[i])
    gr.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): gr.replay()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (iters * sets_n)
    return ms, 4.0 * B * 12 * S * S * 64 / ms / 1e9
for S, n in ((8192, 6), (16384, 3), (32768, 2)):
    ms, tf = t(S, 1, 20 if S < 32768 else 5, n)
    print(f"S={S}: {ms*1e3:.1f} us  {tf:.0f} TFLOP/s", end="; ")
print()
