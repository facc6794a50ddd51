"""Developer probe: the head_dim-128 kernel at 8K / 16K through rf_fa_plan launches (burst: 0.5 s idle, 3 warm-up, 20 timed)."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_2603_12646_b200 as P
from paper_2603_12646_b200.attention import FaPlan
for S in (8192, 16384):
    g = torch.Generator(device="cuda").manual_seed(1)
    n = 4
    sets = [[(torch.rand(1, 12, S, 128, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) for _ in range(3)] for _ in range(n)]
    outs = [torch.empty_like(s[0]) for s in sets]
    plans = [FaPlan(*sets[i], P.AttentionSpec(), out=outs[i]) for i in range(n)]
    for pl in plans:
        pl.launch(); pl.launch()
    torch.cuda.synchronize()
    time.sleep(0.5)
    for i in range(3): plans[i % n].launch()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20): plans[i % n].launch()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"d128 S={S}: {ms*1e3:.1f} us {4.0*12*S*S*128/ms/1e9:.0f} TFLOP/s  (workspace {plans[0].stats.workspace_bytes} B)")
