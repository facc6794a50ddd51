import os, sys, time, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2603_12646_b200 as P
B,H,S,D=1,12,8192,64
host=[torch.rand((B,H,S,D),dtype=torch.float32).pin_memory() for _ in range(3)]
dev=[torch.empty((B,H,S,D),device='cuda') for _ in range(3)]
ho=torch.empty((B,H,S,D),dtype=torch.float32,pin_memory=True)
for _ in range(3):
    for h,d in zip(host,dev): d.copy_(h,non_blocking=True)
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(10):
    for h,d in zip(host,dev): d.copy_(h,non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/10
print("H2D 75.5MB ms", dt*1e3, "GB/s", 75.5e-3/dt)
t=time.perf_counter()
for _ in range(10): ho.copy_(dev[0],non_blocking=True)
torch.cuda.synchronize(); dt=(time.perf_counter()-t)/10
print("D2H 25MB ms", dt*1e3, "GB/s", 25.2e-3/dt)
hq,hk,hv=[h.numpy() for h in host]
for _ in range(4): o=P.flash_attention(hq,hk,hv,P.AttentionSpec())
os.environ["RF_FA_HOST_TIMING"]="1"
t=time.perf_counter(); o=P.flash_attention(hq,hk,hv,P.AttentionSpec()); print("call ms",(time.perf_counter()-t)*1e3)
t=time.perf_counter(); o=P.flash_attention(hq,hk,hv,P.AttentionSpec()); print("call ms",(time.perf_counter()-t)*1e3)
