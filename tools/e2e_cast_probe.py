import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2603_12646_b200 as P
B,H,S,D=1,12,8192,64
host=[torch.empty((B,H,S,D),dtype=torch.float32,pin_memory=True) for _ in range(3)]
g=torch.Generator().manual_seed(0)
for t in host: t.copy_(torch.rand((B,H,S,D),generator=g)*2-1)
hq,hk,hv=[t.numpy() for t in host]
spec=P.AttentionSpec()
for _ in range(6): out=P.flash_attention(hq,hk,hv,spec,device=0)
t0=time.perf_counter()
for _ in range(20): out=P.flash_attention(hq,hk,hv,spec,device=0)
dt=(time.perf_counter()-t0)/20
print("e2e %.3f ms  %.1f TFLOP/s  cast threads env=%s" % (dt*1e3, 4.0*B*H*S*S*D/dt/1e12, os.environ.get("RF_FA_HOST_CAST","default")))
# reference result through the device-cast path must be identical
os.environ["RF_FA_HOST_TIMING"]="1"
out2=P.flash_attention(hq,hk,hv,spec,device=0)
