import torch, sys
sys.path.insert(0, '.')
import paper_2603_12646_b200 as P
g = torch.Generator(device="cuda").manual_seed(3)
def rep(name, B, H, S, wl, wr, n=300, pad=None):
    q,k,v = [(torch.rand((B,H,S,64), device="cuda", generator=g)*2-1).to(torch.bfloat16) for _ in range(3)]
    pb = None
    if pad:
        pb = torch.zeros((B,1,1,S), device="cuda"); pb[..., pad:] = -65504.0
    spec = P.AttentionSpec(0.0, wl, wr, pb)
    st = P.FlashStats()
    o0 = P.flash_attention(q,k,v,spec,out_dtype=torch.float32, stats=st)
    bad = []
    for i in range(n):
        o = P.flash_attention(q,k,v,spec,out_dtype=torch.float32)
        if not torch.equal(o, o0):
            d = (o-o0).abs()
            nz = (d.amax(-1) > 0).nonzero()
            bad.append((i, d.max().item(), len(nz), nz[:3].tolist(), nz[-1].tolist()))
    print(name, "grid", st.grid_ctas, "mismatches", len(bad), bad[:4], flush=True)
rep("global8k_mode1", 1, 12, 8192, -1, -1)
rep("local8k_mode1", 1, 12, 8192, 63, 64, n=600)
rep("local8k_pad_mode1", 1, 12, 8192, 63, 64, pad=7000)
rep("global2k_mode0", 1, 12, 2048, -1, -1)
rep("local2k_mode0", 1, 12, 2048, 63, 64, n=600)
rep("local4k_b1_mode0", 1, 12, 4096, 63, 64, n=600)
