"""CPU tests of the N > 1 host logic with world_size-2 gloo process groups: the split-KV
exchange sequence (with numpy stand-ins for the three device steps -- test infrastructure) and
the request-batch scheduler."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class NumpyOps:
    """Stand-in for the CUDA steps so that the collective sequence can run on CPU."""

    def partial(self, q, k, v, spec, kv_range):
        B, H, S, d = q.shape
        scale = spec.effective_scale(d) * 1.4426950408889634
        s = torch.einsum("bhid,bhjd->bhij", q.double(), k.double()) * scale
        i = torch.arange(S)[:, None]
        j = torch.arange(S)[None, :]
        live = ((j >= kv_range[0]) & (j < kv_range[1])).expand(S, S).clone()
        if spec.window_left >= 0:
            live &= (i - j) <= spec.window_left
        if spec.window_right >= 0:
            live &= (j - i) <= spec.window_right
        live = live[None, None].expand(B, 1, S, S)
        if spec.pad_bias is not None:
            pb = torch.as_tensor(spec.pad_bias).double()
            s = s + pb * 1.4426950408889634
            live = live & (pb > -30000.0)
        s = s.masked_fill(~live, float("-inf"))
        m = s.amax(-1)
        msafe = torch.where(torch.isinf(m), torch.zeros_like(m), m)
        p = torch.exp2(s - msafe[..., None])
        return (p @ v.double()).float(), m.float(), p.sum(-1).float()

    def rescale(self, o, l, m, m_star):
        w = torch.where(torch.isinf(m), torch.zeros_like(m), torch.exp2(m - m_star))
        o.mul_(w[..., None])
        l.mul_(w)

    def normalize(self, o_sum, l_sum, out_dtype):
        safe = torch.where(l_sum > 0, l_sum, torch.ones_like(l_sum))
        return torch.where(l_sum[:, None] > 0, o_sum / safe[:, None], torch.zeros_like(o_sum)).to(out_dtype)


def _splitkv_worker(rank, world, port, S, wl, wr, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_12646_b200.attention import AttentionSpec
        from paper_2603_12646_b200.splitkv import split_kv_attention
        g = torch.Generator().manual_seed(0)
        q, k, v = [torch.rand((1, 2, S, 32), generator=g) * 2 - 1 for _ in range(3)]
        pb = torch.zeros((1, 1, 1, S))
        pb[..., S - S // 5:] = -65504.0
        spec = AttentionSpec(0.0, wl, wr, pb)
        out = split_kv_attention(q, k, v, spec, ops=NumpyOps())
        if rank == 0:
            ret["out"] = out.numpy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("S,wl,wr", [(300, -1, -1), (257, 63, 64), (100, 1, 2)])
def test_split_kv_exchange_sequence_gloo(oracle, S, wl, wr):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        ret = mgr.dict()
        procs = [ctx.Process(target=_splitkv_worker, args=(r, world, port, S, wl, wr, ret))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        got = ret["out"]
    g = torch.Generator().manual_seed(0)
    q, k, v = [(torch.rand((1, 2, S, 32), generator=g) * 2 - 1).numpy() for _ in range(3)]
    pb = np.zeros((1, 1, 1, S), np.float32)
    pb[..., S - S // 5:] = -65504.0
    want = oracle.flash_attention(q, k, v, 0.0, wl, wr, pb)
    assert np.abs(got - want).max() <= 1e-5



def test_kv_blocks_partition():
    from paper_2603_12646_b200.splitkv import kv_block
    for S in (1, 100, 128, 129, 1000, 32768):
        for world in (1, 2, 3, 4, 8):
            blocks = [kv_block(S, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == S
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0 and a0 <= a1
            assert all(b0 % 128 == 0 for b0, _ in blocks)
    assert kv_block(32768, 3, 8) == (12288, 16384)


def test_lpt_assignment_properties():
    from paper_2603_12646_b200.scheduler import ModelShape, Unit, attention_flops, lpt_assign, makespan, unit_cost
    shape = ModelShape()
    # config 3: 3 classifiers x batch 4 at S = 16384 -> 12 equal units; ideal speed-up at G=8 is 6x
    units = [Unit(i, m, r, 16384) for i, (m, r) in enumerate((m, r) for m in ("safety", "domain", "pii") for r in range(4))]
    for G in (1, 2, 4, 8):
        a = lpt_assign(units, G, shape)
        assert sorted(u.uid for part in a for u in part) == list(range(12))
        sizes = sorted(len(p) for p in a)
        assert sizes[-1] == -(-12 // G) and sizes[-1] - sizes[0] <= 1
    assert makespan(lpt_assign(units, 1, shape), shape) / makespan(lpt_assign(units, 8, shape), shape) == pytest.approx(6.0)
    # mixed lengths: LPT never exceeds 4/3 of the lower bound, and is deterministic
    rng = np.random.default_rng(0)
    mixed = [Unit(i, "safety", i, int(s), int(s * f)) for i, (s, f) in
             enumerate(zip(rng.choice([512, 2048, 8192, 32768], 40), rng.uniform(0.5, 1.0, 40)))]
    for G in (2, 4, 8):
        a = lpt_assign(mixed, G, shape)
        total = sum(unit_cost(u, shape) for u in mixed)
        lower = max(total / G, max(unit_cost(u, shape) for u in mixed))
        assert makespan(a, shape) <= 4.0 / 3.0 * lower + 1e-6
        assert [[u.uid for u in p] for p in a] == [[u.uid for u in p] for p in lpt_assign(list(reversed(mixed)), G, shape)]
    # the cost model is the algorithmic FLOP count of SURVEY 8(d)
    assert attention_flops(8192, None, ModelShape(n_layers=1, global_every=1)) == 4.0 * 64 * 12 * 8192 * 8192


def _sched_worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_12646_b200.scheduler import BatchScheduler, Unit
        units = [Unit(i, "pii", i, s) for i, s in enumerate([512, 8192, 2048, 16384, 1024, 4096, 512])]
        calls = {"n": 0}

        def run_unit(u):
            calls["n"] += 1
            if u.uid == 2 and calls.get("failed") is None:  # transient failure: retried once
                calls["failed"] = True
                raise RuntimeError("transient")
            return {"logits": [float(u.seq_len), float(rank)], "rank": rank}

        res = BatchScheduler().run(units, run_unit)
        if rank == 0:
            ret["res"] = dict(res)
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


def test_scheduler_two_ranks_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        ret = mgr.dict()
        procs = [ctx.Process(target=_sched_worker, args=(r, world, port, ret)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        res = ret["res"]
    assert sorted(res) == list(range(7))
    assert all(res[i]["logits"][0] == s for i, s in enumerate([512, 8192, 2048, 16384, 1024, 4096, 512]))
    assert {res[i]["rank"] for i in res} == {0, 1}          # both ranks did work
    assert res[3]["rank"] != res[1]["rank"]                  # the two largest units are split
