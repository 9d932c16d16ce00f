"""Expert-parallel dispatch / return / combine (paper_2310_02410_b200/ep.py) at
world_size 2 over gloo on CPU. The per-rank compute is injected (oracle
router + oracle expert FFN on the rank's expert shard); the layer output on
every rank must equal the single-process oracle top-2 forward bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, E, d, f, bits, T, top_k, q, ret16=False):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import oracle
    from helpers import make_layer
    from paper_2310_02410_b200.ep import ExpertParallelMoE, shard_range

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", world_size=world, rank=rank)
    try:
        orc = oracle.orc()
        L = make_layer(orc, 77, E, d, f, bits, T * world, with_bias=True)  # same layer on every rank
        h_all = L["h"]
        h = h_all[rank * T:(rank + 1) * T]
        lo, hi = shard_range(E, world, rank)

        def route_fn(x):
            ex, g = orc.route(x.numpy(), L["wg"], top_k)
            return torch.from_numpy(ex.reshape(x.shape[0], -1)), torch.from_numpy(g.reshape(x.shape[0], -1))

        def expert_fn(x, e_local, g):
            out = np.zeros((x.shape[0], d), np.float32)
            xn = x.numpy()
            for r in range(x.shape[0]):
                e = lo + int(e_local[r])
                y = orc.expert_ffn(xn[r:r + 1], L["q1"][e], L["s1"][e], L["q2"][e], L["s2"][e],
                                   L["b1"][e], L["b2"][e])
                out[r] = np.float32(g[r]) * y[0]
            return torch.from_numpy(out)

        moe = ExpertParallelMoE(None, None, E, top_k=top_k, route_fn=route_fn, expert_fn=expert_fn,
                                return_dtype=torch.float16 if ret16 else torch.float32)
        got = moe.forward(torch.from_numpy(np.ascontiguousarray(h))).numpy()
        want = orc.moe_forward(h, L["wg"], L["q1"], L["s1"], L["q2"], L["s2"], top_k=top_k,
                               b1=L["b1"], b2=L["b2"])[0]
        if ret16:  # fp16 return rows: one rounding of each gated row (north_star tolerance)
            ok = bool((np.abs(got - want) <= 2e-3 + 1e-2 * np.abs(want)).all())
        else:
            ok = bool(np.array_equal(got, want))
        q.put((rank, ok, float(np.abs(got - want).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,top_k,ret16", [(2, 1, False), (2, 2, False), (4, 2, False), (4, 2, True)])
def test_ep_matches_single_process(world, top_k, ret16):
    """world 2 / 4 over gloo: fp32 return rows are bit-exact with the single-process oracle;
    fp16 return rows (the GPU default) stay within the north_star tolerance."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    E, d, f, bits, T = 8, 32, 64, 4, 13
    procs = [ctx.Process(target=_worker, args=(r, world, port, E, d, f, bits, T, top_k, q, ret16))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, mx in sorted(res):
        assert ok, f"rank {rank}: max abs diff {mx}"


def test_dispatch_plan_stable_order():
    from paper_2310_02410_b200.ep import dispatch_plan
    ex = torch.tensor([[3, 0], [1, 2], [0, 3], [2, 1]], dtype=torch.int32)
    order, tok, dest, counts = dispatch_plan(ex, 4, 2)
    assert counts.tolist() == [4, 4]
    # owner 0 gets experts {0,1} in ascending (token, slot) order, then owner 1
    flat = ex.reshape(-1)[order].tolist()
    assert flat == [0, 1, 0, 1, 3, 2, 3, 2]
    assert tok[order].tolist() == [0, 1, 2, 3, 0, 1, 2, 3]
