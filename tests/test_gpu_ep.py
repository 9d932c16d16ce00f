"""GPU expert_ffn (pre-routed rows) and the expert-parallel layer over NCCL at
world size 1 (real kernels end to end; multi-rank exchange logic is covered by
tests/test_ep_gloo.py on CPU)."""
import os
import socket

import numpy as np
import pytest

from helpers import allclose_report, make_layer

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("rows,bits", [(7, 4), (40, 3), (300, 2)])
def test_expert_ffn_vs_oracle(gpu, orc, rows, bits):
    E, d, f = 6, 128, 256
    L = make_layer(orc, rows + bits, E, d, f, bits, rows, with_bias=True)
    rng = np.random.default_rng(rows)
    ex = rng.integers(0, E, rows).astype(np.int32)
    g = rng.random(rows).astype(np.float32)
    want = np.stack([g[r] * orc.expert_ffn(L["h"][r:r + 1], L["q1"][ex[r]], L["s1"][ex[r]], L["q2"][ex[r]],
                                           L["s2"][ex[r]], L["b1"][ex[r]], L["b2"][ex[r]])[0] for r in range(rows)])
    bank = gpu.ExpertBank(E, d, f, bits, _t(L["p1"]), _t(L["s1"]), _t(L["p2"]), _t(L["s2"]), _t(L["b1"]), _t(L["b2"]))
    for path in ("auto", "gemv", "gemm"):
        out = gpu.expert_ffn(_t(L["h"]).half(), bank, _t(ex), _t(g), path=path)
        nbad, mx = allclose_report(out.cpu().numpy(), want)
        assert nbad == 0, (path, mx)


def test_ep_world1_nccl(gpu, orc):
    import torch
    import torch.distributed as dist
    from paper_2310_02410_b200.ep import ExpertParallelMoE
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0)
    try:
        E, d, f, bits, T = 8, 256, 512, 2, 70
        L = make_layer(orc, 3, E, d, f, bits, T)
        bank = gpu.ExpertBank(E, d, f, bits, _t(L["p1"]), _t(L["s1"]), _t(L["p2"]), _t(L["s2"]))
        want = orc.moe_forward(L["h"], L["wg"], L["q1"], L["s1"], L["q2"], L["s2"], top_k=2)[0]
        ref = gpu.moe_ffn_forward(_t(L["h"]).half(), bank, _t(L["wg"]), top_k=2)
        for rdt in (torch.float16, torch.float32):
            moe = ExpertParallelMoE(bank, _t(L["wg"]), E, top_k=2, return_dtype=rdt)
            out = moe.forward(_t(L["h"]).half())
            nbad, mx = allclose_report(out.cpu().numpy(), want)
            assert nbad == 0, (rdt, mx)
            if rdt == torch.float32:  # fp32 return: same kernels, same combine as the 1-GPU forward
                assert torch.allclose(out, ref, rtol=0, atol=1e-6)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T,k,E,G,d", [(0, 2, 8, 2, 64), (1, 1, 8, 4, 64), (24, 1, 32, 8, 1024), (1000, 2, 128, 8, 2048),
                                       (3000, 2, 64, 4, 256), (2500, 1, 96, 3, 100), (50, 2, 8, 2, 98)])
def test_ep_dispatch_combine_kernels(gpu, T, k, E, G, d):
    """moqe_gpu_ep_dispatch / ep_combine (csrc/ep.cu) against the torch form of the same
    plan (ep.dispatch_plan: stable sort by owner rank) — bit-exact records, counts, combine;
    includes empty input, a >1024-assignment (multi-chunk) plan and d % 4 != 0 rows (scalar paths)."""
    import torch
    from paper_2310_02410_b200.ep import dispatch_plan
    g = torch.Generator().manual_seed(T * 7 + G)
    h = torch.randn((T, d), generator=g).half().cuda()
    ex = torch.randint(0, E, (T, k), generator=g, dtype=torch.int32).cuda()
    gt = torch.rand((T, k), generator=g).cuda()
    rec, pos, counts, err = gpu.ep_dispatch(h, ex, gt, E, G)
    order, tok, dest_sorted, want_counts = dispatch_plan(ex, E, G)
    assert int(err.item()) == 0
    assert torch.equal(counts.cpu(), want_counts.cpu())
    src = tok[order]
    assert torch.equal(rec[:, :d], h.index_select(0, src))
    meta = rec[:, d:].view(torch.int32)
    assert torch.equal(meta[:, 0], (ex.reshape(-1)[order] - dest_sorted * (E // G)).int())
    assert torch.equal(meta[:, 1].view(torch.float32), gt.reshape(-1)[order])
    want_pos = torch.empty_like(order)
    want_pos[order] = torch.arange(order.numel(), device=order.device)
    assert torch.equal(pos.long(), want_pos)
    for dt in (torch.float16, torch.float32):
        back = torch.randn((T * k, d), generator=g).to(dt).cuda()
        out = gpu.ep_combine(back, pos, T, k)
        exp = back.float().index_select(0, pos.long()).reshape(T, k, d)
        ref = torch.zeros((T, d), dtype=torch.float32, device="cuda")
        for s in range(k):
            ref = ref + exp[:, s]
        assert torch.equal(out, ref)


def test_ep_dispatch_rejects_bad_ids(gpu):
    import torch
    h = torch.zeros((4, 64), dtype=torch.float16, device="cuda")
    ex = torch.tensor([[0], [9], [3], [-1]], dtype=torch.int32, device="cuda")
    _, _, _, err = gpu.ep_dispatch(h, ex, torch.ones((4, 1), device="cuda"), 8, 2)
    assert int(err.item()) == 1
    with pytest.raises(ValueError):
        gpu.ep_dispatch(h, ex, torch.ones((4, 1), device="cuda"), 9, 2)
