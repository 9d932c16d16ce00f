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
