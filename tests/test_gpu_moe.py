"""GPU moe_forward parity against the oracle / reference goldens.

Tolerance (BASELINE.json north_star): |gpu - ref| <= 2e-3 + 1e-2*|ref|
elementwise; routing ids bit-exact (logits are bit-identical by construction,
so no near-tie exemption is needed)."""
import numpy as np
import pytest

from helpers import allclose_report, check_routing, fp16_valued, make_layer

pytestmark = pytest.mark.gpu
ATOL, RTOL = 2e-3, 1e-2


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _bank(gpu, L):
    return gpu.ExpertBank(L["E"], L["d"], L["f"], L["bits"], _t(L["p1"]), _t(L["s1"]), _t(L["p2"]),
                          _t(L["s2"]), None if L["b1"] is None else _t(L["b1"]),
                          None if L["b2"] is None else _t(L["b2"]))


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_golden_moe(gpu, golden, bits):
    G = golden["moe"]
    E, d, f = G[f"q1_{bits}"].shape
    b1 = _t(G[f"b1_{bits}"]) if f"b1_{bits}" in G else None
    b2 = _t(G[f"b2_{bits}"]) if f"b2_{bits}" in G else None
    bank = gpu.ExpertBank(E, d, f, bits, _t(G[f"p1_{bits}"]), _t(G[f"s1_{bits}"]), _t(G[f"p2_{bits}"]),
                          _t(G[f"s2_{bits}"]), b1, b2)
    for path in ("auto", "gemv"):
        out, ex, g = gpu.moe_ffn_forward(_t(G[f"h_{bits}"]), bank, _t(G[f"wg_{bits}"]), path=path,
                                         return_routing=True)
        assert np.array_equal(ex.cpu().numpy(), G[f"expert_{bits}"])
        nbad, mx = allclose_report(out.cpu().numpy(), G[f"out_{bits}"], ATOL, RTOL)
        assert nbad == 0, (path, mx)


CASES = [
    # (E, d, f, bits, T, topk, bias)
    (32, 1024, 4096, 3, 24, 1, False),   # north-star decode shape
    (32, 1024, 4096, 2, 24, 1, False),
    (32, 1024, 4096, 4, 24, 1, False),
    (32, 1024, 4096, 8, 24, 1, False),
    (8, 256, 512, 4, 16, 1, True),
    (8, 256, 512, 3, 7, 2, False),
    (5, 72, 200, 2, 13, 1, True),        # ragged dims (padding paths)
    (4, 64, 128, 8, 1, 1, False),
    (16, 128, 256, 4, 200, 1, False),    # > 32 rows per expert: GEMV passes / GEMM
    (16, 128, 256, 3, 300, 2, True),
    # decode-path boundaries: self-planned GEMV (T*k <= 64, T <= 32), decode router EPL 2 / 8
    (64, 1024, 2048, 3, 32, 2, False),   # T*k = 64 (self-plan limit), fc2 split-K over 2 CTAs
    (256, 256, 512, 2, 32, 1, True),     # E = 256: multi-round expert scans in the self plan
    (256, 512, 256, 4, 24, 2, False),    # E > 64 with 32 < T*k < 64: partly filled second row half of the self plan
    (100, 256, 512, 3, 20, 2, True),
    (32, 512, 1024, 4, 33, 1, False),    # T = 33: routed plan + packed GEMV table path
    (8, 2048, 1024, 3, 8, 1, True),      # d = 2048: fc1 split-K over a 2-CTA cluster
    (4, 256, 8192, 2, 6, 2, False),      # f = 8192: fc2 split-K over an 8-CTA cluster
    # mid-size top-1 batches: batched router + k_dec on the experts with <= 32 rows (k_dec_prep units)
    (24, 256, 512, 3, 150, 1, True),
    (40, 72, 200, 4, 320, 1, False),     # ragged dims on the mid path
]


@pytest.mark.parametrize("E,d,f,bits,T,topk,bias", CASES)
def test_moe_vs_oracle(gpu, orc, E, d, f, bits, T, topk, bias):
    import torch
    L = make_layer(orc, E * 31 + T + bits, E, d, f, bits, T, with_bias=bias)
    want, ex_o, g_o = orc.moe_forward(L["h"], L["wg"], L["q1"], L["s1"], L["q2"], L["s2"], top_k=topk,
                                      b1=L["b1"], b2=L["b2"])
    bank = _bank(gpu, L)
    paths = ["auto", "gemv"] + (["gemm"] if gpu.api._lib.load() and _gemm_ok(gpu) else [])
    for path in paths:
        for hdt in (torch.float32, torch.float16):
            out, ex, g = gpu.moe_ffn_forward(_t(L["h"]).to(hdt), bank, _t(L["wg"]), top_k=topk, path=path,
                                             return_routing=True)
            check_routing(orc, L["h"], L["wg"], topk, ex.cpu().numpy(), g.cpu().numpy())
            nbad, mx = allclose_report(out.cpu().numpy(), want, ATOL, RTOL)
            assert nbad == 0, (path, hdt, mx)
    # the bank's router (set once; its blocked copy feeds the decode chain router)
    bank.set_router(_t(L["wg"]))
    for hdt in (torch.float32, torch.float16):
        out, ex, g = gpu.moe_ffn_forward(_t(L["h"]).to(hdt), bank, top_k=topk, return_routing=True)
        check_routing(orc, L["h"], L["wg"], topk, ex.cpu().numpy(), g.cpu().numpy())
        nbad, mx = allclose_report(out.cpu().numpy(), want, ATOL, RTOL)
        assert nbad == 0, ("bank router", hdt, mx)


def _gemm_ok(gpu):
    try:
        import torch
        L = {"E": 2, "d": 64, "f": 128, "bits": 4}
        rng = np.random.default_rng(0)
        p = np.zeros((2, gpu.packed_size(4, 64 * 128)), np.uint8)
        bank = gpu.ExpertBank(2, 64, 128, 4, _t(p), _t(np.ones((2, 128), np.float32)), _t(p),
                              _t(np.ones((2, 64), np.float32)))
        gpu.moe_ffn_forward(_t(np.ones((40, 64), np.float32)), bank, _t(np.zeros((64, 2), np.float32)), path="gemm")
        return True
    except gpu.NotSupported:
        return False


def test_moe_f16_output_and_determinism(gpu, orc):
    import torch
    L = make_layer(orc, 5, 32, 1024, 4096, 3, 24)
    bank = _bank(gpu, L)
    h, wg = _t(L["h"]).half(), _t(L["wg"])
    a = gpu.moe_ffn_forward(h, bank, wg)
    b = gpu.moe_ffn_forward(h, bank, wg)
    assert torch.equal(a, b)  # bit-identical across runs (test_model.cpp:170-181)
    o16 = gpu.moe_ffn_forward(h, bank, wg, out_dtype=torch.float16)
    assert o16.dtype == torch.float16
    want = orc.moe_forward(L["h"], L["wg"], L["q1"], L["s1"], L["q2"], L["s2"])[0]
    nbad, mx = allclose_report(o16.float().cpu().numpy(), want, ATOL, RTOL)
    assert nbad == 0, mx


def test_moe_empty_and_errors(gpu, orc):
    import torch
    L = make_layer(orc, 6, 4, 64, 128, 4, 3)
    bank = _bank(gpu, L)
    out = gpu.moe_ffn_forward(torch.zeros((0, 64), device="cuda"), bank, _t(L["wg"]))
    assert out.shape == (0, 64)
    with pytest.raises(gpu.InvalidArgument):
        gpu.moe_ffn_forward(_t(L["h"]), bank, None)  # no router (top1_route: no gate weights)
    with pytest.raises(gpu.InvalidArgument):
        gpu.moe_ffn_forward(_t(L["h"][:, :32]), bank, _t(L["wg"]))
    with pytest.raises(gpu.InvalidArgument):
        gpu.ExpertBank(0, 64, 128, 4, _t(L["p1"]), _t(L["s1"]), _t(L["p2"]), _t(L["s2"]))


def test_bank_from_float_and_host_api(gpu, orc):
    import torch
    L = make_layer(orc, 7, 8, 128, 256, 4, 20)
    bank = gpu.ExpertBank.from_float(_t(L["w1"]), _t(L["w2"]), 4, router=_t(L["wg"]))
    want = orc.moe_forward(L["h"], L["wg"], L["q1"], L["s1"], L["q2"], L["s2"])[0]
    out = gpu.moe_ffn_forward(_t(L["h"]), bank)  # bank's router
    assert allclose_report(out.cpu().numpy(), want, ATOL, RTOL)[0] == 0
    h_host = torch.from_numpy(L["h"]).pin_memory()
    out_h = gpu.moe_ffn_forward_host(h_host, bank)  # page-locked output: the kernel stores into it
    assert torch.equal(out_h, out.cpu())
    out_p = torch.full((L["h"].shape[0], 128), float("nan"))  # pageable output: the D2H copy path
    gpu.moe_ffn_forward_host(torch.from_numpy(L["h"]), bank, out=out_p)
    assert torch.equal(out_p, out.cpu())
    out_16 = torch.empty((L["h"].shape[0], 128), dtype=torch.float16).pin_memory()
    gpu.moe_ffn_forward_host(h_host.half(), bank, out=out_16)
    assert torch.equal(out_16, gpu.moe_ffn_forward(_t(L["h"]).half(), bank, out_dtype=torch.float16).cpu())


def test_zero_input_gives_gated_bias(gpu):
    # proj/tests/test_model.cpp:118-134 (zero weights quantize to zero codes/scales)
    import torch
    E, d, f = 3, 4, 8
    p = np.zeros((E, gpu.packed_size(4, d * f)), np.uint8) + 0x88  # code 0 everywhere
    bank = gpu.ExpertBank(E, d, f, 4, _t(p), _t(np.zeros((E, f), np.float32)), _t(p),
                          _t(np.zeros((E, d), np.float32)), _t(np.zeros((E, f), np.float32)),
                          _t(np.tile((np.arange(d) - 1.5).astype(np.float32), (E, 1))))
    out, ex, g = gpu.moe_ffn_forward(torch.zeros((2, d), device="cuda"), bank,
                                     torch.zeros((d, E), device="cuda"), return_routing=True)
    assert (ex.cpu().numpy() == 0).all()
    assert np.allclose(out.cpu().numpy(), (np.arange(d) - 1.5) / 3.0, rtol=1e-6)


@pytest.mark.parametrize("bits,T,topk", [(4, 24, 1), (3, 300, 2), (2, 2048, 1)])
def test_moe_per_tensor_bank(gpu, orc, bits, T, topk):
    """Per-tensor experts (Granularity::PerTensor, quant.cpp:53-55: one scale per matrix,
    scale_index) through the forward, decode / mixed / tcgen05 paths."""
    import torch
    E, d, f = 8, 256, 512
    rng = np.random.default_rng(bits * 13 + T)
    w1 = (rng.standard_normal((E, d, f)) * 0.02).astype(np.float32)
    w2 = (rng.standard_normal((E, f, d)) * 0.02).astype(np.float32)
    wg = (rng.standard_normal((d, E)) * 0.02).astype(np.float32)
    h = fp16_valued(rng.standard_normal((T, d)))
    q1 = np.zeros(w1.shape, np.int8); q2 = np.zeros(w2.shape, np.int8)
    s1 = np.zeros((E, f), np.float32); s2 = np.zeros((E, d), np.float32)
    for e in range(E):
        q1[e], t1 = orc.quantize_linear(w1[e], bits, per_tensor=True)
        q2[e], t2 = orc.quantize_linear(w2[e], bits, per_tensor=True)
        s1[e], s2[e] = t1[0], t2[0]
    bank = gpu.ExpertBank.from_float(_t(w1), _t(w2), bits, router=_t(wg), granularity=gpu.PER_TENSOR)
    want, ex_o, g_o = orc.moe_forward(h, wg, q1, s1, q2, s2, top_k=topk)
    out, ex, g = gpu.moe_ffn_forward(_t(h).half(), bank, top_k=topk, return_routing=True)
    check_routing(orc, h, wg, topk, ex.cpu().numpy(), g.cpu().numpy())
    nbad, mx = allclose_report(out.cpu().numpy(), want, ATOL, RTOL)
    assert nbad == 0, mx
