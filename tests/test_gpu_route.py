"""GPU gating parity: expert ids bit-exact with the reference (logits are
computed in the reference's exact fp32 order), gates within float rounding."""
import math

import numpy as np
import pytest

from helpers import check_routing, fp16_valued

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_route_known_answers(gpu):
    # proj/tests/test_model.cpp:35-61
    ex, g = gpu.top1_route(_t(np.array([[1, 2], [-1, 0], [4, 4]], np.float32)),
                           _t(np.array([[0.5], [-0.25]], np.float32)))
    assert (ex.cpu().numpy() == 0).all() and (g.cpu().numpy() == 1.0).all()
    ex, g = gpu.top1_route(_t(np.array([[1, 2, 3], [-1, -2, -3]], np.float32)), _t(np.zeros((3, 4), np.float32)))
    assert (ex.cpu().numpy() == 0).all() and np.allclose(g.cpu().numpy(), 0.25, rtol=1e-6)
    ex, g = gpu.top1_route(_t(np.array([[1.0]], np.float32)), _t(np.array([[2.0, 0.0]], np.float32)))
    assert ex.item() == 0 and math.isclose(g.item(), math.exp(2) / (math.exp(2) + 1), rel_tol=1e-6)
    with pytest.raises(gpu.InvalidArgument):
        gpu.top1_route(_t(np.ones((2, 2), np.float32)), None)


def test_route_golden(gpu, golden):
    G = golden["route"]
    for i in range(3):
        ex, g = gpu.top1_route(_t(G[f"h_{i}"]), _t(G[f"wg_{i}"]))
        assert np.array_equal(ex.cpu().numpy(), G[f"expert_{i}"])
        assert np.allclose(g.cpu().numpy(), G[f"gate_{i}"], rtol=2e-7, atol=0)


@pytest.mark.parametrize("T,d,E,topk", [(24, 1024, 32, 1), (4096, 1024, 32, 1), (3000, 1024, 64, 1),
                                        (257, 2048, 128, 2), (5000, 256, 128, 2), (1, 8, 3, 2),
                                        (70, 33, 200, 1)])
def test_route_vs_oracle(gpu, orc, T, d, E, topk):
    rng = np.random.default_rng(T * 7 + E)
    h = fp16_valued(rng.standard_normal((T, d)))
    wg = (rng.standard_normal((d, E)) * 0.02).astype(np.float32)
    ex_o, g_o = orc.route(h, wg, topk)
    for dt in ("f32", "f16"):
        import torch
        hh = _t(h) if dt == "f32" else _t(h).half()
        ex, g = gpu.route(hh, _t(wg), topk)
        assert np.array_equal(ex.cpu().numpy(), ex_o), dt
        assert np.allclose(g.cpu().numpy(), g_o, rtol=1e-6, atol=0), dt


def test_route_nonfinite_weights_under_zero_activations(gpu, orc):
    # the reference skips zero activations (model.cpp:160-162), so an inf weight met only
    # by zeros never reaches the sum: the decode router's unguarded fast chain must fall
    # back to the exact skip when its Wg scan finds a non-finite value
    rng = np.random.default_rng(11)
    for T, d, E in ((4, 256, 32), (24, 1024, 32)):
        h = fp16_valued(rng.standard_normal((T, d)))
        h[:, 5] = 0.0
        wg = (rng.standard_normal((d, E)) * 0.02).astype(np.float32)
        wg[5, 3] = np.inf
        wg[5, 7] = -np.inf
        ex_o, g_o = orc.route(h, wg, 1)
        import torch
        ex, g = gpu.route(_t(h).half(), _t(wg), 1)
        assert np.array_equal(ex.cpu().numpy(), ex_o)
        assert np.allclose(g.cpu().numpy(), g_o, rtol=1e-6, atol=0)


@pytest.mark.parametrize("topk,E,d", [(1, 32, 1024), (2, 32, 1024), (1, 64, 1024), (2, 256, 512),
                                       (1, 40, 2048), (1, 128, 256)])
def test_decode_forward_routing_finite_and_nonfinite_bank_router(gpu, orc, topk, E, d):
    # decode forward (T*k <= 64): the bank's blocked router copy and the one-warp chain
    # (ffn decode self plan). Finite Wg: the select-free chain; an inf weight met only by
    # zero activations (model.cpp:160-162 skips them) must switch the bank to the exact skip.
    # Shapes: Wg as one chunk (E=32, d=1024; E=128, d=256) and as ~64 KB chunks through two
    # slots (E=64, E=256, d=2048), one to eight experts per lane, E not a multiple of 32.
    import torch
    rng = np.random.default_rng(5 + topk + E + d)
    f = 256
    w1 = torch.randn(E, d, f, device="cuda") * 0.02
    w2 = torch.randn(E, f, d, device="cuda") * 0.02
    for T, nonfinite in ((24, False), (24, True), (5, False), (1, True)):  # odd T: a half-used router CTA
        h = fp16_valued(rng.standard_normal((T, d)))
        wg = (rng.standard_normal((d, E)) * 0.02).astype(np.float32)
        if nonfinite:
            h[:, 5] = 0.0
            wg[5, 3] = np.inf
            wg[5, 7] = -np.nan
        bank = gpu.ExpertBank.from_float(w1, w2, 4, router=_t(wg))
        _, ex, g = gpu.moe_ffn_forward(_t(h).half(), bank, top_k=topk, return_routing=True)
        # the decode forward sums logits in a parallel order: near-tie exemption (north_star)
        check_routing(orc, h, wg, topk, ex.cpu().numpy(), g.cpu().numpy())
