"""BASELINE config 3: 36-layer pre-LN residual FFN stack, even layers
32-expert top-1 int3 MoE, odd layers dense fp16 FFNs with 0.1 % outliers, 24 x 32 tokens.

Oracle: composed from the restated reference pieces (oracle/moqe_oracle.c: layer_norm
model.cpp:193-212, dense_ffn / matmul model.cpp:152-167, :315-322, route + expert FFN
model.cpp:328-393) on a seeded sample of rows; the stack is row-independent (run_stack,
model.cpp:419-435, has no attention here), so the sample is exact.

Tolerances: outputs |gpu - ref| <= 2e-3 + 1e-2 |ref| (north_star). Routing: after 2*i layers of
fp16 activations the GPU's router input differs from the oracle's by ~1e-3 relative, so a token
whose oracle top-2 logit gap is below 5e-3 may pick another expert; such rows leave the
comparison (at most a quarter of the sample). Any other routing difference fails the test.
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ATOL, RTOL, STACK_GAP = 2e-3, 1e-2, 5e-3


def _stack_case(gpu, orc, n_layers, E, d, f, T, n_sample, seed):
    import torch
    from paper_2310_02410_b200.workloads import build_config3
    from helpers import allclose_report
    stack, raw = build_config3(gpu, torch, seed, n_layers=n_layers, E=E, d=d, f=f, keep_f32=True)
    rng = np.random.default_rng(seed)
    h = rng.standard_normal((T, d)).astype(np.float16)
    out, routing = stack.forward(torch.from_numpy(h).cuda(), return_routing=True)
    out = out.cpu().numpy()
    rows = np.sort(rng.choice(T, n_sample, replace=False))
    keep = np.ones(len(rows), bool)
    xs = h[rows].astype(np.float32)
    mi = 0
    for L, R in zip(stack.layers, raw):
        fn = orc.layer_norm(xs, L.gain.cpu().numpy(), L.bias.cpu().numpy())
        if R["kind"] == "moe":
            wg = R["wg"].cpu().numpy()
            ex_o, g_o = orc.route(fn, wg, 1)
            lg = orc.router_logits(fn, wg)
            top = -np.sort(-lg, axis=1)[:, :2]
            gap = top[:, 0] - top[:, 1]
            ex_g = routing[mi].cpu().numpy()[rows]
            mi += 1
            diff = ex_g != ex_o
            assert not (diff & keep & (gap >= STACK_GAP)).any(), "routing differs on a well-separated row"
            keep &= ~diff
            y = np.zeros_like(xs)
            for e in np.unique(ex_o):
                sel = np.flatnonzero(ex_o == e)
                q1, s1 = orc.quantize_linear(R["w1"][e].cpu().numpy(), 3)
                q2, s2 = orc.quantize_linear(R["w2"][e].cpu().numpy(), 3)
                ye = orc.expert_ffn(fn[sel], q1, s1, q2, s2)
                y[sel] = g_o[sel, None] * ye
        else:
            D = L.dense
            y = orc.dense_ffn(fn, D.w1.float().cpu().numpy(), D.w2.float().cpu().numpy(),
                              D.b1.cpu().numpy(), D.b2.cpu().numpy())
        xs = xs + y
    want = orc.layer_norm(xs, stack.final_gain.cpu().numpy(), stack.final_bias.cpu().numpy())
    assert keep.mean() >= 0.75, f"too many near-tie routing divergences ({(~keep).sum()} of {len(keep)})"
    nbad, mx = allclose_report(out[rows][keep], want[keep], ATOL, RTOL)
    assert nbad == 0, (nbad, mx)
    assert np.isfinite(out).all()
    return mx


def test_config3_stack_36_layers(gpu, orc):
    """The BASELINE config 3 shape: 36 layers, d=1024, f=4096, E=32 int3, 768 tokens."""
    _stack_case(gpu, orc, 36, 32, 1024, 4096, 768, 16, 3)


def test_small_stack_all_rows_checked(gpu, orc):
    """A small stack (6 layers, d=256, f=512, E=8) with 64 sampled tokens."""
    _stack_case(gpu, orc, 6, 8, 256, 512, 200, 64, 7)


def test_layer_norm_vs_oracle(gpu, orc):
    import torch
    rng = np.random.default_rng(1)
    for rows, n in ((5, 1024), (3, 72), (1, 4096)):
        x = (rng.standard_normal((rows, n)) * 3 + 0.5).astype(np.float32)
        dl = rng.standard_normal((rows, n)).astype(np.float32)
        g = (1 + 0.1 * rng.standard_normal(n)).astype(np.float32)
        b = (0.1 * rng.standard_normal(n)).astype(np.float32)
        xt = torch.from_numpy(x).cuda()
        out = gpu.stack.add_layer_norm(xt, torch.from_numpy(dl).cuda(), torch.from_numpy(g).cuda(),
                                       torch.from_numpy(b).cuda())
        xs = x + dl
        assert np.array_equal(xt.cpu().numpy(), xs)  # the fp32 residual add is exact
        want = orc.layer_norm(xs, g, b)
        assert np.allclose(out.cpu().numpy(), want, rtol=1e-6, atol=1e-6)
