"""Log-scale quantized experts (quant.cpp:97-243): moe_ffn_forward accepts
log banks (model.cpp:370-372 dequantizes them). The GPU decodes each field (sign + k) to the
exact fp16 +-2^-k in the tcgen05 staging and applies the per-channel scale in the epilogue.

Checker: the compiled, unmodified reference (oracle/_ref): quantize_log (MSE-optimal scales)
for the codes and moe_ffn_forward over the same log bank for the expected output.
Tolerance (north_star): |gpu - ref| <= 2e-3 + 1e-2 |ref|."""
import numpy as np
import pytest

from helpers import allclose_report, check_routing, fp16_valued

pytestmark = pytest.mark.gpu


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("bits,E,d,f,T", [(4, 8, 256, 512, 5), (3, 8, 256, 512, 300), (2, 4, 512, 1024, 64),
                                          (4, 8, 1024, 4096, 24)])
def test_log_bank_vs_reference(gpu, orc, bits, E, d, f, T):
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = oracle.ref()
    rng = np.random.default_rng(bits * 100 + T)
    w1 = (rng.standard_normal((E, d, f)) * 0.02).astype(np.float32)
    w2 = (rng.standard_normal((E, f, d)) * 0.02).astype(np.float32)
    wg = (rng.standard_normal((d, E)) * 0.02).astype(np.float32)
    h = fp16_valued(rng.standard_normal((T, d)))
    q1 = np.zeros(w1.shape, np.int8); q2 = np.zeros(w2.shape, np.int8)
    s1 = np.zeros((E, f), np.float32); s2 = np.zeros((E, d), np.float32)
    for e in range(E):
        # the reference's MSE-optimal scale search costs ~3.5 s per 256x512 matrix on one core:
        # expert 0 takes it on the small shapes, the rest use the max-abs scale
        mse = e == 0 and d * f <= 256 * 512
        q1[e], s1[e] = ref.quantize_log(w1[e], bits, mse_optimal=mse)
        q2[e], s2[e] = ref.quantize_log(w2[e], bits, mse_optimal=mse)
    p1 = np.stack([orc.pack(q1[e], bits) for e in range(E)])
    p2 = np.stack([orc.pack(q2[e], bits) for e in range(E)])
    bank = gpu.ExpertBank(E, d, f, bits, _t(p1), _t(s1), _t(p2), _t(s2), router=_t(wg), scheme="log")
    want = ref.log_bank(q1, s1, q2, s2, bits).forward(h, wg, 8)
    out, ex, g = gpu.moe_ffn_forward(_t(h).half(), bank, return_routing=True)
    check_routing(orc, h, wg, 1, ex.cpu().numpy(), g.cpu().numpy())
    nbad, mx = allclose_report(out.cpu().numpy(), want)
    assert nbad == 0, mx


def test_log_int8_not_supported(gpu):
    import torch
    p = torch.zeros((1, 64 * 128), dtype=torch.uint8, device="cuda")
    s = torch.ones((1, 128), device="cuda")
    with pytest.raises(gpu.NotSupported):
        gpu.ExpertBank(1, 64, 128, 8, p, s, p, torch.ones((1, 64), device="cuda"), scheme="log")
