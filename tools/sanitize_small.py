"""Small forwards through every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck): fused decode (T=5, top-1 and top-2), prefill with the tensor-core router (T=600),
the tcgen05 GEMM path, quantize, the config-3 LayerNorm.

usage: compute-sanitizer --tool racecheck python tools/sanitize_small.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_02410_b200 as m  # noqa: E402
from paper_2310_02410_b200.stack import add_layer_norm  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(3)
E, d, f = 32, 256, 512
w1 = torch.randn(E, d, f, device="cuda", generator=g) * 0.02
w2 = torch.randn(E, f, d, device="cuda", generator=g) * 0.02
wg = torch.randn(d, E, device="cuda", generator=g) * 0.02
for bits in (3, 4):
    bank = m.ExpertBank.from_float(w1, w2, bits, router=wg)
    for T, k, path in ((5, 1, "auto"), (5, 2, "auto"), (600, 1, "auto"), (600, 2, "gemm")):
        h = torch.randn(T, d, device="cuda", generator=g).half()
        out = m.moe_ffn_forward(h, bank, top_k=k, path=path)
        torch.cuda.synchronize()
        assert torch.isfinite(out).all()
x = torch.randn(64, d, device="cuda", generator=g)
add_layer_norm(x, torch.randn(64, d, device="cuda", generator=g), torch.ones(d, device="cuda"),
               torch.zeros(d, device="cuda"))
torch.cuda.synchronize()
print("sanitize_small: ok")
