"""Profiling driver (ncu target): one MoE layer, a few forwards, nothing else.

usage: python tools/prof_layer.py [--bits 3] [--tokens 24] [--experts 32] [--d 1024] [--f 4096] [--banks 1]
                                  [--top-k 1] [--iters 3] [--path auto]
Weights are random fp32 N(0, 0.02) quantized on the GPU; activations N(0,1) fp16.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_02410_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=3)
ap.add_argument("--tokens", type=int, default=24)
ap.add_argument("--experts", type=int, default=32)
ap.add_argument("--d", type=int, default=1024)
ap.add_argument("--f", type=int, default=4096)
ap.add_argument("--top-k", type=int, default=1)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--path", default="auto")
ap.add_argument("--banks", type=int, default=1, help="rotate over N weight copies (N x weights > L2 = cold)")
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
w1 = torch.randn(a.experts, a.d, a.f, device="cuda", generator=g) * 0.02
w2 = torch.randn(a.experts, a.f, a.d, device="cuda", generator=g) * 0.02
wg = torch.randn(a.d, a.experts, device="cuda", generator=g) * 0.02
banks = [m.ExpertBank.from_float(w1 + 1e-6 * i, w2, a.bits, router=wg) for i in range(a.banks)]
del w1, w2
h = torch.randn(a.tokens, a.d, device="cuda", generator=g).half()
for _ in range(a.iters):
    for bank in banks:
        out = m.moe_ffn_forward(h, bank, top_k=a.top_k, path=a.path)
torch.cuda.synchronize()
print("ok", out.float().abs().mean().item())
