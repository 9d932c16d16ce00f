"""Forward time of one MoE layer: eager vs CUDA graph, warm (1 layer) vs cold (N layers rotating).

usage: python tools/time_layer.py [--bits 3] [--tokens 24] [--banks 8]
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
ap.add_argument("--banks", type=int, default=8)
ap.add_argument("--path", default="auto")
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
w1 = torch.randn(a.experts, a.d, a.f, device="cuda", generator=g) * 0.02
w2 = torch.randn(a.experts, a.f, a.d, device="cuda", generator=g) * 0.02
wg = torch.randn(a.d, a.experts, device="cuda", generator=g) * 0.02
banks = [m.ExpertBank.from_float(w1 + 1e-6 * i, w2, a.bits, router=wg) for i in range(a.banks)]
del w1, w2
hs = [torch.randn(a.tokens, a.d, device="cuda", generator=g).half() for _ in banks]
outs = [torch.empty(a.tokens, a.d, device="cuda", dtype=torch.float16) for _ in banks]


def fwd(i):
    outs[i].copy_(m.moe_ffn_forward(hs[i], banks[i], top_k=1, out_dtype=torch.float16, path=a.path))


def run(fn, n):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / n


for nb in (1, a.banks):
    def eager():
        for i in range(nb):
            fwd(i)
    us = run(eager, 50) / nb
    gr = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        eager()
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=st):
            eager()
    us_g = run(gr.replay, 50) / nb
    print(f"layers={nb}: eager {us:.1f} us/forward, graph {us_g:.1f} us/forward")
