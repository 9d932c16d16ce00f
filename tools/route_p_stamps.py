"""Persistent prefill router (k_route_mma_p) per-CTA stamps, us after the earliest start.

usage: python tools/route_p_stamps.py [--tokens 16384]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_02410_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=16384)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
E, d, f = 32, 1024, 4096
w1 = torch.randn(E, d, f, device="cuda", generator=g) * 0.02
w2 = torch.randn(E, f, d, device="cuda", generator=g) * 0.02
wg = torch.randn(d, E, device="cuda", generator=g) * 0.02
bank = m.ExpertBank.from_float(w1, w2, 3, router=wg)
del w1, w2
h = torch.randn(a.tokens, d, device="cuda", generator=g).half()
for _ in range(3):
    m.moe_ffn_forward(h, bank)
torch.cuda.synchronize()
bank.trace(True)
m.moe_ffn_forward(h, bank)
torch.cuda.synchronize()
_, rt = bank.trace_read()
rt = rt.astype(np.int64)
t0 = rt[:63, 0][rt[:63, 0] > 0].min()
f = lambda v: f"{(v - t0) / 1e3:6.2f}" if v > 0 else "   -  "
for c in range(0, 63, 9):
    r = rt[c]
    tiles = "  ".join(f"[{f(r[2 + 3 * i])} {f(r[3 + 3 * i])} {f(r[4 + 3 * i])}]" for i in range(3))
    print(f"CTA {c:2d}: start {f(r[0])} wg {f(r[1])} tiles(rows, mma, done) {tiles} ticket {f(r[11])}")
print("plan: start %s end %s" % (f(rt[63, 13]), f(rt[63, 14])))
