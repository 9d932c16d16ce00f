"""Prefill tensor-core router (k_route_mma) per-CTA phase stamps (us after the earliest start).

usage: python tools/route_mma_stamps.py [--tokens 16384] [--experts 32]
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
ap.add_argument("--experts", type=int, default=32)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
E, d, f = a.experts, 1024, 4096
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
t0 = rt[:, 0][rt[:, 0] > 0].min()
names = ["start", "rows", "c0", "c1", "c2", "c3", "mma", "logits", "select", "", "", "ticket", "plan"]
trs = (a.tokens // 32 + 63) // 64
for c in range(0, 64, 4):
    row = rt[c]
    if row[0] == 0:
        continue
    print(f"CTA {c * trs:3d}: " + " ".join(f"{names[i]} {(row[i] - t0) / 1e3:6.2f}" for i in range(13) if row[i] > 0))
print("last CTA plan: start %.2f end %.2f" % ((rt[63, 13] - t0) / 1e3, (rt[63, 14] - t0) / 1e3))
print("plan phases: loaded %.2f scanned %.2f written %.2f" % tuple((rt[63, k] - t0) / 1e3 for k in (9, 10, 15)))
