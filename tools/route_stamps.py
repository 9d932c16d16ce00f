"""Decode router (k_route_chain) per-chunk stage stamps of CTA 0 (MOQE_ROUTE_DBG=9).

usage: MOQE_ROUTE_DBG=9 python tools/route_stamps.py [--banks 8]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_02410_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--banks", type=int, default=8)
ap.add_argument("--tokens", type=int, default=24)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
w1 = torch.randn(32, 1024, 4096, device="cuda", generator=g) * 0.02
w2 = torch.randn(32, 4096, 1024, device="cuda", generator=g) * 0.02
wg = torch.randn(1024, 32, device="cuda", generator=g) * 0.02
banks = [m.ExpertBank.from_float(w1 + 1e-6 * i, w2, 3, router=wg) for i in range(a.banks)]
h = torch.randn(a.tokens, 1024, device="cuda", generator=g).half()
for _ in range(3):
    for b in banks:
        m.moe_ffn_forward(h, b, top_k=1)
torch.cuda.synchronize()
banks[0].trace(True)
for b in banks[1:]:
    m.moe_ffn_forward(h, b, top_k=1)
m.moe_ffn_forward(h, banks[0], top_k=1)
_, rt = banks[0].trace_read()
ds = rt.reshape(-1)[16:16 + 61].astype(np.int64)
t0 = ds[60]
names = {0: "tma issue", 3: "chain: chunk landed", 4: "chain: chunk done"}
print("cycles since kernel start (clock64), CTA 0")
for c in range(8):
    print(f"chunk {c}: " + "  ".join(f"{n} {ds[c * 6 + i] - t0:6d}" for i, n in names.items()))
