"""Per-CTA event timeline of the decode expert-FFN kernel (k_dec TRACE events):
0 start (after PDL wait), 1 W1 stage landed, 2 mid ready, 3 fc2 done, 4 flush done, 5 unit finished, 6 exit.
usage: python tools/dec_trace.py [--bits 3] [--tokens 24]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_02410_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=3)
ap.add_argument("--tokens", type=int, default=24)
ap.add_argument("--experts", type=int, default=32)
ap.add_argument("--banks", type=int, default=8, help="layers rotated (8: the traced layer's weights are out of L2)")
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
d, f, E = 1024, 4096, a.experts
banks = []
for i in range(a.banks):
    w1 = torch.randn(E, d, f, device="cuda", generator=g) * 0.02
    w2 = torch.randn(E, f, d, device="cuda", generator=g) * 0.02
    wg = torch.randn(d, E, device="cuda", generator=g) * 0.02
    banks.append(m.ExpertBank.from_float(w1, w2, a.bits, router=wg))
h = torch.randn(a.tokens, d, device="cuda", generator=g).half()
for b in banks:
    m.moe_ffn_forward(h, b)
torch.cuda.synchronize()
b = banks[-1]
b.trace(True)
for bb in banks:
    m.moe_ffn_forward(h, bb)
torch.cuda.synchronize()
tr, _ = b.trace_read()
ev = tr[:, :64, :]  # [cta][64][(event, ns)]
t0 = ev[:, :, 1][ev[:, :, 1] > 0].min()
names = {7: "F2:reds", 8: "FIN", 6: "EXIT", 20: "START", 1: "F1:w1", 2: "F1:mid", 3: "F2:w2", 4: "F2:mid", 5: "F2:flush", 10: "P:w1", 11: "P:w2"}
ends = []
for c in range(ev.shape[0]):
    row = [(int(e), (int(t) - int(t0)) / 1e3) for e, t in ev[c] if t > 0]
    row.sort(key=lambda x: x[1])
    if not row:
        continue
    ends.append(max(t for e, t in row))
    if c < 6 or c % 37 == 0:
        print(c, " ".join(f"{names.get(e, e)}@{t:.2f}" for e, t in row))
print("exit us: min %.2f median %.2f max %.2f" % (min(ends), float(np.median(ends)), max(ends)))
q = np.quantile(ends, [0.1, 0.25, 0.5, 0.75, 0.9, 1.0])
print("last event quantiles (10/25/50/75/90/100 %):", " ".join("%.2f" % x for x in q), " n", len(ends))
slow = sorted(range(len(ends)), key=lambda i: -ends[i])[:4]
for c in slow:
    row = sorted([(int(e), (int(t) - int(t0)) / 1e3) for e, t in ev[c] if t > 0], key=lambda x: x[1])
    print("late", c, " ".join(f"{names.get(e, e)}@{t:.2f}" for e, t in row))
st = ev[:, 63, 1].astype(np.int64)
st = (st[st > 0] - int(t0)) / 1e3
print("start (after PDL wait) us: n %d min %.2f median %.2f max %.2f" % (len(st), st.min(), np.median(st), st.max()))
# router events (k_dec_route, rank r at slots (160 + r) * 64): 20 after PDL wait, 21 h staged,
# 22 Wg landed, 23/24 around each cluster barrier, 25 plan built, 26 rows written
rt = tr.reshape(-1, 2)[160 * 64: 168 * 64].reshape(8, 64, 2)
for r in range(8):
    row = [(int(e) & 255, (int(t) - int(t0)) / 1e3, int(e) >> 8) for e, t in rt[r] if t > 0]
    row.sort(key=lambda x: x[2])
    ghz = (row[-1][2] - row[0][2]) / max(1e-9, (row[-1][1] - row[0][1]) * 1e3) if len(row) > 1 else 0
    print("router", r, " ".join(f"{e}@{t:.2f}" for e, t, c in row), f"  SM clock {ghz:.2f} GHz")
    print("   cycles", " ".join(f"{e}:{c - row[0][2]}" for e, t, c in row))
