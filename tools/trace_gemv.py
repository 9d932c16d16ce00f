"""Decode-kernel pipeline trace: run one layer with the device event trace on and
summarise per-role timing (what each CTA waits on).

usage: python tools/trace_gemv.py [--bits 3] [--tokens 24] [--experts 32] [--dump file.npy]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_02410_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=3)
ap.add_argument("--tokens", type=int, default=24)
ap.add_argument("--experts", type=int, default=32)
ap.add_argument("--d", type=int, default=1024)
ap.add_argument("--f", type=int, default=4096)
ap.add_argument("--dump", default=None)
ap.add_argument("--banks", type=int, default=1, help="rotate over N layers (N x weights > L2 = cold)")
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
w1 = torch.randn(a.experts, a.d, a.f, device="cuda", generator=g) * 0.02
w2 = torch.randn(a.experts, a.f, a.d, device="cuda", generator=g) * 0.02
wg = torch.randn(a.d, a.experts, device="cuda", generator=g) * 0.02
banks = [m.ExpertBank.from_float(w1, w2, a.bits, router=wg)]
for i in range(1, a.banks):  # same routing, distinct weight copies
    banks.append(m.ExpertBank.from_float(w1 + 1e-6 * i, w2, a.bits, router=wg))
del w1, w2
h = torch.randn(a.tokens, a.d, device="cuda", generator=g).half()
for _ in range(3):
    for b in banks:
        m.moe_ffn_forward(h, b, top_k=1)
torch.cuda.synchronize()
bank = banks[0]
bank.trace(True)
for b in banks[1:]:
    m.moe_ffn_forward(h, b, top_k=1)
m.moe_ffn_forward(h, bank, top_k=1)
tr, rt = bank.trace_read()
if a.dump:
    np.save(a.dump, tr)
t = tr[:, :, 0].astype(np.int64)
w = tr[:, :, 1]
valid = t > 0
t0 = t[valid].min()
rv = rt[:, 0] > 0
if rv.any():
    r = (rt[rv].astype(np.int64) - t0) / 1e3
    print(f"router CTAs {rv.sum()} (us rel. to GEMV first stamp): start {r[:, 0].min():.2f}  row {r[:, 1].max():.2f}  "
          f"chunks " + " ".join(f"{r[:, 2 + c].max():.2f}" for c in range(8)) +
          f"  chain {r[:, 10].max():.2f}  ticket {r[:, 11].max():.2f}  plan {r[:, 12].max():.2f}")
role = (w >> np.uint64(60)).astype(int)
ev = ((w >> np.uint64(56)) & np.uint64(0xF)).astype(int)
ph = ((w >> np.uint64(48)) & np.uint64(0xFF)).astype(int)
us = (t - t0) / 1e3
print(f"CTAs {tr.shape[0]}, events {valid.sum()}, span {us[valid].max():.2f} us")

for phase in (1, 2):
    sel_s = valid & (role == 2) & (ev == 0) & (ph == phase)
    sel_e = valid & (role == 2) & (ev == 2) & (ph == phase)
    if sel_s.any():
        print(f"phase {phase}: items {sel_s.sum()}  first start {us[sel_s].min():.2f}  last start {us[sel_s].max():.2f}  "
              f"first end {us[sel_e].min():.2f}  last end {us[sel_e].max():.2f} us")
        durs = []
        for c in range(tr.shape[0]):
            st = sorted(us[c][sel_s[c]]); en = sorted(us[c][sel_e[c]])
            durs += [b - a for a, b in zip(st, en)]
        if durs:
            print(f"   item start->end: mean {np.mean(durs):.2f} p50 {np.median(durs):.2f} max {np.max(durs):.2f} us (rank-0 CTAs incl. reduction)")
        sel_m = valid & (role == 2) & (ev == 1) & (ph == phase)
        ml = []
        gaps = []
        for c in range(tr.shape[0]):
            st = sorted(us[c][sel_s[c]]); mm = sorted(us[c][sel_m[c]]); en = sorted(us[c][sel_e[c]])
            ml += [b - a for a, b in zip(st, mm)]
            gaps += [b - a for a, b in zip(en[:-1], st[1:])]
        if ml:
            print(f"   mainloop: mean {np.mean(ml):.2f} us; gap end->next start: mean {np.mean(gaps) if gaps else 0:.2f} max {np.max(gaps) if gaps else 0:.2f}")
        evs = {}
        cyc = {}
        for c in range(tr.shape[0]):
            sel = valid[c] & (role[c] == 2) & (ph[c] == phase)
            tt = us[c][sel]; ee = ev[c][sel]; cc = (w[c][sel] & np.uint64(0xffff)).astype(np.int64)
            order = np.argsort(tt, kind="stable")
            tt = tt[order]; ee = ee[order]; cc = cc[order]
            for k in range(1, len(tt)):
                if ee[k] != 0:
                    evs.setdefault((ee[k - 1], ee[k]), []).append(tt[k] - tt[k - 1])
                    cyc.setdefault((ee[k - 1], ee[k]), []).append((cc[k] - cc[k - 1]) % 65536)
        print("   segments: " + "  ".join(f"{a}->{b}: {np.mean(v):.2f}" for (a, b), v in sorted(evs.items())))
        print("   cycles:   " + "  ".join(f"{a}->{b}: {np.mean(v):.0f}" for (a, b), v in sorted(cyc.items())))
        sel_b = valid & (role == 1) & (ev == 1) & (ph == phase)
        if sel_b.any():
            print(f"   builder done: first {us[sel_b].min():.2f} median {np.median(us[sel_b]):.2f} last {us[sel_b].max():.2f}")
