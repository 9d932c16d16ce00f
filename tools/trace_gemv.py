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
# each CTA row: two halves (fc1, fc2) of S slots; slot 0 / S-1 = (globaltimer, clock64) anchors
S = tr.shape[1] // 2
raw = tr.astype(np.int64)
t = np.zeros(tr.shape[:2], dtype=np.int64)
# globaltimer values are ~1.8e18 ns: convert relative to a base, or float64 rounds to 256 ns
gbase = int(raw[:, 0, 0][raw[:, 0, 0] > 0].min()) - 1_000_000
for hlf in range(2):
    blk = raw[:, hlf * S:(hlf + 1) * S]
    g0, c0_, g1, c1_ = blk[:, 0, 0], blk[:, 0, 1], blk[:, S - 1, 0], blk[:, S - 1, 1]
    ok = (g0 > 0) & (g1 > g0) & (c1_ > c0_)
    rate = np.where(ok, (g1 - g0) / np.maximum(c1_ - c0_, 1), 0.0)  # ns per clock
    ev_ok = (blk[:, 1:S - 1, 1] & 1) == 1
    tt = (g0 - gbase)[:, None] + (blk[:, 1:S - 1, 0] - c0_[:, None]) * rate[:, None]
    t[:, hlf * S + 1:(hlf + 1) * S - 1] = np.where(ev_ok & ok[:, None], tt, 0).astype(np.int64)
w = tr[:, :, 1]
valid = t > 0
t0 = t[valid].min()
rv = rt[:, 0] > 0
if rv.any():
    print("router chain cycles (clock64, per CTA thread 0): mean %.0f" % rt[rv][:, 13].astype(np.float64).mean())
    r = (rt[rv].astype(np.int64) - gbase - t0) / 1e3
    print(f"router CTAs {rv.sum()} (us rel. to GEMV first stamp): start {r[:, 0].min():.2f}  row {r[:, 1].max():.2f}  "
          f"chunks " + " ".join(f"{r[:, 2 + c].max():.2f}" for c in range(8)) +
          f"  chain {r[:, 10].max():.2f}  ticket {r[:, 11].max():.2f}  counts {r[:, 13].max():.2f}  lists {r[:, 14].max():.2f}  perm {r[:, 15].max():.2f}  plan {r[:, 12].max():.2f}")
role = (w >> np.uint64(60)).astype(int)
ev = ((w >> np.uint64(56)) & np.uint64(0xF)).astype(int)
ph = ((w >> np.uint64(48)) & np.uint64(0xFF)).astype(int)
us = (t - t0) / 1e3
print(f"CTAs {tr.shape[0]}, events {valid.sum()}, span {us[valid].max():.2f} us")
ent = raw[:, 0, 0]
print(f"kernel entry (globaltimer anchor) rel. first stamp: min {(ent[ent > 0].min() - gbase - t0) / 1e3:.2f} max {(ent[ent > 0].max() - gbase - t0) / 1e3:.2f} us")

for phase in (1, 2):
    c0 = valid & (role == 2) & (ev == 0) & (ph == phase)
    c1 = valid & (role == 2) & (ev == 1) & (ph == phase)
    e0 = valid & (role == 3) & (ev == 0) & (ph == phase)
    e2 = valid & (role == 3) & (ev == 2) & (ph == phase)
    if not c0.any():
        continue
    print(f"phase {phase}: items {c0.sum()}  consumer first start {us[c0].min():.2f} last mainloop end {us[c1].max():.2f}  "
          f"epilogue first end {us[e2].min():.2f} last end {us[e2].max():.2f} us")
    ml, ep, gap, lag = [], [], [], []
    for c in range(tr.shape[0]):
        a = sorted(us[c][c0[c]]); b = sorted(us[c][c1[c]]); x = sorted(us[c][e0[c]]); y = sorted(us[c][e2[c]])
        ml += [q - p for p, q in zip(a, b)]
        gap += [q - p for p, q in zip(b[:-1], a[1:])]
        ep += [q - p for p, q in zip(x, y)]
        lag += [q - p for p, q in zip(b, y)]
    f = lambda v: f"{np.mean(v):.2f}" if v else "-"
    print(f"   per item: mainloop {f(ml)}  consumer gap {f(gap)}  epilogue {f(ep)}  mainloop-end -> epilogue-end {f(lag)} us")
    # unit latency: k-th issue (role 4) -> k-th landed (role 5), per CTA in order
    lat, bw, top, sw = [], [], [], []
    for c in range(tr.shape[0]):
        iss = sorted(us[c][valid[c] & (role[c] == 4) & (ph[c] == phase)])
        lnd = sorted(us[c][valid[c] & (role[c] == 5) & (ph[c] == phase)])
        lat += [q - p for p, q in zip(iss, lnd)]
        w3 = sorted(us[c][valid[c] & (role[c] == 2) & (ev[c] == 3) & (ph[c] == phase)])
        w0 = sorted(us[c][c0[c]])
        bw += [q - p for p, q in zip(w3, w0)]
        if iss: top.append(iss[0])
        w4 = sorted(us[c][valid[c] & (role[c] == 2) & (ev[c] == 4) & (ph[c] == phase)])
        sw.extend([q - p for p, q in zip(b, w4)])
    print(f"   unit issue->landed {f(lat)} (max {max(lat) if lat else 0:.2f})  consumer bfull wait {f(bw)}  first issue {min(top) if top else 0:.2f} us  scratch wait {f(sw)}")

if os.environ.get("TRACE_CTA"):
    c = int(os.environ["TRACE_CTA"])
    names = {(7, 0): "K pdl_wait done", (7, 1): "K tables+cluster ok", (7, 2): "P self plan done", (7, 3): "P first item issued", (7, 4): "P self plan again", (2, 5): "U B tile", (6, 0): "M item start", (6, 1): "M item issued", (6, 2): "M unit A ok", (6, 3): "M unit issued", (2, 3): "C top", (2, 0): "C bfull ok", (5, 0): "C unit0 in", (5, 1): "C unit+ in", (2, 1): "C mloop end",
             (2, 4): "C scr ok/U B done", (3, 0): "E start", (3, 2): "E end", (4, 0): "P unit0 iss", (4, 1): "P unit+ iss"}
    sel = valid[c]
    order = np.argsort(us[c][sel], kind="stable")
    rr, ee, pp, tt = role[c][sel][order], ev[c][sel][order], ph[c][sel][order], us[c][sel][order]
    mt = ((w[c][sel][order] >> np.uint64(20)) & np.uint64(0xfff)).astype(int)
    ex = ((w[c][sel][order] >> np.uint64(32)) & np.uint64(0xffff)).astype(int)
    for a, b, p_, t_, m_, e_ in zip(rr, ee, pp, tt, mt, ex):
        if p_ == int(os.environ.get("TRACE_PHASE", "1")):
            print(f"{t_:8.2f}  {names.get((a, b), (a, b))!s:12s} e{e_} mt{m_}")
