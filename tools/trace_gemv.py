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
names = {(3, 1): "CTA entry (pre-PDL)", (3, 0): "kernel start", (2, 3): "cons: END item", (0, 0): "prod: ticket", (0, 1): "prod: weights issued",
         (1, 0): "conv: prep start", (1, 1): "conv: prep end", (1, 2): "conv: B-load issued",
         (2, 0): "cons: item start", (2, 2): "cons: item end", (4, 0): "pub: item done"}
for (r, e), nm in names.items():
    sel = valid & (role == r) & (ev == e)
    if sel.any():
        v = us[sel]
        print(f"  {nm:22s} n={sel.sum():5d}  first {v.min():7.2f}  median {np.median(v):7.2f}  last {v.max():7.2f} us")
for p in (1, 2, 3, 4):
    for (r, e) in ((2, 0), (2, 2), (1, 0), (1, 1)):
        sel = valid & (role == r) & (ev == e) & (ph == p)
        if sel.any():
            v = us[sel]
            print(f"  phase {p} {names[(r, e)]:22s} n={sel.sum():4d} first {v.min():7.2f} last {v.max():7.2f}")
# per-CTA consumer busy: item start -> end durations
dur = []
for c in range(tr.shape[0]):
    s = [(us[c, i], ph[c, i]) for i in range(tr.shape[1]) if valid[c, i] and role[c, i] == 2 and ev[c, i] == 0]
    e_ = [us[c, i] for i in range(tr.shape[1]) if valid[c, i] and role[c, i] == 2 and ev[c, i] == 2]
    for (a0, p), b0 in zip(s, e_):
        dur.append((p, b0 - a0))
dur = np.array(dur)
for p in (1, 2):
    d = dur[dur[:, 0] == p, 1]
    if d.size:
        print(f"  consumer item phase {p}: n={d.size} mean {d.mean():.2f} us  p50 {np.median(d):.2f}  max {d.max():.2f}")
# publisher lag: consumer item end -> publish done, matched per CTA by (phase, e, mt, ks)
key = (w & np.uint64(0x0000FFFFFFFFFFFF))
for p in (1, 2):
    lags = []
    for c in range(tr.shape[0]):
        ends = {int(key[c, i]): us[c, i] for i in range(tr.shape[1]) if valid[c, i] and role[c, i] == 2 and ev[c, i] == 2 and ph[c, i] == p}
        for i in range(tr.shape[1]):
            if valid[c, i] and role[c, i] == 4 and ev[c, i] == 0 and ph[c, i] == p and int(key[c, i]) in ends:
                lags.append(us[c, i] - ends[int(key[c, i])])
    if lags:
        print(f"  phase {p} publish lag after consumer end: mean {np.mean(lags):.2f} us  p50 {np.median(lags):.2f}  max {np.max(lags):.2f}")
for p in (1, 2):
    dd = []
    for c in range(tr.shape[0]):
        st_ = {int(key[c, i]): us[c, i] for i in range(tr.shape[1]) if valid[c, i] and role[c, i] == 4 and ev[c, i] == 1 and ph[c, i] == p}
        for i in range(tr.shape[1]):
            if valid[c, i] and role[c, i] == 4 and ev[c, i] == 0 and ph[c, i] == p and int(key[c, i]) in st_:
                dd.append(us[c, i] - st_[int(key[c, i])])
    if dd:
        print(f"  phase {p} publish service time: mean {np.mean(dd):.2f} us  p50 {np.median(dd):.2f}  max {np.max(dd):.2f}")
# publisher internals (fc1): start -> y computed (4,4) -> before fence (4,2) -> after fence (4,3) -> done (4,0)
seq = []
for c in range(tr.shape[0]):
    evs = sorted((us[c, i], ev[c, i]) for i in range(tr.shape[1]) if valid[c, i] and role[c, i] == 4)
    cur = {}
    for tt, e in evs:
        if e == 1: cur = {1: tt}
        elif cur: cur[e] = tt
        if e == 0 and all(k in cur for k in (1, 4, 2, 3)):
            seq.append((cur[4] - cur[1], cur[2] - cur[4], cur[3] - cur[2], tt - cur[3]))
            cur = {}
if seq:
    a_ = np.array(seq)
    print(f"  fc1 publish: start->y {a_[:,0].mean():.2f}  y->prefence {a_[:,1].mean():.2f}  fence {a_[:,2].mean():.2f}  after {a_[:,3].mean():.2f} us (n={len(seq)})")
# consumer epilogue sub-steps (thread 0): mainloop end (2,1) -> scratch (5,1) -> V (5,2) -> barrier (5,3) -> encode (5,4) -> item end (2,2)
for p in (1, 2):
    segs = []
    for c in range(tr.shape[0]):
        evs = sorted((us[c, i], role[c, i], ev[c, i], ph[c, i]) for i in range(tr.shape[1]) if valid[c, i] and role[c, i] in (2, 5))
        cur = None
        for tt, ro, e, pp in evs:
            if ro == 2 and e == 1 and pp == p: cur = {'m': tt}
            elif cur is not None and ro == 5: cur[e] = tt
            elif cur is not None and ro == 2 and e == 2:
                cur['end'] = tt
                keys = ['m'] + [k for k in (1, 2, 3, 4) if k in cur] + ['end']
                if len(keys) == (6 if p == 1 else 4):
                    segs.append([cur[keys[i + 1]] - cur[keys[i]] for i in range(len(keys) - 1)])
                cur = None
    if segs:
        print(f"  phase {p} epilogue segments (us):", np.round(np.mean(np.array(segs), axis=0), 2), len(segs))
# mainloop: time from item start to mainloop end, and the part spent waiting for weights
ks = (w & np.uint64(0xFFFF)).astype(np.int64)
for p in (1, 2):
    ml, wt = [], []
    for c in range(tr.shape[0]):
        s0 = [us[c, i] for i in range(tr.shape[1]) if valid[c, i] and role[c, i] == 2 and ev[c, i] == 0 and ph[c, i] == p]
        s1 = [(us[c, i], ks[c, i]) for i in range(tr.shape[1]) if valid[c, i] and role[c, i] == 2 and ev[c, i] == 1 and ph[c, i] == p]
        for a0, (b0, wn) in zip(s0, s1):
            ml.append(b0 - a0)
            wt.append(wn / 1e3)
    if ml:
        print(f"  phase {p} mainloop: mean {np.mean(ml):.2f} us, of which waiting for weights {np.mean(wt):.2f} us")
# mainloop clock split (warp 0): mt = wait cycles/16, ks = compute cycles/16
mtv = ((w >> np.uint64(16)) & np.uint64(0xFFFF)).astype(np.int64)
for p in (1, 2):
    sel = valid & (role == 2) & (ev == 1) & (ph == p)
    if sel.any():
        print(f"  phase {p} mainloop cycles (warp 0): wait {16 * mtv[sel].mean():.0f}  compute {16 * ks[sel].mean():.0f} per item")
# consumer idle gaps (end -> next start) per CTA
gaps = []
for c in range(tr.shape[0]):
    s = sorted(us[c, i] for i in range(tr.shape[1]) if valid[c, i] and role[c, i] == 2 and ev[c, i] == 0)
    e_ = sorted(us[c, i] for i in range(tr.shape[1]) if valid[c, i] and role[c, i] == 2 and ev[c, i] == 2)
    for a0, b0 in zip(e_[:-1], s[1:]):
        gaps.append(b0 - a0)
if gaps:
    g_ = np.array(gaps)
    print(f"  consumer gaps between items: n={g_.size} mean {g_.mean():.2f} us  p50 {np.median(g_):.2f}  max {g_.max():.2f}")
