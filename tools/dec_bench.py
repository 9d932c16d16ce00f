"""Decode-layer timing: N independent layers rotating (working set > L2), one CUDA graph
of N forwards replayed; prints us/forward and the in-kernel spans (router, expert FFN).

usage: python tools/dec_bench.py [--bits 3] [--tokens 24] [--experts 32] [--layers 8] [--topk 1]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_02410_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, nargs="+", default=[3])
ap.add_argument("--tokens", type=int, default=24)
ap.add_argument("--experts", type=int, default=32)
ap.add_argument("--d", type=int, default=1024)
ap.add_argument("--f", type=int, default=4096)
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--topk", type=int, default=1)
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--isolated", action="store_true", help="also report the span of isolated (synchronised) forwards")
a = ap.parse_args()
lib = m.load_library()


def packed(bits, n):
    return 3 * ((n + 7) // 8) if bits == 3 else (n * bits + 7) // 8


for bits in a.bits:
    banks, hs, outs, touched = [], [], [], []
    for li in range(a.layers):
        g = torch.Generator(device="cuda").manual_seed(100 + li)
        w1 = torch.randn(a.experts, a.d, a.f, device="cuda", generator=g) * 0.02
        w2 = torch.randn(a.experts, a.f, a.d, device="cuda", generator=g) * 0.02
        wg = torch.randn(a.d, a.experts, device="cuda", generator=g) * 0.02
        banks.append(m.ExpertBank.from_float(w1, w2, bits, router=wg))
        del w1, w2
        hs.append(torch.randn(a.tokens, a.d, device="cuda", generator=g).half())
        outs.append(torch.empty(a.tokens, a.d, device="cuda"))
        _, ex, _ = m.moe_ffn_forward(hs[-1], banks[-1], top_k=a.topk, return_routing=True)
        touched.append(int((torch.bincount(ex.reshape(-1).long(), minlength=a.experts) > 0).sum()))

    def fwd():
        for i in range(a.layers):
            m.moe_ffn_forward(hs[i], banks[i], top_k=a.topk, out=outs[i])

    fwd()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(gr, stream=st):
            fwd()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        gr.replay()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) * 1e3 / (a.reps * a.layers)
    # spans
    for b in banks:
        lib.moqe_gpu_bank_span(b._h, 1)
    gr2 = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        with torch.cuda.graph(gr2, stream=st):
            fwd()
    for b in banks:
        lib.moqe_gpu_bank_span(b._h, 0)
    tot = (C.c_double * 2)()
    cnt = (C.c_int64 * 2)()
    for b in banks:
        lib.moqe_gpu_bank_span_read(b._h, tot, cnt)
    sums = np.zeros(2)
    ns = np.zeros(2)
    for _ in range(a.reps):
        gr2.replay()
    for b in banks:
        lib.moqe_gpu_bank_span_read(b._h, tot, cnt)
        sums += np.array(tot[:])
        ns += np.array(cnt[:])
    span = sums / np.maximum(ns, 1)
    if a.isolated:
        for b in banks:
            lib.moqe_gpu_bank_span(b._h, 1)
            lib.moqe_gpu_bank_span_read(b._h, tot, cnt)
        isums, ins = np.zeros(2), np.zeros(2)
        for _ in range(10):
            for i in range(a.layers):
                m.moe_ffn_forward(hs[i], banks[i], top_k=a.topk, out=outs[i])
                torch.cuda.synchronize()
        for b in banks:
            lib.moqe_gpu_bank_span_read(b._h, tot, cnt)
            isums += np.array(tot[:])
            ins += np.array(cnt[:])
            lib.moqe_gpu_bank_span(b._h, 0)
        print(f"  isolated forwards: span ffn {isums[1] / max(ins[1], 1):.2f} us")
    wbytes = np.mean(touched) * (2 * packed(bits, a.d * a.f) + 2 * (a.d + a.f))
    print(f"int{bits} T={a.tokens} k={a.topk} E={a.experts}: {us:.2f} us/forward ({a.tokens / us * 1e6:,.0f} tok/s), "
          f"touched {np.mean(touched):.1f}, weights {wbytes / 1e6:.1f} MB -> {wbytes / us / 1e3:.0f} GB/s per step; "
          f"span router {span[0]:.2f} us, ffn {span[1]:.2f} us ({wbytes / max(span[1], 1e-9) / 1e3:.0f} GB/s)",
          flush=True)
    del banks, gr, gr2
    torch.cuda.empty_cache()
