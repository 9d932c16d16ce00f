"""Breakdown of the host-buffer forward (moqe_gpu_moe_forward_host) on the headline layer:
the by-value call, its pieces, and variants (kernel writing the pinned host output directly).
usage: python tools/e2e_probe.py"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_02410_b200 as m  # noqa: E402
from paper_2310_02410_b200 import _lib  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(1)
E, d, f, T = 32, 1024, 4096, 24
banks = []
for i in range(8):
    w1 = torch.randn(E, d, f, device="cuda", generator=g) * 0.02
    w2 = torch.randn(E, f, d, device="cuda", generator=g) * 0.02
    wg = torch.randn(d, E, device="cuda", generator=g) * 0.02
    banks.append(m.ExpertBank.from_float(w1, w2, 3, router=wg))
    del w1, w2
hs = [torch.randn(T, d, device="cuda", generator=g).half().cpu().pin_memory() for _ in banks]
outs = [torch.empty(T, d).pin_memory() for _ in banks]
hd = [h.cuda() for h in hs]
od = [torch.empty(T, d, device="cuda") for _ in banks]
lib = _lib.load()


def bench(fn, n=400):
    for i in range(24):
        fn(i % 8)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        fn(i % 8)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


s = torch.cuda.current_stream()
sp = C.c_void_p(s.cuda_stream)


def fwd_dev_out(i, out_ptr):
    r = lib.moqe_gpu_moe_forward(banks[i]._h, C.c_void_p(hd[i].data_ptr()), _lib.F16, T, None, 1,
                                 C.c_void_p(out_ptr), _lib.F32, None, None, 0, sp)
    assert r == 0, r


print("host API e2e            %.1f us" % bench(lambda i: m.moe_ffn_forward_host(hs[i], banks[i], out=outs[i])))
print("device fwd + sync       %.1f us" % bench(lambda i: (fwd_dev_out(i, od[i].data_ptr()), s.synchronize())))
print("device fwd no sync      %.1f us" % bench(lambda i: fwd_dev_out(i, od[i].data_ptr())))
print("fwd -> pinned out + sync %.1f us" % bench(lambda i: (fwd_dev_out(i, outs[i].data_ptr()), s.synchronize())))


def h2d_fwd_pinned(i):
    hd[i].copy_(hs[i], non_blocking=True)
    fwd_dev_out(i, outs[i].data_ptr())
    s.synchronize()


print("H2D + fwd->pinned + sync %.1f us" % bench(h2d_fwd_pinned))


def copies(i):
    hd[i].copy_(hs[i], non_blocking=True)
    outs[i].copy_(od[i], non_blocking=True)
    s.synchronize()


print("H2D+D2H+sync only       %.1f us" % bench(copies))
print("H2D+sync only           %.1f us" % bench(lambda i: (hd[i].copy_(hs[i], non_blocking=True), s.synchronize())))
print("sync only               %.1f us" % bench(lambda i: s.synchronize()))
ok = torch.equal(outs[0], od[0].cpu()) if False else None
fwd_dev_out(0, od[0].data_ptr()); fwd_dev_out(0, outs[0].data_ptr()); s.synchronize()
print("pinned-out result identical:", torch.equal(outs[0], od[0].cpu()))

# the same call replayed from a CUDA graph (H2D copy node + forward kernel, output stored into the
# pinned host buffer by the kernel): what a per-signature graph cache in the C-ABI would buy
graphs = []
gs = torch.cuda.Stream()
for i in range(8):
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(gs):
        fwd_dev_out(i, outs[i].data_ptr())  # warm (workspace, lazy init) outside capture
        gs.synchronize()
        with torch.cuda.graph(gr, stream=gs):
            hd[i].copy_(hs[i], non_blocking=True)
            r = lib.moqe_gpu_moe_forward(banks[i]._h, C.c_void_p(hd[i].data_ptr()), _lib.F16, T, None, 1,
                                         C.c_void_p(outs[i].data_ptr()), _lib.F32, None, None, 0,
                                         C.c_void_p(gs.cuda_stream))
            assert r == 0
    graphs.append(gr)
torch.cuda.synchronize()
print("graph(H2D + fwd->pinned) + sync %.1f us" % bench(lambda i: (graphs[i].replay(), torch.cuda.current_stream().synchronize(), gs.synchronize())))
