import time, sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2310_02410_b200 as m
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
def bench(fn, n=400):
    for _ in range(20): fn(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n): fn(i % 8)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6
s = torch.cuda.current_stream()
print("host API e2e        %.1f us" % bench(lambda i: m.moe_ffn_forward_host(hs[i], banks[i], out=outs[i])))
print("device fwd + sync   %.1f us" % bench(lambda i: (m.moe_ffn_forward(hd[i], banks[i], out=od[i]), s.synchronize())))
print("device fwd no sync  %.1f us" % bench(lambda i: m.moe_ffn_forward(hd[i], banks[i], out=od[i])))
def copies(i):
    hd[i].copy_(hs[i], non_blocking=True); outs[i].copy_(od[i], non_blocking=True); s.synchronize()
print("H2D+D2H+sync only   %.1f us" % bench(copies))
