"""Small forced-GEMM-path parity probe (used before the full suite)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle, paper_2310_02410_b200 as m
from helpers import make_layer, allclose_report
orc = oracle.orc()
for (E, d, f, bits, T, k) in [(2, 128, 128, 4, 40, 1), (4, 256, 512, 3, 300, 1), (8, 1024, 4096, 2, 1000, 1), (4, 200, 300, 8, 77, 2)]:
    L = make_layer(orc, 5, E, d, f, bits, T)
    want, ex_o, _ = orc.moe_forward(L["h"], L["wg"], L["q1"], L["s1"], L["q2"], L["s2"], top_k=k)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    bank = m.ExpertBank(E, d, f, bits, t(L["p1"]), t(L["s1"]), t(L["p2"]), t(L["s2"]))
    out = m.moe_ffn_forward(t(L["h"]).half(), bank, t(L["wg"]), top_k=k, path="gemm")
    torch.cuda.synchronize()
    nbad, mx = allclose_report(out.cpu().numpy(), want)
    print(f"E={E} d={d} f={f} int{bits} T={T} k={k}: bad={nbad} maxabs={mx:.3e}", flush=True)
