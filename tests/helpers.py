"""Seeded synthetic layers shared by the parity tests (inputs only; the
oracle computes every expected value)."""
from __future__ import annotations

import numpy as np


def fp16_valued(a):
    return np.asarray(a, np.float32).astype(np.float16).astype(np.float32)


def make_layer(orc, seed, E, d, f, bits, T, wscale=0.02, with_bias=False, zipf_bias=None):
    """Expert bank quantized by the oracle (reference quantizer restatement)."""
    rng = np.random.default_rng(seed)
    w1 = (rng.standard_normal((E, d, f)) * wscale).astype(np.float32)
    w2 = (rng.standard_normal((E, f, d)) * wscale).astype(np.float32)
    q1 = np.zeros(w1.shape, np.int8)
    q2 = np.zeros(w2.shape, np.int8)
    s1 = np.zeros((E, f), np.float32)
    s2 = np.zeros((E, d), np.float32)
    for x in range(E):
        q1[x], s1[x] = orc.quantize_linear(w1[x], bits)
        q2[x], s2[x] = orc.quantize_linear(w2[x], bits)
    h = fp16_valued(rng.standard_normal((T, d)))
    wg = (rng.standard_normal((d, E)) * 0.02).astype(np.float32)
    if zipf_bias is not None:
        h[:, 0] = 1.0
        wg[0, :] = zipf_bias
    b1 = (rng.standard_normal((E, f)) * 0.05).astype(np.float32) if with_bias else None
    b2 = (rng.standard_normal((E, d)) * 0.05).astype(np.float32) if with_bias else None
    p1 = np.stack([orc.pack(q1[x], bits) for x in range(E)])
    p2 = np.stack([orc.pack(q2[x], bits) for x in range(E)])
    return dict(w1=w1, w2=w2, q1=q1, q2=q2, s1=s1, s2=s2, p1=p1, p2=p2, h=h, wg=wg, b1=b1, b2=b2,
                E=E, d=d, f=f, bits=bits)


def allclose_report(got, ref, atol=2e-3, rtol=1e-2):
    """Tolerance from BASELINE.json north_star: |gpu-ref| <= atol + rtol*|ref|."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    diff = np.abs(got - ref)
    bad = diff > atol + rtol * np.abs(ref)
    return int(bad.sum()), float(diff.max() if diff.size else 0.0)


def sampled_moe_expected(orc, h, wg, top_k, tokens, expert_codes, ex_all, g_all, b1=None, b2=None,
                         threads=8):
    """Oracle MoE outputs for a SAMPLE of tokens (rows are independent:
    /root/reference/proj/src/model.cpp:360-391 touches a token only through its own
    experts). expert_codes(e) -> (q1, s1, q2, s2) from the oracle quantizer; ex_all /
    g_all are the oracle's routing of ALL tokens ([T] or [T, k]). out[t] = g0*y0
    (+ g1*y1), fp32, in slot order like oracle/moqe_oracle.c run_shard."""
    from concurrent.futures import ThreadPoolExecutor
    ex = np.asarray(ex_all).reshape(len(ex_all), -1)
    g = np.asarray(g_all, np.float32).reshape(len(g_all), -1)
    need = {}
    for i, t in enumerate(tokens):
        for k in range(top_k):
            need.setdefault(int(ex[t, k]), []).append((i, k))
    ys = {}

    def run(e):
        q1, s1, q2, s2 = expert_codes(e)
        rows = need[e]
        x = np.stack([h[tokens[i]] for i, _ in rows]).astype(np.float32)
        y = orc.expert_ffn(x, q1, s1, q2, s2, None if b1 is None else b1[e], None if b2 is None else b2[e])
        return e, y

    with ThreadPoolExecutor(threads) as pool:  # ctypes releases the GIL
        for e, y in pool.map(run, sorted(need)):
            for r, (i, k) in enumerate(need[e]):
                ys[(i, k)] = y[r]
    d = h.shape[1]
    out = np.zeros((len(tokens), d), np.float32)
    for i, t in enumerate(tokens):
        o = g[t, 0] * ys[(i, 0)]
        for k in range(1, top_k):
            o = o + g[t, k] * ys[(i, k)]
        out[i] = o
    return out


def check_routing(orc, h, wg, top_k, ex, g, gap_tol=1e-4, gate_rtol=1e-5):
    """Routing parity (BASELINE.json north_star): expert ids equal the oracle's except for
    tokens whose oracle top-(k+1) logit gap is below 1e-4 (the GPU sums the logits in a
    parallel order); gates of the other tokens within gate_rtol."""
    ex_o, g_o = orc.route(h, wg, top_k)
    lg = orc.router_logits(h, wg)
    top = -np.sort(-lg, axis=1)[:, : top_k + 1]
    gap = np.min(top[:, :-1] - top[:, 1:], axis=1) if lg.shape[1] > top_k else np.full(len(h), np.inf)
    sep = ~(gap < gap_tol)  # NaN gaps (non-finite logits) count as separated
    ex = np.asarray(ex).reshape(ex_o.shape)
    g = np.asarray(g, np.float64).reshape(g_o.shape)
    bad = (ex != ex_o).reshape(len(ex_o), -1).any(axis=1) & sep
    assert not bad.any(), ("routing differs on well-separated tokens", np.flatnonzero(bad)[:8])
    gs = sep if g.ndim == 1 else sep[:, None]
    with np.errstate(invalid="ignore", divide="ignore"):
        rel = np.abs(g - g_o) / np.abs(g_o)
    ok = (rel <= gate_rtol) | (g == g_o) | (np.isnan(g) & np.isnan(g_o)) | ~gs
    assert ok.all(), ("gate mismatch", float(np.nanmax(np.where(gs, rel, 0))))
    return ex_o, g_o
