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
