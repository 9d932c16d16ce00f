"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the dev container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
The fixtures are committed; the GPU box never needs /root/reference.
Inputs are seeded numpy draws; the reference computes every output.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def fp16_valued(a: np.ndarray) -> np.ndarray:
    return a.astype(np.float16).astype(np.float32)


def main() -> None:
    oracle.build(ref=True)
    ref = oracle.ref()
    rng = np.random.default_rng(20260823)

    # quantizer + packer: per-channel and per-tensor, every width
    quant = {}
    for bits in (2, 3, 4, 8):
        w = (rng.standard_normal((96, 80)) * 0.3).astype(np.float32)
        w[:, 7] = 0.0  # an all-zero channel -> scale 0, codes 0
        for gname, pt in (("channel", False), ("tensor", True)):
            q, s = ref.quantize_linear(w, bits, pt)
            quant[f"w_{bits}_{gname}"] = w
            quant[f"codes_{bits}_{gname}"] = q
            quant[f"scales_{bits}_{gname}"] = s
            quant[f"packed_{bits}_{gname}"] = ref.pack(q, bits)
        # ragged counts (not multiples of 8): packing of flat arrays
        for count in (0, 1, 5, 9, 26, 63):
            c = rng.integers(-(1 << (bits - 1)), 1 << (bits - 1), count).astype(np.int8)
            quant[f"ragged_codes_{bits}_{count}"] = c
            quant[f"ragged_packed_{bits}_{count}"] = ref.pack(c, bits)
    np.savez_compressed(os.path.join(OUT, "quant.npz"), **quant)

    # routing (top-1): reference argmax + softmax gate
    route = {}
    for i, (t, d, e) in enumerate(((32, 8, 5), (24, 64, 8), (40, 1024, 32))):
        h = fp16_valued(rng.standard_normal((t, d)))
        wg = (rng.standard_normal((d, e)) * (1.0 if d <= 8 else 0.02)).astype(np.float32)
        ex, g = ref.top1_route(h, wg)
        route[f"h_{i}"], route[f"wg_{i}"], route[f"expert_{i}"], route[f"gate_{i}"] = h, wg, ex, g
    np.savez_compressed(os.path.join(OUT, "route.npz"), **route)

    # full MoE layer through moqe::moe_ffn_forward (quantized bank), each width
    E, d, f, T = 4, 64, 128, 24
    moe = {}
    for bits in (2, 3, 4, 8):
        w1 = (rng.standard_normal((E, d, f)) * 0.02).astype(np.float32)
        w2 = (rng.standard_normal((E, f, d)) * 0.02).astype(np.float32)
        q1 = np.zeros(w1.shape, np.int8)
        q2 = np.zeros(w2.shape, np.int8)
        s1 = np.zeros((E, f), np.float32)
        s2 = np.zeros((E, d), np.float32)
        for x in range(E):
            q1[x], s1[x] = ref.quantize_linear(w1[x], bits)
            q2[x], s2[x] = ref.quantize_linear(w2[x], bits)
        b1 = (rng.standard_normal((E, f)) * 0.1).astype(np.float32) if bits == 4 else None
        b2 = (rng.standard_normal((E, d)) * 0.1).astype(np.float32) if bits == 4 else None
        h = fp16_valued(rng.standard_normal((T, d)))
        wg = (rng.standard_normal((d, E)) * 0.02).astype(np.float32)
        bank = ref.bank(q1, s1, q2, s2, bits, b1, b2)
        out = bank.forward(h, wg, 1)
        ex, g = ref.top1_route(h, wg)
        rec = dict(q1=q1, s1=s1, q2=q2, s2=s2, h=h, wg=wg, out=out, expert=ex, gate=g)
        rec["p1"] = np.stack([ref.pack(q1[x], bits) for x in range(E)])
        rec["p2"] = np.stack([ref.pack(q2[x], bits) for x in range(E)])
        if b1 is not None:
            rec["b1"], rec["b2"] = b1, b2
        for k, v in rec.items():
            moe[f"{k}_{bits}"] = v
    np.savez_compressed(os.path.join(OUT, "moe.npz"), **moe)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
