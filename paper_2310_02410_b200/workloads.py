"""Seeded synthetic inputs for the BASELINE.json configs (bench + tests).

The reference measures nothing at the MoE-layer level on real data; every
BASELINE config is synthetic (activations ~N(0,1) rounded to fp16, weights and
gate ~N(0,0.02)). Config 5 asks for Zipf(1.2) expert popularity. The reference
router has no bias term (top1_route, /root/reference/proj/src/model.cpp:328-346),
so the bias is folded into the gate weights the way SURVEY.md §8(d) prescribes:
h[:, 0] = 1 and Wg[0, :] = bias. `zipf_bias` calibrates that bias once, from a
fixed seed, so argmax(logits) follows Zipf(1.2) over the experts.
"""
from __future__ import annotations

import numpy as np

ZIPF_S = 1.2


def zipf_target(E: int, s: float = ZIPF_S, seed: int = 5) -> np.ndarray:
    """Target routing probabilities: p(rank r) ~ r^-s, ranks assigned to experts
    by a seeded permutation (the popular experts are not simply 0, 1, 2 ...)."""
    p = np.arange(1, E + 1, dtype=np.float64) ** -s
    p /= p.sum()
    perm = np.random.default_rng(seed).permutation(E)
    out = np.empty(E)
    out[perm] = p
    return out


def zipf_bias(wg: np.ndarray, s: float = ZIPF_S, seed: int = 5, samples: int = 16384,
              iters: int = 200) -> np.ndarray:
    """Per-expert logit bias b (to be written into wg[0, :], with h[:, 0] = 1) such that
    argmax_e(h[1:] . wg[1:, e] + b_e) over h ~ N(0,1) follows zipf_target(E)."""
    d, E = wg.shape
    rng = np.random.default_rng(seed + 1)
    h = rng.standard_normal((samples, d - 1)).astype(np.float32)
    noise = (h @ wg[1:].astype(np.float32)).astype(np.float64)
    target = zipf_target(E, s, seed)
    b = np.log(target) * noise.std()
    for _ in range(iters):
        cnt = np.bincount(np.argmax(noise + b, axis=1), minlength=E)
        emp = (cnt + 0.5) / (samples + 0.5 * E)
        b += 0.5 * noise.std() * (np.log(target) - np.log(emp))
        b -= b.max()
    return b.astype(np.float32)


def apply_bias(h: np.ndarray, wg: np.ndarray, bias: np.ndarray):
    """Fold the bias into the router inputs."""
    h = np.array(h, copy=True)
    wg = np.array(wg, copy=True)
    h[:, 0] = 1.0
    wg[0, :] = bias
    return h, wg
