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


def build_config3(m, torch, seed: int, n_layers: int = 36, E: int = 32, d: int = 1024, f: int = 4096,
                  bits: int = 3, outlier_frac: float = 1e-3, keep_f32: bool = False):
    """BASELINE config 3: a pre-LN residual FFN stack (no attention). Even layers are E-expert
    top-1 MoE FFNs with `bits`-bit per-channel experts, odd layers dense fp16 FFNs
    d -> f -> d with weights ~N(0,0.02) and `outlier_frac` of entries scaled x8. LayerNorm
    gains ~1 + N(0,0.05), biases ~N(0,0.05); dense biases ~N(0,0.01); routers ~N(0,0.02).
    Weights are drawn on the device from `seed`. keep_f32: also return the f32 expert weights
    and the gate weights (the oracle re-quantizes them)."""
    from .stack import DenseFFN, FfnStack, StackLayer
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(seed)
    layers, raw = [], []
    for i in range(n_layers):
        gain = 1.0 + 0.05 * torch.randn(d, generator=g, device=dev)
        bias = 0.05 * torch.randn(d, generator=g, device=dev)
        if i % 2 == 0:
            w1 = torch.randn((E, d, f), generator=g, device=dev) * 0.02
            w2 = torch.randn((E, f, d), generator=g, device=dev) * 0.02
            wg = torch.randn((d, E), generator=g, device=dev) * 0.02
            bank = m.ExpertBank.from_float(w1, w2, bits, router=wg)
            layers.append(StackLayer(gain, bias, moe=bank))
            raw.append({"kind": "moe", "w1": w1 if keep_f32 else None, "w2": w2 if keep_f32 else None, "wg": wg})
            if not keep_f32:
                del w1, w2
        else:
            def dense_w(k, n):
                w = torch.randn((k, n), generator=g, device=dev) * 0.02
                mask = torch.rand((k, n), generator=g, device=dev) < outlier_frac
                return torch.where(mask, w * 8.0, w).to(torch.float16)
            w1 = dense_w(d, f)
            w2 = dense_w(f, d)
            b1 = 0.01 * torch.randn(f, generator=g, device=dev)
            b2 = 0.01 * torch.randn(d, generator=g, device=dev)
            layers.append(StackLayer(gain, bias, dense=DenseFFN(w1, w2, b1, b2)))
            raw.append({"kind": "dense"})
    fg = 1.0 + 0.05 * torch.randn(d, generator=g, device=dev)
    fb = 0.05 * torch.randn(d, generator=g, device=dev)
    return FfnStack(layers, fg, fb), raw
