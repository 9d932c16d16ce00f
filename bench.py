#!/usr/bin/env python
"""bench.py — MoQE expert-FFN layer throughput on B200.

Headline workload (BASELINE.json configs[1], north-star decode point): one
MoE FFN layer, d_model=1024, d_ffn=4096, 32 experts, top-1, int3
per-channel experts, T=24 tokens (one decode step, batch 24), fp16
activations ~N(0,1), weights ~N(0,0.02), gate ~N(0,0.02). One step = one
moe_forward (route -> permute -> expert FFN -> combine) of one layer.
L2 hygiene: 8 independent layer replicas (different weights, routers and
inputs) rotate, so each step's weights were last touched 7 steps earlier
(total working set > 126 MB L2).

Prints ONE JSON line (rank 0). `--impl reference` times the reference's own
CPU moe_ffn_forward (oracle/_ref, built from /root/reference) on the host
cores on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE FFN tokens/s & packed-weight HBM GB/s (vs 8TB/s), int4/3/2, 1-8 B200"
SEED = 20231004
N_LAYERS = 8


def gemv_extra(d, T, top_k):
    """Kernels beside the timed "gemv" scope's first: the fc2 grid unless fc1 and fc2 run as
    one fused grid (capi.cu: self plan, fc1 in one 1024-k chunk), plus k_xrows unless the
    decode router writes the fc1 row blocks itself (self plan with the bank's router)."""
    fused = (T * top_k <= 64 and T <= 32 and d <= 1024 and os.environ.get("MOQE_GEMV_FUSED", "1") != "0")
    in_router = T * top_k <= 64 and T <= 32 and os.environ.get("MOQE_XROWS_IN_ROUTER", "1") != "0"
    return (0 if fused else 1) + (0 if in_router else 1)


def packed_bytes(bits: int, n: int) -> int:
    return 3 * ((n + 7) // 8) if bits == 3 else (n * bits + 7) // 8


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.15)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm = []
        mx = None
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for n, v in zip(names, r[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------
# workload

def layer0_numpy(E, d, f):
    """Layer 0 weights/inputs, generated identically for both arms (seeded numpy)."""
    rng = np.random.default_rng(SEED)
    w1 = (rng.standard_normal((E, d, f), dtype=np.float32) * np.float32(0.02))
    w2 = (rng.standard_normal((E, f, d), dtype=np.float32) * np.float32(0.02))
    wg = (rng.standard_normal((d, E), dtype=np.float32) * np.float32(0.02))
    return w1, w2, wg, rng


def tokens_numpy(rng, T, d):
    return rng.standard_normal((T, d), dtype=np.float32).astype(np.float16)


class GpuLayer:
    def __init__(self, m, bank, wg, h, touched, counts):
        self.m, self.bank, self.wg, self.h = m, bank, wg, h
        self.touched, self.counts = touched, counts


def build_gpu_layers(m, torch, E, d, f, bits, T, top_k, n_layers, dev, zipf=False):
    """zipf: BASELINE config 5 popularity (bias folded into Wg[0,:] with h[:,0] = 1,
    paper_2310_02410_b200.workloads.zipf_bias)."""
    from paper_2310_02410_b200.workloads import zipf_bias
    layers = []
    w1n, w2n, wgn, rng = layer0_numpy(E, d, f)
    for li in range(n_layers):
        if li == 0:
            w1 = torch.from_numpy(w1n).to(dev)
            w2 = torch.from_numpy(w2n).to(dev)
            wg = torch.from_numpy(wgn).to(dev)
            h = torch.from_numpy(tokens_numpy(rng, T, d)).to(dev)
        else:
            g = torch.Generator(device=dev).manual_seed(SEED + li)
            w1 = torch.randn((E, d, f), generator=g, device=dev) * 0.02
            w2 = torch.randn((E, f, d), generator=g, device=dev) * 0.02
            wg = torch.randn((d, E), generator=g, device=dev) * 0.02
            h = torch.randn((T, d), generator=g, device=dev).half()
        if zipf:
            wg = wg.clone()
            wg[0, :] = torch.from_numpy(zipf_bias(wg.float().cpu().numpy())).to(dev)
            h = h.clone()
            h[:, 0] = 1.0
        bank = m.ExpertBank.from_float(w1, w2, bits, router=wg)
        del w1, w2
        _, ex, _ = m.moe_ffn_forward(h, bank, top_k=top_k, return_routing=True)
        counts = torch.bincount(ex.reshape(-1).long(), minlength=E).cpu().numpy()
        layers.append(GpuLayer(m, bank, wg, h, int((counts > 0).sum()), counts))
    torch.cuda.synchronize()
    return layers


def kernel_bytes(L, d, f, bits, T, top_k, out_bytes=4):
    """Algorithmic bytes of the fused expert-FFN kernel (minus router):
    packed W1+W2 + fp16-equivalent scales of every touched expert + fp16 input
    rows + output rows."""
    per_expert = packed_bytes(bits, d * f) * 2 + 2 * (f + d)
    return L.touched * per_expert + T * top_k * d * 2 + T * d * out_bytes


def step_flops(d, f, E, T, top_k):
    return 2 * T * d * E + 4 * d * f * T * top_k


def capture(torch, fn, layers, idxs):
    """Capture one forward per listed layer into a CUDA graph (the forward is
    stream-ordered with no host sync, so the whole route -> FFN chain replays
    without host launch overhead)."""
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in idxs:
            fn(layers[i])
    return g


def time_steps(torch, fn, layers, steps, warmup, dist=None, graphs=True):
    """Device time of EXACTLY `steps` steps (layer i % L at step i), CUDA events
    on the replay stream, barrier + synchronize on both sides, max over ranks."""
    L = len(layers)
    if graphs:
        full = capture(torch, fn, layers, list(range(L)))
        rem = steps % L
        grem = capture(torch, fn, layers, list(range(rem))) if rem else None
        run = lambda: ([full.replay() for _ in range(steps // L)], grem.replay() if grem else None)
        for _ in range(max(1, -(-warmup // L))):
            full.replay()
    else:
        run = lambda: [fn(layers[i % L]) for i in range(steps)]
        for i in range(warmup):
            fn(layers[i % L])
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    st = torch.cuda.current_stream()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    run()
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms


def profile_spans(m, torch, layers, steps, fwd):
    """In-pipeline durations of the decode kernels, measured on the device (moqe_gpu_bank_span:
    first CTA start after the programmatic-launch wait -> last CTA exit, summed by the kernel
    itself), from a graph of one forward per layer replayed until >= `steps` forwards. No event
    nodes, so the launch chain keeps its programmatic edges. Returns per kind (0 router, 1 expert
    FFN incl. fused routing): (total us, launches)."""
    import ctypes as C
    lib = m.load_library()
    for L in layers:
        lib.moqe_gpu_bank_span(L.bank._h, 1)
    g = capture(torch, fwd, layers, list(range(len(layers))))
    for L in layers:
        lib.moqe_gpu_bank_span(L.bank._h, 0)
    tot = (C.c_double * 2)()
    cnt = (C.c_int64 * 2)()
    g.replay()
    for L in layers:
        lib.moqe_gpu_bank_span_read(L.bank._h, tot, cnt)  # discard the warm replay
    us = np.zeros(2)
    n = np.zeros(2, np.int64)
    for _ in range(max(1, -(-steps // len(layers)))):
        g.replay()
    for L in layers:
        lib.moqe_gpu_bank_span_read(L.bank._h, tot, cnt)
        us += np.array(tot[:])
        n += np.array(cnt[:])
    del g
    return us, n


def profile_kernels(m, torch, layers, steps, fwd):
    """Per-kernel CUDA-event durations on the launching stream (prefill kernels): a graph of one
    forward per layer with event nodes around every kernel, replayed until >= `steps` steps have
    been measured."""
    import ctypes as C
    lib = m.load_library()
    for L in layers:
        lib.moqe_gpu_bank_profile(L.bank._h, 1)
    g = capture(torch, fwd, layers, list(range(len(layers))))
    for L in layers:
        lib.moqe_gpu_bank_profile(L.bank._h, 0)
    g.replay()
    ms = (C.c_double * 6)()
    n = (C.c_int64 * 6)()
    for L in layers:
        lib.moqe_gpu_bank_profile_read(L.bank._h, ms, n, 1)  # discard the warm replay
    tot_ms = np.zeros(6)
    tot_n = np.zeros(6, np.int64)
    per_layer = [(np.zeros(6), np.zeros(6, np.int64)) for _ in layers]
    reps = max(1, -(-steps // len(layers)))
    for _ in range(reps):
        g.replay()
        for j, L in enumerate(layers):
            lib.moqe_gpu_bank_profile_read(L.bank._h, ms, n, 1)
            tot_ms += np.array(ms[:])
            tot_n += np.array(n[:])
            per_layer[j][0][:] += np.array(ms[:])
            per_layer[j][1][:] += np.array(n[:])
    for L in layers:
        lib.moqe_gpu_bank_profile_read(L.bank._h, ms, n, 0)
    del g
    return tot_ms, tot_n, per_layer


KINDS = ["route", "scatter", "gemv", "gemm_fc1", "gemm_fc2", "convert"]


def run_point(m, torch, E, d, f, bits, T, top_k, steps, warmup, dev, hbm_peak, tc_peak, dist=None,
              n_layers=N_LAYERS, detail=False, zipf=False):
    layers = build_gpu_layers(m, torch, E, d, f, bits, T, top_k, n_layers, dev, zipf=zipf)
    outs = [torch.empty((T, d), dtype=torch.float32, device=dev) for _ in layers]

    # reuse preallocated outputs to keep allocator traffic out of the loop
    def fwd_out(L, _o={id(L): o for L, o in zip(layers, outs)}):
        # the bank's router (set once per layer, like the reference's gate weights): its
        # blocked copy feeds the decode router's fast chain
        m.moe_ffn_forward(L.h, L.bank, top_k=top_k, out=_o[id(L)])

    ms = time_steps(torch, fwd_out, layers, steps, warmup, dist)
    span_us, span_n = profile_spans(m, torch, layers, steps, fwd_out)
    if span_n[1] > 0:
        # decode path (dec.cu): one k_dec launch per forward (routing fused in, or behind the
        # k_dec_route cluster); span = first CTA start after the PDL wait -> last CTA exit
        avg_us = span_us[1] / span_n[1]
        per_launch = float(np.mean([kernel_bytes(L, d, f, bits, T, top_k) + d * E * 4 for L in layers]))
        achieved = per_launch / (avg_us * 1e-6) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": None,
                "kernel": "k_dec (routing + expert FFN, one launch)" if span_n[0] == 0 else "k_dec expert FFN",
                "bytes_per_launch": int(per_launch), "avg_launch_us": round(avg_us, 3),
                "timing": "in-kernel globaltimer span (first CTA after PDL wait -> last CTA exit), inside the graph"}
        if span_n[0] > 0:
            roof["router_avg_us"] = round(span_us[0] / span_n[0], 3)
        prof_ms = np.zeros(6)
        prof_n = np.zeros(6, np.int64)
        prof_ms[2] = span_us[1] * 1e-3
        prof_n[2] = span_n[1]
        if span_n[0] > 0:
            prof_ms[0] = span_us[0] * 1e-3
            prof_n[0] = span_n[0]
        launches = (1 + (1 if span_n[0] > 0 else 0))
    else:
        prof_ms, prof_n, per_layer = profile_kernels(m, torch, layers, steps, fwd_out)
        # dominant expert-FFN kernel (the path's hot loop; the router is reported in kernel_share)
        ffn = [2, 3, 4]
        dom = ffn[int(np.argmax(prof_ms[ffn]))]
        avg_launch_ms = prof_ms[dom] / max(prof_n[dom], 1)
        if KINDS[dom] == "gemv":
            tot_b = sum(kernel_bytes(L, d, f, bits, T, top_k) * n[2] for L, (_, n) in zip(layers, per_layer))
            per_launch = tot_b / max(prof_n[2], 1)
            achieved = per_launch / (avg_launch_ms * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(achieved / hbm_peak, 4), "traffic": None,
                    "kernel": "k_gemv fc1+fc2", "bytes_per_launch": int(per_launch),
                    "avg_launch_us": round(avg_launch_ms * 1e3, 3)}
        else:
            # each tcgen05 phase is half of the expert-FFN FLOPs (2*d*f*T*k per phase)
            fl = 2 * d * f * T * top_k
            achieved = fl / (avg_launch_ms * 1e-3) / 1e12
            both_ms = (prof_ms[3] + prof_ms[4]) / max(prof_n[3], 1)
            roof = {"bound": "tensor", "achieved": round(achieved, 1), "peak": tc_peak, "unit": "TFLOP/s",
                    "frac": round(achieved / tc_peak, 4), "traffic": None, "kernel": "k_ffn_gemm " + KINDS[dom],
                    "flops_per_launch": int(fl), "avg_launch_us": round(avg_launch_ms * 1e3, 3),
                    "fc1_plus_fc2_TFLOPs": round(2 * fl / (both_ms * 1e-3) / 1e12, 1),
                    "timing": "CUDA event nodes around each kernel in the graph"}
        launches = None
    try:  # ncu-measured DRAM bytes per launch (dram__bytes_read+write.sum) of this kernel/config
        with open(os.path.join(ROOT, "profiles", "round2", "traffic.json")) as fh:
            tr = json.load(fh).get(f"int{bits}/T{T}/E{E}/k{top_k}")
        if tr:
            roof["traffic"] = tr["bytes_per_launch"]
            roof["traffic_source"] = tr["source"]
    except Exception:
        pass
    touched = float(np.mean([L.touched for L in layers]))
    step_b = np.mean([kernel_bytes(L, d, f, bits, T, top_k) for L in layers]) + d * E * 4
    res = {
        "bits": bits, "tokens": T, "top_k": top_k, "ms_per_step": ms,
        "tokens_per_s": T / (ms * 1e-3),
        "step_GBps": step_b / (ms * 1e-3) / 1e9,
        "step_TFLOPs": step_flops(d, f, E, T, top_k) / (ms * 1e-3) / 1e12,
        "touched_experts": touched, "roofline": roof,
        "kernel_share": {KINDS[k]: round(float(prof_ms[k] / max(prof_ms.sum(), 1e-12)), 4)
                         for k in range(6) if prof_n[k]},
        # kernels per forward: a "gemv" scope launches k_gemv (one fused fc1+fc2 grid for
        # decode batches of <= 64 routed rows, else fc1 + fc2) and is preceded by k_xrows
        # (token-row encoding, timed inside the "route" scope)
        "launches_per_step": launches if launches is not None else
        int(round((prof_n.sum() + gemv_extra(d, T, top_k) * prof_n[2]) / max(1, -(-steps // len(layers)) * len(layers)))),
    }
    return res, layers


def e2e_point(m, torch, layers, steps, warmup, top_k, d):
    """Through the by-value C-ABI call with pinned HOST buffers (H2D + D2H inside)."""
    hs = [L.h.cpu().pin_memory() for L in layers]
    T = hs[0].shape[0]
    outs = [torch.empty((T, d), dtype=torch.float32).pin_memory() for _ in layers]
    idx = {id(L): i for i, L in enumerate(layers)}

    def fn(L):
        i = idx[id(L)]
        m.moe_ffn_forward_host(hs[i], L.bank, top_k=top_k, out=outs[i])

    for L in layers:  # every replica's first host call sizes its staging buffers: not timed
        fn(L)
    ms = time_steps(torch, fn, layers, steps, warmup, graphs=False)
    return {"value": round(T / (ms * 1e-3), 1), "unit": "tokens/s",
            "h2d_bytes_per_step": int(T * d * 2), "d2h_bytes_per_step": int(T * d * 4),
            "ms_per_step": round(ms, 5)}


def run_config3(m, torch, steps, warmup, n_layers=36, T=768, seed=SEED):
    """BASELINE config 3: 36-layer pre-LN residual FFN stack (even layers 32-expert top-1 int3
    MoE, odd layers dense fp16 FFNs with 0.1 % outliers), 24 x 32 = 768 fp16 tokens. One step
    = one forward of the whole stack, replayed from a CUDA graph (weights 1.8 GB >> L2)."""
    from paper_2310_02410_b200.workloads import build_config3
    stack, _ = build_config3(m, torch, seed, n_layers=n_layers)
    g = torch.Generator(device="cuda").manual_seed(seed + 3)
    h = torch.randn((T, 1024), generator=g, device="cuda").half()
    stack.forward(h)
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        with torch.cuda.graph(gr, stream=st):
            stack.forward(h)
    for _ in range(max(warmup, 3)):
        gr.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        gr.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    del gr, stack
    torch.cuda.empty_cache()
    return {"config": "config3", "layers": n_layers, "tokens": T, "ms_per_step": round(ms, 4),
            "tokens_per_s": round(T / (ms * 1e-3), 1), "ms_per_layer": round(ms / n_layers, 5),
            "launch": "CUDA graph of the whole stack forward"}


# ---------------------------------------------------------------------------------------
# expert parallelism (N > 1): experts sharded E/G, T tokens per rank (weak scaling)

def run_point_ep(m, torch, dist, E, d, f, bits, T, top_k, steps, warmup, dev, rank, world, n_layers=N_LAYERS):
    from paper_2310_02410_b200.ep import ExpertParallelMoE, shard_range
    lo, hi = shard_range(E, world, rank)
    layers = []
    for li in range(n_layers):
        w1 = torch.empty((hi - lo, d, f), device=dev)
        w2 = torch.empty((hi - lo, f, d), device=dev)
        for e in range(lo, hi):  # expert e's weights are the same whichever rank owns it
            g = torch.Generator(device=dev).manual_seed(SEED + 1000 * li + e)
            w1[e - lo] = torch.randn((d, f), generator=g, device=dev) * 0.02
            w2[e - lo] = torch.randn((f, d), generator=g, device=dev) * 0.02
        gr = torch.Generator(device=dev).manual_seed(SEED + 1000 * li + 999)
        wg = torch.randn((d, E), generator=gr, device=dev) * 0.02
        gh = torch.Generator(device=dev).manual_seed(SEED + 7919 * (li + 1) + rank)
        h = torch.randn((T, d), generator=gh, device=dev).half()
        bank = m.ExpertBank.from_float(w1, w2, bits)
        del w1, w2
        layers.append((ExpertParallelMoE(bank, wg, E, top_k=top_k), h))
    torch.cuda.synchronize()
    fwd = lambda L: L[0].forward(L[1])
    ms = time_steps(torch, fwd, layers, steps, warmup, dist, graphs=False)
    # e2e: the same step from pinned HOST token rows to a pinned HOST output (H2D + D2H timed)
    hosts = {id(L): (L[1].cpu().pin_memory(), torch.empty((T, d), dtype=torch.float32).pin_memory())
             for L in layers}

    def fwd_host(L):
        hh, oh = hosts[id(L)]
        oh.copy_(L[0].forward(hh.to(dev, non_blocking=True)), non_blocking=True)

    ms_e2e = time_steps(torch, fwd_host, layers, max(steps // 2, 5), warmup, dist, graphs=False)
    # this library's kernels per step (CUPTI kernel records of one step per layer; NCCL excluded)
    launches = None
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for L in layers:
                fwd(L)
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
        ours = [n for n in names if "moqe_gpu::" in n or n.startswith("k_")]
        launches = len(ours) // len(layers) * steps if ours else None
    except Exception:  # profiler unavailable: no claim
        launches = None

    e2e = {"value": round(T * world / (ms_e2e * 1e-3), 1), "unit": "tokens/s", "h2d_bytes_per_step": int(T * d * 2),
           "d2h_bytes_per_step": int(T * d * 4), "ms_per_step": round(ms_e2e, 5)}
    return {"ms_per_step": ms, "tokens_per_s_per_rank": T / (ms * 1e-3), "experts_per_rank": hi - lo, "e2e": e2e,
            "gpu_launches": launches}


def ep_cpu_baseline(E, d, f, bits, top_k, sample_tokens=16, threads=None):
    """CPU baseline of the expert-parallel layer (BASELINE config 4). The reference routes
    top-1 only (top-2 is not in it), so this is the oracle port (oracle/moqe_oracle.c: the
    reference's router and per-row dequantize-on-the-fly FFN, model.cpp:328-393) on a bounded
    sample: `sample_tokens` rows x top-2 experts over the host threads, extrapolated to
    tokens/s (the per-token work does not depend on which expert it meets)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    orc = oracle.orc()
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(SEED)
    q1 = rng.integers(-(1 << (bits - 1)), 1 << (bits - 1), size=(d, f), dtype=np.int8)
    q2 = rng.integers(-(1 << (bits - 1)), 1 << (bits - 1), size=(f, d), dtype=np.int8)
    s1 = np.full(f, 0.01, np.float32)
    s2 = np.full(d, 0.01, np.float32)
    wg = (rng.standard_normal((d, E)) * 0.02).astype(np.float32)
    h = rng.standard_normal((sample_tokens, d)).astype(np.float16).astype(np.float32)
    t0 = time.perf_counter()
    orc.route(h, wg, top_k)
    with ThreadPoolExecutor(threads) as pool:  # ctypes releases the GIL
        list(pool.map(lambda i: orc.expert_ffn(h[i:i + 1].repeat(top_k, 0), q1, s1, q2, s2), range(sample_tokens)))
    dt = time.perf_counter() - t0
    return {"value": round(sample_tokens / dt, 3), "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"{sample_tokens} tokens x top-{top_k} of the d={d} f={f} int{bits} layer (oracle port: the "
                      f"reference has no top-2), {threads} threads, extrapolated per token"}


# ---------------------------------------------------------------------------------------
# reference CPU arm

def reference_baseline(E, d, f, bits, T, reps=3, threads=None, one_thread=True):
    """Time the reference moqe::moe_ffn_forward (oracle/_ref) on the host cores the way
    BASELINE.md §2 / SURVEY.md §8(d) ask (bench.cpp:96-107 convention: 1 discarded warm-up,
    median of `reps`): token-sharded over all host threads (bit-identical to 1 thread) and,
    when one_thread, single-threaded as the reference runs. The one-time quantize-experts cost
    (quantize_linear + pack of every expert matrix, 1 thread) is timed too."""
    import oracle
    kind = "reference" if oracle.ref_available() else "port"
    lib = oracle.ref() if kind == "reference" else oracle.orc()
    orc = oracle.orc()
    w1, w2, wg, rng = layer0_numpy(E, d, f)
    h = tokens_numpy(rng, T, d).astype(np.float32)
    q1 = np.empty((E, d, f), np.int8)
    q2 = np.empty((E, f, d), np.int8)
    s1 = np.empty((E, f), np.float32)
    s2 = np.empty((E, d), np.float32)
    t0 = time.perf_counter()
    for e in range(E):  # quantize-experts (model.cpp:577-636), packed as write_checkpoint does
        q1[e], s1[e] = lib.quantize_linear(w1[e], bits)
        q2[e], s2[e] = lib.quantize_linear(w2[e], bits)
        lib.pack(q1[e], bits)
        lib.pack(q2[e], bits)
    quant_s = time.perf_counter() - t0
    del w1, w2
    threads = threads or os.cpu_count() or 1
    if kind == "reference":
        bank = oracle.ref().bank(q1, s1, q2, s2, bits)
        run = lambda n: bank.forward(h, wg, n)
    else:
        run = lambda n: orc.moe_forward(h, wg, q1, s1, q2, s2, n_threads=n)

    def timed(n):
        run(n)  # discarded warm-up
        ts = []
        for _ in range(reps):
            t1 = time.perf_counter()
            run(n)
            ts.append(time.perf_counter() - t1)
        return statistics.median(ts)

    med = timed(threads)
    res = {"value": round(T / med, 3), "unit": "tokens/s", "cores": threads, "kind": kind,
           "sample": f"T={T} int{bits} E={E} d={d} f={f} top-1 layer; 1 warm-up + median of {reps} "
                     f"timed moe_ffn_forward calls, token-sharded over {threads} threads",
           "seconds_per_step": round(med, 4),
           "quantize_experts_s_1thread": round(quant_s, 3)}
    if one_thread and threads > 1:
        med1 = timed(1)
        res["one_thread"] = {"value": round(T / med1, 3), "unit": "tokens/s", "cores": 1,
                             "seconds_per_step": round(med1, 4)}
    return res


# ---------------------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--bits", type=int, default=3)
    ap.add_argument("--tokens", type=int, default=24)
    ap.add_argument("--experts", type=int, default=32)
    ap.add_argument("--d-model", type=int, default=1024)
    ap.add_argument("--d-ffn", type=int, default=4096)
    ap.add_argument("--top-k", type=int, default=1)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ep", action="store_true", help="expert-parallel path (config 4) even at one rank")
    ap.add_argument("--keep-shape", action="store_true", help="EP runs keep the given shape instead of config 4")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if (world > 1 or args.ep) and not args.keep_shape:
        # multi-GPU runs measure BASELINE config 4: d=2048, f=8192, 128 experts sharded over the
        # ranks, top-2 renormalised, int2, 16384 tokens per rank
        args.experts, args.d_model, args.d_ffn, args.top_k, args.bits, args.tokens = 128, 2048, 8192, 2, 2, 16384
        args.steps = min(args.steps, 40)
    E, d, f, bits, T, k = args.experts, args.d_model, args.d_ffn, args.bits, args.tokens, args.top_k
    config = {"workload": f"config2 decode: MoE FFN layer d_model={d} d_ffn={f} {E} experts top-{k} "
                          f"int{bits} per-channel, T={T} tokens",
              "d_model": d, "d_ffn": f, "experts": E, "top_k": k, "weight_bits": bits, "tokens": T,
              "activations": "fp16 ~N(0,1)", "weights": "~N(0,0.02) quantized per output channel",
              "l2": f"{N_LAYERS} rotating layer replicas (working set > 126 MB L2)", "seed": SEED,
              "launch": f"CUDA graph replay, one graph = {N_LAYERS} layer forwards"}

    if args.impl == "reference":
        if rank != 0:
            return
        base = reference_baseline(E, d, f, bits, T, one_thread=False)
        line = {"metric": METRIC, "value": base["value"], "unit": "tokens/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": base["seconds_per_step"] * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": config, "impl": "reference",
                "cpu_baseline": {k2: base[k2] for k2 in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": base["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2310_02410_b200 as m

    dist = None
    if world > 1:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        dist = tdist
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    m.load_library()
    hbm_peak, tc_peak, peak_kind = load_peaks()

    if world > 1 or args.ep:
        if dist is None:
            import torch.distributed as tdist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            tdist.init_process_group("nccl", world_size=1, rank=0, device_id=dev)
            dist = tdist
        sampler = ClockSampler(local) if rank == 0 else None
        if sampler:
            sampler.start()
        ep = run_point_ep(m, torch, dist, E, d, f, bits, T, k, args.steps, args.warmup, dev, rank, world,
                          n_layers=4)
        clocks = sampler.stop() if sampler else None
        if rank == 0:
            config["workload"] = (f"config4 expert-parallel MoE FFN layer d_model={d} d_ffn={f} {E} experts "
                                  f"({ep['experts_per_rank']}/rank) top-{k} renormalised int{bits}, "
                                  f"T={T} tokens per rank")
            config["parallelism"] = f"ep{world}"
            fl = 2 * T * d * E + 4 * d * f * T * k  # per rank (router + fc1 + fc2 of every routed row)
            ach = fl / (ep["ms_per_step"] * 1e-3) / 1e12
            roof = {"bound": "tensor", "achieved": round(ach, 1), "peak": tc_peak, "unit": "TFLOP/s",
                    "frac": round(ach / tc_peak, 4), "traffic": None, "kernel": "whole EP layer step per rank",
                    "flops_per_step_per_rank": int(fl), "peak_kind": peak_kind,
                    "timing": "CUDA events around the eager step, max over ranks"}
            cpu = ep_cpu_baseline(E, d, f, bits, k) if not args.no_cpu else None
            line = {"metric": METRIC, "value": round(ep["tokens_per_s_per_rank"] * world, 1), "unit": "tokens/s",
                    "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                    "ms_per_step": round(ep["ms_per_step"], 5), "higher_is_better": True, "scaling": "weak",
                    "vs_baseline": None, "dtype": "f16", "data": "synthetic", "config": config,
                    "roofline": roof, "cpu_baseline": cpu, "e2e": ep["e2e"], "gpu_launches": ep["gpu_launches"], "clocks": clocks,
                    "detail": {"note": "eager EP steps: router kernel, device dispatch (k_ep_plan + k_ep_pack: "
                                       "packed fp16 records, one NCCL all_to_all + a G-int count exchange), owner "
                                       "expert FFN kernels, fp16 return all_to_all, k_ep_combine; max over ranks"}}
            print(json.dumps(line), flush=True)
        dist.barrier()
        dist.destroy_process_group()
        return

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    head, layers = run_point(m, torch, E, d, f, bits, T, k, args.steps, args.warmup, dev, hbm_peak,
                             tc_peak, dist)
    clocks = sampler.stop() if sampler else None
    e2e = e2e_point(m, torch, layers, max(args.steps // 4, 20), args.warmup, k, d) if rank == 0 else None
    del layers
    torch.cuda.empty_cache()

    sweep = []
    if rank == 0 and world == 1 and not args.no_sweep:
        # (config, E, bits, T, zipf): BASELINE config 2 bit sweep (+ T=16384 tensor point), config 1,
        # config 5 Zipf(1.2) skew over 64 experts
        pts = [("config2", E, b, t, False) for b in (8, 4, 3, 2) for t in (24, 4096)]
        pts += [("config2", E, 3, 16384, False), ("config2", E, 2, 16384, False), ("config1", 32, 4, 512, False)]
        pts += [("config5", 64, 4, t, True) for t in (1, 8, 64, 512, 4096, 32768)]
        for cfg, e_, b, t, zf in pts:
            if (cfg, e_, b, t) == ("config2", E, bits, T):
                continue
            try:
                r, lay = run_point(m, torch, e_, d, f, b, t, 1, max(min(args.steps, 60), 10), 5, dev,
                                   hbm_peak, tc_peak, n_layers=4 if t >= 4096 else N_LAYERS, zipf=zf)
                del lay
                torch.cuda.empty_cache()
                r = {kk: (round(v, 5) if isinstance(v, float) else v) for kk, v in r.items()}
                r["config"] = cfg
                r["experts"] = e_
                sweep.append(r)
            except Exception as ex:  # report, never hide
                sweep.append({"config": cfg, "experts": e_, "bits": b, "tokens": t, "error": str(ex)[:200]})

        try:
            sweep.append(run_config3(m, torch, max(min(args.steps // 20, 20), 5), 3))
        except Exception as ex:  # report, never hide
            sweep.append({"config": "config3", "error": str(ex)[:200]})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = reference_baseline(E, d, f, bits, T)
        cpu.pop("seconds_per_step", None)
        if "one_thread" in cpu:
            cpu["one_thread"].pop("seconds_per_step", None)

    if rank == 0:
        value = head["tokens_per_s"] * world
        roof = dict(head["roofline"])
        roof["peak_kind"] = peak_kind
        line = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(head["ms_per_step"], 5),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
                "data": "synthetic", "config": config, "roofline": roof, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": head["launches_per_step"] * args.steps,
                "clocks": clocks,
                "detail": {"step_GBps": round(head["step_GBps"], 1),
                           "step_TFLOPs": round(head["step_TFLOPs"], 3),
                           "touched_experts": head["touched_experts"],
                           "kernel_share": head["kernel_share"],
                           "accumulate": "f32", "weights": f"int{bits} codes -> f16 in registers/smem"},
                "sweep": sweep}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
