// route.cu — fused gating (top-1 / top-2) + stable token permutation.
//
// Reference: top1_route proj/src/model.cpp:328-346 (logits = matmul :152-167,
// softmax_rows :214-227), gather loop :360-364 / :377-379.
//
// Logits are computed exactly as the reference does: fp32, products rounded
// (__fmul_rn) then added (__fadd_rn) in ascending k, zero activations
// skipped — so they are bit-identical and the argmax (strict '>', ties to the
// lowest index) matches the reference on every token. The gate is the softmax
// probability of the winner computed in fp64. Top-2 (BASELINE config 4) adds a
// second argmax over the remaining experts and renormalised gates
// g1 = 1/(1+exp(l2-l1)), g2 = exp(l2-l1)/(1+exp(l2-l1)).
//
// Permutation: rows are grouped by expert in ascending (token, slot) order,
// exactly the order of the reference's per-expert gather. Each routing CTA
// computes its local histogram and stable local ranks; the last CTA to finish
// (ticket) scans the per-CTA histograms, builds offsets, the per-path expert
// lists and resets the downstream schedulers — no extra launch, no host sync.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "ptx.cuh"
#include "xrow.cuh"

namespace moqe_gpu {

__device__ __forceinline__ float load_act(const void* h, int h_f16, int64_t idx) {
    return h_f16 ? __half2float(static_cast<const __half*>(h)[idx]) : static_cast<const float*>(h)[idx];
}

// Warp-wide argmax with the reference's tie rule (lowest index among equal
// maxima); `skip` excludes one expert (for the second choice).
template <int EPL>
__device__ __forceinline__ void warp_argmax(const float (&l)[EPL], int E, int skip, float& bv, int& bi) {
    const int lane = threadIdx.x & 31;
    bv = -INFINITY;
    bi = 0x7FFFFFFF;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        const int j = lane + 32 * e;
        if (j < E && j != skip && (bi == 0x7FFFFFFF || l[e] > bv)) { bv = l[e]; bi = j; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_down_sync(0xffffffffu, bv, off);
        const int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (oi != 0x7FFFFFFF && (bi == 0x7FFFFFFF || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
    }
    bv = __shfl_sync(0xffffffffu, bv, 0);
    bi = __shfl_sync(0xffffffffu, bi, 0);
}

// Offsets, per-path expert lists, GEMM tile prefix, meta and scheduler resets
// from per-expert counts `cnt` (global or shared); the first warp works, the
// others return. `s_off` (optional, shared) receives a copy of the offsets.
__device__ void plan_lists(const RouteArgs& a, Plan& P, const int* cnt, int* s_off) {
    const int E = a.E, lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        int run = 0, ngemv = 0, ngemm = 0, tiles = 0, mx = 0;
        for (int e0 = 0; e0 < E; e0 += 32) {
            const int e = e0 + lane;
            const int n = e < E ? cnt[e] : 0;
            int incl = n;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            const int off_e = run + incl - n;
            if (e < E) {
                P.offsets[e] = off_e;
                if (s_off) s_off[e] = off_e;
            }
            run += __shfl_sync(0xffffffffu, incl, 31);
            int m = n;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
            mx = max(mx, m);
            const int gmax = a.gemv_max > 0 ? a.gemv_max : kGemvMaxRows;
            const bool gemv = n > 0 && (a.path == 1 || (a.path == 0 && n <= gmax));
            const bool gemm = n > 0 && !gemv;
            const unsigned bg = __ballot_sync(0xffffffffu, gemv), bm = __ballot_sync(0xffffffffu, gemm);
            const unsigned lt = (1u << lane) - 1u;
            if (gemv) {
                P.gemv_list[ngemv + __popc(bg & lt)] = e;
                P.gtab[1 + ngemv + __popc(bg & lt)] = make_int4(e, n, off_e, 0);
            }
            const int nt = gemm ? (n + a.gemm_bn - 1) / a.gemm_bn : 0;
            int tincl = nt;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, tincl, off);
                if (lane >= off) tincl += y;
            }
            if (gemm) {
                const int slot = ngemm + __popc(bm & lt);
                P.gemm_list[slot] = e;
                P.gemm_tile_start[slot] = tiles + tincl - nt;
            }
            tiles += __shfl_sync(0xffffffffu, tincl, 31);
            ngemv += __popc(bg);
            ngemm += __popc(bm);
        }
        if (lane == 0) {
            P.offsets[E] = run;
            P.gemm_tile_start[ngemm] = tiles;
            P.meta[0] = ngemv;
            P.gtab[0] = make_int4(ngemv, 0, 0, 0);
            P.meta[1] = ngemm;
            P.meta[2] = tiles;
            P.meta[3] = mx;
            P.meta[5] += 1;  // forward epoch (GEMV fragment-ready flags compare against it)
            P.tickets[1] = 0;
            P.tickets[2] = 0;
            P.tickets[3] = 0;
            P.tickets[4] = 0;
            P.tickets[0] = 0;  // self-reset for the next forward
        }
    }
}

// Last-CTA planning: per-CTA bases, counts, offsets, expert lists, resets.
// `scr` (optional, >= n_ctas*E ints of smem) stages the per-CTA histograms so
// the cross-CTA scan costs one L2 round trip instead of one per expert.
__device__ void plan_tail(const RouteArgs& a, Plan P, int n_ctas, int tt, int* scr, int scr_ints) {
    const int E = a.E, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    const int RB = blockDim.x >= E ? int(blockDim.x) / E : 1;  // row blocks of the two-level scan
    // staging: [rows][E] histogram rows (as many as fit), s_cnt [E] carries, seg [RB][E]
    const int rows_fit = scr ? int((int64_t(scr_ints) - E - int64_t(RB) * E) / E) & ~3 : 0;
    const bool staged = rows_fit >= 32;
    int* s_cnt = staged ? scr + rows_fit * E : nullptr;
    if (staged) {
        int* seg = s_cnt + E;  // [RB][E]
        const int e = threadIdx.x % E, rb = threadIdx.x / E;
        for (int i = threadIdx.x; i < E; i += blockDim.x) s_cnt[i] = 0;
        // blocks of rows_fit histogram rows; each: load (16-byte loads, 8 in flight per thread),
        // two-level exclusive scan per expert carried across blocks, write back
        for (int blk0 = 0; blk0 < n_ctas; blk0 += rows_fit) {
            const int nb = min(rows_fit, n_ctas - blk0);
            const int n = nb * E;
            int32_t* gsrc = P.cta_counts + int64_t(blk0) * E;
            if ((E & 3) == 0) {
                const int n4 = n >> 2;
                const int4* src = reinterpret_cast<const int4*>(gsrc);
                int4* dst = reinterpret_cast<int4*>(scr);
                for (int i0 = threadIdx.x; i0 < n4; i0 += 8 * blockDim.x) {
                    int4 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int i = i0 + u * blockDim.x;
                        v[u] = i < n4 ? __ldcg(src + i) : make_int4(0, 0, 0, 0);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int i = i0 + u * blockDim.x;
                        if (i < n4) dst[i] = v[u];
                    }
                }
            } else {
                for (int i = threadIdx.x; i < n; i += blockDim.x) scr[i] = __ldcg(gsrc + i);
            }
            __syncthreads();
            const int per = (nb + RB - 1) / RB, r0 = rb * per, r1 = min(nb, r0 + per);
            if (rb < RB) {
                int sum = 0;
#pragma unroll 8
                for (int r = r0; r < r1; ++r) sum += scr[r * E + e];
                seg[rb * E + e] = sum;
            }
            __syncthreads();
            if (rb < RB) {
                int run = s_cnt[e];
                for (int q = 0; q < rb; ++q) run += seg[q * E + e];
#pragma unroll 8
                for (int r = r0; r < r1; ++r) {
                    const int v = scr[r * E + e];
                    scr[r * E + e] = run;
                    run += v;
                }
            }
            __syncthreads();
            if (rb == 0) {  // carry into the next block: + this block's column total
                int tot = 0;
                for (int q = 0; q < RB; ++q) tot += seg[q * E + e];
                s_cnt[e] += tot;
            }
            if ((E & 3) == 0) {
                for (int i = threadIdx.x; i < (n >> 2); i += blockDim.x)
                    reinterpret_cast<int4*>(gsrc)[i] = reinterpret_cast<const int4*>(scr)[i];
            } else {
                for (int i = threadIdx.x; i < n; i += blockDim.x) gsrc[i] = scr[i];
            }
            __syncthreads();
        }
        for (int i = threadIdx.x; i < E; i += blockDim.x) P.counts[i] = s_cnt[i];
    } else {
    // 1. exclusive scan of per-CTA counts over CTAs, per expert (warp per expert)
    for (int e = warp; e < E; e += nw) {
        int running = 0;
        for (int c0 = 0; c0 < n_ctas; c0 += 32 * 8) {
            int v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int c = c0 + u * 32 + lane;
                v[u] = c < n_ctas ? __ldcg(P.cta_counts + int64_t(c) * E + e) : 0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                int incl = v[u];
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += y;
                }
                const int c = c0 + u * 32 + lane;
                if (c < n_ctas) P.cta_counts[int64_t(c) * E + e] = running + incl - v[u];
                running += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        if (lane == 0) P.counts[e] = running;
    }
    }
    __syncthreads();
        if (a.trace && threadIdx.x == 0) a.trace[(kTraceRouteCtas - 1) * 16 + 15] = gtime_ns();
    // 2. offsets + expert lists (warp 0, expert order)
    plan_lists(a, P, staged ? s_cnt : P.counts, nullptr);
    for (int e = threadIdx.x; e < E; e += blockDim.x) P.done[e] = 0;
    __syncthreads();
    // 3. small problems: scatter routing metadata here (no extra launch)
    if (a.inline_scatter) {
        const int64_t n = a.T * a.topk;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const int64_t t = i / a.topk;
            const int e = __ldcg(P.expert + i);
            const int base = staged && n_ctas <= rows_fit ? scr[(t / tt) * E + e] : __ldcg(P.cta_counts + (t / tt) * E + e);
            const int pos = P.offsets[e] + base + __ldcg(P.lrank + i);
            P.perm_token[pos] = int32_t(t);
            P.perm_gate[pos] = __ldcg(P.gate + i);
            P.inv_pos[i] = pos;
        }
        if (a.zero_out) {
            float4* z = reinterpret_cast<float4*>(a.zero_out);
            const int64_t n4 = a.T * a.d / 4;
            for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int64_t i = n4 * 4 + threadIdx.x; i < a.T * a.d; i += blockDim.x) a.zero_out[i] = 0.f;
        }
    }
}

// Shared tail of both routing kernels: per-token argmax / gate from logits
// held by the warp (lane j <-> experts j, j+32, ...), stable local ranks, CTA
// histogram, last-CTA planning.
template <int EPL>
__device__ __forceinline__ void finish_token(const RouteArgs& a, Plan& P, const float (&acc)[EPL], int64_t t,
                                             int lt, int* s_exp) {
    const int lane = threadIdx.x & 31, E = a.E, k = a.topk;
    float b1v, b2v = 0.f;
    int b1i, b2i = 0;
    warp_argmax<EPL>(acc, E, -1, b1v, b1i);
    float g1, g2 = 0.f;
    if (k == 1) {
        // softmax in double (model.cpp:214-227); gate = prob[best] (:343)
        const double mx = double(b1v);
        double s = 0.0;
#pragma unroll
        for (int e = 0; e < EPL; ++e)
            if (lane + 32 * e < E) s += exp(double(acc[e]) - mx);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        const float eb = float(exp(double(b1v) - mx));
        g1 = float(double(eb) / s);
    } else {
        warp_argmax<EPL>(acc, E, b1i, b2v, b2i);
        const double z = exp(double(b2v) - double(b1v));
        g1 = float(1.0 / (1.0 + z));
        g2 = float(z / (1.0 + z));
    }
    if (lane == 0) {
        P.expert[t * k] = b1i;
        P.gate[t * k] = g1;
        s_exp[lt * k] = b1i;
        if (k == 2) {
            P.expert[t * k + 1] = b2i;
            P.gate[t * k + 1] = g2;
            s_exp[lt * k + 1] = b2i;
        }
    }
}

__device__ __forceinline__ void ranks_hist_plan(const RouteArgs& a, Plan& P, int* s_exp, int* s_hist, int tt,
                                                int* scr = nullptr, int scr_ints = 0,
                                                unsigned long long* tr = nullptr) {
    const int E = a.E, k = a.topk;
    __syncthreads();
    for (int i = threadIdx.x; i < tt * k; i += blockDim.x) {
        const int e = s_exp[i];
        if (e < 0) continue;
        int r = 0;
        for (int j = 0; j < i; ++j) r += s_exp[j] == e;
        P.lrank[int64_t(blockIdx.x) * tt * k + i] = r;
        atomicAdd(&s_hist[e], 1);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) P.cta_counts[int64_t(blockIdx.x) * E + e] = s_hist[e];
    __syncthreads();
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        __threadfence();  // release this CTA's routing results (ordered by the barrier)
        s_last = atomicAdd(&P.tickets[0], 1u) == gridDim.x - 1;
        if (s_last) __threadfence();  // acquire everyone else's
    }
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[11] = gtime_ns();
    if (!s_last) return;
    if (a.trace && threadIdx.x == 0) a.trace[(kTraceRouteCtas - 1) * 16 + 13] = gtime_ns();  // plan start
    plan_tail(a, P, gridDim.x, tt, scr, scr_ints);
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[12] = gtime_ns();
    if (a.trace && threadIdx.x == 0) a.trace[(kTraceRouteCtas - 1) * 16 + 14] = gtime_ns();  // plan end
}

constexpr int kRouteSmallWarps = 4;   // token warps per CTA (one token each, one per SM sub-partition)
constexpr int kRouteSlots = 8;        // Wg chunk ring (8 x 16 KB)
constexpr int kRouteChunkFloats = 4096;

// Wg rows per 16 KB chunk (a multiple of 4 so chunk byte offsets stay 16-byte aligned).
__host__ __device__ constexpr int route_chunk_rows(int E) {
    return E <= 1024 ? ((kRouteChunkFloats / E) & ~3) > 0 ? ((kRouteChunkFloats / E) & ~3) : 4 : 4;
}
__host__ __device__ inline int route_dpad(int d, int E) {
    const int r = route_chunk_rows(E);
    return (d + r - 1) / r * r;
}
size_t route_small_smem(int d, int E) {
    return size_t(kRouteSlots) * route_chunk_rows(E) * E * sizeof(float) +
           size_t(kRouteSmallWarps) * route_dpad(d, E) * sizeof(float) + 2 * kRouteSlots * sizeof(uint64_t);
}

// Small T (decode): one warp per token, lane j <-> experts j, j+32, ...
// Warp 4 streams Wg through an 8-slot smem ring with TMA bulk copies
// (mbarrier full/empty pairs, no CTA-wide barriers in the k loop); the token
// warps hold their row in smem as fp32 and run the reference's exact
// sequential fp32 chain (FMUL then FADD in ascending k, zero activations
// skipped), reading 4 activations per LDS.128 broadcast and one Wg word per
// k. EFIX > 0 compiles the expert count in (E == EFIX).
template <int EPL, int EFIX>
__global__ void __launch_bounds__((kRouteSmallWarps + 1) * 32, 1) k_route_small(RouteArgs a, Plan P) {
    constexpr int TT = kRouteSmallWarps;
    extern __shared__ __align__(128) float s_dyn[];
    __shared__ int s_exp[TT * 2];
    __shared__ int s_hist[256];
    pdl_trigger();  // the expert-FFN grid may launch and run its prologue now
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* tr = (a.trace && blockIdx.x < kTraceRouteCtas) ? a.trace + blockIdx.x * 16 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = gtime_ns();
    const int E = EFIX ? EFIX : a.E, d = a.d;
    const int rows = route_chunk_rows(E);
    const int chunk = rows * E;
    const int nch = (d + rows - 1) / rows;
    const int dpad = nch * rows;
    float* ring = s_dyn;                                   // [kRouteSlots][chunk]
    float* s_hrow = s_dyn + kRouteSlots * chunk;           // [TT][dpad]
    uint64_t* full = reinterpret_cast<uint64_t*>(s_hrow + TT * dpad);
    uint64_t* empty = full + kRouteSlots;
    const int64_t t = int64_t(blockIdx.x) * TT + (warp < TT ? warp : 0);
    const bool live = warp < TT && t < a.T;
    for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kRouteSlots; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], TT); }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == TT) {
        // ===== producer: Wg chunks -> ring (bulk copies need 16-byte aligned sources)
        if (lane == 0) {
            const bool bulk = (reinterpret_cast<uintptr_t>(a.wg) & 15) == 0;
            for (int c = 0; c < nch; ++c) {
                const int s = c % kRouteSlots;
                if (c >= kRouteSlots) mbar_wait(&empty[s], ((c / kRouteSlots) - 1) & 1);
                const int nr = min(rows, d - c * rows);
                const float* src = a.wg + int64_t(c) * chunk;
                if (bulk && ((nr * E) & 3) == 0) {
                    mbar_arrive_expect_tx(&full[s], uint32_t(nr * E * 4));
                    bulk_g2s(ring + s * chunk, src, uint32_t(nr * E * 4), &full[s]);
                } else {
                    for (int i = 0; i < nr * E; ++i) ring[s * chunk + i] = __ldg(src + i);
                    mbar_arrive(&full[s]);
                }
            }
        }
    } else {
        // ===== token warps: row -> smem (fp32, zero padded), then the exact chain
        float* hr = s_hrow + warp * dpad;
        if (live && a.h_f16 && (d % 8) == 0 && (reinterpret_cast<uintptr_t>(a.h) & 15) == 0) {
            const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __half*>(a.h) + t * d);
            for (int j = lane; j < d / 8; j += 32) {
                const uint4 v = __ldg(src + j);
                const __half2* h2 = reinterpret_cast<const __half2*>(&v);
                float4 lo, hi;
                float2 f;
                f = __half22float2(h2[0]); lo.x = f.x; lo.y = f.y;
                f = __half22float2(h2[1]); lo.z = f.x; lo.w = f.y;
                f = __half22float2(h2[2]); hi.x = f.x; hi.y = f.y;
                f = __half22float2(h2[3]); hi.z = f.x; hi.w = f.y;
                reinterpret_cast<float4*>(hr)[2 * j] = lo;
                reinterpret_cast<float4*>(hr)[2 * j + 1] = hi;
            }
            for (int p = d + lane; p < dpad; p += 32) hr[p] = 0.0f;
        } else {
            for (int p = lane; p < dpad; p += 32) hr[p] = (live && p < d) ? load_act(a.h, a.h_f16, t * d + p) : 0.0f;
        }
        __syncwarp();
        if (tr && threadIdx.x == 0) tr[1] = gtime_ns();
        float acc[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[e] = 0.0f;
        for (int c = 0; c < nch; ++c) {
            const int s = c % kRouteSlots;
            mbar_wait(&full[s], (c / kRouteSlots) & 1);
            if (live) {
                const float* wb = ring + s * chunk + lane;
                const float* hc = hr + c * rows;
                const int nr = min(rows, d - c * rows);  // rows beyond d are never read
                // software pipeline: the next 16 rows' operands load while the
                // current 16-step dependent FADD chain runs
                constexpr int U = EPL >= 4 ? 4 : 16 / EPL;
                int q = 0;
                if (nr >= U) {
                    float a_c[U], w_c[U][EPL];
                    auto fetch = [&](int q0, float (&av)[U], float (&wv)[U][EPL]) {
#pragma unroll
                        for (int u = 0; u < U; u += 4) {
                            const float4 t4 = *reinterpret_cast<const float4*>(hc + q0 + u);
                            av[u] = t4.x; av[u + 1] = t4.y; av[u + 2] = t4.z; av[u + 3] = t4.w;
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int e = 0; e < EPL; ++e)
                                wv[u][e] = (EFIX || lane + 32 * e < E) ? wb[(q0 + u) * E + 32 * e] : 0.0f;
                    };
                    fetch(0, a_c, w_c);
                    for (; q + U <= nr; q += U) {
                        float a_n[U], w_n[U][EPL];
                        if (q + 2 * U <= nr) fetch(q + U, a_n, w_n);
#pragma unroll
                        for (int u = 0; u < U; ++u) {
#pragma unroll
                            for (int e = 0; e < EPL; ++e) {
                                // reference: `if (av == 0.0f) continue; orow[j] += av * brow[j];`
                                const float pr = __fmul_rn(a_c[u], w_c[u][e]);
                                if (a_c[u] != 0.0f) acc[e] = __fadd_rn(acc[e], pr);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            a_c[u] = a_n[u];
#pragma unroll
                            for (int e = 0; e < EPL; ++e) w_c[u][e] = w_n[u][e];
                        }
                    }
                }
                for (; q < nr; ++q) {
                    const float av = hc[q];
#pragma unroll
                    for (int e = 0; e < EPL; ++e) {
                        const float w = (EFIX || lane + 32 * e < E) ? wb[q * E + 32 * e] : 0.0f;
                        const float pr = __fmul_rn(av, w);
                        if (av != 0.0f) acc[e] = __fadd_rn(acc[e], pr);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (tr && threadIdx.x == 0 && c < 8) tr[2 + c] = gtime_ns();
        }
        if (live) finish_token<EPL>(a, P, acc, t, warp, s_exp);
        else if (lane == 0) { s_exp[warp * a.topk] = -1; if (a.topk == 2) s_exp[warp * a.topk + 1] = -1; }
        if (tr && threadIdx.x == 0) tr[10] = gtime_ns();
    }
    // the Wg ring is free now: it stages the per-CTA histograms for the plan
    __syncthreads();
    ranks_hist_plan(a, P, s_exp, s_hist, TT, reinterpret_cast<int*>(ring), kRouteSlots * chunk, tr);
}

// ---- decode (T <= 32): one cluster, plan built in the leader CTA's shared memory ----
// Same per-token exact chain as k_route_small (warp = token, lane j <-> experts
// j, j+32, ...), with the operands of the next BK rows loaded ahead of the
// current BK-step dependent FADD chain (ping-pong register blocks, clamped
// addresses so the loads are unconditional). Each token's choice and gate go
// straight into cluster rank 0's shared memory (DSMEM); after one cluster
// barrier rank 0 builds counts, offsets, lists and the permutation from shared
// memory — no tickets, no global round trips before the plan is written.
constexpr int kRouteDecMaxCtas = 8;
constexpr int kRouteDecMaxT = kRouteDecMaxCtas * kRouteSmallWarps;
constexpr int kRouteDecMaxE = 256;

template <int BK, int EPL, int EFIX>
__device__ __forceinline__ void chain_load(const float* hc, const float* wb, int q0, int E, int lane,
                                           float (&x)[BK], float (&w)[BK][EPL]) {
#pragma unroll
    for (int u = 0; u < BK; u += 4) {
        const float4 t4 = *reinterpret_cast<const float4*>(hc + q0 + u);
        x[u] = t4.x; x[u + 1] = t4.y; x[u + 2] = t4.z; x[u + 3] = t4.w;
    }
#pragma unroll
    for (int u = 0; u < BK; ++u)
#pragma unroll
        for (int e = 0; e < EPL; ++e) w[u][e] = (EFIX || lane + 32 * e < E) ? wb[(q0 + u) * E + 32 * e] : 0.0f;
}
template <int BK, int EPL>
__device__ __forceinline__ void chain_run(float (&acc)[EPL], const float (&x)[BK], const float (&w)[BK][EPL]) {
#pragma unroll
    for (int u = 0; u < BK; ++u)
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
            // reference: `if (av == 0.0f) continue; orow[j] += av * brow[j];` — the skip is
            // folded into the addend (+0 leaves a round-to-nearest sum that started at +0
            // unchanged, and 0 * inf never forms), so the dependent FADD chain carries no
            // predicate from the ALU pipe: bit-identical, shorter critical path
            const float pr = x[u] != 0.0f ? __fmul_rn(x[u], w[u][e]) : 0.0f;
            acc[e] = __fadd_rn(acc[e], pr);
        }
}

// TT tokens (warps) per CTA: 4 with the in-cluster plan; 1 in no_plan mode, where
// the CTAs are independent — one token warp per SM keeps the chain off the shared-
// memory wavefront limit (~1.25 wavefronts per step per warp, ~1 per cycle per SM).
template <int EPL, int EFIX, int TT>
__global__ void __launch_bounds__((TT + 1) * 32, 1) k_route_decode(RouteArgs a, Plan P) {
    constexpr int BK = EPL <= 2 ? 16 : EPL <= 4 ? 8 : 4;  // rows per pipelined block
    extern __shared__ __align__(128) float s_dyn[];
    __shared__ int s_exp[kRouteDecMaxT * 2];
    __shared__ float s_gate[kRouteDecMaxT * 2];
    __shared__ int s_cnt[kRouteDecMaxE];
    __shared__ int s_off[kRouteDecMaxE];
    pdl_trigger();  // the expert-FFN grid may launch and run its prologue now
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = int(cta_rank());
    unsigned long long* tr = (a.trace && blockIdx.x < kTraceRouteCtas) ? a.trace + blockIdx.x * 16 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = gtime_ns();
    const int E = EFIX ? EFIX : a.E, d = a.d, k = a.topk;
    const int rows = route_chunk_rows(E);
    const int chunk = rows * E;
    const int nch = (d + rows - 1) / rows;
    const int dpad = nch * rows;
    float* ring = s_dyn;
    float* s_hrow = s_dyn + kRouteSlots * chunk;
    uint64_t* full = reinterpret_cast<uint64_t*>(s_hrow + TT * dpad);
    uint64_t* empty = full + kRouteSlots;
    const int64_t t = int64_t(blockIdx.x) * TT + (warp < TT ? warp : 0);
    const bool live = warp < TT && t < a.T;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kRouteSlots; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], TT); }
        fence_barrier_init();
    }
    __syncthreads();
    const bool plan = !a.no_plan;  // uniform: with no_plan the CTAs never touch each other
    if (plan) cluster_arrive_release();  // rank 0 has started before anyone writes its shared memory (wait below)

    if (warp == TT) {
        if (lane == 0) {
            const bool bulk = (reinterpret_cast<uintptr_t>(a.wg) & 15) == 0;
            for (int c = 0; c < nch; ++c) {
                const int s = c % kRouteSlots;
                if (c >= kRouteSlots) mbar_wait(&empty[s], ((c / kRouteSlots) - 1) & 1);
                const int nr = min(rows, d - c * rows);
                const float* src = a.wg + int64_t(c) * chunk;
                if (bulk && ((nr * E) & 3) == 0) {
                    mbar_arrive_expect_tx(&full[s], uint32_t(nr * E * 4));
                    bulk_g2s(ring + s * chunk, src, uint32_t(nr * E * 4), &full[s]);
                } else {
                    for (int i = 0; i < nr * E; ++i) ring[s * chunk + i] = __ldg(src + i);
                    mbar_arrive(&full[s]);
                }
            }
        }
        __syncwarp();
        if (plan) cluster_wait_acquire();
    } else {
        float* hr = s_hrow + warp * dpad;
        if (live && a.h_f16 && (d % 8) == 0 && (reinterpret_cast<uintptr_t>(a.h) & 15) == 0) {
            const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __half*>(a.h) + t * d);
            for (int j = lane; j < d / 8; j += 32) {
                const uint4 v = __ldg(src + j);
                const __half2* h2 = reinterpret_cast<const __half2*>(&v);
                float4 lo, hi;
                float2 f;
                f = __half22float2(h2[0]); lo.x = f.x; lo.y = f.y;
                f = __half22float2(h2[1]); lo.z = f.x; lo.w = f.y;
                f = __half22float2(h2[2]); hi.x = f.x; hi.y = f.y;
                f = __half22float2(h2[3]); hi.z = f.x; hi.w = f.y;
                reinterpret_cast<float4*>(hr)[2 * j] = lo;
                reinterpret_cast<float4*>(hr)[2 * j + 1] = hi;
            }
            for (int p = d + lane; p < dpad; p += 32) hr[p] = 0.0f;
        } else {
            for (int p = lane; p < dpad; p += 32) hr[p] = (live && p < d) ? load_act(a.h, a.h_f16, t * d + p) : 0.0f;
        }
        if (live && a.inline_scatter && a.zero_out)  // top-2: fp32 accumulation rows start at zero
            for (int j = lane; j < d; j += 32) a.zero_out[t * d + j] = 0.f;
        __syncwarp();
        if (tr && threadIdx.x == 0) tr[1] = gtime_ns();
        const long long clk0 = clock64();
        float acc[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[e] = 0.0f;
        for (int c = 0; c < nch; ++c) {
            const int s = c % kRouteSlots;
            mbar_wait(&full[s], (c / kRouteSlots) & 1);
            if (live && a.dbg != 1) {
                const float* wb = ring + s * chunk + lane;
                const float* hc = hr + c * rows;
                const int nr = min(rows, d - c * rows);
                int q = 0;
                if (nr >= 2 * BK) {
                    const int qlast = (nr - BK) & ~3;  // clamp target: in range and 16-byte aligned
                    float xa[BK], wa[BK][EPL], xb[BK], wbk[BK][EPL];
                    chain_load<BK, EPL, EFIX>(hc, wb, 0, E, lane, xa, wa);
                    for (; q + 2 * BK <= nr; q += 2 * BK) {
                        chain_load<BK, EPL, EFIX>(hc, wb, q + BK, E, lane, xb, wbk);
                        chain_run<BK, EPL>(acc, xa, wa);
                        chain_load<BK, EPL, EFIX>(hc, wb, min(q + 2 * BK, qlast), E, lane, xa, wa);
                        chain_run<BK, EPL>(acc, xb, wbk);
                    }
                }
                for (; q < nr; ++q) {
                    const float av = hc[q];
#pragma unroll
                    for (int e = 0; e < EPL; ++e) {
                        const float w = (EFIX || lane + 32 * e < E) ? wb[q * E + 32 * e] : 0.0f;
                        const float pr = __fmul_rn(av, w);
                        if (av != 0.0f) acc[e] = __fadd_rn(acc[e], pr);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (tr && threadIdx.x == 0 && c < 8) tr[2 + c] = gtime_ns();
        }
        // argmax / gate (reference tie rule, fp64 softmax) -> rank 0's shared memory
        float b1v = 0.f, b2v = 0.f, g1 = 0.f, g2 = 0.f;
        int b1i = 0, b2i = 0;
        if (live) {
            warp_argmax<EPL>(acc, E, -1, b1v, b1i);
            if (k == 1) {
                const double mx = double(b1v);
                double sm = 0.0;
#pragma unroll
                for (int e = 0; e < EPL; ++e)
                    if (lane + 32 * e < E) sm += exp(double(acc[e]) - mx);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, off);
                const float eb = float(exp(double(b1v) - mx));
                g1 = float(double(eb) / sm);
            } else {
                warp_argmax<EPL>(acc, E, b1i, b2v, b2i);
                const double z = exp(double(b2v) - double(b1v));
                g1 = float(1.0 / (1.0 + z));
                g2 = float(z / (1.0 + z));
            }
        }
        if (tr && threadIdx.x == 0) { tr[10] = gtime_ns(); tr[13] = clock64() - clk0; }
        if (!plan) {  // the GEMV kernels build the plan themselves: expert / gate only
            if (live && lane == 0) {
                P.expert[t * k] = b1i;
                P.gate[t * k] = g1;
                if (k == 2) {
                    P.expert[t * k + 1] = b2i;
                    P.gate[t * k + 1] = g2;
                }
            }
        } else {
        cluster_wait_acquire();  // rank 0 is running
        if (live && lane == 0) {
            st_cluster_u32(map_rank(&s_exp[t * k], 0), uint32_t(b1i));
            st_cluster_u32(map_rank(&s_gate[t * k], 0), __float_as_uint(g1));
            if (k == 2) {
                st_cluster_u32(map_rank(&s_exp[t * k + 1], 0), uint32_t(b2i));
                st_cluster_u32(map_rank(&s_gate[t * k + 1], 0), __float_as_uint(g2));
            }
        }
        }
    }
    if (!plan) {
        // launched behind k_xrows (PDL): the grid completes only after it (see below)
        if (blockIdx.x == 0 && threadIdx.x == 0) pdl_wait();
        return;
    }
    cluster_arrive_release();
    cluster_wait_acquire();  // every token's choice is in rank 0's shared memory
    if (tr && threadIdx.x == 0) tr[11] = gtime_ns();
    if (rank != 0) return;

    // ===== rank 0: the whole plan from shared memory
    const int n = int(a.T) * k;
    const int nct = int((a.T + TT - 1) / TT);
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        int c = 0;
        for (int i = 0; i < n; ++i) c += s_exp[i] == e;
        s_cnt[e] = c;
        P.counts[e] = c;
        P.done[e] = 0;
    }
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[13] = gtime_ns();
    plan_lists(a, P, s_cnt, s_off);
    if (threadIdx.x == 0) P.tickets[0] = 0;
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[14] = gtime_ns();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int e = s_exp[i];
        const int c0 = (i / k) / TT * TT * k;  // first (token, slot) of this row's route group
        int r = 0, base = 0;
        for (int j = 0; j < i; ++j)
            if (s_exp[j] == e) { ++r; base += j < c0; }
        const int pos = s_off[e] + r;
        const float gt = s_gate[i];
        P.expert[i] = e;
        P.gate[i] = gt;
        P.lrank[i] = r - base;
        if (a.inline_scatter) {
            P.perm_token[pos] = i / k;
            P.perm_gate[pos] = gt;
            P.inv_pos[i] = pos;
        }
    }
    if (tr && threadIdx.x == 0) tr[15] = gtime_ns();
    for (int idx = threadIdx.x; idx < nct * E; idx += blockDim.x) {  // route-group bases (k_scatter)
        const int c = idx / E, e = idx - c * E, lim = min(c * TT * k, n);
        int b = 0;
        for (int j = 0; j < lim; ++j) b += s_exp[j] == e;
        P.cta_counts[idx] = b;
    }
    if (tr) {
        __syncthreads();
        if (threadIdx.x == 0) tr[12] = gtime_ns();
    }
    // launched behind k_xrows (PDL): finish only after it, so the expert-FFN grid's
    // own dependency wait on this grid covers the row blocks too
    if (threadIdx.x == 0) pdl_wait();
}

// ---- decode without a plan (the GEMV grid builds it): one chain warp, blocked Wg -------
// The bank keeps a second copy of the router weights, transposed and blocked (built once by
// route_block_wg): chunks [chunk][expert][rows + 4] (rc_rows; a 16-byte pad per expert row, so
// eight lanes' LDS.128 cover all 32 banks). One token per CTA. The chain warp (lane j <->
// experts j, j + 32, ...) reads four consecutive k of its expert per LDS.128 and four
// activations per broadcast LDS.128, and runs the reference's sequential fp32 chain (FMUL,
// then FADD, ascending k; model.cpp matmul) — ~2.5 instructions per k instead of a strided
// load per k. With an all-finite Wg (checked at bank creation) the zero-activation skip
// needs no select: 0 * w is +-0, and adding +-0 leaves the sum unchanged (it starts at +0
// and round-to-nearest never yields -0 from a nonzero sum); otherwise x != 0 selects. A TMA
// warp streams the chunks through a ring. kRCTok tokens per CTA, one chain warp each (one per
// SM sub-partition), sharing the ring: fewer router SMs means fewer expert-FFN CTAs launching
// late behind it, but with the one-chunk layout 1 token per CTA measured best (32.6 us per
// layer vs 33.0 with 2 and 33.8 with 4).
constexpr int kRCTok = 1;
static_assert(kRCTok <= 4, "row index math below covers up to 4 tokens");
// Chunking (measured: every chunk boundary restarts the register pipeline and costs the
// chain more than the copy latency it hides): the whole Wg as ONE chunk when it fits
// ~136 KB (E = 32, d = 1024: 128 KB), else ~64 KB chunks through two slots.
constexpr int kRCOneChunk = 136 * 1024;
__host__ __device__ constexpr int rc_ps(int rows);
__host__ __device__ inline int rc_rows(int d, int E) {
    const int whole = (d + 31) / 32 * 32;  // a multiple of 32: full chunks take the fast path
    if (int64_t(E) * (whole + 4) * 4 <= kRCOneChunk) return whole;
    return 4 * route_chunk_rows(E);
}
__host__ __device__ inline int rc_slots(int d, int E) { return rc_rows(d, E) >= d ? 1 : 2; }
constexpr int kRCSlotsMax = 2;
constexpr int kRCPad = 64;  // floats after the token row: the chain's look-ahead loads past a chunk stay in bounds
__host__ __device__ constexpr int rc_ps(int rows) { return rows + 4; }
size_t route_chain_smem(int d, int E) {
    const int rows = rc_rows(d, E);
    return size_t(rc_slots(d, E)) * E * rc_ps(rows) * 4 + size_t(kRCTok) * ((d + rows - 1) / rows * rows + kRCPad) * 4 +
           size_t(2 * kRCSlotsMax) * 8;
}

// fc1 row blocks of a router CTA's tokens from their rows in smem (the decode router's
// copy warp; out of line so the chain warp's code and registers are unaffected).
// The fields it needs come by value: taking the kernel parameter's address would force a
// local-memory copy of RouteArgs into every thread.
__device__ __noinline__ void route_xrows(int d, int h_f16, int nch1, int xr_bits, uint8_t* xr, const float* hrow, int hs,
                                         int ntok, int64_t t0, int lane) {
    for (int r = 0; r < ntok; ++r) {
        const float* hr = hrow + r * hs;
        auto q16 = [&](float x) { return h_f16 ? x : __half2float(__float2half_rn(x)); };
        float m = 0.f, l1 = 0.f;
        for (int kk = lane; kk < d; kk += 32) {
            const float x = fabsf(q16(hr[kk]));
            m = fmaxf(m, x);
            l1 += x;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
            l1 += __shfl_xor_sync(0xffffffffu, l1, off);
        }
        const int st = lane >> 2, tq = lane & 3;
        for (int c = 0; c < nch1; ++c) {
            float v[32];
            const int k0 = c * kChunkK + st * kStageK + 16 * tq;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                v[i] = k0 + i < d ? q16(hr[k0 + i]) : 0.f;
                v[16 + i] = k0 + 64 + i < d ? q16(hr[k0 + 64 + i]) : 0.f;
            }
            const int64_t row = (t0 + r) * nch1 + c;
            switch (xr_bits) {
                case 2: xrow_encode<2>(v, m, l1, xr + row * RB<2>::XR1, lane); break;
                case 3: xrow_encode<3>(v, m, l1, xr + row * RB<3>::XR1, lane); break;
                case 4: xrow_encode<4>(v, m, l1, xr + row * RB<4>::XR1, lane); break;
                default: xrow_encode<8>(v, m, l1, xr + row * RB<8>::XR1, lane); break;
            }
        }
    }
}

// thread 0..kSelfPlanRows-1 zero the GEMV readiness counters below
static_assert((kRCTok + 1) * 32 >= kSelfPlanRows, "k_route_chain blocks must cover the readiness counters");
template <int EPL, int EFIX, bool SEL>
__global__ void __launch_bounds__((kRCTok + 1) * 32, 1) k_route_chain(RouteArgs a, Plan P) {
    extern __shared__ __align__(128) float s_dyn[];
    if (a.first) pdl_wait();  // leads the decode chain: the previous grid made the token rows
    pdl_trigger();            // the expert-FFN grid may launch and run its prologue now
    if (a.first && a.ready && blockIdx.x == 0 && threadIdx.x < kSelfPlanRows) a.ready[threadIdx.x] = 0u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long* tr = (a.trace && blockIdx.x < kTraceRouteCtas && (a.dbg != 9 || blockIdx.x == 0))
                                 ? a.trace + blockIdx.x * 16 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = gtime_ns();
    const int E = EFIX ? EFIX : a.E, d = a.d, k = a.topk;
    const int rows = rc_rows(d, E), PS = rc_ps(rows), cf = E * PS;  // floats per chunk
    const int nslot = rc_slots(d, E), sh = nslot - 1;                 // 1 or 2 slots: c >> sh = use count
    const int nch = (d + rows - 1) / rows, dpad = nch * rows;
    const int hs = dpad + kRCPad;         // floats per token row
    float* ring = s_dyn;                  // [nslot][E][PS]
    float* hrow = ring + nslot * cf;      // [kRCTok][hs] the token rows in fp32 (zero padded)
    uint64_t* full = reinterpret_cast<uint64_t*>(hrow + kRCTok * hs);
    uint64_t* empty = full + kRCSlotsMax;
    const int64_t t0 = int64_t(blockIdx.x) * kRCTok;
    const int ntok = int(min(int64_t(kRCTok), a.T - t0));
    constexpr int kTma = kRCTok;  // the TMA warp
    // dbg 9: per-chunk clock64 stamps of CTA 0 in the trace slots of CTAs 1.. (diagnostics)
    unsigned long long* ds = a.dbg == 9 && a.trace && blockIdx.x == 0 ? a.trace + 16 : nullptr;
    auto dstamp = [&](int c, int ev) { if (ds && c < 8) ds[c * 6 + ev] = clock64(); };
    if (ds && threadIdx.x == 0) ds[60] = clock64();
    auto issue = [&](int c) {  // chunk c -> slot c & sh
        const int s = c & sh;
        dstamp(c, 0);
        mbar_arrive_expect_tx(&full[s], uint32_t(cf * 4));
        bulk_g2s(ring + s * cf, a.wg_blk + int64_t(c) * cf, uint32_t(cf * 4), &full[s]);
    };
    if (warp == kTma && lane == 0) {  // barriers, then the first chunks while the rows load
        for (int s = 0; s < nslot; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kRCTok); }
        fence_barrier_init();
        for (int c = 0; c < min(nch, nslot); ++c) issue(c);
    }
    {  // token rows -> fp32 (every warp)
        const int tid = threadIdx.x, nthr = (kRCTok + 1) * 32;
        if (a.h_f16 && (d % 8) == 0 && (reinterpret_cast<uintptr_t>(a.h) & 15) == 0) {
            const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __half*>(a.h) + t0 * d);
            const int d8 = d / 8;
            for (int jj = tid; jj < ntok * d8; jj += nthr) {
                const int r = jj >= d8 ? (jj >= 2 * d8 ? (jj >= 3 * d8 ? 3 : 2) : 1) : 0, j = jj - r * d8;
                float* hr = hrow + r * hs;
                const uint4 v = __ldg(src + jj);
                const __half2* h2 = reinterpret_cast<const __half2*>(&v);
                float4 lo, hi;
                float2 f;
                f = __half22float2(h2[0]); lo.x = f.x; lo.y = f.y;
                f = __half22float2(h2[1]); lo.z = f.x; lo.w = f.y;
                f = __half22float2(h2[2]); hi.x = f.x; hi.y = f.y;
                f = __half22float2(h2[3]); hi.z = f.x; hi.w = f.y;
                reinterpret_cast<float4*>(hr)[2 * j] = lo;
                reinterpret_cast<float4*>(hr)[2 * j + 1] = hi;
            }
            for (int r = 0; r < kRCTok; ++r)  // padding (and the rows of absent tokens)
                for (int p = (r < ntok ? d : 0) + tid; p < hs; p += nthr) hrow[r * hs + p] = 0.0f;
        } else {
            for (int pp = tid; pp < kRCTok * hs; pp += nthr) {
                const int r = pp / hs, p = pp - r * hs;
                hrow[pp] = (p < d && r < ntok) ? load_act(a.h, a.h_f16, (t0 + r) * d + p) : 0.0f;
            }
        }
        if (a.inline_scatter && a.zero_out)  // top-2: fp32 accumulation rows start at zero
            for (int j = tid; j < ntok * d; j += nthr) a.zero_out[t0 * d + j] = 0.f;
    }
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[1] = gtime_ns();

    if (warp == kTma) {
        if (lane == 0)
            for (int c = nslot; c < nch; ++c) {
                while (!mbar_try_wait_sleep(&empty[c & sh], ((c >> sh) - 1) & 1)) {
                }
                issue(c);
            }
        __syncwarp();
        // this warp is otherwise idle during the chain: the tokens' fc1 row blocks from the
        // rows in smem (fp16-valued, as k_xrows reads them; same exponent, digits and planes)
        if (a.xr) route_xrows(a.d, a.h_f16, a.nch1, a.xr_bits, a.xr, hrow, hs, ntok, t0, lane);
    } else {
        // ===== chain warp: token t0 + warp
        const int64_t t = t0 + warp;
        const bool live = warp < ntok;
        const float* hr = hrow + warp * hs;
        const long long clk0 = clock64();
        float acc[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[e] = 0.0f;
        constexpr int V = EPL == 1 ? 4 : EPL <= 4 ? 2 : 1;  // 4-k groups per register block
        int col[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) col[e] = (EFIX || lane + 32 * e < E) ? lane + 32 * e : 0;
        auto mul = [](float x, float w) { return SEL ? (x != 0.0f ? __fmul_rn(x, w) : 0.0f) : __fmul_rn(x, w); };
        for (int c = 0; c < nch; ++c) {
            const int s = c & sh;
            mbar_wait(&full[s], (c >> sh) & 1);
            if (threadIdx.x == 0) dstamp(c, 3);
            const float* wc = ring + s * cf;
            const float* hc = hr + c * rows;
            const int ng = (min(rows, d - c * rows) + 3) / 4;
            if (live && a.dbg != 1 && ng == rows / 4 && ng % (2 * V) == 0) {
                // full chunk: ping-pong register blocks, the next block's loads in flight during
                // this block's dependent FADDs; no clamps or guards (immediate-offset loads; the
                // look-ahead past the chunk reads padding or the next slot, never used)
                const float* wp[EPL];
#pragma unroll
                for (int e = 0; e < EPL; ++e) wp[e] = wc + col[e] * PS;
                float4 xa[V], xb[V], wa[V][EPL], wb[V][EPL];
                auto ld = [&](float4 (&x)[V], float4 (&w)[V][EPL], int g0) {
#pragma unroll
                    for (int i = 0; i < V; ++i) {
                        x[i] = *reinterpret_cast<const float4*>(hc + 4 * (g0 + i));
#pragma unroll
                        for (int e = 0; e < EPL; ++e) w[i][e] = *reinterpret_cast<const float4*>(wp[e] + 4 * (g0 + i));
                    }
                };
                auto run = [&](const float4 (&x)[V], const float4 (&w)[V][EPL]) {
#pragma unroll
                    for (int i = 0; i < V; ++i)
#pragma unroll
                        for (int e = 0; e < EPL; ++e) {
                            float v = __fadd_rn(acc[e], mul(x[i].x, w[i][e].x));
                            v = __fadd_rn(v, mul(x[i].y, w[i][e].y));
                            v = __fadd_rn(v, mul(x[i].z, w[i][e].z));
                            acc[e] = __fadd_rn(v, mul(x[i].w, w[i][e].w));
                        }
                };
                ld(xa, wa, 0);
#pragma unroll 1
                for (int g = 0; g < ng; g += 2 * V) {
                    ld(xb, wb, g + V);
                    run(xa, wa);
                    ld(xa, wa, g + 2 * V);
                    run(xb, wb);
                }
            } else if (live && a.dbg != 1) {
                // partial chunk: the same with clamped addresses and guarded adds
                float4 xa[V], xb[V], wa[V][EPL], wb[V][EPL];
                auto ld = [&](float4 (&x)[V], float4 (&w)[V][EPL], int g0) {
#pragma unroll
                    for (int i = 0; i < V; ++i) {
                        const int g = min(g0 + i, ng - 1);
                        x[i] = *reinterpret_cast<const float4*>(hc + 4 * g);
#pragma unroll
                        for (int e = 0; e < EPL; ++e) w[i][e] = *reinterpret_cast<const float4*>(wc + col[e] * PS + 4 * g);
                    }
                };
                auto run = [&](const float4 (&x)[V], const float4 (&w)[V][EPL], int g0) {
#pragma unroll
                    for (int i = 0; i < V; ++i)
                        if (g0 + i < ng)
#pragma unroll
                            for (int e = 0; e < EPL; ++e) {
                                float v = __fadd_rn(acc[e], mul(x[i].x, w[i][e].x));
                                v = __fadd_rn(v, mul(x[i].y, w[i][e].y));
                                v = __fadd_rn(v, mul(x[i].z, w[i][e].z));
                                acc[e] = __fadd_rn(v, mul(x[i].w, w[i][e].w));
                            }
                };
                ld(xa, wa, 0);
                for (int g = 0; g < ng; g += 2 * V) {
                    ld(xb, wb, g + V);
                    run(xa, wa, g);
                    ld(xa, wa, g + 2 * V);
                    run(xb, wb, g + V);
                }
            }
            __syncwarp();
            if (lane == 0) {
                if (warp == 0) dstamp(c, 4);
                mbar_arrive(&empty[s]);
            }
            if (tr && threadIdx.x == 0 && c < 8) tr[2 + c] = gtime_ns();
        }
        // argmax / gate (reference tie rule, fp64 softmax)
        float b1v = 0.f, b2v = 0.f, g1 = 0.f, g2 = 0.f;
        int b1i = 0, b2i = 0;
        warp_argmax<EPL>(acc, E, -1, b1v, b1i);
        if (k == 1) {
            const double mx = double(b1v);
            double sm = 0.0;
#pragma unroll
            for (int e = 0; e < EPL; ++e)
                if (lane + 32 * e < E) sm += exp(double(acc[e]) - mx);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, off);
            const float eb = float(exp(double(b1v) - mx));
            g1 = float(double(eb) / sm);
        } else {
            warp_argmax<EPL>(acc, E, b1i, b2v, b2i);
            const double z = exp(double(b2v) - double(b1v));
            g1 = float(1.0 / (1.0 + z));
            g2 = float(z / (1.0 + z));
        }
        if (tr && threadIdx.x == 0) { tr[10] = gtime_ns(); tr[13] = clock64() - clk0; }
        if (live && lane == 0) {  // the GEMV grid builds the plan from these
            P.expert[t * k] = b1i;
            P.gate[t * k] = g1;
            if (k == 2) {
                P.expert[t * k + 1] = b2i;
                P.gate[t * k + 1] = g2;
            }
        }
    }
    // launched behind k_xrows (PDL): the grid completes only after it, so the expert-FFN
    // grid's own dependency wait on this grid covers the row blocks too
    if (!a.first && blockIdx.x == 0 && threadIdx.x == 0) pdl_wait();
}

// Router weights [d][E] -> the blocked, transposed copy k_route_chain streams; flags any
// non-finite weight (then the chain keeps the explicit zero-activation select).
__global__ void k_wg_block(const float* __restrict__ wg, int d, int E, float* __restrict__ out, int* nonfinite) {
    const int rows = rc_rows(d, E), PS = rc_ps(rows);
    const int nch = (d + rows - 1) / rows;
    const int64_t n = int64_t(nch) * E * PS;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int r = int(i % PS);
        const int64_t ce = i / PS;
        const int e = int(ce % E), c = int(ce / E);
        const int kk = c * rows + r;
        const float v = (r < rows && kk < d) ? wg[int64_t(kk) * E + e] : 0.0f;
        if (!isfinite(v)) atomicOr(nonfinite, 1);
        out[i] = v;
    }
}
int64_t route_wg_block_floats(int d, int E) {
    const int rows = rc_rows(d, E);
    return int64_t((d + rows - 1) / rows) * E * rc_ps(rows);
}
cudaError_t route_block_wg(const float* wg, int d, int E, float* out, int* d_flag, int* finite) {
    cudaError_t e = cudaMemset(d_flag, 0, sizeof(int));
    if (e != cudaSuccess) return e;
    const int64_t n = route_wg_block_floats(d, E);
    k_wg_block<<<unsigned(std::min<int64_t>((n + 255) / 256, 4096)), 256>>>(wg, d, E, out, d_flag);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    int h = 0;
    if ((e = cudaMemcpy(&h, d_flag, sizeof(int), cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
    *finite = h == 0;
    return cudaSuccess;
}

// ---- large T, E in {32, 64}, fp16 rows with d % 8 == 0 (the prefill shapes) ----------
// CTA = 32 tokens x all E experts; 8 compute warps, warp w owns experts
// [w*EPL, (w+1)*EPL) (EPL = E/8) for the 32 tokens of its lanes, so each lane runs
// EPL independent exact chains (FMUL then FADD, ascending k, zero activations
// skipped) and the FADD latency is covered without CTA-wide barriers. A producer
// warp stages the 32 token rows once (TMA, padded rows: conflict-free LDS.128) and
// streams Wg through an mbarrier ring in 128-row chunks.
constexpr int kRL2Warps = 8, kRL2Rows = 128;
__host__ __device__ constexpr int rl2_hstride(int d) { return d * 2 + 16; }
__host__ __device__ constexpr int rl2_slots(int E) { return E <= 32 ? 6 : 4; }
size_t rl2_smem(int d, int E) {
    return size_t((32 * rl2_hstride(d) + 127) / 128 * 128) + size_t(rl2_slots(E)) * kRL2Rows * E * 4 + 256 +
           size_t(32) * (E + 1) * 4;
}

template <int EPL>
__global__ void __launch_bounds__((kRL2Warps + 1) * 32, 1) k_route_logits2(RouteArgs a, Plan P) {
    constexpr int E = 8 * EPL, NS = rl2_slots(8 * EPL);
    extern __shared__ __align__(128) uint8_t sm[];
    const int d = a.d, hs = rl2_hstride(d);
    float* ring = reinterpret_cast<float*>(sm + (32 * hs + 127) / 128 * 128);
    uint64_t* hbar = reinterpret_cast<uint64_t*>(ring + NS * kRL2Rows * E);
    uint64_t* full = hbar + 1;
    uint64_t* empty = full + NS;
    float* s_l = reinterpret_cast<float*>(empty + NS);  // [32 tokens][E + 1] logits of this CTA
    __shared__ int s_exp[64];
    __shared__ int s_hist[256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t0 = int64_t(blockIdx.x) * 32;
    for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;
    const int ntok = a.T - t0 < 32 ? int(a.T - t0) : 32;
    const int nch = (d + kRL2Rows - 1) / kRL2Rows;
    if (threadIdx.x == 0) {
        mbar_init(hbar, 1);
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kRL2Warps); }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == kRL2Warps) {
        if (lane == 0) {
            const __half* h = static_cast<const __half*>(a.h);
            mbar_arrive_expect_tx(hbar, uint32_t(ntok * d * 2));
            for (int r = 0; r < ntok; ++r) bulk_g2s(sm + r * hs, h + (t0 + r) * d, uint32_t(d * 2), hbar);
            for (int c = 0; c < nch; ++c) {
                const int s = c % NS;
                if (c >= NS) mbar_wait(&empty[s], ((c / NS) - 1) & 1);
                const int nr = min(kRL2Rows, d - c * kRL2Rows);
                mbar_arrive_expect_tx(&full[s], uint32_t(nr * E * 4));
                bulk_g2s(ring + s * kRL2Rows * E, a.wg + int64_t(c) * kRL2Rows * E, uint32_t(nr * E * 4), &full[s]);
            }
        }
        __syncwarp();
    } else {
    const bool live = lane < ntok;
    const uint8_t* hr = sm + lane * hs;
    float acc[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[e] = 0.0f;
    mbar_wait(hbar, 0);
    for (int c = 0; c < nch; ++c) {
        const int s = c % NS;
        mbar_wait(&full[s], (c / NS) & 1);
        const float* wc = ring + s * kRL2Rows * E + warp * EPL;
        const int nr = min(kRL2Rows, d - c * kRL2Rows);  // a multiple of 8
        const uint8_t* hc = hr + c * kRL2Rows * 2;
#pragma unroll 2
        for (int q = 0; q < nr; q += 8) {
            const uint4 hv = *reinterpret_cast<const uint4*>(hc + q * 2);
            const __half2* h2 = reinterpret_cast<const __half2*>(&hv);
            float x[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = __half22float2(h2[i]);
                x[2 * i] = f.x;
                x[2 * i + 1] = f.y;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                float w[EPL];
#pragma unroll
                for (int e = 0; e < EPL; e += 4) {
                    const float4 v = *reinterpret_cast<const float4*>(wc + (q + u) * E + e);
                    w[e] = v.x; w[e + 1] = v.y; w[e + 2] = v.z; w[e + 3] = v.w;
                }
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    // reference: `if (av == 0.0f) continue; orow[j] += av * brow[j];`
                    const float pr = __fmul_rn(x[u], w[e]);
                    if (x[u] != 0.0f) acc[e] = __fadd_rn(acc[e], pr);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
#pragma unroll
    for (int e = 0; e < EPL; ++e) s_l[lane * (E + 1) + warp * EPL + e] = acc[e];
    named_bar_sync(1, kRL2Warps * 32);  // all 32 x E logits of the CTA in smem
    // selection: warp w finishes tokens 4w .. 4w+3 (lane j <-> experts j, j + 32)
    for (int lt = 4 * warp; lt < 4 * warp + 4; ++lt) {
        if (lt < ntok) {
            float l[E / 32];
#pragma unroll
            for (int e = 0; e < E / 32; ++e) l[e] = s_l[lt * (E + 1) + lane + 32 * e];
            finish_token<E / 32>(a, P, l, t0 + lt, lt, s_exp);
        } else if (lane == 0) {
            s_exp[lt * a.topk] = -1;
            if (a.topk == 2) s_exp[lt * a.topk + 1] = -1;
        }
    }
    }
    // ranks, CTA histogram, last-CTA plan (every thread of the CTA takes part;
    // the drained Wg ring stages the per-CTA histograms)
    ranks_hist_plan(a, P, s_exp, s_hist, 32, reinterpret_cast<int*>(ring), NS * kRL2Rows * E);
}

// ---- large T, tensor-core logits (E in {32, 64}, finite Wg, fp16 rows) -----------------
// The exact-order chains above cost one FMUL + one FADD per MAC (~130 us at T = 16384).
// north_star lets tokens whose top-2 logit gap is < 1e-4 route differently, so the prefill
// logits run on the tensor cores instead: the bank's split copy Wg * 2^s = hi + lo (fp16,
// ~22 significant bits; see dec_split_wg) is the B operand, the fp16 token rows the A operand,
// fp32 accumulation in a fixed per-CTA order (deterministic, |error| ~1e-7 relative). CTA =
// 32 tokens (two 16-row A tiles) x all E experts, 8 MMA warps: warp w owns A tile w & 1 and the
// 8-expert B tiles w >> 1 (+4 for E = 64), over the whole K. A producer warp stages the token
// rows (zero-padded to Kp1) and streams the four Wg chunks through one slot (~100 KB of smem:
// two CTAs per SM, so one CTA's loads overlap the other's MMAs). Selection,
// ranks and the last-CTA plan are the shared tail (finish_token, ranks_hist_plan).
constexpr int kRMWarps = 8, kRMSlots = 1;  // one Wg slot: two CTAs per SM overlap each other's loads
__host__ __device__ inline int rm_hpitch(int Kp1) { return Kp1 * 2 + 16; }  // 16 mod 128: conflict-free
__host__ __device__ inline uint32_t rm_chunk_bytes(int E, int Kp1) {
    return uint32_t(2 * ((E + 7) & ~7)) * uint32_t((Kp1 / 4 + 8) * 2);
}
size_t rm_smem(int E, int Kp1) {
    return size_t((32 * rm_hpitch(Kp1) + 127) / 128 * 128) + size_t(kRMSlots) * rm_chunk_bytes(E, Kp1) + 128 +
           size_t(32) * (E + 1) * 4;
}

template <int EPL>
__global__ void __launch_bounds__((kRMWarps + 1) * 32, 2) k_route_mma(RouteArgs a, Plan P) {
    constexpr int E = 32 * EPL, NT = E / 8, IPW = 2 * NT / kRMWarps;  // B tiles; items per warp
    extern __shared__ __align__(128) uint8_t sm[];
    const int d = a.d, Kp1 = a.Kp1, hp = rm_hpitch(Kp1);
    const int Kc = Kp1 / 4, cpitch = (Kc + 8) * 2, nsteps = Kc / 16;
    const uint32_t cb = rm_chunk_bytes(E, Kp1);
    uint8_t* ring = sm + (32 * hp + 127) / 128 * 128;
    uint64_t* hbar = reinterpret_cast<uint64_t*>(ring + kRMSlots * cb);
    uint64_t* full = hbar + 1;
    uint64_t* empty = full + kRMSlots;
    float* s_l = reinterpret_cast<float*>(sm + (32 * hp + 127) / 128 * 128 + kRMSlots * cb + 128);  // [32][E + 1]
    __shared__ int s_exp[64];
    __shared__ int s_hist[256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int64_t t0 = int64_t(blockIdx.x) * 32;
    // diagnostics: globaltimer stamps of CTAs < kTraceRouteCtas (0 start, 1 rows, 2-5 chunks,
    // 6 MMAs done, 7 logits in smem, 8 selection done, 11 ticket, 12 plan)
    const int trs = (gridDim.x + kTraceRouteCtas - 1) / kTraceRouteCtas;  // every trs-th CTA
    unsigned long long* tr = a.trace && blockIdx.x % trs == 0 ? a.trace + (blockIdx.x / trs) * 16 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = gtime_ns();
    for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;
    const int ntok = a.T - t0 < 32 ? int(a.T - t0) : 32;
    if (threadIdx.x == 0) {
        mbar_init(hbar, 1);
        for (int s = 0; s < kRMSlots; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kRMWarps); }
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < 32 * (Kp1 - d); i += blockDim.x) {  // K padding of the rows: zeros
        const int r = i / (Kp1 - d), k = d + i % (Kp1 - d);
        reinterpret_cast<__half*>(sm + r * hp)[k] = __float2half_rn(0.f);
    }
    __syncthreads();
    if (warp == kRMWarps) {
        if (lane == 0) {
            const __half* h = static_cast<const __half*>(a.h);
            mbar_arrive_expect_tx(hbar, uint32_t(ntok * d * 2));
            for (int r = 0; r < ntok; ++r) bulk_g2s(sm + r * hp, h + (t0 + r) * d, uint32_t(d * 2), hbar);
            for (int c = 0; c < 4; ++c) {
                const int s = c % kRMSlots;
                if (c >= kRMSlots) mbar_wait(&empty[s], ((c / kRMSlots) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], cb);
                bulk_g2s(ring + s * cb, reinterpret_cast<const uint8_t*>(a.wgt) + size_t(c) * cb, cb, &full[s]);
            }
        }
        __syncwarp();
    } else {
        float acc[IPW][2][2][4];  // [item][hi, lo][even, odd k-step][4]
#pragma unroll
        for (int x = 0; x < IPW; ++x)
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
                for (int q = 0; q < 2; ++q)
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[x][h2][q][i] = 0.f;
        const int mt = warp & 1;
        // ldmatrix row addresses. A (token rows): matrices (rows 0-7 | 8-15) x (k 0-7 | 8-15) ->
        // a0..a3; B (expert rows of the hi | lo halves) x (k 0-7 | 8-15) -> b0, b1 of hi and lo.
        const int lr = lane & 7, lm = lane >> 3;
        const uint32_t a_row = smem_u32(sm) + min(mt * 16 + lr + (lm & 1) * 8, ntok - 1) * hp + (lm >> 1) * 16;
        mbar_wait(hbar, 0);
        if (tr && threadIdx.x == 0) tr[1] = gtime_ns();
        for (int c = 0; c < 4; ++c) {
            const int s = c % kRMSlots;
            mbar_wait(&full[s], (c / kRMSlots) & 1);
            if (tr && threadIdx.x == 0) tr[2 + c] = gtime_ns();
            const uint32_t buf = smem_u32(ring + s * cb);
#pragma unroll
            for (int x = 0; x < IPW; ++x) {
                const int nt = (warp >> 1) + x * (kRMWarps / 2);
                const uint32_t b_row = buf + ((lm >> 1) * E + nt * 8 + lr) * cpitch + (lm & 1) * 16;
                const uint32_t a_c = a_row + c * Kc * 2;
#pragma unroll 2
                for (int s2 = 0; s2 < nsteps; s2 += 2) {  // nsteps is even (Kp1 % 128 == 0)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {  // even / odd k-step: two accumulator sets
                        const int st = s2 + q;
                        uint32_t a0, a1, a2, a3, bh0, bh1, bl0, bl1;
                        ldsm_x4(a_c + st * 32, a0, a1, a2, a3);
                        ldsm_x4(b_row + st * 32, bh0, bh1, bl0, bl1);
                        mma_16816(acc[x][0][q], a0, a1, a2, a3, bh0, bh1);
                        mma_16816(acc[x][1][q], a0, a1, a2, a3, bl0, bl1);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (tr && threadIdx.x == 0) tr[6] = gtime_ns();
        // c0, c1: token mt*16+g, experts nt*8+2t, +1; c2, c3: token + 8 (fixed summation order)
        const float us = __int_as_float((127 - a.wg_shift) << 23);  // exact power of two
#pragma unroll
        for (int x = 0; x < IPW; ++x) {
            const int nt = (warp >> 1) + x * (kRMWarps / 2);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float v = ((acc[x][0][0][i] + acc[x][0][1][i]) + (acc[x][1][0][i] + acc[x][1][1][i])) * us;
                const int tok = mt * 16 + g + 8 * (i >> 1), e = nt * 8 + 2 * t + (i & 1);
                s_l[tok * (E + 1) + e] = v;
            }
        }
        named_bar_sync(1, kRMWarps * 32);  // all 32 x E logits of the CTA in smem
        if (tr && threadIdx.x == 0) tr[7] = gtime_ns();
        // selection: 8 lanes per token, all 32 tokens at once (lane j of a group holds experts
        // j, j+8, ...); argmax with the reference's scan semantics (NaN skipped unless at the
        // first index, ties -> lowest index), softmax gate in double (model.cpp:214-227)
        {
            constexpr int PER = E / 8;
            const int lt = warp * 4 + (lane >> 3), sub = lane & 7;
            const int ltc = lt < ntok ? lt : ntok - 1;
            const float* lrow = s_l + ltc * (E + 1);
            float l[PER];
#pragma unroll
            for (int j = 0; j < PER; ++j) l[j] = lrow[sub + 8 * j];
            int best[2] = {0, 0};
            float bvs[2] = {0.f, 0.f};
#pragma unroll
            for (int slot = 0; slot < 2; ++slot) {
                if (slot == 1 && a.topk == 1) break;
                const int skip = slot == 0 ? -1 : best[0];
                const int first = skip == 0 ? 1 : 0;
                float bv = -INFINITY;
                int bi = 1 << 30;
#pragma unroll
                for (int j = 0; j < PER; ++j) {
                    const int e = sub + 8 * j;
                    if (e == skip || l[j] != l[j]) continue;
                    if (bi == (1 << 30) || l[j] > bv) { bv = l[j]; bi = e; }
                }
#pragma unroll
                for (int o = 4; o; o >>= 1) {
                    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    if (oi != (1 << 30) && (bi == (1 << 30) || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
                }
                const float lf = lrow[first];
                if (lf != lf) { bi = first; bv = lf; }
                else if (bi == (1 << 30)) { bi = first; bv = lf; }
                best[slot] = bi;
                bvs[slot] = bv;
            }
            float g1, g2 = 0.f;
            if (a.topk == 1) {
                const double mx = double(bvs[0]);
                double sum = 0.0;
#pragma unroll
                for (int j = 0; j < PER; ++j) sum += exp(double(l[j]) - mx);
#pragma unroll
                for (int o = 4; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                g1 = float(double(float(exp(double(bvs[0]) - mx))) / sum);
            } else {
                const double z = exp(double(bvs[1]) - double(bvs[0]));
                g1 = float(1.0 / (1.0 + z));
                g2 = float(z / (1.0 + z));
            }
            if (sub == 0) {
                const int k = a.topk;
                if (lt < ntok) {
                    const int64_t t = t0 + lt;
                    P.expert[t * k] = best[0];
                    P.gate[t * k] = g1;
                    s_exp[lt * k] = best[0];
                    if (k == 2) {
                        P.expert[t * k + 1] = best[1];
                        P.gate[t * k + 1] = g2;
                        s_exp[lt * k + 1] = best[1];
                    }
                } else {
                    s_exp[lt * k] = -1;
                    if (k == 2) s_exp[lt * k + 1] = -1;
                }
            }
        }
        if (tr && threadIdx.x == 0) tr[8] = gtime_ns();
    }
    // the drained token rows + Wg slot stage the per-CTA histograms of the last-CTA plan
    ranks_hist_plan(a, P, s_exp, s_hist, 32, reinterpret_cast<int*>(sm), int((ring - sm + kRMSlots * cb) / 4), tr);
}

// ---- persistent tensor-core router (E = 32, Kp1 <= 1024): Wg resident, token rows streamed ----
// k_route_mma reloads all of Wg (135 KB at d = 1024) for every 32-token CTA and pays the
// two-wave tail; here one CTA per SM keeps the split Wg in shared memory for the whole launch
// and walks the 32-token tiles tile = blockIdx.x, + gridDim.x, ... (the same tiles, histograms
// and lrank layout as the per-CTA kernels, so scatter and plan_tail are unchanged). Each tile
// is two 16-token halves streamed by a producer warp through two row buffers; warp w computes
// expert tile w & 3 over K half w >> 2 (hi + lo, even / odd k-step accumulators) and the two K
// halves meet in a fixed order at selection. Each CTA adds its tile count to the ticket once;
// the CTA that completes the count runs the plan, with all of its shared memory as staging.
constexpr int kRPWarps = 8;
__host__ __device__ inline size_t rp_smem(int Kp1) {
    return size_t(4) * rm_chunk_bytes(32, Kp1) + 2 * size_t(16) * rm_hpitch(Kp1) + 2 * 32 * 33 * 4 + 128;
}

__global__ void __launch_bounds__((kRPWarps + 1) * 32, 1) k_route_mma_p(RouteArgs a, Plan P) {
    constexpr int E = 32, NTHR = kRPWarps * 32;
    extern __shared__ __align__(128) uint8_t sm[];
    const int d = a.d, Kp1 = a.Kp1, hp = rm_hpitch(Kp1);
    const int Kc = Kp1 / 4, cpitch = (Kc + 8) * 2, nsteps = Kc / 16;
    const uint32_t cb = rm_chunk_bytes(E, Kp1);
    uint8_t* wgs = sm;                                  // [4 chunks][hi, lo][32][Kc + 8]
    uint8_t* hb = wgs + 4 * cb;                         // [2 buffers][16 rows][hp]
    float* part = reinterpret_cast<float*>(hb + 2 * 16 * hp);  // [K half][32 tokens][33]
    uint64_t* bars = reinterpret_cast<uint64_t*>(part + 2 * 32 * 33);
    uint64_t* wbar = bars;          // Wg landed
    uint64_t* hfull = bars + 1;     // [2]
    uint64_t* hempty = bars + 3;    // [2]
    __shared__ int s_exp[64];
    __shared__ int s_hist[E];
    __shared__ int s_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = int((a.T + 31) / 32);
    // diagnostics (CTAs < kTraceRouteCtas): 0 start, 1 Wg landed, per tile i < 3: 2+3i rows,
    // 3+3i MMAs, 4+3i tile done; 11 ticket
    unsigned long long* tr = a.trace && blockIdx.x < kTraceRouteCtas ? a.trace + blockIdx.x * 16 : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = gtime_ns();
    if (threadIdx.x == 0) {
        mbar_init(wbar, 1);
        for (int b = 0; b < 2; ++b) { mbar_init(hfull + b, 1); mbar_init(hempty + b, kRPWarps); }
        fence_barrier_init();
        s_last = 0;
    }
    // K padding columns of both row buffers: zeros (the copies never touch them)
    for (int i = threadIdx.x; i < 2 * 16 * (Kp1 - d); i += blockDim.x) {
        const int r = i / (Kp1 - d), k = d + i % (Kp1 - d);
        reinterpret_cast<__half*>(hb + r * hp)[k] = __float2half_rn(0.f);
    }
    __syncthreads();
    if (warp == kRPWarps) {
        // ------------------------------ producer ------------------------------
        if (lane == 0) {
            mbar_arrive_expect_tx(wbar, 4 * cb);
            bulk_g2s(wgs, a.wgt, 4 * cb, wbar);
            const __half* h = static_cast<const __half*>(a.h);
            int n = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
                for (int half = 0; half < 2; ++half, ++n) {
                    const int b = n & 1;
                    if (n >= 2) mbar_wait(hempty + b, ((n >> 1) - 1) & 1);
                    const int64_t r0 = int64_t(tile) * 32 + half * 16;
                    const int rows = int(a.T - r0 < 16 ? a.T - r0 : 16);
                    mbar_arrive_expect_tx(hfull + b, rows > 0 ? uint32_t(rows * d * 2) : 0u);
                    for (int r = 0; r < rows; ++r)
                        bulk_g2s(hb + (b * 16 + r) * hp, h + (r0 + r) * d, uint32_t(d * 2), hfull + b);
                }
        }
        __syncwarp();
    } else {
        // ------------------------------ MMA + selection warps ------------------------------
        const int nt = warp & 3, kq = warp >> 2;  // expert tile, K half (chunks 2kq, 2kq + 1)
        const int lr = lane & 7, lm = lane >> 3, g = lane >> 2, t = lane & 3;
        const float us = __int_as_float((127 - a.wg_shift) << 23);
        mbar_wait(wbar, 0);
        if (tr && threadIdx.x == 0) tr[1] = gtime_ns();
        int n = 0, it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int64_t t0 = int64_t(tile) * 32;
            const int ntok = int(a.T - t0 < 32 ? a.T - t0 : 32);
            for (int e = threadIdx.x; e < E; e += NTHR) s_hist[e] = 0;
            for (int half = 0; half < 2; ++half, ++n) {
                const int b = n & 1;
                mbar_wait(hfull + b, (n >> 1) & 1);
                if (tr && threadIdx.x == 0 && half == 0 && it < 3) tr[2 + 3 * it] = gtime_ns();
                const int hrows = max(1, min(16, ntok - half * 16));
                const uint32_t a_row = smem_u32(hb) + (b * 16 + min(lr + (lm & 1) * 8, hrows - 1)) * hp + (lm >> 1) * 16;
                float acc[2][2][4];  // [hi, lo][even, odd][4]
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
                    for (int q = 0; q < 2; ++q)
#pragma unroll
                        for (int i = 0; i < 4; ++i) acc[h2][q][i] = 0.f;
                for (int c = 2 * kq; c < 2 * kq + 2; ++c) {
                    const uint32_t b_row = smem_u32(wgs + c * cb) + ((lm >> 1) * E + nt * 8 + lr) * cpitch + (lm & 1) * 16;
                    const uint32_t a_c = a_row + c * Kc * 2;
#pragma unroll 2
                    for (int s2 = 0; s2 < nsteps; s2 += 2) {
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const int st = s2 + q;
                            uint32_t a0, a1, a2, a3, bh0, bh1, bl0, bl1;
                            ldsm_x4(a_c + st * 32, a0, a1, a2, a3);
                            ldsm_x4(b_row + st * 32, bh0, bh1, bl0, bl1);
                            mma_16816(acc[0][q], a0, a1, a2, a3, bh0, bh1);
                            mma_16816(acc[1][q], a0, a1, a2, a3, bl0, bl1);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(hempty + b);  // this warp is done with the rows
                // c0, c1: token g, experts nt*8+2t, +1; c2, c3: token g + 8
                float* pk = part + kq * 32 * 33;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int tok = half * 16 + g + 8 * (i >> 1), e = nt * 8 + 2 * t + (i & 1);
                    pk[tok * 33 + e] = (acc[0][0][i] + acc[0][1][i]) + (acc[1][0][i] + acc[1][1][i]);
                }
            }
            named_bar_sync(1, NTHR);  // the tile's partial logits are in smem
            if (tr && threadIdx.x == 0 && it < 3) tr[3 + 3 * it] = gtime_ns();
            // selection: 8 lanes per token, all 32 tokens (see k_route_mma)
            {
                constexpr int PER = E / 8;
                const int lt = warp * 4 + (lane >> 3), sub = lane & 7;
                const int ltc = lt < ntok ? lt : ntok - 1;
                float l[PER];
#pragma unroll
                for (int j = 0; j < PER; ++j)
                    l[j] = (part[ltc * 33 + sub + 8 * j] + part[32 * 33 + ltc * 33 + sub + 8 * j]) * us;
                int best[2] = {0, 0};
                float bvs[2] = {0.f, 0.f};
#pragma unroll
                for (int slot = 0; slot < 2; ++slot) {
                    if (slot == 1 && a.topk == 1) break;
                    const int skip = slot == 0 ? -1 : best[0];
                    const int first = skip == 0 ? 1 : 0;
                    float bv = -INFINITY;
                    int bi = 1 << 30;
                    float lf = 0.f;
#pragma unroll
                    for (int j = 0; j < PER; ++j) {
                        const int e = sub + 8 * j;
                        if (e == first) lf = l[j];
                        if (e == skip || l[j] != l[j]) continue;
                        if (bi == (1 << 30) || l[j] > bv) { bv = l[j]; bi = e; }
                    }
#pragma unroll
                    for (int o = 4; o; o >>= 1) {
                        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
                        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                        if (oi != (1 << 30) && (bi == (1 << 30) || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
                    }
                    lf = __shfl_sync(0xffffffffu, lf, (lane & ~7) | first);  // the scan's first logit
                    if (lf != lf || bi == (1 << 30)) { bi = first; bv = lf; }
                    best[slot] = bi;
                    bvs[slot] = bv;
                }
                float g1, g2 = 0.f;
                if (a.topk == 1) {
                    const double mx = double(bvs[0]);
                    double sum = 0.0;
#pragma unroll
                    for (int j = 0; j < PER; ++j) sum += exp(double(l[j]) - mx);
#pragma unroll
                    for (int o = 4; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                    g1 = float(double(float(exp(double(bvs[0]) - mx))) / sum);
                } else {
                    const double z = exp(double(bvs[1]) - double(bvs[0]));
                    g1 = float(1.0 / (1.0 + z));
                    g2 = float(z / (1.0 + z));
                }
                if (sub == 0) {
                    const int k = a.topk;
                    if (lt < ntok) {
                        const int64_t tk = t0 + lt;
                        P.expert[tk * k] = best[0];
                        P.gate[tk * k] = g1;
                        s_exp[lt * k] = best[0];
                        if (k == 2) {
                            P.expert[tk * k + 1] = best[1];
                            P.gate[tk * k + 1] = g2;
                            s_exp[lt * k + 1] = best[1];
                        }
                    } else {
                        s_exp[lt * k] = -1;
                        if (k == 2) s_exp[lt * k + 1] = -1;
                    }
                }
            }
            named_bar_sync(1, NTHR);
            // stable ranks inside the tile + tile histogram (as ranks_hist_plan)
            for (int i = threadIdx.x; i < 32 * a.topk; i += NTHR) {
                const int e = s_exp[i];
                if (e < 0) continue;
                int r = 0;
                for (int j = 0; j < i; ++j) r += s_exp[j] == e;
                P.lrank[int64_t(tile) * 32 * a.topk + i] = r;
                atomicAdd(&s_hist[e], 1);
            }
            named_bar_sync(1, NTHR);
            for (int e = threadIdx.x; e < E; e += NTHR) P.cta_counts[int64_t(tile) * E + e] = s_hist[e];
            named_bar_sync(1, NTHR);
            if (tr && threadIdx.x == 0 && it < 3) tr[4 + 3 * it] = gtime_ns();
        }
    }
    __syncthreads();  // producer and consumers: the loop is over, all of smem is free
    if (threadIdx.x == 0) {  // one ticket per CTA: its tile count
        const unsigned mine = unsigned((ntiles - 1 - int(blockIdx.x)) / int(gridDim.x) + 1);
        __threadfence();  // release this CTA's tiles (ordered by the barrier)
        if (atomicAdd(&P.tickets[0], mine) + mine == unsigned(ntiles)) {
            __threadfence();  // acquire every other CTA's
            s_last = 1;
        }
        if (tr) tr[11] = gtime_ns();
    }
    __syncthreads();
    if (!s_last) return;
    if (a.trace && threadIdx.x == 0) a.trace[(kTraceRouteCtas - 1) * 16 + 13] = gtime_ns();  // plan start
    plan_tail(a, P, ntiles, 32, reinterpret_cast<int*>(sm), int(rp_smem(Kp1) / 4) - 64);
    __syncthreads();
    if (a.trace && threadIdx.x == 0) a.trace[(kTraceRouteCtas - 1) * 16 + 14] = gtime_ns();  // plan end
}

// ---- large T (prefill) ----------------------------------------------------------------
// k_route_logits: one warp = 32 tokens (lane = token) x 8 experts; a CTA = 4
// warps = 32 tokens x 32 experts, grid (T/32, E/32). Each Wg row is a smem
// broadcast (2 x LDS.128 per warp per k), so a MAC costs one FMUL + one FADD
// in the reference's exact order. Staging is double-buffered in registers.
constexpr int kRLTok = 32, kRLExp = 32, kRLRows = 32;
// VEC: fp16 activations with d % 8 == 0 and E % 32 == 0 -> one 16-byte h load
// and two float4 Wg loads per thread per 32-row chunk; otherwise scalar.
template <bool VEC>
__global__ void __launch_bounds__(128) k_route_logits(RouteArgs a, float* __restrict__ logits) {
    __shared__ __align__(16) float s_h[2][kRLRows][kRLTok + 1];
    __shared__ __align__(16) float s_w[2][kRLRows][kRLExp];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int E = a.E, d = a.d;
    const int64_t t0 = int64_t(blockIdx.x) * kRLTok;
    const int e0 = blockIdx.y * kRLExp;
    const int nchunks = (d + kRLRows - 1) / kRLRows;
    float ph[8], pw[8];
    auto load = [&](int c) {
        const int p0 = c * kRLRows;
        if constexpr (VEC) {
            const int r = tid >> 2, c8 = tid & 3;  // token row, 8-wide p segment
            const int64_t t = t0 + r;
            uint4 hv = make_uint4(0, 0, 0, 0);
            if (t < a.T && p0 + 8 * c8 < d)
                hv = __ldg(reinterpret_cast<const uint4*>(static_cast<const __half*>(a.h) + t * d + p0 + 8 * c8));
            const __half2* h2 = reinterpret_cast<const __half2*>(&hv);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = __half22float2(h2[i]);
                ph[2 * i] = f.x;
                ph[2 * i + 1] = f.y;
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int idx = i * 128 + tid, q = idx >> 3, c4 = idx & 7;
                float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
                if (p0 + q < d) w = __ldg(reinterpret_cast<const float4*>(a.wg + int64_t(p0 + q) * E + e0 + 4 * c4));
                pw[4 * i] = w.x; pw[4 * i + 1] = w.y; pw[4 * i + 2] = w.z; pw[4 * i + 3] = w.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int r = i * 4 + warp;
                const int64_t t = t0 + r;
                ph[i] = (t < a.T && p0 + lane < d) ? load_act(a.h, a.h_f16, t * d + p0 + lane) : 0.0f;
                const int q = i * 4 + warp;
                pw[i] = (p0 + q < d && e0 + lane < E) ? __ldg(a.wg + int64_t(p0 + q) * E + e0 + lane) : 0.0f;
            }
        }
    };
    auto store = [&](int b) {
        if constexpr (VEC) {
            const int r = tid >> 2, c8 = tid & 3;
#pragma unroll
            for (int i = 0; i < 8; ++i) s_h[b][8 * c8 + i][r] = ph[i];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int idx = i * 128 + tid, q = idx >> 3, c4 = idx & 7;
                *reinterpret_cast<float4*>(&s_w[b][q][4 * c4]) = make_float4(pw[4 * i], pw[4 * i + 1], pw[4 * i + 2], pw[4 * i + 3]);
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                s_h[b][lane][i * 4 + warp] = ph[i];
                s_w[b][i * 4 + warp][lane] = pw[i];
            }
        }
    };
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
    load(0);
    for (int c = 0; c < nchunks; ++c) {
        const int b = c & 1;
        store(b);
        __syncthreads();
        if (c + 1 < nchunks) load(c + 1);
        const int pn = min(kRLRows, d - c * kRLRows);
#pragma unroll 8
        for (int q = 0; q < kRLRows; ++q) {
            if (q >= pn) break;
            const float av = s_h[b][q][lane];
            const float4 w0 = *reinterpret_cast<const float4*>(&s_w[b][q][8 * warp]);
            const float4 w1 = *reinterpret_cast<const float4*>(&s_w[b][q][8 * warp + 4]);
            const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            float pr[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) pr[e] = __fmul_rn(av, w[e]);
            // reference: `if (av == 0.0f) continue; orow[j] += av * brow[j];`
            if (av != 0.0f) {
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[e] = __fadd_rn(acc[e], pr[e]);
            }
        }
    }
    const int64_t t = t0 + lane;
    if (t < a.T) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int j = e0 + 8 * warp + e;
            if (j < E) logits[t * E + j] = acc[e];
        }
    }
}

// k_route_logits2t: the VEC case with two tokens per lane (lane, lane + 32): a CTA = 64 tokens x
// 32 experts, so each Wg smem broadcast feeds 16 products instead of 8. Same exact chain per
// (token, expert) as k_route_logits (FMUL then FADD in ascending k, zero activations skipped).
constexpr int kRL2Tok = 64;
__global__ void __launch_bounds__(128) k_route_logits2t(RouteArgs a, float* __restrict__ logits) {
    __shared__ __align__(16) float s_h[2][kRLRows][kRL2Tok + 1];
    __shared__ __align__(16) float s_w[2][kRLRows][kRLExp];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int E = a.E, d = a.d;
    const int64_t t0 = int64_t(blockIdx.x) * kRL2Tok;
    const int e0 = blockIdx.y * kRLExp;
    const int nchunks = (d + kRLRows - 1) / kRLRows;
    float ph[16], pw[8];
    auto load = [&](int c) {
        const int p0 = c * kRLRows;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int r = (tid >> 2) + 32 * u, c8 = tid & 3;  // token row, 8-wide p segment
            const int64_t t = t0 + r;
            uint4 hv = make_uint4(0, 0, 0, 0);
            if (t < a.T && p0 + 8 * c8 < d)
                hv = __ldg(reinterpret_cast<const uint4*>(static_cast<const __half*>(a.h) + t * d + p0 + 8 * c8));
            const __half2* h2 = reinterpret_cast<const __half2*>(&hv);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = __half22float2(h2[i]);
                ph[8 * u + 2 * i] = f.x;
                ph[8 * u + 2 * i + 1] = f.y;
            }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int idx = i * 128 + tid, q = idx >> 3, c4 = idx & 7;
            float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
            if (p0 + q < d) w = __ldg(reinterpret_cast<const float4*>(a.wg + int64_t(p0 + q) * E + e0 + 4 * c4));
            pw[4 * i] = w.x; pw[4 * i + 1] = w.y; pw[4 * i + 2] = w.z; pw[4 * i + 3] = w.w;
        }
    };
    auto store = [&](int b) {
        const int c8 = tid & 3;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int r = (tid >> 2) + 32 * u;
#pragma unroll
            for (int i = 0; i < 8; ++i) s_h[b][8 * c8 + i][r] = ph[8 * u + i];
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int idx = i * 128 + tid, q = idx >> 3, c4 = idx & 7;
            *reinterpret_cast<float4*>(&s_w[b][q][4 * c4]) = make_float4(pw[4 * i], pw[4 * i + 1], pw[4 * i + 2], pw[4 * i + 3]);
        }
    };
    float acc0[8], acc1[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc0[e] = acc1[e] = 0.0f;
    load(0);
    for (int c = 0; c < nchunks; ++c) {
        const int b = c & 1;
        store(b);
        __syncthreads();
        if (c + 1 < nchunks) load(c + 1);
        const int pn = min(kRLRows, d - c * kRLRows);
#pragma unroll 8
        for (int q = 0; q < kRLRows; ++q) {
            if (q >= pn) break;
            const float av0 = s_h[b][q][lane], av1 = s_h[b][q][lane + 32];
            const float4 w0 = *reinterpret_cast<const float4*>(&s_w[b][q][8 * warp]);
            const float4 w1 = *reinterpret_cast<const float4*>(&s_w[b][q][8 * warp + 4]);
            const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            // reference: `if (av == 0.0f) continue; orow[j] += av * brow[j];`
            if (av0 != 0.0f) {
#pragma unroll
                for (int e = 0; e < 8; ++e) acc0[e] = __fadd_rn(acc0[e], __fmul_rn(av0, w[e]));
            }
            if (av1 != 0.0f) {
#pragma unroll
                for (int e = 0; e < 8; ++e) acc1[e] = __fadd_rn(acc1[e], __fmul_rn(av1, w[e]));
            }
        }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const int64_t t = t0 + lane + 32 * u;
        if (t < a.T) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int j = e0 + 8 * warp + e;
                if (j < E) logits[t * E + j] = u ? acc1[e] : acc0[e];
            }
        }
    }
}

constexpr int kRouteSelWarps = 32;  // tokens per selection CTA
// k_route_select: one warp per token reads its E logits, applies the
// reference argmax / softmax gate (or top-2), then stable ranks, CTA
// histogram and the last-CTA plan as in the small-T kernel.
__global__ void __launch_bounds__(kRouteSelWarps * 32) k_route_select(RouteArgs a, Plan P) {
    __shared__ int s_exp[kRouteSelWarps * 2];
    __shared__ int s_hist[256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int E = a.E;
    for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;
    const int64_t t = int64_t(blockIdx.x) * kRouteSelWarps + warp;
    if (t < a.T) {
        float l[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int j = lane + 32 * e;
            l[e] = j < E ? __ldcg(P.logits + t * E + j) : 0.0f;
        }
        finish_token<8>(a, P, l, t, warp, s_exp);
    } else if (lane == 0) {
        s_exp[warp * a.topk] = -1;
        if (a.topk == 2) s_exp[warp * a.topk + 1] = -1;
    }
    ranks_hist_plan(a, P, s_exp, s_hist, kRouteSelWarps);
}

// Pre-routed rows (expert-parallel owner side): expert ids / gates are inputs (one expert per
// row); build stable ranks, per-CTA histograms and the plan exactly as routing does. Tiles of
// kPlanIdsTile rows keep the last CTA's plan scan short (config 4 owner: 32 K rows -> 128
// tiles x E counts instead of 1024).
__global__ void __launch_bounds__(kPlanIdsTile) k_plan_from_ids(RouteArgs a, Plan P) {
    __shared__ int s_exp[kPlanIdsTile];
    __shared__ int s_hist[256];
    for (int e = threadIdx.x; e < a.E; e += blockDim.x) s_hist[e] = 0;
    {
        const int64_t t = int64_t(blockIdx.x) * kPlanIdsTile + threadIdx.x;
        int e = -1;
        if (t < a.T) {
            e = P.expert[t];
            if (e < 0 || e >= a.E) e = -1;  // validated on the host; never index out of range
        }
        s_exp[threadIdx.x] = e;
    }
    ranks_hist_plan(a, P, s_exp, s_hist, kPlanIdsTile);
}

cudaError_t launch_plan_from_ids(const RouteArgs& a, const Plan& P, cudaStream_t st) {
    if (a.topk != 1) return cudaErrorInvalidValue;
    const unsigned grid = unsigned((a.T + kPlanIdsTile - 1) / kPlanIdsTile);
    k_plan_from_ids<<<grid, kPlanIdsTile, 0, st>>>(a, P);
    return cudaGetLastError();
}

// Scatter routing metadata and gather token rows into the expert-grouped
// fp16 activation matrix x_perm [T*k x ldx] (tcgen05 B operand; zero-padded
// to ldx columns). One warp per (token, slot).
__global__ void __launch_bounds__(256) k_scatter(const void* h, int h_f16, int64_t T, int d, int topk,
                                                 int E, int tt, int path, int gemv_max, Plan P, __half* x_perm,
                                                 int ldx, float* zero_out) {
    const int64_t i = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= T * topk) return;
    const int64_t t = i / topk;
    const int e = P.expert[i];
    const int n_e = P.counts[e];
    const int pos = P.offsets[e] + P.cta_counts[(t / tt) * E + e] + P.lrank[i];
    if (lane == 0) {
        P.perm_token[pos] = int32_t(t);
        P.perm_gate[pos] = P.gate[i];
        P.inv_pos[i] = pos;
    }
    if (zero_out && (i % topk) == 0)
        for (int j = lane; j < d; j += 32) zero_out[t * d + j] = 0.f;
    const bool gemm = n_e > 0 && (path == 2 || (path == 0 && n_e > gemv_max));
    if (!gemm || x_perm == nullptr) return;
    __half* dst = x_perm + int64_t(pos) * ldx;
    if (h_f16 && (d % 8) == 0) {
        const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __half*>(h) + t * d);
        uint4* o = reinterpret_cast<uint4*>(dst);
        for (int j = lane; j < d / 8; j += 32) o[j] = __ldg(src + j);
    } else {
        for (int j = lane; j < d; j += 32) dst[j] = __float2half_rn(load_act(h, h_f16, t * d + j));
    }
    for (int j = d + lane; j < ldx; j += 32) dst[j] = __float2half_rn(0.f);
}

namespace {
template <int EPL, int EFIX, int TT>
cudaError_t launch_dec_tt(const RouteArgs& a, const Plan& P, size_t smem, cudaStream_t st) {
    static bool configured_dev[kMaxDevices] = {};
    int dev_ = 0;
    cudaGetDevice(&dev_);
    bool& configured = configured_dev[dev_ < kMaxDevices ? dev_ : 0];
    if (!configured) {
        cudaFuncSetAttribute(k_route_decode<EPL, EFIX, TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        configured = true;
    }
    const unsigned nct = unsigned((a.T + TT - 1) / TT);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nct);
    cfg.blockDim = dim3((TT + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = TT == 1 ? 1 : nct;  // no_plan: independent CTAs
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = a.pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k_route_decode<EPL, EFIX, TT>, a, P);
}
template <int EPL, int EFIX, bool SEL>
cudaError_t launch_chain(const RouteArgs& a, const Plan& P, size_t smem, cudaStream_t st) {
    static bool configured_dev[kMaxDevices] = {};
    int dev_ = 0;
    cudaGetDevice(&dev_);
    bool& configured = configured_dev[dev_ < kMaxDevices ? dev_ : 0];
    if (!configured) {
        cudaFuncSetAttribute(k_route_chain<EPL, EFIX, SEL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((a.T + kRCTok - 1) / kRCTok));
    cfg.blockDim = dim3((kRCTok + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = a.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_route_chain<EPL, EFIX, SEL>, a, P);
}
template <int EPL, int EFIX>
cudaError_t launch_dec(const RouteArgs& a, const Plan& P, size_t smem, cudaStream_t st) {
    if (a.no_plan) {
        const size_t cs = route_chain_smem(a.d, EFIX ? EFIX : a.E);
        if (a.wg_blk && cs <= 220 * 1024 && a.dbg != 7)  // dbg 7: the strided-Wg chain (comparison)
            return a.wg_finite ? launch_chain<EPL, EFIX, false>(a, P, cs, st) : launch_chain<EPL, EFIX, true>(a, P, cs, st);
        // only the chain kernel writes the fc1 row blocks: a caller that skipped k_xrows because
        // route_chain_used() said so must not silently get k_route_decode
        if (a.xr) return cudaErrorInvalidValue;
        return launch_dec_tt<EPL, EFIX, 1>(a, P, smem, st);
    }
    return launch_dec_tt<EPL, EFIX, kRouteSmallWarps>(a, P, smem, st);
}
}  // namespace

bool route_chain_one_chunk(int d, int E) { return rc_slots(d, E) == 1; }
bool route_chain_used(const RouteArgs& a) {
    return a.no_plan && a.wg_blk && a.T <= kRouteDecMaxT && a.E <= kRouteDecMaxE && a.dbg != 7 &&
           route_chain_smem(a.d, a.E) <= 220 * 1024 && route_small_smem(a.d, a.E) <= 220 * 1024;
}
cudaError_t launch_route_decode(const RouteArgs& a, const Plan& P, size_t smem, cudaStream_t st) {
    switch (a.E) {
        case 32: return launch_dec<1, 32>(a, P, smem, st);
        case 64: return launch_dec<2, 64>(a, P, smem, st);
        case 128: return launch_dec<4, 128>(a, P, smem, st);
        case 256: return launch_dec<8, 256>(a, P, smem, st);
        default: return launch_dec<8, 0>(a, P, smem, st);
    }
}

// MOQE_ROUTE_EXACT=1: prefill routing keeps the reference's exact-order fp32 chains
bool route_mma_enabled() {
    static const bool v = [] { const char* s = getenv("MOQE_ROUTE_EXACT"); return !(s && atoi(s) == 1); }();
    return v;
}

// Route tile: tokens per routing CTA for a given T (must match scatter's tt). Above the
// threshold the batched routers run (tensor-core logits for E = 32 / 64 with the bank's split
// gate weights); at or below it the per-token exact-order kernels. MOQE_ROUTE_BIG_T overrides.
int64_t route_big_threshold() {
    static const int64_t v = [] {
        const char* s = getenv("MOQE_ROUTE_BIG_T");
        return s ? std::max<int64_t>(32, atoll(s)) : int64_t(32);
    }();
    return v;
}
int route_tokens_per_cta(int64_t T) { return T <= route_big_threshold() ? kRouteSmallWarps : kRouteSelWarps; }

static bool route_logits2t_enabled() {  // MOQE_ROUTE_LOGITS_2T=0: one token per lane (A/B)
    static const bool v = [] {
        const char* s = getenv("MOQE_ROUTE_LOGITS_2T");
        return !(s && s[0] == '0');
    }();
    return v;
}

cudaError_t launch_route(const RouteArgs& a, const Plan& P, cudaStream_t st) {
    const int tt = route_tokens_per_cta(a.T);
    const unsigned grid = unsigned((a.T + tt - 1) / tt);
    if (a.T > route_big_threshold()) {
        if (P.logits == nullptr) return cudaErrorInvalidValue;
        dim3 lg(unsigned((a.T + kRLTok - 1) / kRLTok), unsigned((a.E + kRLExp - 1) / kRLExp));
        const bool vec = a.h_f16 && (a.d % 8) == 0 && (a.E % 32) == 0 && (reinterpret_cast<uintptr_t>(a.h) & 15) == 0;
        const size_t sm2 = rl2_smem(a.d, a.E);
        int dev_ = 0;
        cudaGetDevice(&dev_);
        const int di = dev_ < kMaxDevices ? dev_ : 0;
        const size_t smm = rm_smem(a.E, a.Kp1);
        if (vec && a.wgt && a.wg_finite && a.E == 32 && a.Kp1 % 128 == 0 && a.Kp1 >= a.d &&
            rp_smem(a.Kp1) <= 220 * 1024 && route_mma_enabled()) {
            static bool cfgp[kMaxDevices] = {};
            static int nsm[kMaxDevices] = {};
            if (!cfgp[di]) {
                cudaFuncSetAttribute(k_route_mma_p, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
                cudaDeviceGetAttribute(&nsm[di], cudaDevAttrMultiProcessorCount, dev_);
                cfgp[di] = true;
            }
            const unsigned gp = unsigned(std::min<int64_t>((a.T + 31) / 32, nsm[di]));
            k_route_mma_p<<<gp, (kRPWarps + 1) * 32, rp_smem(a.Kp1), st>>>(a, P);
            return cudaGetLastError();
        }
        if (vec && a.wgt && a.wg_finite && (a.E == 32 || a.E == 64) && a.Kp1 % 128 == 0 && a.Kp1 >= a.d &&
            smm <= 220 * 1024 && route_mma_enabled()) {
            static bool cfgm[kMaxDevices][2] = {};
            const unsigned gm = unsigned((a.T + 31) / 32);
            if (a.E == 32) {
                if (!cfgm[di][0]) { cudaFuncSetAttribute(k_route_mma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024); cfgm[di][0] = true; }
                k_route_mma<1><<<gm, (kRMWarps + 1) * 32, smm, st>>>(a, P);
            } else {
                if (!cfgm[di][1]) { cudaFuncSetAttribute(k_route_mma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024); cfgm[di][1] = true; }
                k_route_mma<2><<<gm, (kRMWarps + 1) * 32, smm, st>>>(a, P);
            }
            return cudaGetLastError();
        }
        if (vec && (a.E == 32 || a.E == 64) && sm2 <= 220 * 1024 && (reinterpret_cast<uintptr_t>(a.wg) & 15) == 0) {
            static bool cfg2[kMaxDevices][2] = {};
            bool& cfg32 = cfg2[di][0];
            bool& cfg64 = cfg2[di][1];
            const unsigned g2 = unsigned((a.T + 31) / 32);
            if (a.E == 32) {
                if (!cfg32) { cudaFuncSetAttribute(k_route_logits2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024); cfg32 = true; }
                k_route_logits2<4><<<g2, (kRL2Warps + 1) * 32, sm2, st>>>(a, P);
            } else {
                if (!cfg64) { cudaFuncSetAttribute(k_route_logits2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024); cfg64 = true; }
                k_route_logits2<8><<<g2, (kRL2Warps + 1) * 32, sm2, st>>>(a, P);
            }
            return cudaGetLastError();  // selection and plan are fused into the logits kernel
        } else if (vec && route_logits2t_enabled()) {
            dim3 lg2(unsigned((a.T + kRL2Tok - 1) / kRL2Tok), unsigned((a.E + kRLExp - 1) / kRLExp));
            k_route_logits2t<<<lg2, 128, 0, st>>>(a, P.logits);
        } else if (vec) k_route_logits<true><<<lg, 128, 0, st>>>(a, P.logits);
        else k_route_logits<false><<<lg, 128, 0, st>>>(a, P.logits);
        k_route_select<<<grid, kRouteSelWarps * 32, 0, st>>>(a, P);
        return cudaGetLastError();
    }
    const size_t smem = route_small_smem(a.d, a.E);
    if (smem > 220 * 1024) return cudaErrorInvalidValue;
    if (a.T <= kRouteDecMaxT && a.E <= kRouteDecMaxE) return launch_route_decode(a, P, smem, st);
    static bool configured_dev[kMaxDevices] = {};
    int dev_ = 0;
    cudaGetDevice(&dev_);
    bool& configured = configured_dev[dev_ < kMaxDevices ? dev_ : 0];
    if (!configured) {
        const int mx = 220 * 1024;
        cudaFuncSetAttribute(k_route_small<1, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_route_small<2, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_route_small<4, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_route_small<8, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_route_small<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        configured = true;
    }
    constexpr int nthr = (kRouteSmallWarps + 1) * 32;
    switch (a.E) {
        case 32: k_route_small<1, 32><<<grid, nthr, smem, st>>>(a, P); break;
        case 64: k_route_small<2, 64><<<grid, nthr, smem, st>>>(a, P); break;
        case 128: k_route_small<4, 128><<<grid, nthr, smem, st>>>(a, P); break;
        case 256: k_route_small<8, 256><<<grid, nthr, smem, st>>>(a, P); break;
        default: k_route_small<8, 0><<<grid, nthr, smem, st>>>(a, P); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_scatter(const void* h, int h_f16, int64_t T, int d, int topk, int E, int path, int gemv_max, int tt,
                           const Plan& P, __half* x_perm, int ldx, float* zero_out, cudaStream_t st) {
    const int64_t n = T * topk;
    if (n == 0) return cudaSuccess;
    k_scatter<<<unsigned((n + 7) / 8), 256, 0, st>>>(h, h_f16, T, d, topk, E, tt, path,
                                                     gemv_max > 0 ? gemv_max : kGemvMaxRows, P, x_perm, ldx, zero_out);
    return cudaGetLastError();
}

}  // namespace moqe_gpu
