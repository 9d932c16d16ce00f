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

#include "kernels.cuh"

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

// Last-CTA planning: per-CTA bases, counts, offsets, expert lists, resets.
__device__ void plan_tail(const RouteArgs& a, Plan P, int n_ctas, int tt) {
    const int E = a.E, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
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
    __syncthreads();
    // 2. offsets + expert lists (warp 0, expert order)
    if (warp == 0) {
        int run = 0, ngemv = 0, ngemm = 0, tiles = 0, mx = 0;
        for (int e0 = 0; e0 < E; e0 += 32) {
            const int e = e0 + lane;
            const int n = e < E ? P.counts[e] : 0;
            int incl = n;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            if (e < E) P.offsets[e] = run + incl - n;
            run += __shfl_sync(0xffffffffu, incl, 31);
            int m = n;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
            mx = max(mx, m);
            const bool gemv = n > 0 && (a.path == 1 || (a.path == 0 && n <= kGemvMaxRows));
            const bool gemm = n > 0 && !gemv;
            const unsigned bg = __ballot_sync(0xffffffffu, gemv), bm = __ballot_sync(0xffffffffu, gemm);
            const unsigned lt = (1u << lane) - 1u;
            if (gemv) P.gemv_list[ngemv + __popc(bg & lt)] = e;
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
            P.meta[1] = ngemm;
            P.meta[2] = tiles;
            P.meta[3] = mx;
            P.tickets[1] = 0;
            P.tickets[2] = 0;
            P.tickets[3] = 0;
            P.tickets[0] = 0;  // self-reset for the next forward
        }
    }
    for (int e = threadIdx.x; e < E; e += blockDim.x) P.done[e] = 0;
    __syncthreads();
    // 3. small problems: scatter routing metadata here (no extra launch)
    if (a.inline_scatter) {
        const int64_t n = a.T * a.topk;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const int64_t t = i / a.topk;
            const int e = __ldcg(P.expert + i);
            const int pos = P.offsets[e] + P.cta_counts[(t / tt) * E + e] + __ldcg(P.lrank + i);
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

__device__ __forceinline__ void ranks_hist_plan(const RouteArgs& a, Plan& P, int* s_exp, int* s_hist, int tt) {
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
    __threadfence();
    __syncthreads();
    __shared__ bool s_last;
    if (threadIdx.x == 0) s_last = atomicAdd(&P.tickets[0], 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    plan_tail(a, P, gridDim.x, tt);
}

constexpr int kRouteSmallWarps = 4;   // one token per warp; a warp per SM sub-partition

// Wg rows staged per chunk for a given expert count.
__host__ __device__ constexpr int route_chunk_rows(int E) { return E <= 128 ? 4096 / (E < 32 ? 32 : E) : 32; }

// Small T (decode): one warp per token, lane j <-> experts j, j+32, ...
// The token rows sit in smem (loaded once); Wg streams through a
// double-buffered smem chunk (register prefetch of the next chunk overlaps the
// current chunk's sequential fp32 chain). EFIX > 0 compiles the expert count
// in (E == EFIX): the chunk copy is unpredicated float4 and the 32-row inner
// loop unrolls to immediate smem offsets; EFIX == 0 is the generic path.
template <int EPL, int EFIX>
__global__ void __launch_bounds__(kRouteSmallWarps * 32) k_route_small(RouteArgs a, Plan P) {
    constexpr int TT = kRouteSmallWarps;
    constexpr int NT = kRouteSmallWarps * 32;
    extern __shared__ __align__(16) float s_dyn[];
    __shared__ int s_exp[TT * 2];
    __shared__ int s_hist[256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int E = EFIX ? EFIX : a.E, d = a.d;
    const int rows = EFIX ? route_chunk_rows(EFIX) : route_chunk_rows(a.E);
    const int chunk = rows * E;
    const int nchunks = (d + rows - 1) / rows;
    const int dpad = nchunks * rows;
    float* s_w = s_dyn;                     // [2][chunk]
    float* s_hrow = s_dyn + 2 * chunk;      // [TT][dpad] token rows, zero padded
    const int64_t t = int64_t(blockIdx.x) * TT + warp;
    const bool live = t < a.T;
    for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;
    for (int p = lane; p < dpad; p += 32)
        s_hrow[warp * dpad + p] = (live && p < d) ? load_act(a.h, a.h_f16, t * d + p) : 0.0f;

    float acc[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[e] = 0.0f;
    // EFIX: chunk == 4096 floats (E <= 128) or 32*E; each thread moves chunk/NT floats as float4
    constexpr int V4 = EFIX ? (route_chunk_rows(EFIX) * EFIX) / (4 * NT) : 1;
    float4 pre[V4];
    const int64_t lim = int64_t(d) * E;
    auto load_chunk = [&](int c) {
        const int64_t base = int64_t(c) * chunk;
        if constexpr (EFIX != 0) {
#pragma unroll
            for (int i = 0; i < V4; ++i) {
                const int64_t idx = base + 4 * (int64_t(i) * NT + threadIdx.x);
                pre[i] = idx + 3 < lim ? __ldg(reinterpret_cast<const float4*>(a.wg + idx)) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    };
    auto store_chunk = [&](int c, float* buf) {
        if constexpr (EFIX != 0) {
#pragma unroll
            for (int i = 0; i < V4; ++i) reinterpret_cast<float4*>(buf)[i * NT + threadIdx.x] = pre[i];
        } else {
            const int64_t base = int64_t(c) * chunk;
            for (int i = threadIdx.x; i < chunk; i += NT) buf[i] = base + i < lim ? __ldg(a.wg + base + i) : 0.0f;
        }
    };
    load_chunk(0);
    for (int c = 0; c < nchunks; ++c) {
        float* buf = s_w + (c & 1) * chunk;
        store_chunk(c, buf);
        __syncthreads();
        if (c + 1 < nchunks) load_chunk(c + 1);
        if (live) {
            const float* hr = s_hrow + warp * dpad + c * rows;
            for (int q0 = 0; q0 < rows; q0 += 32) {
                const float* wb = buf + q0 * E + lane;
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const float av = hr[q0 + q];  // smem broadcast; 0 beyond d
#pragma unroll
                    for (int e = 0; e < EPL; ++e) {
                        const float w = (EFIX || lane + 32 * e < E) ? wb[q * E + 32 * e] : 0.0f;
                        // reference: `if (av == 0.0f) continue; orow[j] += av * brow[j];`
                        const float pr = __fmul_rn(av, w);
                        if (av != 0.0f) acc[e] = __fadd_rn(acc[e], pr);
                    }
                }
            }
        }
        // buffer (c&1) is rewritten at c+2, after the next iteration's barrier
    }
    if (live) finish_token<EPL>(a, P, acc, t, warp, s_exp);
    else if (lane == 0) { s_exp[warp * a.topk] = -1; if (a.topk == 2) s_exp[warp * a.topk + 1] = -1; }
    ranks_hist_plan(a, P, s_exp, s_hist, TT);
}

constexpr int kRouteBigWarps = 2;     // 64 tokens per CTA, one token per thread
constexpr int kRouteBigGroup = 32;    // experts accumulated per pass
constexpr int kRouteBigRows = 32;     // Wg / h rows staged per chunk

// Large T (prefill): one token per thread; each Wg row is broadcast from smem
// to the warp (LDS.128 = 4 experts), so a MAC costs one FMUL + one FADD.
// Staging is double-buffered through registers (all loads of chunk c+1 are in
// flight while chunk c is consumed). Experts are processed in groups of 32
// (logits kept in smem) so registers stay bounded for any E <= 256;
// argmax/softmax then run one warp per token.
__global__ void __launch_bounds__(kRouteBigWarps * 32) k_route_big(RouteArgs a, Plan P) {
    constexpr int TT = kRouteBigWarps * 32;
    constexpr int NT = TT;
    constexpr int HS = TT + 1;  // transposed h stride (conflict-free)
    extern __shared__ __align__(16) float sm[];
    float* s_h = sm;                                     // [2][kRouteBigRows][HS]
    float* s_w = s_h + 2 * kRouteBigRows * HS;           // [2][kRouteBigRows][kRouteBigGroup] (16B aligned: 2*32*65 floats)
    float* s_log = s_w + 2 * kRouteBigRows * kRouteBigGroup;  // [TT][E+1]
    int* s_exp = reinterpret_cast<int*>(s_log + TT * (a.E + 1));
    int* s_hist = s_exp + TT * 2;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int E = a.E, d = a.d, LS = a.E + 1;
    const int64_t t0 = int64_t(blockIdx.x) * TT;
    for (int e = tid; e < E; e += blockDim.x) s_hist[e] = 0;
    const int nchunks = (d + kRouteBigRows - 1) / kRouteBigRows;
    // per thread per chunk: h = TT*32 values -> 32 per thread (token row segments);
    // Wg = 32 rows x 32 experts -> 16 per thread
    constexpr int HV = kRouteBigRows * TT / NT, WV = kRouteBigRows * kRouteBigGroup / NT;
    float ph[HV], pw[WV];
    for (int g0 = 0; g0 < E; g0 += kRouteBigGroup) {
        const int gn = min(kRouteBigGroup, E - g0);
        auto load = [&](int c) {
            const int p0 = c * kRouteBigRows;
#pragma unroll
            for (int i = 0; i < HV; ++i) {  // element (r = token, q = p offset), q fastest per warp
                const int r = i * (NT / 32) + warp, q = lane;
                const int64_t tt = t0 + r;
                ph[i] = (tt < a.T && p0 + q < d) ? load_act(a.h, a.h_f16, tt * d + p0 + q) : 0.0f;
            }
#pragma unroll
            for (int i = 0; i < WV; ++i) {
                const int idx = i * NT + tid, q = idx / kRouteBigGroup, e = idx % kRouteBigGroup;
                pw[i] = (p0 + q < d && e < gn) ? __ldg(a.wg + int64_t(p0 + q) * E + g0 + e) : 0.0f;
            }
        };
        float acc[kRouteBigGroup];
#pragma unroll
        for (int e = 0; e < kRouteBigGroup; ++e) acc[e] = 0.0f;
        load(0);
        for (int c = 0; c < nchunks; ++c) {
            float* bh = s_h + (c & 1) * kRouteBigRows * HS;
            float* bw = s_w + (c & 1) * kRouteBigRows * kRouteBigGroup;
#pragma unroll
            for (int i = 0; i < HV; ++i) bh[lane * HS + i * (NT / 32) + warp] = ph[i];
#pragma unroll
            for (int i = 0; i < WV; ++i) bw[i * NT + tid] = pw[i];
            __syncthreads();
            if (c + 1 < nchunks) load(c + 1);
            const int pn = min(kRouteBigRows, d - c * kRouteBigRows);
            for (int q = 0; q < pn; ++q) {
                const float av = bh[q * HS + tid];
                const float4* wr = reinterpret_cast<const float4*>(bw + q * kRouteBigGroup);
#pragma unroll
                for (int e4 = 0; e4 < kRouteBigGroup / 4; ++e4) {
                    const float4 w = wr[e4];
                    const float p0f = __fmul_rn(av, w.x), p1f = __fmul_rn(av, w.y);
                    const float p2f = __fmul_rn(av, w.z), p3f = __fmul_rn(av, w.w);
                    if (av != 0.0f) {
                        acc[4 * e4 + 0] = __fadd_rn(acc[4 * e4 + 0], p0f);
                        acc[4 * e4 + 1] = __fadd_rn(acc[4 * e4 + 1], p1f);
                        acc[4 * e4 + 2] = __fadd_rn(acc[4 * e4 + 2], p2f);
                        acc[4 * e4 + 3] = __fadd_rn(acc[4 * e4 + 3], p3f);
                    }
                }
            }
        }
#pragma unroll
        for (int e = 0; e < kRouteBigGroup; ++e)
            if (e < gn) s_log[tid * LS + g0 + e] = acc[e];
        __syncthreads();
    }
    // per-token argmax + gate (one warp per token, reusing the warp helpers)
    for (int r = warp; r < TT; r += kRouteBigWarps) {
        const int64_t t = t0 + r;
        if (t >= a.T) {
            if (lane == 0) { s_exp[r * a.topk] = -1; if (a.topk == 2) s_exp[r * a.topk + 1] = -1; }
            continue;
        }
        float l[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int j = lane + 32 * e;
            l[e] = j < E ? s_log[r * LS + j] : 0.0f;
        }
        finish_token<8>(a, P, l, t, r, s_exp);
    }
    ranks_hist_plan(a, P, s_exp, s_hist, TT);
}

// Scatter routing metadata and gather token rows into the expert-grouped
// fp16 activation matrix x_perm [T*k x ldx] (tcgen05 B operand; zero-padded
// to ldx columns). One warp per (token, slot).
__global__ void __launch_bounds__(256) k_scatter(const void* h, int h_f16, int64_t T, int d, int topk,
                                                 int E, int tt, int path, Plan P, __half* x_perm,
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
    const bool gemm = n_e > 0 && (path == 2 || (path == 0 && n_e > kGemvMaxRows));
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

// Route tile: tokens per routing CTA for a given T (must match scatter's tt).
constexpr int64_t kRouteBigThreshold = 512;
int route_tokens_per_cta(int64_t T) {
    return T <= kRouteBigThreshold ? kRouteSmallWarps : kRouteBigWarps * 32;
}

namespace {
size_t route_big_smem(int E) {
    return sizeof(float) * (2 * kRouteBigRows * (kRouteBigWarps * 32 + 1) + 2 * kRouteBigRows * kRouteBigGroup +
                            kRouteBigWarps * 32 * (E + 1)) +
           sizeof(int) * (kRouteBigWarps * 32 * 2 + E);
}
}  // namespace

cudaError_t launch_route(const RouteArgs& a, const Plan& P, cudaStream_t st) {
    const int tt = route_tokens_per_cta(a.T);
    const unsigned grid = unsigned((a.T + tt - 1) / tt);
    if (a.T > kRouteBigThreshold) {
        const size_t smem = route_big_smem(a.E);
        static int configured = 0;
        if (!configured) {
            cudaError_t e = cudaFuncSetAttribute(k_route_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 int(route_big_smem(256)));
            if (e != cudaSuccess) return e;
            configured = 1;
        }
        k_route_big<<<grid, kRouteBigWarps * 32, smem, st>>>(a, P);
        return cudaGetLastError();
    }
    const int rows = route_chunk_rows(a.E);
    const int dpad = (a.d + rows - 1) / rows * rows;
    const size_t smem = (size_t(2) * rows * a.E + size_t(kRouteSmallWarps) * dpad) * sizeof(float);
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    static bool configured = false;
    if (!configured) {
        const int mx = 200 * 1024;
        cudaFuncSetAttribute(k_route_small<1, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_route_small<2, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_route_small<4, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_route_small<8, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(k_route_small<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        configured = true;
    }
    switch (a.E) {
        case 32: k_route_small<1, 32><<<grid, kRouteSmallWarps * 32, smem, st>>>(a, P); return cudaGetLastError();
        case 64: k_route_small<2, 64><<<grid, kRouteSmallWarps * 32, smem, st>>>(a, P); return cudaGetLastError();
        case 128: k_route_small<4, 128><<<grid, kRouteSmallWarps * 32, smem, st>>>(a, P); return cudaGetLastError();
        case 256: k_route_small<8, 256><<<grid, kRouteSmallWarps * 32, smem, st>>>(a, P); return cudaGetLastError();
        default: k_route_small<8, 0><<<grid, kRouteSmallWarps * 32, smem, st>>>(a, P); return cudaGetLastError();
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_scatter(const void* h, int h_f16, int64_t T, int d, int topk, int E, int path,
                           const Plan& P, __half* x_perm, int ldx, float* zero_out, cudaStream_t st) {
    const int64_t n = T * topk;
    if (n == 0) return cudaSuccess;
    k_scatter<<<unsigned((n + 7) / 8), 256, 0, st>>>(h, h_f16, T, d, topk, E, route_tokens_per_cta(T),
                                                     path, P, x_perm, ldx, zero_out);
    return cudaGetLastError();
}

}  // namespace moqe_gpu
