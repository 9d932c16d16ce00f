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

// One warp computes TPW tokens x E experts (lane j handles experts j, j+32, ...).
template <int EPL, int TPW>
__global__ void __launch_bounds__(kRouteWarps * 32) k_route(RouteArgs a, Plan P) {
    constexpr int TT = kRouteWarps * TPW;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int E = a.E, d = a.d, k = a.topk;
    const int64_t tok0 = int64_t(blockIdx.x) * TT + warp * TPW;

    float acc[TPW][EPL];
#pragma unroll
    for (int i = 0; i < TPW; ++i)
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[i][e] = 0.0f;

    for (int p0 = 0; p0 < d; p0 += 32) {
        float hv[TPW];
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
            const int64_t t = tok0 + i;
            hv[i] = (t < a.T && p0 + lane < d) ? load_act(a.h, a.h_f16, t * d + p0 + lane) : 0.0f;
        }
        const int qn = min(32, d - p0);
#pragma unroll 4
        for (int q = 0; q < qn; ++q) {
            float w[EPL];
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                const int j = lane + 32 * e;
                w[e] = j < E ? __ldg(a.wg + int64_t(p0 + q) * E + j) : 0.0f;
            }
#pragma unroll
            for (int i = 0; i < TPW; ++i) {
                const float av = __shfl_sync(0xffffffffu, hv[i], q);
#pragma unroll
                for (int e = 0; e < EPL; ++e) {
                    // reference: `if (av == 0.0f) continue; orow[j] += av * brow[j];`
                    const float pr = __fmul_rn(av, w[e]);
                    acc[i][e] = av != 0.0f ? __fadd_rn(acc[i][e], pr) : acc[i][e];
                }
            }
        }
    }

    __shared__ int s_exp[TT * 2];
    __shared__ int s_hist[256];
    for (int e = threadIdx.x; e < E; e += blockDim.x) s_hist[e] = 0;

#pragma unroll
    for (int i = 0; i < TPW; ++i) {
        const int64_t t = tok0 + i;
        const int lt = warp * TPW + i;
        if (t >= a.T) {  // warp-uniform
            if (lane == 0) { s_exp[lt * k] = -1; if (k == 2) s_exp[lt * k + 1] = -1; }
            continue;
        }
        float b1v, b2v = 0.f;
        int b1i, b2i = 0;
        warp_argmax<EPL>(acc[i], E, -1, b1v, b1i);
        float g1, g2 = 0.f;
        if (k == 1) {
            // softmax in double (model.cpp:214-227); gate = prob[best] (:343)
            const double mx = double(b1v);
            double s = 0.0;
#pragma unroll
            for (int e = 0; e < EPL; ++e)
                if (lane + 32 * e < E) s += exp(double(acc[i][e]) - mx);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            const float eb = float(exp(double(b1v) - mx));
            g1 = float(double(eb) / s);
        } else {
            warp_argmax<EPL>(acc[i], E, b1i, b2v, b2i);
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
    __syncthreads();
    // stable local ranks + CTA histogram
    for (int i = threadIdx.x; i < TT * k; i += blockDim.x) {
        const int e = s_exp[i];
        if (e < 0) continue;
        int r = 0;
        for (int j = 0; j < i; ++j) r += s_exp[j] == e;
        P.lrank[int64_t(blockIdx.x) * TT * k + i] = r;
        atomicAdd(&s_hist[e], 1);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) P.cta_counts[int64_t(blockIdx.x) * E + e] = s_hist[e];

    // last CTA plans
    __threadfence();
    __syncthreads();
    __shared__ bool s_last;
    if (threadIdx.x == 0) s_last = atomicAdd(&P.tickets[0], 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    plan_tail(a, P, gridDim.x, TT);
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

namespace {
template <int EPL, int TPW>
cudaError_t launch_route_t(const RouteArgs& a, const Plan& P, cudaStream_t st) {
    constexpr int TT = kRouteWarps * TPW;
    const unsigned grid = unsigned((a.T + TT - 1) / TT);
    k_route<EPL, TPW><<<grid, kRouteWarps * 32, 0, st>>>(a, P);
    return cudaGetLastError();
}
}  // namespace

// Route tile: tokens per routing CTA for a given T (must match scatter's tt).
int route_tokens_per_cta(int64_t T) { return T <= 2048 ? kRouteWarps : kRouteWarps * 8; }

cudaError_t launch_route(const RouteArgs& a, const Plan& P, cudaStream_t st) {
    const bool big = a.T > 2048;
    const int epl = (a.E + 31) / 32;
#define MOQE_ROUTE_CASE(EPLV)                                                              \
    if (epl <= EPLV) return big ? launch_route_t<EPLV, 8>(a, P, st) : launch_route_t<EPLV, 1>(a, P, st);
    MOQE_ROUTE_CASE(1)
    MOQE_ROUTE_CASE(2)
    MOQE_ROUTE_CASE(4)
    MOQE_ROUTE_CASE(8)
#undef MOQE_ROUTE_CASE
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
