// dec.cu — decode path (T*k <= 64 routed rows, d_model <= 1024): two launches.
//
//   k_dec_route  one thread-block cluster. Each CTA owns a slice of d_model: it stages its
//                rows of Wg (before the PDL wait, so the copy overlaps the previous grid) and
//                its columns of h, and forms partial logits with FFMA; the partials are summed
//                over DSMEM in CTA-rank order (a fixed order: deterministic). Each token's
//                (expert, gate) is broadcast to every CTA, every CTA builds the same plan
//                (stable expert-grouped row order, units of <= 16 rows) and writes its share
//                of the permuted fp16 activation rows.
//   k_dec<BITS>  persistent weight-streaming expert FFN, one CTA per SM. The work is the
//                sequence (unit u, f-slice j) over every routed unit and the S = d_ffn/64
//                slices of its expert; CTA c takes a contiguous range of it (stream-K).
//                A slice is self-contained: fc1 for 64 channels (all of d_model) -> ReLU ->
//                fp16 mid -> fc2 partial over those 64 k. fc2 partials accumulate in registers
//                while the CTA stays on one unit and are flushed as 2^-24 fixed point with
//                integer atomics (order-independent, so the sum is deterministic). The CTA
//                whose flush completes a unit's S slices applies scale, bias and gate and
//                stores the rows (top-2: the second finisher of a token adds the two slots).
//                No grid-wide waits, so partial residency cannot deadlock.
//
// Reference path replaced: moqe::top1_route + moe_ffn_forward (proj/src/model.cpp:328-393);
// top-2 renormalisation per BASELINE config 4 (oracle/moqe_oracle.c orc_route).
// Numerics: logits in parallel FFMA order (north_star allows different routing for tokens
// whose top-2 logit gap is < 1e-4); the reference's zero-activation skip is kept (a zero
// activation never multiplies a weight). Codes x fp16 activations are exact products,
// fp32 accumulation, scale in the epilogue, fp16 mid (as the prefill GEMM).
#include <cuda_fp16.h>

#include <algorithm>
#include <type_traits>

#include "codec.cuh"
#include "kernels.cuh"

namespace moqe_gpu {

namespace {

constexpr int kDecThreads = 256;     // router CTA
constexpr int kMidPitch = 64 * 2 + 16;  // bytes per mid row (pitch = 16 mod 128: conflict-free LDS.128)
constexpr float kFix = 16777216.0f;     // 2^24 fixed-point scale of the fc2 partials
constexpr int kMaxRouteSmem = 200 * 1024;
#ifndef DEC_ROLE_SPLIT
#define DEC_ROLE_SPLIT 0
#endif
#ifndef DEC_F1_UNROLL
#define DEC_F1_UNROLL 8
#endif
constexpr int kF1Unroll = DEC_F1_UNROLL;
#ifndef DEC_PLAN_ROWS
#define DEC_PLAN_ROWS 16
#endif
// rows per planned unit (<= kDecUnitRows, the buffer capacity); an expert with more rows gets
// several units. Units of <= 8 rows keep their fc2 partials in registers for the whole run.
constexpr int kDecPlanRows = DEC_PLAN_ROWS;

__device__ __forceinline__ void red_add_s64(long long* p, long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ float ld_cluster_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// ---- span profiler: first CTA's start (after the PDL wait) to the last CTA's exit ----
__device__ __forceinline__ void span_begin(DecSpan* s) {
    if (s) atomicMin(&s->start_min, gtime_ns());
}
__device__ __forceinline__ void span_end(DecSpan* s, unsigned nctas) {
    if (!s) return;
    const unsigned long long t = gtime_ns();
    __threadfence();
    if (atomicAdd(&s->ticket, 1u) == nctas - 1) {
        __threadfence();
        const unsigned long long t0 = atomicExch(&s->start_min, ~0ull);
        if (t > t0) atomicAdd(&s->total_ns, t - t0);
        atomicAdd(&s->count, 1ull);
        s->ticket = 0;
    }
}

// Strict '>' argmax with the reference's sequential semantics (model.cpp:339-341,
// oracle argmax_excluding): ties -> lowest index, a NaN never wins unless it sits at the
// scan's first index. Warp-wide; lane owns experts lane, lane+32, ...
__device__ __forceinline__ int warp_argmax(const float* l, int E, int skip) {
    const int lane = threadIdx.x & 31;
    const int first = skip == 0 ? 1 : 0;
    if (l[first] != l[first]) return first;  // NaN at the scan start stays the best
    float bv = -__int_as_float(0x7f800000);
    int bi = 1 << 30;
    for (int e = lane; e < E; e += 32) {
        const float v = l[e];
        if (e == skip || v != v) continue;
        if (bi == (1 << 30) || v > bv) { bv = v; bi = e; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (oi != (1 << 30) && (bi == (1 << 30) || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
    }
    return bi == (1 << 30) ? first : bi;
}

}  // namespace

// power of two of the codec field holding code position p (0..15) of a 16-code chunk
// (codec.cuh / unpack_chunk_raw)
__device__ __forceinline__ int dec_field_shift(int bits, int p) {
    // one nibble per code pair (p / 2): int2 0,2,4,6,8,0,2,4; int3 0,3,0,3,6,6,0,3; int4 0,4,...
    const uint32_t tab = bits == 2 ? 0x42086420u : bits == 3 ? 0x30663030u : bits == 4 ? 0x40404040u : 0u;
    return int((tab >> (4 * (p >> 1))) & 0xFu);
}

// diagnostics: per-CTA event log (a.trace: [grid][kDecTrace][2] = (event, globaltimer ns)),
// slots [base, base + 21) per role
__device__ __forceinline__ void dec_trace(const DecArgs& a, int base, int& n, int ev) {
    if (a.trace && n < 21) {
        unsigned long long* p = a.trace + (size_t(blockIdx.x) * kDecTrace + base + n) * 2;
        p[0] = unsigned(ev);
        p[1] = gtime_ns();
        ++n;
    }
}

// router events: absolute slots after the FFN kernel's [grid][kDecTrace] block
__device__ __forceinline__ void route_trace(const DecArgs& a, int rank, int& n, int ev) {
    if (a.trace && n < 32 && threadIdx.x == 0) {
        unsigned long long* p = a.trace + (size_t(160 + rank) * kDecTrace + (ev >= 28 ? ev - 28 + 16 : n)) * 2;
        p[0] = unsigned(ev) | (static_cast<unsigned long long>(clock64()) << 8);
        p[1] = gtime_ns();
        ++n;
    }
}

// =====================================================================================
// Router + plan (one cluster)
// =====================================================================================
__global__ void __launch_bounds__(kDecThreads) k_dec_route(const DecArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int C = int(cluster_nctas());
    const int rank = int(cta_rank());
    const int T = a.T, E = a.E, K = a.topk, R = T * K, d = a.d;
    const int rpc = ((d + C - 1) / C + 3) & ~3;  // rows of Wg per CTA (multiple of 4: 16-B aligned rows)
    const int r0 = rank * rpc, nr = max(0, min(d, r0 + rpc) - r0);
    const int Tp = (T + 7) & ~7;
    const int ntile = (Tp / 8) * ((E + 31) / 32);               // 8-token x 32-expert output tiles
    const int ks = ntile >= 8 ? 1 : (ntile >= 4 ? 2 : (ntile >= 2 ? 4 : 8));  // row splits per tile
    float* wgs = reinterpret_cast<float*>(smem);                 // [rpc][E]
    float* hsT = wgs + rpc * E;                                   // [rpc][Tp] (token-minor)
    float* part = hsT + rpc * Tp;                                 // [ks][T][E], later per-warp logit rows
    float* plog = part + max(ks * T * E, 8 * 256);                // [T][E]
    int* ch_e = reinterpret_cast<int*>(plog + T * E);             // [64] (token, slot) choices
    float* ch_g = reinterpret_cast<float*>(ch_e + 64);            // [64]
    int* cnt = reinterpret_cast<int*>(ch_g + 64);                 // [E]
    int* off = cnt + E;                                           // [E + 1] row offsets
    int* ubase = off + E + 1;                                     // [E + 1] unit offsets
    int* pos = ubase + E + 1;                                     // [64]
    uint64_t* bar = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(pos + 64) + 15) & ~uintptr_t(15));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // Wg rows [r0, r0+nr) are contiguous (Wg is [d][E] row-major): one bulk copy, issued
    // before the PDL wait (the gate weights are not produced by the previous grid).
    const uint32_t wbytes = uint32_t(nr) * E * 4;
    const bool bulk = (wbytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(a.wg + size_t(r0) * E) & 15) == 0);
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (tid == 0 && bulk && nr > 0) {
        mbar_arrive_expect_tx(bar, wbytes);
        for (uint32_t o = 0; o < wbytes; o += 32768u)
            bulk_g2s(reinterpret_cast<unsigned char*>(wgs) + o, reinterpret_cast<const unsigned char*>(a.wg + size_t(r0) * E) + o,
                     min(32768u, wbytes - o), bar);
    }
    if (!bulk)
        for (int i = tid; i < nr * E; i += kDecThreads) wgs[i] = a.wg[size_t(r0) * E + i];
    pdl_trigger();
    pdl_wait();
    int rtr = 0;
    route_trace(a, rank, rtr, 20);
    span_begin(tid == 0 ? a.span_route : nullptr);
    // token columns [r0, r0+nr) of h -> f32, transposed (8 consecutive tokens per LDS.128 pair).
    // 8-column chunks with one vector load each (rows of fp16 h are 16-B aligned when d % 8 == 0)
    const bool vec = a.h_f16 && (d % 8 == 0) && ((reinterpret_cast<uintptr_t>(a.h) & 15) == 0);
    if (vec) {
        const int nc = rpc / 4;  // 4-column units (rpc is a multiple of 4); load 8 when both halves exist
        for (int i = tid; i < Tp * (nc / 2 + (nc & 1)); i += kDecThreads) {
            const int per = nc / 2 + (nc & 1);
            const int t = i / per, k = (i - t * per) * 8;
            float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (t < T && k < nr) {
                const __half* src = static_cast<const __half*>(a.h) + size_t(t) * d + r0 + k;
                if (k + 8 <= nr) {
                    const uint4 q = *reinterpret_cast<const uint4*>(src);
                    const __half2* hp = reinterpret_cast<const __half2*>(&q);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = __half22float2(hp[e]);
                        v[2 * e] = f.x;
                        v[2 * e + 1] = f.y;
                    }
                } else {
                    for (int e = 0; k + e < nr && e < 8; ++e) v[e] = __half2float(src[e]);
                }
            }
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (k + e < rpc) hsT[(k + e) * Tp + t] = v[e];
        }
    } else {
        for (int i = tid; i < Tp * rpc; i += kDecThreads) {
            const int t = i / rpc, k = i - t * rpc;
            float v = 0.f;
            if (t < T && k < nr) {
                const size_t gi = size_t(t) * d + r0 + k;
                v = a.h_f16 ? __half2float(static_cast<const __half*>(a.h)[gi]) : static_cast<const float*>(a.h)[gi];
            }
            hsT[k * Tp + t] = v;
        }
    }
    route_trace(a, rank, rtr, 21);
    if (bulk && nr > 0) mbar_wait(bar, 0);
    route_trace(a, rank, rtr, 22);
    // non-finite gate weights: keep the reference's zero-activation skip (0 * inf must not
    // reach the sum, model.cpp:160); otherwise a plain FMA is the same sum
    bool nonfinite = false;
    for (int i = tid; i < nr * E; i += kDecThreads) nonfinite |= !isfinite(wgs[i]);
    nonfinite = __syncthreads_or(nonfinite);
    // partial logits: warp = (8-token x 32-expert tile, row split); lane = expert; 8 FMA chains
    {
        const int rps = (nr + ks - 1) / ks;
        for (int wi = warp; wi < ntile * ks; wi += kDecThreads / 32) {
            const int tile = wi / ks, sp = wi - tile * ks;
            const int tb = tile % (Tp / 8), eg = tile / (Tp / 8);
            const int e = eg * 32 + lane;
            const int k0 = sp * rps, k1 = min(nr, k0 + rps);
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (e < E) {
                if (!nonfinite) {
#pragma unroll 4
                    for (int k = k0; k < k1; ++k) {
                        const float w = wgs[k * E + e];
                        const float4 x0 = *reinterpret_cast<const float4*>(hsT + k * Tp + tb * 8);
                        const float4 x1 = *reinterpret_cast<const float4*>(hsT + k * Tp + tb * 8 + 4);
                        acc[0] = fmaf(x0.x, w, acc[0]); acc[1] = fmaf(x0.y, w, acc[1]);
                        acc[2] = fmaf(x0.z, w, acc[2]); acc[3] = fmaf(x0.w, w, acc[3]);
                        acc[4] = fmaf(x1.x, w, acc[4]); acc[5] = fmaf(x1.y, w, acc[5]);
                        acc[6] = fmaf(x1.z, w, acc[6]); acc[7] = fmaf(x1.w, w, acc[7]);
                    }
                } else {
                    for (int k = k0; k < k1; ++k) {
                        const float w = wgs[k * E + e];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float x = hsT[k * Tp + tb * 8 + i];
                            if (x != 0.f) acc[i] = fmaf(x, w, acc[i]);
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int t = tb * 8 + i;
                    if (t < T) part[(sp * T + t) * E + e] = acc[i];
                }
            }
        }
    }
    __syncthreads();
    for (int o = tid; o < T * E; o += kDecThreads) {  // row splits summed in a fixed order
        float v = part[o];
        for (int sp = 1; sp < ks; ++sp) v += part[sp * T * E + o];
        plog[o] = v;
    }
    route_trace(a, rank, rtr, 23);
    cluster_sync();
    route_trace(a, rank, rtr, 24);
    // reduce partials in rank order; this CTA owns tokens t = rank, rank + C, ...
    for (int t = rank + warp * C; t < T; t += C * (kDecThreads / 32)) {
        float* lt = part + warp * 256;  // per-warp logit row (the partials are consumed)
        for (int e = lane; e < E; e += 32) {
            float v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c)
                if (c < C) v[c] = ld_cluster_f32(map_rank(plog + t * E + e, uint32_t(c)));
            float s = v[0];
#pragma unroll
            for (int c = 1; c < 16; ++c)
                if (c < C) s += v[c];
            lt[e] = s;
        }
        __syncwarp();
        const int b1 = warp_argmax(lt, E, -1);
        int b2 = -1;
        if (K == 2) b2 = warp_argmax(lt, E, b1);
        float g1 = 1.f, g2 = 0.f;
        if (K == 1) {
            // softmax probability of the winner in double (model.cpp:214-227, :343)
            double mx = -1e300;
            for (int e = lane; e < E; e += 32)
                if (double(lt[e]) > mx) mx = double(lt[e]);
            for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            double s = 0.0;
            for (int e = lane; e < E; e += 32) s += exp(double(lt[e]) - mx);
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            g1 = float(double(float(exp(double(lt[b1]) - mx))) / s);
        } else {
            const double z = exp(double(lt[b2]) - double(lt[b1]));
            g1 = float(1.0 / (1.0 + z));
            g2 = float(z / (1.0 + z));
        }
        if (lane < C) {  // broadcast the choice to every CTA of the cluster
            st_cluster_u32(map_rank(ch_e + t * K, uint32_t(lane)), uint32_t(b1));
            st_cluster_u32(map_rank(ch_g + t * K, uint32_t(lane)), __float_as_uint(g1));
            if (K == 2) {
                st_cluster_u32(map_rank(ch_e + t * K + 1, uint32_t(lane)), uint32_t(b2));
                st_cluster_u32(map_rank(ch_g + t * K + 1, uint32_t(lane)), __float_as_uint(g2));
            }
        }
        if (lane == 0) {
            a.expert[t * K] = b1;
            a.gate[t * K] = g1;
            if (K == 2) {
                a.expert[t * K + 1] = b2;
                a.gate[t * K + 1] = g2;
            }
        }
        __syncwarp();
    }
    route_trace(a, rank, rtr, 23);
    cluster_sync();
    route_trace(a, rank, rtr, 24);
    // every CTA builds the same plan: rows grouped by expert, ascending (token, slot) inside
    for (int e = tid; e < E; e += kDecThreads) {
        int c = 0;
        for (int i = 0; i < R; ++i) c += ch_e[i] == e;
        cnt[e] = c;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scans of rows and of units (<= 16 rows each), E <= 256
        const int per = (E + 31) / 32, e0 = lane * per;
        int sr = 0, su = 0;
        for (int e = e0; e < min(E, e0 + per); ++e) { sr += cnt[e]; su += (cnt[e] + kDecPlanRows - 1) / kDecPlanRows; }
        int ir = sr, iu = su;
        for (int o = 1; o < 32; o <<= 1) {
            const int vr = __shfl_up_sync(0xffffffffu, ir, o), vu = __shfl_up_sync(0xffffffffu, iu, o);
            if (lane >= o) { ir += vr; iu += vu; }
        }
        int pr = ir - sr, pu = iu - su;
        for (int e = e0; e < min(E, e0 + per); ++e) {
            off[e] = pr;
            ubase[e] = pu;
            pr += cnt[e];
            pu += (cnt[e] + kDecPlanRows - 1) / kDecPlanRows;
        }
        if (lane == 31) { off[E] = ir; ubase[E] = iu; }
    }
    __syncthreads();
    for (int i = tid; i < R; i += kDecThreads) {
        const int e = ch_e[i];
        int r = 0;
        for (int j = 0; j < i; ++j) r += ch_e[j] == e;
        pos[i] = off[e] + r;
    }
    __syncthreads();
    if (rank == 0) {
        for (int i = tid; i < R; i += kDecThreads) {
            a.perm_token[pos[i]] = i / K;
            a.perm_gate[pos[i]] = ch_g[i];
            a.row_of[i] = pos[i];
        }
        for (int e = tid; e < E; e += kDecThreads) {
            const int n = cnt[e];
            for (int p = 0; p * kDecPlanRows < n; ++p)
                a.units[ubase[e] + p] = make_int4(e, off[e] + p * kDecPlanRows, min(kDecPlanRows, n - p * kDecPlanRows), 0);
        }
        if (tid == 0) *a.n_units = ubase[E];
    }
    route_trace(a, rank, rtr, 25);
    // permuted fp16 rows (zero padded to Kp1), one warp per row, rows split over the CTAs.
    // Value k is stored as fp16(x_k) * 2^-s(k mod 16) (the fc1 weight field's power of two,
    // see unpack_chunk_raw) and Z = Sum_k (1024 + bias * 2^s) * stored_k goes behind the row.
    const int bias = 1 << (a.bits - 1);
    for (int i = rank + warp * C; i < R; i += C * (kDecThreads / 32)) {
        const int t = i / K;
        unsigned char* rowp = reinterpret_cast<unsigned char*>(a.xperm) + size_t(pos[i]) * a.xpitch;
        double z = 0.0;
        // 8 values per lane step: all loads of the row first, then scale / store / Z
        for (int k0 = lane * 8; k0 < a.Kp1; k0 += 32 * 8) {
            float v[8];
            if (vec && k0 + 8 <= d) {
                const uint4 q = __ldg(reinterpret_cast<const uint4*>(static_cast<const __half*>(a.h) + size_t(t) * d + k0));
                const __half2* hp = reinterpret_cast<const __half2*>(&q);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __half22float2(hp[e]);
                    v[2 * e] = f.x;
                    v[2 * e + 1] = f.y;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const int k = k0 + e;
                    const size_t gi = size_t(t) * d + k;
                    v[e] = k >= d ? 0.f
                                  : a.h_f16 ? __half2float(static_cast<const __half*>(a.h)[gi])
                                            : __half2float(__float2half_rn(static_cast<const float*>(a.h)[gi]));
                }
            }
            uint4 o;
            __half2* op = reinterpret_cast<__half2*>(&o);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int sh = dec_field_shift(a.bits, (k0 + 2 * e) & 15);  // one shift per code pair
                const float sc = __int_as_float((127 - sh) << 23);            // 2^-sh, exact
                const __half2 hv = __floats2half2_rn(v[2 * e] * sc, v[2 * e + 1] * sc);
                op[e] = hv;
                const double m = 1024.0 + double(bias) * double(1 << sh);
                z += m * (double(__low2float(hv)) + double(__high2float(hv)));
            }
            *reinterpret_cast<uint4*>(rowp + size_t(k0) * 2) = o;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
        if (lane == 0) *reinterpret_cast<float*>(rowp + a.Kp1 * 2) = float(z);
    }
    __syncthreads();
    route_trace(a, rank, rtr, 26);
    span_end(tid == 0 ? a.span_route : nullptr, gridDim.x);
    cluster_sync();  // no CTA exits while a peer may still read its plog / write its choices
}

// =====================================================================================
// Expert FFN, stream-K over (unit, f-slice)
// =====================================================================================
namespace {

template <int BITS>
struct DecGeom {
    static constexpr int RB = 8 * BITS;  // tile-row bytes (64 codes)
};

// fc1 weights without the fp16 magic subtraction: pair p of a 16-code chunk becomes
// (1024 + u * 2^s_p) exactly (codec.cuh field positions; u = code + 2^(bits-1)). The MMA's
// B values carry 2^-s_k instead (the router writes x_k * 2^-s_k), so each product is
// 1024 * 2^-s_k * x_k + u_k * x_k and Sum q_k x_k = acc - Z with the per-token constant
// Z = Sum_k (1024 + bias * 2^s_k) * B_k (k_dec_route). No HFMA2, no constants.
template <int BITS>
__device__ __forceinline__ void unpack_chunk_raw(const uint8_t* row, int t, uint32_t (&o)[8], const uint32_t (&mg)[8]) {
    if constexpr (BITS == 4) {
        const uint2 w = *reinterpret_cast<const uint2*>(row + 8 * t);
        const uint32_t ws[2] = {w.x, w.y};
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const uint32_t a = ws[q], a8 = ws[q] >> 8;
            o[4 * q + 0] = lop_magic<0x000F000Fu>(a, mg[4 * q + 0]);
            o[4 * q + 1] = lop_magic<0x00F000F0u>(a, mg[4 * q + 1]);
            o[4 * q + 2] = lop_magic<0x000F000Fu>(a8, mg[4 * q + 2]);
            o[4 * q + 3] = lop_magic<0x00F000F0u>(a8, mg[4 * q + 3]);
        }
    } else if constexpr (BITS == 2) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(row + 4 * t);
        const uint32_t w10 = w >> 10;
        o[0] = lop_magic<0x00030003u>(w, mg[0]);
        o[1] = lop_magic<0x000C000Cu>(w, mg[1]);
        o[2] = lop_magic<0x00300030u>(w, mg[2]);
        o[3] = lop_magic<0x00C000C0u>(w, mg[3]);
        o[4] = lop_magic<0x03000300u>(w, mg[4]);
        o[5] = lop_magic<0x00030003u>(w10, mg[5]);
        o[6] = lop_magic<0x000C000Cu>(w10, mg[6]);
        o[7] = lop_magic<0x00300030u>(w10, mg[7]);
    } else if constexpr (BITS == 3) {
        const uint32_t A = *reinterpret_cast<const uint32_t*>(row + 4 * t);
        const uint32_t B = *reinterpret_cast<const uint16_t*>(row + 16 + 2 * t);
        const uint32_t A8 = A >> 8;
        const uint32_t Bx = prmt(B, 0u, 0x4140u);  // (B.lo, 0, B.hi, 0)
        o[0] = lop_magic<0x00070007u>(A, mg[0]);
        o[1] = lop_magic<0x00380038u>(A, mg[1]);
        o[2] = lop_magic<0x00070007u>(A8, mg[2]);
        o[3] = lop_magic<0x00380038u>(A8, mg[3]);
        o[4] = lop_magic<0x00C000C0u>(A, mg[4]) | ((Bx << 2) & 0x01000100u);
        o[5] = lop_magic<0x00C000C0u>(A8, mg[5]) | ((Bx << 1) & 0x01000100u);
        o[6] = lop_magic<0x00070007u>(Bx, mg[6]);
        o[7] = lop_magic<0x00380038u>(Bx, mg[7]);
    } else {  // 8: the magic's high byte (0x64 or 0xE4) joins each code byte
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t wq = reinterpret_cast<const uint32_t*>(row + 16 * t)[q];
            o[2 * q] = prmt(wq, mg[2 * q], 0x7170u);      // (byte0, magic hi, byte1, magic hi)
            o[2 * q + 1] = prmt(wq, mg[2 * q + 1], 0x7372u);
        }
    }
}

template <int BITS>
constexpr int kBias = 1 << (BITS - 1);
template <int BITS>
__device__ __forceinline__ int field_shift_c(int p) {  // p = code position mod 16 (see dec_field_shift)
    constexpr uint32_t tab = BITS == 2 ? 0x42086420u : BITS == 3 ? 0x30663030u : BITS == 4 ? 0x40404040u : 0u;
    return int((tab >> (4 * ((p & 15) >> 1))) & 0xFu);
}

// per-pair magic registers (all 0x6400: fp16 1024 + field)
__device__ __forceinline__ void make_magics(uint32_t (&mg)[8]) {
    uint32_t pos;
    asm("mov.b32 %0, 0x64006400;" : "=r"(pos));  // opaque: keeps the LOP3 a single instruction
#pragma unroll
    for (int p = 0; p < 8; ++p) mg[p] = pos;
}

// ---- warp roles of k_dec -------------------------------------------------------------
constexpr int kF1Warps = 8;   // fc1: (16-channel group of the slice's 64, half of Kp1) each
constexpr int kF2Warps = 8;   // fc2: Np2 / 8 channels each, the slice's 64 k
// + one warpgroup for the TMA producer (warp 16; warps 17-19 only help the routing phase).
// 17 warps would cap every thread at 96 registers (5 warps on one SM sub-partition); with 20,
// the producer warpgroup drops to kDecProdRegs after the routing phase and the fc1 / fc2
// warpgroups grow to kDecMathRegs (setmaxnreg). The increases draw only on what the CTA got at
// launch (640 x 96): 512 x 112 + 128 x 24 fits, 512 x 120 + 128 x 32 never completes.
// Measured: parity-green, no faster (int3 32.6 vs 32.4 us, int2 30.5 vs 29.8), so off by
// default; the slice loops are not register-bound.
#ifndef DEC_SETMAXNREG
#define DEC_SETMAXNREG 0
#endif
constexpr int kDecFfnWarps = DEC_SETMAXNREG ? kF1Warps + kF2Warps + 4 : kF1Warps + kF2Warps + 1;
#if DEC_SETMAXNREG
constexpr int kDecProdRegs = 24, kDecMathRegs = 112;
#endif

// fc1 of one slice for one warp: channels gw*16 .. +15, KP k-tiles from global k-tile kt0.
// xrow[nb] = this lane's activation row (row g of n-block nb) scaled by 2^-s(k).
// Two accumulator sets (even / odd k-tiles) halve the HMMA dependency chain.
template <int BITS, int KP, int NB>
__device__ __forceinline__ void dec_fc1_piece(const unsigned char* piece, int kt0, int gw, int g, int t,
                                              const unsigned char* const (&xrow)[2], float (&ca)[2][4],
                                              float (&cb)[2][4]) {
    constexpr int RB = DecGeom<BITS>::RB;
    const unsigned char* ra = piece + (gw * 16 + g) * RB;
    uint32_t mg[8];
    make_magics(mg);
#pragma unroll kF1Unroll
    for (int i = 0; i < KP; ++i) {
        uint32_t oa[8], ob[8];
        unpack_chunk_raw<BITS>(ra + i * 64 * RB, t, oa, mg);
        unpack_chunk_raw<BITS>(ra + i * 64 * RB + 8 * RB, t, ob, mg);
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
            float(&c)[4] = (i & 1) ? cb[nb] : ca[nb];
            const unsigned char* xr = xrow[nb] + (kt0 + i) * 128 + t * 32;
            const uint4 x0 = *reinterpret_cast<const uint4*>(xr);
            const uint4 x1 = *reinterpret_cast<const uint4*>(xr + 16);
            mma_16816(c, oa[0], ob[0], oa[1], ob[1], x0.x, x0.y);
            mma_16816(c, oa[2], ob[2], oa[3], ob[3], x0.z, x0.w);
            mma_16816(c, oa[4], ob[4], oa[5], ob[5], x1.x, x1.y);
            mma_16816(c, oa[6], ob[6], oa[7], ob[7], x1.z, x1.w);
        }
    }
}

// fc2 partial of one slice for one warp: QW channel groups starting at group q0 of a piece.
// fc2 converts exactly (codec.cuh unpack_chunk: LOP3 + HFMA2 per code pair). A raw variant (the
// fc1 unpack against mid rows pre-scaled by 2^-s(k), per-slice correction Z) was built twice
// and measured parity-green but no faster: removing the fc2 math entirely (DEC_SKIP_FC2) saves
// only ~4 us of the ~32 us step, the slice pipeline being bound by data arrival and the
// tail, not by the converter ALU.
template <int BITS, int QW, int NB>
__device__ __forceinline__ void dec_fc2_piece(const unsigned char* piece, int q0, int g, int t,
                                              const unsigned char* mid, float (&c2)[QW][NB][4]) {
    constexpr int RB = DecGeom<BITS>::RB;
    uint4 m0[NB], m1[NB];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
        const unsigned char* mr = mid + (nb * 8 + g) * kMidPitch + t * 32;
        m0[nb] = *reinterpret_cast<const uint4*>(mr);
        m1[nb] = *reinterpret_cast<const uint4*>(mr + 16);
    }
#pragma unroll
    for (int q = 0; q < QW; ++q) {
        const unsigned char* ra = piece + size_t((q0 + q) * 16 + g) * RB;
        uint32_t oa[8], ob[8];
        unpack_chunk<BITS>(ra, t, oa);
        unpack_chunk<BITS>(ra + 8 * RB, t, ob);
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
            mma_16816(c2[q][nb], oa[0], ob[0], oa[1], ob[1], m0[nb].x, m0[nb].y);
            mma_16816(c2[q][nb], oa[2], ob[2], oa[3], ob[3], m0[nb].z, m0[nb].w);
            mma_16816(c2[q][nb], oa[4], ob[4], oa[5], ob[5], m1[nb].x, m1[nb].y);
            mma_16816(c2[q][nb], oa[6], ob[6], oa[7], ob[7], m1[nb].z, m1[nb].w);
        }
    }
}

}  // namespace

// Per-CTA plan (shared memory) of the fused decode kernel, or pointers into the router's
// global plan (separate-router path).
struct DecPlanSmem {
    int4 units[kDecMaxRows];
    int perm_token[kDecMaxRows];
    float perm_gate[kDecMaxRows];
    int row_of[kDecMaxRows];
    float z[32];            // per-token correction Z of the scaled rows (fused path)
    int ch_e[kDecMaxRows];  // (token, slot) choices
    float ch_g[kDecMaxRows];
    int cnt[256], off[257], ubase[257], pos[kDecMaxRows];
    int n_units;
};

// Fused routing (every CTA, redundantly and bit-identically): logits = Wg^T . h on the tensor
// cores, Wg (pre-split by the bank into fp16 hi + lo, x 2^sw, four K chunks) as the 16-expert A
// tiles and the activation rows as 8-token B tiles; parallel-order fp32 sums, so north_star's
// near-tie exemption applies. In a cluster of cl CTAs (2 or 4), rank r owns chunks
// [r*4/cl, (r+1)*4/cl) (staged before the PDL wait). Warp w owns expert tile w % mtiles and the
// K steps s = w / mtiles (mod KP) of the CTA's range, for EVERY token tile: each Wg byte is read
// from shared memory once per CTA (the routing phase is bound by shared-memory wavefronts, not
// by the HMMAs). The KP partial tables of an expert tile meet in shared memory (fixed kp order),
// and each (expert tile, token tile) table goes into every CTA of the cluster (its own included)
// with st.async (mbarrier complete_tx: no cluster barrier, no fence), transposed to
// [token][expert]. The top-k adds the cl tables in rank order, so every CTA of every cluster
// holds the same logits. Without a cluster the four chunks stream through nbuf buffers.
// Layout behind the chunk buffers: the per-rank tables [cl][8 ceil(T / 8) tokens][Ep16 + 4], the K-part
// scratch [16 warps][ceil(T / 8) token tiles][32 lanes][4].
struct DecRouteGeom {
    int Ep, Ep16, tp, cl, tt;
    __host__ __device__ DecRouteGeom(int E, int cl_, int T) {
        Ep = (E + 7) & ~7;
        Ep16 = (E + 15) & ~15;
        tp = Ep16 + 4;  // 16 B row skew
        cl = cl_;
        tt = (T + 7) >> 3;  // token tiles
    }
    __host__ __device__ size_t tab() const { return size_t(tt) * 8 * tp; }
    __host__ __device__ size_t pair_off() const { return size_t(cl) * tab(); }
    __host__ __device__ size_t lg_off() const { return pair_off() + size_t(16) * tt * 32 * 4; }
    __host__ __device__ size_t floats() const { return lg_off() + size_t(tt) * 8 * tp; }
};

__device__ __forceinline__ void st_async_f32(uint32_t addr, float x, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr),
                 "r"(__float_as_uint(x)), "r"(bar)
                 : "memory");
}

template <int BITS>
__device__ __forceinline__ void dec_fused_route(const DecArgs& a, unsigned char* hs, int hpitch, unsigned char* rbase,
                                                int nbuf, float* lg, uint64_t* rbar, int warp, int lane) {
    const int T = a.T, E = a.E, Kp1 = a.Kp1;
    const int cl = int(cluster_nctas()), crank = int(cta_rank());
    const DecRouteGeom G(E, cl, T);
    const int Ep = G.Ep, Ep16 = G.Ep16;
    const int Kc = Kp1 / 4, cpitch = (Kc + 8) * 2, nsteps = Kc / 16;
    const uint32_t cbytes = uint32_t(2 * Ep) * cpitch;
    const int tid = threadIdx.x, g = lane >> 2, t = lane & 3;
    constexpr int NW = kF1Warps + kF2Warps;  // compute warps (16)
    const int mtiles = Ep16 / 16, ttiles = (T + 7) >> 3, items = mtiles * ttiles;
    const int KP = NW / mtiles;  // K parts per expert tile (E <= 256: mtiles <= 16)
    const int mt = warp % mtiles, kp = warp / mtiles;
    const bool mma_warp = warp < mtiles * KP;
    if (tid == 0) mbar_arrive_expect_tx(rbar + 5, uint32_t(cl) * items * 128 * 4);
    int rtr = 0;
    const int rk = blockIdx.x < 8 ? int(blockIdx.x) : 7;
    if (blockIdx.x < 8) route_trace(a, rk, rtr, 30);
    const int cpr = 4 / cl;  // K chunks of this CTA
    const int c_begin = crank * cpr, c_end = c_begin + cpr;
    float acc[4][2][4];  // [token tile][hi, lo][4]
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[x][h2][i] = 0.f;
    const unsigned char* br[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) br[x] = hs + size_t(min(x * 8 + g, T - 1)) * hpitch + 4 * t;
    for (int c = c_begin; c < c_end; ++c) {
        const int bi = cl > 1 ? c - c_begin : c % nbuf;
        const unsigned char* buf = rbase + size_t(bi) * cbytes;
        mbar_wait(rbar + bi, cl > 1 ? 0 : (c / nbuf) & 1);
#ifdef DEC_PLAN_TRACE
        if (blockIdx.x < 8 && c == c_begin) route_trace(a, rk, rtr, 41);
#endif
        if (mma_warp) {
            const unsigned char* ar = buf + size_t(mt * 16 + g) * cpitch + 4 * t;
            const int gs0 = (c - c_begin) * nsteps;  // K steps are dealt round-robin over the kp warps
            for (int st = ((kp - gs0) % KP + KP) % KP; st < nsteps; st += KP) {
                const int kk = st * 16;
                uint32_t af[2][4];
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    const unsigned char* aa = ar + size_t(h2 * Ep) * cpitch + kk * 2;
                    af[h2][0] = *reinterpret_cast<const uint32_t*>(aa);
                    af[h2][1] = *reinterpret_cast<const uint32_t*>(aa + 8 * cpitch);
                    af[h2][2] = *reinterpret_cast<const uint32_t*>(aa + 16);
                    af[h2][3] = *reinterpret_cast<const uint32_t*>(aa + 8 * cpitch + 16);
                }
                const int ko = (c * Kc + kk) * 2;
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    if (x < ttiles) {
                        const uint32_t b0 = *reinterpret_cast<const uint32_t*>(br[x] + ko);
                        const uint32_t b1 = *reinterpret_cast<const uint32_t*>(br[x] + ko + 16);
#pragma unroll
                        for (int h2 = 0; h2 < 2; ++h2)
                            mma_16816(acc[x][h2], af[h2][0], af[h2][1], af[h2][2], af[h2][3], b0, b1);
                    }
                }
            }
        }
        if (cl == 1 && c + nbuf < 4) {
            __syncthreads();  // buffer bi is free again
            if (tid == 0) {
                mbar_arrive_expect_tx(rbar + bi, cbytes);
                bulk_g2s(const_cast<unsigned char*>(buf), reinterpret_cast<const unsigned char*>(a.wgt) + size_t(c + nbuf) * cbytes,
                         cbytes, rbar + bi);
            }
        }
    }
#ifdef DEC_PLAN_TRACE
    if (blockIdx.x < 8) route_trace(a, rk, rtr, 40);
#endif
    // the K parts of each expert tile meet in shared memory (kp order), then each table goes to
    // every CTA of the cluster
    float* pair = lg + G.pair_off();  // [NW][token tiles][32 lanes][4]
    if (mma_warp) {
#pragma unroll
        for (int x = 0; x < 4; ++x)
            if (x < ttiles)
                reinterpret_cast<float4*>(pair)[(warp * ttiles + x) * 32 + lane] =
                    make_float4(acc[x][0][0] + acc[x][1][0], acc[x][0][1] + acc[x][1][1], acc[x][0][2] + acc[x][1][2],
                                acc[x][0][3] + acc[x][1][3]);
    }
    if (cl > 1) cluster_wait_acquire();  // the peers' barriers are initialised (arrived at kernel start)
    __syncthreads();
    float* recv = lg;  // [cl][8 ceil(T / 8) tokens][tp]
    for (int it = warp; it < items; it += kDecFfnWarps) {
        const int imt = it % mtiles, x = it / mtiles;
        float4 v = reinterpret_cast<const float4*>(pair)[(imt * ttiles + x) * 32 + lane];
        for (int q = 1; q < KP; ++q) {
            const float4 o = reinterpret_cast<const float4*>(pair)[((q * mtiles + imt) * ttiles + x) * 32 + lane];
            v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
        }
        // c0, c1: expert imt*16+g, tokens x*8+2t, +1; c2, c3: expert + 8
        const int e0 = imt * 16 + g, tk0 = x * 8 + 2 * t;
        float* tb = recv + size_t(crank) * G.tab();
        for (int r = 0; r < cl; ++r) {
            const uint32_t bar = map_rank(rbar + 5, uint32_t(r));
            st_async_f32(map_rank(tb + tk0 * G.tp + e0, uint32_t(r)), v.x, bar);
            st_async_f32(map_rank(tb + (tk0 + 1) * G.tp + e0, uint32_t(r)), v.y, bar);
            st_async_f32(map_rank(tb + tk0 * G.tp + e0 + 8, uint32_t(r)), v.z, bar);
            st_async_f32(map_rank(tb + (tk0 + 1) * G.tp + e0 + 8, uint32_t(r)), v.w, bar);
        }
    }
#ifdef DEC_PLAN_TRACE
    if (blockIdx.x < 8) route_trace(a, rk, rtr, 42);
#endif
    mbar_wait(rbar + 5, 0);
    // the logits, once: the cl tables in rank order, then the exact 2^-sw scale
    {
        const float unscale = __int_as_float((127 - a.wg_shift) << 23);
        float* lgt = lg + G.lg_off();  // [8 ceil(T / 8) tokens][tp]
        for (int i = threadIdx.x; i < T * E; i += blockDim.x) {
            const int tk = i / E, e = i - tk * E;
            float v = recv[size_t(tk) * G.tp + e];
            for (int r = 1; r < cl; ++r) v += recv[size_t(r) * G.tab() + size_t(tk) * G.tp + e];
            lgt[size_t(tk) * G.tp + e] = v * unscale;
        }
    }
    __syncthreads();
    if (blockIdx.x < 8) route_trace(a, rk, rtr, 32);
}

// Top-k, gates and the plan from the logit tables (every CTA computes the same plan),
// and the activation rows scaled in place by 2^-s(k) (the fc1 weight field shifts) with the
// per-token correction Z (see unpack_chunk_raw).
//
// Top-k: 8 lanes per token on the assembled logits (one load per logit); each lane
// scans its experts ascending with strict '>', then shuffle max (value) and min (index among
// the lanes holding the max) give the reference's argmax semantics (model.cpp:339-341: ties -> lowest index, NaN skipped unless it sits at the
// scan's first index). Gates in fp32 (expf is within 2 ulp; the logits already differ from the
// reference's in the last bits).
// Plan (the producer warp, while the other warps scale the rows; it then streams its first
// slices without waiting for the rows): lane l owns rows l and l + 32 (row =
// token * k + slot). Equal-expert masks come from ten ballots per half (expert bits + a unique
// tag for empty rows), giving each row's stable rank and its expert's count; experts are
// ordered by their first row, and one shuffle scan over those first rows yields row offsets and
// unit bases (units of <= 16 rows).
template <int BITS>
__device__ __forceinline__ void dec_fused_decide(const DecArgs& a, DecPlanSmem& P, unsigned char* hs, int hpitch,
                                                 const float* lg, uint64_t* rbar6, int warp, int lane) {
    const int T = a.T, E = a.E, K = a.topk, R = T * K, Kp1 = a.Kp1;
    const int cl = int(cluster_nctas());
    const DecRouteGeom G(E, cl, T);
    int rtr = 8;
    const int rk = blockIdx.x < 8 ? int(blockIdx.x) : 7;
    {
        // 8 lanes per token; lane sub scans experts [sub * EPL, (sub + 1) * EPL) ascending
        const int sub = lane & 7, EPL = G.Ep16 / 8, e_lo = sub * EPL, e_hi = min(E, e_lo + EPL);
        const float* lgt = lg + G.lg_off();
        auto logit = [&](int tk, int e) { return lgt[size_t(tk) * G.tp + e]; };
        for (int tb = warp * 4; tb < T; tb += kDecFfnWarps * 4) {  // warp-uniform trip count
            const bool live = tb + (lane >> 3) < T;
            const int tk = live ? tb + (lane >> 3) : T - 1;  // idle groups redo the last token
            int best[2] = {0, 0};
            float mx0 = 0.f;
#pragma unroll
            for (int slot = 0; slot < 2; ++slot) {
                if (slot == 1 && K == 1) break;
                const int skip = slot == 0 ? -1 : best[0];
                const int first = skip == 0 ? 1 : 0;
                float bv = -__int_as_float(0x7f800000);
                int bi = 1 << 30;
                for (int e = e_lo; e < e_hi; ++e) {  // ascending, strict '>': lowest index per lane
                    const float v = logit(tk, e);
                    if (e == skip || v != v) continue;
                    if (bi == (1 << 30) || v > bv) { bv = v; bi = e; }
                }
                float m = bv;
#pragma unroll
                for (int o = 4; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                unsigned bmin = bi != (1 << 30) && bv == m ? unsigned(bi) : 0xffffffffu;
#pragma unroll
                for (int o = 4; o; o >>= 1) bmin = min(bmin, __shfl_xor_sync(0xffffffffu, bmin, o));
                const float lf = logit(tk, first);
                best[slot] = (lf != lf) ? first : (bmin == 0xffffffffu ? first : int(bmin));
                if (slot == 0) mx0 = m;
            }
            float g1 = 1.f, g2 = 0.f;
#ifdef DEC_PLAN_TRACE
            if (blockIdx.x < 8) route_trace(a, rk, rtr, 44);
#endif
            if (K == 1) {
                const float mx = mx0;  // = fmaxf over every logit (fmaxf drops NaNs)
                float sm = 0.f;
                for (int e = e_lo; e < e_hi; ++e) sm += expf(logit(tk, e) - mx);
#pragma unroll
                for (int o = 4; o; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
                g1 = expf(logit(tk, best[0]) - mx) / sm;
            } else {
                const float z = expf(logit(tk, best[1]) - logit(tk, best[0]));
                g1 = 1.f / (1.f + z);
                g2 = z / (1.f + z);
            }
#ifdef DEC_PLAN_TRACE
            if (blockIdx.x < 8) route_trace(a, rk, rtr, 46);
#endif
            if (sub == 0 && live) {
                P.ch_e[tk * K] = best[0];
                P.ch_g[tk * K] = g1;
                if (K == 2) {
                    P.ch_e[tk * K + 1] = best[1];
                    P.ch_g[tk * K + 1] = g2;
                }
                if (blockIdx.x == 0) {
                    a.expert[tk * K] = best[0];
                    a.gate[tk * K] = g1;
                    if (K == 2) {
                        a.expert[tk * K + 1] = best[1];
                        a.gate[tk * K + 1] = g2;
                    }
                }
            }
        }
    }
    __syncthreads();
    if (blockIdx.x < 8) route_trace(a, rk, rtr, 33);
#ifdef DEC_PLAN_TRACE
    if (blockIdx.x < 8) route_trace(a, rk, rtr, 47);
#endif
    if (warp == kF1Warps + kF2Warps) {  // the producer warp: it needs the plan first
        int ee[2];
        float gg[2];
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
            const int row = lane + 32 * hb;
            const bool ok = row < R;
            ee[hb] = ok ? P.ch_e[row] : (0x200 | row);  // empty rows: unique tags >= 512
            gg[hb] = ok ? P.ch_g[row] : 0.f;
        }
        // equal-expert masks: m[x][y] = lanes of half y whose row has the expert of my row in half x
        unsigned m00 = 0xffffffffu, m01 = 0xffffffffu, m10 = 0xffffffffu, m11 = 0xffffffffu;
#pragma unroll
        for (int b = 0; b < 10; ++b) {
            const unsigned ba = __ballot_sync(0xffffffffu, (ee[0] >> b) & 1);
            const unsigned bb = __ballot_sync(0xffffffffu, (ee[1] >> b) & 1);
            const bool xa = (ee[0] >> b) & 1, xb = (ee[1] >> b) & 1;
            m00 &= xa ? ba : ~ba;
            m01 &= xa ? bb : ~bb;
            m10 &= xb ? ba : ~ba;
            m11 &= xb ? bb : ~bb;
        }
        const unsigned ltm = (1u << lane) - 1u;
        const int rank0 = __popc(m00 & ltm), rank1 = __popc(m10) + __popc(m11 & ltm);
        const bool first0 = lane < R && (m00 & ltm) == 0;
        const bool first1 = lane + 32 < R && m10 == 0 && (m11 & ltm) == 0;
        const int cnt0 = __popc(m00) + __popc(m01), cnt1 = __popc(m11);  // first rows only
        // (rows, units) of each expert at its first row, packed: rows | units << 16
        const int v0 = first0 ? (cnt0 | (((cnt0 + kDecPlanRows - 1) / kDecPlanRows) << 16)) : 0;
        const int v1 = first1 ? (cnt1 | (((cnt1 + kDecPlanRows - 1) / kDecPlanRows) << 16)) : 0;
        int i0 = v0, i1 = v1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u0 = __shfl_up_sync(0xffffffffu, i0, o), u1 = __shfl_up_sync(0xffffffffu, i1, o);
            if (lane >= o) { i0 += u0; i1 += u1; }
        }
        const int tot0 = __shfl_sync(0xffffffffu, i0, 31);
        const int x0 = i0 - v0, x1 = i1 - v1 + tot0;  // exclusive (rows | units << 16)
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
            const bool fr = hb == 0 ? first0 : first1;
            if (fr) {
                const int x = hb == 0 ? x0 : x1, c = hb == 0 ? cnt0 : cnt1, e = ee[hb];
                for (int q = 0; q * kDecPlanRows < c; ++q)
                    P.units[(x >> 16) + q] =
                        make_int4(e, (x & 0xFFFF) + q * kDecPlanRows, min(kDecPlanRows, c - q * kDecPlanRows), 0);
            }
        }
        // row positions: offset of the expert's first row + rank
        const int f0 = __ffs(m00) - 1;
        const int f1 = m10 ? __ffs(m10) - 1 : __ffs(m11) - 1;
        const int o00 = __shfl_sync(0xffffffffu, x0, f0 & 31);
        const int o10 = __shfl_sync(0xffffffffu, x0, f1 & 31), o11 = __shfl_sync(0xffffffffu, x1, f1 & 31);
        if (lane < R) {
            const int ps = (o00 & 0xFFFF) + rank0;
            P.perm_token[ps] = K == 2 ? lane >> 1 : lane;
            P.perm_gate[ps] = gg[0];
            P.row_of[lane] = ps;
        }
        if (lane + 32 < R) {
            const int ps = ((m10 ? o10 : o11) & 0xFFFF) + rank1;
            P.perm_token[ps] = K == 2 ? (lane + 32) >> 1 : lane + 32;
            P.perm_gate[ps] = gg[1];
            P.row_of[lane + 32] = ps;
        }
        if (lane == 31) P.n_units = (i1 + tot0) >> 16;
        if (blockIdx.x < 8) route_trace(a, rk, rtr, 34);
    } else {
        // activation rows scaled in place by 2^-s(k) (HMUL2 by a power of two: the same
        // rounding as scaling in fp32 and converting) + Z per token (warps 1..), once the rest of
        // each row (outside this CTA's routing K range) has landed
        if (a.h_f16 && (a.d % 8 == 0) && ((reinterpret_cast<uintptr_t>(a.h) & 15) == 0)) mbar_wait(rbar6, 0);
        constexpr int bias = 1 << (BITS - 1);
        for (int tk = warp; tk < T; tk += kDecFfnWarps - 1) {  // warps 0-15 (and 17-19)
            unsigned char* row = hs + size_t(tk) * hpitch;
            float zf = 0.f;
            for (int k0 = lane * 8; k0 < Kp1; k0 += 256) {
                uint4 q = *reinterpret_cast<const uint4*>(row + k0 * 2);
                __half2* hp = reinterpret_cast<__half2*>(&q);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int sh = field_shift_c<BITS>((k0 + 2 * e) & 15);
                    hp[e] = __hmul2(hp[e], __half2half2(__ushort_as_half(uint16_t((15 - sh) << 10))));
                    const float2 f = __half22float2(hp[e]);
                    const float m = 1024.f + float(bias << sh);  // exact; products of 11-bit factors
                    zf = fmaf(m, f.x, zf);
                    zf = fmaf(m, f.y, zf);
                }
                *reinterpret_cast<uint4*>(row + k0 * 2) = q;
            }
            double z = zf;
#pragma unroll
            for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
            if (lane == 0) P.z[tk] = float(z);
        }
    }
    // the plan (producer warp) and the scaled rows (the others) meet at barrier 7; the producer
    // only arrives, so it starts streaming its first slices while the rows are still scaled
    if (warp == kF1Warps + kF2Warps) {
        __syncwarp();
        asm volatile("bar.arrive 7, %0;" ::"r"(kDecFfnWarps * 32) : "memory");
    } else {
        named_bar_sync(7, kDecFfnWarps * 32);
    }
    if (blockIdx.x < 8) route_trace(a, rk, rtr, 35);
}

// Warp-specialised stream-K decode FFN. Warps 0-7 (fc1) and 8-15 (fc2) work on different
// slices at once: fc1 of slice n+1 overlaps fc2 of slice n through a double-buffered mid.
// QN = Kp1 / 256, GQ = Np2 / 256, NP = pieces per weight part (2 for int8: smaller stages).
// FU: routing fused in (dec_fused_route, T <= 32); else the plan and the permuted scaled rows
// come from k_dec_route (global).
template <int BITS, int QN, int GQ, int NP, bool FU>
__global__ void __launch_bounds__(kDecFfnWarps * 32, 1) k_dec(const DecArgs a) {
    constexpr int RB = DecGeom<BITS>::RB;
    constexpr int Kt = 4 * QN;          // fc1 k-tiles
    constexpr int KP = Kt / NP;         // k-tiles per W1 piece
    constexpr int QW = 2 * GQ;          // fc2 groups per warp (Np2 / 16 / kF2Warps)
    constexpr int KH = KP / 2;          // k-tiles per fc1 warp per piece
    constexpr int WPP = kF2Warps / NP;  // fc2 warps per W2 piece
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int S = a.S, Np2 = a.Np2, d = a.d;
    const uint32_t sb1 = a.stage_bytes, sb2 = a.stage2_bytes;
    const int n1 = a.n_stages, n2 = a.n_stages2;
    unsigned char* ring1 = smem;
    unsigned char* ring2 = ring1 + size_t(n1) * sb1;
    unsigned char* xsb = ring2 + size_t(n2) * sb2;  // FU: hs [T][hpitch]; else 2 x [16 rows][xpitch]
    const int xregion = FU ? ((a.T * a.xpitch + 127) & ~127) : 2 * kDecUnitRows * a.xpitch;
    unsigned char* midb = xsb + xregion;                                          // 2 x [16][kMidPitch]
    float* z2b = reinterpret_cast<float*>(midb + 2 * kDecUnitRows * kMidPitch);  // [2][4 warps][16 cols]
    float* redb = z2b + 2 * 64;                                                  // [2][4 groups][32][8]
    DecPlanSmem* PS = reinterpret_cast<DecPlanSmem*>(redb + 2 * 4 * 32 * 8);
    uint64_t* full1 = reinterpret_cast<uint64_t*>(PS + 1);
    uint64_t* empty1 = full1 + n1;
    uint64_t* full2 = empty1 + n1;
    uint64_t* empty2 = full2 + n2;
    uint64_t* xfull = empty2 + n2;
    uint64_t* xempty = xfull + 2;
    uint64_t* mfull = xempty + 2;
    uint64_t* mempty = mfull + 2;
    uint64_t* rbar = mempty + 2;  // [4] routing Wg chunks, [4] activation rows
    int* flag = reinterpret_cast<int*>(rbar + 8);
    int* comb = flag + 2;  // [kDecUnitRows] tokens to combine (top-2)

    if (tid == 0) {
        for (int s = 0; s < n1; ++s) {
            mbar_init(full1 + s, 1);
            mbar_init(empty1 + s, kF1Warps);
        }
        for (int s = 0; s < n2; ++s) {
            mbar_init(full2 + s, 1);
            mbar_init(empty2 + s, WPP);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(xfull + b, 1);
            mbar_init(xempty + b, kF1Warps);
            mbar_init(mfull + b, kF1Warps / 2);  // the epilogue warps (kh = 0)
            mbar_init(mempty + b, kF2Warps);
        }
        for (int b = 0; b < 8; ++b) mbar_init(rbar + b, 1);
        fence_barrier_init();
    }
    __syncthreads();
    // the cluster's barrier inits are published before any peer pushes logits (the matching
    // wait sits in dec_fused_route, long after this arrive)
    if (FU && cluster_nctas() > 1) cluster_arrive_relaxed();
    // fused routing: gate-weight chunks that fit in the rings (bank constants: before the PDL wait)
    const int Ep_ = (a.E + 7) & ~7;
    const uint32_t cbytes_ = uint32_t(2 * Ep_) * ((a.Kp1 / 4 + 8) * 2);
    const int nbuf_ = FU ? a.route_nbuf : 1;
    if (FU && tid == 0) {
        const int cl = int(cluster_nctas());
        if (cl > 1) {  // this CTA's K chunks only
            const int cpr = 4 / cl, c0 = int(cta_rank()) * cpr;
            for (int i = 0; i < cpr; ++i) {
                mbar_arrive_expect_tx(rbar + i, cbytes_);
                bulk_g2s(ring1 + size_t(i) * cbytes_, reinterpret_cast<const unsigned char*>(a.wgt) + size_t(c0 + i) * cbytes_,
                         cbytes_, rbar + i);
            }
        } else {
            for (int c = 0; c < nbuf_; ++c) {
                mbar_arrive_expect_tx(rbar + c, cbytes_);
                bulk_g2s(ring1 + size_t(c) * cbytes_, reinterpret_cast<const unsigned char*>(a.wgt) + size_t(c) * cbytes_,
                         cbytes_, rbar + c);
            }
        }
    }
    pdl_trigger();
    pdl_wait();
    if (tid == 0) span_begin(a.span_ffn);
    if (a.trace && tid == 0) {  // slot 63: this CTA's start after the PDL wait
        unsigned long long* p = a.trace + (size_t(blockIdx.x) * kDecTrace + 63) * 2;
        p[0] = 20u;
        p[1] = gtime_ns();
    }
    int rtr0 = 0;
    if (FU && blockIdx.x < 8) route_trace(a, blockIdx.x, rtr0, 28);
    if constexpr (FU) {
        // activation rows -> hs (one bulk copy per row), zero padding columns / rows
        const int T = a.T;
        const bool bulk = a.h_f16 && (d % 8 == 0) && ((reinterpret_cast<uintptr_t>(a.h) & 15) == 0);
        if (bulk && warp == 0) {  // one row per lane
            // this CTA's K range of the routing logits first (rbar 4, waited for below), the rest of
            // each row behind it (rbar 6, waited for by the row scaling in dec_fused_decide)
            const int cl = int(cluster_nctas());
            int k_lo = 0, k_hi = d;
            if (cl > 1) {
                const int span = (4 / cl) * (a.Kp1 / 4);
                k_lo = min(d, int(cta_rank()) * span);
                k_hi = min(d, k_lo + span);
            }
            if (lane == 0) {
                mbar_arrive_expect_tx(rbar + 4, uint32_t(T) * (k_hi - k_lo) * 2);
                mbar_arrive_expect_tx(rbar + 6, uint32_t(T) * (d - (k_hi - k_lo)) * 2);
            }
            __syncwarp();
            const __half* hh = static_cast<const __half*>(a.h);
            for (int r = lane; r < T; r += 32)
                if (k_hi > k_lo)
                    bulk_g2s(xsb + size_t(r) * a.xpitch + k_lo * 2, hh + size_t(r) * d + k_lo, (k_hi - k_lo) * 2, rbar + 4);
            for (int r = lane; r < T; r += 32) {
                if (k_lo > 0) bulk_g2s(xsb + size_t(r) * a.xpitch, hh + size_t(r) * d, k_lo * 2, rbar + 6);
                if (k_hi < d)
                    bulk_g2s(xsb + size_t(r) * a.xpitch + k_hi * 2, hh + size_t(r) * d + k_hi, (d - k_hi) * 2, rbar + 6);
            }
        }
        if (!bulk) {
            for (int i = tid; i < T * d; i += blockDim.x) {
                const int r = i / d, k = i - r * d;
                const float v = a.h_f16 ? __half2float(static_cast<const __half*>(a.h)[i]) : static_cast<const float*>(a.h)[i];
                reinterpret_cast<__half*>(xsb + size_t(r) * a.xpitch)[k] = __float2half_rn(v);
            }
        }
        for (int i = tid; i < T * (a.Kp1 - d); i += blockDim.x) {
            const int r = i / (a.Kp1 - d), k = d + i % (a.Kp1 - d);
            reinterpret_cast<__half*>(xsb + size_t(r) * a.xpitch)[k] = __float2half_rn(0.f);
        }
        if (bulk) mbar_wait(rbar + 4, 0);
        __syncthreads();
        if (blockIdx.x < 8) route_trace(a, blockIdx.x, rtr0, 29);
        float* lg = reinterpret_cast<float*>(ring1 + size_t(nbuf_) * cbytes_);
        // one instantiation (two token m-tiles) keeps the kernel's instruction footprint small
        dec_fused_route<BITS>(a, xsb, a.xpitch, ring1, nbuf_, lg, rbar, warp, lane);
        dec_fused_decide<BITS>(a, *PS, xsb, a.xpitch, lg, rbar + 6, warp, lane);
    }
    const int4* units = FU ? PS->units : a.units;
    const int* perm_token = FU ? PS->perm_token : a.perm_token;
    const float* perm_gate = FU ? PS->perm_gate : a.perm_gate;
    const int* row_of = FU ? PS->row_of : a.row_of;
    const int U = FU ? PS->n_units : *a.n_units;
    const int W = U * S;
    const int w0 = int((long long)W * blockIdx.x / gridDim.x), w1 = int((long long)W * (blockIdx.x + 1) / gridDim.x);
    const int u0 = w0 / S, j0 = w0 - u0 * S;
#if DEC_SETMAXNREG
    if (warp >= kF1Warps + kF2Warps) {  // warpgroup 4: hand registers to the math warpgroups
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kDecProdRegs));
        if (warp != kF1Warps + kF2Warps) return;
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kDecMathRegs));
    }
#endif

    if (warp == kF1Warps + kF2Warps) {
        // ------------------------------ producer ------------------------------
        if (lane == 0 && w0 < w1) {
            const uint64_t pol = policy_evict_first();
            int s1 = 0, s2 = 0, nu = 0, ntr = 0;
            uint32_t p1 = 0, p2 = 0;
            int u = u0, j = j0;
            int4 un = units[u];
            for (int w = w0; w < w1; ++w) {
                if (w == w0 || j == 0) {
                    if (w != w0) un = units[u];
                    if (!FU) {
                        const int b = nu & 1;
                        mbar_wait(xempty + b, ((nu >> 1) & 1) ^ 1);
                        const uint32_t xb = uint32_t(un.z) * a.xpitch;
                        mbar_arrive_expect_tx(xfull + b, xb);
                        bulk_g2s(xsb + size_t(b) * kDecUnitRows * a.xpitch,
                                 reinterpret_cast<const unsigned char*>(a.xperm) + size_t(un.y) * a.xpitch, xb, xfull + b);
                    }
                    ++nu;
                }
                const uint8_t* sl = a.wdec + size_t(un.x) * a.wdec_stride + size_t(j) * a.slice_bytes;
                dec_trace(a, 42, ntr, 10);
#pragma unroll
                for (int p = 0; p < NP; ++p) {  // W1 pieces; the last one carries the slice's s1 / b1
                    const uint32_t bytes = uint32_t(KP) * 64 * RB;
                    const uint32_t extra = p == NP - 1 ? (a.b1 ? 512u : 256u) : 0u;
                    mbar_wait(empty1 + s1, p1 ^ 1);
                    mbar_arrive_expect_tx(full1 + s1, bytes + extra);
                    unsigned char* dst = ring1 + size_t(s1) * sb1;
                    bulk_g2s_hint(dst, sl + size_t(p) * bytes, bytes, full1 + s1, pol);
                    if (p == NP - 1) {
                        bulk_g2s(dst + sb1 - 512, a.s1 + size_t(un.x) * a.Np1 + j * 64, 256u, full1 + s1);
                        if (a.b1) bulk_g2s(dst + sb1 - 256, a.b1 + size_t(un.x) * a.Np1 + j * 64, 256u, full1 + s1);
                    }
                    if (++s1 == n1) { s1 = 0; p1 ^= 1; }
                }
                dec_trace(a, 42, ntr, 11);
#pragma unroll
                for (int p = 0; p < NP; ++p) {  // W2 pieces
                    const uint32_t bytes = uint32_t(Np2 / NP) * RB;
                    mbar_wait(empty2 + s2, p2 ^ 1);
                    mbar_arrive_expect_tx(full2 + s2, bytes);
                    bulk_g2s_hint(ring2 + size_t(s2) * sb2, sl + size_t(Kt) * 64 * RB + size_t(p) * bytes, bytes,
                                  full2 + s2, pol);
                    if (++s2 == n2) { s2 = 0; p2 ^= 1; }
                }
                if (++j == S) { j = 0; ++u; }
            }
        }
        return;
    }

    // roles by SM sub-partition (warp % 4): fc1 on SMSPs 0-1, fc2 on SMSPs 2-3, so each
    // sub-partition's L0 instruction cache (~6 KB) holds one role's unrolled loop
#if DEC_ROLE_SPLIT
    const bool is_f1 = (warp & 2) == 0;
    const int rix = (warp >> 2) * 2 + (warp & 1);  // index within the role, 0..7
#else
    const bool is_f1 = warp < kF1Warps;
    const int rix = is_f1 ? warp : warp - kF1Warps;
#endif
    if (is_f1) {
        // ------------------------------ fc1 warps ------------------------------
        const int gw = rix & 3, kh = rix >> 2;
        int s1 = 0, nu = 0, n = 0, ntr = 0;
        uint32_t p1 = 0;
        int u = u0, j = j0;
        int4 un = units[u];
        const unsigned char* xrow[2] = {xsb, xsb};
        float zc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};  // Z of this lane's epilogue columns
        const bool has_b1 = a.b1 != nullptr;
        for (int w = w0; w < w1; ++w, ++n) {
            if (w == w0 || j == 0) {
                if (w != w0) un = units[u];
                if (FU) {
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb) {
                        const int r = nb * 8 + g;
                        xrow[nb] = xsb + size_t(perm_token[un.y + (r < un.z ? r : 0)]) * a.xpitch;
#pragma unroll
                        for (int lo = 0; lo < 2; ++lo) {
                            const int col = nb * 8 + 2 * t + lo;
                            zc[nb][lo] = col < un.z ? PS->z[perm_token[un.y + col]] : 0.f;
                        }
                    }
                } else {
                    const int b = nu & 1;
                    const unsigned char* xs = xsb + size_t(b) * kDecUnitRows * a.xpitch;
                    mbar_wait(xfull + b, (nu >> 1) & 1);
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb) {
                        xrow[nb] = xs + (nb * 8 + g) * a.xpitch;
#pragma unroll
                        for (int lo = 0; lo < 2; ++lo)
                            zc[nb][lo] = *reinterpret_cast<const float*>(xs + (nb * 8 + 2 * t + lo) * a.xpitch + QN * 512);
                    }
                }
            }
            const int NBr = un.z > 8 ? 2 : 1;
            float ca[2][4], cb[2][4];
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                for (int i = 0; i < 4; ++i) ca[nb][i] = cb[nb][i] = 0.f;
            int sl1 = s1;
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                sl1 = s1;
                mbar_wait(full1 + s1, p1);
                if (lane == 0 && rix == 0) dec_trace(a, 0, ntr, 1);
                const unsigned char* piece = ring1 + size_t(s1) * sb1 + size_t(kh * KH) * 64 * RB;
#ifndef DEC_SKIP_FC1  // timing experiments only (tools/ab_build.sh): results are wrong
                if (NBr == 1) dec_fc1_piece<BITS, KH, 1>(piece, p * KP + kh * KH, gw, g, t, xrow, ca, cb);
                else dec_fc1_piece<BITS, KH, 2>(piece, p * KP + kh * KH, gw, g, t, xrow, ca, cb);
#endif
                if (p < NP - 1 || kh == 1) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty1 + s1);
                }
                if (++s1 == n1) { s1 = 0; p1 ^= 1; }
            }
            // the K halves meet in smem (double-buffered by slice parity): kh = 1 hands over,
            // kh = 0 adds (fixed order) and runs the epilogue
            float* rw = redb + ((n & 1) * 4 + gw) * 32 * 8 + lane * 8;
            if (kh == 1) {
#pragma unroll
                for (int nb = 0; nb < 2; ++nb)
                    if (nb < NBr)
                        *reinterpret_cast<float4*>(rw + nb * 4) =
                            make_float4(ca[nb][0] + cb[nb][0], ca[nb][1] + cb[nb][1], ca[nb][2] + cb[nb][2], ca[nb][3] + cb[nb][3]);
                named_bar_sync(3 + gw, 64);
                if (++j == S) { j = 0; ++u; }
                if (w + 1 == w1 || j == 0) {  // this CTA's run on the unit ends: release its rows
                    if (!FU && lane == 0) mbar_arrive(xempty + (nu & 1));
                    ++nu;
                }
                continue;
            }
            named_bar_sync(3 + gw, 64);
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
                if (nb < NBr) {
                    const float4 o = *reinterpret_cast<const float4*>(rw + nb * 4);
                    ca[nb][0] += cb[nb][0]; ca[nb][1] += cb[nb][1]; ca[nb][2] += cb[nb][2]; ca[nb][3] += cb[nb][3];
                    cb[nb][0] = o.x; cb[nb][1] = o.y; cb[nb][2] = o.z; cb[nb][3] = o.w;
                }
            // epilogue: (acc - Z) * s1 + b1 -> ReLU -> fp16 mid[n & 1]
            const int mb = n & 1;
            mbar_wait(mempty + mb, ((n >> 1) & 1) ^ 1);
            unsigned char* mid = midb + mb * kDecUnitRows * kMidPitch;
            const unsigned char* last = ring1 + size_t(sl1) * sb1;
            const float* sc1 = reinterpret_cast<const float*>(last + sb1 - 512);
            const float* bi1 = reinterpret_cast<const float*>(last + sb1 - 256);
#pragma unroll
            for (int nb = 0; nb < 2; ++nb) {
                if (nb < NBr) {
#pragma unroll
                    for (int hi = 0; hi < 2; ++hi) {
                        const int ch = gw * 16 + g + 8 * hi;
                        const float sc = sc1[ch], bi = has_b1 ? bi1[ch] : 0.f;
#pragma unroll
                        for (int lo = 0; lo < 2; ++lo) {
                            const int i = hi * 2 + lo;
                            float v = ((ca[nb][i] + cb[nb][i]) - zc[nb][lo]) * sc + bi;
                            v = v > 0.f ? v : 0.f;  // ReLU (model.cpp:189-191)
                            *reinterpret_cast<__half*>(mid + (nb * 8 + 2 * t + lo) * kMidPitch + ch * 2) = __float2half_rn(v);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(mfull + mb);
                mbar_arrive(empty1 + sl1);  // last W1 piece (and its scales) consumed
                if (gw == 0) dec_trace(a, 0, ntr, 2);
            }
            if (++j == S) { j = 0; ++u; }
            if (w + 1 == w1 || j == 0) {  // this CTA's run on the unit ends: release its rows
                if (!FU && lane == 0) mbar_arrive(xempty + (nu & 1));
                ++nu;
            }
        }
        return;
    }

    // ------------------------------ fc2 warps ------------------------------
    constexpr int NT2 = kF2Warps * 32;
    const int v = rix, tid2 = rix * 32 + lane;
    const int vp = v / WPP, q0 = (v % WPP) * QW;  // W2 piece of this warp, first group in it
    int s2 = 0, n = 0, ntr = 0;
    uint32_t p2 = 0;
    int u = u0, j = j0;
    int w = w0;
    while (w < w1) {
        // one run: this CTA's consecutive slices of unit u, accumulated in registers
        const int4 un = units[u];
        const int ulo = j, len = min(S - j, w1 - w);
        long long* acc = a.acc + size_t(un.y) * Np2;
        auto wait_slice = [&](int& myst) {
            int st = s2;  // skip the W2 pieces of the other warps, wait for this warp's piece
            uint32_t ph = p2;
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                if (p == vp) { st = s2; ph = p2; }
                if (++s2 == n2) { s2 = 0; p2 ^= 1; }
            }
            myst = st;
            mbar_wait(full2 + st, ph);
            if (tid2 == 0) dec_trace(a, 21, ntr, 3);
            mbar_wait(mfull + (n & 1), (n >> 1) & 1);
            if (tid2 == 0) dec_trace(a, 21, ntr, 4);
        };
        auto release_slice = [&](int myst) {
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(empty2 + myst);
                mbar_arrive(mempty + (n & 1));
            }
        };
        if (un.z <= 8) {
            // <= 8 rows: the run's fc2 partials stay in registers, one flush at the end
            float c2[QW][1][4];
#pragma unroll
            for (int q = 0; q < QW; ++q)
#pragma unroll
                for (int i = 0; i < 4; ++i) c2[q][0][i] = 0.f;
            for (int r = 0; r < len; ++r, ++n) {
                int myst;
                wait_slice(myst);
#ifndef DEC_SKIP_FC2
                dec_fc2_piece<BITS, QW, 1>(ring2 + size_t(myst) * sb2, q0, g, t, midb + (n & 1) * kDecUnitRows * kMidPitch,
                                           c2);
#endif
                release_slice(myst);
            }
#pragma unroll
            for (int q = 0; q < QW; ++q) {
                const int gi = vp * (QW * WPP) + q0 + q;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int col = 2 * t + (i & 1);
                    const int ch = gi * 16 + g + 8 * (i >> 1);
                    if (col < un.z) red_add_s64(acc + size_t(col) * Np2 + ch, __float2ll_rn(c2[q][0][i] * kFix));
                }
            }
        } else {
            // 9..16 rows: flush every slice, QW/2 groups at a time (bounded registers)
            constexpr int QH = QW / 2 > 0 ? QW / 2 : 1;
            for (int r = 0; r < len; ++r, ++n) {
                int myst;
                wait_slice(myst);
#pragma unroll
                for (int hb = 0; hb < QW / QH; ++hb) {
                    float c2[QH][2][4];
#pragma unroll
                    for (int q = 0; q < QH; ++q)
#pragma unroll
                        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                            for (int i = 0; i < 4; ++i) c2[q][nb][i] = 0.f;
                    dec_fc2_piece<BITS, QH, 2>(ring2 + size_t(myst) * sb2, q0 + hb * QH, g, t,
                                               midb + (n & 1) * kDecUnitRows * kMidPitch, c2);
#pragma unroll
                    for (int q = 0; q < QH; ++q) {
                        const int gi = vp * (QW * WPP) + q0 + hb * QH + q;
#pragma unroll
                        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const int col = nb * 8 + 2 * t + (i & 1);
                                const int ch = gi * 16 + g + 8 * (i >> 1);
                                if (col < un.z)
                                    red_add_s64(acc + size_t(col) * Np2 + ch, __float2ll_rn(c2[q][nb][i] * kFix));
                            }
                    }
                }
                release_slice(myst);
            }
        }
        const int uu = u, ju = j + len - 1;
        w += len;
        j += len;
        if (j == S) { j = 0; ++u; }
        if (a.trace && tid2 == 0) {  // slot 60: the run's reds are issued (diagnostics)
            unsigned long long* p = a.trace + (size_t(blockIdx.x) * kDecTrace + 60) * 2;
            p[0] = 7u;
            p[1] = gtime_ns();
        }
        {
            // the fc2 warps' reds are ordered before one acq_rel counter update (bar.sync + the
            // cumulative release of thread 0); the finisher's acquire covers its reads of acc
            named_bar_sync(2, NT2);
            if (tid2 == 0) {
                const unsigned mine = unsigned(ju + 1 - ulo);
                const unsigned old = atom_add_acq_rel(a.unit_done + uu, mine);
                const int fin = old + mine == unsigned(S);
                if (fin) a.unit_done[uu] = 0;
                flag[0] = fin;
            }
            named_bar_sync(2, NT2);
            if (tid2 == 0) dec_trace(a, 21, ntr, 5);
            if (flag[0]) {
                // final epilogue of the unit: y = s2 * acc * 2^-24 + b2, gated (model.cpp:385-390)
                const float* s2p = a.s2 + size_t(un.x) * Np2;
                const float* b2p = a.b2 ? a.b2 + size_t(un.x) * Np2 : nullptr;
                // four channels per thread and step (two 16-byte acc loads in flight): the unit's
                // tail is a chain of L2 round trips under full HBM load, so fewer, wider steps
                const int dq = d >> 2;
                for (int idx = tid2; idx < ((d & 3) ? 0 : un.z * dq); idx += NT2) {
                    const int r = idx / dq, ch = 4 * (idx - r * dq);
                    longlong2* ap = reinterpret_cast<longlong2*>(acc + size_t(r) * Np2 + ch);
                    const longlong2 v0 = __ldcg(ap), v1 = __ldcg(ap + 1);
                    ap[0] = make_longlong2(0, 0);  // self-cleaning for the next forward
                    ap[1] = make_longlong2(0, 0);
                    const float4 sc = *reinterpret_cast<const float4*>(s2p + ch);
                    float y[4] = {float(v0.x) * (1.0f / kFix) * sc.x, float(v0.y) * (1.0f / kFix) * sc.y,
                                  float(v1.x) * (1.0f / kFix) * sc.z, float(v1.y) * (1.0f / kFix) * sc.w};
                    if (b2p) {
                        const float4 bb = *reinterpret_cast<const float4*>(b2p + ch);
                        y[0] = y[0] + bb.x;
                        y[1] = y[1] + bb.y;
                        y[2] = y[2] + bb.z;
                        y[3] = y[3] + bb.w;
                    }
                    const int row = un.y + r;
                    const float gt = perm_gate[row];
                    const float4 g4 = make_float4(gt * y[0], gt * y[1], gt * y[2], gt * y[3]);
                    if (a.topk == 1) {
                        const size_t o = size_t(perm_token[row]) * d + ch;
                        if (a.out_f16) {
                            __half2* op = reinterpret_cast<__half2*>(static_cast<__half*>(a.out) + o);
                            op[0] = __floats2half2_rn(g4.x, g4.y);
                            op[1] = __floats2half2_rn(g4.z, g4.w);
                        } else {
                            *reinterpret_cast<float4*>(static_cast<float*>(a.out) + o) = g4;
                        }
                    } else {
                        *reinterpret_cast<float4*>(a.ybuf + size_t(row) * d + ch) = g4;
                    }
                }
                for (int idx = tid2; idx < ((d & 3) ? un.z * d : 0); idx += NT2) {  // d_model % 4 != 0
                    const int r = idx / d, ch = idx - r * d;
                    long long* ap = acc + size_t(r) * Np2 + ch;
                    const long long vv = __ldcg(ap);
                    *ap = 0;  // self-cleaning for the next forward
                    float y = float(vv) * (1.0f / kFix) * s2p[ch];
                    if (b2p) y = y + b2p[ch];
                    const int row = un.y + r;
                    const float gy = perm_gate[row] * y;
                    if (a.topk == 1) {
                        const size_t o = size_t(perm_token[row]) * d + ch;
                        if (a.out_f16) static_cast<__half*>(a.out)[o] = __float2half_rn(gy);
                        else static_cast<float*>(a.out)[o] = gy;
                    } else {
                        a.ybuf[size_t(row) * d + ch] = gy;
                    }
                }
                if (a.topk == 2) {
                    named_bar_sync(2, NT2);  // ybuf rows written; each token's acq_rel count below
                    if (tid2 < un.z) {      // releases them (cumulative) and acquires the other slot's
                        const int tok = perm_token[un.y + tid2];
                        const unsigned old = atom_add_acq_rel(a.tok_cnt + tok, 1u);
                        comb[tid2] = old == 1 ? tok : -1;
                        if (old == 1) a.tok_cnt[tok] = 0;
                    }
                    named_bar_sync(2, NT2);
                    // four channels per step (16-byte ybuf loads), as the unit epilogue above
                    const int dq = d >> 2;
                    for (int idx = tid2; idx < ((d & 3) ? 0 : un.z * dq); idx += NT2) {
                        const int r = idx / dq, ch = 4 * (idx - r * dq);
                        const int tok = comb[r];
                        if (tok < 0) continue;
                        // o = g0*y0; o = o + g1*y1 (slot order, like the oracle's combine)
                        const float4 y0 = __ldcg(reinterpret_cast<const float4*>(a.ybuf + size_t(row_of[2 * tok]) * d + ch));
                        const float4 y1 = __ldcg(reinterpret_cast<const float4*>(a.ybuf + size_t(row_of[2 * tok + 1]) * d + ch));
                        const float4 o = make_float4(y0.x + y1.x, y0.y + y1.y, y0.z + y1.z, y0.w + y1.w);
                        const size_t oi = size_t(tok) * d + ch;
                        if (a.out_f16) {
                            __half2* op = reinterpret_cast<__half2*>(static_cast<__half*>(a.out) + oi);
                            op[0] = __floats2half2_rn(o.x, o.y);
                            op[1] = __floats2half2_rn(o.z, o.w);
                        } else {
                            *reinterpret_cast<float4*>(static_cast<float*>(a.out) + oi) = o;
                        }
                    }
                    for (int idx = tid2; idx < ((d & 3) ? un.z * d : 0); idx += NT2) {  // d_model % 4 != 0
                        const int r = idx / d, ch = idx - r * d;
                        const int tok = comb[r];
                        if (tok < 0) continue;
                        // o = g0*y0; o = o + g1*y1 (slot order, like the oracle's combine)
                        const float y0 = __ldcg(a.ybuf + size_t(row_of[2 * tok]) * d + ch);
                        const float y1 = __ldcg(a.ybuf + size_t(row_of[2 * tok + 1]) * d + ch);
                        const float o = y0 + y1;
                        const size_t oi = size_t(tok) * d + ch;
                        if (a.out_f16) static_cast<__half*>(a.out)[oi] = __float2half_rn(o);
                        else static_cast<float*>(a.out)[oi] = o;
                    }
                }
                named_bar_sync(2, NT2);
                if (a.trace && tid2 == 0) {  // slot 61: the unit's final epilogue is done
                    unsigned long long* p = a.trace + (size_t(blockIdx.x) * kDecTrace + 61) * 2;
                    p[0] = 8u;
                    p[1] = gtime_ns();
                }
            }
        }
    }
    named_bar_sync(2, NT2);
    if (a.trace && tid2 == 0) {  // slot 62: this CTA's exit
        unsigned long long* p = a.trace + (size_t(blockIdx.x) * kDecTrace + 62) * 2;
        p[0] = 6u;
        p[1] = gtime_ns();
    }
    if (tid2 == 0) span_end(a.span_ffn, gridDim.x);
}

// Mid-size batches: the plan of the batched router + k_scatter (counts, offsets, perm_token)
// becomes k_dec's work list. The last block's warp 0 turns every expert with 0 < rows <=
// gemv_max (path 1: every expert) into units of <= kDecMidUnitRows permuted rows (expert order);
// the other warps write those rows, scaled by 2^-s(k) with the per-row correction Z in the
// 16 bytes after Kp1 (the layout k_dec's non-fused path reads; same arithmetic as
// dec_fused_decide). Top-1 only (one row per token).
template <int BITS>
__global__ void __launch_bounds__(256) k_dec_prep(const void* h, int h_f16, int T, int d, int E, int Kp1, int path,
                                                  int gemv_max, Plan P, int4* units, int* n_units, __half* xperm,
                                                  int xpitch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (blockIdx.x == gridDim.x - 1) {
        if (warp != 0) return;
        int base = 0;
        for (int e0 = 0; e0 < E; e0 += 32) {
            const int e = e0 + lane;
            const int n = e < E ? P.counts[e] : 0;
            const bool sel = n > 0 && (path == 1 || n <= gemv_max);
            const int nu = sel ? (n + kDecMidUnitRows - 1) / kDecMidUnitRows : 0;
            int incl = nu;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (sel) {
                const int off = P.offsets[e];
                for (int q = 0; q < nu; ++q)
                    units[base + incl - nu + q] =
                        make_int4(e, off + q * kDecMidUnitRows, min(kDecMidUnitRows, n - q * kDecMidUnitRows), 0);
            }
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) *n_units = base;
        return;
    }
    const int r = blockIdx.x * 8 + warp;  // permuted row
    if (r >= T) return;
    const int t = P.perm_token[r];
    const int n = P.counts[P.expert[t]];
    if (!(n > 0 && (path == 1 || n <= gemv_max))) return;
    unsigned char* row = reinterpret_cast<unsigned char*>(xperm) + size_t(r) * xpitch;
    constexpr int bias = 1 << (BITS - 1);
    const bool vec = h_f16 && (d % 8) == 0 && ((reinterpret_cast<uintptr_t>(h) & 15) == 0);
    float zf = 0.f;
    for (int k0 = lane * 8; k0 < Kp1; k0 += 256) {
        uint4 q;
        if (vec && k0 < d) {
            q = __ldg(reinterpret_cast<const uint4*>(static_cast<const __half*>(h) + size_t(t) * d + k0));
        } else {
            __half v8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int k = k0 + i;
                const float v = k < d ? (h_f16 ? __half2float(static_cast<const __half*>(h)[size_t(t) * d + k])
                                                : static_cast<const float*>(h)[size_t(t) * d + k])
                                      : 0.f;
                v8[i] = __float2half_rn(v);
            }
            q = *reinterpret_cast<const uint4*>(v8);
        }
        __half2* hp = reinterpret_cast<__half2*>(&q);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int sh = field_shift_c<BITS>((k0 + 2 * e) & 15);
            hp[e] = __hmul2(hp[e], __half2half2(__ushort_as_half(uint16_t((15 - sh) << 10))));
            const float2 f = __half22float2(hp[e]);
            const float m = 1024.f + float(bias << sh);  // exact; products of 11-bit factors
            zf = fmaf(m, f.x, zf);
            zf = fmaf(m, f.y, zf);
        }
        *reinterpret_cast<uint4*>(row + k0 * 2) = q;
    }
    double z = zf;
#pragma unroll
    for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if (lane == 0) *reinterpret_cast<float*>(row + size_t(Kp1) * 2) = float(z);
}

// Bank layout for the decode kernel: per expert, per 64-channel f-slice j, contiguous
// [W1 part: Kp1/64 k-tiles x 64 channel rows][W2 part: Np2/128 x 128 channel rows] of
// tile rows (64 codes each, the codec of codec.cuh), copied from the tiled bank.
__global__ void k_dec_layout(const uint8_t* __restrict__ w1, const uint8_t* __restrict__ w2, int64_t w1_stride,
                             int64_t w2_stride, int Kp1, int Np1, int Np2, int bits, uint8_t* __restrict__ out,
                             int64_t out_stride, int64_t slice_bytes) {
    const int e = blockIdx.z, j = blockIdx.y;
    const int RB = 8 * bits, Kt = Kp1 / 64, Kt2 = Np1 / 64;
    const int tb = 128 * RB;
    const int nblk = Kt + Np2 / 128;  // Kt half-tiles of W1, Np2/128 tiles of W2
    for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
        const uint8_t* src;
        uint8_t* dst = out + size_t(e) * out_stride + size_t(j) * slice_bytes;
        int bytes;
        if (b < Kt) {  // W1 tile (nt = j/2, kb = b), rows (j%2)*64 .. +63
            src = w1 + size_t(e) * w1_stride + (size_t(j / 2) * Kt + b) * tb + (j & 1) * 64 * RB;
            dst += size_t(b) * 64 * RB;
            bytes = 64 * RB;
        } else {  // W2 tile (nt = b - Kt, kb = j)
            const int nt = b - Kt;
            src = w2 + size_t(e) * w2_stride + (size_t(nt) * Kt2 + j) * tb;
            dst += size_t(Kt) * 64 * RB + size_t(nt) * tb;
            bytes = tb;
        }
        for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16)
            *reinterpret_cast<uint4*>(dst + i) = *reinterpret_cast<const uint4*>(src + i);
    }
}

// =====================================================================================
// host side
// =====================================================================================
namespace {
constexpr int kMaxDev = 64;

int route_cluster(int d, int E) {
    return (int64_t(((d + 7) / 8 + 3) & ~3) * E * 4 <= 64 * 1024) ? 8 : 16;
}
size_t route_smem(int T, int d, int E, int C) {
    const int rpc = ((d + C - 1) / C + 3) & ~3;
    const int Tp = (T + 7) & ~7;
    const int ntile = (Tp / 8) * ((E + 31) / 32);
    const int ks = ntile >= 8 ? 1 : (ntile >= 4 ? 2 : (ntile >= 2 ? 4 : 8));
    size_t s = size_t(rpc) * E * 4 + size_t(rpc) * Tp * 4 + size_t(std::max(ks * T * E, 8 * 256)) * 4 +
               size_t(T) * E * 4;
    s += 64 * 4 * 2 + size_t(3 * E + 2 + 64) * 4 + 32;
    return s;
}
}  // namespace

int64_t dec_slice_bytes(int bits, int Kp1, int Np2) { return int64_t(Kp1 + Np2) * 8 * bits; }

bool dec_mid_supported(int d, int E, int Kp1, int Np1, int Np2) {
    return d <= Kp1 && Kp1 <= 1024 && Kp1 % 256 == 0 && Np2 <= 1024 && Np2 % 256 == 0 && Np1 % 64 == 0 && E <= 256;
}

cudaError_t launch_dec_prep(int bits, const void* h, int h_f16, int64_t T, int d, int E, int Kp1, int path,
                            int gemv_max, const Plan& P, int4* units, int* n_units, __half* xperm, int xpitch,
                            cudaStream_t st) {
    const unsigned grid = unsigned((T + 7) / 8 + 1);
    switch (bits) {
        case 2: k_dec_prep<2><<<grid, 256, 0, st>>>(h, h_f16, int(T), d, E, Kp1, path, gemv_max, P, units, n_units, xperm, xpitch); break;
        case 3: k_dec_prep<3><<<grid, 256, 0, st>>>(h, h_f16, int(T), d, E, Kp1, path, gemv_max, P, units, n_units, xperm, xpitch); break;
        case 4: k_dec_prep<4><<<grid, 256, 0, st>>>(h, h_f16, int(T), d, E, Kp1, path, gemv_max, P, units, n_units, xperm, xpitch); break;
        case 8: k_dec_prep<8><<<grid, 256, 0, st>>>(h, h_f16, int(T), d, E, Kp1, path, gemv_max, P, units, n_units, xperm, xpitch); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

bool dec_supported(int64_t T, int topk, int d, int E, int Kp1, int Np1, int Np2) {
    if (T * topk > kDecMaxRows || T < 1) return false;
    // compile-time warp tiling: fc1 k-tiles a multiple of 4 (Kp1 in {256, 512, 768, 1024}),
    // fc2 channel groups a multiple of 16 (Np2 in {256, 512, 768, 1024})
    if (Kp1 > 1024 || Kp1 % 256 || Np2 > 1024 || Np2 % 256 || Np1 % 64 || E > 256) return false;
    const int C = route_cluster(d, E);
    return route_smem(int(T), d, E, C) <= size_t(kMaxRouteSmem);
}

cudaError_t dec_build_layout(const uint8_t* w1, const uint8_t* w2, int64_t w1_stride, int64_t w2_stride, int E,
                             int Kp1, int Np1, int Np2, int bits, uint8_t* out, cudaStream_t st) {
    const int64_t sb = dec_slice_bytes(bits, Kp1, Np2);
    dim3 grid(8, Np1 / 64, E);
    k_dec_layout<<<grid, 256, 0, st>>>(w1, w2, w1_stride, w2_stride, Kp1, Np1, Np2, bits, out, sb * (Np1 / 64), sb);
    return cudaGetLastError();
}

template <int BITS, int QN, int GQ, int NP, bool FU>
static cudaError_t launch_dec_t(const DecArgs& a, cudaStream_t st, int num_sms, size_t smem) {
    static bool configured[kMaxDev] = {};
    static int clusters[kMaxDev][3] = {};  // co-resident clusters of 2 / 4 CTAs (fused routing)
    int dev = 0;
    cudaGetDevice(&dev);
    const int di = dev < kMaxDev ? dev : 0;
    auto kern = k_dec<BITS, QN, GQ, NP, FU>;
    if (!configured[di]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(227 * 1024));
        if (e != cudaSuccess) return e;
        configured[di] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(kDecFfnWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    const int cl = (FU && (a.route_cluster == 2 || a.route_cluster == 4)) ? a.route_cluster : 1;
    attr[1].val.clusterDim.x = unsigned(cl);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    int grid = num_sms;
    if (cl > 1) {
        int& nc = clusters[di][cl / 2];
        if (nc == 0) {
            cudaLaunchConfig_t q = cfg;
            q.gridDim = dim3(unsigned(num_sms / cl * cl));
            q.attrs = attr + 1;
            q.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess || n <= 0) n = num_sms / cl;
            nc = std::min(n, num_sms / cl);
        }
        grid = nc * cl;
        cfg.numAttrs = 2;
    } else {
        cfg.numAttrs = 1;
    }
    cfg.gridDim = dim3(unsigned(grid));
    return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int BITS, int QN, int GQ>
static cudaError_t launch_dec_f(const DecArgs& a, cudaStream_t st, int num_sms, size_t smem) {
    constexpr int NP = BITS == 8 ? 2 : 1;
    return a.fused ? launch_dec_t<BITS, QN, GQ, NP, true>(a, st, num_sms, smem)
                   : launch_dec_t<BITS, QN, GQ, NP, false>(a, st, num_sms, smem);
}

template <int BITS, int QN>
static cudaError_t launch_dec_q(const DecArgs& a, cudaStream_t st, int num_sms, size_t smem) {
    switch (a.Np2 / 256) {
#ifndef DEC_AB_ONLY  // experiment builds (tools/ab_build.sh): d_model = 1024 only
        case 1: return launch_dec_f<BITS, QN, 1>(a, st, num_sms, smem);
        case 2: return launch_dec_f<BITS, QN, 2>(a, st, num_sms, smem);
        case 3: return launch_dec_f<BITS, QN, 3>(a, st, num_sms, smem);
#endif
        case 4: return launch_dec_f<BITS, QN, 4>(a, st, num_sms, smem);
    }
    return cudaErrorInvalidValue;
}

template <int BITS>
static cudaError_t launch_dec_b(const DecArgs& a, cudaStream_t st, int num_sms, size_t smem) {
    switch (a.Kp1 / 256) {
#ifndef DEC_AB_ONLY
        case 1: return launch_dec_q<BITS, 1>(a, st, num_sms, smem);
        case 2: return launch_dec_q<BITS, 2>(a, st, num_sms, smem);
        case 3: return launch_dec_q<BITS, 3>(a, st, num_sms, smem);
#endif
        case 4: return launch_dec_q<BITS, 4>(a, st, num_sms, smem);
    }
    return cudaErrorInvalidValue;
}

// Gate weights for the fused routing: Wg [d x E] f32 -> [4 K chunks][hi, lo][Ep][Kp1/4 + 8] fp16
// with Wg * 2^shift = hi + lo (shift keeps hi in range and lo out of the subnormals).
__global__ void k_wg_split(const float* __restrict__ wg, int d, int E, int Ep, int Kp1, int shift,
                           __half* __restrict__ out) {
    const int Kc = Kp1 / 4, cp = Kc + 8;
    const int64_t n = int64_t(4) * 2 * Ep * cp;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int kk = int(i % cp);
        const int e = int((i / cp) % Ep);
        const int h2 = int((i / (int64_t(cp) * Ep)) % 2);
        const int c = int(i / (int64_t(cp) * Ep * 2));
        const int k = c * Kc + kk;
        float v = 0.f;
        if (kk < Kc && k < d && e < E) v = ldexpf(wg[size_t(k) * E + e], shift);
        const __half hi = __float2half_rn(v);
        out[i] = h2 == 0 ? hi : __float2half_rn(v - __half2float(hi));
    }
}

int64_t dec_wgt_halves(int E, int Kp1) { return int64_t(4) * 2 * ((E + 7) & ~7) * (Kp1 / 4 + 8); }

cudaError_t dec_split_wg(const float* wg, int d, int E, int Kp1, int shift, __half* out, cudaStream_t st) {
    const int64_t n = dec_wgt_halves(E, Kp1);
    k_wg_split<<<unsigned(std::min<int64_t>((n + 255) / 256, 4096)), 256, 0, st>>>(wg, d, E, (E + 7) & ~7, Kp1, shift, out);
    return cudaGetLastError();
}

// Shared-memory plan of k_dec for a mode (fused routing or not); false when it does not fit.
static bool dec_config(int bits, DecArgs& a, size_t* smem_out) {
    const int RB = 8 * bits, NP = bits == 8 ? 2 : 1;
    a.stage_bytes = uint32_t(a.Kp1 / NP) * RB + 512;  // W1 piece + the slice's fc1 scales / biases
    a.stage2_bytes = uint32_t(a.Np2 / NP) * RB;
    const size_t xregion = a.fused ? ((size_t(a.T) * a.xpitch + 127) & ~size_t(127)) : 2 * size_t(kDecUnitRows) * a.xpitch;
    const size_t fixed = xregion + 2 * kDecUnitRows * kMidPitch + 512 + 2 * 4 * 32 * 8 * 4 + sizeof(DecPlanSmem) + 256;
    if (fixed >= 227 * 1024) return false;
    const size_t budget = 227 * 1024 - fixed;
    // stages split evenly between the W1 and W2 rings (both parts have the same bytes)
    const int pairs = int(std::min<size_t>(8, budget / (a.stage_bytes + a.stage2_bytes + 32)));
    if (pairs < 2) return false;
    if (a.fused) {  // the routing phase borrows the rings: 2..4 Wg chunks + the partial logits
        const DecRouteGeom G(a.E, a.route_cluster, a.T);
        const size_t cb = size_t(2 * G.Ep) * ((a.Kp1 / 4 + 8) * 2), pb = G.floats() * 4;
        const size_t ring = size_t(pairs) * (a.stage_bytes + a.stage2_bytes);
        a.route_nbuf = ring < pb ? 0 : int(std::min<size_t>(4, (ring - pb) / cb));
        // a cluster CTA holds its 4/cl chunks at once; alone it streams them through >= 2 buffers
        const int cl = a.route_cluster == 2 || a.route_cluster == 4 ? a.route_cluster : 1;
        if (a.route_nbuf < (cl > 1 ? 4 / cl : 2)) return false;
    }
    a.n_stages = a.n_stages2 = pairs;
    *smem_out = size_t(pairs) * (a.stage_bytes + a.stage2_bytes) + fixed + size_t(pairs) * 32;
    return true;
}

cudaError_t launch_dec(int bits, const DecArgs& a0, cudaStream_t st, int num_sms) {
    DecArgs a = a0;
    size_t smem = 0;
    if (a.fused && !dec_config(bits, a, &smem)) {
        // a larger cluster needs fewer gate-weight chunks per CTA (e.g. E = 64 at d = 1024)
        if (a.route_cluster == 2) a.route_cluster = 4;
        if (a.route_cluster != 4 || !dec_config(bits, a, &smem)) a.fused = 0;  // separate router launch
    }
    if (!a.fused && !dec_config(bits, a, &smem)) return cudaErrorInvalidConfiguration;
    if (!a.fused && !a.plan_ready) {  // ---- router (one cluster) ----
        const int C = route_cluster(a.d, a.E);
        const size_t rs = route_smem(int(a.T), a.d, a.E, C);
        static bool configured[kMaxDev] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < kMaxDev && !configured[dev]) {
            cudaError_t e = cudaFuncSetAttribute(k_dec_route, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxRouteSmem);
            if (e != cudaSuccess) return e;
            e = cudaFuncSetAttribute(k_dec_route, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
            configured[dev] = true;
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(C);
        cfg.blockDim = dim3(kDecThreads);
        cfg.dynamicSmemBytes = rs;
        cfg.stream = st;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_dec_route, a);
        if (e != cudaSuccess) return e;
    }
    // ---- expert FFN ----
    switch (bits) {
        case 2: return launch_dec_b<2>(a, st, num_sms, smem);
        case 3: return launch_dec_b<3>(a, st, num_sms, smem);
#ifndef DEC_AB_ONLY
        case 4: return launch_dec_b<4>(a, st, num_sms, smem);
        case 8: return launch_dec_b<8>(a, st, num_sms, smem);
#endif
    }

    return cudaErrorInvalidValue;
}

}  // namespace moqe_gpu
