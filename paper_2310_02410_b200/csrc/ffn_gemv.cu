// ffn_gemv.cu — decode path: expert FFN (fc1 -> ReLU -> fc2 -> gate combine)
// as persistent weight-streaming kernels, plus the token-row encoder k_xrows
// that runs beside the router. Decode batches (<= 64 routed rows, d <= 1024)
// run fc1 and fc2 in ONE grid: every CTA streams its fc1 items, then its
// cluster's fc2 items; an fc2 item waits only for its own pass's readiness
// counter (release by the fc1 epilogues), so fc2 weights stream while fc1
// finishes. Larger batches chain an fc1 and an fc2 grid with programmatic
// dependent launch (PDL).
//
// Reference: the per-expert loop of moe_ffn_forward proj/src/model.cpp:360-391
// (dequantize :370-375, matmul :381/:384, add_bias/relu :382-385, scatter
// :387-390). The reference re-dequantizes whole experts to f32 (27 ms per
// 4M-element matrix); here packed codes stream from HBM exactly once and are
// never widened beyond 8 bits.
//
// Integer dot products (frag.cuh). A weight code q = u - 2^(b-1) is kept as
// its offset binary u; one LOP3 yields four u8 values u * 2^s that feed IMMA
// m16n8k32 (u8 x s8 -> s32). The activations of a row are a per-row
// fixed-point integer X = rint(x * 2^p) split into signed base-256 digit
// planes; each plane is one MMA column. Sum_k u*X is exact in integers; the
// zero point 2^(b-1) * Sum X, the plane weights 256^s and 2^-p are applied
// once per item, the per-channel scale in the epilogue.
//   fc1 rows (fp16 tokens): 3 planes, p from the row maximum — exact for every
//     activation within 2^11 of the row max.
//   fc2 rows (mid = ReLU(fc1)): 4 planes, p from a rigorous per-row bound
//     |mid| <= max_scale * 2^(b-1) * |x|_1 + max|bias|, so every fc1 item
//     encodes its own 128 output channels (one fc2 k-stage) independently;
//     resolution ~2^-29 of the bound, far finer than the reference's fp32 chain.
//
// Row blocks. The B operand of an item is up to 4 rows; each row's digits of
// one 1024-k chunk live in a self-contained "row block" (header + one plane
// per digit, every plane already in the k-order the IMMA B fragments want), so
// the producer fetches a row with a single TMA bulk copy and a consumer lane
// reads its B registers with one LDS.64 per fragment. fc1 row blocks are
// written once per token by k_xrows (not once per item), fc2 row blocks by the
// fc1 epilogue (one 128-k stage per fc1 item).
//
// Work: an item is (expert, row pass, 128-channel m-tile); its K is split into
// 1024-k chunks, one per CTA of a thread-block cluster (fc1: d/1024 CTAs, fc2:
// f/1024). Each CTA streams its chunk's packed tiles — one contiguous stripe —
// with TMA bulk copies of >= 16 KB (smaller copies cap the chip at 1-3.6 TB/s,
// profiles/round1/tma_copy_size.md). Items are statically scheduled over the
// clusters (all the same size): no tickets, no cross-cluster synchronisation.
//   warps 0-7   consumers: 16 channels each; LOP3 unpack + IMMA; per item the
//               exact group sums go to a double-buffered scratch and the warp
//               moves straight on to the next item (the stream never waits
//               for an epilogue)
//   warps 8-15  epilogue, two groups of four taking alternate items: thread =
//               channel; exact int64 partials, split-K reduction into cluster
//               rank 0 over DSMEM, scale/bias, and
//               fc1: ReLU -> fc2 fixed point -> fc2 row blocks in global memory
//               (fused grid: then a per-pass readiness release)
//               fc2: gate-weighted output rows (one writer per element)
//   warp 16     producer: row blocks + weight copy units (TMA, evict-first)
#include <cuda_fp16.h>

#include <algorithm>

#include "codec.cuh"
#include "frag.cuh"
#include "kernels.cuh"
#include "ptx.cuh"
#include "xrow.cuh"

namespace moqe_gpu {

constexpr int kMaxCluster = 8;
constexpr int kPassRows = 4;         // rows per item pass
constexpr int kMaxNT = 2;            // n8 column tiles (4 rows x 4 planes = 16 columns)
constexpr int kMaxListed = 256;
constexpr int kConsumers = 8;        // MMA warps: 16 channels (one m16 block) each
constexpr int kEpiWarps = 4;         // warps per epilogue group: one thread per channel
constexpr int kEpiGroups = 2;        // epilogue groups, alternating items (an item's epilogue may take
                                     // longer than its mainloop without stalling the consumers)
constexpr int kProdWarp = kConsumers + kEpiGroups * kEpiWarps;
constexpr int kGemvThreads = (kProdWarp + 1) * 32;
constexpr int kBufs = 3;             // row-block buffers (B operands of 3 items in flight)
constexpr int kScrBufs = 2;          // accumulator scratch buffers (consumer -> epilogue)
constexpr int kScrStride = 20;       // ints per channel row of the scratch (16 columns; conflict-free LDS.128)
constexpr int kSmemMax = 227 * 1024;

__host__ __device__ constexpr int planes_of(int phase) { return phase == 1 ? 3 : 4; }
__host__ __device__ constexpr int nt_of(int phase, int rows) { return (planes_of(phase) * rows + 7) / 8; }
template <int BITS>
__host__ __device__ constexpr int unit_stages() { return BITS == 8 ? 2 : 4; }  // >= 16 KB per weight copy

template <int BITS>
struct Cfg {
    static constexpr int F = Frag<BITS>::F;
    static constexpr int TB = tile_bytes(BITS);
    static constexpr int SB = 2 * TB;          // one IMMA stage of weights
    static constexpr int US = unit_stages<BITS>();
    static constexpr int UB = US * SB;         // one weight copy
};

struct GemvItem {
    int e, mt, row0, nrows;  // e < 0: none
};

constexpr int kTokCache = 512;       // routed rows whose token ids the producer keeps in smem
constexpr int kItemCache = 64;       // this CTA's first items, decoded once at kernel start

struct GemvTables {
    int list[kMaxListed], cnt[kMaxListed], off[kMaxListed];
    int start[kMaxListed + 1];  // item prefix per listed expert
    int tok[kTokCache];         // perm_token[0, kTokCache) (fc1 row-block sources)
    int4 items[kItemCache];     // (e, mt, row0, nrows) of this CTA's k-th item
    int n;                      // n_gemv
    // self plan (decode, GEMV only): the router's raw choices -> positions
    int rexp[kSelfPlanRows];    // expert of routed row i = (token, slot)
    int eoff[kMaxListed];       // first permuted row of expert e
    float gate[kSelfPlanRows];  // gate of permuted row (fc2 epilogue)
};

__device__ __forceinline__ int find_listed(const int* st, int n, int v, int sc) {  // largest a with st[a] * sc <= v
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (st[mid] * sc <= v) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Item tables from the plan's GEMV table (one warp, ONE load round: the header and
// the first 32 entries are fetched together; prefix by a warp scan). Returns n_gemv
// in T.n.
__device__ void build_tables(GemvTables& T, const Plan& P, int nmt, int lane, int64_t rows) {
    const int nr = rows < kTokCache ? int(rows) : kTokCache;
    const int n = P.gtab[0].x;
    int4 v = P.gtab[1 + lane];  // speculative: valid if lane < n
    for (int r = lane; r < nr; r += 32) T.tok[r] = P.perm_token[r];
    int running = 0;
    for (int a0 = 0; a0 < n; a0 += 32) {
        if (a0 > 0) v = P.gtab[1 + a0 + lane];
        const int a = a0 + lane;
        const bool ok = a < n;
        const int np = ok ? nmt * ((v.y + kPassRows - 1) / kPassRows) : 0;
        int incl = np;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        if (ok) {
            T.list[a] = v.x;
            T.cnt[a] = v.y;
            T.off[a] = v.z;
            T.start[a] = running + incl - np;
        }
        running += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
        T.start[n] = running;
        T.n = n;
    }
}

// Self plan (decode, every routed expert on the GEMV path, T*k <= kSelfPlanRows):
// the same counts, expert-order offsets, item prefix and stable row order as the
// router's plan (route.cu plan_lists / the decode router's leader), built by one
// warp from P.expert / P.gate in one load round — the router then only writes the
// choices and never serialises a plan step.
// The loads go through L2 only (__ldcg): the GEMV grid also runs this as a dry pass while
// the router still writes the choices, and must not keep stale lines in L1; ids are
// clamped to [0, E) so a dry pass over stale data stays in bounds.
__device__ void build_tables_self(GemvTables& T, const Plan& P, int nr, int E, int k, int nmt, int lane) {
    // rows i = lane and lane + 32; per-expert counts by smem atomics, stable ranks by
    // __match_any (no per-lane loops over the rows)
    const int i0 = lane, i1 = lane + 32;
    const int e0 = i0 < nr ? int(min(unsigned(__ldcg(P.expert + i0)), unsigned(E - 1))) : -1;
    const int e1 = i1 < nr ? int(min(unsigned(__ldcg(P.expert + i1)), unsigned(E - 1))) : -1;
    const float g0 = i0 < nr ? __ldcg(P.gate + i0) : 0.f, g1 = i1 < nr ? __ldcg(P.gate + i1) : 0.f;
    int* h1 = T.rexp;  // scratch: [E] counts of rows 0..31 (E <= kSelfPlanRows handled below)
    int* cnt = T.eoff;  // [E] total counts; the scan below reads each and overwrites it with the offset
    for (int e = lane; e < E; e += 32) cnt[e] = 0;
    const bool small = E <= kSelfPlanRows;
    if (small) for (int e = lane; e < E; e += 32) h1[e] = 0;
    __syncwarp();
    const unsigned lt = (1u << lane) - 1u;
    const unsigned m0 = __match_any_sync(0xffffffffu, e0), m1 = __match_any_sync(0xffffffffu, e1);
    if (e0 >= 0 && (m0 & lt) == 0) atomicAdd(&cnt[e0], __popc(m0));   // leader of each group adds its size
    if (e1 >= 0 && (m1 & lt) == 0) atomicAdd(&cnt[e1], __popc(m1));
    if (small && e0 >= 0 && (m0 & lt) == 0) h1[e0] = __popc(m0);
    __syncwarp();
    int running = 0, nlisted = 0, items = 0;
    for (int eb = 0; eb < E; eb += 32) {
        const int e = eb + lane;
        const int c = e < E ? cnt[e] : 0;
        int incl = c;
        const int np = c > 0 ? nmt * ((c + kPassRows - 1) / kPassRows) : 0;
        int inp = np;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, off);
            const int z = __shfl_up_sync(0xffffffffu, inp, off);
            if (lane >= off) { incl += y; inp += z; }
        }
        if (e < E) T.eoff[e] = running + incl - c;
        const unsigned bl = __ballot_sync(0xffffffffu, c > 0);
        if (c > 0) {
            const int a = nlisted + __popc(bl & lt);
            T.list[a] = e;
            T.cnt[a] = c;
            T.off[a] = running + incl - c;
            T.start[a] = items + inp - np;
        }
        running += __shfl_sync(0xffffffffu, incl, 31);
        items += __shfl_sync(0xffffffffu, inp, 31);
        nlisted += __popc(bl);
    }
    if (lane == 0) {
        T.start[nlisted] = items;
        T.n = nlisted;
    }
    __syncwarp();
    // stable positions: row i -> eoff[e] + #{j < i : e_j == e}
    if (e0 >= 0) {
        const int pos = T.eoff[e0] + __popc(m0 & lt);
        T.tok[pos] = i0 / k;
        T.gate[pos] = g0;
    }
    int before = 0;  // rows 0..31 with the same expert
    if (small) {
        if (e1 >= 0) before = h1[e1];
    } else {
        // every lane takes part in the full-mask shuffles (rows >= nr have e1 = -1)
        for (int j = 0; j < 32; ++j) before += __shfl_sync(0xffffffffu, e0, j) == e1;
    }
    if (e1 >= 0) {
        const int pos = T.eoff[e1] + before + __popc(m1 & lt);
        T.tok[pos] = i1 / k;
        T.gate[pos] = g1;
    }
    __syncwarp();
}

// Item i (expert-major: expert, pass, m-tile). T.start counts items (sc = 1) or, for the
// fused kernel whose two phases differ in m-tiles, passes (sc = nmt).
__device__ __forceinline__ GemvItem item_at(int i, const GemvTables& T, int n_gemv, int nmt, int sc) {
    GemvItem it{};
    if (i >= T.start[n_gemv] * sc) { it.e = -1; return it; }
    const int a = find_listed(T.start, n_gemv, i, sc);
    const int r = i - T.start[a] * sc;
    const int pass = r / nmt;
    it.e = T.list[a];
    it.mt = r - pass * nmt;
    it.row0 = T.off[a] + pass * kPassRows;
    it.nrows = min(kPassRows, T.cnt[a] - pass * kPassRows);
    return it;
}

// One phase (fc1 or fc2) as this CTA sees it.
struct PhaseGeo {
    int CS, rank, clu, nclu;  // split-K cluster of this phase (fused fc1: one CTA)
    int Kp, Np, k0, nst, nunits, nmt;
    int n, nitems, sc;        // listed experts, items, unit of T.start (see item_at)
    int cbase, ccap;          // this phase's slice of T.items
    const uint8_t* wbase0;
    int64_t wstride;
};

// k-th item of this CTA in phase Q (global index i): the cached decode, else the table lookup
__device__ __forceinline__ GemvItem item_of(int k, int i, const GemvTables& T, const PhaseGeo& Q) {
    if (k < Q.ccap) {
        const int4 v = T.items[Q.cbase + k];
        GemvItem it;
        it.e = v.x; it.mt = v.y; it.row0 = v.z; it.nrows = v.w;
        return it;
    }
    return item_at(i, T, Q.n, Q.nmt, Q.sc);
}

// ---- optional event trace (diagnostics; off unless the bank enables it) ----------------
// Per CTA and phase a row of kTraceCap/2 slots: slot 0 / last = (globaltimer, clock64)
// anchors at start / end; consumers log into [1, 128), epilogue [128, 192), producer
// [192, last). Events carry clock64 (cheap, no atomics); the reader maps them to ns.
// role 2 = consumers (3 top, 0 row blocks in, 1 mainloop end, 4 scratch free),
// 3 = epilogue (0 start, 2 end), 4 = producer (0/1 unit issued), 5 = unit landed.
struct Tracer {
    unsigned long long* p;
    int n, cap;
    __device__ __forceinline__ void ev(int role, int e, const GemvItem& it, int phase) {
        if (p == nullptr || n >= cap) return;
        unsigned long long* q = p + 2 * n++;
        q[0] = clock64();
        q[1] = (unsigned long long)role << 60 | (unsigned long long)e << 56 | (unsigned long long)phase << 48 |
               (unsigned long long)(it.e & 0xffff) << 32 | (unsigned long long)(it.mt & 0xfff) << 20 |
               (unsigned long long)(it.nrows & 0xf) << 16 | 1ull;
    }
};
__device__ __forceinline__ Tracer tracer(unsigned long long* row, int lo, int hi) {
    Tracer t;
    t.p = row ? row + 2 * lo : nullptr;
    t.n = 0;
    t.cap = hi - lo;
    return t;
}

// ---- k_xrows: token rows -> fc1 row blocks ------------------------------------------------
// Warp per (token, 1024-k chunk); lane = (stage st, quad tq) owns the 32
// activations that quad's IMMA lanes meet in stage st. The row maximum and
// |x|_1 cover the whole row, so every chunk of a row derives the same exponent.
__device__ __forceinline__ float act16(const XrowArgs& a, int64_t t, int k) {  // fp16 value of h[t][k] (0 beyond d)
    if (k >= a.d) return 0.f;
    return a.h_f16 ? __half2float(static_cast<const __half*>(a.h)[t * a.d + k])
                   : __half2float(__float2half_rn(static_cast<const float*>(a.h)[t * a.d + k]));
}
__device__ __forceinline__ void load16(const XrowArgs& a, int64_t t, int k, bool vec, float* v) {
    if (vec) {
        const __half* row = static_cast<const __half*>(a.h) + t * a.d;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            uint4 w = make_uint4(0u, 0u, 0u, 0u);
            if (k + 8 * q < a.d) w = __ldg(reinterpret_cast<const uint4*>(row + k + 8 * q));  // d % 8 == 0
            const __half2* h2 = reinterpret_cast<const __half2*>(&w);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = __half22float2(h2[i]);
                v[8 * q + 2 * i] = f.x;
                v[8 * q + 2 * i + 1] = f.y;
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = act16(a, t, k + i);
    }
}

template <int BITS>
__global__ void __launch_bounds__(128) k_xrows(XrowArgs a) {
    // Launched with PDL behind the previous forward's expert-FFN grid, so this grid can be
    // resident before that one drains: wait for the previous grid, then let the decode router
    // launch (it reads the token rows, never the row blocks).
    pdl_wait();
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t w = int64_t(blockIdx.x) * 4 + warp;
    const int64_t t = w / a.nch1;
    const int c = int(w - t * a.nch1);
    if (a.ready && blockIdx.x == 0 && threadIdx.x < kSelfPlanRows) a.ready[threadIdx.x] = 0u;
    if (t >= a.T) return;
    const bool vec = a.h_f16 && (a.d % 8) == 0 && (reinterpret_cast<uintptr_t>(a.h) & 15) == 0;
    const int st = lane >> 2, tq = lane & 3, k0 = c * kChunkK;
    float v[32];
    load16(a, t, k0 + st * kStageK + 16 * tq, vec, v);
    load16(a, t, k0 + st * kStageK + 64 + 16 * tq, vec, v + 16);
    float m = 0.f, l1 = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) { m = fmaxf(m, fabsf(v[i])); l1 += fabsf(v[i]); }
    for (int k = lane * 16; k < a.d; k += 32 * 16) {  // the other chunks of the row: max and |x|_1 only
        if (k >= k0 && k < k0 + kChunkK) continue;
        float u[16];
        load16(a, t, k, vec, u);
#pragma unroll
        for (int i = 0; i < 16; ++i) { m = fmaxf(m, fabsf(u[i])); l1 += fabsf(u[i]); }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    xrow_encode<BITS>(v, m, l1, a.xr + (t * a.nch1 + c) * int64_t(RB<BITS>::XR1), lane);
}

// ---- consumer pieces -------------------------------------------------------------------
// One 128-k stage of one m16 block: LOP3 unpack + IMMA against the stage's B words.
template <int BITS, int NT>
__device__ __forceinline__ void stage_mma(const uint8_t* T0, int r0, int tq, const uint8_t* const (&bp)[kMaxNT],
                                          int soff, int (&acc)[Frag<BITS>::G][kMaxNT][4]) {
    using FR = Frag<BITS>;
    constexpr int F = FR::F;
    uint32_t a[F][4];
    FR::load(T0, T0 + tile_bytes(BITS), r0, tq, a);
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const uint2 b = *reinterpret_cast<const uint2*>(bp[j] + soff + f * 32);
            imma(acc[FR::grp(f)][j], a[f], b.x, b.y);
        }
}

template <int BITS, int NT>
__device__ __forceinline__ void unit_mma(const uint8_t* U, int nst_u, int s0, int r0, int tq,
                                         const uint8_t* const (&bp)[kMaxNT], int (&acc)[Frag<BITS>::G][kMaxNT][4]) {
    using FR = Frag<BITS>;
    constexpr int F = FR::F, US = unit_stages<BITS>();
    constexpr int SB = 2 * tile_bytes(BITS), STG = RB<BITS>::STG;
    if (nst_u == US) {
        // full unit: every stage's A and B words are loaded before the first IMMA
        // (two consumer warps per SM sub-partition cannot hide the LDS -> IMMA chain)
        uint32_t a[US][F][4];
        uint2 b[US][F][NT];
#pragma unroll
        for (int s = 0; s < US; ++s) {
            const uint8_t* T0 = U + s * SB;
            FR::load(T0, T0 + tile_bytes(BITS), r0, tq, a[s]);
#pragma unroll
            for (int f = 0; f < F; ++f)
#pragma unroll
                for (int j = 0; j < NT; ++j)
                    b[s][f][j] = *reinterpret_cast<const uint2*>(bp[j] + (s0 + s) * STG + f * 32);
        }
#pragma unroll
        for (int s = 0; s < US; ++s)
#pragma unroll
            for (int f = 0; f < F; ++f)
#pragma unroll
                for (int j = 0; j < NT; ++j) imma(acc[FR::grp(f)][j], a[s][f], b[s][f][j].x, b[s][f][j].y);
        return;
    }
#pragma unroll 1
    for (int s = 0; s < nst_u; ++s) stage_mma<BITS, NT>(U + s * SB, r0, tq, bp, (s0 + s) * STG, acc);
}

// V * 2^-sh in fp32: one rounding (int64 -> fp32), exact power-of-two scale
__device__ __forceinline__ float scale_pow2(long long V, int sh) {
    const float v = float(V);
    return (sh > -127 && sh < 127) ? v * __int_as_float((127 - sh) << 23) : ldexpf(v, -sh);
}

// fc2 exponent of one fc1 row: |mid| <= smax * 2^(b-1) * |x|_1 + bmax, and
// |X| = |mid| * 2^p2 < 2^30 keeps four signed base-256 digits.
template <int BITS>
__device__ __forceinline__ int fc2_exp(float smax, float bmax, float l1) {
    const float bound = (smax * float(1 << (BITS - 1)) * l1 + bmax) * (1.0f + 0x1p-16f);
    return bound < 0x1p-100f ? kZeroRow : 29 - ilogbf(bound);
}

// ---- smem layout (host and device agree) ------------------------------------------------
// Fixed parts first, then the split-K partials (only for clusters of >= 2 CTAs,
// sized by the cluster), then the weight ring takes everything that is left:
// the in-flight bytes per SM are what bounds the stream at loaded HBM latency.
template <int BITS, int PHASE>  // PHASE 0: the fused kernel (both phases share the carve-up)
struct Layout {
    using R = RB<BITS>;
    static_assert(R::XR2 >= R::XR1, "fc2 row blocks are the larger");
    static constexpr int kMaxNU = 8;
    static constexpr int XR = PHASE == 1 ? R::XR1 : R::XR2;                    // row-block buffer stride
    static constexpr int BUFS = kBufs * kPassRows * XR;
    static constexpr int ZERO = rup(R::PB, 128);                               // all-zero plane (idle columns)
    static constexpr int SCR = kScrBufs * TILE_N * kScrStride * 4;
    static constexpr int STG1 = PHASE != 2 ? rup(kPassRows * 4 * R::STG + kEpiWarps * kPassRows * 8, 128) : 0;
    static constexpr int STG = kEpiGroups * STG1;  // per epilogue group
    static constexpr int TABLES = rup(int(sizeof(GemvTables)), 128);
    static constexpr int BARS = rup((2 * kMaxNU + 2 * kBufs + 2 * kScrBufs + 4) * 8, 128);
    static constexpr int O_ZERO = BUFS, O_SCR = O_ZERO + ZERO, O_STG = O_SCR + SCR, O_TAB = O_STG + STG;
    static constexpr int O_BARS = O_TAB + TABLES, O_RED = O_BARS + BARS;
    __host__ __device__ static constexpr int red_bytes(int cs) { return cs > 1 ? 2 * (cs - 1) * TILE_N * kPassRows * 8 : 0; }
    __host__ __device__ static constexpr int ring_off(int cs) { return rup(O_RED + red_bytes(cs), 128); }
    __host__ __device__ static constexpr int nu(int cs) {
        return (kSmemMax - ring_off(cs)) / Cfg<BITS>::UB < kMaxNU ? (kSmemMax - ring_off(cs)) / Cfg<BITS>::UB : kMaxNU;
    }
    __host__ __device__ static constexpr int total(int cs) { return ring_off(cs) + nu(cs) * Cfg<BITS>::UB; }
    static_assert(nu(kMaxCluster) >= 2, "weight ring needs two slots");
};

// ---- per-phase pieces ---------------------------------------------------------------------
// Shared-memory carve-up of one CTA (both phases of the fused kernel share it).
struct GemvSmem {
    uint8_t* bufs;        // [kBufs][4 rows][XRB]: row blocks of 3 items in flight
    const uint8_t* zero;  // zero plane (idle B columns)
    int* scr;             // [2][128][kScrStride]: exact group sums, consumers -> epilogue
    uint8_t* stg;         // fc1: per epilogue group [4 rows][4 planes][STG] + zred
    GemvTables* TBL;
    long long* red;       // [2][CS-1][128][4]: split-K partials (rank 0)
    uint8_t* ring;        // [NU][UB]: weight copy units
    uint64_t *full, *empty, *bfull, *bempty, *sfull, *sempty, *red_full, *red_empty;
    int NU, XRB;
};

template <int BITS, int PH>
__device__ __forceinline__ PhaseGeo phase_geo(const GemvArgs& g, int CS, int rank, int clu, int nclu) {
    PhaseGeo G;
    G.CS = CS;
    G.rank = rank;
    G.clu = clu;
    G.nclu = nclu;
    G.Kp = PH == 1 ? g.Kp1 : g.Kp2;
    G.Np = PH == 1 ? g.Np1 : g.Np2;
    G.k0 = rank * kChunkK;
    G.nst = (min(kChunkK, G.Kp - G.k0) + kStageK - 1) / kStageK;
    G.nunits = (G.nst + Cfg<BITS>::US - 1) / Cfg<BITS>::US;
    G.nmt = G.Np / TILE_N;
    G.n = G.nitems = G.cbase = G.ccap = 0;
    G.sc = 1;
    G.wbase0 = PH == 1 ? g.w1 : g.w2;
    G.wstride = PH == 1 ? g.w1_stride : g.w2_stride;
    return G;
}

// Finalise both phases' item counts and cache slices from the built tables (every thread).
__device__ __forceinline__ void finish_geo(const GemvTables& T, PhaseGeo& G1, PhaseGeo& G2, int tsc, bool fused) {
    const int n = T.n;
    G1.n = G2.n = n;
    G1.sc = tsc;
    G1.nitems = n > 0 ? T.start[n] * tsc : 0;
    G1.cbase = 0;
    G1.ccap = fused ? kItemCache / 2 : kItemCache;  // fused: half per phase
    G2.sc = G2.nmt;
    G2.nitems = n > 0 ? T.start[n] * G2.nmt : 0;
    G2.cbase = kItemCache / 2;
    G2.ccap = fused ? kItemCache / 2 : 0;
}
// Decode this CTA's first items of both phases into T.items (threads tid < nthr of one warp
// group, after the tables are built; read after the CTA barrier).
__device__ __forceinline__ void fill_items(GemvTables& T, PhaseGeo G1, PhaseGeo G2, int tsc, bool fused, int tid,
                                           int nthr) {
    finish_geo(T, G1, G2, tsc, fused);
    for (int k = tid; k < G1.ccap; k += nthr) {
        const int i = G1.clu + k * G1.nclu;
        if (i >= G1.nitems) break;
        const GemvItem it = item_at(i, T, G1.n, G1.nmt, G1.sc);
        T.items[G1.cbase + k] = make_int4(it.e, it.mt, it.row0, it.nrows);
    }
    for (int k = tid; k < G2.ccap; k += nthr) {
        const int i = G2.clu + k * G2.nclu;
        if (i >= G2.nitems) break;
        const GemvItem it = item_at(i, T, G2.n, G2.nmt, G2.sc);
        T.items[G2.cbase + k] = make_int4(it.e, it.mt, it.row0, it.nrows);
    }
}

// ===== producer (one thread): each item's row blocks, then its weight copy units
template <int BITS, int PH>
__device__ __forceinline__ void produce(const GemvArgs& g, const Plan& P, const GemvSmem& S, const PhaseGeo& Q,
                                        int& slot, int& sph, int& seq, int early_units, bool early_rows, bool fused,
                                        bool& waited, Tracer& T) {
    using C = Cfg<BITS>;
    constexpr int XR = PH == 1 ? RB<BITS>::XR1 : RB<BITS>::XR2;
    const GemvTables& TBL = *S.TBL;
    const uint64_t pol = policy_evict_first();
    const int nch2 = (g.Kp2 + kChunkK - 1) / kChunkK;
    for (int k = 0, i = Q.clu; i < Q.nitems; i += Q.nclu, ++k, ++seq) {
        const GemvItem it = item_of(k, i, TBL, Q);
        const int b = seq % kBufs, bph = ((seq / kBufs) & 1) ^ 1;
        auto issue_rows = [&]() {
            if (PH == 2 && fused) {  // the pass's fc2 row blocks come from fc1 items of every CTA
                const unsigned need = unsigned(g.Np1 / TILE_N);
                while (ld_acquire_u32(g.ready + it.row0) < need) {
                }
                fence_proxy_async_global();  // generic writes (fc1 epilogues) -> this CTA's TMA reads
            }
            mbar_wait(&S.bempty[b], bph);
            mbar_arrive_expect_tx(&S.bfull[b], uint32_t(it.nrows * XR));
            for (int t = 0; t < it.nrows; ++t) {
                const uint8_t* src =
                    PH == 1 ? g.xr + (int64_t(it.row0 + t < kTokCache ? TBL.tok[it.row0 + t]
                                                                      : __ldg(P.perm_token + it.row0 + t)) *
                                          g.nch1 + Q.rank) * XR
                            : g.xb + (int64_t(it.row0 + t) * nch2 + Q.rank) * XR;
                bulk_g2s(S.bufs + (b * kPassRows + t) * S.XRB, src, uint32_t(XR), &S.bfull[b]);
            }
        };
        // fc2 (first item of the fc2 kernel; every item of the fused one): the weights do not
        // depend on fc1 and are queued first; the row blocks follow once the ring is full or
        // the item is issued
        const bool late = PH == 2 && (fused || k == 0);
        if (!late && !(k == 0 && early_rows)) issue_rows();
        const uint8_t* wb =
            Q.wbase0 + int64_t(it.e) * Q.wstride + (int64_t(it.mt) * (Q.Kp / TILE_K) + Q.k0 / TILE_K) * C::TB;
        bool rows_due = late;
        for (int u = k == 0 ? early_units : 0; u <= Q.nunits; ++u) {
            if (rows_due && (u == Q.nunits || u == S.NU)) {
                if (!waited) pdl_wait();
                waited = true;
                rows_due = false;
                issue_rows();
            }
            if (u == Q.nunits) break;
            const int bytes = min(C::US, Q.nst - u * C::US) * C::SB;
            mbar_wait(&S.empty[slot], sph ^ 1);
            T.ev(4, u == 0 ? 0 : 1, it, PH);
            mbar_arrive_expect_tx(&S.full[slot], uint32_t(bytes));
            bulk_g2s_hint(S.ring + size_t(slot) * C::UB, wb + int64_t(u) * C::UB, uint32_t(bytes), &S.full[slot], pol);
            if (++slot == S.NU) { slot = 0; sph ^= 1; }
        }
    }
}

// ===== consumers: warp -> m16 block (16 channels) of the 128-channel item
template <int BITS, int PH>
__device__ __forceinline__ void consume(const GemvArgs& g, const GemvSmem& S, const PhaseGeo& Q, int& slot, int& sph,
                                        int& seq, int warp, int lane, Tracer& T) {
    using FR = Frag<BITS>;
    using C = Cfg<BITS>;
    using R = RB<BITS>;
    constexpr int G = FR::G, HDR = PH == 1 ? R::HDR1 : R::HDR2, PL = planes_of(PH);
    const int gq = lane >> 2, tq = lane & 3;
    const int r0 = 16 * warp + gq;
    for (int k = 0, i = Q.clu; i < Q.nitems; i += Q.nclu, ++k, ++seq) {
        const GemvItem it = item_of(k, i, *S.TBL, Q);
        const int b = seq % kBufs, sb = seq & 1;
        const int NT = nt_of(PH, it.nrows), ncol = PL * it.nrows;
        // B column c = s * nrows + t (plane s of row t); idle columns read the zero plane
        const uint8_t* bp[kMaxNT];
        const int inv = it.nrows == 1 ? 65536 : it.nrows == 2 ? 32768 : it.nrows == 3 ? 21846 : 16384;
#pragma unroll
        for (int j = 0; j < kMaxNT; ++j) {
            const int c = 8 * j + gq;
            const int sq = (c * inv) >> 16;  // c / nrows (exact for c < 16)
            const int t = c < ncol ? c - sq * it.nrows : 0, s = c < ncol ? sq : 0;
            bp[j] = c < ncol ? S.bufs + (b * kPassRows + t) * S.XRB + HDR + s * R::PB + tq * 8 : S.zero + tq * 8;
        }
        T.ev(2, 3, it, PH);
        mbar_wait(&S.bfull[b], (seq / kBufs) & 1);
        T.ev(2, 0, it, PH);
        int acc[G][kMaxNT][4];
#pragma unroll
        for (int a = 0; a < G; ++a)
#pragma unroll
            for (int j = 0; j < kMaxNT; ++j)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[a][j][q] = 0;
        for (int u = 0; u < Q.nunits; ++u) {
            mbar_wait(&S.full[slot], sph);
            T.ev(5, u == 0 ? 0 : 1, it, PH);
            const uint8_t* U = S.ring + size_t(slot) * C::UB;
            const int ns = min(C::US, Q.nst - u * C::US);
            if (g.dbg == 1) {
            } else if (NT == 1) unit_mma<BITS, 1>(U, ns, u * C::US, r0, tq, bp, acc);
            else unit_mma<BITS, 2>(U, ns, u * C::US, r0, tq, bp, acc);
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.empty[slot]);
            if (++slot == S.NU) { slot = 0; sph ^= 1; }
        }
        T.ev(2, 1, it, PH);
        if (lane == 0) {
            mbar_arrive(&S.bempty[b]);
            mbar_wait(&S.sempty[sb], ((seq >> 1) & 1) ^ 1);
        }
        T.ev(2, 4, it, PH);
        __syncwarp();
        // groups -> D * Sum_k u * digit per (channel, column): exact in int32 for 1024-k chunks
        int* sc = S.scr + sb * TILE_N * kScrStride;
#pragma unroll
        for (int j = 0; j < kMaxNT; ++j) {
            if (j >= NT) break;
#pragma unroll
            for (int hq = 0; hq < 2; ++hq) {
                int s0 = 0, s1 = 0;
#pragma unroll
                for (int a = 0; a < G; ++a) {
                    s0 += FR::mult(a) * acc[a][j][2 * hq];
                    s1 += FR::mult(a) * acc[a][j][2 * hq + 1];
                }
                *reinterpret_cast<int2*>(sc + (r0 + 8 * hq) * kScrStride + 8 * j + 2 * tq) = make_int2(s0, s1);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.sfull[sb]);
    }
}

// ===== epilogue: group grp takes the items whose CTA sequence number is grp mod 2;
// thread = channel. seq0 = sequence number of this phase's first item.
template <int BITS, int PH>
__device__ __forceinline__ void epilogue(const GemvArgs& g, const Plan& P, const GemvSmem& S, const PhaseGeo& Q,
                                         int seq0, int grp, uint8_t* stg, bool fused, Tracer& T) {
    using FR = Frag<BITS>;
    using R = RB<BITS>;
    constexpr int F = FR::F, PL = planes_of(PH);
    constexpr int LOGD = FR::D == 64 ? 6 : FR::D == 16 ? 4 : 0;
    constexpr long long Z = 1ll << (BITS - 1);
    const GemvTables& TBL = *S.TBL;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ew = (warp - kConsumers) % kEpiWarps;
    const int ch = threadIdx.x - (kConsumers + grp * kEpiWarps) * 32;
    const int ebar = 2 + grp;  // this group's named barrier
    const int CS = Q.CS, rank = Q.rank;
    const int nch2 = (g.Kp2 + kChunkK - 1) / kChunkK;
    const uint32_t red_rank0 = CS > 1 ? map_rank(S.red, 0) : 0u, full_rank0 = CS > 1 ? map_rank(S.red_full, 0) : 0u;
    // fc1: this channel's byte positions in a fc2 stage block (k = ch within the stage)
    int pos0 = 0, pos1 = -1;
    if (PH == 1) {
        const int q = (ch & 63) >> 4, kid = (ch >> 6) * 16 + (ch & 15);
        bool first = true;
        for (int f = 0; f < F; ++f)
            for (int h = 0; h < 2; ++h)
                for (int i = 0; i < 4; ++i)
                    if (FR::kidx(f, h, i) == kid) {
                        const int o = f * 32 + q * 8 + h * 4 + i;
                        if (first) { pos0 = o; first = false; } else pos1 = o;
                    }
    }
    const int k1 = ((grp - seq0) % kEpiGroups + kEpiGroups) % kEpiGroups;
    for (int k = k1, seq = seq0 + k1, i = Q.clu + k1 * Q.nclu; i < Q.nitems;
         k += kEpiGroups, seq += kEpiGroups, i += kEpiGroups * Q.nclu) {
        const GemvItem it = item_of(k, i, TBL, Q);
        const int b = seq % kBufs, sb = seq & 1;
        const int chg = it.mt * TILE_N + ch;
        float sc = 0.f, bias = 0.f, gate[kPassRows] = {0.f, 0.f, 0.f, 0.f};
        int tok[kPassRows] = {0, 0, 0, 0};
        float es = 0.f, eb = 0.f;
        if (rank == 0) {  // epilogue operands, fetched before the wait
            sc = __ldg((PH == 1 ? g.s1 : g.s2) + int64_t(it.e) * Q.Np + chg);
            const float* bb = PH == 1 ? g.b1 : g.b2;
            bias = bb ? __ldg(bb + int64_t(it.e) * Q.Np + chg) : 0.f;
            if (PH == 1) { es = __ldg(g.smax1 + it.e); eb = __ldg(g.bmax1 + it.e); }
            if (PH == 2)
#pragma unroll
                for (int t = 0; t < kPassRows; ++t)
                    if (t < it.nrows) {
                        if (g.self_plan) { gate[t] = TBL.gate[it.row0 + t]; tok[t] = TBL.tok[it.row0 + t]; }
                        else { gate[t] = __ldg(P.perm_gate + it.row0 + t); tok[t] = __ldg(P.perm_token + it.row0 + t); }
                    }
        }
        mbar_wait(&S.sfull[sb], (seq >> 1) & 1);
        T.ev(3, 0, it, PH);
        // exact partial of this chunk: V = Sum_s 256^s S_s - D Z Sum X (int64)
        const uint8_t* rb = S.bufs + b * kPassRows * S.XRB;
        const int* srow = S.scr + sb * TILE_N * kScrStride + ch * kScrStride;
        long long V[kPassRows];
        int pe[kPassRows];
        float l1[kPassRows];
#pragma unroll
        for (int t = 0; t < kPassRows; ++t) {
            V[t] = 0;
            pe[t] = kZeroRow;
            l1[t] = 0.f;
            if (t >= it.nrows) continue;
            const uint8_t* hb = rb + t * S.XRB;
            long long zs = 0;
            if (PH == 1) {
                const XHead1 hd = *reinterpret_cast<const XHead1*>(hb);
                pe[t] = hd.p;
                l1[t] = hd.l1;
                zs = hd.zsum;
            } else {
                pe[t] = *reinterpret_cast<const int*>(hb);
                for (int s = 0; s < Q.nst; ++s) zs += *reinterpret_cast<const long long*>(hb + 64 + 8 * s);
            }
            long long v = -(long long)FR::D * Z * zs;
#pragma unroll
            for (int s = 0; s < PL; ++s) v += (long long)srow[s * it.nrows + t] << (8 * s);
            V[t] = v;
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&S.sempty[sb]);
            mbar_arrive(&S.bempty[b]);
        }
        if (CS > 1) {  // split-K: every rank's partial into rank 0 (DSMEM), fixed-order sum there
            // partials double-buffered by item parity: rank r may run one item ahead of rank 0
            const int q = seq - seq0, rbuf = q & 1;
            const long long* redb = S.red + rbuf * (CS - 1) * TILE_N * kPassRows;
            if (rank != 0) {
                if (lane == 0) wait_cluster(&S.red_empty[rbuf], ((q >> 1) & 1) ^ 1);  // rank 0 took item q - 2
                __syncwarp();
                const uint32_t dst = red_rank0 + uint32_t((rbuf * (CS - 1) + rank - 1) * TILE_N * kPassRows * 8);
#pragma unroll
                for (int t = 0; t < kPassRows; ++t)
                    if (t < it.nrows) st_cluster_s64(dst + uint32_t((ch * kPassRows + t) * 8), V[t]);
                __syncwarp();
                if (lane == 0) arrive_cluster(full_rank0 + uint32_t(rbuf * 8));
                T.ev(3, 2, it, PH);
                continue;
            }
            if (lane == 0) wait_cluster(&S.red_full[rbuf], (q >> 1) & 1);
            __syncwarp();
#pragma unroll
            for (int t = 0; t < kPassRows; ++t)
                if (t < it.nrows)
                    for (int r = 1; r < CS; ++r) V[t] += redb[((r - 1) * TILE_N + ch) * kPassRows + t];
            named_bar_sync(ebar, kEpiWarps * 32);  // every epilogue warp read this buffer
            if (ch >= 1 && ch < CS) arrive_cluster(map_rank(&S.red_empty[rbuf], ch));
        }
        if (PH == 2) {
#pragma unroll
            for (int t = 0; t < kPassRows; ++t) {
                if (t >= it.nrows || chg >= g.d) continue;
                const float y = pe[t] == kZeroRow ? 0.f : scale_pow2(V[t], pe[t] + LOGD);
                const float yg = fmaf(y, sc, bias) * gate[t];
                const int64_t o = int64_t(tok[t]) * g.d + chg;
                if (g.out_acc) atomicAdd(g.out_acc + o, yg);  // top-2: two addends onto zero
                else if (g.out_f16) static_cast<__half*>(g.out)[o] = __float2half_rn(yg);
                else static_cast<float*>(g.out)[o] = yg;
            }
        } else {
            // mid = ReLU(y s + b) in fc2 fixed point -> stage mt % 8 of the rows' fc2 blocks
            long long* zred = reinterpret_cast<long long*>(stg + kPassRows * 4 * R::STG);  // [4 warps][4 rows]
            int p2[kPassRows];
#pragma unroll
            for (int t = 0; t < kPassRows; ++t) {
                p2[t] = kZeroRow;
                long long X2 = 0;
                if (t < it.nrows) {
                    p2[t] = fc2_exp<BITS>(es, eb, l1[t]);
                    const float y = pe[t] == kZeroRow ? 0.f : scale_pow2(V[t], pe[t] + LOGD);
                    const float mid = fmaxf(fmaf(y, sc, bias), 0.0f);  // ReLU, model.cpp:190
                    X2 = p2[t] == kZeroRow ? 0 : __float2int_rn(ldexpf(mid, p2[t]));
                    const uint32_t dg = (uint32_t(int(X2)) + 0x80808080u) ^ 0x80808080u;  // 4 signed digits
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        uint8_t* pl = stg + (t * 4 + s) * R::STG;
                        const uint8_t byte = uint8_t(dg >> (8 * s));
                        pl[pos0] = byte;
                        if (pos1 >= 0) pl[pos1] = byte;
                    }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) X2 += __shfl_xor_sync(0xffffffffu, X2, off);
                if (lane == 0) zred[ew * kPassRows + t] = X2;
            }
            named_bar_sync(ebar, kEpiWarps * 32);  // the stage blocks and warp sums are complete
            const int st2 = it.mt % kChunkStages, c2 = it.mt / kChunkStages;
            constexpr int V16 = R::STG / 16;
            for (int idx = ch; idx < it.nrows * 4 * V16; idx += kEpiWarps * 32) {
                const int t = idx / (4 * V16), s = (idx / V16) & 3, u = idx % V16;
                uint8_t* dst = g.xb + (int64_t(it.row0 + t) * nch2 + c2) * R::XR2 + R::HDR2 + s * R::PB +
                               st2 * R::STG + 16 * u;
                *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(stg + (t * 4 + s) * R::STG + 16 * u);
            }
            if (ch < it.nrows) {
                const int t = ch;
                int p2t = kZeroRow;
#pragma unroll
                for (int u = 0; u < kPassRows; ++u)
                    if (u == t) p2t = p2[u];
                uint8_t* hb = g.xb + (int64_t(it.row0 + t) * nch2 + c2) * R::XR2;
                long long z = 0;
                for (int w = 0; w < kEpiWarps; ++w) z += zred[w * kPassRows + t];
                *reinterpret_cast<long long*>(hb + 64 + 8 * st2) = z;
                *reinterpret_cast<int*>(hb) = p2t;  // the same value from every m-tile of the pass
            }
            named_bar_sync(ebar, kEpiWarps * 32);  // stage blocks / warp sums reused by the next item
            if (fused && ch == 0) {
                // publish: this m-tile's stage of the pass's fc2 row blocks is in global memory
                // (the barrier orders the group's stores before this thread's release)
                fence_proxy_async_global();
                red_release_add(g.ready + it.row0, 1u);
            }
        }
        T.ev(3, 2, it, PH);
    }
}

// MODE 1: fc1, 2: fc2 (two grids chained by PDL), 3: fc1 then fc2 in one persistent grid
// (decode with the self plan and a one-CTA fc1 chunk: no second launch, no second
// prologue; a cluster starts fc2 as soon as its own fc1 items are done, each fc2 item
// waiting only for its pass's readiness counter).
template <int BITS, int MODE>
__global__ void __launch_bounds__(kGemvThreads, 1) k_gemv(GemvArgs g, Plan P) {
    constexpr bool FUSED = MODE == 3;
    constexpr int PH0 = MODE == 2 ? 2 : 1;  // the first (or only) phase
    using C = Cfg<BITS>;
    using L = Layout<BITS, FUSED ? 0 : MODE>;
    constexpr int XR0 = PH0 == 1 ? RB<BITS>::XR1 : RB<BITS>::XR2;
    extern __shared__ __align__(128) uint8_t smem[];
    if (MODE != 1 && threadIdx.x == 0) pdl_trigger();  // the next forward's k_xrows may become resident
    const int CS = int(cluster_nctas()), rank = int(cta_rank());
    GemvSmem S;
    S.NU = L::nu(CS);
    S.XRB = L::XR;
    S.bufs = smem;
    S.zero = smem + L::O_ZERO;
    S.scr = reinterpret_cast<int*>(smem + L::O_SCR);
    S.stg = smem + L::O_STG;
    S.TBL = reinterpret_cast<GemvTables*>(smem + L::O_TAB);
    S.red = reinterpret_cast<long long*>(smem + L::O_RED);
    S.ring = smem + L::ring_off(CS);
    S.full = reinterpret_cast<uint64_t*>(smem + L::O_BARS);
    S.empty = S.full + S.NU;
    S.bfull = S.empty + S.NU;
    S.bempty = S.bfull + kBufs;
    S.sfull = S.bempty + kBufs;
    S.sempty = S.sfull + kScrBufs;
    S.red_full = S.sempty + kScrBufs;  // [2] rank 0: every other rank's partials of the item landed
    S.red_empty = S.red_full + 2;      // [2] rank r: rank 0 consumed that buffer
    GemvTables& TBL = *S.TBL;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kSlots = kTraceCap / 2;
    // trace rows: fc1 events in the first half of each CTA row, fc2 in the second
    unsigned long long* trow = g.trace ? g.trace + size_t(blockIdx.x) * kTraceCap * 2 : nullptr;
    unsigned long long* tr = trow ? trow + (PH0 == 2 ? kTraceCap : 0) : nullptr;
    unsigned long long* tr2 = FUSED && trow ? trow + kTraceCap : nullptr;
    if (threadIdx.x == 0) {  // anchors: kernel entry
        if (tr) { tr[0] = gtime_ns(); tr[1] = clock64(); }
        if (tr2) { tr2[0] = gtime_ns(); tr2[1] = clock64(); }
    }
    // first phase: its split-K cluster (fused fc1: every CTA on its own); fused fc2: the cluster
    PhaseGeo G1 = phase_geo<BITS, PH0>(g, FUSED ? 1 : CS, FUSED ? 0 : rank, FUSED ? int(blockIdx.x) : int(blockIdx.x) / CS,
                                       FUSED ? int(gridDim.x) : int(gridDim.x) / CS);
    PhaseGeo G2 = phase_geo<BITS, 2>(g, CS, rank, int(blockIdx.x) / CS, int(gridDim.x) / CS);
    const int tsc = FUSED ? G1.nmt : 1;  // fused: TBL.start counts passes (the phases differ in m-tiles)
    int early_units = 0;     // producer: weight units of this CTA's first item issued before the CTA barrier
    bool early_rows = false; // producer: its fc1 row blocks too
    for (int i = threadIdx.x; i < L::ZERO / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(const_cast<uint8_t*>(S.zero))[i] = make_uint4(0u, 0u, 0u, 0u);
    if (warp == kProdWarp) {
        // The producer owns the barriers' initialisation, builds the item tables and starts
        // its first item before the CTA-wide synchronisation. Self plan: the build, the
        // first issue and the item cache run twice through the same code — a dry pass while
        // the router still runs (this grid launched early, PDL), then the real one: the
        // dry pass pulls the cold prologue code into the instruction cache (cold, the real
        // pass took ~3x its warm time).
        if (lane == 0) {
            for (int s = 0; s < S.NU; ++s) { mbar_init(&S.full[s], 1); mbar_init(&S.empty[s], kConsumers); }
            for (int b = 0; b < kBufs; ++b) { mbar_init(&S.bfull[b], 1); mbar_init(&S.bempty[b], kConsumers + kEpiWarps); }
            for (int b = 0; b < kScrBufs; ++b) { mbar_init(&S.sfull[b], kConsumers); mbar_init(&S.sempty[b], kEpiWarps); }
            for (int b = 0; b < 2; ++b) {
                mbar_init(&S.red_full[b], kEpiWarps * max(CS - 1, 1));
                mbar_init(&S.red_empty[b], 1);
            }
            fence_barrier_init();
        }
        __syncwarp();
#pragma unroll 1
        for (int pass = g.self_plan ? 0 : 1; pass < 2; ++pass) {
            const bool real = pass == 1;
            if (real && PH0 == 1) pdl_wait();  // routing plan and fc1 row blocks
            int e0 = -1, mt0 = 0, row00 = 0, nrows0 = 0;  // this CTA's first item, if any
            if (g.self_plan) {
                build_tables_self(TBL, P, int(g.T * g.topk), g.E, g.topk, FUSED ? 1 : G1.nmt, lane);
                if (real && tr && lane == 0) { tr[6] = clock64(); tr[7] = 7ull << 60 | 2ull << 56 | (unsigned long long)PH0 << 48 | 1ull; }
                const int n = TBL.n;
                if (G1.clu < TBL.start[n] * tsc) {
                    const GemvItem it = item_at(G1.clu, TBL, n, G1.nmt, tsc);
                    e0 = it.e; mt0 = it.mt; row00 = it.row0; nrows0 = it.nrows;
                }
            } else {
                const int n = P.gtab[0].x;
                const int4 v = P.gtab[1 + lane];
                if (n > 0 && n <= 32) {
                    const int np = lane < n ? G1.nmt * ((v.y + kPassRows - 1) / kPassRows) : 0;
                    int incl = np;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, off);
                        if (lane >= off) incl += y;
                    }
                    const unsigned own = __ballot_sync(0xffffffffu, lane < n && incl - np <= G1.clu && G1.clu < incl);
                    if (own) {
                        const int src = __ffs(own) - 1;
                        const int cnt = __shfl_sync(0xffffffffu, v.y, src);
                        const int off0 = __shfl_sync(0xffffffffu, v.z, src), st0 = __shfl_sync(0xffffffffu, incl - np, src);
                        const int r = G1.clu - st0, pass1 = r / G1.nmt;
                        e0 = __shfl_sync(0xffffffffu, v.x, src);
                        mt0 = r - pass1 * G1.nmt;
                        row00 = off0 + pass1 * kPassRows;
                        nrows0 = min(kPassRows, cnt - pass1 * kPassRows);
                    }
                }
            }
            if (e0 >= 0) {
                const uint8_t* wb = G1.wbase0 + int64_t(e0) * G1.wstride +
                                    (int64_t(mt0) * (G1.Kp / TILE_K) + G1.k0 / TILE_K) * C::TB;
                early_units = min(G1.nunits, S.NU);
                if (lane == 0 && real) {
                    const uint64_t pol = policy_evict_first();
                    for (int u = 0; u < early_units; ++u) {
                        const int bytes = min(C::US, G1.nst - u * C::US) * C::SB;
                        mbar_arrive_expect_tx(&S.full[u], uint32_t(bytes));
                        bulk_g2s_hint(S.ring + size_t(u) * C::UB, wb + int64_t(u) * C::UB, uint32_t(bytes), &S.full[u], pol);
                    }
                }
                if (PH0 == 1) {
                    const int tok = lane < nrows0 ? (g.self_plan ? TBL.tok[row00 + lane] : P.perm_token[row00 + lane]) : 0;
                    if (lane == 0 && real) mbar_arrive_expect_tx(&S.bfull[0], uint32_t(nrows0 * XR0));
                    __syncwarp();
                    if (lane < nrows0 && real)
                        bulk_g2s(S.bufs + lane * S.XRB, g.xr + (int64_t(tok) * g.nch1 + G1.rank) * XR0, uint32_t(XR0),
                                 &S.bfull[0]);
                    early_rows = real;
                }
                if (real && tr && lane == 0) { tr[8] = clock64(); tr[9] = 7ull << 60 | 3ull << 56 | (unsigned long long)PH0 << 48 | 1ull; }
            }
            if (!real) early_units = 0;
            if (g.self_plan) {
                __syncwarp();
                fill_items(TBL, G1, G2, tsc, FUSED, lane, 32);
            }
        }
    }
    if (PH0 == 1 && warp != kProdWarp) pdl_wait();  // every thread that reads the plan waits for it
    if (tr && threadIdx.x == 0) { tr[2] = clock64(); tr[3] = 7ull << 60 | 0ull << 56 | (unsigned long long)PH0 << 48 | 1ull; }
    if (warp == 0 && !g.self_plan) {
        build_tables(TBL, P, G1.nmt, lane, PH0 == 1 ? g.T * g.topk : 0);
        __syncwarp();
        fill_items(TBL, G1, G2, tsc, FUSED, lane, 32);
    }
    __syncthreads();
    finish_geo(TBL, G1, G2, tsc, FUSED);
    // Split cluster barrier: this CTA's barriers are initialised (arrive here); a thread waits
    // only before its first remote access (the split-K epilogue), so no role stalls on the
    // slowest peer's prologue.
    if (CS > 1) cluster_arrive_relaxed();
    if (MODE == 1 && threadIdx.x == 0) pdl_trigger();  // the fc2 grid may launch as CTAs retire (one thread per CTA)
    if (tr && threadIdx.x == 0) { tr[4] = clock64(); tr[5] = 7ull << 60 | 1ull << 56 | (unsigned long long)PH0 << 48 | 1ull; }

    if (warp == kProdWarp) {
        if (lane == 0) {
            int slot = early_units, sph = 0, seq = 0;
            if (slot == S.NU) { slot = 0; sph = 1; }
            bool waited = PH0 == 1;
            Tracer T1 = tracer(tr, 192, kSlots - 1);
            produce<BITS, PH0>(g, P, S, G1, slot, sph, seq, early_units, early_rows, false, waited, T1);
            if (FUSED) {
                Tracer T2 = tracer(tr2, 192, kSlots - 1);
                produce<BITS, 2>(g, P, S, G2, slot, sph, seq, 0, false, true, waited, T2);
            }
            if (!waited) pdl_wait();
        }
        __syncwarp();
        if (CS > 1) cluster_wait_acquire();
    } else if (warp < kConsumers) {
        int slot = 0, sph = 0, seq = 0;
        Tracer T1 = tracer(threadIdx.x == 0 ? tr : nullptr, 6, 128);
        consume<BITS, PH0>(g, S, G1, slot, sph, seq, warp, lane, T1);
        if (FUSED) {
            Tracer T2 = tracer(threadIdx.x == 0 ? tr2 : nullptr, 6, 128);
            consume<BITS, 2>(g, S, G2, slot, sph, seq, warp, lane, T2);
        }
        if (CS > 1) cluster_wait_acquire();
    } else {
        const int grp = (warp - kConsumers) / kEpiWarps;
        const bool lead = threadIdx.x == (kConsumers + grp * kEpiWarps) * 32 && grp == 0;
        Tracer T1 = tracer(lead ? tr : nullptr, 128, 192);
        if (!FUSED && CS > 1) cluster_wait_acquire();  // every peer's barriers initialised
        epilogue<BITS, PH0>(g, P, S, G1, 0, grp, S.stg + grp * L::STG1, FUSED, T1);
        if (FUSED && CS > 1) cluster_wait_acquire();
        if (FUSED) {
            const int n1 = G1.clu < G1.nitems ? (G1.nitems - G1.clu + G1.nclu - 1) / G1.nclu : 0;
            Tracer T2 = tracer(lead ? tr2 : nullptr, 128, 192);
            epilogue<BITS, 2>(g, P, S, G2, n1, grp, nullptr, false, T2);
        }
    }
    if (CS > 1) cluster_sync();  // no CTA leaves while a peer may still write its shared memory
    if (threadIdx.x == 0) {
        if (tr) { tr[2 * (kSlots - 1)] = gtime_ns(); tr[2 * (kSlots - 1) + 1] = clock64(); }
        if (tr2) { tr2[2 * (kSlots - 1)] = gtime_ns(); tr2[2 * (kSlots - 1) + 1] = clock64(); }
    }
}

// ---- launch -----------------------------------------------------------------------------
namespace {
template <class K>
int active_clusters(K kern, int cs, size_t smem, int threads, int num_sms) {
    if (cs == 1) return num_sms;
    cudaLaunchConfig_t q{};
    q.gridDim = dim3(unsigned(num_sms / cs * cs));
    q.blockDim = dim3(threads);
    q.dynamicSmemBytes = smem;
    cudaLaunchAttribute qa[1];
    qa[0].id = cudaLaunchAttributeClusterDimension;
    qa[0].val.clusterDim.x = cs;
    qa[0].val.clusterDim.y = 1;
    qa[0].val.clusterDim.z = 1;
    q.attrs = qa;
    q.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess || n <= 0) n = num_sms / cs;
    return std::min(n, num_sms / cs);
}

template <int BITS, int MODE>
cudaError_t launch_phase(const GemvArgs& g, const Plan& P, cudaStream_t st, int num_sms) {
    using L = Layout<BITS, MODE == 3 ? 0 : MODE>;
    auto kern = k_gemv<BITS, MODE>;
    const int Kp = MODE == 1 ? g.Kp1 : g.Kp2;
    const int cs = (Kp + kChunkK - 1) / kChunkK;
    const int smem = L::total(cs);
    static bool configured_dev[kMaxDevices] = {};
    static int ncl_dev[kMaxDevices][kMaxCluster + 1] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int di = dev < kMaxDevices ? dev : 0;
    int* ncl = ncl_dev[di];
    if (!configured_dev[di]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
        if (e != cudaSuccess) return e;
        configured_dev[di] = true;
    }
    if (ncl[cs] == 0) ncl[cs] = active_clusters(kern, cs, smem, kGemvThreads, num_sms);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(ncl[cs] * cs));
    cfg.blockDim = dim3(kGemvThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(cs);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, g, P);
}

template <int BITS>
cudaError_t launch_gemv_t(const GemvArgs& g, const Plan& P, cudaStream_t st, int num_sms) {
    // fused: every fc1 item must fit one CTA (its cluster is the fc2 one) and the per-pass
    // readiness counters (indexed by the pass's first permuted row) cover the self plan
    if (g.ready && g.self_plan && g.Kp1 <= kChunkK) return launch_phase<BITS, 3>(g, P, st, num_sms);
    cudaError_t e = launch_phase<BITS, 1>(g, P, st, num_sms);
    if (e != cudaSuccess) return e;
    return launch_phase<BITS, 2>(g, P, st, num_sms);
}
}  // namespace

bool gemv_supported(int Kp1, int Kp2) {
    return Kp1 <= kMaxCluster * kChunkK && Kp2 <= kMaxCluster * kChunkK && Kp2 >= kStageK;
}
int64_t gemv_xr_bytes(int bits) {
    switch (bits) {
        case 2: return RB<2>::XR1;
        case 3: return RB<3>::XR1;
        case 4: return RB<4>::XR1;
    }
    return RB<8>::XR1;
}
int64_t gemv_xb_bytes(int bits) {
    switch (bits) {
        case 2: return RB<2>::XR2;
        case 3: return RB<3>::XR2;
        case 4: return RB<4>::XR2;
    }
    return RB<8>::XR2;
}
int gemv_chunks(int Kp) { return (Kp + kChunkK - 1) / kChunkK; }

cudaError_t launch_gemv(int bits, const GemvArgs& g, const Plan& P, cudaStream_t st, int num_sms) {
    if (!gemv_supported(g.Kp1, g.Kp2)) return cudaErrorInvalidValue;
    switch (bits) {
        case 2: return launch_gemv_t<2>(g, P, st, num_sms);
        case 3: return launch_gemv_t<3>(g, P, st, num_sms);
        case 4: return launch_gemv_t<4>(g, P, st, num_sms);
        case 8: return launch_gemv_t<8>(g, P, st, num_sms);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_xrows(int bits, const XrowArgs& a, cudaStream_t st) {
    if (a.T <= 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((a.T * a.nch1 + 3) / 4));
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    switch (bits) {
        case 2: return cudaLaunchKernelEx(&cfg, k_xrows<2>, a);
        case 3: return cudaLaunchKernelEx(&cfg, k_xrows<3>, a);
        case 4: return cudaLaunchKernelEx(&cfg, k_xrows<4>, a);
        case 8: return cudaLaunchKernelEx(&cfg, k_xrows<8>, a);
        default: return cudaErrorInvalidValue;
    }
}

// Per expert: max fc1 scale and max |fc1 bias| — the constants of the fc2
// fixed-point bound (bank creation).
__global__ void k_expert_max(const float* __restrict__ s1, const float* __restrict__ b1, int Np1, float* smax,
                             float* bmax) {
    const int e = blockIdx.x;
    float ms = 0.f, mb = 0.f;
    for (int n = threadIdx.x; n < Np1; n += blockDim.x) {
        ms = fmaxf(ms, fabsf(s1[int64_t(e) * Np1 + n]));
        if (b1) mb = fmaxf(mb, fabsf(b1[int64_t(e) * Np1 + n]));
    }
    for (int off = 16; off > 0; off >>= 1) {
        ms = fmaxf(ms, __shfl_xor_sync(0xffffffffu, ms, off));
        mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, off));
    }
    __shared__ float red[2][32];
    if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = ms; red[1][threadIdx.x >> 5] = mb; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) { ms = fmaxf(ms, red[0][w]); mb = fmaxf(mb, red[1][w]); }
        smax[e] = ms;
        bmax[e] = mb;
    }
}

cudaError_t launch_expert_max(const float* s1, const float* b1, int E, int Np1, float* smax, float* bmax,
                              cudaStream_t st) {
    k_expert_max<<<E, 256, 0, st>>>(s1, b1, Np1, smax, bmax);
    return cudaGetLastError();
}

}  // namespace moqe_gpu
