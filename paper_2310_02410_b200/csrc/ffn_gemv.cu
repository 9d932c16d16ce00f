// ffn_gemv.cu — decode path: expert FFN (fc1 -> ReLU -> fc2 -> gate combine)
// as two persistent weight-streaming kernels (one per layer of the FFN),
// chained with programmatic dependent launch (PDL).
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
// Work: an item is (expert, row pass, 128-channel m-tile); its K is split into
// 1024-k chunks, one per CTA of a thread-block cluster (fc1: d/1024 CTAs, fc2:
// f/1024). Each CTA streams its chunk's packed tiles — one contiguous stripe —
// with TMA bulk copies of >= 16 KB (smaller copies cap the chip at 1-3.6 TB/s,
// profiles/round1/tma_copy_size.md), runs the IMMA k-loop, and sends its exact
// int64 partial sums to cluster rank 0 through distributed shared memory; rank 0
// finishes the item. Items are statically scheduled over the clusters (all the
// same size), so there are no tickets and no cross-cluster synchronisation.
//   fc1 roles: warps 0-7 consumers (16 channels each), 8-10 builders (token rows
//     -> digit fragments in smem, two items ahead), 11 producer (weights).
//     Rank 0's epilogue writes fc2's fragments + Sum X parts to global memory.
//   fc2 roles: warps 0-7 consumers, 8 producer (weights, then each item's
//     fragment slot, issued after the PDL wait on fc1); rank 0 writes the
//     gate-weighted output rows (exactly one writer per element: deterministic).
#include <cuda_fp16.h>

#include <algorithm>

#include "codec.cuh"
#include "frag.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace moqe_gpu {

constexpr int kStageK = 2 * TILE_K;  // k per IMMA stage (2 tiles)
constexpr int kChunkK = 1024;        // k per CTA of a cluster
constexpr int kChunkStages = kChunkK / kStageK;
constexpr int kMaxCluster = 8;
constexpr int kPassRows = 4;         // token rows per item pass
constexpr int kMaxNT = 2;            // n8 column tiles (4 rows x 4 planes = 16 columns)
constexpr int kScrCols = 8 * kMaxNT;
constexpr int kMaxListed = 256;
constexpr int kConsumers = 8;        // consumer warps: 16 channels (one m16 block) each
constexpr int kBuilders = 3;         // fc1 fragment builders (= fragment buffers)
constexpr int kBufs = 3;             // fragment buffers
constexpr int kHead = 352;           // fragment buffer / fc2 slot head (see below)
constexpr int kZeroRow = -0x40000000;  // exponent sentinel: the row is (numerically) zero

__host__ __device__ constexpr int planes_of(int phase) { return phase == 1 ? 3 : 4; }
__host__ __device__ constexpr int nt_of(int phase, int rows) { return (planes_of(phase) * rows + 7) / 8; }
__host__ __device__ constexpr int w_of(int phase, int nt) { return 8 * nt / planes_of(phase); }
__host__ __device__ constexpr int threads_of(int phase) {
    return (phase == 1 ? kConsumers + kBuilders + 1 : kConsumers + 1) * 32;
}
template <int BITS>
__host__ __device__ constexpr int unit_stages() { return BITS == 8 ? 2 : 4; }  // >= 16 KB per weight copy

// Fragment buffer head (352 bytes):
//   fc1 (built in smem): p[4] (row exponent), zsum[4] (Sum X of the chunk), l1[4] (|x|_1 of the row)
//   fc2 slot (global, copied with the fragments): p[4] = p2, zpart[8 stages][4 rows] (Sum X2 per fc1 item)
struct __align__(16) Head {
    int p[4];
    int pad0[4];
    long long zsum[4];
    float l1[4];
    int pad1[4];
    long long zpart[kChunkStages][4];
};
static_assert(sizeof(Head) == kHead, "head layout");

template <int BITS>
struct Cfg {
    static constexpr int F = Frag<BITS>::F;
    static constexpr int TB = tile_bytes(BITS);
    static constexpr int SB = 2 * TB;                             // one IMMA stage of weights
    static constexpr int US = unit_stages<BITS>();
    static constexpr int UB = US * SB;                            // one weight copy
    static constexpr int BBUF = kChunkStages * F * kMaxNT * 256;  // fragments of a 1024-k chunk
    static constexpr int64_t SLOT = kHead + BBUF;                 // fc2 fragment slot in global memory
};

struct GemvItem {
    int e, mt, row0, nrows, gp;  // gp: global row-pass index (fc2 fragment slots); e < 0: none
};

struct GemvTables {
    int list[kMaxListed], cnt[kMaxListed], off[kMaxListed];
    int pst[kMaxListed + 1];    // row-pass prefix per listed expert
    int start[kMaxListed + 1];  // item prefix per listed expert
};

__device__ __forceinline__ int find_listed(const int* st, int n, int v) {  // largest a with st[a] <= v
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (st[mid] <= v) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Item tables from the plan (one warp: lane-parallel loads, serial prefix).
__device__ void build_tables(GemvTables& T, const Plan& P, int n_gemv, int nmt, int lane) {
    for (int a = lane; a < n_gemv; a += 32) {
        const int e = P.gemv_list[a];
        T.list[a] = e;
        T.cnt[a] = P.counts[e];
        T.off[a] = P.offsets[e];
    }
    __syncwarp();
    if (lane == 0) {
        int t = 0, tp = 0;
        for (int a = 0; a < n_gemv; ++a) {
            const int np = (T.cnt[a] + kPassRows - 1) / kPassRows;
            T.pst[a] = tp;
            T.start[a] = t;
            tp += np;
            t += nmt * np;
        }
        T.pst[n_gemv] = tp;
        T.start[n_gemv] = t;
    }
}

// Item i (expert-major: expert, pass, m-tile).
__device__ GemvItem item_at(int i, const GemvTables& T, int n_gemv, int nmt) {
    GemvItem it{};
    if (i >= T.start[n_gemv]) { it.e = -1; return it; }
    const int a = find_listed(T.start, n_gemv, i);
    const int r = i - T.start[a];
    const int pass = r / nmt;
    it.e = T.list[a];
    it.mt = r % nmt;
    it.row0 = T.off[a] + pass * kPassRows;
    it.nrows = min(kPassRows, T.cnt[a] - pass * kPassRows);
    it.gp = T.pst[a] + pass;
    return it;
}

// ---- optional event trace (diagnostics; off unless the bank enables it) ----------------
__device__ __forceinline__ void trace_ev(unsigned long long* trace, unsigned* cnt, int role, int ev,
                                         const GemvItem& it, int phase) {
    if (trace == nullptr) return;
    const unsigned i = atomicAdd(cnt, 1u);
    if (i >= unsigned(kTraceCap / 2)) return;
    unsigned long long* p = trace + (size_t(blockIdx.x) * kTraceCap + i) * 2;
    p[0] = gtime_ns();
    p[1] = (unsigned long long)role << 60 | (unsigned long long)ev << 56 | (unsigned long long)phase << 48 |
           (unsigned long long)(it.e & 0xffff) << 32 | (unsigned long long)(it.mt & 0xfff) << 20 |
           (unsigned long long)(it.nrows & 0xf) << 16 | (unsigned long long)(clock64() & 0xffff);
}

// ---- fc1 builders: token rows -> 3-plane digit fragments of one 1024-k chunk ----------
// One warp per row; lane = (stage st, quad tq) owns the 32 activations that quad's
// IMMA lanes meet in stage st of the chunk. The row maximum and |x|_1 cover the
// whole row (every CTA of the cluster derives the same exponent).
template <int BITS>
__device__ void build_row(const GemvArgs& g, const Plan& P, const GemvItem& it, int t, int lane, bool vec_h,
                          int k0, int nst, uint8_t* bb, Head& hd) {
    using FR = Frag<BITS>;
    constexpr int F = FR::F;
    const int NT = nt_of(1, it.nrows), W = w_of(1, NT);
    const int st = lane >> 2, tq = lane & 3;
    const int64_t tok = P.perm_token[it.row0 + t];
    auto load16 = [&](int k, float* v) {  // 16 activations from k (zeros beyond d)
        if (vec_h) {
            const __half* row = static_cast<const __half*>(g.h) + tok * g.d;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                uint4 w = make_uint4(0u, 0u, 0u, 0u);
                if (k + 8 * q < g.d) w = __ldg(reinterpret_cast<const uint4*>(row + k + 8 * q));  // d % 8 == 0
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
            for (int i = 0; i < 16; ++i) {
                float x = 0.f;
                if (k + i < g.d)  // activations enter as fp16 values (the GEMM path's x_perm is fp16 too)
                    x = g.h_f16 ? __half2float(static_cast<const __half*>(g.h)[tok * g.d + k + i])
                                : __half2float(__float2half_rn(static_cast<const float*>(g.h)[tok * g.d + k + i]));
                v[i] = x;
            }
        }
    };
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.f;
    const bool act = st < nst;
    if (act) {
        load16(k0 + st * kStageK + 16 * tq, v);
        load16(k0 + st * kStageK + 64 + 16 * tq, v + 16);
    }
    float m = 0.f, l1 = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) { m = fmaxf(m, fabsf(v[i])); l1 += fabsf(v[i]); }
    // the rest of the row (other chunks of the cluster): maximum and |x|_1 only
    for (int k = lane * 16; k < g.Kp1; k += 32 * 16) {
        if (k >= k0 && k < k0 + kChunkK) continue;
        float u[16];
        load16(k, u);
#pragma unroll
        for (int i = 0; i < 16; ++i) { m = fmaxf(m, fabsf(u[i])); l1 += fabsf(u[i]); }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    // |x| * 2^p < 2^22 (three digits); rows below 2^-100 count as zero
    const int p = m < 0x1p-100f ? kZeroRow : 21 - ilogbf(m);
    const float sc = p == kZeroRow ? 0.f : exp2f(float(p));
    uint32_t D[32];
    int sum = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const int X = __float2int_rn(v[i] * sc);
        sum += X;
        D[i] = (uint32_t(X) + 0x808080u) ^ 0x808080u;  // bytes 0..2 = signed base-256 digits
    }
    long long zs = sum;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) zs += __shfl_xor_sync(0xffffffffu, zs, off);
    if (lane == 0) {
        hd.p[t] = p;
        hd.zsum[t] = zs;
        hd.l1[t] = l1 * (1.0f + 0x1p-9f);  // covers the fp32 summation error: an upper bound
    }
    if (!act) return;
#pragma unroll
    for (int s = 0; s < 3; ++s) {
        const int col = s * W + t, j = col >> 3, gq = col & 7;
        const uint32_t sel = uint32_t(s) | (uint32_t(4 + s) << 4);
        uint8_t* dst = bb + (size_t(st * F) * NT + j) * 256 + (4 * gq + tq) * 8;
#pragma unroll
        for (int f = 0; f < F; ++f) {
            uint32_t b[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t lo = prmt(D[FR::kidx(f, h, 0)], D[FR::kidx(f, h, 1)], sel);
                const uint32_t hi = prmt(D[FR::kidx(f, h, 2)], D[FR::kidx(f, h, 3)], sel);
                b[h] = prmt(lo, hi, 0x5410u);
            }
            *reinterpret_cast<uint2*>(dst + size_t(f) * NT * 256) = make_uint2(b[0], b[1]);
        }
    }
}

// ---- consumer pieces -------------------------------------------------------------------
// One 128-k stage of one m16 block: LOP3 unpack + IMMA against the stage's B fragments.
template <int BITS, int NT>
__device__ __forceinline__ void stage_mma(const uint8_t* T0, int r0, int lane, const uint8_t* bstage,
                                          int (&acc)[Frag<BITS>::G][kMaxNT][4]) {
    using FR = Frag<BITS>;
    constexpr int F = FR::F;
    uint32_t a[F][4];
    FR::load(T0, T0 + tile_bytes(BITS), r0, lane & 3, a);
    const uint8_t* bs = bstage + lane * 8;
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const uint2 b = *reinterpret_cast<const uint2*>(bs + (f * NT + j) * 256);
            imma(acc[FR::grp(f)][j], a[f], b.x, b.y);
        }
}

template <int BITS, int NT>
__device__ __forceinline__ void unit_mma(const uint8_t* U, int nst_u, int s0, int r0, int lane, const uint8_t* bb,
                                         int (&acc)[Frag<BITS>::G][kMaxNT][4]) {
    constexpr int F = Frag<BITS>::F, SB = 2 * tile_bytes(BITS);
#pragma unroll 2
    for (int s = 0; s < nst_u; ++s) stage_mma<BITS, NT>(U + s * SB, r0, lane, bb + size_t((s0 + s) * F) * NT * 256, acc);
}

__device__ __forceinline__ void scale_bias(const float* s, const float* b, int64_t idx, float& sc, float& bias) {
    sc = __ldg(s + idx);
    bias = b ? __ldg(b + idx) : 0.f;
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
template <int BITS, int PHASE>
struct Layout {
    static constexpr int NU = 116 * 1024 / Cfg<BITS>::UB;  // weight-copy ring slots (~96-112 KB in flight)
    static constexpr size_t RING = size_t(NU) * Cfg<BITS>::UB;
    static constexpr size_t BUFS = size_t(kBufs) * (kHead + Cfg<BITS>::BBUF);
    static constexpr size_t SCR = size_t(TILE_N) * kScrCols * 4;
    static constexpr size_t RED = size_t(kMaxCluster) * TILE_N * kPassRows * 8;  // int64 partials per rank
    static constexpr size_t XS = PHASE == 1 ? TILE_N * kPassRows * 4 + kPassRows * 8 : 0;
    static constexpr size_t BARS = size_t(2 * NU + 2 * kBufs + 2) * 8;
    static constexpr size_t TOTAL = RING + BUFS + SCR + RED + XS + BARS + sizeof(GemvTables) + 64;
};

template <int BITS, int PHASE>
__global__ void __launch_bounds__(threads_of(PHASE), 1) k_gemv(GemvArgs g, Plan P) {
    using FR = Frag<BITS>;
    using C = Cfg<BITS>;
    using L = Layout<BITS, PHASE>;
    constexpr int F = FR::F, G = FR::G, NU = L::NU, UB = C::UB, US = C::US, SB = C::SB, TB = C::TB;
    constexpr int LOGD = FR::D == 64 ? 6 : FR::D == 16 ? 4 : 0;
    constexpr long long Z = 1ll << (BITS - 1);
    constexpr int PROD = PHASE == 1 ? kConsumers + kBuilders : kConsumers;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* ring = smem;
    uint8_t* bufs = ring + L::RING;                                   // [kBufs][head | fragments]
    int* scr = reinterpret_cast<int*>(bufs + L::BUFS);                 // [128][16]
    long long* red = reinterpret_cast<long long*>(reinterpret_cast<uint8_t*>(scr) + L::SCR);  // [CS][128][4]
    int* xs = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(red) + L::RED);  // fc1: [128][4] + zs[4]
    long long* zs = reinterpret_cast<long long*>(xs + TILE_N * kPassRows);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(xs) + L::XS);
    uint64_t* empty = full + NU;
    uint64_t* bfull = empty + NU;
    uint64_t* bempty = bfull + kBufs;
    uint64_t* red_full = bempty + kBufs;   // rank 0: every rank's partials landed
    uint64_t* red_empty = red_full + 1;    // rank r: rank 0 consumed the previous partials
    GemvTables& TBL = *reinterpret_cast<GemvTables*>(red_empty + 1);
    __shared__ unsigned s_tn;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int CS = int(cluster_nctas()), rank = int(cta_rank());
    const int Kp = PHASE == 1 ? g.Kp1 : g.Kp2;
    const int Np = PHASE == 1 ? g.Np1 : g.Np2;
    const int k0 = rank * kChunkK, nst = (min(kChunkK, Kp - k0) + kStageK - 1) / kStageK;
    const int nunits = (nst + US - 1) / US;
    if (threadIdx.x == 0) {
        s_tn = 0;
        for (int s = 0; s < NU; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kConsumers); }
        for (int b = 0; b < kBufs; ++b) { mbar_init(&bfull[b], 1); mbar_init(&bempty[b], kConsumers); }
        mbar_init(red_full, kConsumers * CS);
        mbar_init(red_empty, 1);
        if (PHASE == 1) for (int t = 0; t < kPassRows; ++t) zs[t] = 0;
        fence_barrier_init();
    }
    if (PHASE == 1) pdl_wait();  // routing plan (fc2: the plan is older than fc1's own wait)
    const int n_gemv = P.meta[0];
    const int nmt = Np / TILE_N;
    if (warp == 0 && n_gemv > 0) build_tables(TBL, P, n_gemv, nmt, lane);
    __syncthreads();
    cluster_sync();  // barriers of every CTA initialised before any remote arrive
    if (PHASE == 1) pdl_trigger();  // the fc2 grid may launch as CTAs of this grid retire
    const int nitems = n_gemv > 0 ? TBL.start[n_gemv] : 0;
    const int clu = int(blockIdx.x) / CS, nclu = int(gridDim.x) / CS;
    const int nchunk2 = (g.Kp2 + kChunkK - 1) / kChunkK;
    // trace rows: fc1 events in the first half of each CTA row, fc2 in the second
    unsigned long long* tr = g.trace ? g.trace + (PHASE == 2 ? kTraceCap : 0) : nullptr;

    if (warp == PROD) {
        // ===== producer: weight copy units (+ fc2: the fragment slot of each item)
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            bool waited = PHASE == 1;
            int slot = 0, sph = 0, seq = 0;
            const uint8_t* wbase0 = PHASE == 1 ? g.w1 : g.w2;
            const int64_t wstride = PHASE == 1 ? g.w1_stride : g.w2_stride;
            for (int i = clu; i < nitems; i += nclu, ++seq) {
                const GemvItem it = item_at(i, TBL, n_gemv, nmt);
                if (PHASE == 2 && seq > 0) {
                    const int buf = seq % kBufs;
                    mbar_wait(&bempty[buf], ((seq / kBufs) & 1) ^ 1);
                    const uint32_t bytes = uint32_t(kHead + F * nt_of(2, it.nrows) * 256 * nst);
                    mbar_arrive_expect_tx(&bfull[buf], bytes);
                    bulk_g2s(bufs + size_t(buf) * (kHead + C::BBUF),
                             g.xb + (int64_t(it.gp) * nchunk2 + rank) * g.xb_slot_bytes, bytes, &bfull[buf]);
                }
                const uint8_t* wb = wbase0 + int64_t(it.e) * wstride + (int64_t(it.mt) * (Kp / TILE_K) + k0 / TILE_K) * TB;
                for (int u = 0; u <= nunits; ++u) {
                    // fc2, first item: its weights stream while fc1 finishes; the fragment
                    // slot (written by fc1) is fetched once the ring is full or the item issued
                    if (PHASE == 2 && seq == 0 && !waited && (u == nunits || u == NU)) {
                        pdl_wait();
                        waited = true;
                        const uint32_t bytes = uint32_t(kHead + F * nt_of(2, it.nrows) * 256 * nst);
                        mbar_arrive_expect_tx(&bfull[0], bytes);
                        bulk_g2s(bufs, g.xb + (int64_t(it.gp) * nchunk2 + rank) * g.xb_slot_bytes, bytes, &bfull[0]);
                    }
                    if (u == nunits) break;
                    const int bytes = min(US, nst - u * US) * SB;
                    mbar_wait(&empty[slot], sph ^ 1);
                    mbar_arrive_expect_tx(&full[slot], uint32_t(bytes));
                    bulk_g2s_hint(ring + size_t(slot) * UB, wb + int64_t(u) * UB, uint32_t(bytes), &full[slot], pol);
                    if (++slot == NU) { slot = 0; sph ^= 1; }
                }
            }
            if (!waited) pdl_wait();
        }
        __syncwarp();
    } else if (PHASE == 1 && warp >= kConsumers) {
        // ===== builders: builder b fills fragment buffer b (every kBufs-th item)
        const int bw = warp - kConsumers;
        const bool vec_h = g.h_f16 && (g.d % 8) == 0 && (reinterpret_cast<uintptr_t>(g.h) & 15) == 0;
        int seq = bw;
        for (int i = clu + bw * nclu; i < nitems; i += kBufs * nclu, seq += kBufs) {
            const GemvItem it = item_at(i, TBL, n_gemv, nmt);
            if (lane == 0) mbar_wait(&bempty[bw], ((seq / kBufs) & 1) ^ 1);
            __syncwarp();
            uint8_t* b = bufs + size_t(bw) * (kHead + C::BBUF);
            Head& hd = *reinterpret_cast<Head*>(b);
            for (int t = 0; t < it.nrows; ++t) build_row<BITS>(g, P, it, t, lane, vec_h, k0, nst, b + kHead, hd);
            __syncwarp();
            if (lane == 0) {
                trace_ev(tr, &s_tn, 1, 1, it, PHASE);
                mbar_arrive(&bfull[bw]);
            }
        }
    } else if (warp < kConsumers) {
        // ===== consumers: warp -> m16 block (16 channels) of the 128-channel item
        const int r = lane & 15;  // epilogue: lane -> channel 16 warp + r, rows (lane >> 4) + 2 u
        const uint32_t red_rank0 = map_rank(red, 0), full_rank0 = map_rank(red_full, 0);
        int slot = 0, sph = 0, seq = 0;
        for (int i = clu; i < nitems; i += nclu, ++seq) {
            const GemvItem it = item_at(i, TBL, n_gemv, nmt);
            const int buf = seq % kBufs;
            const int ch = it.mt * TILE_N + 16 * warp + r;
            float sc = 0.f, bias = 0.f, gate[2] = {0.f, 0.f};  // epilogue operands, fetched early
            int tok[2] = {0, 0};
            float smax = 0.f, bmax = 0.f;
            if (rank == 0) {
                scale_bias(PHASE == 1 ? g.s1 : g.s2, PHASE == 1 ? g.b1 : g.b2, int64_t(it.e) * Np + ch, sc, bias);
                if (PHASE == 1) { smax = __ldg(g.smax1 + it.e); bmax = __ldg(g.bmax1 + it.e); }
                if (PHASE == 2)
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int t = (lane >> 4) + 2 * u;
                        if (t < it.nrows) { gate[u] = P.perm_gate[it.row0 + t]; tok[u] = P.perm_token[it.row0 + t]; }
                    }
            }
            mbar_wait(&bfull[buf], (seq / kBufs) & 1);
            if (threadIdx.x == 0) trace_ev(tr, &s_tn, 2, 0, it, PHASE);
            const uint8_t* bb = bufs + size_t(buf) * (kHead + C::BBUF);
            const Head& hd = *reinterpret_cast<const Head*>(bb);
            const int NT = nt_of(PHASE, it.nrows);
            int acc[G][kMaxNT][4];
#pragma unroll
            for (int a = 0; a < G; ++a)
#pragma unroll
                for (int j = 0; j < kMaxNT; ++j)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[a][j][q] = 0;
            const int r0 = 16 * warp + (lane >> 2);
            for (int u = 0; u < nunits; ++u) {
                mbar_wait(&full[slot], sph);
                const uint8_t* U = ring + size_t(slot) * UB;
                const int ns = min(US, nst - u * US);
                if (NT == 1) unit_mma<BITS, 1>(U, ns, u * US, r0, lane, bb + kHead, acc);
                else unit_mma<BITS, 2>(U, ns, u * US, r0, lane, bb + kHead, acc);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                if (++slot == NU) { slot = 0; sph ^= 1; }
            }
            if (threadIdx.x == 0) trace_ev(tr, &s_tn, 2, 1, it, PHASE);
            // groups -> D * Sum_k u * digit per (row, column) (exact in int32 for 1024-k chunks)
            {
                const int tq = lane & 3, gq = lane >> 2;
#pragma unroll
                for (int j = 0; j < kMaxNT; ++j) {
                    if (j >= NT) break;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        int s = 0;
#pragma unroll
                        for (int a = 0; a < G; ++a) s += FR::mult(a) * acc[a][j][q];
                        scr[(16 * warp + gq + 8 * (q >> 1)) * kScrCols + 8 * j + 2 * tq + (q & 1)] = s;
                    }
                }
            }
            __syncwarp();
            // this chunk's exact partial: V = Sum_s 256^s S_s - D Z Sum X (int64) -> rank 0
            const int PL = planes_of(PHASE), W = w_of(PHASE, NT);
            const int* wr = scr + (16 * warp + r) * kScrCols;
            if (lane == 0 && rank != 0) wait_cluster(red_empty, (seq & 1) ^ 1);  // rank 0 took the previous item
            __syncwarp();
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int t = (lane >> 4) + 2 * u;
                if (t >= it.nrows) continue;
                long long zsum = 0;
                if (PHASE == 1) {
                    zsum = hd.zsum[t];
                } else {
                    for (int st = 0; st < nst; ++st) zsum += hd.zpart[st][t];
                }
                long long V = -(long long)FR::D * Z * zsum;
                for (int s = 0; s < PL; ++s) V += (long long)wr[s * W + t] << (8 * s);
                const int idx = ((rank * TILE_N) + 16 * warp + r) * kPassRows + t;
                if (rank == 0) red[idx] = V;
                else st_cluster_s64(red_rank0 + uint32_t(idx) * 8u, V);
            }
            // exponents needed by rank 0 after the buffer is recycled
            int pe[2] = {kZeroRow, kZeroRow};
            float l1e[2] = {0.f, 0.f};
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int t = (lane >> 4) + 2 * u;
                if (t < it.nrows) { pe[u] = hd.p[t]; l1e[u] = PHASE == 1 ? hd.l1[t] : 0.f; }
            }
            const float l1row = (PHASE == 1 && threadIdx.x < it.nrows) ? hd.l1[threadIdx.x] : 0.f;
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&bempty[buf]);
                arrive_cluster(full_rank0);  // this warp's partials are in rank 0's smem
            }
            if (threadIdx.x == 0) trace_ev(tr, &s_tn, 2, 3, it, PHASE);
            if (rank != 0) continue;
            // ===== rank 0: reduce the cluster's partials and finish the item
            wait_cluster(red_full, seq & 1);
            if (threadIdx.x == 0) trace_ev(tr, &s_tn, 2, 4, it, PHASE);
            float y[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int t = (lane >> 4) + 2 * u;
                long long V = 0;
                if (t < it.nrows)
                    for (int c = 0; c < CS; ++c) V += red[((c * TILE_N) + 16 * warp + r) * kPassRows + t];
                y[u] = (t >= it.nrows || pe[u] == kZeroRow) ? 0.f : scale_pow2(V, pe[u] + LOGD);
            }
            named_bar_sync(1, kConsumers * 32);  // every warp read red
            if (threadIdx.x == 0) trace_ev(tr, &s_tn, 2, 6, it, PHASE);
            if (threadIdx.x < CS && threadIdx.x > 0) arrive_cluster(map_rank(red_empty, threadIdx.x));
            if (PHASE == 2) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int t = (lane >> 4) + 2 * u;
                    if (t < it.nrows && ch < g.d) {
                        const float yg = fmaf(y[u], sc, bias) * gate[u];
                        const int64_t o = int64_t(tok[u]) * g.d + ch;
                        if (g.out_acc) atomicAdd(g.out_acc + o, yg);  // top-2: two addends onto zero
                        else if (g.out_f16) static_cast<__half*>(g.out)[o] = __float2half_rn(yg);
                        else static_cast<float*>(g.out)[o] = yg;
                    }
                }
            } else {
                // mid = ReLU(y s + b) in fc2 fixed point -> fc2 fragment stage mt % 8 of slot (pass, mt / 8)
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int t = (lane >> 4) + 2 * u;
                    long long X2 = 0;
                    if (t < it.nrows) {
                        const int p2 = fc2_exp<BITS>(smax, bmax, l1e[u]);
                        const float mid = fmaxf(fmaf(y[u], sc, bias), 0.0f);  // ReLU, model.cpp:190
                        X2 = p2 == kZeroRow ? 0 : __float2int_rn(ldexpf(mid, p2));
                        xs[(16 * warp + r) * kPassRows + t] = int(X2);
                    }
#pragma unroll
                    for (int off = 1; off < 16; off <<= 1) X2 += __shfl_xor_sync(0xffffffffu, X2, off);
                    if (r == 0 && t < it.nrows)
                        atomicAdd(reinterpret_cast<unsigned long long*>(&zs[t]), (unsigned long long)X2);
                }
                named_bar_sync(1, kConsumers * 32);  // all 128 channels of X2 are in xs
                if (threadIdx.x == 0) trace_ev(tr, &s_tn, 2, 5, it, PHASE);
                const int NT2 = nt_of(2, it.nrows), W2 = w_of(2, NT2);
                uint8_t* sl = g.xb + (int64_t(it.gp) * nchunk2 + it.mt / kChunkStages) * g.xb_slot_bytes;
                const int st2 = it.mt % kChunkStages;
                uint8_t* bstage = sl + kHead + size_t(st2 * F) * NT2 * 256;
                const int nwords = it.nrows * 4 * 4 * F;
                for (int wd = threadIdx.x; wd < nwords; wd += kConsumers * 32) {
                    const int f = wd % F, s = (wd / F) & 3, tq = (wd / (4 * F)) & 3, t = wd / (16 * F);
                    uint32_t b[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t word = 0;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int k = FR::kidx(f, h, q);  // tile * 16 + code
                            const int X = xs[(64 * (k >> 4) + 16 * tq + (k & 15)) * kPassRows + t];
                            word |= ((((uint32_t(X) + 0x80808080u) ^ 0x80808080u) >> (8 * s)) & 0xffu) << (8 * q);
                        }
                        b[h] = word;
                    }
                    const int col = s * W2 + t, j = col >> 3, gq = col & 7;
                    __stcg(reinterpret_cast<uint2*>(bstage + (size_t(f) * NT2 + j) * 256 + (4 * gq + tq) * 8),
                           make_uint2(b[0], b[1]));
                }
                if (threadIdx.x == 0) trace_ev(tr, &s_tn, 2, 7, it, PHASE);
                if (threadIdx.x < it.nrows) {
                    const int t = threadIdx.x;
                    Head* gh = reinterpret_cast<Head*>(sl);
                    gh->zpart[st2][t] = zs[t];
                    gh->p[t] = fc2_exp<BITS>(smax, bmax, l1row);  // the same value from every m-tile
                }
                named_bar_sync(1, kConsumers * 32);  // xs / zs reuse
                if (threadIdx.x < kPassRows) zs[threadIdx.x] = 0;
            }
            if (threadIdx.x == 0) trace_ev(tr, &s_tn, 2, 2, it, PHASE);
        }
    }
    cluster_sync();  // no CTA leaves while a peer may still write its shared memory
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

template <int BITS, int PHASE>
cudaError_t launch_phase(const GemvArgs& g, const Plan& P, cudaStream_t st, int num_sms) {
    using L = Layout<BITS, PHASE>;
    auto kern = k_gemv<BITS, PHASE>;
    const int Kp = PHASE == 1 ? g.Kp1 : g.Kp2;
    const int cs = (Kp + kChunkK - 1) / kChunkK;
    static bool configured = false;
    static int ncl[kMaxCluster + 1] = {0};
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L::TOTAL));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    if (ncl[cs] == 0) ncl[cs] = active_clusters(kern, cs, L::TOTAL, threads_of(PHASE), num_sms);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(ncl[cs] * cs));
    cfg.blockDim = dim3(threads_of(PHASE));
    cfg.dynamicSmemBytes = L::TOTAL;
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
    cudaError_t e = launch_phase<BITS, 1>(g, P, st, num_sms);
    if (e != cudaSuccess) return e;
    return launch_phase<BITS, 2>(g, P, st, num_sms);
}
}  // namespace

bool gemv_supported(int Kp1, int Kp2) {
    return Kp1 <= kMaxCluster * kChunkK && Kp2 <= kMaxCluster * kChunkK && Kp2 >= kStageK;
}
int64_t gemv_xb_slot_bytes(int bits) {
    switch (bits) {
        case 2: return Cfg<2>::SLOT;
        case 3: return Cfg<3>::SLOT;
        case 4: return Cfg<4>::SLOT;
    }
    return Cfg<8>::SLOT;
}
// every listed expert may end in a partial pass; one slot per (pass, 1024-k chunk of fc2)
int64_t gemv_xb_slots(int64_t rows, int E, int Kp2) {
    return ((rows + kPassRows - 1) / kPassRows + E) * ((Kp2 + kChunkK - 1) / kChunkK);
}

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
