// ffn_gemv.cu — decode path: fused expert FFN (fc1 -> ReLU -> fc2 -> gate
// combine) as ONE persistent, warp-specialised weight-streaming kernel.
//
// Reference: the per-expert loop of moe_ffn_forward proj/src/model.cpp:360-391
// (dequantize :370-375, matmul :381/:384, add_bias/relu :382-385, scatter
// :387-390). The reference re-dequantizes whole experts to f32 (27 ms per
// 4M-element matrix); here packed codes stream from HBM exactly once and are
// never widened beyond 8 bits.
//
// Integer dot products (frag.cuh). A weight code q = u - 2^(b-1) is kept as
// its offset binary u; one LOP3 yields four u8 values u * 2^s that feed IMMA
// m16n8k32 (u8 x s8 -> s32). Activations of a row are a per-row fixed-point
// integer X = rint(x * 2^p) split into signed base-256 digit planes; each
// plane is one MMA column. Sum_k u*X is exact in integers; the zero point
// (2^(b-1) Sum X), the plane weights 256^s and 2^-p are applied once per item
// in fp64, the per-channel scale in the epilogue.
//   fc1 rows (fp16 tokens): 3 planes, p from the row maximum — exact for every
//     activation within 2^11 of the row max.
//   fc2 rows (mid = ReLU(fc1)): 4 planes, p from a rigorous per-row bound
//     |mid| <= max_scale * 2^(b-1) * |x|_1 + max|bias|, so every fc1 item can
//     encode its own 128 output channels (one fc2 k-stage) without waiting for
//     the rest of the row; resolution ~2^-29 of the bound, far finer than the
//     fp32 chain of the reference.
//
// Work items (device-side, no host sync): fc1 (expert, 128-channel m-tile,
// k-chunk, row pass) for every expert in the GEMV list, then fc2 items.
//   warp 12      producer: item tickets, packed weight tiles -> smem ring via
//                TMA bulk copies (evict-first), 2 tiles (128 k) per stage
//   warps 8-10   builders: fc1 item rows -> digit fragments in smem (two items
//                ahead of the consumers, warp per row)
//   warp 11      loader: fc2 item -> waits for the 8 fc1 stage flags of its
//                fragment slot, TMA bulk copy slot -> smem
//   warps 0-7    consumers: 16 output channels each; LOP3 unpack, IMMA;
//                accumulators -> smem scratch (double buffered)
//   warps 13-14  publishers: exact epilogue, scale/bias, fc1 -> fc2 fragment
//                slots (+ ready flags), fc2 -> gate-weighted output; split-K
//                partials reduced in fixed order by the last arriving CTA
// Results are deterministic (integer accumulation, fixed-order reductions).
#include <cuda_fp16.h>

#include "codec.cuh"
#include "frag.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace moqe_gpu {

constexpr int kGemvKC = 1024;        // k per item
constexpr int kStageK = 2 * TILE_K;  // k per ring stage (2 tiles)
constexpr int kStagesPerChunk = kGemvKC / kStageK;
constexpr int kConsumers = 4;        // IMMA warps (32 channels = two m16 blocks each: every B fragment feeds 2 IMMAs)
constexpr int kBlk = 2;              // m16 blocks per consumer warp
constexpr int kBuilders = 3;         // fc1 fragment builders
constexpr int kLoader = kConsumers + kBuilders;
constexpr int kProducer = kLoader + 1;
constexpr int kPublisher = kProducer + 1;
constexpr int kGemvThreads = (kPublisher + 1) * 32;
constexpr int kItemQ = 6;
constexpr int kBBufs = kBuilders;    // fragment buffers (builder warp b owns buffer b); two items of lead
constexpr int kScrBufs = 3;          // accumulator scratch / epilogue buffers (warps may drift two items apart)
constexpr int kPassRows = 4;         // token rows per item pass
constexpr int kMaxNT = 2;            // n8 column tiles per item (4 rows x 4 planes = 16 columns)
constexpr int kMaxListed = 256;
constexpr int kRingBytes = 96 * 1024;
constexpr int kScrCols = 8 * kMaxNT;
constexpr int kZeroRow = -0x40000000;  // exponent sentinel: the row is (numerically) zero

__host__ __device__ constexpr int gemv_ksplit_c(int Kp) { return (Kp + kGemvKC - 1) / kGemvKC; }
__host__ __device__ constexpr int planes_of(int phase) { return phase == 1 ? 3 : 4; }
__host__ __device__ constexpr int nt_of(int phase, int rows) { return (planes_of(phase) * rows + 7) / 8; }
__host__ __device__ constexpr int w_of(int phase, int nt) { return 8 * nt / planes_of(phase); }

template <int BITS>
struct GemvCfg {
    static constexpr int TB = tile_bytes(BITS);
    static constexpr int SB = 2 * TB;                 // ring stage = 2 tiles (128 k)
    static constexpr int NST = kRingBytes / SB;
    static constexpr int F = Frag<BITS>::F;
    static constexpr int BBUF = kStagesPerChunk * F * kMaxNT * 256;  // digit fragments per item
};

struct GemvItem {
    int phase;  // 1 fc1, 2 fc2, 0 end
    int e, mt, ks, row0, nrows, npass, slot;  // slot: fc2 fragment slot (fc1: of the pass's chunk 0)
};

struct GemvTables {
    int list[kMaxListed], cnt[kMaxListed], off[kMaxListed];
    int pst[kMaxListed + 1];                             // row-pass prefix per listed expert
    int start1[kMaxListed + 1], start2[kMaxListed + 1];  // item prefix per listed expert
};

// Per-item fragment meta (128 bytes, copied with the fragments).
struct __align__(16) BufMeta {
    int p[8];                     // row exponent (kZeroRow: zero row)
    unsigned long long zsum[8];   // fc1: Sum_k X per row (fc2 slots keep it per stage, after the fragments)
    float l1[8];                  // fc1: |x|_1 of the row chunk (bounds the fc2 exponent)
};
static_assert(sizeof(BufMeta) == 128, "BufMeta is copied as one 128-byte block");

__device__ __forceinline__ int find_listed(const int* st, int n, int v) {  // largest a with st[a] <= v
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (st[mid] <= v) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Ticket order: fc1 items (expert, pass, m-tile, k-split) then fc2 items.
__device__ GemvItem decode_item(unsigned ticket, const GemvTables& T, int n_gemv, int nmt1, int s1, int nmt2,
                                int s2) {
    GemvItem it{};
    const unsigned c1 = unsigned(T.start1[n_gemv]), c2 = c1 + unsigned(T.start2[n_gemv]);
    int phase, r;
    if (ticket < c1) { phase = 1; r = int(ticket); }
    else if (ticket < c2) { phase = 2; r = int(ticket - c1); }
    else { it.phase = 0; return it; }
    const int* st = phase == 1 ? T.start1 : T.start2;
    const int a = find_listed(st, n_gemv, r);
    const int nmt = phase == 1 ? nmt1 : nmt2, S = phase == 1 ? s1 : s2;
    const int rr = r - st[a];
    const int pass = rr / (nmt * S), r2 = rr % (nmt * S);
    const int n = T.cnt[a];
    it.phase = phase;
    it.e = T.list[a];
    it.mt = r2 / S;
    it.ks = r2 % S;
    it.row0 = T.off[a] + pass * kPassRows;
    it.nrows = min(kPassRows, n - pass * kPassRows);
    it.npass = (n + kPassRows - 1) / kPassRows;
    it.slot = (T.pst[a] + pass) * s2 + (phase == 2 ? it.ks : 0);
    return it;
}

// ---- optional event trace (diagnostics; off unless the bank enables it) ----------------
// event word: role << 60 | ev << 56 | phase << 48 | e << 32 | mt << 16 | ks
__device__ __forceinline__ void trace_ev(const GemvArgs& g, unsigned* cnt, int role, int ev, const GemvItem& it) {
    if (g.trace == nullptr) return;
    const unsigned i = atomicAdd(cnt, 1u);
    if (i >= unsigned(kTraceCap)) return;
    unsigned long long* p = g.trace + (size_t(blockIdx.x) * kTraceCap + i) * 2;
    p[0] = gtime_ns();
    p[1] = (unsigned long long)role << 60 | (unsigned long long)ev << 56 | (unsigned long long)(it.phase & 0xff) << 48 |
           (unsigned long long)(it.e & 0xffff) << 32 | (unsigned long long)(it.mt & 0xffff) << 16 |
           (unsigned long long)(it.ks & 0xffff);
}

// Scatter one lane's 32 digit words (byte s = plane s) into the B fragments of
// one stage: column (t, s) -> n-tile j, group g; lane quad tq.
template <int BITS, int PL>
__device__ __forceinline__ void scatter_digits(const uint32_t (&D)[32], uint8_t* bstage, int NT, int W, int t,
                                               int tq, bool global) {
    using FR = Frag<BITS>;
    constexpr int F = FR::F;
#pragma unroll
    for (int s = 0; s < PL; ++s) {
        const int col = s * W + t, j = col >> 3, gq = col & 7;
        const uint32_t sel = uint32_t(s) | (uint32_t(4 + s) << 4);
        uint8_t* dst = bstage + size_t(j) * 256 + (4 * gq + tq) * 8;
#pragma unroll
        for (int f = 0; f < F; ++f) {
            uint32_t b[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t lo = prmt(D[FR::kidx(f, h, 0)], D[FR::kidx(f, h, 1)], sel);
                const uint32_t hi = prmt(D[FR::kidx(f, h, 2)], D[FR::kidx(f, h, 3)], sel);
                b[h] = prmt(lo, hi, 0x5410u);
            }
            uint2* p = reinterpret_cast<uint2*>(dst + size_t(f) * NT * 256);
            if (global) __stcg(p, make_uint2(b[0], b[1]));
            else *p = make_uint2(b[0], b[1]);
        }
    }
}

// ---- builders: fc1 rows -> 3-plane digit fragments in smem ----------------------------
// One warp per row; lane = (stage st, quad tq) owns the 32 activations that
// quad's IMMA lanes meet in that stage, so the row maximum, Sum X and |x|_1
// are warp reductions.
template <int BITS>
__device__ void build_row(const GemvArgs& g, const Plan& P, const GemvItem& it, int t, int lane, bool vec_h,
                          uint8_t* bb, BufMeta& meta) {
    constexpr int F = Frag<BITS>::F;
    const int k0 = it.ks * kGemvKC;
    const int nst = min(kGemvKC, g.Kp1 - k0) / kStageK;
    const int NT = nt_of(1, it.nrows), W = w_of(1, NT);
    const int st = lane >> 2, tq = lane & 3;
    const bool act = st < nst;
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.f;
    const int kb = k0 + st * kStageK + 16 * tq;  // tile 0 run; tile 1 run at +64
    const int64_t tok = P.perm_token[it.row0 + t];
    if (act) {
        if (vec_h) {
            const __half* row = static_cast<const __half*>(g.h) + tok * g.d;
#pragma unroll
            for (int tile = 0; tile < 2; ++tile)
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int kk = kb + 64 * tile + 8 * q;
                    uint4 w = make_uint4(0u, 0u, 0u, 0u);
                    if (kk < g.d) w = __ldg(reinterpret_cast<const uint4*>(row + kk));  // d % 8 == 0
                    const __half2* h2 = reinterpret_cast<const __half2*>(&w);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float2 f = __half22float2(h2[i]);
                        v[16 * tile + 8 * q + 2 * i] = f.x;
                        v[16 * tile + 8 * q + 2 * i + 1] = f.y;
                    }
                }
        } else {
#pragma unroll
            for (int tile = 0; tile < 2; ++tile)
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int kk = kb + 64 * tile + i;
                    float x = 0.f;
                    if (kk < g.d)  // activations enter as fp16 values (the GEMM path's x_perm is fp16 too)
                        x = g.h_f16 ? __half2float(static_cast<const __half*>(g.h)[tok * g.d + kk])
                                    : __half2float(__float2half_rn(static_cast<const float*>(g.h)[tok * g.d + kk]));
                    v[16 * tile + i] = x;
                }
        }
    }
    float m = 0.f, l1 = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) { m = fmaxf(m, fabsf(v[i])); l1 += fabsf(v[i]); }
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
        meta.p[t] = p;
        meta.zsum[t] = (unsigned long long)zs;
        meta.l1[t] = l1 * (1.0f + 0x1p-9f);  // covers the fp32 summation error: an upper bound
    }
    if (act) scatter_digits<BITS, 3>(D, bb + size_t(st * F) * NT * 256, NT, W, t, tq, false);
}

// ---- consumers ------------------------------------------------------------------------
template <int BITS, int NT>
__device__ __forceinline__ void gemv_mainloop(const uint8_t* ring, const uint8_t* bb, uint64_t* full,
                                              uint64_t* empty, int& stage, int& sphase, int nst, int warp,
                                              int lane, int (&acc)[kBlk][Frag<BITS>::G][kMaxNT][4],
                                              long long* cyc = nullptr) {
    using Cfg = GemvCfg<BITS>;
    using FR = Frag<BITS>;
    constexpr int F = FR::F;
    const int tq = lane & 3, r0 = 16 * kBlk * warp + (lane >> 2);
    auto compute = [&](int stg, int s) {
        const uint8_t* T0 = ring + stg * Cfg::SB;
        uint32_t a[kBlk][F][4];
#pragma unroll
        for (int bk = 0; bk < kBlk; ++bk) FR::load(T0, T0 + Cfg::TB, r0 + 16 * bk, tq, a[bk]);
        const uint8_t* bs = bb + size_t(s * F) * NT * 256 + lane * 8;
#pragma unroll
        for (int f = 0; f < F; ++f)
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const uint2 b = *reinterpret_cast<const uint2*>(bs + (f * NT + j) * 256);
#pragma unroll
                for (int bk = 0; bk < kBlk; ++bk) imma(acc[bk][FR::grp(f)][j], a[bk][f], b.x, b.y);
            }
    };
    // two ring stages per iteration: both waits first, so the second stage's
    // shared-memory loads overlap the first stage's IMMAs
    for (int s = 0; s < nst; s += 2) {
        const bool two = s + 1 < nst;
        const int st0 = stage, ph0 = sphase;
        if (++stage == Cfg::NST) { stage = 0; sphase ^= 1; }
        const int st1 = stage, ph1 = sphase;
        if (two && ++stage == Cfg::NST) { stage = 0; sphase ^= 1; }
        long long c0 = 0;
        if (cyc) c0 = clock64();
        mbar_wait(&full[st0], ph0);
        if (two) mbar_wait(&full[st1], ph1);
        if (cyc) { const long long c1 = clock64(); cyc[0] += c1 - c0; c0 = c1; }
        compute(st0, s);
        if (two) compute(st1, s + 1);
        __syncwarp();
        if (cyc) cyc[1] += clock64() - c0;
        if (lane == 0) {
            mbar_arrive(&empty[st0]);
            if (two) mbar_arrive(&empty[st1]);
        }
    }
}

// ---- epilogue helpers -------------------------------------------------------------------
__device__ __forceinline__ void scale_bias(const GemvArgs& g, bool p1, int e, int ch, float& sc, float& bias) {
    const int Np = p1 ? g.Np1 : g.Np2;
    sc = __ldg((p1 ? g.s1 : g.s2) + int64_t(e) * Np + ch);
    const float* bi = p1 ? g.b1 : g.b2;
    bias = bi ? __ldg(bi + int64_t(e) * Np + ch) : 0.f;
}

// V * 2^-sh in fp32: one rounding (int64 -> fp32), exact power-of-two scale
__device__ __forceinline__ float scale_pow2(long long V, int sh) {
    const float v = float(V);
    return (sh > -127 && sh < 127) ? v * __int_as_float((127 - sh) << 23) : ldexpf(v, -sh);
}

// fc2 output element: y -> scale/bias -> x gate -> output row
__device__ __forceinline__ void fc2_finish(const GemvArgs& g, int ch, float y, float sc, float bias, float gate,
                                           int tok) {
    if (ch >= g.d) return;
    const float yg = fmaf(y, sc, bias) * gate;
    const int64_t o = int64_t(tok) * g.d + ch;
    if (g.out_acc) atomicAdd(g.out_acc + o, yg);
    else if (g.out_f16) static_cast<__half*>(g.out)[o] = __float2half_rn(yg);
    else static_cast<float*>(g.out)[o] = yg;
}

// fc2 exponent of one fc1 row: |mid| <= smax * 2^(b-1) * |x|_1 + bmax, and
// |X| = |mid| * 2^p2 < 2^30 keeps four signed base-256 digits.
template <int BITS>
__device__ __forceinline__ int fc2_exp(float smax, float bmax, float l1) {
    const float bound = (smax * float(1 << (BITS - 1)) * l1 + bmax) * (1.0f + 0x1p-16f);
    return bound < 0x1p-100f ? kZeroRow : 29 - ilogbf(bound);
}
__device__ __forceinline__ int encode_x2(float mid, int p2) {
    return p2 == kZeroRow ? 0 : __float2int_rn(ldexpf(mid, p2));
}

// fc2 fragment words of one stage from the X2 of 128 channels x rows (xs),
// spread over `nthr` threads: word (row t, quad tq, plane s, fragment f).
template <int BITS>
__device__ __forceinline__ void encode_stage(const int* xs, int nrows, uint8_t* bstage, int tid, int nthr) {
    using FR = Frag<BITS>;
    constexpr int F = FR::F;
    const int NT = nt_of(2, nrows), W = w_of(2, NT);
    const int nwords = nrows * 4 * 4 * F;
    for (int w = tid; w < nwords; w += nthr) {
        const int f = w % F, s = (w / F) & 3, tq = (w / (4 * F)) & 3, t = w / (16 * F);
        uint32_t b[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t word = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = FR::kidx(f, h, i);  // tile * 16 + code
                const int X = xs[(64 * (k >> 4) + 16 * tq + (k & 15)) * kPassRows + t];
                const uint32_t dig = (((uint32_t(X) + 0x80808080u) ^ 0x80808080u) >> (8 * s)) & 0xffu;
                word |= dig << (8 * i);
            }
            b[h] = word;
        }
        const int col = s * W + t, j = col >> 3, gq = col & 7;
        __stcg(reinterpret_cast<uint2*>(bstage + (size_t(f) * NT + j) * 256 + (4 * gq + tq) * 8),
               make_uint2(b[0], b[1]));
    }
}

// ---- consumers: mainloop + the item's epilogue for the warp's 16 channels -------------
struct EpiSmem {  // per epilogue buffer
    int xs[TILE_N * kPassRows];   // fc1: fixed-point mid of the item (the fc2 stage)
    unsigned long long zs[kPassRows];
};

template <int BITS, int NT>
__device__ void consume_item(const GemvArgs& g, const Plan& P, const GemvItem& it, const uint8_t* ring,
                             const uint8_t* bb, const BufMeta& meta, const long long* bzsum, uint64_t* full,
                             uint64_t* empty, int& stage, int& sphase, int* ws, EpiSmem& es, int s1, int s2,
                             unsigned* tn) {
    using FR = Frag<BITS>;
    constexpr int G = FR::G;
    constexpr int LOGD = FR::D == 64 ? 6 : FR::D == 16 ? 4 : 0;
    constexpr long long Z = 1ll << (BITS - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tq = lane & 3, gq = lane >> 2;
    const bool p1 = it.phase == 1;
    const int Kp = p1 ? g.Kp1 : g.Kp2;
    const int nst = min(kGemvKC, Kp - it.ks * kGemvKC) / kStageK;
    const int S = p1 ? s1 : s2;
    const int Np = p1 ? g.Np1 : g.Np2;
    const int nrows = it.nrows;
    // epilogue operands fetched early (latency overlaps the k-loop): lane -> channel r, all rows
    const int r = lane, ch = it.mt * TILE_N + 32 * warp + r;
    float sc, bias;
    scale_bias(g, p1, it.e, ch, sc, bias);
    const int ks2 = it.mt / kStagesPerChunk;
    const float smax = p1 ? __ldg(g.smax1 + it.e * s2 + ks2) : 0.f;
    const float bmax = p1 ? __ldg(g.bmax1 + it.e * s2 + ks2) : 0.f;
    float gate[kPassRows];
    int tok[kPassRows];
#pragma unroll
    for (int t = 0; t < kPassRows; ++t) {
        gate[t] = 0.f;
        tok[t] = 0;
        if (!p1 && S == 1 && t < nrows) { gate[t] = P.perm_gate[it.row0 + t]; tok[t] = P.perm_token[it.row0 + t]; }
    }
    int acc[kBlk][G][kMaxNT][4];
#pragma unroll
    for (int bk = 0; bk < kBlk; ++bk)
#pragma unroll
        for (int q = 0; q < G; ++q)
#pragma unroll
            for (int j = 0; j < kMaxNT; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[bk][q][j][i] = 0;
    long long cyc[2] = {0, 0};
    gemv_mainloop<BITS, NT>(ring, bb, full, empty, stage, sphase, nst, warp, lane, acc,
                            (g.trace && threadIdx.x == 0) ? cyc : nullptr);
    if (g.trace && threadIdx.x == 0) {  // mainloop end; mt/ks carry the wait / compute clock cycles (/16)
        GemvItem w = it;
        w.mt = int(min(cyc[0] >> 4, 0xffffll));
        w.ks = int(min(cyc[1] >> 4, 0xffffll));
        trace_ev(g, tn, 2, 1, w);
    }
    if (g.dbg & 1) {  // diagnostics: keep the accumulators alive, skip the epilogue
        int s = 0;
#pragma unroll
        for (int bk = 0; bk < kBlk; ++bk)
#pragma unroll
            for (int q = 0; q < G; ++q)
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) s += acc[bk][q][j][i];
        if (s == 0x7fffffff) ws[0] = s;
        return;
    }
    // groups -> D * Sum_k u * digit (exact in int32 for k-chunks <= 1024), per column (warp's own rows)
#pragma unroll
    for (int bk = 0; bk < kBlk; ++bk)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                int s = 0;
#pragma unroll
                for (int q = 0; q < G; ++q) s += FR::mult(q) * acc[bk][q][j][i];
                ws[(32 * warp + 16 * bk + gq + 8 * (i >> 1)) * kScrCols + 8 * j + 2 * tq + (i & 1)] = s;
            }
    __syncwarp();
    if (g.trace && threadIdx.x == 0) trace_ev(g, tn, 5, 1, it);
    // digits -> D * Sum_k q * X (int64) -> y = 2^-p * that / D (fp32, one rounding)
    const int PL = planes_of(it.phase), W = w_of(it.phase, NT);
    const int* wr = ws + (32 * warp + r) * kScrCols;
    float* part = g.partial + (p1 || s1 == 1 ? 0 : int64_t(s1) * g.part_rows * g.Np1);
    long long zsum_part[kPassRows];
#pragma unroll
    for (int t = 0; t < kPassRows; ++t) {
        zsum_part[t] = 0;
        if (t >= nrows) continue;
        const long long zs = p1 ? (long long)meta.zsum[t] : bzsum[t];
        long long V = -(long long)FR::D * Z * zs;
        for (int s = 0; s < PL; ++s) V += (long long)wr[s * W + t] << (8 * s);
        const int p = meta.p[t];
        const float y = p == kZeroRow ? 0.f : scale_pow2(V, p + LOGD);
        const int pos = it.row0 + t;
        if (S > 1) {
            __stcg(part + (int64_t(it.ks) * g.part_rows + pos) * Np + ch, y);
        } else if (p1) {
            const int X = encode_x2(fmaxf(fmaf(y, sc, bias), 0.0f), fc2_exp<BITS>(smax, bmax, meta.l1[t]));  // ReLU
            es.xs[(32 * warp + r) * kPassRows + t] = X;
            zsum_part[t] = X;
        } else {
            fc2_finish(g, ch, y, sc, bias, gate[t], tok[t]);
        }
    }
    if (g.trace && threadIdx.x == 0) trace_ev(g, tn, 5, 2, it);
    if (p1 && S > 1 && warp == 0 && lane < nrows)  // |x|_1 per row and k-split (the last CTA bounds the fc2 exponent)
        g.l1part[int64_t(it.row0 + lane) * s1 + it.ks] = meta.l1[lane];
    if (p1 && S == 1) {
        // Sum X2 per row over the 128 channels (the fc2 zero-point term of this stage)
#pragma unroll
        for (int t = 0; t < kPassRows; ++t) {
            long long z = zsum_part[t];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
            if (lane == 0 && t < nrows) atomicAdd(&es.zs[t], (unsigned long long)z);
        }
        named_bar_sync(1, kConsumers * 32);  // all 128 channels of X2 are in xs
        if (g.trace && threadIdx.x == 0) trace_ev(g, tn, 5, 3, it);
        const int slot = it.slot + ks2, st2 = it.mt % kStagesPerChunk;
        uint8_t* sl = g.xb + int64_t(slot) * g.xb_slot_bytes;
        encode_stage<BITS>(es.xs, nrows, sl + sizeof(BufMeta) + size_t(st2 * FR::F) * nt_of(2, nrows) * 256,
                           threadIdx.x, kConsumers * 32);
        if (g.trace && threadIdx.x == 0) trace_ev(g, tn, 5, 4, it);
        const int ctid = threadIdx.x;
        if (ctid < nrows) {
            long long* zpart = reinterpret_cast<long long*>(sl + sizeof(BufMeta) + GemvCfg<BITS>::BBUF);
            __stcg(zpart + st2 * 8 + ctid, (long long)es.zs[ctid]);
            es.zs[ctid] = 0;  // reused three items later (after two more barriers)
            reinterpret_cast<BufMeta*>(sl)->p[ctid] = fc2_exp<BITS>(smax, bmax, meta.l1[ctid]);
        }
    }
}

// ---- publisher: release the item's global results -------------------------------------
// fc1: fence + epoch flag of the fc2 stage; split-K items: fence + arrival
// count; the last arriving CTA reduces the partials in fixed k order.
template <int BITS>
__device__ void publish_item(const GemvArgs& g, const Plan& P, const GemvItem& it, int lane, int s1, int s2,
                             int nmt1, int nmt2, unsigned epoch, EpiSmem& es) {
    const bool p1 = it.phase == 1;
    const int S = p1 ? s1 : s2;
    const int ks2 = it.mt / kStagesPerChunk;
    if (S == 1) {
        if (p1 && lane == 0) {
            fence_proxy_async_global();  // the slot is read back by TMA bulk copies
            __threadfence();             // the consumers' fragment stores (acquired through the mbarrier)
            st_release_u32(g.xb_flag + (it.slot + ks2) * kStagesPerChunk + it.mt % kStagesPerChunk, epoch);
        }
        return;
    }
    const int maxmt = max(nmt1, nmt2);
    unsigned* cnt = g.split_cnt + (p1 ? 0 : g.E * maxmt) + it.e * maxmt + it.mt;
    int last = 0;
    if (lane == 0) {
        __threadfence();  // release the CTA's partials
        last = atomicAdd(cnt, 1u) == unsigned(S * it.npass - 1);
        if (last) {
            __threadfence();  // acquire the other CTAs' partials
            *cnt = 0;         // self-reset for the next forward
        }
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    const int Np = p1 ? g.Np1 : g.Np2;
    const float* part = g.partial + (p1 || s1 == 1 ? 0 : int64_t(s1) * g.part_rows * g.Np1);
    const int n = P.counts[it.e], off = P.offsets[it.e];
    const int slot0 = it.slot - (it.row0 - off) / kPassRows * s2;  // fc2 slot of the expert's first pass
    constexpr int NQ = TILE_N / 32;
    float sc[NQ], bias[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) scale_bias(g, p1, it.e, it.mt * TILE_N + lane + 32 * q, sc[q], bias[q]);
    const float smax = p1 ? __ldg(g.smax1 + it.e * s2 + ks2) : 0.f;
    const float bmax = p1 ? __ldg(g.bmax1 + it.e * s2 + ks2) : 0.f;
    for (int pass = 0; pass * kPassRows < n; ++pass) {
        const int row0 = off + pass * kPassRows, nr = min(kPassRows, n - pass * kPassRows);
        float y[NQ][kPassRows];
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int t = 0; t < kPassRows; ++t) y[q][t] = 0.f;
        for (int ks = 0; ks < S; ++ks)  // fixed k order; each step's loads are independent
#pragma unroll
            for (int q = 0; q < NQ; ++q)
#pragma unroll
                for (int t = 0; t < kPassRows; ++t)
                    if (t < nr) y[q][t] += __ldcg(part + (int64_t(ks) * g.part_rows + row0 + t) * Np + it.mt * TILE_N + lane + 32 * q);
        if (p1) {
            int p2[kPassRows];
#pragma unroll
            for (int t = 0; t < kPassRows; ++t) {
                float l = 0.f;
                if (t < nr)
                    for (int ks = 0; ks < S; ++ks) l += __ldcg(g.l1part + int64_t(row0 + t) * s1 + ks);
                p2[t] = t < nr ? fc2_exp<BITS>(smax, bmax, l * (1.0f + 0x1p-12f)) : kZeroRow;
            }
#pragma unroll
            for (int q = 0; q < NQ; ++q)
#pragma unroll
                for (int t = 0; t < kPassRows; ++t)
                    if (t < nr) es.xs[(lane + 32 * q) * kPassRows + t] = encode_x2(fmaxf(fmaf(y[q][t], sc[q], bias[q]), 0.f), p2[t]);
            __syncwarp();
            const int slot = slot0 + pass * s2 + ks2, st2 = it.mt % kStagesPerChunk;
            uint8_t* sl = g.xb + int64_t(slot) * g.xb_slot_bytes;
            encode_stage<BITS>(es.xs, nr, sl + sizeof(BufMeta) + size_t(st2 * Frag<BITS>::F) * nt_of(2, nr) * 256,
                               lane, 32);
            if (lane < nr) {
                long long z = 0;
                for (int c = 0; c < TILE_N; ++c) z += es.xs[c * kPassRows + lane];
                long long* zpart = reinterpret_cast<long long*>(sl + sizeof(BufMeta) + GemvCfg<BITS>::BBUF);
                __stcg(zpart + st2 * 8 + lane, z);
                reinterpret_cast<BufMeta*>(sl)->p[lane] = p2[lane];
            }
            __syncwarp();
            if (lane == 0) {
                fence_proxy_async_global();
                __threadfence();
                st_release_u32(g.xb_flag + slot * kStagesPerChunk + st2, epoch);
            }
            __syncwarp();
        } else {
#pragma unroll
            for (int t = 0; t < kPassRows; ++t) {
                if (t >= nr) break;
                const float gt = P.perm_gate[row0 + t];
                const int tk = P.perm_token[row0 + t];
#pragma unroll
                for (int q = 0; q < NQ; ++q) fc2_finish(g, it.mt * TILE_N + lane + 32 * q, y[q][t], sc[q], bias[q], gt, tk);
            }
        }
    }
}

template <int BITS>
__global__ void __launch_bounds__(kGemvThreads, 1) k_ffn_gemv(GemvArgs g, Plan P) {
    using Cfg = GemvCfg<BITS>;
    constexpr int SB = Cfg::SB, NST = Cfg::NST;
    constexpr int BSTRIDE = int(sizeof(BufMeta)) + Cfg::BBUF;
    constexpr int SCR = TILE_N * kScrCols;  // ints per scratch buffer
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* ring = smem;
    uint8_t* bbuf = ring + NST * SB;                                  // [kBBufs][meta | fragments]
    int* scr = reinterpret_cast<int*>(bbuf + kBBufs * BSTRIDE);        // [kScrBufs][128][16]
    EpiSmem* epi = reinterpret_cast<EpiSmem*>(scr + kScrBufs * SCR);   // [kScrBufs] (+1: the publisher's)
    long long* bzsum = reinterpret_cast<long long*>(epi + kScrBufs + 1);  // [kBBufs][kPassRows] fc2 Sum X
    GemvItem* pub = reinterpret_cast<GemvItem*>(bzsum + kBBufs * kPassRows);  // [kScrBufs]
    uint64_t* full = reinterpret_cast<uint64_t*>(pub + kScrBufs);
    uint64_t* empty = full + NST;
    uint64_t* ifull = empty + NST;
    uint64_t* iempty = ifull + kItemQ;
    uint64_t* bfull = iempty + kItemQ;
    uint64_t* bempty = bfull + kBBufs;
    uint64_t* pfull = bempty + kBBufs;
    uint64_t* pempty = pfull + kScrBufs;
    GemvItem* items = reinterpret_cast<GemvItem*>(pempty + kScrBufs);
    GemvTables& TBL = *reinterpret_cast<GemvTables*>(items + kItemQ);
    __shared__ unsigned s_tn;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned long long t_entry = gtime_ns();
    if (threadIdx.x == 0) {
        s_tn = 0;
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kConsumers); }
        for (int q = 0; q < kItemQ; ++q) { mbar_init(&ifull[q], 1); mbar_init(&iempty[q], kConsumers + kBuilders + 1); }
        for (int b = 0; b < kBBufs; ++b) { mbar_init(&bfull[b], 1); mbar_init(&bempty[b], kConsumers); }
        for (int b = 0; b < kScrBufs; ++b) { mbar_init(&pfull[b], kConsumers); mbar_init(&pempty[b], 1); }
    }
    for (int i = threadIdx.x; i < (kScrBufs + 1) * kPassRows; i += blockDim.x) epi[i / kPassRows].zs[i % kPassRows] = 0;
    if (threadIdx.x == 0) fence_barrier_init();
    __syncthreads();
    pdl_wait();  // routing plan of the preceding grid
    const int n_gemv = P.meta[0];
    if (n_gemv == 0) return;
    const unsigned epoch = unsigned(P.meta[5]);
    if (threadIdx.x == 0 && g.trace) {  // CTA entry (before the PDL wait) and after it
        const unsigned i = atomicAdd(&s_tn, 1u);
        g.trace[(size_t(blockIdx.x) * kTraceCap + i) * 2] = t_entry;
        g.trace[(size_t(blockIdx.x) * kTraceCap + i) * 2 + 1] = 3ull << 60 | 1ull << 56;
        trace_ev(g, &s_tn, 3, 0, GemvItem{});
    }
    const int nmt1 = g.Np1 / TILE_N, nmt2 = g.Np2 / TILE_N;
    const int s1 = gemv_ksplit_c(g.Kp1), s2 = gemv_ksplit_c(g.Kp2);

    if (warp == kProducer) {
        // ===== producer: item tables, tickets (one atomic in flight ahead), weight tiles
        unsigned ticket = 0;
        if (lane == 0) ticket = atomicAdd(&P.tickets[1], 1u);  // latency overlaps the table build
        for (int a = lane; a < n_gemv; a += 32) {
            const int e = P.gemv_list[a];
            TBL.list[a] = e;
            TBL.cnt[a] = P.counts[e];
            TBL.off[a] = P.offsets[e];
        }
        __syncwarp();
        if (lane != 0) return;
        {
            int t1 = 0, t2 = 0, tp = 0;
            for (int a = 0; a < n_gemv; ++a) {
                const int np = (TBL.cnt[a] + kPassRows - 1) / kPassRows;
                TBL.pst[a] = tp;
                TBL.start1[a] = t1;
                TBL.start2[a] = t2;
                tp += np;
                t1 += nmt1 * s1 * np;
                t2 += nmt2 * s2 * np;
            }
            TBL.pst[n_gemv] = tp;
            TBL.start1[n_gemv] = t1;
            TBL.start2[n_gemv] = t2;
        }
        const uint64_t pol = policy_evict_first();
        int stage = 0, sphase = 0, q = 0, qphase = 0;
        for (;;) {
            const GemvItem it = decode_item(ticket, TBL, n_gemv, nmt1, s1, nmt2, s2);
            trace_ev(g, &s_tn, 0, 0, it);
            mbar_wait(&iempty[q], qphase ^ 1);
            items[q] = it;
            mbar_arrive(&ifull[q]);
            if (++q == kItemQ) { q = 0; qphase ^= 1; }
            if (it.phase == 0) break;
            ticket = atomicAdd(&P.tickets[1], 1u);  // next ticket while this item's weights stream
            const bool p1 = it.phase == 1;
            const int Kp = p1 ? g.Kp1 : g.Kp2;
            const int k0 = it.ks * kGemvKC, klen = min(kGemvKC, Kp - k0);
            const int kbs = Kp / TILE_K;
            const uint8_t* base = (p1 ? g.w1 + int64_t(it.e) * g.w1_stride : g.w2 + int64_t(it.e) * g.w2_stride) +
                                  (int64_t(it.mt) * kbs + k0 / TILE_K) * Cfg::TB;
            for (int s = 0; s < klen / kStageK; ++s) {  // 2 consecutive tiles are contiguous
                mbar_wait(&empty[stage], sphase ^ 1);
                mbar_arrive_expect_tx(&full[stage], SB);
                bulk_g2s_hint(ring + stage * SB, base + int64_t(s) * SB, SB, &full[stage], pol);
                if (++stage == NST) { stage = 0; sphase ^= 1; }
            }
            trace_ev(g, &s_tn, 0, 1, it);
        }
        return;
    }

    if (warp == kPublisher) {
        // ===== publisher: fences, ready flags, split-K arrivals (in item order)
        int ps = 0, pph = 0;
        for (;;) {
            mbar_wait(&pfull[ps], pph);
            const GemvItem it = pub[ps];
            if (it.phase == 0) break;
            if (lane == 0) trace_ev(g, &s_tn, 4, 1, it);
            publish_item<BITS>(g, P, it, lane, s1, s2, nmt1, nmt2, epoch, epi[kScrBufs]);
            if (lane == 0) trace_ev(g, &s_tn, 4, 0, it);
            __syncwarp();
            if (lane == 0) mbar_arrive(&pempty[ps]);
            if (++ps == kScrBufs) { ps = 0; pph ^= 1; }
        }
        return;
    }

    if (warp == kLoader) {
        // ===== loader: fc2 items: fragment slot (all stages ready) -> smem buffer, in item order
        int q = 0, qphase = 0, bseq = 0;
        for (;;) {
            mbar_wait(&ifull[q], qphase);
            const GemvItem it = items[q];
            __syncwarp();
            if (lane == 0) mbar_arrive(&iempty[q]);
            if (++q == kItemQ) { q = 0; qphase ^= 1; }
            if (it.phase == 0) break;
            const int buf = bseq % kBBufs;
            if (it.phase == 2) {
                if (lane == 0) mbar_wait(&bempty[buf], ((bseq / kBBufs) & 1) ^ 1);
                __syncwarp();
                const int nst = min(kGemvKC, g.Kp2 - it.ks * kGemvKC) / kStageK;
                // lane (stage st, row t): acquire the stage flag, then its Sum X part
                const int st = lane >> 2, t = lane & 3;
                long long z = 0;
                if (st < nst) {
                    while (ld_acquire_u32(g.xb_flag + it.slot * kStagesPerChunk + st) != epoch) __nanosleep(32);
                    if (t < it.nrows)
                        z = __ldcg(reinterpret_cast<const long long*>(g.xb + int64_t(it.slot) * g.xb_slot_bytes +
                                                                      sizeof(BufMeta) + Cfg::BBUF) + st * 8 + t);
                }
#pragma unroll
                for (int off = 4; off < 32; off <<= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
                if (lane < kPassRows) bzsum[buf * kPassRows + lane] = z;
                __syncwarp();
                if (lane == 0) {
                    fence_proxy_async_global();
                    trace_ev(g, &s_tn, 1, 2, it);
                    const uint32_t bytes = uint32_t(sizeof(BufMeta) + nst * Cfg::F * nt_of(2, it.nrows) * 256);
                    mbar_arrive_expect_tx(&bfull[buf], bytes);
                    bulk_g2s(bbuf + buf * BSTRIDE, g.xb + int64_t(it.slot) * g.xb_slot_bytes, bytes, &bfull[buf]);
                }
            }
            __syncwarp();
            ++bseq;
        }
        return;
    }

    if (warp >= kConsumers) {
        // ===== builders (warps 8..10): builder b fills buffer b, i.e. every kBBufs-th weight item (fc1)
        const int bw = warp - kConsumers;
        const bool vec_h = g.h_f16 && (g.d % 8) == 0 && (reinterpret_cast<uintptr_t>(g.h) & 15) == 0;
        int q = 0, qphase = 0, bseq = 0;
        for (;;) {
            mbar_wait(&ifull[q], qphase);
            const GemvItem it = items[q];
            __syncwarp();
            if (lane == 0) mbar_arrive(&iempty[q]);
            if (++q == kItemQ) { q = 0; qphase ^= 1; }
            if (it.phase == 0) break;
            const int buf = bseq % kBBufs;
            if (it.phase == 1 && buf == bw) {
                if (lane == 0) mbar_wait(&bempty[buf], ((bseq / kBBufs) & 1) ^ 1);
                __syncwarp();
                BufMeta& bm = *reinterpret_cast<BufMeta*>(bbuf + buf * BSTRIDE);
                for (int t = 0; t < it.nrows; ++t)
                    build_row<BITS>(g, P, it, t, lane, vec_h, bbuf + buf * BSTRIDE + sizeof(BufMeta), bm);
                __syncwarp();
                if (lane == 0) {
                    trace_ev(g, &s_tn, 1, 1, it);
                    mbar_arrive(&bfull[buf]);
                }
            }
            ++bseq;
        }
        return;
    }

    // ===== consumers (warps 0..7): mainloop + epilogue -> publisher
    int stage = 0, sphase = 0, q = 0, qphase = 0, bseq = 0, ps = 0, pph = 0;
    for (;;) {
        mbar_wait(&ifull[q], qphase);
        const GemvItem it = items[q];
        __syncwarp();
        if (lane == 0) mbar_arrive(&iempty[q]);
        if (++q == kItemQ) { q = 0; qphase ^= 1; }
        if (lane == 0) mbar_wait(&pempty[ps], pph ^ 1);  // publisher slot ps is free
        __syncwarp();
        if (it.phase != 0) {
            const int buf = bseq % kBBufs;
            if (!(g.dbg & 2)) mbar_wait(&bfull[buf], (bseq / kBBufs) & 1);
            if (threadIdx.x == 0) trace_ev(g, &s_tn, 2, 0, it);
            const BufMeta& bm = *reinterpret_cast<const BufMeta*>(bbuf + buf * BSTRIDE);
            const uint8_t* bb = bbuf + buf * BSTRIDE + sizeof(BufMeta);
            const long long* bz = bzsum + buf * kPassRows;
            int* ws = scr + ps * SCR;
            if (nt_of(it.phase, it.nrows) == 1)
                consume_item<BITS, 1>(g, P, it, ring, bb, bm, bz, full, empty, stage, sphase, ws, epi[ps], s1, s2, &s_tn);
            else
                consume_item<BITS, 2>(g, P, it, ring, bb, bm, bz, full, empty, stage, sphase, ws, epi[ps], s1, s2, &s_tn);
            __syncwarp();
            if (lane == 0) mbar_arrive(&bempty[buf]);
            if (threadIdx.x == 0) trace_ev(g, &s_tn, 2, 2, it);
            ++bseq;
        } else if (threadIdx.x == 0) {
            trace_ev(g, &s_tn, 2, 3, it);
        }
        if (warp == 0 && lane == 0) pub[ps] = it;
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[ps]);  // release: this warp's global results of the item
        if (++ps == kScrBufs) { ps = 0; pph ^= 1; }
        if (it.phase == 0) break;
    }
}

namespace {
template <int BITS>
size_t gemv_smem() {
    using Cfg = GemvCfg<BITS>;
    return size_t(Cfg::NST) * Cfg::SB + kBBufs * (sizeof(BufMeta) + size_t(Cfg::BBUF)) +
           size_t(kScrBufs) * TILE_N * kScrCols * 4 + (kScrBufs + 1) * sizeof(EpiSmem) +
           kBBufs * kPassRows * 8 + kScrBufs * sizeof(GemvItem) +
           (2 * Cfg::NST + 2 * kItemQ + 2 * kBBufs + 2 * kScrBufs) * 8 + kItemQ * sizeof(GemvItem) +
           sizeof(GemvTables) + 64;
}

template <int BITS>
cudaError_t launch_gemv_t(const GemvArgs& g, const Plan& P, cudaStream_t st, int num_sms) {
    auto kern = k_ffn_gemv<BITS>;
    const size_t smem = gemv_smem<BITS>();
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    return launch_pdl(kern, dim3(num_sms), dim3(kGemvThreads), smem, st, g, P);
}
}  // namespace

int gemv_ksplit(int Kp) { return gemv_ksplit_c(Kp); }
// fc2 fragment slot: [meta | fragments (4 planes) | Sum X per (stage, row)]
int64_t gemv_xb_slot_bytes(int bits) {
    const int64_t tail = 8 * 8 * sizeof(long long);
    switch (bits) {
        case 2: return sizeof(BufMeta) + GemvCfg<2>::BBUF + tail;
        case 3: return sizeof(BufMeta) + GemvCfg<3>::BBUF + tail;
        case 4: return sizeof(BufMeta) + GemvCfg<4>::BBUF + tail;
    }
    return sizeof(BufMeta) + GemvCfg<8>::BBUF + tail;
}
// upper bound on row passes: every listed expert may end in a partial pass
int64_t gemv_xb_passes(int64_t rows, int E) { return (rows + kPassRows - 1) / kPassRows + E; }
int gemv_stages_per_chunk() { return kStagesPerChunk; }

// Partial-sum buffer size (floats) for `rows` GEMV rows.
int64_t gemv_partial_floats(int64_t rows, int Kp1, int Np1, int Kp2, int Np2) {
    const int s1 = gemv_ksplit_c(Kp1), s2 = gemv_ksplit_c(Kp2);
    return (s1 > 1 ? int64_t(s1) * rows * Np1 : 0) + int64_t(s2) * rows * Np2;
}

cudaError_t launch_gemv(int bits, bool, const GemvArgs& g, const Plan& P, cudaStream_t st, int num_sms) {
    switch (bits) {
        case 2: return launch_gemv_t<2>(g, P, st, num_sms);
        case 3: return launch_gemv_t<3>(g, P, st, num_sms);
        case 4: return launch_gemv_t<4>(g, P, st, num_sms);
        case 8: return launch_gemv_t<8>(g, P, st, num_sms);
    }
    return cudaErrorInvalidValue;
}

// Per (expert, fc2 k-chunk): max fc1 scale and max |fc1 bias| over the chunk's
// channels — the constants of the fc2 fixed-point bound (bank creation).
__global__ void k_chunk_max(const float* __restrict__ s1, const float* __restrict__ b1, int Np1, float* smax,
                            float* bmax) {
    const int e = blockIdx.x, ks = blockIdx.y, n0 = ks * kGemvKC;
    float ms = 0.f, mb = 0.f;
    for (int n = n0 + threadIdx.x; n < min(n0 + kGemvKC, Np1); n += blockDim.x) {
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
        smax[e * gridDim.y + ks] = ms;
        bmax[e * gridDim.y + ks] = mb;
    }
}

cudaError_t launch_chunk_max(const float* s1, const float* b1, int E, int Np1, int Kp2, float* smax, float* bmax,
                             cudaStream_t st) {
    k_chunk_max<<<dim3(E, gemv_ksplit_c(Kp2)), 256, 0, st>>>(s1, b1, Np1, smax, bmax);
    return cudaGetLastError();
}

}  // namespace moqe_gpu
