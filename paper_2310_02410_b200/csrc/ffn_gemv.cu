// ffn_gemv.cu — decode path: fused expert FFN (fc1 -> ReLU -> fc2 -> gate
// combine) as ONE persistent, warp-specialised weight-streaming kernel.
//
// Reference: the per-expert loop of moe_ffn_forward proj/src/model.cpp:360-391
// (dequantize :370-375, matmul :381/:384, add_bias/relu :382-385, scatter
// :387-390). The reference re-dequantizes whole experts to f32 (27 ms per
// 4M-element matrix); here packed codes stream from HBM exactly once.
//
// Work items (device-side, no host sync): fc1 (expert, 128-channel m-tile,
// k-chunk) for every expert in the GEMV list, then fc2 items likewise. A
// producer warp grabs items from a global ticket and streams each item's
// packed weight tiles (TILE_N x 64 codes, 1024*bits bytes) with TMA bulk
// copies (cp.async.bulk, evict-first) into an NSTAGE smem ring. Eight
// consumer warps each own 16 output channels: they unpack codes straight
// into m16n8k16 A-fragments (codec.cuh: one LOP3 + one HFMA2 per code pair,
// no smem round trip) and multiply by the routed tokens' activations
// (B-fragments, n8 = 8 tokens per tile, fp32 accumulation). Per-output-channel
// scales factor out of the k-sum and are applied once in the epilogue (codes
// x fp16 activations are exact products). fc2 items wait on a per-expert fc1
// completion counter while their weights are already in flight. Split-K
// partials are reduced in fixed k order by the last arriving CTA, so results
// are deterministic.
#include <cuda_fp16.h>

#include "codec.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace moqe_gpu {

constexpr int kGemvKC = 1024;       // k-chunk (codes) per item
constexpr int kGemvConsumers = 8;   // consumer warps (16 channels each)
constexpr int kGemvThreads = (kGemvConsumers + 1) * 32;
constexpr int kItemQ = 4;           // item queue depth
constexpr int kGemvRows = kGemvMaxRows;  // token rows per pass (2 n8 tiles)
constexpr int kActStride = kGemvKC * 2 + 16;  // bytes: 16B-aligned rows for bulk copies
constexpr int kMaxListed = 256;

struct GemvItem {
    int phase;  // 1, 2, or 0 = end
    int e, mt, ks, row0, nrows, npass;
};

template <int BITS>
struct GemvCfg {
    static constexpr int TB = tile_bytes(BITS);
    static constexpr int KPS = 2;  // k-blocks (tiles) per ring stage
    static constexpr int SB = KPS * TB;
    static constexpr int NST = BITS == 2 ? 8 : BITS == 3 ? 6 : BITS == 4 ? 4 : 3;
};

struct GemvTables {
    int list[kMaxListed], cnt[kMaxListed], off[kMaxListed];
    int start1[kMaxListed + 1], start2[kMaxListed + 1];  // item prefix per listed expert
};

// Decode ticket -> item from the smem tables (binary search over experts).
__device__ GemvItem decode_item(unsigned ticket, const GemvTables& T, int n_gemv, int nmt1, int s1, int nmt2,
                                int s2) {
    GemvItem it{};
    const unsigned tot1 = unsigned(T.start1[n_gemv]), tot2 = unsigned(T.start2[n_gemv]);
    int phase;
    unsigned rem;
    const int* st;
    if (ticket < tot1) { phase = 1; rem = ticket; st = T.start1; }
    else if (ticket < tot1 + tot2) { phase = 2; rem = ticket - tot1; st = T.start2; }
    else { it.phase = 0; return it; }
    int lo = 0, hi = n_gemv - 1;  // largest a with st[a] <= rem
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (unsigned(st[mid]) <= rem) lo = mid; else hi = mid - 1;
    }
    const int a = lo;
    const int nmt = phase == 1 ? nmt1 : nmt2, S = phase == 1 ? s1 : s2;
    const int r = int(rem - unsigned(st[a]));
    const int pass = r / (nmt * S), r2 = r % (nmt * S);
    const int n = T.cnt[a];
    it.phase = phase;
    it.e = T.list[a];
    it.mt = r2 / S;
    it.ks = r2 % S;
    it.row0 = T.off[a] + pass * kGemvRows;
    it.nrows = min(kGemvRows, n - pass * kGemvRows);
    it.npass = (n + kGemvRows - 1) / kGemvRows;
    return it;
}

// One k-block (64 codes) of the warp's 16 channels against NT token tiles.
template <int BITS, int NT>
__device__ __forceinline__ void gemv_kblock(const uint8_t* tile, const uint8_t* act, int kb, int warp, int gq,
                                            int tq, float (&acc)[2][4]) {
    uint32_t lo[8], hi[8];  // rows g and g+8 of the warp's m16 tile
    unpack_chunk<BITS>(tile + (16 * warp + gq) * row_bytes(BITS), tq, lo);
    unpack_chunk<BITS>(tile + (16 * warp + gq + 8) * row_bytes(BITS), tq, hi);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int off = (kb * 64 + tq * 16 + 4 * j) * 2;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            const uint2 b = *reinterpret_cast<const uint2*>(act + (8 * n + gq) * kActStride + off);
            mma_16816(acc[n], lo[2 * j], hi[2 * j], lo[2 * j + 1], hi[2 * j + 1], b.x, b.y);
        }
    }
}

template <int BITS, int NT>
__device__ __forceinline__ void gemv_mainloop(const uint8_t* ring, const uint8_t* act, uint64_t* full,
                                              uint64_t* empty, int& stage, int& sphase, int nblk, int warp,
                                              int lane, float (&acc)[2][4]) {
    constexpr int TB = GemvCfg<BITS>::TB, SB = GemvCfg<BITS>::SB, NST = GemvCfg<BITS>::NST;
    const int gq = lane >> 2, tq = lane & 3;
    for (int kb = 0; kb < nblk; kb += 2) {  // nblk is even (k-chunks are multiples of 128)
        mbar_wait(&full[stage], sphase);
        const uint8_t* st = ring + stage * SB;
        gemv_kblock<BITS, NT>(st, act, kb, warp, gq, tq, acc);
        gemv_kblock<BITS, NT>(st + TB, act, kb + 1, warp, gq, tq, acc);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == NST) { stage = 0; sphase ^= 1; }
    }
}

template <int BITS>
__global__ void __launch_bounds__(kGemvThreads, 2) k_ffn_gemv(GemvArgs g, Plan P) {
    using Cfg = GemvCfg<BITS>;
    constexpr int TB = Cfg::TB, SB = Cfg::SB, NST = Cfg::NST;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* ring = smem;
    uint8_t* actbuf = smem + NST * SB;  // [2][kGemvRows][kActStride]
    uint64_t* full = reinterpret_cast<uint64_t*>(actbuf + 2 * kGemvRows * kActStride);
    uint64_t* empty = full + NST;
    uint64_t* ifull = empty + NST;
    uint64_t* iempty = ifull + kItemQ;
    uint64_t* afull = iempty + kItemQ;
    uint64_t* aempty = afull + 2;
    GemvItem* items = reinterpret_cast<GemvItem*>(aempty + 2);
    GemvTables& TBL = *reinterpret_cast<GemvTables*>(items + kItemQ);
    __shared__ int s_flag;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_gemv = P.meta[0];
    const int nmt1 = g.Np1 / TILE_N, nmt2 = g.Np2 / TILE_N;
    const int s1 = (g.Kp1 + kGemvKC - 1) / kGemvKC, s2 = (g.Kp2 + kGemvKC - 1) / kGemvKC;
    if (n_gemv == 0) return;
    // bulk activation copies need 16-byte rows of fp16 input
    const bool bulk_h = g.h_f16 && (g.d % 8) == 0 && (reinterpret_cast<uintptr_t>(g.h) & 15) == 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kGemvConsumers); }
        for (int q = 0; q < kItemQ; ++q) { mbar_init(&ifull[q], 1); mbar_init(&iempty[q], kGemvConsumers); }
        for (int b = 0; b < 2; ++b) { mbar_init(&afull[b], 1); mbar_init(&aempty[b], kGemvConsumers); }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kGemvConsumers) {
        // ===== producer warp: item decode (lane 0), activation rows (all lanes), weight tiles (lane 0)
        for (int a = lane; a < n_gemv; a += 32) {
            const int e = P.gemv_list[a];
            TBL.list[a] = e;
            TBL.cnt[a] = P.counts[e];
            TBL.off[a] = P.offsets[e];
        }
        __syncwarp();
        if (lane == 0) {
            int t1 = 0, t2 = 0;
            for (int a = 0; a < n_gemv; ++a) {
                const int np = (TBL.cnt[a] + kGemvRows - 1) / kGemvRows;
                TBL.start1[a] = t1;
                TBL.start2[a] = t2;
                t1 += nmt1 * s1 * np;
                t2 += nmt2 * s2 * np;
            }
            TBL.start1[n_gemv] = t1;
            TBL.start2[n_gemv] = t2;
        }
        __syncwarp();
        const uint64_t pol = policy_evict_first();
        int stage = 0, sphase = 0, q = 0, qphase = 0;
        for (int seq = 0;; ++seq) {
            GemvItem it;
            if (lane == 0) it = decode_item(atomicAdd(&P.tickets[1], 1u), TBL, n_gemv, nmt1, s1, nmt2, s2);
            it.phase = __shfl_sync(0xffffffffu, it.phase, 0);
            it.e = __shfl_sync(0xffffffffu, it.e, 0);
            it.mt = __shfl_sync(0xffffffffu, it.mt, 0);
            it.ks = __shfl_sync(0xffffffffu, it.ks, 0);
            it.row0 = __shfl_sync(0xffffffffu, it.row0, 0);
            it.nrows = __shfl_sync(0xffffffffu, it.nrows, 0);
            it.npass = __shfl_sync(0xffffffffu, it.npass, 0);
            const bool p1 = it.phase == 1;
            const int Kp = p1 ? g.Kp1 : g.Kp2;
            const int k0 = it.ks * kGemvKC;
            const int klen = it.phase ? min(kGemvKC, Kp - k0) : 0;
            if (it.phase != 0) {
                // activation rows -> act buffer (seq & 1)
                const int ab = seq & 1;
                uint8_t* act = actbuf + ab * kGemvRows * kActStride;
                if (lane == 0) {
                    mbar_wait(&aempty[ab], ((seq >> 1) & 1) ^ 1);
                    if (!p1) {  // fc2 needs every fc1 m-tile of this expert (all passes)
                        const unsigned need = unsigned(nmt1 * it.npass);
                        while (ld_acquire_u32(&P.done[it.e]) < need) __nanosleep(32);
                    }
                }
                __syncwarp();
                if (!p1 || bulk_h) {
                    if (lane == 0) mbar_arrive_expect_tx(&afull[ab], uint32_t(it.nrows * klen * 2));
                    __syncwarp();
                    if (lane < it.nrows) {
                        const __half* src = p1 ? static_cast<const __half*>(g.h) + int64_t(P.perm_token[it.row0 + lane]) * g.d + k0
                                               : g.mid + int64_t(it.row0 + lane) * g.Np1 + k0;
                        bulk_g2s(act + lane * kActStride, src, uint32_t(klen * 2), &afull[ab]);
                    }
                } else {
                    // f32 or unaligned input: convert through registers
                    for (int r = 0; r < it.nrows; ++r) {
                        const int64_t tok = P.perm_token[it.row0 + r];
                        __half* dst = reinterpret_cast<__half*>(act + r * kActStride);
                        for (int kk = lane; kk < klen; kk += 32) {
                            const int64_t kx = k0 + kk;
                            float x = 0.f;
                            if (kx < g.d)
                                x = g.h_f16 ? __half2float(static_cast<const __half*>(g.h)[tok * g.d + kx])
                                            : static_cast<const float*>(g.h)[tok * g.d + kx];
                            dst[kk] = __float2half_rn(x);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&afull[ab]);
                }
            }
            if (lane == 0) {
                mbar_wait(&iempty[q], qphase ^ 1);
                items[q] = it;
                mbar_arrive(&ifull[q]);
            }
            if (++q == kItemQ) { q = 0; qphase ^= 1; }
            if (it.phase == 0) break;
            if (lane == 0) {
                const int kbs = Kp / TILE_K;
                const int kb0 = k0 / TILE_K, kb1 = kb0 + klen / TILE_K;
                const uint8_t* base = (p1 ? g.w1 + int64_t(it.e) * g.w1_stride : g.w2 + int64_t(it.e) * g.w2_stride) +
                                      (int64_t(it.mt) * kbs) * TB;
                for (int kb = kb0; kb < kb1; kb += Cfg::KPS) {  // KPS consecutive tiles are contiguous
                    mbar_wait(&empty[stage], sphase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], SB);
                    bulk_g2s_hint(ring + stage * SB, base + int64_t(kb) * TB, SB, &full[stage], pol);
                    if (++stage == NST) { stage = 0; sphase ^= 1; }
                }
            }
            __syncwarp();
        }
        return;
    }

    // ===== consumers (warps 0..7, 256 threads) =====
    const int gq = lane >> 2, tq = lane & 3;
    const int ctid = threadIdx.x;
    constexpr int NCT = kGemvConsumers * 32;
    int stage = 0, sphase = 0, q = 0, qphase = 0;
    for (int seq = 0;; ++seq) {
        mbar_wait(&ifull[q], qphase);
        const GemvItem it = items[q];
        if (it.phase == 0) break;
        const bool p1 = it.phase == 1;
        const int Kp = p1 ? g.Kp1 : g.Kp2;
        const int klen = min(kGemvKC, Kp - it.ks * kGemvKC);
        const int nblk = klen / TILE_K;
        const int ab = seq & 1;
        const uint8_t* act = actbuf + ab * kGemvRows * kActStride;
        const int chb = it.mt * TILE_N + 16 * warp + gq;
        // epilogue operands fetched early (latency overlaps the k-loop)
        const float* sc = p1 ? g.s1 + int64_t(it.e) * g.Np1 : g.s2 + int64_t(it.e) * g.Np2;
        const float* bi = p1 ? g.b1 : g.b2;
        const int Np = p1 ? g.Np1 : g.Np2;
        const float sc0 = __ldg(sc + chb), sc1 = __ldg(sc + chb + 8);
        const float bi0 = bi ? __ldg(bi + int64_t(it.e) * Np + chb) : 0.f;
        const float bi1 = bi ? __ldg(bi + int64_t(it.e) * Np + chb + 8) : 0.f;

        mbar_wait(&afull[ab], (seq >> 1) & 1);
        float acc[2][4];
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[n][i] = 0.f;
        const int ntl = (it.nrows + 7) / 8;
        if (ntl <= 1) gemv_mainloop<BITS, 1>(ring, act, full, empty, stage, sphase, nblk, warp, lane, acc);
        else gemv_mainloop<BITS, 2>(ring, act, full, empty, stage, sphase, nblk, warp, lane, acc);
        __syncwarp();
        if (lane == 0) mbar_arrive(&aempty[ab]);

        // ---- split-K reduction (fixed order) + epilogue ----
        // fragment (n, i): channel ch = chb + 8*(i>>1), row r = 8n + 2tq + (i&1)
        const int S = p1 ? s1 : s2;
        float* part = g.partial + (p1 || s1 == 1 ? 0 : int64_t(s1) * g.part_rows * g.Np1);
        bool do_epi = true;
        if (S > 1) {
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int r = 8 * n + 2 * tq + (i & 1);
                    if (n < ntl && r < it.nrows)
                        __stcg(part + (int64_t(it.ks) * g.part_rows + it.row0 + r) * Np + chb + 8 * (i >> 1), acc[n][i]);
                }
            named_bar_sync(1, NCT);
            const int maxmt = max(nmt1, nmt2);
            unsigned* cnt = g.split_cnt + (p1 ? 0 : g.E * maxmt) + it.e * maxmt + it.mt;
            if (ctid == 0) {
                __threadfence();  // release the CTA's partials (ordered by the barrier above)
                const bool last = atomicAdd(cnt, 1u) == unsigned(S * it.npass - 1);
                if (last) {
                    __threadfence();  // acquire the other CTAs' partials
                    *cnt = 0;         // self-reset for the next forward
                }
                s_flag = last;
            }
            named_bar_sync(1, NCT);
            do_epi = s_flag;
        }
        if (do_epi) {
            const int npass_here = S > 1 ? it.npass : 1;
            for (int ps = 0; ps < npass_here; ++ps) {
                const int row0 = S > 1 ? P.offsets[it.e] + ps * kGemvRows : it.row0;
                const int nrows = S > 1 ? min(kGemvRows, P.counts[it.e] - ps * kGemvRows) : it.nrows;
#pragma unroll
                for (int n = 0; n < 2; ++n)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int r = 8 * n + 2 * tq + (i & 1);
                        if (r >= nrows) continue;
                        const int ch = chb + 8 * (i >> 1);
                        const int pos = row0 + r;
                        float v;
                        if (S > 1) {
                            v = 0.f;
                            for (int ks = 0; ks < S; ++ks) v += __ldcg(part + (int64_t(ks) * g.part_rows + pos) * Np + ch);
                        } else {
                            v = acc[n][i];
                        }
                        const float y = v * ((i >> 1) ? sc1 : sc0) + ((i >> 1) ? bi1 : bi0);
                        if (p1) {
                            g.mid[int64_t(pos) * g.Np1 + ch] = __float2half_rn(y > 0.f ? y : 0.f);
                        } else if (ch < g.d) {
                            const float yg = y * P.perm_gate[pos];
                            const int64_t o = int64_t(P.perm_token[pos]) * g.d + ch;
                            if (g.out_acc) atomicAdd(g.out_acc + o, yg);
                            else if (g.out_f16) static_cast<__half*>(g.out)[o] = __float2half_rn(yg);
                            else static_cast<float*>(g.out)[o] = yg;
                        }
                    }
            }
            if (p1) {
                named_bar_sync(1, NCT);
                if (ctid == 0) {
                    __threadfence();  // publish mid rows before counting the m-tile done
                    atomicAdd(&P.done[it.e], unsigned(S > 1 ? it.npass : 1));
                }
            }
        }
        named_bar_sync(1, NCT);
        if (lane == 0) mbar_arrive(&iempty[q]);
        if (++q == kItemQ) { q = 0; qphase ^= 1; }
    }
}

namespace {
template <int BITS>
size_t gemv_smem() {
    return size_t(GemvCfg<BITS>::NST) * GemvCfg<BITS>::SB + size_t(2 * kGemvRows) * kActStride +
           (2 * GemvCfg<BITS>::NST + 2 * kItemQ + 4) * 8 + kItemQ * sizeof(GemvItem) + sizeof(GemvTables) + 64;
}

template <int BITS>
cudaError_t launch_gemv_t(const GemvArgs& g, const Plan& P, cudaStream_t st, int num_sms) {
    auto kern = k_ffn_gemv<BITS>;
    const size_t smem = gemv_smem<BITS>();
    static bool configured = false;
    static int occ = 1;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGemvThreads, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
        configured = true;
    }
    kern<<<num_sms * occ, kGemvThreads, smem, st>>>(g, P);
    return cudaGetLastError();
}
}  // namespace

// Partial-sum buffer size (floats) for `rows` GEMV rows.
int64_t gemv_partial_floats(int64_t rows, int Kp1, int Np1, int Kp2, int Np2) {
    const int s1 = (Kp1 + kGemvKC - 1) / kGemvKC, s2 = (Kp2 + kGemvKC - 1) / kGemvKC;
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

}  // namespace moqe_gpu
