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
// producer warp grabs items from a global ticket and streams the item's
// packed weight tiles (TILE_N x 64 codes, 1024*bits bytes) with TMA bulk
// copies into an NSTAGE smem ring; 8 consumer warps unpack codes to fp16 in
// registers (magic-number / PRMT tricks, no smem round trip) and accumulate
// in fp32 with m16n8k16 register MMAs (tokens = M, channels = N). Scales are
// per output channel, so they are applied once in the epilogue (codes and
// fp16 activations multiply exactly). fc2 items wait on a per-expert fc1
// completion counter while their weights are already in flight. Split-K
// partials are reduced in fixed k order by the last arriving CTA
// (deterministic).
#include <cuda_fp16.h>

#include "kernels.cuh"
#include "ptx.cuh"

namespace moqe_gpu {

constexpr int kGemvKC = 1024;       // k-chunk (codes) per item
constexpr int kGemvConsumers = 8;   // consumer warps (16 channels each)
constexpr int kGemvThreads = (kGemvConsumers + 1) * 32;
constexpr int kItemQ = 4;           // item queue depth

struct GemvItem {
    int phase;  // 1, 2, or 0 = end
    int e, a, mt, ks, row0, nrows, npass;
};

template <int BITS>
struct GemvCfg {
    static constexpr int TB = tile_bytes(BITS);
    static constexpr int NST = BITS == 2 ? 16 : BITS == 3 ? 12 : BITS == 4 ? 8 : 4;
};

// Fragment order of the 16 codes a thread unpacks per 64-code row: position p
// of the staged activation group holds actual k offset perm(p).
template <int BITS>
__device__ __forceinline__ int frag_pos_of(int off) {
    if (BITS == 8) return off;
    if (BITS == 4) {  // perm = [0,4,1,5, 2,6,3,7, 8,12,9,13, 10,14,11,15]
        const int hi = off & 8, r = off & 7;
        return hi + ((r & 3) << 1) + (r >> 2);
    }
    // BITS 2/3: perm = [0,8,1,9, 2,10,3,11, 4,12,5,13, 6,14,7,15]
    return ((off & 7) << 1) + (off >> 3);
}

// Unpack the thread's 16 codes (row bytes [2*BITS*t, 2*BITS*(t+1))) into
// b[j][0..1] = half2 pairs for mma k-steps j = 0..3.
template <int BITS>
__device__ __forceinline__ void unpack16(const uint8_t* p, uint32_t (&b)[4][2]) {
    if constexpr (BITS == 4) {
        const uint2 w = *reinterpret_cast<const uint2*>(p);
        const __half2 bias = __float2half2_rn(1032.0f);
        const uint32_t ws[2] = {w.x, w.y};
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                uint32_t v = ((ws[q] >> (4 * s)) & 0x000F000Fu) | 0x64006400u;
                __half2 hv = __hsub2(*reinterpret_cast<__half2*>(&v), bias);
                b[q * 2 + (s >> 1)][s & 1] = *reinterpret_cast<uint32_t*>(&hv);
            }
    } else if constexpr (BITS == 2) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
        const __half2 bias = __float2half2_rn(1026.0f);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            uint32_t v = ((w >> (2 * s)) & 0x00030003u) | 0x64006400u;
            __half2 hv = __hsub2(*reinterpret_cast<__half2*>(&v), bias);
            b[s >> 1][s & 1] = *reinterpret_cast<uint32_t*>(&hv);
        }
    } else if constexpr (BITS == 3) {
        const uint16_t* q = reinterpret_cast<const uint16_t*>(p);
        const uint32_t g0 = uint32_t(q[0]) | (uint32_t(q[1] & 0xFFu) << 16);
        const uint32_t g1 = uint32_t(q[1] >> 8) | (uint32_t(q[2]) << 8);
        const uint32_t w = (g0 & 0xFFFFu) | (g1 << 16);
        const uint32_t w2 = ((g0 >> 15) & 0xFFFFu) | ((g1 >> 15) << 16);
        const __half2 bias = __float2half2_rn(1028.0f);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const uint32_t src = s < 5 ? (w >> (3 * s)) : (w2 >> (3 * (s - 5)));
            uint32_t v = (src & 0x00070007u) | 0x64006400u;
            __half2 hv = __hsub2(*reinterpret_cast<__half2*>(&v), bias);
            b[s >> 1][s & 1] = *reinterpret_cast<uint32_t*>(&hv);
        }
    } else {  // 8
        const uint4 w = *reinterpret_cast<const uint4*>(p);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        const __half2 bias = __float2half2_rn(1152.0f);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t lo = prmt(ws[q], 0x64646464u, 0x4140u);
            uint32_t hi = prmt(ws[q], 0x64646464u, 0x4342u);
            __half2 hl = __hsub2(*reinterpret_cast<__half2*>(&lo), bias);
            __half2 hh = __hsub2(*reinterpret_cast<__half2*>(&hi), bias);
            b[q][0] = *reinterpret_cast<uint32_t*>(&hl);
            b[q][1] = *reinterpret_cast<uint32_t*>(&hh);
        }
    }
}

// Decode ticket -> item. Items: phase 1 = sum_a Nmt1*S1*P_a, then phase 2.
__device__ GemvItem decode_item(unsigned ticket, const Plan& P, int n_gemv, int rows_per_pass,
                                int nmt1, int s1, int nmt2, int s2) {
    GemvItem it{};
    unsigned rem = ticket;
    for (int phase = 1; phase <= 2; ++phase) {
        const int nmt = phase == 1 ? nmt1 : nmt2, S = phase == 1 ? s1 : s2;
        for (int a = 0; a < n_gemv; ++a) {
            const int e = P.gemv_list[a];
            const int n = P.counts[e];
            const int npass = (n + rows_per_pass - 1) / rows_per_pass;
            const unsigned cnt = unsigned(nmt * S * npass);
            if (rem < cnt) {
                const int pass = int(rem) / (nmt * S);
                const int r2 = int(rem) % (nmt * S);
                it.phase = phase;
                it.e = e;
                it.a = a;
                it.mt = r2 / S;
                it.ks = r2 % S;
                it.row0 = P.offsets[e] + pass * rows_per_pass;
                it.nrows = min(rows_per_pass, n - pass * rows_per_pass);
                it.npass = npass;
                return it;
            }
            rem -= cnt;
        }
    }
    it.phase = 0;
    return it;
}

template <int BITS, int MT>
__global__ void __launch_bounds__(kGemvThreads, 1) k_ffn_gemv(GemvArgs g, Plan P) {
    using Cfg = GemvCfg<BITS>;
    constexpr int TB = Cfg::TB, NST = Cfg::NST, ROWS = 16 * MT;
    constexpr int ASTR = kGemvKC * 2 + 8;  // bytes; == 8 mod 128 -> conflict-free A loads
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* ring = smem;
    uint8_t* act = smem + NST * TB;
    uint64_t* full = reinterpret_cast<uint64_t*>(act + ROWS * ASTR);
    uint64_t* empty = full + NST;
    uint64_t* ifull = empty + NST;
    uint64_t* iempty = ifull + kItemQ;
    GemvItem* items = reinterpret_cast<GemvItem*>(iempty + kItemQ);
    __shared__ int s_flag;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_gemv = P.meta[0];
    const int nmt1 = g.Np1 / TILE_N, nmt2 = g.Np2 / TILE_N;
    const int s1 = (g.Kp1 + kGemvKC - 1) / kGemvKC, s2 = (g.Kp2 + kGemvKC - 1) / kGemvKC;
    if (n_gemv == 0) return;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], kGemvConsumers); }
        for (int q = 0; q < kItemQ; ++q) { mbar_init(&ifull[q], 1); mbar_init(&iempty[q], kGemvConsumers); }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == kGemvConsumers) {
        // ===== producer =====
        if (lane != 0) return;
        const uint64_t pol = policy_evict_first();
        int stage = 0, sphase = 0, q = 0, qphase = 0;
        for (;;) {
            const unsigned ticket = atomicAdd(&P.tickets[1], 1u);
            GemvItem it = decode_item(ticket, P, n_gemv, ROWS, nmt1, s1, nmt2, s2);
            mbar_wait(&iempty[q], qphase ^ 1);
            items[q] = it;
            mbar_arrive(&ifull[q]);
            if (++q == kItemQ) { q = 0; qphase ^= 1; }
            if (it.phase == 0) break;
            const bool p1 = it.phase == 1;
            const int Kp = p1 ? g.Kp1 : g.Kp2;
            const int kbs = Kp / TILE_K;
            const int kb0 = it.ks * (kGemvKC / TILE_K);
            const int kb1 = min(kbs, kb0 + kGemvKC / TILE_K);
            const uint8_t* base = (p1 ? g.w1 + int64_t(it.e) * g.w1_stride : g.w2 + int64_t(it.e) * g.w2_stride) +
                                  (int64_t(it.mt) * kbs) * TB;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&empty[stage], sphase ^ 1);
                mbar_arrive_expect_tx(&full[stage], TB);
                bulk_g2s_hint(ring + stage * TB, base + int64_t(kb) * TB, TB, &full[stage], pol);
                if (++stage == NST) { stage = 0; sphase ^= 1; }
            }
        }
        return;
    }

    // ===== consumers (warps 0..7, 256 threads) =====
    const int gq = lane >> 2, tq = lane & 3;
    const int ctid = threadIdx.x;  // 0..255
    int stage = 0, sphase = 0, q = 0, qphase = 0;
    for (;;) {
        mbar_wait(&ifull[q], qphase);
        const GemvItem it = items[q];
        if (it.phase == 0) break;
        const bool p1 = it.phase == 1;
        const int Kp = p1 ? g.Kp1 : g.Kp2;
        const int k0 = it.ks * kGemvKC;
        const int klen = min(kGemvKC, Kp - k0);
        const int nblk = klen / TILE_K;

        if (!p1) {
            // fc2 needs every fc1 m-tile of this expert (all passes)
            if (ctid == 0) {
                const unsigned need = unsigned(nmt1 * it.npass);
                while (ld_acquire_u32(&P.done[it.e]) < need) __nanosleep(100);
            }
            named_bar_sync(1, kGemvConsumers * 32);
        }
        // ---- stage activations (fp16, fragment-permuted) ----
        {
            const int chunks = klen / 8;
            for (int idx = ctid; idx < it.nrows * chunks; idx += kGemvConsumers * 32) {
                const int r = idx / chunks, c = idx % chunks;
                const int kk = c * 8;  // local k
                __half v[8];
                if (p1) {
                    const int64_t tok = P.perm_token[it.row0 + r];
                    const int64_t kg = k0 + kk;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int64_t kx = kg + u;
                        float x = 0.f;
                        if (kx < g.d)
                            x = g.h_f16 ? __half2float(static_cast<const __half*>(g.h)[tok * g.d + kx])
                                        : static_cast<const float*>(g.h)[tok * g.d + kx];
                        v[u] = __float2half_rn(x);
                    }
                } else {
                    const uint4 raw = __ldcg(reinterpret_cast<const uint4*>(g.mid + int64_t(it.row0 + r) * g.Np1 + k0 + kk));
                    *reinterpret_cast<uint4*>(v) = raw;
                }
                __half* dst = reinterpret_cast<__half*>(act + r * ASTR);
                const int gbase = kk & ~15;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int off = (kk & 15) + u;
                    dst[gbase + frag_pos_of<BITS>(off)] = v[u];
                }
            }
        }
        named_bar_sync(1, kGemvConsumers * 32);

        float acc[MT][2][4];
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[m][n][i] = 0.f;
        const bool two = MT == 2 && it.nrows > 16;

        for (int kb = 0; kb < nblk; ++kb) {
            mbar_wait(&full[stage], sphase);
            const uint8_t* tile = ring + stage * TB;
            uint32_t bf[2][4][2];
#pragma unroll
            for (int n = 0; n < 2; ++n)
                unpack16<BITS>(tile + (16 * warp + 8 * n + gq) * row_bytes(BITS) + tq * 2 * BITS, bf[n]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == NST) { stage = 0; sphase ^= 1; }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int pos = (kb * 64 + tq * 16 + 4 * j) * 2;  // byte offset inside the row
#pragma unroll
                for (int m = 0; m < MT; ++m) {
                    if (m == 1 && !two) break;
                    const uint2 lo = *reinterpret_cast<const uint2*>(act + (16 * m + gq) * ASTR + pos);
                    const uint2 hi = *reinterpret_cast<const uint2*>(act + (16 * m + gq + 8) * ASTR + pos);
#pragma unroll
                    for (int n = 0; n < 2; ++n) mma_16816(acc[m][n], lo.x, hi.x, lo.y, hi.y, bf[n][j][0], bf[n][j][1]);
                }
            }
        }

        // ---- split-K reduction (fixed order) + epilogue ----
        const int S = p1 ? s1 : s2;
        const int Np = p1 ? g.Np1 : g.Np2;
        float* part = g.partial + (p1 || s1 == 1 ? 0 : int64_t(s1) * g.part_rows * g.Np1);
        bool do_epi = true;
        if (S > 1) {
#pragma unroll
            for (int m = 0; m < MT; ++m)
#pragma unroll
                for (int n = 0; n < 2; ++n)
#pragma unroll
                    for (int hr = 0; hr < 2; ++hr) {
                        const int r = 16 * m + gq + 8 * hr;
                        if (r >= it.nrows) continue;
                        const int ch = it.mt * TILE_N + 16 * warp + 8 * n + 2 * tq;
                        float2* dst = reinterpret_cast<float2*>(part + (int64_t(it.ks) * g.part_rows + it.row0 + r) * Np + ch);
                        __stcg(dst, make_float2(acc[m][n][2 * hr], acc[m][n][2 * hr + 1]));
                    }
            __threadfence();
            named_bar_sync(1, kGemvConsumers * 32);
            unsigned* cnt = g.split_cnt + (p1 ? 0 : g.E * max(nmt1, nmt2)) + it.e * max(nmt1, nmt2) + it.mt;
            if (ctid == 0) s_flag = atomicAdd(cnt, 1u) == unsigned(S * it.npass - 1);
            named_bar_sync(1, kGemvConsumers * 32);
            do_epi = s_flag;
            if (do_epi) {
                __threadfence();
                if (ctid == 0) *cnt = 0;  // self-reset
                // rows of every pass of this (expert, m-tile) are ours to finish
            }
        }
        if (do_epi) {
            const int npass_here = S > 1 ? it.npass : 1;
            for (int ps = 0; ps < npass_here; ++ps) {
                const int row0 = S > 1 ? P.offsets[it.e] + ps * ROWS : it.row0;
                const int nrows = S > 1 ? min(ROWS, P.counts[it.e] - ps * ROWS) : it.nrows;
#pragma unroll
                for (int m = 0; m < MT; ++m)
#pragma unroll
                    for (int n = 0; n < 2; ++n)
#pragma unroll
                        for (int hr = 0; hr < 2; ++hr) {
                            const int r = 16 * m + gq + 8 * hr;
                            if (r >= nrows) continue;
                            const int ch = it.mt * TILE_N + 16 * warp + 8 * n + 2 * tq;
                            float v0, v1;
                            if (S > 1) {
                                v0 = 0.f;
                                v1 = 0.f;
                                for (int ks = 0; ks < S; ++ks) {
                                    const float2 pv = __ldcg(reinterpret_cast<const float2*>(
                                        part + (int64_t(ks) * g.part_rows + row0 + r) * Np + ch));
                                    v0 += pv.x;
                                    v1 += pv.y;
                                }
                            } else {
                                v0 = acc[m][n][2 * hr];
                                v1 = acc[m][n][2 * hr + 1];
                            }
                            const int pos = row0 + r;
                            if (p1) {
                                const float* sc = g.s1 + int64_t(it.e) * g.Np1;
                                float y0 = v0 * sc[ch], y1 = v1 * sc[ch + 1];
                                if (g.b1) { y0 += g.b1[int64_t(it.e) * g.Np1 + ch]; y1 += g.b1[int64_t(it.e) * g.Np1 + ch + 1]; }
                                y0 = y0 > 0.f ? y0 : 0.f;
                                y1 = y1 > 0.f ? y1 : 0.f;
                                *reinterpret_cast<__half2*>(g.mid + int64_t(pos) * g.Np1 + ch) = __floats2half2_rn(y0, y1);
                            } else {
                                const float* sc = g.s2 + int64_t(it.e) * g.Np2;
                                float y0 = v0 * sc[ch], y1 = v1 * sc[ch + 1];
                                if (g.b2) { y0 += g.b2[int64_t(it.e) * g.Np2 + ch]; y1 += g.b2[int64_t(it.e) * g.Np2 + ch + 1]; }
                                const float gt = P.perm_gate[pos];
                                const int64_t tok = P.perm_token[pos];
                                y0 *= gt;
                                y1 *= gt;
                                if (g.out_acc) {
                                    if (ch < g.d) atomicAdd(g.out_acc + tok * g.d + ch, y0);
                                    if (ch + 1 < g.d) atomicAdd(g.out_acc + tok * g.d + ch + 1, y1);
                                } else if (g.out_f16) {
                                    __half* o = static_cast<__half*>(g.out) + tok * g.d;
                                    if (ch < g.d) o[ch] = __float2half_rn(y0);
                                    if (ch + 1 < g.d) o[ch + 1] = __float2half_rn(y1);
                                } else {
                                    float* o = static_cast<float*>(g.out) + tok * g.d;
                                    if (ch < g.d) o[ch] = y0;
                                    if (ch + 1 < g.d) o[ch + 1] = y1;
                                }
                            }
                        }
            }
            if (p1) {
                __threadfence();
                named_bar_sync(1, kGemvConsumers * 32);
                if (ctid == 0) atomicAdd(&P.done[it.e], unsigned(S > 1 ? it.npass : 1));
            }
        }
        // release the item slot (activations are re-staged for the next item)
        named_bar_sync(1, kGemvConsumers * 32);
        if (lane == 0) mbar_arrive(&iempty[q]);
        if (++q == kItemQ) { q = 0; qphase ^= 1; }
    }
}

namespace {
template <int BITS, int MT>
size_t gemv_smem() {
    return size_t(GemvCfg<BITS>::NST) * GemvCfg<BITS>::TB + size_t(16 * MT) * (kGemvKC * 2 + 8) +
           (2 * GemvCfg<BITS>::NST + 2 * kItemQ) * 8 + kItemQ * sizeof(GemvItem) + 64;
}

template <int BITS, int MT>
cudaError_t launch_gemv_t(const GemvArgs& g, const Plan& P, cudaStream_t st, int num_sms) {
    auto kern = k_ffn_gemv<BITS, MT>;
    const size_t smem = gemv_smem<BITS, MT>();
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

cudaError_t launch_gemv(int bits, bool two_m16, const GemvArgs& g, const Plan& P, cudaStream_t st, int num_sms) {
#define MOQE_GEMV_CASE(B)                                                                \
    if (bits == B) return two_m16 ? launch_gemv_t<B, 2>(g, P, st, num_sms) : launch_gemv_t<B, 1>(g, P, st, num_sms);
    MOQE_GEMV_CASE(2)
    MOQE_GEMV_CASE(3)
    MOQE_GEMV_CASE(4)
    MOQE_GEMV_CASE(8)
#undef MOQE_GEMV_CASE
    return cudaErrorInvalidValue;
}

}  // namespace moqe_gpu
