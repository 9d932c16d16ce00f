// ffn_gemm_tc.cu — prefill path: tcgen05 grouped GEMM over experts with the
// weight dequantization done in smem staging (fc1 -> ReLU, then fc2 -> gate
// combine; one persistent launch per layer of the FFN).
//
// Reference: moe_ffn_forward proj/src/model.cpp:370-390 (dequantize + matmul +
// add_bias + relu + matmul + add_bias + gate scatter) and its fused CPU
// analogue matmul_dequant_fused proj/src/bench.cpp:11-47.
//
// Orientation (swap-AB): D[128 channels x BN tokens] += Wq^T[ch][k] . X[tok][k]
//   A = weights, M = 128 output channels, K-major fp16 codes (exact integers),
//       built in smem by converter warps from the packed device tiles;
//   B = activations (expert-grouped rows of x_perm or mid), K-major, loaded
//       by TMA with 128-byte swizzle;
//   D = fp32 in TMEM (two 256-column accumulators, MMA of tile i+1 overlaps
//       the epilogue of tile i).
// The per-output-channel scale factors out of the k-sum and is applied in the
// epilogue together with the bias and ReLU (fc1) or gate-weighted combine (fc2).
//
// Warp roles (512 threads, one CTA per SM, persistent static tile schedule):
//   warp 0      TMA producer (packed weight tile: 1-D bulk; activation tile: 2-D tensor,
//               optionally multicast across a cluster along M)
//   warp 1      MMA issuer (one elected lane issues tcgen05.mma, commits to mbarriers)
//   warp 2      TMEM allocator
//   warps 4-11  converters: packed codes -> fp16 SW128 K-major A tile (codec.cuh),
//               A double-buffered apart from the 4-deep TMA ring
//   warps 12-15 epilogue: tcgen05.ld -> scale/bias/act -> global
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "codec.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace moqe_gpu {

constexpr int kBM = 128;           // output channels per tile (UMMA M)
constexpr int kBN = 256;           // tokens per tile (UMMA N)
constexpr int kBK = 64;            // k per stage (one 128-byte swizzle atom of fp16)
constexpr int kStages = 4;        // TMA ring: packed weight tile + activation tile
constexpr int kAStages = 2;       // converted fp16 A tiles (double buffer)
constexpr int kConvThreads = 256; // warps 4..11
constexpr int kGemmThreads = 512;
constexpr int kATile = kBM * kBK * 2;   // 16 KB
constexpr int kBTile = kBN * kBK * 2;   // 32 KB
constexpr int kTmemCols = 512;

bool gemm_available() { return true; }
int gemm_block_n() { return kBN; }
// UMMA N of a 2-SM tile with `nvalid` tokens: a multiple of 32 (N/2 rows per CTA, whole
// 8-row swizzle atoms), at most kBN
__host__ __device__ constexpr int tile_n(int nvalid) { return nvalid >= kBN ? kBN : (nvalid + 31) / 32 * 32; }

struct GemmParams {
    CUtensorMap tmap_b;  // activation matrix (x_perm for fc1, mid for fc2)
};

// ---- tcgen05 / TMEM helpers -------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)), "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// 32 lanes x 32 columns of 32-bit, one register per column
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major operand, 128-byte swizzle, 8-row
// core-matrix groups 1024 B apart (SBO), sm_100 descriptor version 1.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFFu);        // start address
    d |= uint64_t(1) << 16;                        // LBO (unused for swizzled K-major)
    d |= uint64_t(1024 >> 4) << 32;                // SBO
    d |= uint64_t(1) << 46;                        // version (sm_100)
    d |= uint64_t(2) << 61;                        // SWIZZLE_128B
    return d;
}
// Instruction descriptor: kind::f16, A/B fp16, D fp32, both K-major, M=128, N=kBN.
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
    return (1u << 4) | (0u << 7) | (0u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-D TMA load multicast to every CTA of the cluster in `mask` (same smem offset, same mbarrier offset).
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const void* tmap, int32_t c0, int32_t c1, uint64_t* bar,
                                               uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
// MMA completion -> arrive on the same mbarrier in every CTA of `mask`.
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

struct GemmTile {
    int e, mt, row0, nvalid;
};

// Super-tile t -> (expert, m-group, n-tile); the CTA of cluster rank r takes
// m-tile mg*CS + r. Tiles are ordered (expert, m-group, n-tile).
__device__ __forceinline__ GemmTile decode_tile(int t, const int* s_list, const int* s_off, const int* s_cnt,
                                                const int* s_tstart, int n_gemm, int nmg, int cs, int rank) {
    int lo = 0, hi = n_gemm - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_tstart[mid] * nmg <= t) lo = mid; else hi = mid - 1;
    }
    const int r = t - s_tstart[lo] * nmg;
    const int ntl = s_tstart[lo + 1] - s_tstart[lo];
    const int mg = r / ntl, nt = r % ntl;
    GemmTile g;
    g.e = s_list[lo];
    g.mt = mg * cs + rank;
    g.row0 = s_off[lo] + nt * kBN;
    g.nvalid = min(kBN, s_cnt[lo] - nt * kBN);
    return g;
}


// Epilogue for one accumulator tile (128 channels x nvalid tokens) owned by the
// 4 epilogue warps: TMEM (lane = channel, column = token) -> registers ->
// scale/bias/act -> smem transpose [32 tokens][128 channels] -> coalesced
// 16-byte row stores (fc1: fp16 mid rows; fc2: gate-scaled fp32/fp16 output rows
// of the routed tokens, or fp32 atomics for top-2 accumulation).
__device__ __forceinline__ void epilogue_tile(const GemmArgs& g, bool p1, const GemmTile& tl, uint32_t taddr,
                                              float scale, float bias, const int* s_tok, const float* s_gate,
                                              float* stage, int q, int lane, int et) {
    const int mt0 = tl.mt * kBM;
    for (int c0 = 0; c0 < tl.nvalid; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(taddr + uint32_t(c0), r);
        const int nj = min(32, tl.nvalid - c0);
        const int cl = 32 * q + lane;  // local channel
        named_bar_sync(2, 128);        // previous chunk's readers are done with `stage`
        if (p1) {
            __half* st = reinterpret_cast<__half*>(stage);  // [32][128] fp16
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float y = __uint_as_float(r[j]) * scale + bias;
                st[j * kBM + cl] = __float2half_rn(y > 0.f ? y : 0.f);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) stage[j * (kBM + 4) + cl] = __uint_as_float(r[j]) * scale + bias;
        }
        named_bar_sync(2, 128);
        if (p1) {
            // 32 rows x 256 B: 512 16-byte pieces, 4 per thread
            const uint4* st4 = reinterpret_cast<const uint4*>(stage);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int idx = i * 128 + et, j = idx >> 4, c16 = idx & 15;
                if (j < nj)
                    *reinterpret_cast<uint4*>(g.mid + int64_t(tl.row0 + c0 + j) * g.Np1 + mt0 + c16 * 8) = st4[j * 16 + c16];
            }
        } else {
            // 32 rows x 128 channels fp32: a warp per row at a time, 4 channels per lane
            for (int j = q; j < nj; j += 4) {
                const int chl = 4 * lane, ch = mt0 + chl;
                if (ch >= g.d) continue;
                const float gt = s_gate[c0 + j];
                const float4 v = *reinterpret_cast<const float4*>(stage + j * (kBM + 4) + chl);
                const float y0 = v.x * gt, y1 = v.y * gt, y2 = v.z * gt, y3 = v.w * gt;
                const int64_t o = int64_t(s_tok[c0 + j]) * g.d + ch;
                const bool full4 = ch + 3 < g.d;
                if (g.out_acc) {
                    atomicAdd(g.out_acc + o, y0);
                    if (ch + 1 < g.d) atomicAdd(g.out_acc + o + 1, y1);
                    if (ch + 2 < g.d) atomicAdd(g.out_acc + o + 2, y2);
                    if (ch + 3 < g.d) atomicAdd(g.out_acc + o + 3, y3);
                } else if (g.out_f16) {
                    __half* op = static_cast<__half*>(g.out) + o;
                    if (full4 && (o & 3) == 0) {
                        __half2 a = __floats2half2_rn(y0, y1), b = __floats2half2_rn(y2, y3);
                        uint2 pk;
                        pk.x = *reinterpret_cast<uint32_t*>(&a);
                        pk.y = *reinterpret_cast<uint32_t*>(&b);
                        *reinterpret_cast<uint2*>(op) = pk;
                    } else {
                        op[0] = __float2half_rn(y0);
                        if (ch + 1 < g.d) op[1] = __float2half_rn(y1);
                        if (ch + 2 < g.d) op[2] = __float2half_rn(y2);
                        if (ch + 3 < g.d) op[3] = __float2half_rn(y3);
                    }
                } else {
                    float* op = static_cast<float*>(g.out) + o;
                    if (full4 && (o & 3) == 0) {
                        *reinterpret_cast<float4*>(op) = make_float4(y0, y1, y2, y3);
                    } else {
                        op[0] = y0;
                        if (ch + 1 < g.d) op[1] = y1;
                        if (ch + 2 < g.d) op[2] = y2;
                        if (ch + 3 < g.d) op[3] = y3;
                    }
                }
            }
        }
    }
}

template <int BITS, int CS>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_ffn_gemm(const __grid_constant__ GemmParams prm, GemmArgs g, Plan P, int phase) {
    constexpr int TB = tile_bytes(BITS);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;                                 // [kAStages][16 KB]
    uint8_t* sB = sA + kAStages * kATile;               // [kStages][32 KB]
    uint8_t* sP = sB + kStages * kBTile;                // [kStages][TB] packed codes
    uint64_t* full = reinterpret_cast<uint64_t*>(sP + kStages * TB);
    uint64_t* empty = full + kStages;
    uint64_t* afull = empty + kStages;                  // [kAStages]
    uint64_t* aempty = afull + kAStages;                // [kAStages]
    uint64_t* accf = aempty + kAStages;                 // [2]
    uint64_t* acce = accf + 2;                          // [2]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acce + 2);
    int* s_list = reinterpret_cast<int*>(s_tmem + 4);   // [256]
    int* s_off = s_list + 256;
    int* s_cnt = s_off + 256;
    int* s_tstart = s_cnt + 256;                        // [257]
    int* s_tok = s_tstart + 260;                        // [kBN] epilogue token ids (fc2)
    float* s_gate = reinterpret_cast<float*>(s_tok + kBN);  // [kBN] gates (fc2)
    float* s_stage = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(s_gate + kBN) + 15) & ~uintptr_t(15));  // [32][132] epilogue transpose

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_gemm = P.meta[1];
    if (n_gemm == 0) return;
    const bool p1 = phase == 1;
    const int Kp = p1 ? g.Kp1 : g.Kp2;
    const int Np = p1 ? g.Np1 : g.Np2;
    const int nmt = Np / kBM;
    const int nmg = nmt / CS;          // m-groups (one per cluster super-tile)
    const int nkb = Kp / kBK;
    const int ntiles = nmg * P.meta[2];
    const int rank = CS > 1 ? int(cluster_rank()) : 0;
    const int cid = int(blockIdx.x) / CS, ncl = int(gridDim.x) / CS;
    constexpr uint16_t kMask = uint16_t((1u << CS) - 1u);
    constexpr int kSlice = kBN / CS;   // B rows each CTA fetches and multicasts

    for (int a = threadIdx.x; a < n_gemm; a += blockDim.x) {
        const int e = P.gemm_list[a];
        s_list[a] = e;
        s_off[a] = P.offsets[e];
        s_cnt[a] = P.counts[e];
        s_tstart[a] = P.gemm_tile_start[a];
    }
    if (threadIdx.x == 0) {
        s_tstart[n_gemm] = P.gemm_tile_start[n_gemm];
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CS);  // one MMA-commit arrival from every CTA of the cluster
        }
        for (int s = 0; s < kAStages; ++s) {
            mbar_init(&afull[s], kConvThreads);
            mbar_init(&aempty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&accf[s], 1);
            mbar_init(&acce[s], 128);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(s_tmem, kTmemCols);
    tc_fence_before();
    __syncthreads();
    if (CS > 1) cluster_sync_all();  // peers' barriers initialised before any multicast
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            prefetch_tmap(&prm.tmap_b);
            const uint8_t* wbase = p1 ? g.w1 : g.w2;
            const int64_t wstride = p1 ? g.w1_stride : g.w2_stride;
            int s = 0, ph = 0;
            for (int t = cid; t < ntiles; t += ncl) {
                const GemmTile tl = decode_tile(t, s_list, s_off, s_cnt, s_tstart, n_gemm, nmg, CS, rank);
                const uint8_t* wt = wbase + int64_t(tl.e) * wstride + int64_t(tl.mt) * nkb * TB;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);  // every CTA of the cluster is done with stage s
                    mbar_arrive_expect_tx(&full[s], TB + kBTile);
                    bulk_g2s(sP + s * TB, wt + int64_t(kb) * TB, TB, &full[s]);
                    if (CS == 1)
                        tma_load_2d(sB + s * kBTile, &prm.tmap_b, kb * kBK, tl.row0, &full[s]);
                    else  // this CTA's slice of the shared activation tile, to all CTAs of the cluster
                        tma_load_2d_mc(sB + s * kBTile + rank * kSlice * 128, &prm.tmap_b, kb * kBK,
                                       tl.row0 + rank * kSlice, &full[s], kMask);
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16(kBM, kBN);
            int s = 0, ph = 0, a = 0, aph2 = 0, as = 0, aph = 0;
            for (int t = cid; t < ntiles; t += ncl) {
                mbar_wait(&acce[as], aph ^ 1);
                tc_fence_after();
                const uint32_t dt = tmem + uint32_t(as * kBN);
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&afull[a], aph2);
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint64_t ad = smem_desc_sw128(smem_u32(sA + a * kATile));
                    const uint64_t bd = smem_desc_sw128(smem_u32(sB + s * kBTile));
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)  // +32 bytes per k16 step inside the swizzle atom
                        tc_mma_f16(dt, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb | k) != 0);
                    tc_commit(&aempty[a]);
                    if (CS == 1) tc_commit(&empty[s]);
                    else tc_commit_mc(&empty[s], kMask);  // frees stage s in every CTA of the cluster
                    if (++s == kStages) { s = 0; ph ^= 1; }
                    if (++a == kAStages) { a = 0; aph2 ^= 1; }
                }
                tc_commit(&accf[as]);
                if (++as == 2) { as = 0; aph ^= 1; }
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ===== converters: thread -> (A row m, chunk pair hc) =====
        const int ct = threadIdx.x - 128;
        const int m = ct & 127, hc = ct >> 7;  // chunks 2hc, 2hc+1 of the row
        int s = 0, ph = 0, a = 0, aph2 = 0;
        for (int t = cid; t < ntiles; t += ncl) {
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&full[s], ph);
                mbar_wait(&aempty[a], aph2 ^ 1);
                const uint8_t* row = sP + s * TB + m * row_bytes(BITS);
                uint8_t* arow = sA + a * kATile + m * 128;
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    const int c = 2 * hc + cc;
                    uint32_t o[8];
                    if (g.log_codes) unpack_chunk_log<BITS>(row, c, o);  // log-scale bank (quant.cpp:226-243)
                    else unpack_chunk<BITS>(row, c, o);
                    // 16-byte chunks 2c, 2c+1 of the 128-byte row, swizzled by (row % 8)
                    *reinterpret_cast<uint4*>(arow + (((2 * c) ^ (m & 7)) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
                    *reinterpret_cast<uint4*>(arow + (((2 * c + 1) ^ (m & 7)) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
                }
                fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
                mbar_arrive(&afull[a]);
                if (++s == kStages) { s = 0; ph ^= 1; }
                if (++a == kAStages) { a = 0; aph2 ^= 1; }
            }
        }
    } else if (warp >= 12) {
        // ===== epilogue: TMEM lanes (channels) 32*(warp%4) .. +31 =====
        const int q = warp & 3;
        const int et = threadIdx.x - 384;  // 0..127
        int as = 0, aph = 0;
        for (int t = cid; t < ntiles; t += ncl) {
            const GemmTile tl = decode_tile(t, s_list, s_off, s_cnt, s_tstart, n_gemm, nmg, CS, rank);
            const int ch = tl.mt * kBM + 32 * q + lane;
            const float* sc = p1 ? g.s1 + int64_t(tl.e) * g.Np1 : g.s2 + int64_t(tl.e) * g.Np2;
            const float* bi = p1 ? g.b1 : g.b2;
            const float scale = __ldg(sc + ch);
            const float bias = bi ? __ldg(bi + int64_t(tl.e) * Np + ch) : 0.f;
            if (!p1) {
                // token ids / gates of this tile's rows -> smem (shared by the 4 warps)
                named_bar_sync(2, 128);
                for (int j = et; j < tl.nvalid; j += 128) {
                    s_tok[j] = P.perm_token[tl.row0 + j];
                    s_gate[j] = P.perm_gate[tl.row0 + j];
                }
                named_bar_sync(2, 128);
            }
            mbar_wait(&accf[as], aph);
            tc_fence_after();
            const uint32_t taddr = tmem + (uint32_t(32 * q) << 16) + uint32_t(as * kBN);
            epilogue_tile(g, p1, tl, taddr, scale, bias, s_tok, s_gate, s_stage, q, lane, et);
            tc_fence_before();
            mbar_arrive(&acce[as]);
            if (++as == 2) { as = 0; aph ^= 1; }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (CS > 1) cluster_sync_all();  // no CTA leaves while peers may still multicast into it
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, kTmemCols);
    }
}

// ============================ 2-SM variant (cta_group::2) ==============================
// A CTA pair (cluster of 2 on one TPC) computes a 256-channel x 256-token tile:
// each CTA converts its own 128 weight rows into its A buffer and TMA-loads its
// own 128-token half of the activation tile; the leader (rank 0) issues
// tcgen05.mma.cta_group::2 (M=256, N=256) that reads A and B from both SMs'
// shared memory and writes each CTA's 128 accumulator rows into its own TMEM.
// Per-SM operand traffic is half of the 1-SM kernel's.
constexpr int kBHalf = kBTile / 2;  // 16 KB: 128 token rows x 64 k
// TMA ring depth for the 2-SM kernel: as many (B half + packed tile) stages as
// fit next to the double-buffered A tiles (~200 KB of shared memory).
__host__ __device__ constexpr int stages2(int bits) { return (184 * 1024 - kAStages * kATile) / (kBHalf + tile_bytes(bits)); }

__device__ __forceinline__ uint32_t leader_addr(const void* p) { return smem_u32(p) & 0xFEFFFFFFu; }
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const void* tmap, int32_t c0, int32_t c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tc_mma_f16_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tc_commit_2sm_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

template <int BITS>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_ffn_gemm2(const __grid_constant__ GemmParams prm, GemmArgs g, Plan P, int phase) {
    constexpr int TB = tile_bytes(BITS);
    constexpr int kStages = stages2(BITS);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;                                 // [kAStages][16 KB]  own 128 rows
    uint8_t* sB = sA + kAStages * kATile;               // [kStages][16 KB]   own 128 tokens
    uint8_t* sP = sB + kStages * kBHalf;                // [kStages][TB]      own packed rows
    uint64_t* pfull = reinterpret_cast<uint64_t*>(sP + kStages * TB);  // local: packed landed
    uint64_t* bfull = pfull + kStages;                  // leader: both B halves landed
    uint64_t* empty = bfull + kStages;                  // local: MMA done with stage (multicast commit)
    uint64_t* afull = empty + kStages;                  // leader: both CTAs' A converted
    uint64_t* aempty = afull + kAStages;                // local: MMA done with A buffer
    uint64_t* accf = aempty + kAStages;                 // local: accumulator ready
    uint64_t* acce = accf + 2;                          // leader: both epilogues drained
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acce + 2);
    int* s_list = reinterpret_cast<int*>(s_tmem + 4);
    int* s_off = s_list + 256;
    int* s_cnt = s_off + 256;
    int* s_tstart = s_cnt + 256;
    int* s_tok = s_tstart + 260;
    float* s_gate = reinterpret_cast<float*>(s_tok + kBN);
    float* s_stage = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(s_gate + kBN) + 15) & ~uintptr_t(15));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_gemm = P.meta[1];
    if (n_gemm == 0) return;
    const bool p1 = phase == 1;
    const int Kp = p1 ? g.Kp1 : g.Kp2;
    const int Np = p1 ? g.Np1 : g.Np2;
    const int nmg = Np / (2 * kBM);
    const int nkb = Kp / kBK;
    const int ntiles = nmg * P.meta[2];
    const int rank = int(cluster_rank());
    const int cid = int(blockIdx.x) >> 1, ncl = int(gridDim.x) >> 1;

    for (int a = threadIdx.x; a < n_gemm; a += blockDim.x) {
        const int e = P.gemm_list[a];
        s_list[a] = e;
        s_off[a] = P.offsets[e];
        s_cnt[a] = P.counts[e];
        s_tstart[a] = P.gemm_tile_start[a];
    }
    if (threadIdx.x == 0) {
        s_tstart[n_gemm] = P.gemm_tile_start[n_gemm];
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&pfull[s], 1);
            mbar_init(&bfull[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < kAStages; ++s) {
            mbar_init(&afull[s], 2 * (kConvThreads / 32));  // one arrival per converter warp, both CTAs
            mbar_init(&aempty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&accf[s], 1);
            mbar_init(&acce[s], 2 * 4);  // one arrival per epilogue warp, both CTAs
        }
        fence_barrier_init();
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 0) {
        // ===== TMA producer (both CTAs) =====
        if (lane == 0) {
            prefetch_tmap(&prm.tmap_b);
            const uint8_t* wbase = p1 ? g.w1 : g.w2;
            const int64_t wstride = p1 ? g.w1_stride : g.w2_stride;
            int s = 0, ph = 0;
            for (int t = cid; t < ntiles; t += ncl) {
                const GemmTile tl = decode_tile(t, s_list, s_off, s_cnt, s_tstart, n_gemm, nmg, 2, rank);
                const uint8_t* wt = wbase + int64_t(tl.e) * wstride + int64_t(tl.mt) * nkb * TB;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&pfull[s], TB);
                    bulk_g2s(sP + s * TB, wt + int64_t(kb) * TB, TB, &pfull[s]);
                    if (rank == 0) mbar_arrive_expect_tx(&bfull[s], 2 * kBHalf);
                    // the pair splits the tile's N = tile_n(nvalid) rows: CTA r holds rows [r N/2, (r+1) N/2)
                    // (the fixed kBN/2-row box is a superset; the MMA reads the first N/2 rows)
                    tma_load_2d_2sm(sB + s * kBHalf, &prm.tmap_b, kb * kBK, tl.row0 + rank * (tile_n(tl.nvalid) / 2),
                                    leader_addr(&bfull[s]));
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (leader only) =====
        if (rank == 0 && lane == 0) {
            int s = 0, ph = 0, a = 0, aph2 = 0, as = 0, aph = 0;
            for (int t = cid; t < ntiles; t += ncl) {
                // UMMA N sized to the tile's tokens (a 130-token expert no longer pays for 256)
                const GemmTile tl = decode_tile(t, s_list, s_off, s_cnt, s_tstart, n_gemm, nmg, 2, rank);
                const uint32_t idesc = idesc_f16(2 * kBM, tile_n(tl.nvalid));
                mbar_wait(&acce[as], aph ^ 1);
                tc_fence_after();
                const uint32_t dt = tmem + uint32_t(as * kBN);
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&afull[a], aph2);
                    mbar_wait(&bfull[s], ph);
                    tc_fence_after();
                    const uint64_t ad = smem_desc_sw128(smem_u32(sA + a * kATile));
                    const uint64_t bd = smem_desc_sw128(smem_u32(sB + s * kBHalf));
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                        tc_mma_f16_2sm(dt, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb | k) != 0);
                    tc_commit_2sm_mc(&aempty[a], 0x3);
                    tc_commit_2sm_mc(&empty[s], 0x3);
                    if (++s == kStages) { s = 0; ph ^= 1; }
                    if (++a == kAStages) { a = 0; aph2 ^= 1; }
                }
                tc_commit_2sm_mc(&accf[as], 0x3);
                if (++as == 2) { as = 0; aph ^= 1; }
            }
        }
    } else if (warp >= 4 && warp < 12) {
        // ===== converters (both CTAs): thread -> (A row m, chunk pair hc) =====
        const int ct = threadIdx.x - 128;
        const int m = ct & 127, hc = ct >> 7;
        const uint32_t afull_l = leader_addr(afull);
        int s = 0, ph = 0, a = 0, aph2 = 0;
        for (int t = cid; t < ntiles; t += ncl) {
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&pfull[s], ph);
                mbar_wait(&aempty[a], aph2 ^ 1);
                const uint8_t* row = sP + s * TB + m * row_bytes(BITS);
                uint8_t* arow = sA + a * kATile + m * 128;
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    const int c = 2 * hc + cc;
                    uint32_t o[8];
                    if (g.log_codes) unpack_chunk_log<BITS>(row, c, o);  // log-scale bank (quant.cpp:226-243)
                    else unpack_chunk<BITS>(row, c, o);
                    *reinterpret_cast<uint4*>(arow + (((2 * c) ^ (m & 7)) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
                    *reinterpret_cast<uint4*>(arow + (((2 * c + 1) ^ (m & 7)) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(afull_l + uint32_t(a * 8));
                if (++s == kStages) { s = 0; ph ^= 1; }
                if (++a == kAStages) { a = 0; aph2 ^= 1; }
            }
        }
    } else if (warp >= 12) {
        // ===== epilogue (both CTAs): own TMEM lanes = own 128 channels =====
        const int q = warp & 3;
        const int et = threadIdx.x - 384;
        const uint32_t acce_l = leader_addr(acce);
        int as = 0, aph = 0;
        for (int t = cid; t < ntiles; t += ncl) {
            const GemmTile tl = decode_tile(t, s_list, s_off, s_cnt, s_tstart, n_gemm, nmg, 2, rank);
            const int ch = tl.mt * kBM + 32 * q + lane;
            const float* sc = p1 ? g.s1 + int64_t(tl.e) * g.Np1 : g.s2 + int64_t(tl.e) * g.Np2;
            const float* bi = p1 ? g.b1 : g.b2;
            const float scale = __ldg(sc + ch);
            const float bias = bi ? __ldg(bi + int64_t(tl.e) * Np + ch) : 0.f;
            if (!p1) {
                named_bar_sync(2, 128);
                for (int j = et; j < tl.nvalid; j += 128) {
                    s_tok[j] = P.perm_token[tl.row0 + j];
                    s_gate[j] = P.perm_gate[tl.row0 + j];
                }
                named_bar_sync(2, 128);
            }
            mbar_wait(&accf[as], aph);
            tc_fence_after();
            const uint32_t taddr = tmem + (uint32_t(32 * q) << 16) + uint32_t(as * kBN);
            epilogue_tile(g, p1, tl, taddr, scale, bias, s_tok, s_gate, s_stage, q, lane, et);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acce_l + uint32_t(as * 8));
            if (++as == 2) { as = 0; aph ^= 1; }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

bool make_tmap(CUtensorMap* m, const __half* base, int64_t rows, int64_t cols, int box_rows) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(cols * 2)};
    cuuint32_t box[2] = {cuuint32_t(kBK), cuuint32_t(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BITS>
size_t gemm_smem() {
    return 1024 + size_t(kAStages) * kATile + size_t(kStages) * (kBTile + tile_bytes(BITS)) +
           (2 * kStages + 2 * kAStages + 4) * 8 + 16 +
           sizeof(int) * (256 * 3 + 260 + kBN) + sizeof(float) * kBN + 64 + 16 + 32 * (kBM + 4) * 4;
}

template <int BITS>
size_t gemm2_smem() {
    constexpr int ns = stages2(BITS);
    return 1024 + size_t(kAStages) * kATile + size_t(ns) * (kBHalf + tile_bytes(BITS)) +
           (3 * ns + 2 * kAStages + 4) * 8 + 16 + sizeof(int) * (256 * 3 + 260 + kBN) + sizeof(float) * kBN + 64 + 16 + 32 * (kBM + 4) * 4;
}

template <int BITS>
cudaError_t launch_gemm_2sm(const GemmArgs& g, const Plan& P, int phase, cudaStream_t st, int num_sms) {
    GemmParams prm;
    const bool ok = phase == 1 ? make_tmap(&prm.tmap_b, g.x_perm, g.R, g.Kp1, kBN / 2)
                               : make_tmap(&prm.tmap_b, g.mid, g.R, g.Np1, kBN / 2);
    if (!ok) return cudaErrorInvalidValue;
    auto kern = k_ffn_gemm2<BITS>;
    const size_t smem = gemm2_smem<BITS>();
    static int max_clusters_dev[kMaxDevices] = {};  // per device: attribute + co-resident clusters
    int dev = 0;
    cudaGetDevice(&dev);
    int& max_clusters = max_clusters_dev[dev < kMaxDevices ? dev : 0];
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    if (max_clusters == 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t q{};
        q.gridDim = dim3(unsigned(num_sms / 2 * 2));
        q.blockDim = dim3(kGemmThreads);
        q.dynamicSmemBytes = smem;
        q.attrs = attr;
        q.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &q) != cudaSuccess || max_clusters <= 0)
            max_clusters = num_sms / 2;
        max_clusters = std::min(max_clusters, num_sms / 2);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(max_clusters * 2));
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, prm, g, P, phase);
}

template <int BITS, int CS>
cudaError_t launch_gemm_cs(const GemmArgs& g, const Plan& P, int phase, cudaStream_t st, int num_sms) {
    GemmParams prm;
    const bool ok = phase == 1 ? make_tmap(&prm.tmap_b, g.x_perm, g.R, g.Kp1, kBN / CS)
                               : make_tmap(&prm.tmap_b, g.mid, g.R, g.Np1, kBN / CS);
    if (!ok) return cudaErrorInvalidValue;
    auto kern = k_ffn_gemm<BITS, CS>;
    const size_t smem = gemm_smem<BITS>();
    static bool configured_dev[kMaxDevices] = {};
    static int max_clusters_dev[kMaxDevices] = {};  // co-resident clusters (GPC packing leaves SMs idle for CS=4)
    int dev = 0;
    cudaGetDevice(&dev);
    const int di = dev < kMaxDevices ? dev : 0;
    if (!configured_dev[di]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        configured_dev[di] = true;
    }
    cudaLaunchConfig_t cfg{};
    int& max_clusters = max_clusters_dev[di];
    if (max_clusters == 0) {
        cudaLaunchConfig_t q{};
        q.gridDim = dim3(unsigned(num_sms / CS * CS));
        q.blockDim = dim3(kGemmThreads);
        q.dynamicSmemBytes = smem;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = CS;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        q.attrs = qa;
        q.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &q) != cudaSuccess || max_clusters <= 0)
            max_clusters = num_sms / CS;
        max_clusters = std::min(max_clusters, num_sms / CS);
    }
    cfg.gridDim = dim3(unsigned(max_clusters * CS));
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, prm, g, P, phase);
}

template <int BITS>
cudaError_t launch_gemm_t(const GemmArgs& g, const Plan& P, int phase, cudaStream_t st, int num_sms) {
    // cluster of CS CTAs along M shares (multicasts) the activation tile
    const int nmt = (phase == 1 ? g.Np1 : g.Np2) / kBM;
    static const int pref = [] {
        const char* v = getenv("MOQE_GEMM_CLUSTER");
        return v ? atoi(v) : 1;
    }();
    static const bool two_sm = [] {
        const char* v = getenv("MOQE_GEMM_2SM");
        return v ? atoi(v) != 0 : true;
    }();
    if (two_sm && nmt % 2 == 0) return launch_gemm_2sm<BITS>(g, P, phase, st, num_sms);
    if (pref >= 4 && nmt % 4 == 0) return launch_gemm_cs<BITS, 4>(g, P, phase, st, num_sms);
    if (pref >= 2 && nmt % 2 == 0) return launch_gemm_cs<BITS, 2>(g, P, phase, st, num_sms);
    return launch_gemm_cs<BITS, 1>(g, P, phase, st, num_sms);
}

}  // namespace

cudaError_t launch_gemm(int bits, int phase, const GemmArgs& g, const Plan& P, cudaStream_t st, int num_sms) {
    switch (bits) {
        case 2: return launch_gemm_t<2>(g, P, phase, st, num_sms);
        case 3: return launch_gemm_t<3>(g, P, phase, st, num_sms);
        case 4: return launch_gemm_t<4>(g, P, phase, st, num_sms);
        case 8: return launch_gemm_t<8>(g, P, phase, st, num_sms);
    }
    return cudaErrorInvalidValue;
}

}  // namespace moqe_gpu
