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
// Warp roles (384 threads, one CTA per SM, persistent static tile schedule):
//   warp 0      TMA producer (packed weight tile: 1-D bulk; activation tile: 2-D tensor)
//   warp 1      MMA issuer (one elected lane issues tcgen05.mma, commits to mbarriers)
//   warp 2      TMEM allocator
//   warps 4-7   converters: packed codes -> fp16 SW128 K-major A tile (codec.cuh)
//   warps 8-11  epilogue: tcgen05.ld -> scale/bias/act -> global
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "codec.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace moqe_gpu {

constexpr int kBM = 128;           // output channels per tile (UMMA M)
constexpr int kBN = 256;           // tokens per tile (UMMA N)
constexpr int kBK = 64;            // k per stage (one 128-byte swizzle atom of fp16)
constexpr int kStages = 3;
constexpr int kGemmThreads = 384;
constexpr int kATile = kBM * kBK * 2;   // 16 KB
constexpr int kBTile = kBN * kBK * 2;   // 32 KB
constexpr int kTmemCols = 512;

bool gemm_available() { return true; }
int gemm_block_n() { return kBN; }

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

struct GemmTile {
    int e, mt, row0, nvalid;
};

__device__ __forceinline__ GemmTile decode_tile(int t, const int* s_list, const int* s_off, const int* s_cnt,
                                                const int* s_tstart, int n_gemm, int nmt) {
    int lo = 0, hi = n_gemm - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_tstart[mid] * nmt <= t) lo = mid; else hi = mid - 1;
    }
    const int r = t - s_tstart[lo] * nmt;
    const int ntl = s_tstart[lo + 1] - s_tstart[lo];
    const int mt = r / ntl, nt = r % ntl;
    GemmTile g;
    g.e = s_list[lo];
    g.mt = mt;
    g.row0 = s_off[lo] + nt * kBN;
    g.nvalid = min(kBN, s_cnt[lo] - nt * kBN);
    return g;
}

template <int BITS>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_ffn_gemm(const __grid_constant__ GemmParams prm, GemmArgs g, Plan P, int phase) {
    constexpr int TB = tile_bytes(BITS);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;                                 // [kStages][16 KB]
    uint8_t* sB = sA + kStages * kATile;                // [kStages][32 KB]
    uint8_t* sP = sB + kStages * kBTile;                // [kStages][TB] packed codes
    uint64_t* full = reinterpret_cast<uint64_t*>(sP + kStages * TB);
    uint64_t* afull = full + kStages;
    uint64_t* empty = afull + kStages;
    uint64_t* accf = empty + kStages;                   // [2]
    uint64_t* acce = accf + 2;                          // [2]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(acce + 2);
    int* s_list = reinterpret_cast<int*>(s_tmem + 4);   // [256]
    int* s_off = s_list + 256;
    int* s_cnt = s_off + 256;
    int* s_tstart = s_cnt + 256;                        // [257]
    int* s_tok = s_tstart + 260;                        // [kBN] epilogue token ids (fc2)
    float* s_gate = reinterpret_cast<float*>(s_tok + kBN);  // [kBN] gates (fc2)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_gemm = P.meta[1];
    if (n_gemm == 0) return;
    const bool p1 = phase == 1;
    const int Kp = p1 ? g.Kp1 : g.Kp2;
    const int Np = p1 ? g.Np1 : g.Np2;
    const int nmt = Np / kBM;
    const int nkb = Kp / kBK;
    const int ntiles = nmt * P.meta[2];

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
            mbar_init(&afull[s], 128);
            mbar_init(&empty[s], 1);
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
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            prefetch_tmap(&prm.tmap_b);
            const uint8_t* wbase = p1 ? g.w1 : g.w2;
            const int64_t wstride = p1 ? g.w1_stride : g.w2_stride;
            int s = 0, ph = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const GemmTile tl = decode_tile(t, s_list, s_off, s_cnt, s_tstart, n_gemm, nmt);
                const uint8_t* wt = wbase + int64_t(tl.e) * wstride + int64_t(tl.mt) * nkb * TB;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], TB + kBTile);
                    bulk_g2s(sP + s * TB, wt + int64_t(kb) * TB, TB, &full[s]);
                    tma_load_2d(sB + s * kBTile, &prm.tmap_b, kb * kBK, tl.row0, &full[s]);
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16(kBM, kBN);
            int s = 0, ph = 0, as = 0, aph = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(&acce[as], aph ^ 1);
                tc_fence_after();
                const uint32_t dt = tmem + uint32_t(as * kBN);
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&afull[s], ph);
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint64_t ad = smem_desc_sw128(smem_u32(sA + s * kATile));
                    const uint64_t bd = smem_desc_sw128(smem_u32(sB + s * kBTile));
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)  // +32 bytes per k16 step inside the swizzle atom
                        tc_mma_f16(dt, ad + uint64_t(2 * k), bd + uint64_t(2 * k), idesc, (kb | k) != 0);
                    tc_commit(&empty[s]);
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
                tc_commit(&accf[as]);
                if (++as == 2) { as = 0; aph ^= 1; }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ===== converters: one output channel (A row) per thread =====
        const int m = threadIdx.x - 128;
        int s = 0, ph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&full[s], ph);
                const uint8_t* row = sP + s * TB + m * row_bytes(BITS);
                uint8_t* arow = sA + s * kATile + m * 128;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t o[8];
                    unpack_chunk<BITS>(row, c, o);
                    // 16-byte chunks 2c, 2c+1 of the 128-byte row, swizzled by (row % 8)
                    *reinterpret_cast<uint4*>(arow + (((2 * c) ^ (m & 7)) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
                    *reinterpret_cast<uint4*>(arow + (((2 * c + 1) ^ (m & 7)) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
                }
                fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
                mbar_arrive(&afull[s]);
                if (++s == kStages) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp >= 8) {
        // ===== epilogue: TMEM lanes (channels) 32*(warp%4) .. +31 =====
        const int q = warp & 3;
        const int et = threadIdx.x - 256;  // 0..127
        int as = 0, aph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const GemmTile tl = decode_tile(t, s_list, s_off, s_cnt, s_tstart, n_gemm, nmt);
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
            for (int c0 = 0; c0 < tl.nvalid; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(taddr + uint32_t(c0), r);
                const int nj = min(32, tl.nvalid - c0);
                if (p1) {
                    __half* mrow = g.mid + int64_t(tl.row0 + c0) * g.Np1 + ch;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (j < nj) {
                            const float y = __uint_as_float(r[j]) * scale + bias;
                            mrow[int64_t(j) * g.Np1] = __float2half_rn(y > 0.f ? y : 0.f);
                        }
                    }
                } else if (ch < g.d) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (j < nj) {
                            const float y = (__uint_as_float(r[j]) * scale + bias) * s_gate[c0 + j];
                            const int64_t o = int64_t(s_tok[c0 + j]) * g.d + ch;
                            if (g.out_acc) atomicAdd(g.out_acc + o, y);
                            else if (g.out_f16) static_cast<__half*>(g.out)[o] = __float2half_rn(y);
                            else static_cast<float*>(g.out)[o] = y;
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&acce[as]);
            if (++as == 2) { as = 0; aph ^= 1; }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, kTmemCols);
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

bool make_tmap(CUtensorMap* m, const __half* base, int64_t rows, int64_t cols) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(cols * 2)};
    cuuint32_t box[2] = {cuuint32_t(kBK), cuuint32_t(kBN)};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BITS>
size_t gemm_smem() {
    return 1024 + size_t(kStages) * (kATile + kBTile + tile_bytes(BITS)) + (3 * kStages + 4) * 8 + 16 +
           sizeof(int) * (256 * 3 + 260 + kBN) + sizeof(float) * kBN + 64;
}

template <int BITS>
cudaError_t launch_gemm_t(const GemmArgs& g, const Plan& P, int phase, cudaStream_t st, int num_sms) {
    GemmParams prm;
    const bool ok = phase == 1 ? make_tmap(&prm.tmap_b, g.x_perm, g.R, g.Kp1) : make_tmap(&prm.tmap_b, g.mid, g.R, g.Np1);
    if (!ok) return cudaErrorInvalidValue;
    auto kern = k_ffn_gemm<BITS>;
    const size_t smem = gemm_smem<BITS>();
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    kern<<<num_sms, kGemmThreads, smem, st>>>(prm, g, P, phase);
    return cudaGetLastError();
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
