// xrow.cuh — fc1 row blocks: the decode GEMV's B operand for one token and one 1024-k
// chunk (fixed-point digit planes in IMMA fragment order). Written by k_xrows, or by the
// decode router's copy warp (route.cu) from the token row it already holds in smem.
#pragma once
#include <stdint.h>

#include "common.cuh"
#include "frag.cuh"
#include "ptx.cuh"

namespace moqe_gpu {

constexpr int kStageK = 2 * TILE_K;  // k per IMMA stage (2 tiles)
constexpr int kChunkK = 1024;        // k per CTA of a cluster
constexpr int kChunkStages = kChunkK / kStageK;
constexpr int kZeroRow = -0x40000000;  // exponent sentinel: the row is (numerically) zero
__host__ __device__ constexpr int rup(int x, int a) { return (x + a - 1) / a * a; }

// Row block geometry. A plane holds 8 stages of STG bytes: stage st, fragment
// f, quad tq, register h -> the u32 at st*STG + f*32 + tq*8 + h*4 whose byte i
// is the digit of activation Frag::kidx(f, h, i) of that quad (codec order).
// Planes are PB bytes apart (PB = 32 mod 128) and row blocks XR bytes apart
// (XR = 64 mod 128), so the 8 column groups of a warp's LDS.64 hit distinct
// bank groups (two wavefronts, the minimum for 256 bytes).
template <int BITS>
struct RB {
    static constexpr int F = Frag<BITS>::F;
    static constexpr int STG = F * 32;
    static constexpr int PB = kChunkStages * STG + 32;
    static constexpr int HDR1 = 32;   // fc1: int p, float l1 (whole row), int64 Sum X (this chunk)
    static constexpr int HDR2 = 128;  // fc2: int p2 at 0, int64 Sum X2 of stage st at 64 + 8 st
    static constexpr int XR1 = rup(HDR1 + 3 * PB, 128) + 64;
    static constexpr int XR2 = rup(HDR2 + 4 * PB, 128) + 64;
};
struct XHead1 {
    int p;
    float l1;
    long long zsum;
};

// Lane (stage st = lane / 4, quad tq = lane % 4) of a warp owns the 32 activations of chunk
// positions st * kStageK + 16 tq + i and st * kStageK + 64 + 16 tq + i (i < 16): v[0..15],
// v[16..31]. m = max |x| and l1 = Sum |x| over the WHOLE row (every chunk of a row derives
// the same exponent). Writes the chunk's row block at blk (whole warp).
template <int BITS>
__device__ __forceinline__ void xrow_encode(const float (&v)[32], float m, float l1, uint8_t* blk, int lane) {
    using FR = Frag<BITS>;
    using R = RB<BITS>;
    constexpr int F = FR::F;
    const int st = lane >> 2, tq = lane & 3;
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
        XHead1 hd;
        hd.p = p;
        hd.l1 = l1 * (1.0f + 0x1p-9f);  // covers the fp32 summation error: an upper bound
        hd.zsum = zs;
        *reinterpret_cast<XHead1*>(blk) = hd;
    }
#pragma unroll
    for (int s = 0; s < 3; ++s) {
        const uint32_t sel = uint32_t(s) | (uint32_t(4 + s) << 4);
        uint8_t* dst = blk + R::HDR1 + s * R::PB + st * R::STG + tq * 8;
#pragma unroll
        for (int f = 0; f < F; ++f) {
            uint32_t b[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t lo = prmt(D[FR::kidx(f, h, 0)], D[FR::kidx(f, h, 1)], sel);
                const uint32_t hi = prmt(D[FR::kidx(f, h, 2)], D[FR::kidx(f, h, 3)], sel);
                b[h] = prmt(lo, hi, 0x5410u);
            }
            *reinterpret_cast<uint2*>(dst + f * 32) = make_uint2(b[0], b[1]);
        }
    }
}

}  // namespace moqe_gpu
