// codec.cuh — device weight-tile codec (the bank's re-tiled format).
//
// A tile row holds the 64 codes W[kb*64 + kk][n] of one output channel n.
// It is split into four 16-code chunks (kk = 16t .. 16t+15, t = 0..3); each
// chunk is re-encoded — same bits, same byte count as the reference packing —
// so that one 32-bit word yields half2 PAIRS OF CONSECUTIVE CODES
// (k, k+1) with a single LOP3 (mask | 0x6400 magic) and one HFMA2, for most
// pairs without any shift: even codes live in the low 16-bit half, odd codes
// at the same bit position in the high half, and codes are kept inside the
// 10-bit fp16 mantissa wherever possible. The fp16 value of (magic | u<<s)
// is 1024 + u*2^s, so HFMA2(v, 2^-s, -(1024*2^-s + bias)) = u - bias exactly.
//
//   bits  row bytes  chunk t layout
//   8     64         bytes [16t, 16t+16): natural order (the reference packing)
//   4     32         two u32 at 8t: per word, low half nibbles c0 c2 c4 c6,
//                    high half c1 c3 c5 c7
//   3     24         u32 A at 4t: byte0 = c0 | c2<<3 | (c8&3)<<6, byte1 = c4 | c6<<3
//                    | (c10&3)<<6, byte2 = c1 | c3<<3 | (c9&3)<<6, byte3 = c5 | c7<<3 |
//                    (c11&3)<<6; u16 B at 16+2t: lo byte c12 | c14<<3 | (c8>>2)<<6 |
//                    (c10>>2)<<7, hi byte c13 | c15<<3 | (c9>>2)<<6 | (c11>>2)<<7
//                    (every field byte-aligned at the same offset in each byte, so
//                    one LOP3 yields four u8 codes for the decode IMMA path too)
//   2     16         u32 at 4t: low half c0 c2 .. c14 @2-bit slots, high half
//                    c1 c3 .. c15
// (u = code + 2^(bits-1), offset binary like bitpack.cpp:18-39.)
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "ptx.cuh"

namespace moqe_gpu {

// ---- encode (bank creation, one-time) --------------------------------------------
template <int BITS>
__device__ __forceinline__ void encode_row(const int (&q)[64], uint8_t* row) {
    const int bias = 1 << (BITS - 1);
    for (int t = 0; t < 4; ++t) {
        uint32_t u[16];
        for (int i = 0; i < 16; ++i) u[i] = uint32_t(q[16 * t + i] + bias);
        if (BITS == 8) {
            for (int i = 0; i < 16; ++i) row[16 * t + i] = uint8_t(u[i]);
        } else if (BITS == 4) {
            for (int w = 0; w < 2; ++w) {
                uint32_t W = 0;
                for (int i = 0; i < 4; ++i) W |= (u[8 * w + 2 * i] << (4 * i)) | (u[8 * w + 2 * i + 1] << (16 + 4 * i));
                for (int b = 0; b < 4; ++b) row[8 * t + 4 * w + b] = uint8_t(W >> (8 * b));
            }
        } else if (BITS == 2) {
            uint32_t W = 0;
            for (int p = 0; p < 8; ++p) W |= (u[2 * p] << (2 * p)) | (u[2 * p + 1] << (16 + 2 * p));
            for (int b = 0; b < 4; ++b) row[4 * t + b] = uint8_t(W >> (8 * b));
        } else {  // 3
            const uint32_t A = (u[0] | u[2] << 3 | (u[8] & 3u) << 6) | (u[4] | u[6] << 3 | (u[10] & 3u) << 6) << 8 |
                               (u[1] | u[3] << 3 | (u[9] & 3u) << 6) << 16 | (u[5] | u[7] << 3 | (u[11] & 3u) << 6) << 24;
            const uint32_t lo = u[12] | u[14] << 3 | (u[8] >> 2) << 6 | (u[10] >> 2) << 7;
            const uint32_t hi = u[13] | u[15] << 3 | (u[9] >> 2) << 6 | (u[11] >> 2) << 7;
            for (int b = 0; b < 4; ++b) row[4 * t + b] = uint8_t(A >> (8 * b));
            row[16 + 2 * t] = uint8_t(lo);
            row[16 + 2 * t + 1] = uint8_t(hi);
        }
    }
}

// ---- unpack (hot loops) --------------------------------------------------------------
__device__ __forceinline__ uint32_t h2_fma(uint32_t v, float s, float o) {
    __half2 r = __hfma2(*reinterpret_cast<__half2*>(&v), __float2half2_rn(s), __float2half2_rn(o));
    return *reinterpret_cast<uint32_t*>(&r);
}
// (w & mask) | 0x64006400 as ONE LOP3: the magic lives in a register (an
// opaque mov stops the compiler from splitting it into AND + OR immediates).
__device__ __forceinline__ uint32_t magic_reg() {
    uint32_t m;
    asm("mov.b32 %0, 0x64006400;" : "=r"(m));
    return m;
}
template <uint32_t MASK>
__device__ __forceinline__ uint32_t lop_magic(uint32_t w, uint32_t magic) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(w), "n"(MASK), "r"(magic));
    return d;
}

// Unpack chunk t of a tile row into 8 half2 pairs: out[p] = (code[16t+2p], code[16t+2p+1]).
template <int BITS>
__device__ __forceinline__ void unpack_chunk(const uint8_t* row, int t, uint32_t (&o)[8]) {
    const uint32_t mg = magic_reg();
    if constexpr (BITS == 4) {
        const uint2 w = *reinterpret_cast<const uint2*>(row + 8 * t);
        const uint32_t ws[2] = {w.x, w.y};
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const uint32_t a = ws[q], a8 = ws[q] >> 8;
            o[4 * q + 0] = h2_fma(lop_magic<0x000F000Fu>(a, mg), 1.0f, -1032.0f);
            o[4 * q + 1] = h2_fma(lop_magic<0x00F000F0u>(a, mg), 1.0f / 16, -72.0f);
            o[4 * q + 2] = h2_fma(lop_magic<0x000F000Fu>(a8, mg), 1.0f, -1032.0f);
            o[4 * q + 3] = h2_fma(lop_magic<0x00F000F0u>(a8, mg), 1.0f / 16, -72.0f);
        }
    } else if constexpr (BITS == 2) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(row + 4 * t);
        const uint32_t w10 = w >> 10;
        o[0] = h2_fma(lop_magic<0x00030003u>(w, mg), 1.0f, -1026.0f);
        o[1] = h2_fma(lop_magic<0x000C000Cu>(w, mg), 1.0f / 4, -258.0f);
        o[2] = h2_fma(lop_magic<0x00300030u>(w, mg), 1.0f / 16, -66.0f);
        o[3] = h2_fma(lop_magic<0x00C000C0u>(w, mg), 1.0f / 64, -18.0f);
        o[4] = h2_fma(lop_magic<0x03000300u>(w, mg), 1.0f / 256, -6.0f);
        o[5] = h2_fma(lop_magic<0x00030003u>(w10, mg), 1.0f, -1026.0f);
        o[6] = h2_fma(lop_magic<0x000C000Cu>(w10, mg), 1.0f / 4, -258.0f);
        o[7] = h2_fma(lop_magic<0x00300030u>(w10, mg), 1.0f / 16, -66.0f);
    } else if constexpr (BITS == 3) {
        const uint32_t A = *reinterpret_cast<const uint32_t*>(row + 4 * t);
        const uint32_t B = *reinterpret_cast<const uint16_t*>(row + 16 + 2 * t);
        const uint32_t A8 = A >> 8;
        const uint32_t Bx = prmt(B, 0u, 0x4140u);  // (B.lo, 0, B.hi, 0)
        o[0] = h2_fma(lop_magic<0x00070007u>(A, mg), 1.0f, -1028.0f);
        o[1] = h2_fma(lop_magic<0x00380038u>(A, mg), 1.0f / 8, -132.0f);
        o[2] = h2_fma(lop_magic<0x00070007u>(A8, mg), 1.0f, -1028.0f);
        o[3] = h2_fma(lop_magic<0x00380038u>(A8, mg), 1.0f / 8, -132.0f);
        o[4] = h2_fma(lop_magic<0x00C000C0u>(A, mg) | ((Bx << 2) & 0x01000100u), 1.0f / 64, -20.0f);
        o[5] = h2_fma(lop_magic<0x00C000C0u>(A8, mg) | ((Bx << 1) & 0x01000100u), 1.0f / 64, -20.0f);
        o[6] = h2_fma(lop_magic<0x00070007u>(Bx, mg), 1.0f, -1028.0f);
        o[7] = h2_fma(lop_magic<0x00380038u>(Bx, mg), 1.0f / 8, -132.0f);
    } else {  // 8
        const uint4 w = *reinterpret_cast<const uint4*>(row + 16 * t);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            o[2 * q] = h2_fma(prmt(ws[q], 0x64646464u, 0x4140u), 1.0f, -1152.0f);
            o[2 * q + 1] = h2_fma(prmt(ws[q], 0x64646464u, 0x4342u), 1.0f, -1152.0f);
        }
    }
}

}  // namespace moqe_gpu

namespace moqe_gpu {

// Log-scale codes (quant.cpp:18-27, :226-243): a field u = code + 2^(b-1) holds the sign in its
// top bit and k = u & (2^(b-1) - 1); the weight is +-s * 2^-k. Two fields x (one per 16-bit
// half, already shifted down to bit 0) become the exact fp16 pair (+-2^-k) as
// (sign << 15) | ((15 - k) << 10); the per-channel s is applied in the epilogue like the
// linear scale. b <= 4 (k <= 7: normal fp16).
template <int BITS>
__device__ __forceinline__ uint32_t log_pair(uint32_t x) {
    constexpr uint32_t kmask = ((1u << (BITS - 1)) - 1u) * 0x00010001u;
    const uint32_t sgn = (x >> (BITS - 1)) & 0x00010001u;
    return (sgn << 15) | ((0x000F000Fu - (x & kmask)) << 10);
}

// Unpack chunk t of a tile row of log codes into 8 fp16 pairs (same field positions as
// unpack_chunk; each field is shifted down by its position s before the exponent build).
template <int BITS>
__device__ __forceinline__ void unpack_chunk_log(const uint8_t* row, int t, uint32_t (&o)[8]) {
    if constexpr (BITS == 4) {
        const uint2 w = *reinterpret_cast<const uint2*>(row + 8 * t);
        const uint32_t ws[2] = {w.x, w.y};
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const uint32_t a = ws[q], a8 = ws[q] >> 8;
            o[4 * q + 0] = log_pair<4>(a & 0x000F000Fu);
            o[4 * q + 1] = log_pair<4>((a >> 4) & 0x000F000Fu);
            o[4 * q + 2] = log_pair<4>(a8 & 0x000F000Fu);
            o[4 * q + 3] = log_pair<4>((a8 >> 4) & 0x000F000Fu);
        }
    } else if constexpr (BITS == 2) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(row + 4 * t);
        const uint32_t w10 = w >> 10;
        o[0] = log_pair<2>(w & 0x00030003u);
        o[1] = log_pair<2>((w >> 2) & 0x00030003u);
        o[2] = log_pair<2>((w >> 4) & 0x00030003u);
        o[3] = log_pair<2>((w >> 6) & 0x00030003u);
        o[4] = log_pair<2>((w >> 8) & 0x00030003u);
        o[5] = log_pair<2>(w10 & 0x00030003u);
        o[6] = log_pair<2>((w10 >> 2) & 0x00030003u);
        o[7] = log_pair<2>((w10 >> 4) & 0x00030003u);
    } else if constexpr (BITS == 3) {
        const uint32_t A = *reinterpret_cast<const uint32_t*>(row + 4 * t);
        const uint32_t B = *reinterpret_cast<const uint16_t*>(row + 16 + 2 * t);
        const uint32_t A8 = A >> 8;
        const uint32_t Bx = prmt(B, 0u, 0x4140u);  // (B.lo, 0, B.hi, 0)
        o[0] = log_pair<3>(A & 0x00070007u);
        o[1] = log_pair<3>((A >> 3) & 0x00070007u);
        o[2] = log_pair<3>(A8 & 0x00070007u);
        o[3] = log_pair<3>((A8 >> 3) & 0x00070007u);
        o[4] = log_pair<3>(((A >> 6) & 0x00030003u) | ((Bx >> 4) & 0x00040004u));
        o[5] = log_pair<3>(((A8 >> 6) & 0x00030003u) | ((Bx >> 5) & 0x00040004u));
        o[6] = log_pair<3>(Bx & 0x00070007u);
        o[7] = log_pair<3>((Bx >> 3) & 0x00070007u);
    } else {
        for (int i = 0; i < 8; ++i) o[i] = 0u;  // log8 is not a GPU scheme (k up to 127)
    }
}

}  // namespace moqe_gpu
