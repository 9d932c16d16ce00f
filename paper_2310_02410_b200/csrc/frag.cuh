// frag.cuh — IMMA fragment recipes of the decode GEMV (shared with probes).
//
// The bank codec (codec.cuh) keeps every packed field byte-aligned at the same
// offset in each byte, so one LOP3 with a byte-lane mask turns a packed word
// into four u8 codes u * 2^s that feed mma.sync m16n8k32 (u8 x s8 -> s32)
// directly as A operands.
#pragma once
#include <stdint.h>

#include "ptx.cuh"

namespace moqe_gpu {

// ---- per-width fragment recipes ---------------------------------------------------
// For each stage (tiles T0, T1 = 128 k of 16 rows per warp) a lane builds F
// A-fragments. Fragment f accumulates into group grp(f); groups differ by the
// power of two the LOP3 left on the codes, undone by mult(g)/D at the end.
// kidx(f, h, i) names the activation (tile*16 + code within the lane's 16-code
// chunk) that meets byte i of A register a0/a1 (h = 0) or a2/a3 (h = 1).
template <int BITS>
struct Frag;

template <>
struct Frag<2> {
    static constexpr int F = 4, G = 4, D = 64;
    __host__ __device__ static constexpr int grp(int f) { return f; }
    __host__ __device__ static constexpr int mult(int g) { return 64 >> (2 * g); }
    __host__ __device__ static constexpr int kidx(int f, int h, int i) {
        return 16 * h + (i == 0 ? 2 * f : i == 1 ? 8 + 2 * f : i == 2 ? 2 * f + 1 : 9 + 2 * f);
    }
    __device__ static __forceinline__ void load(const uint8_t* T0, const uint8_t* T1, int r0, int tq,
                                                uint32_t (&a)[F][4]) {
        const uint32_t w00 = *reinterpret_cast<const uint32_t*>(T0 + r0 * 16 + 4 * tq);
        const uint32_t w01 = *reinterpret_cast<const uint32_t*>(T0 + (r0 + 8) * 16 + 4 * tq);
        const uint32_t w10 = *reinterpret_cast<const uint32_t*>(T1 + r0 * 16 + 4 * tq);
        const uint32_t w11 = *reinterpret_cast<const uint32_t*>(T1 + (r0 + 8) * 16 + 4 * tq);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t M = 0x03030303u << (2 * j);
            a[j][0] = w00 & M; a[j][1] = w01 & M; a[j][2] = w10 & M; a[j][3] = w11 & M;
        }
    }
};

template <>
struct Frag<3> {
    static constexpr int F = 5, G = 5, D = 64;  // f0 and f3 share a scale but not an accumulator (no IMMA chain)
    __host__ __device__ static constexpr int grp(int f) { return f; }
    __host__ __device__ static constexpr int mult(int g) { return g == 0 || g == 3 ? 64 : g == 1 ? 8 : g == 2 ? 1 : 4; }
    __host__ __device__ static constexpr int kidx(int f, int h, int i) {
        return f == 0 ? 16 * h + (i == 0 ? 0 : i == 1 ? 4 : i == 2 ? 1 : 5)
             : f == 1 ? 16 * h + (i == 0 ? 2 : i == 1 ? 6 : i == 2 ? 3 : 7)
             : f == 2 ? 16 * h + (i == 0 ? 8 : i == 1 ? 10 : i == 2 ? 9 : 11)
             : f == 3 ? 16 * (i >> 1) + 12 + 2 * h + (i & 1)
                      : 16 * (i >> 1) + 8 + 2 * h + (i & 1);
    }
    __device__ static __forceinline__ void load(const uint8_t* T0, const uint8_t* T1, int r0, int tq,
                                                uint32_t (&a)[F][4]) {
        const int o0 = r0 * 24, o1 = (r0 + 8) * 24;
        const uint32_t A00 = *reinterpret_cast<const uint32_t*>(T0 + o0 + 4 * tq);
        const uint32_t A01 = *reinterpret_cast<const uint32_t*>(T0 + o1 + 4 * tq);
        const uint32_t A10 = *reinterpret_cast<const uint32_t*>(T1 + o0 + 4 * tq);
        const uint32_t A11 = *reinterpret_cast<const uint32_t*>(T1 + o1 + 4 * tq);
        const uint32_t B00 = *reinterpret_cast<const uint16_t*>(T0 + o0 + 16 + 2 * tq);
        const uint32_t B01 = *reinterpret_cast<const uint16_t*>(T0 + o1 + 16 + 2 * tq);
        const uint32_t B10 = *reinterpret_cast<const uint16_t*>(T1 + o0 + 16 + 2 * tq);
        const uint32_t B11 = *reinterpret_cast<const uint16_t*>(T1 + o1 + 16 + 2 * tq);
        const uint32_t Bc0 = prmt(B00, B10, 0x5410u), Bc1 = prmt(B01, B11, 0x5410u);
        a[0][0] = A00 & 0x07070707u; a[0][1] = A01 & 0x07070707u; a[0][2] = A10 & 0x07070707u; a[0][3] = A11 & 0x07070707u;
        a[1][0] = A00 & 0x38383838u; a[1][1] = A01 & 0x38383838u; a[1][2] = A10 & 0x38383838u; a[1][3] = A11 & 0x38383838u;
        a[2][0] = A00 & 0xC0C0C0C0u; a[2][1] = A01 & 0xC0C0C0C0u; a[2][2] = A10 & 0xC0C0C0C0u; a[2][3] = A11 & 0xC0C0C0C0u;
        a[3][0] = Bc0 & 0x07070707u; a[3][1] = Bc1 & 0x07070707u;
        a[3][2] = (Bc0 >> 3) & 0x07070707u; a[3][3] = (Bc1 >> 3) & 0x07070707u;
        a[4][0] = Bc0 & 0x40404040u; a[4][1] = Bc1 & 0x40404040u;
        a[4][2] = (Bc0 >> 1) & 0x40404040u; a[4][3] = (Bc1 >> 1) & 0x40404040u;
    }
};

template <>
struct Frag<4> {
    static constexpr int F = 4, G = 2, D = 16;
    __host__ __device__ static constexpr int grp(int f) { return f & 1; }
    __host__ __device__ static constexpr int mult(int g) { return g == 0 ? 16 : 1; }
    __host__ __device__ static constexpr int kidx(int f, int h, int i) {
        return 16 * (f >> 1) + 8 * h + 2 * (f & 1) + (i == 0 ? 0 : i == 1 ? 4 : i == 2 ? 1 : 5);
    }
    __device__ static __forceinline__ void load(const uint8_t* T0, const uint8_t* T1, int r0, int tq,
                                                uint32_t (&a)[F][4]) {
        const uint2 w00 = *reinterpret_cast<const uint2*>(T0 + r0 * 32 + 8 * tq);
        const uint2 w01 = *reinterpret_cast<const uint2*>(T0 + (r0 + 8) * 32 + 8 * tq);
        const uint2 w10 = *reinterpret_cast<const uint2*>(T1 + r0 * 32 + 8 * tq);
        const uint2 w11 = *reinterpret_cast<const uint2*>(T1 + (r0 + 8) * 32 + 8 * tq);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const uint32_t M = g ? 0xF0F0F0F0u : 0x0F0F0F0Fu;
            a[g][0] = w00.x & M; a[g][1] = w01.x & M; a[g][2] = w00.y & M; a[g][3] = w01.y & M;
            a[2 + g][0] = w10.x & M; a[2 + g][1] = w11.x & M; a[2 + g][2] = w10.y & M; a[2 + g][3] = w11.y & M;
        }
    }
};

template <>
struct Frag<8> {
    static constexpr int F = 4, G = 1, D = 1;
    __host__ __device__ static constexpr int grp(int) { return 0; }
    __host__ __device__ static constexpr int mult(int) { return 1; }
    __host__ __device__ static constexpr int kidx(int f, int h, int i) { return 16 * (f >> 1) + 8 * (f & 1) + 4 * h + i; }
    __device__ static __forceinline__ void load(const uint8_t* T0, const uint8_t* T1, int r0, int tq,
                                                uint32_t (&a)[F][4]) {
        const uint4 w00 = *reinterpret_cast<const uint4*>(T0 + r0 * 64 + 16 * tq);
        const uint4 w01 = *reinterpret_cast<const uint4*>(T0 + (r0 + 8) * 64 + 16 * tq);
        const uint4 w10 = *reinterpret_cast<const uint4*>(T1 + r0 * 64 + 16 * tq);
        const uint4 w11 = *reinterpret_cast<const uint4*>(T1 + (r0 + 8) * 64 + 16 * tq);
        a[0][0] = w00.x; a[0][1] = w01.x; a[0][2] = w00.y; a[0][3] = w01.y;
        a[1][0] = w00.z; a[1][1] = w01.z; a[1][2] = w00.w; a[1][3] = w01.w;
        a[2][0] = w10.x; a[2][1] = w11.x; a[2][2] = w10.y; a[2][3] = w11.y;
        a[3][0] = w10.z; a[3][1] = w11.z; a[3][2] = w10.w; a[3][3] = w11.w;
    }
};

__device__ __forceinline__ void imma(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

}  // namespace moqe_gpu
