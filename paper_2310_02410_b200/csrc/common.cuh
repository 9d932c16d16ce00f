// common.cuh — shared device/host helpers for the MoQE B200 path (sm_100a only).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/moqe_gpu.h"

namespace moqe_gpu {

// ---- error plumbing ------------------------------------------------------
void set_error(const std::string& msg);
moqe_status fail(moqe_status st, const std::string& msg);
moqe_status cuda_fail(cudaError_t err, const char* what);

#define MOQE_CUDA(expr)                                              \
    do {                                                             \
        cudaError_t e__ = (expr);                                    \
        if (e__ != cudaSuccess) return ::moqe_gpu::cuda_fail(e__, #expr); \
    } while (0)

#define MOQE_CHECK_LAUNCH(what)                                      \
    do {                                                             \
        cudaError_t e__ = cudaGetLastError();                        \
        if (e__ != cudaSuccess) return ::moqe_gpu::cuda_fail(e__, what); \
    } while (0)

constexpr int kMaxDevices = 64;  // per-process launch caches are indexed by device ordinal

inline bool valid_bits(int b) { return b == 2 || b == 3 || b == 4 || b == 8; }

// bitpack.cpp:12-16
__host__ __device__ inline int64_t packed_size(int bits, int64_t count) {
    return bits == 3 ? 3 * ((count + 7) / 8) : (count * bits + 7) / 8;
}

// ---- device weight-tile layout ---------------------------------------------
// A quantized matrix W [K x N] (N = output channel) lives on the device as
// tiles of TILE_N output channels x TILE_K input rows. Tile (nt, kb) holds
// TILE_N "rows" (one per output channel n), each the TILE_K codes
// W[kb*64 + kk][n], kk = 0..63, packed exactly like the reference packs a flat
// code array (offset binary, LSB-first, 3-bit in 24-bit groups,
// bitpack.cpp:18-39). Row bytes = 8*bits; tile bytes = 1024*bits. Tiles are
// ordered nt-major so one output-channel tile streams contiguously over K.
constexpr int TILE_N = 128;
constexpr int TILE_K = 64;
__host__ __device__ constexpr int row_bytes(int bits) { return 8 * bits; }
__host__ __device__ constexpr int tile_bytes(int bits) { return TILE_N * 8 * bits; }
__host__ __device__ inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ---- binary16 ----------------------------------------------------------------
// Reference scale rounding: fp64 -> fp32 (RN) -> binary16 (RNE), tensor.cpp:38-72,
// quant.cpp:67. __float2half_rn is exactly the reference's f32_to_f16_bits on
// every finite float.
__device__ inline float f16_round(float x, bool* overflow) {
    __half h = __float2half_rn(x);
    unsigned short b = __half_as_ushort(h);
    *overflow = (b & 0x7FFFu) == 0x7C00u;
    return __half2float(h);
}

// ---- small PTX helpers -----------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

}  // namespace moqe_gpu
