// quant.cu — "quantize experts" on the GPU: per-channel abs-max scales,
// linear codes and reference-layout bit-packing, plus the device re-tiling
// used by the expert bank.
//
// Reference: linear_scales/quantize_linear proj/src/quant.cpp:38-95,
// pack/unpack proj/src/bitpack.cpp:18-68, binary16 proj/src/tensor.cpp:38-106.
// All integer/byte outputs are bit-exact with the reference:
//  * column max |a| is exact (fabs + max are exact in any order);
//  * scale = f16_RNE(f32_RN(2.0*m/(2^b-1))) computed in fp64 like quant.cpp:67;
//  * code = clamp(rint(double(a)/double(s))) with IEEE fp64 division (the
//    reference's exact expression, quant.cpp:88); no reciprocal multiply.
// HBM-bound streaming kernels: each thread owns one 8-code group (one packed
// unit of b bytes, 3 bytes for int3), so loads are 2x float4 and stores are a
// single 2/4/8-byte word.
#include <cuda_fp16.h>

#include "common.cuh"
#include "codec.cuh"

namespace moqe_gpu {

namespace {

constexpr int kFlagNonFinite = 1;
constexpr int kFlagRange = 2;
constexpr int kFlagOutOfRange = 4;

// ---- column abs-max (+ finiteness) -------------------------------------------------
// grid: (ceil(cols/32), batch), block (32, 16). Each block reduces 32 columns
// over all rows of one matrix.
__global__ void k_colmax(const float* __restrict__ a, int64_t rows, int64_t cols,
                         float* __restrict__ colmax, int* __restrict__ flag) {
    const int64_t b = blockIdx.y;
    const int64_t j = int64_t(blockIdx.x) * 32 + threadIdx.x;
    const float* m = a + b * rows * cols;
    float mx = 0.0f;
    bool bad = false;
    if (j < cols) {
        for (int64_t i = threadIdx.y; i < rows; i += blockDim.y) {
            const float v = __ldg(m + i * cols + j);
            bad |= !isfinite(v);
            mx = fmaxf(mx, fabsf(v));
        }
    }
    __shared__ float red[16][33];
    red[threadIdx.y][threadIdx.x] = mx;
    if (__syncthreads_or(bad) && threadIdx.x == 0 && threadIdx.y == 0) atomicOr(flag, kFlagNonFinite);
    if (threadIdx.y == 0 && j < cols) {
        float r = red[0][threadIdx.x];
        for (int y = 1; y < blockDim.y; ++y) r = fmaxf(r, red[y][threadIdx.x]);
        colmax[b * cols + j] = r;
    }
}

// scales: one thread per output scale. Per-tensor reduces the matrix's column
// maxima inside one block (grid.x == 1 for per-tensor).
__global__ void k_scales(const float* __restrict__ colmax, int64_t cols, int bits, int per_tensor,
                         float* __restrict__ scales, int* __restrict__ flag) {
    const int64_t b = blockIdx.y;
    const double denom = double((1 << bits) - 1);
    if (per_tensor) {
        __shared__ float red[256];
        float mx = 0.0f;
        for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) mx = fmaxf(mx, colmax[b * cols + j]);
        red[threadIdx.x] = mx;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + s]);
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const double m = red[0];
            bool ovf = false;
            float s = m == 0.0 ? 0.0f : f16_round(__double2float_rn(2.0 * m / denom), &ovf);
            if (ovf) atomicOr(flag, kFlagRange);
            scales[b] = s;
        }
        return;
    }
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    const double m = colmax[b * cols + j];
    bool ovf = false;
    const float s = m == 0.0 ? 0.0f : f16_round(__double2float_rn(2.0 * m / denom), &ovf);
    if (ovf) atomicOr(flag, kFlagRange);
    scales[b * cols + j] = s;
}

__device__ __forceinline__ int quant_code(float a, float s, int bits) {
    if (s == 0.0f) return 0;
    double q = rint(__ddiv_rn(double(a), double(s)));
    const double lo = -double(1 << (bits - 1)), hi = double((1 << (bits - 1)) - 1);
    q = fmin(fmax(q, lo), hi);
    return int(q);
}

// Bit offset of code i inside its 8-code group (3-bit: 24-bit group).
// Packing an 8-code group into one little-endian word of b bytes.
__device__ __forceinline__ uint64_t pack_group(const int* q, int bits) {
    const int bias = 1 << (bits - 1);
    uint64_t w = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) w |= uint64_t(uint32_t(q[i] + bias) & ((1u << bits) - 1u)) << (i * bits);
    return w;
}

__device__ __forceinline__ void store_group(uint8_t* out, int64_t g, uint64_t w, int bits,
                                            int64_t nbytes_total, bool aligned) {
    const int64_t off = g * bits;  // each 8-code group is exactly `bits` bytes
    if (aligned && off + bits <= nbytes_total) {
        if (bits == 8) { *reinterpret_cast<uint64_t*>(out + off) = w; return; }
        if (bits == 4) { *reinterpret_cast<uint32_t*>(out + off) = uint32_t(w); return; }
        if (bits == 2) { *reinterpret_cast<uint16_t*>(out + off) = uint16_t(w); return; }
    }
    for (int i = 0; i < bits; ++i)
        if (off + i < nbytes_total) out[off + i] = uint8_t(w >> (8 * i));
}

// quantize (+pack): one thread per 8-code group of the flat [rows x cols] array.
__global__ void k_quant_pack(const float* __restrict__ a, int64_t rows, int64_t cols, int bits,
                             int per_tensor, const float* __restrict__ scales,
                             uint8_t* __restrict__ packed, int8_t* __restrict__ codes,
                             int64_t n_groups_per_mat, int64_t batch) {
    const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= n_groups_per_mat * batch) return;
    const int64_t b = gid / n_groups_per_mat, g = gid % n_groups_per_mat;
    const int64_t n = rows * cols;
    const float* m = a + b * n;
    const float* sc = scales + (per_tensor ? b : b * cols);
    const int64_t i0 = g * 8;
    int q[8];
    const bool vec = (cols % 8 == 0) && (n % 4 == 0) && i0 + 8 <= n &&
                     ((reinterpret_cast<uintptr_t>(m) & 15) == 0);
    if (vec) {
        const float4 v0 = __ldg(reinterpret_cast<const float4*>(m + i0));
        const float4 v1 = __ldg(reinterpret_cast<const float4*>(m + i0 + 4));
        const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        const int64_t j0 = i0 % cols;  // group never straddles a row (cols % 8 == 0)
#pragma unroll
        for (int i = 0; i < 8; ++i) q[i] = quant_code(v[i], per_tensor ? sc[0] : sc[j0 + i], bits);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int64_t idx = i0 + i;
            q[i] = idx < n ? quant_code(m[idx], per_tensor ? sc[0] : sc[idx % cols], bits) : 0;
        }
    }
    if (codes) {
        int8_t* c = codes + b * n;
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i0 + i < n) c[i0 + i] = int8_t(q[i]);
    }
    if (packed) {
        // padding codes beyond n contribute zero bits (reference zero-fills).
        const int64_t psz = packed_size(bits, n);
        uint8_t* p = packed + b * psz;
        const int bias = 1 << (bits - 1);
        int qq[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) qq[i] = i0 + i < n ? q[i] : -bias;  // u = 0 padding
        const bool aligned = (psz % 8 == 0) && ((reinterpret_cast<uintptr_t>(p) & 7) == 0);
        store_group(p, g, pack_group(qq, bits), bits, psz, aligned);
    }
}

// pack(): codes -> bytes, one thread per 8-code group; out-of-range -> flag.
__global__ void k_pack(const int8_t* __restrict__ codes, int64_t count, int bits,
                       uint8_t* __restrict__ out, int* __restrict__ flag) {
    const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t ng = (count + 7) / 8;
    if (g >= ng) return;
    const int lo = -(1 << (bits - 1)), hi = (1 << (bits - 1)) - 1;
    int q[8];
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t idx = g * 8 + i;
        q[i] = idx < count ? int(codes[idx]) : lo;
        bad |= q[i] < lo || q[i] > hi;
    }
    if (bad) { atomicOr(flag, kFlagOutOfRange); return; }
    store_group(out, g, pack_group(q, bits), bits, packed_size(bits, count), false);
}

__device__ __forceinline__ int extract_code(const uint8_t* __restrict__ data, int64_t i, int bits) {
    const int64_t p = bits == 3 ? (i / 8) * 24 + (i % 8) * 3 : i * bits;
    const unsigned sh = unsigned(p & 7);
    uint32_t u = uint32_t(data[p >> 3]) >> sh;
    if (sh + unsigned(bits) > 8u) u |= uint32_t(data[(p >> 3) + 1]) << (8u - sh);
    return int(u & ((1u << bits) - 1u)) - (1 << (bits - 1));
}

__global__ void k_unpack(const uint8_t* __restrict__ data, int64_t count, int bits,
                         int8_t* __restrict__ codes) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < count) codes[i] = int8_t(extract_code(data, i, bits));
}

}  // namespace

// ---- re-tiling: reference-packed [K x N] -> device tiles (common.cuh layout) ----
// One thread per (expert, tile row n, k-block): gathers the 64 codes
// W[kb*64+kk][n] from the flat packed array and re-packs them as one row.
__global__ void k_retile(const uint8_t* __restrict__ src, int64_t K, int64_t N, int bits,
                         int64_t src_stride, uint8_t* __restrict__ dst, int64_t dst_stride,
                         int64_t Kp, int64_t Np, int n_mats) {
    const int64_t kbs = Kp / TILE_K;
    const int64_t per_mat = Np * kbs;
    const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= per_mat * n_mats) return;
    const int64_t m = gid / per_mat, r = gid % per_mat;
    const int64_t n = r / kbs, kb = r % kbs;  // n-major: consecutive threads walk k-blocks
    const uint8_t* s = src + m * src_stride;
    int q[TILE_K];
#pragma unroll 8
    for (int kk = 0; kk < TILE_K; ++kk) {
        const int64_t k = kb * TILE_K + kk;
        q[kk] = (k < K && n < N) ? extract_code(s, k * N + n, bits) : 0;
    }
    // row (n, kb) lives in tile (n/128, kb) at row n%128, re-encoded (codec.cuh)
    const int64_t tile = (n / TILE_N) * kbs + kb;
    uint8_t* row = dst + m * dst_stride + tile * tile_bytes(bits) + (n % TILE_N) * row_bytes(bits);
    switch (bits) {
        case 2: encode_row<2>(q, row); break;
        case 3: encode_row<3>(q, row); break;
        case 4: encode_row<4>(q, row); break;
        default: encode_row<8>(q, row); break;
    }
}

namespace {

struct FlagBuf {
    int* d = nullptr;
    ~FlagBuf() { if (d) cudaFree(d); }
};

moqe_status read_flag(int* dflag, cudaStream_t st, int* out) {
    MOQE_CUDA(cudaMemcpyAsync(out, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
    MOQE_CUDA(cudaStreamSynchronize(st));
    return MOQE_OK;
}

moqe_status flag_status(int f) {
    if (f & kFlagNonFinite) return fail(MOQE_INVALID_ARGUMENT, "quant: non-finite values");
    if (f & kFlagRange)
        return fail(MOQE_RANGE_ERROR, "round_to_binary16: overflow above binary16 max 65504");
    if (f & kFlagOutOfRange) return fail(MOQE_OUT_OF_RANGE, "bitpack: code out of range");
    return MOQE_OK;
}

moqe_status run_quant(const float* a, int64_t batch, int64_t rows, int64_t cols, int bits,
                      moqe_granularity g, float* scales, int8_t* codes, uint8_t* packed,
                      bool scales_only, cudaStream_t st) {
    if (!valid_bits(bits)) return fail(MOQE_INVALID_ARGUMENT, "quant: unsupported bit width");
    if (rows < 0 || cols < 0 || batch < 0) return fail(MOQE_INVALID_ARGUMENT, "quant: tensor must be 2D");
    if (g != MOQE_PER_CHANNEL && g != MOQE_PER_TENSOR)
        return fail(MOQE_INVALID_ARGUMENT, "quant: bad granularity");
    if (batch == 0 || rows * cols == 0) {
        // reference: zero-size matrices give all-zero scales
        if (scales && batch > 0) {
            const int64_t ns = g == MOQE_PER_TENSOR ? batch : batch * cols;
            if (ns) MOQE_CUDA(cudaMemsetAsync(scales, 0, ns * sizeof(float), st));
            MOQE_CUDA(cudaStreamSynchronize(st));
        }
        return MOQE_OK;
    }
    FlagBuf flag;
    float* colmax = nullptr;
    MOQE_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&flag.d), sizeof(int), st));
    MOQE_CUDA(cudaMemsetAsync(flag.d, 0, sizeof(int), st));
    MOQE_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&colmax), batch * cols * sizeof(float), st));
    k_colmax<<<dim3(unsigned((cols + 31) / 32), unsigned(batch)), dim3(32, 16), 0, st>>>(
        a, rows, cols, colmax, flag.d);
    MOQE_CHECK_LAUNCH("k_colmax");
    if (g == MOQE_PER_TENSOR)
        k_scales<<<dim3(1, unsigned(batch)), 256, 0, st>>>(colmax, cols, bits, 1, scales, flag.d);
    else
        k_scales<<<dim3(unsigned((cols + 255) / 256), unsigned(batch)), 256, 0, st>>>(
            colmax, cols, bits, 0, scales, flag.d);
    MOQE_CHECK_LAUNCH("k_scales");
    int f = 0;
    moqe_status s = read_flag(flag.d, st, &f);
    cudaFreeAsync(colmax, st);
    if (s != MOQE_OK) return s;
    if ((s = flag_status(f)) != MOQE_OK) return s;
    if (scales_only) return MOQE_OK;
    const int64_t ng = (rows * cols + 7) / 8;
    const int64_t total = ng * batch;
    k_quant_pack<<<unsigned((total + 255) / 256), 256, 0, st>>>(
        a, rows, cols, bits, g == MOQE_PER_TENSOR, scales, packed, codes, ng, batch);
    MOQE_CHECK_LAUNCH("k_quant_pack");
    MOQE_CUDA(cudaStreamSynchronize(st));
    return MOQE_OK;
}

}  // namespace

moqe_status retile(const uint8_t* src, int64_t K, int64_t N, int bits, int n_mats, uint8_t* dst,
                   int64_t Kp, int64_t Np, cudaStream_t st) {
    const int64_t src_stride = packed_size(bits, K * N);
    const int64_t dst_stride = (Np / TILE_N) * (Kp / TILE_K) * tile_bytes(bits);
    const int64_t total = Np * (Kp / TILE_K) * n_mats;
    k_retile<<<unsigned((total + 127) / 128), 128, 0, st>>>(src, K, N, bits, src_stride, dst,
                                                            dst_stride, Kp, Np, n_mats);
    MOQE_CHECK_LAUNCH("k_retile");
    return MOQE_OK;
}

}  // namespace moqe_gpu

using namespace moqe_gpu;

extern "C" {

size_t moqe_gpu_packed_size(int bits, size_t count) {
    if (!valid_bits(bits)) {
        set_error("bitpack: unsupported width " + std::to_string(bits));
        return size_t(-1);
    }
    return size_t(packed_size(bits, int64_t(count)));
}

moqe_status moqe_gpu_pack(const int8_t* codes, int64_t count, int bits, uint8_t* out,
                          void* stream) {
    if (!valid_bits(bits)) return fail(MOQE_INVALID_ARGUMENT, "bitpack: unsupported width " + std::to_string(bits));
    if (count < 0) return fail(MOQE_INVALID_ARGUMENT, "bitpack: negative count");
    if (count == 0) return MOQE_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FlagBuf flag;
    MOQE_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&flag.d), sizeof(int), st));
    MOQE_CUDA(cudaMemsetAsync(flag.d, 0, sizeof(int), st));
    const int64_t ng = (count + 7) / 8;
    k_pack<<<unsigned((ng + 255) / 256), 256, 0, st>>>(codes, count, bits, out, flag.d);
    MOQE_CHECK_LAUNCH("k_pack");
    int f = 0;
    moqe_status s = read_flag(flag.d, st, &f);
    if (s != MOQE_OK) return s;
    return flag_status(f);
}

moqe_status moqe_gpu_unpack(const uint8_t* data, int64_t len, int bits, int64_t count,
                            int8_t* codes, void* stream) {
    if (!valid_bits(bits)) return fail(MOQE_INVALID_ARGUMENT, "bitpack: unsupported width " + std::to_string(bits));
    if (count < 0 || len != packed_size(bits, count))
        return fail(MOQE_INVALID_ARGUMENT, "bitpack: data length " + std::to_string(len) +
                                               " does not match " + std::to_string(count) +
                                               " codes at " + std::to_string(bits) + " bits");
    if (count == 0) return MOQE_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    k_unpack<<<unsigned((count + 255) / 256), 256, 0, st>>>(data, count, bits, codes);
    MOQE_CHECK_LAUNCH("k_unpack");
    return MOQE_OK;
}

moqe_status moqe_gpu_linear_scales(const float* a, int64_t batch, int64_t rows, int64_t cols,
                                   int bits, moqe_granularity g, float* scales, void* stream) {
    return run_quant(a, batch, rows, cols, bits, g, scales, nullptr, nullptr, true,
                     static_cast<cudaStream_t>(stream));
}

moqe_status moqe_gpu_quantize_linear(const float* a, int64_t batch, int64_t rows, int64_t cols,
                                     int bits, moqe_granularity g, int8_t* codes, float* scales,
                                     void* stream) {
    return run_quant(a, batch, rows, cols, bits, g, scales, codes, nullptr, false,
                     static_cast<cudaStream_t>(stream));
}

moqe_status moqe_gpu_quantize_pack(const float* a, int64_t batch, int64_t rows, int64_t cols,
                                   int bits, moqe_granularity g, uint8_t* packed, float* scales,
                                   int8_t* codes, void* stream) {
    return run_quant(a, batch, rows, cols, bits, g, scales, codes, packed, false,
                     static_cast<cudaStream_t>(stream));
}

}  // extern "C"
