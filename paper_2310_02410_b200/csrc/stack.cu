// stack.cu — the pre-LN residual FFN stack around the MoE layer (BASELINE config 3;
// SURVEY.md §8 f1): x <- x + delta; out = layer_norm(x) per row (eps 1e-5, double statistics).
//
// Reference: run_stack (proj/src/model.cpp:419-435) minus attention: per layer
// fn = layer_norm(x, ln_ffn) (model.cpp:193-212), x += ffn_block(fn) (add_inplace,
// model.cpp:308-310), then the final layer_norm. One CTA per row: the residual add is fused
// into the normalisation that follows it, so the residual stream is read and written once.
#include <cuda_fp16.h>

#include "kernels.cuh"

namespace moqe_gpu {

namespace {
constexpr int kLnThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (w == 0) {
        s = l < kLnThreads / 32 ? red[l] : 0.0;
#pragma unroll
        for (int o = 4; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (l == 0) red[8] = s;
    }
    __syncthreads();
    s = red[8];
    __syncthreads();
    return s;
}
}  // namespace

// x [rows][n] f32 (updated in place when delta != null: x += delta, fp32 like add_inplace),
// out [rows][n] f32 or f16: float((x - mean) * inv * gain + bias) computed in double.
__global__ void __launch_bounds__(kLnThreads) k_add_layer_norm(float* __restrict__ x, const float* __restrict__ delta,
                                                               int64_t n, const float* __restrict__ gain,
                                                               const float* __restrict__ bias, void* out, int out_f16) {
    __shared__ double red[9];
    const int64_t row = blockIdx.x;
    float* xr = x + row * n;
    const float* dr = delta ? delta + row * n : nullptr;
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += kLnThreads) {
        float v = xr[j];
        if (dr) {
            v = v + dr[j];
            xr[j] = v;
        }
        s += double(v);
    }
    const double mean = block_sum(s, red) / double(n);
    double q = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += kLnThreads) {
        const double dv = double(xr[j]) - mean;
        q += dv * dv;
    }
    const double var = block_sum(q, red) / double(n);
    const double inv = 1.0 / sqrt(var + 1e-5);
    for (int64_t j = threadIdx.x; j < n; j += kLnThreads) {
        const float o = float((double(xr[j]) - mean) * inv * double(gain[j]) + double(bias[j]));
        if (out_f16) static_cast<__half*>(out)[row * n + j] = __float2half_rn(o);
        else static_cast<float*>(out)[row * n + j] = o;
    }
}

}  // namespace moqe_gpu

using namespace moqe_gpu;

extern "C" moqe_status moqe_gpu_add_layer_norm(float* x, const float* delta, int64_t rows, int64_t n,
                                               const float* gain, const float* bias, void* out,
                                               moqe_dtype out_dtype, void* stream) {
    if (rows < 0 || n <= 0) return fail(MOQE_INVALID_ARGUMENT, "layer_norm: bad shape");
    if (!x || !gain || !bias || !out) return fail(MOQE_INVALID_ARGUMENT, "layer_norm: null buffer");
    if (out_dtype != MOQE_F32 && out_dtype != MOQE_F16) return fail(MOQE_INVALID_ARGUMENT, "layer_norm: bad out dtype");
    if (rows == 0) return MOQE_OK;
    if (rows > 0x7fffffff) return fail(MOQE_INVALID_ARGUMENT, "layer_norm: too many rows");
    k_add_layer_norm<<<unsigned(rows), kLnThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        x, delta, n, gain, bias, out, out_dtype == MOQE_F16 ? 1 : 0);
    MOQE_CHECK_LAUNCH("k_add_layer_norm");
    return MOQE_OK;
}
