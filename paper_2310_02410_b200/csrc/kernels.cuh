// kernels.cuh — launch interfaces shared by the kernel translation units and capi.cu.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "plan.cuh"

namespace moqe_gpu {

struct RouteArgs {
    const void* h;
    int h_f16;
    int64_t T;
    int d;
    const float* wg;
    int E;
    int topk;
    int path;            // 0 auto, 1 gemv-all, 2 gemm-all
    int inline_scatter;  // plan CTA also scatters metadata (small T, GEMV only)
    int gemm_bn;         // GEMM n-tile rows, for tile counting
    float* zero_out;     // top-2 fp32 accumulation rows to zero (inline scatter), or null
};
cudaError_t launch_route(const RouteArgs& a, const Plan& P, cudaStream_t st);
int route_tokens_per_cta(int64_t T);
// rows already routed: plan with kRouteSelWarps rows per CTA (scatter must use that tile)
cudaError_t launch_plan_from_ids(const RouteArgs& a, const Plan& P, cudaStream_t st);
constexpr int kPlanIdsTile = 32;
cudaError_t launch_scatter(const void* h, int h_f16, int64_t T, int d, int topk, int E, int path, int tt,
                           const Plan& P, __half* x_perm, int ldx, float* zero_out, cudaStream_t st);

moqe_status retile(const uint8_t* src, int64_t K, int64_t N, int bits, int n_mats, uint8_t* dst,
                   int64_t Kp, int64_t Np, cudaStream_t st);

struct GemvArgs {
    const void* h;
    int h_f16;
    int64_t T;
    int d, f, topk, E;
    const uint8_t* w1;
    const uint8_t* w2;
    int64_t w1_stride, w2_stride;  // bytes per expert (tiled)
    const float* s1;               // [E][Np1]
    const float* s2;               // [E][Np2]
    const float* b1;               // [E][Np1] or null
    const float* b2;               // [E][Np2] or null
    int Kp1, Np1, Kp2, Np2;
    __half* mid;                   // [R][Np1]
    void* out;                     // [T][d] (top-1 direct store)
    int out_f16;
    float* out_acc;                // [T][d] fp32 (top-2 accumulation) or null
    float* partial;                // split-K partials: phase1 [S1][R][Np1], phase2 [S2][R][Np2]
    int64_t part_rows;             // R capacity
    unsigned* split_cnt;           // [2][E][max(Nmt)]
};
cudaError_t launch_gemv(int bits, bool two_m16, const GemvArgs& g, const Plan& P, cudaStream_t st,
                        int num_sms);
int64_t gemv_partial_floats(int64_t rows, int Kp1, int Np1, int Kp2, int Np2);

struct GemmArgs {
    const __half* x_perm;  // [R][Kp1] expert-grouped activations
    __half* mid;           // [R][Np1]
    const uint8_t* w1;
    const uint8_t* w2;
    int64_t w1_stride, w2_stride;
    const float* s1;
    const float* s2;
    const float* b1;
    const float* b2;
    int Kp1, Np1, Kp2, Np2;
    int64_t R;             // rows capacity of x_perm / mid
    int d;
    void* out;
    int out_f16;
    float* out_acc;
};
bool gemm_available();
int gemm_block_n();
cudaError_t launch_gemm(int bits, int phase, const GemmArgs& g, const Plan& P, cudaStream_t st, int num_sms);

}  // namespace moqe_gpu
