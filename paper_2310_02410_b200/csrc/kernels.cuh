// kernels.cuh — launch interfaces shared by the kernel translation units and capi.cu.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "common.cuh"
#include "plan.cuh"

namespace moqe_gpu {

// Launch with programmatic stream serialization: the grid may start while the
// preceding kernel in the stream drains; the kernel calls pdl_wait() before it
// reads that kernel's results.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

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
    unsigned long long* trace;  // router phase stamps [kTraceRouteCtas][16] or null (diagnostics)
    int pdl;                    // launched behind k_xrows: the decode router may start early (PDL)
    int no_plan;                // decode GEMV-only: write expert / gate only (the GEMV kernels plan themselves)
    int dbg;                    // diagnostics (env MOQE_ROUTE_DBG; 1 = skip the logit chain, timing only)
    const float* wg_blk;        // the bank's blocked copy of wg (route_block_wg) or null
    int wg_finite;              // wg has no inf / NaN
    // decode chain led by the router (k_route_chain only): it waits for the previous grid
    // itself, zeroes the GEMV readiness counters and writes the fc1 row blocks (no k_xrows)
    int first;
    uint8_t* xr;                // fc1 row blocks [T][nch1][xr bytes] or null
    int nch1, xr_bits;
    unsigned* ready;            // [kSelfPlanRows] or null
    // tensor-core prefill logits (k_route_mma): the bank's split gate weights
    // [4 K chunks][hi, lo][Ep][Kp1/4 + 8] fp16 = Wg * 2^wg_shift (finite Wg only), or null
    const __half* wgt;
    int wg_shift;
    int Kp1;
    int gemv_max;               // experts with <= this many rows are planned for the GEMV-class path (0: kGemvMaxRows)
};
bool route_chain_used(const RouteArgs& a);  // launch_route will run k_route_chain
constexpr int kTraceRouteCtas = 64;
// Router weights -> blocked transposed copy for the decode chain; *finite = no inf / NaN.
int64_t route_wg_block_floats(int d, int E);
cudaError_t route_block_wg(const float* wg, int d, int E, float* out, int* d_flag, int* finite);
cudaError_t launch_route(const RouteArgs& a, const Plan& P, cudaStream_t st);
bool route_chain_one_chunk(int d, int E);  // the decode chain router holds all of Wg in one chunk
int route_tokens_per_cta(int64_t T);
// rows already routed (top-1): plan with kPlanIdsTile rows per CTA (scatter must use that tile)
cudaError_t launch_plan_from_ids(const RouteArgs& a, const Plan& P, cudaStream_t st);
constexpr int kPlanIdsTile = 256;
cudaError_t launch_scatter(const void* h, int h_f16, int64_t T, int d, int topk, int E, int path, int gemv_max, int tt,
                           const Plan& P, __half* x_perm, int ldx, float* zero_out, cudaStream_t st);

moqe_status retile(const uint8_t* src, int64_t K, int64_t N, int bits, int n_mats, uint8_t* dst,
                   int64_t Kp, int64_t Np, cudaStream_t st);

// Decode path (ffn_gemv.cu): two persistent weight-streaming kernels chained
// with programmatic dependent launch — fc1 (expert rows -> ReLU -> fc2's
// fixed-point fragments in global memory) and fc2 (-> gate-weighted output).
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
    void* out;                     // [T][d] (top-1 direct store)
    int out_f16;
    float* out_acc;                // [T][d] fp32 (top-2 accumulation, 2 addends per element) or null
    const uint8_t* xr;             // fc1 row blocks [T][nch1][xr bytes] (k_xrows)
    int nch1;                      // 1024-k chunks of fc1
    uint8_t* xb;                   // fc2 row blocks [T*k][nch2][xb bytes] (written by the fc1 epilogue)
    const float* smax1;            // [E] max fc1 scale (bounds the fc2 fixed-point exponent)
    const float* bmax1;            // [E] max |fc1 bias|
    unsigned long long* trace;     // [grid][kTraceCap][2] (time ns, event) or null
    int dbg;                       // diagnostics (env MOQE_GEMV_DBG; 1 = consumers skip the MMA work)
    int self_plan;                 // plan built in each CTA from P.expert / P.gate (T*k <= kSelfPlanRows)
    unsigned* ready;               // [kSelfPlanRows] fc1 m-tiles done per pass (by first row), zeroed by
                                   // k_xrows; non-null selects the fused fc1+fc2 grid (self plan only)
};
constexpr int kSelfPlanRows = 64;
constexpr int kTraceCap = 512;
cudaError_t launch_gemv(int bits, const GemvArgs& g, const Plan& P, cudaStream_t st, int num_sms);
bool gemv_supported(int Kp1, int Kp2);
// Token rows -> fc1 row blocks (fixed-point digit planes in IMMA fragment order).
struct XrowArgs {
    const void* h;
    int h_f16;
    int64_t T;
    int d;
    int nch1;
    uint8_t* xr;
    unsigned* ready;  // [kSelfPlanRows] zeroed here for the fused decode grid, or null
};
cudaError_t launch_xrows(int bits, const XrowArgs& a, cudaStream_t st);
int64_t gemv_xr_bytes(int bits);  // one fc1 row block (per token and 1024-k chunk)
int64_t gemv_xb_bytes(int bits);  // one fc2 row block (per routed row and 1024-k chunk)
int gemv_chunks(int Kp);
cudaError_t launch_expert_max(const float* s1, const float* b1, int E, int Np1, float* smax, float* bmax,
                              cudaStream_t st);

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
    int log_codes;         // 1: log-scale bank (+-2^-k codes, unpack_chunk_log)
};
bool gemm_available();
int gemm_block_n();
cudaError_t launch_gemm(int bits, int phase, const GemmArgs& g, const Plan& P, cudaStream_t st, int num_sms);

// Decode path (dec.cu): k_dec_route (one cluster: parallel-order logits, top-k, plan,
// permuted fp16 rows) -> PDL -> k_dec<BITS> (stream-K over (unit, 64-channel f-slice)).
constexpr int kDecMaxRows = 64;   // T * top_k handled by the decode path
// Mid-size batches (T * k <= kDecMidMaxRows, top-1): after the batched router + scatter, the
// experts with few rows (<= the plan's GEMV-class limit) run on k_dec from a prepared plan
// (k_dec_prep: units of <= kDecMidUnitRows rows, scaled rows + Z); the rest on tcgen05.
constexpr int kDecMidMaxRows = 1024;
constexpr int kDecMidUnitRows = 8;
constexpr int kDecMidMaxUnits = kDecMidMaxRows / kDecMidUnitRows + 256;
constexpr int kDecTrace = 64;
constexpr int kDecUnitRows = 16;  // rows per unit (an expert with more rows has several units)
struct DecSpan {                  // in-kernel launch span: first CTA start (after PDL wait) -> last CTA exit
    unsigned long long start_min;
    unsigned ticket, pad;
    unsigned long long total_ns, count;
};
struct DecArgs {
    const void* h;
    int h_f16;
    int T, d;
    const float* wg;
    int E, topk, bits;
    int32_t* expert;       // [T*k] routing outputs
    float* gate;
    int4* units;           // [kDecMaxRows] {expert, first permuted row, rows, 0}
    int* n_units;
    int32_t* perm_token;   // [T*k] token of permuted row
    float* perm_gate;      // [T*k]
    int32_t* row_of;       // [T*k] permuted row of (token, slot)
    __half* xperm;         // [T*k][xpitch bytes] fp16 rows * 2^-field shift, zero padded to Kp1; float Z behind
    int xpitch;
    int Kp1, Np1, Np2, S;  // S = Np1 / 64 f-slices
    const uint8_t* wdec;   // decode bank layout (dec_build_layout)
    int64_t wdec_stride, slice_bytes;
    const float* s1;
    const float* b1;
    const float* s2;
    const float* b2;
    long long* acc;        // [T*k][Np2] fixed-point fc2 accumulators (zero between forwards)
    unsigned* unit_done;   // [kDecMaxRows] (zero between forwards)
    float* ybuf;           // [T*k][d] gated rows (top-2)
    unsigned* tok_cnt;     // [T] (top-2; zero between forwards)
    void* out;
    int out_f16;
    DecSpan* span_route;   // or null
    DecSpan* span_ffn;     // or null
    unsigned long long* trace;  // diagnostics: [grid][kDecTrace][2] (event, globaltimer ns) or null
    const __half* wgt;     // fused routing: the bank's split gate weights (dec_split_wg) or null
    int wg_shift;
    int fused;             // routing inside k_dec (T <= 32, bank router, finite Wg)
    int route_nbuf;        // set by launch_dec: Wg chunk buffers of the fused routing
    int route_cluster;     // fused routing: CTAs per cluster sharing the K chunks (2 or 4), 1 = every CTA alone
    int plan_ready;        // units / permuted rows prepared by k_dec_prep (no k_dec_route launch)
    uint32_t stage_bytes, stage2_bytes;  // set by launch_dec: W1 / W2 ring stage sizes
    int n_stages, n_stages2;
};
bool dec_supported(int64_t T, int topk, int d, int E, int Kp1, int Np1, int Np2);
int64_t dec_slice_bytes(int bits, int Kp1, int Np2);
cudaError_t dec_build_layout(const uint8_t* w1, const uint8_t* w2, int64_t w1_stride, int64_t w2_stride, int E,
                             int Kp1, int Np1, int Np2, int bits, uint8_t* out, cudaStream_t st);
cudaError_t launch_dec(int bits, const DecArgs& a, cudaStream_t st, int num_sms);
bool dec_mid_supported(int d, int E, int Kp1, int Np1, int Np2);
// k_dec_prep: units of the experts with 0 < rows <= gemv_max (path 1: every expert) from the
// plan's counts / offsets, and their permuted rows scaled by 2^-s(k) with Z, into xperm.
cudaError_t launch_dec_prep(int bits, const void* h, int h_f16, int64_t T, int d, int E, int Kp1, int path,
                            int gemv_max, const Plan& P, int4* units, int* n_units, __half* xperm, int xpitch,
                            cudaStream_t st);
int64_t dec_wgt_halves(int E, int Kp1);
cudaError_t dec_split_wg(const float* wg, int d, int E, int Kp1, int shift, __half* out, cudaStream_t st);

}  // namespace moqe_gpu
