// capi.cu — C-ABI entry points: device-resident expert bank, workspace and
// the moe_forward orchestration (route -> permute -> GEMV / tcgen05 GEMM ->
// combine), all stream-ordered with no host synchronisation on the hot path.
//
// Reference interface replaced: moqe::moe_ffn_forward
// (include/moqe/model.hpp:87, proj/src/model.cpp:348-393) and the ExpertBank /
// RouterState types (model.hpp:56-82).
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "kernels.cuh"

namespace moqe_gpu {

// ---- errors --------------------------------------------------------------------
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
moqe_status fail(moqe_status st, const std::string& msg) {
    set_error(msg);
    return st;
}
moqe_status cuda_fail(cudaError_t err, const char* what) {
    set_error(std::string(what) + ": " + cudaGetErrorString(err));
    return MOQE_CUDA_ERROR;
}

__global__ void k_f32_to_f16(const float* __restrict__ a, __half* __restrict__ b, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) b[i] = __float2half_rn(a[i]);
}

}  // namespace moqe_gpu

using namespace moqe_gpu;

struct Workspace {
    int64_t cap_rows = 0, cap_tokens = 0;
    void* block = nullptr;
    Plan P{};
    __half* mid = nullptr;
    __half* x_perm = nullptr;
    float* out_acc = nullptr;
    uint8_t* xr = nullptr;         // decode GEMV: fc1 row blocks (k_xrows)
    uint8_t* xb = nullptr;         // decode GEMV: fc2 row blocks (fc1 epilogue -> fc2)
    unsigned* ready = nullptr;     // decode GEMV, fused grid: fc1 m-tiles done per pass
    // decode path (dec.cu), fixed size: kDecMaxRows routed rows
    void* dblock = nullptr;
    int4* d_units = nullptr;
    int* d_nunits = nullptr;
    int32_t* d_perm_token = nullptr;
    float* d_perm_gate = nullptr;
    int32_t* d_row_of = nullptr;
    __half* d_xperm = nullptr;
    long long* d_acc = nullptr;
    unsigned* d_unit_done = nullptr;
    float* d_ybuf = nullptr;
    unsigned* d_tok_cnt = nullptr;
};

struct moqe_bank {
    int E = 0, bits = 0;
    int64_t d = 0, f = 0;
    int Kp1 = 0, Np1 = 0, Kp2 = 0, Np2 = 0;
    uint8_t* w1 = nullptr;
    uint8_t* w2 = nullptr;
    int64_t w1_stride = 0, w2_stride = 0;
    float* s1 = nullptr;
    float* s2 = nullptr;
    float* b1 = nullptr;
    float* b2 = nullptr;
    float* wg = nullptr;
    float* wg_blk = nullptr;  // blocked transposed copy for the decode router (route_block_wg)
    int wg_finite = 0;
    float* smax1 = nullptr;  // [E] fc2 fixed-point bound constants (decode GEMV)
    float* bmax1 = nullptr;
    uint8_t* wdec = nullptr;  // decode layout (dec_build_layout), d_model <= 1024 only
    int log = 0;              // log-scale experts (Scheme::LogScale): tcgen05 path only
    __half* wgt = nullptr;    // split gate weights for the fused decode routing (dec_split_wg)
    int wg_shift = 0;
    int64_t wdec_stride = 0, dec_slice = 0;
    DecSpan* spans = nullptr;  // [2] router / expert-FFN launch spans (moqe_gpu_bank_span)
    bool span_on = false;
    int num_sms = 148;
    int device = 0;
    cudaStream_t host_stream = nullptr;
    void* h_dev = nullptr;   // host-API staging
    void* o_dev = nullptr;
    int64_t host_cap = 0;
    Workspace ws;
    // per-kernel event timing (bench support)
    bool prof = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
    std::vector<std::pair<int, int>> ev_used;  // (kind, pool index)
    double prof_ms[MOQE_PROFILE_KINDS] = {0};
    unsigned long long* trace = nullptr;  // GEMV event trace (moqe_gpu_bank_trace)
    int64_t prof_n[MOQE_PROFILE_KINDS] = {0};
};

namespace {
int route_dbg() {  // diagnostics only
    static const int v = [] { const char* s = getenv("MOQE_ROUTE_DBG"); return s ? atoi(s) : 0; }();
    return v;
}
bool gemv_fused() {  // MOQE_GEMV_FUSED=0: decode as two grids (fc1, fc2) even when one would do
    static const bool v = [] { const char* s = getenv("MOQE_GEMV_FUSED"); return !(s && atoi(s) == 0); }();
    return v;
}
bool dec_enabled() {  // MOQE_DEC=0: decode batches take the round-1 GEMV path instead
    static const bool v = [] { const char* s = getenv("MOQE_DEC"); return !(s && atoi(s) == 0); }();
    return v;
}
bool fused_enabled() {  // MOQE_DEC_FUSED=0: decode keeps the separate router launch
    static const bool v = [] { const char* s = getenv("MOQE_DEC_FUSED"); return !(s && atoi(s) == 0); }();
    return v;
}
int route_cluster_env() {  // MOQE_DEC_CLUSTER=1|2|4: CTAs per routing cluster of the fused decode
    static const int v = [] {
        const char* s = getenv("MOQE_DEC_CLUSTER");
        const int c = s ? atoi(s) : 2;
        return (c == 1 || c == 4) ? c : 2;
    }();
    return v;
}
bool dec_mid_enabled() {  // MOQE_DEC_MID=0: mid-size batches keep the round-1 GEMV for their small experts
    static const bool v = [] { const char* s = getenv("MOQE_DEC_MID"); return !(s && atoi(s) == 0); }();
    return v;
}
int dec_mid_rows() {  // MOQE_DEC_MID_ROWS: experts with at most this many rows run on k_dec (default 32)
    static const int v = [] {
        const char* s = getenv("MOQE_DEC_MID_ROWS");
        const int r = s ? atoi(s) : 32;
        return r < 1 ? 1 : r;
    }();
    return v;
}
int64_t dec_mid_avg() {  // MOQE_DEC_MID_AVG: mid-size path while T*k <= this many rows per expert on average (16)
    static const int64_t v = [] {
        const char* s = getenv("MOQE_DEC_MID_AVG");
        const int r = s ? atoi(s) : 16;
        return int64_t(r < 1 ? 1 : r);
    }();
    return v;
}
bool xrows_in_router() {  // MOQE_XROWS_IN_ROUTER=0: decode keeps the separate k_xrows launch
    static const bool v = [] { const char* s = getenv("MOQE_XROWS_IN_ROUTER"); return !(s && atoi(s) == 0); }();
    return v;
}
int gemv_dbg() {  // diagnostics only
    static const int v = [] { const char* s = getenv("MOQE_GEMV_DBG"); return s ? atoi(s) : 0; }();
    return v;
}
struct KernelTimer {
    moqe_bank* b;
    int kind;
    int idx = -1;
    cudaStream_t st;
    KernelTimer(moqe_bank* bank, int k, cudaStream_t s) : b(bank), kind(k), st(s) {
        if (!b->prof) return;
        idx = int(b->ev_used.size());
        if (idx >= int(b->ev_pool.size())) {
            cudaEvent_t a, z;
            cudaEventCreate(&a);
            cudaEventCreate(&z);
            b->ev_pool.emplace_back(a, z);
        }
        b->ev_used.emplace_back(kind, idx);
        cudaEventRecordWithFlags(b->ev_pool[idx].first, st, cudaEventRecordExternal);
    }
    ~KernelTimer() {
        if (idx >= 0) cudaEventRecordWithFlags(b->ev_pool[idx].second, st, cudaEventRecordExternal);
    }
};
}  // namespace

namespace {

template <class T>
T* carve(char*& p, int64_t n) {
    T* r = reinterpret_cast<T*>(p);
    p += round_up(int64_t(sizeof(T)) * std::max<int64_t>(n, 1), 256);
    return r;
}

moqe_status ensure_workspace(moqe_bank* b, int64_t T, int topk) {
    Workspace& w = b->ws;
    const int64_t R = T * topk;
    if (T <= w.cap_tokens && R <= w.cap_rows) return MOQE_OK;
    const int64_t capT = std::max(T, w.cap_tokens);
    const int64_t capR = std::max<int64_t>(std::max(R, w.cap_rows), capT * 2);  // room for top-2
    if (w.block) {
        MOQE_CUDA(cudaDeviceSynchronize());
        cudaFree(w.block);
        w.block = nullptr;
    }
    const int E = b->E;
    const int64_t nctas = (capT + 3) / 4;  // routing CTAs cover >= 4 tokens each
    // sizing pass
    int64_t bytes = 0;
    auto add = [&](int64_t sz, int64_t n) { bytes += round_up(sz * std::max<int64_t>(n, 1), 256); };
    add(4, capR); add(4, capR); add(4, capR); add(4, nctas * E); add(4, E); add(4, E + 1);
    add(4, capR); add(4, capR); add(4, capR); add(4, E); add(4, E); add(4, E + 1); add(4, 8);
    add(4, 8); add(4, E); add(16, std::max(E + 1, 64));
    add(2, capR * b->Np1); add(2, capR * b->Kp1); add(4, capT * b->d); add(4, capT * E);
    const int64_t xr_bytes = gemv_xr_bytes(b->bits) * gemv_chunks(b->Kp1) * capT;
    const int64_t xb_bytes = gemv_xb_bytes(b->bits) * gemv_chunks(b->Kp2) * capR;
    add(xr_bytes, 1);
    add(xb_bytes, 1);
    add(4, kSelfPlanRows);
    MOQE_CUDA(cudaMalloc(&w.block, bytes));
    MOQE_CUDA(cudaMemset(w.block, 0, bytes));
    char* p = static_cast<char*>(w.block);
    Plan& P = w.P;
    P.expert = carve<int32_t>(p, capR);
    P.gate = carve<float>(p, capR);
    P.lrank = carve<int32_t>(p, capR);
    P.cta_counts = carve<int32_t>(p, nctas * E);
    P.counts = carve<int32_t>(p, E);
    P.offsets = carve<int32_t>(p, E + 1);
    P.perm_token = carve<int32_t>(p, capR);
    P.perm_gate = carve<float>(p, capR);
    P.inv_pos = carve<int32_t>(p, capR);
    P.gemv_list = carve<int32_t>(p, E);
    P.gemm_list = carve<int32_t>(p, E);
    P.gemm_tile_start = carve<int32_t>(p, E + 1);
    P.meta = carve<int32_t>(p, 8);
    P.tickets = carve<unsigned>(p, 8);
    P.done = carve<unsigned>(p, E);
    P.gtab = carve<int4>(p, std::max(E + 1, 64));  // >= 33: the GEMV's speculative first load round
    w.mid = carve<__half>(p, capR * b->Np1);
    w.x_perm = carve<__half>(p, capR * b->Kp1);
    w.out_acc = carve<float>(p, capT * b->d);
    P.logits = carve<float>(p, capT * E);
    w.xr = carve<uint8_t>(p, xr_bytes);
    w.xb = carve<uint8_t>(p, xb_bytes);
    w.ready = carve<unsigned>(p, kSelfPlanRows);
    w.cap_rows = capR;
    w.cap_tokens = capT;
    return MOQE_OK;
}

moqe_status ensure_dec_workspace(moqe_bank* b) {
    Workspace& w = b->ws;
    if (w.dblock) return MOQE_OK;
    const int64_t R = kDecMaxRows, xpitch = int64_t(b->Kp1) * 2 + 16;
    int64_t bytes = 0;
    auto add = [&](int64_t n) { int64_t o = bytes; bytes += round_up(std::max<int64_t>(n, 1), 256); return o; };
    // units, permuted rows, fc2 accumulators and unit counters also serve the mid-size path
    const int64_t RM = kDecMidMaxRows, UM = kDecMidMaxUnits;
    const int64_t o_units = add(16 * UM), o_nu = add(16), o_pt = add(4 * R), o_pg = add(4 * R), o_ro = add(4 * R),
                  o_x = add(xpitch * RM), o_acc = add(8 * RM * b->Np2), o_ud = add(4 * UM), o_yb = add(4 * R * b->d),
                  o_tc = add(4 * R);
    MOQE_CUDA(cudaMalloc(&w.dblock, bytes));
    MOQE_CUDA(cudaMemset(w.dblock, 0, bytes));
    char* p = static_cast<char*>(w.dblock);
    w.d_units = reinterpret_cast<int4*>(p + o_units);
    w.d_nunits = reinterpret_cast<int*>(p + o_nu);
    w.d_perm_token = reinterpret_cast<int32_t*>(p + o_pt);
    w.d_perm_gate = reinterpret_cast<float*>(p + o_pg);
    w.d_row_of = reinterpret_cast<int32_t*>(p + o_ro);
    w.d_xperm = reinterpret_cast<__half*>(p + o_x);
    w.d_acc = reinterpret_cast<long long*>(p + o_acc);
    w.d_unit_done = reinterpret_cast<unsigned*>(p + o_ud);
    w.d_ybuf = reinterpret_cast<float*>(p + o_yb);
    w.d_tok_cnt = reinterpret_cast<unsigned*>(p + o_tc);
    return MOQE_OK;
}

void free_bank(moqe_bank* b) {
    if (!b) return;
    cudaFree(b->w1);
    cudaFree(b->w2);
    cudaFree(b->s1);
    cudaFree(b->s2);
    cudaFree(b->b1);
    cudaFree(b->b2);
    cudaFree(b->wg);
    cudaFree(b->wg_blk);
    cudaFree(b->smax1);
    cudaFree(b->bmax1);
    cudaFree(b->ws.block);
    cudaFree(b->ws.dblock);
    cudaFree(b->wdec);
    cudaFree(b->wgt);
    cudaFree(b->spans);
    cudaFree(b->h_dev);
    cudaFree(b->o_dev);
    cudaFree(b->trace);
    if (b->host_stream) cudaStreamDestroy(b->host_stream);
    delete b;
}

// copy [E][n] (host or device) into a zero-padded device [E][np] array
moqe_status upload_padded(float** dst, const float* src, int E, int64_t n, int64_t np, bool on_dev) {
    MOQE_CUDA(cudaMalloc(dst, sizeof(float) * E * np));
    MOQE_CUDA(cudaMemset(*dst, 0, sizeof(float) * E * np));
    MOQE_CUDA(cudaMemcpy2D(*dst, np * sizeof(float), src, n * sizeof(float), n * sizeof(float), E,
                           on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    return MOQE_OK;
}

}  // namespace

extern "C" {

int moqe_gpu_abi_version(void) { return MOQE_GPU_ABI_VERSION; }
const char* moqe_gpu_last_error(void) { return g_last_error.c_str(); }
const char* moqe_gpu_status_string(moqe_status st) {
    switch (st) {
        case MOQE_OK: return "ok";
        case MOQE_INVALID_ARGUMENT: return "invalid_argument";
        case MOQE_OUT_OF_RANGE: return "out_of_range";
        case MOQE_RANGE_ERROR: return "range_error";
        case MOQE_CUDA_ERROR: return "cuda_error";
        case MOQE_NCCL_ERROR: return "nccl_error";
        case MOQE_NOT_SUPPORTED: return "not_supported";
        case MOQE_CHECKPOINT_ERROR: return "checkpoint_error";
    }
    return "unknown";
}

moqe_status moqe_gpu_bank_create(int n_experts, int64_t d_model, int64_t d_ffn, int bits,
                                 const uint8_t* packed_w1, const float* scales1,
                                 const uint8_t* packed_w2, const float* scales2, const float* b1,
                                 const float* b2, int inputs_on_device, moqe_bank_t* out) {
    if (!out) return fail(MOQE_INVALID_ARGUMENT, "bank_create: null output handle");
    *out = nullptr;
    if (n_experts <= 0) return fail(MOQE_INVALID_ARGUMENT, "moe_ffn_forward: empty expert bank");
    if (n_experts > 256) return fail(MOQE_NOT_SUPPORTED, "bank_create: at most 256 experts");
    if (!valid_bits(bits)) return fail(MOQE_INVALID_ARGUMENT, "quant: unsupported bit width");
    if (d_model <= 0 || d_ffn <= 0) return fail(MOQE_INVALID_ARGUMENT, "bank_create: bad dimensions");
    if (!packed_w1 || !packed_w2 || !scales1 || !scales2)
        return fail(MOQE_INVALID_ARGUMENT, "bank_create: null weights");
    auto* b = new moqe_bank;
    b->E = n_experts;
    b->d = d_model;
    b->f = d_ffn;
    b->bits = bits;
    b->Kp1 = int(round_up(d_model, 2 * TILE_K));  // even number of k-blocks (GEMV stages hold 2)
    b->Np1 = int(round_up(d_ffn, TILE_N));
    b->Kp2 = b->Np1;  // fc2 consumes the full (zero-padded) fc1 output width
    b->Np2 = int(round_up(d_model, TILE_N));
    cudaError_t ce = cudaGetDevice(&b->device);
    if (ce == cudaSuccess) ce = cudaDeviceGetAttribute(&b->num_sms, cudaDevAttrMultiProcessorCount, b->device);
    if (ce != cudaSuccess) {
        free_bank(b);
        return cuda_fail(ce, "cudaGetDevice");
    }
    const bool dev = inputs_on_device != 0;
    b->w1_stride = int64_t(b->Np1 / TILE_N) * (b->Kp1 / TILE_K) * tile_bytes(bits);
    b->w2_stride = int64_t(b->Np2 / TILE_N) * (b->Kp2 / TILE_K) * tile_bytes(bits);
    const int64_t src1 = packed_size(bits, d_model * d_ffn), src2 = src1;
    uint8_t* stage = nullptr;
    moqe_status st = MOQE_OK;
    do {
        if ((ce = cudaMalloc(&b->w1, b->w1_stride * n_experts)) != cudaSuccess) break;
        if ((ce = cudaMalloc(&b->w2, b->w2_stride * n_experts)) != cudaSuccess) break;
        const uint8_t* s1p = packed_w1;
        const uint8_t* s2p = packed_w2;
        if (!dev) {
            if ((ce = cudaMalloc(&stage, std::max(src1, src2) * n_experts)) != cudaSuccess) break;
            if ((ce = cudaMemcpy(stage, packed_w1, src1 * n_experts, cudaMemcpyHostToDevice)) != cudaSuccess) break;
            s1p = stage;
        }
        if ((st = retile(s1p, d_model, d_ffn, bits, n_experts, b->w1, b->Kp1, b->Np1, nullptr)) != MOQE_OK) break;
        if (!dev) {
            if ((ce = cudaDeviceSynchronize()) != cudaSuccess) break;
            if ((ce = cudaMemcpy(stage, packed_w2, src2 * n_experts, cudaMemcpyHostToDevice)) != cudaSuccess) break;
            s2p = stage;
        }
        if ((st = retile(s2p, d_ffn, d_model, bits, n_experts, b->w2, b->Kp2, b->Np2, nullptr)) != MOQE_OK) break;
        if ((st = upload_padded(&b->s1, scales1, n_experts, d_ffn, b->Np1, dev)) != MOQE_OK) break;
        if ((st = upload_padded(&b->s2, scales2, n_experts, d_model, b->Np2, dev)) != MOQE_OK) break;
        if (b1 && (st = upload_padded(&b->b1, b1, n_experts, d_ffn, b->Np1, dev)) != MOQE_OK) break;
        if (b2 && (st = upload_padded(&b->b2, b2, n_experts, d_model, b->Np2, dev)) != MOQE_OK) break;
        {
            if ((ce = cudaMalloc(&b->smax1, sizeof(float) * n_experts)) != cudaSuccess) break;
            if ((ce = cudaMalloc(&b->bmax1, sizeof(float) * n_experts)) != cudaSuccess) break;
            if ((ce = launch_expert_max(b->s1, b->b1, n_experts, b->Np1, b->smax1, b->bmax1, nullptr)) !=
                cudaSuccess)
                break;
        }
        if (b->Kp1 <= 1024 && b->Np2 <= 1024) {
            b->dec_slice = dec_slice_bytes(bits, b->Kp1, b->Np2);
            b->wdec_stride = b->dec_slice * (b->Np1 / 64);
            if ((ce = cudaMalloc(&b->wdec, b->wdec_stride * n_experts)) != cudaSuccess) break;
            if ((ce = dec_build_layout(b->w1, b->w2, b->w1_stride, b->w2_stride, n_experts, b->Kp1, b->Np1, b->Np2,
                                       bits, b->wdec, nullptr)) != cudaSuccess)
                break;
        }
        if ((ce = cudaMalloc(&b->spans, 2 * sizeof(DecSpan))) != cudaSuccess) break;
        {
            DecSpan z[2];
            for (auto& x : z) { x.start_min = ~0ull; x.ticket = x.pad = 0; x.total_ns = x.count = 0; }
            if ((ce = cudaMemcpy(b->spans, z, sizeof(z), cudaMemcpyHostToDevice)) != cudaSuccess) break;
        }
        if ((ce = cudaDeviceSynchronize()) != cudaSuccess) break;
    } while (false);
    if (stage) cudaFree(stage);
    if (ce != cudaSuccess) st = cuda_fail(ce, "bank_create");
    if (st != MOQE_OK) {
        free_bank(b);
        return st;
    }
    *out = b;
    return MOQE_OK;
}

moqe_status moqe_gpu_bank_create_g(int n_experts, int64_t d_model, int64_t d_ffn, int bits, int granularity,
                                   const uint8_t* packed_w1, const float* scales1, const uint8_t* packed_w2,
                                   const float* scales2, const float* b1, const float* b2, int inputs_on_device,
                                   moqe_bank_t* out) {
    if (granularity == 0)
        return moqe_gpu_bank_create(n_experts, d_model, d_ffn, bits, packed_w1, scales1, packed_w2, scales2, b1, b2,
                                    inputs_on_device, out);
    if (granularity != 1) return fail(MOQE_INVALID_ARGUMENT, "bank_create: bad granularity");
    if (n_experts <= 0 || d_model <= 0 || d_ffn <= 0 || !scales1 || !scales2)
        return moqe_gpu_bank_create(n_experts, d_model, d_ffn, bits, packed_w1, scales1, packed_w2, scales2, b1, b2,
                                    inputs_on_device, out);
    // per-tensor: one scale per matrix, broadcast to its channels (scale_index, quant.cpp:53-55)
    std::vector<float> t1(n_experts), t2(n_experts);
    const cudaMemcpyKind k = inputs_on_device ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost;
    MOQE_CUDA(cudaMemcpy(t1.data(), scales1, sizeof(float) * n_experts, k));
    MOQE_CUDA(cudaMemcpy(t2.data(), scales2, sizeof(float) * n_experts, k));
    std::vector<float> e1(size_t(n_experts) * d_ffn), e2(size_t(n_experts) * d_model);
    for (int e = 0; e < n_experts; ++e) {
        std::fill(e1.begin() + size_t(e) * d_ffn, e1.begin() + size_t(e + 1) * d_ffn, t1[e]);
        std::fill(e2.begin() + size_t(e) * d_model, e2.begin() + size_t(e + 1) * d_model, t2[e]);
    }
    if (!inputs_on_device)
        return moqe_gpu_bank_create(n_experts, d_model, d_ffn, bits, packed_w1, e1.data(), packed_w2, e2.data(), b1, b2,
                                    0, out);
    float *d1 = nullptr, *d2 = nullptr;
    MOQE_CUDA(cudaMalloc(&d1, e1.size() * sizeof(float)));
    cudaError_t ce = cudaMalloc(&d2, e2.size() * sizeof(float));
    if (ce == cudaSuccess) ce = cudaMemcpy(d1, e1.data(), e1.size() * sizeof(float), cudaMemcpyHostToDevice);
    if (ce == cudaSuccess) ce = cudaMemcpy(d2, e2.data(), e2.size() * sizeof(float), cudaMemcpyHostToDevice);
    moqe_status st = ce == cudaSuccess ? moqe_gpu_bank_create(n_experts, d_model, d_ffn, bits, packed_w1, d1, packed_w2,
                                                              d2, b1, b2, 1, out)
                                       : cuda_fail(ce, "bank_create_g");
    cudaFree(d1);
    cudaFree(d2);
    return st;
}

moqe_status moqe_gpu_bank_create_ex(int n_experts, int64_t d_model, int64_t d_ffn, int bits, int scheme,
                                    int granularity, const uint8_t* packed_w1, const float* scales1,
                                    const uint8_t* packed_w2, const float* scales2, const float* b1, const float* b2,
                                    int inputs_on_device, moqe_bank_t* out) {
    if (scheme != MOQE_SCHEME_LINEAR && scheme != MOQE_SCHEME_LOG)
        return fail(MOQE_INVALID_ARGUMENT, "bank_create: bad scheme");
    if (scheme == MOQE_SCHEME_LOG && bits == 8)
        return fail(MOQE_NOT_SUPPORTED, "bank_create: log-scale int8 (k up to 127) is not a GPU scheme");
    moqe_status st = moqe_gpu_bank_create_g(n_experts, d_model, d_ffn, bits, granularity, packed_w1, scales1, packed_w2,
                                            scales2, b1, b2, inputs_on_device, out);
    if (st == MOQE_OK && scheme == MOQE_SCHEME_LOG) (*out)->log = 1;
    return st;
}

moqe_status moqe_gpu_bank_destroy(moqe_bank_t bank) {
    if (bank) cudaDeviceSynchronize();
    free_bank(bank);
    return MOQE_OK;
}

moqe_status moqe_gpu_bank_set_router(moqe_bank_t b, const float* wg, int on_device) {
    if (!b || !wg) return fail(MOQE_INVALID_ARGUMENT, "top1_route: no gate weights");
    if (!b->wg) MOQE_CUDA(cudaMalloc(&b->wg, sizeof(float) * b->d * b->E));
    MOQE_CUDA(cudaMemcpy(b->wg, wg, sizeof(float) * b->d * b->E,
                         on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
    if (!b->wg_blk) MOQE_CUDA(cudaMalloc(&b->wg_blk, sizeof(float) * route_wg_block_floats(int(b->d), b->E) + 16));
    int* flag = reinterpret_cast<int*>(b->wg_blk + route_wg_block_floats(int(b->d), b->E));
    MOQE_CUDA(route_block_wg(b->wg, int(b->d), b->E, b->wg_blk, flag, &b->wg_finite));
    if (b->wg_finite && b->Kp1 % 64 == 0) {  // the split copy the fused decode and prefill routers stream
        std::vector<float> hw(size_t(b->d) * b->E);
        MOQE_CUDA(cudaMemcpy(hw.data(), b->wg, hw.size() * sizeof(float), cudaMemcpyDeviceToHost));
        float mx = 0.f;
        for (float v : hw) mx = std::max(mx, std::fabs(v));
        int e2 = 0;
        if (mx > 0.f && std::isfinite(mx)) std::frexp(mx, &e2);  // mx < 2^e2
        b->wg_shift = 14 - e2;
        if (!b->wgt) MOQE_CUDA(cudaMalloc(&b->wgt, sizeof(__half) * dec_wgt_halves(b->E, b->Kp1)));
        MOQE_CUDA(dec_split_wg(b->wg, int(b->d), b->E, b->Kp1, b->wg_shift, b->wgt, nullptr));
        MOQE_CUDA(cudaDeviceSynchronize());
    }
    return MOQE_OK;
}

int64_t moqe_gpu_bank_weight_bytes(moqe_bank_t b) {
    if (!b) return -1;
    return (b->w1_stride + b->w2_stride) * b->E;
}

namespace {
// Shared forward body. With pre_expert/pre_gate (expert-parallel owner side),
// rows arrive already routed: the plan is built from the given ids (top-1 per
// row) and the router is skipped.
// The decode kernel (k_dec) takes the forward: its output is written with plain stores only
// (no atomics), so it may target mapped pinned host memory directly.
bool dec_path_taken(moqe_bank_t b, int64_t t, int top_k, moqe_path path) {
    // 32 < T <= 64 top-1: the batched router + the mid-size k_dec path, unless MOQE_DEC_ROUTER=1
    // keeps the one-cluster decode router (k_dec_route)
    static const bool dec_router = [] { const char* s = getenv("MOQE_DEC_ROUTER"); return s && atoi(s) == 1; }();
    if (t > 32 && top_k == 1 && !dec_router && dec_mid_enabled() && t <= 16 * int64_t(b->E)) return false;
    return !b->log && b->wdec && dec_enabled() && (path == MOQE_PATH_AUTO || path == MOQE_PATH_GEMV) &&
           dec_supported(t, top_k, int(b->d), b->E, b->Kp1, b->Np1, b->Np2);
}

moqe_status forward_impl(moqe_bank_t b, const void* h, moqe_dtype h_dtype, int64_t t, const float* wg, int top_k,
                         void* out, moqe_dtype out_dtype, int32_t* expert_out, float* gate_out, moqe_path path,
                         void* stream, const int32_t* pre_expert, const float* pre_gate) {
    if (!b) return fail(MOQE_INVALID_ARGUMENT, "moe_ffn_forward: empty expert bank");
    if (t < 0) return fail(MOQE_INVALID_ARGUMENT, "moe_ffn_forward: negative token count");
    if (top_k != 1 && top_k != 2) return fail(MOQE_INVALID_ARGUMENT, "moe_forward: top_k must be 1 or 2");
    if (top_k == 2 && b->E < 2) return fail(MOQE_INVALID_ARGUMENT, "moe_forward: top-2 needs >= 2 experts");
    if (h_dtype != MOQE_F32 && h_dtype != MOQE_F16) return fail(MOQE_INVALID_ARGUMENT, "moe_forward: bad h dtype");
    if (out_dtype != MOQE_F32 && out_dtype != MOQE_F16) return fail(MOQE_INVALID_ARGUMENT, "moe_forward: bad out dtype");
    const bool pre = pre_expert != nullptr;
    if (!pre) {
        if (!wg) wg = b->wg;
        if (!wg) return fail(MOQE_INVALID_ARGUMENT, "top1_route: no gate weights");
    }
    if (t == 0) return MOQE_OK;
    if (!h || !out) return fail(MOQE_INVALID_ARGUMENT, "moe_forward: null buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    (void)cudaGetLastError();  // launch checks below must not see a stale error from unrelated calls
    if (b->log) {  // log-scale codes: only the tcgen05 GEMM converts them (unpack_chunk_log)
        if (path == MOQE_PATH_GEMV) return fail(MOQE_NOT_SUPPORTED, "moe_forward: log-scale banks take the GEMM path");
        path = MOQE_PATH_GEMM;
    }
    if (!pre && dec_path_taken(b, t, top_k, path)) {
        moqe_status s = ensure_dec_workspace(b);
        if (s != MOQE_OK) return s;
        s = ensure_workspace(b, t, top_k);  // routing outputs when the caller passes none
        if (s != MOQE_OK) return s;
        Workspace& w = b->ws;
        DecArgs a{};
        a.h = h;
        a.h_f16 = h_dtype == MOQE_F16;
        a.T = int(t);
        a.d = int(b->d);
        a.wg = wg;
        a.E = b->E;
        a.topk = top_k;
        a.bits = b->bits;
        a.expert = expert_out ? expert_out : w.P.expert;
        a.gate = gate_out ? gate_out : w.P.gate;
        a.units = w.d_units;
        a.n_units = w.d_nunits;
        a.perm_token = w.d_perm_token;
        a.perm_gate = w.d_perm_gate;
        a.row_of = w.d_row_of;
        a.xperm = w.d_xperm;
        a.xpitch = b->Kp1 * 2 + 16;
        a.Kp1 = b->Kp1;
        a.Np1 = b->Np1;
        a.Np2 = b->Np2;
        a.S = b->Np1 / 64;
        a.wdec = b->wdec;
        a.wdec_stride = b->wdec_stride;
        a.slice_bytes = b->dec_slice;
        a.s1 = b->s1;
        a.b1 = b->b1;
        a.s2 = b->s2;
        a.b2 = b->b2;
        a.acc = w.d_acc;
        a.unit_done = w.d_unit_done;
        a.ybuf = w.d_ybuf;
        a.tok_cnt = w.d_tok_cnt;
        a.out = out;
        a.out_f16 = out_dtype == MOQE_F16;
        a.span_route = b->span_on ? b->spans : nullptr;
        a.span_ffn = b->span_on ? b->spans + 1 : nullptr;
        a.trace = b->trace;
        a.fused = (wg == b->wg && b->wgt && b->wg_finite && t <= 32 && fused_enabled()) ? 1 : 0;
        a.wgt = b->wgt;
        a.wg_shift = b->wg_shift;
        a.route_cluster = route_cluster_env();
        cudaError_t ce = launch_dec(b->bits, a, st, b->num_sms);
        if (ce != cudaSuccess) return cuda_fail(ce, "k_dec");
        return MOQE_OK;
    }
    moqe_status s = ensure_workspace(b, t, top_k);
    if (s != MOQE_OK) return s;
    Workspace& w = b->ws;
    Plan P = w.P;
    if (pre) {
        P.expert = const_cast<int32_t*>(pre_expert);
        P.gate = const_cast<float*>(pre_gate);
    } else {
        if (expert_out) P.expert = expert_out;
        if (gate_out) P.gate = gate_out;
    }
    const int64_t R = t * top_k;
    int eff_path = int(path);
    if (eff_path == MOQE_PATH_GEMM && !gemm_available())
        return fail(MOQE_NOT_SUPPORTED, "moe_forward: tcgen05 GEMM path not built");
    if (eff_path == MOQE_PATH_AUTO && !gemm_available()) eff_path = MOQE_PATH_GEMV;
    // Small batches: no expert can exceed a few GEMV passes, so skip the (empty)
    // scatter + tcgen05 launches entirely; the GEMV takes every expert.
    if (!gemv_supported(b->Kp1, b->Kp2)) {  // decode kernels hold a whole fc1 row of fragments in smem
        if (eff_path == MOQE_PATH_GEMV) return fail(MOQE_NOT_SUPPORTED, "moe_forward: GEMV path needs d_model <= 2048");
        eff_path = MOQE_PATH_GEMM;
    }
    if (eff_path == MOQE_PATH_AUTO && R <= 4 * kGemvMaxRows) eff_path = MOQE_PATH_GEMV;
    // Large batches: experts almost never stay within GEMV size, and the GEMV
    // launches (+ token-row encoding) would cost ~15 us of empty work.
    if (eff_path == MOQE_PATH_AUTO && R > 1024) eff_path = MOQE_PATH_GEMM;
    const bool need_gemm = eff_path == MOQE_PATH_GEMM || (eff_path == MOQE_PATH_AUTO && R > kGemvMaxRows);
    const bool need_gemv = eff_path != MOQE_PATH_GEMM;
    const bool inline_scatter = !need_gemm && R <= 256;
    // mid-size top-1 batches on a decode-capable bank: the small experts (<= dec_mid_rows() rows)
    // run on k_dec from the router's plan instead of the round-1 GEMV. Not for pre-routed rows:
    // the expert-parallel owner keeps the kernels of the top-k forward it stands in for (an fp32
    // return then equals the single-GPU forward bit for bit, ep.py)
    const bool dec_mid = !pre && need_gemv && top_k == 1 && !b->log && b->wdec && dec_enabled() && dec_mid_enabled() &&
                         R <= kDecMidMaxRows && R <= dec_mid_avg() * int64_t(b->E) &&  // ~1-2 units per expert on average
                         dec_mid_supported(int(b->d), b->E, b->Kp1, b->Np1, b->Np2);
    const int gemv_max = dec_mid ? dec_mid_rows() : kGemvMaxRows;
    float* acc = nullptr;
    if (top_k == 2) acc = out_dtype == MOQE_F32 ? static_cast<float*>(out) : w.out_acc;

    RouteArgs ra{h, h_dtype == MOQE_F16, t, int(b->d), wg, b->E, top_k, eff_path, inline_scatter ? 1 : 0,
                 gemm_block_n(), inline_scatter ? acc : nullptr,
                 b->trace ? b->trace + int64_t(b->num_sms) * kTraceCap * 2 : nullptr};
    ra.gemv_max = gemv_max;
    cudaError_t ce;
    bool self_plan = false;
    {
        KernelTimer kt(b, 0, st);
        // decode, every expert on the GEMV path: the router writes only the choices and the
        // GEMV kernels build the plan themselves (no serial plan step between them)
        self_plan = !dec_mid && !pre && !need_gemm && R <= kSelfPlanRows && t <= 32 && b->E <= 256;
        ra.no_plan = self_plan ? 1 : 0;
        if (wg == b->wg && b->wg_blk) { ra.wg_blk = b->wg_blk; ra.wg_finite = b->wg_finite; }
        if (wg == b->wg && b->wgt) { ra.wgt = b->wgt; ra.wg_shift = b->wg_shift; ra.Kp1 = int(b->Kp1); }
        ra.dbg = route_dbg();
        // the router's copy warp writes the fc1 row blocks only with the one-chunk Wg layout: with
        // two chunks it would run after the chain's last chunk, k_xrows overlaps better
        if (need_gemv && !dec_mid && !pre && route_chain_used(ra) && xrows_in_router() &&
            route_chain_one_chunk(int(b->d), b->E)) {
            // decode: the router leads the chain (waits for the previous grid itself) and its
            // copy warp writes the fc1 row blocks — two launches per forward
            ra.first = 1;
            ra.pdl = 1;
            ra.xr = w.xr;
            ra.nch1 = gemv_chunks(b->Kp1);
            ra.xr_bits = b->bits;
            ra.ready = self_plan && gemv_fused() ? w.ready : nullptr;
        } else if (need_gemv && !dec_mid) {  // token rows -> fc1 row blocks; the decode router overlaps it (PDL)
            XrowArgs xa{h, h_dtype == MOQE_F16, t, int(b->d), gemv_chunks(b->Kp1), w.xr,
                        self_plan && gemv_fused() ? w.ready : nullptr};
            ce = launch_xrows(b->bits, xa, st);
            if (ce != cudaSuccess) return cuda_fail(ce, "k_xrows");
            ra.pdl = 1;
        }
        ce = pre ? launch_plan_from_ids(ra, P, st) : launch_route(ra, P, st);
    }
    if (ce != cudaSuccess) return cuda_fail(ce, pre ? "k_plan_from_ids" : "k_route");
    if (!inline_scatter) {
        KernelTimer kt(b, 1, st);
        const int tt = pre ? kPlanIdsTile : route_tokens_per_cta(t);
        ce = launch_scatter(h, h_dtype == MOQE_F16, t, int(b->d), top_k, b->E, eff_path, gemv_max, tt, P,
                            need_gemm ? w.x_perm : nullptr, b->Kp1, acc, st);
        if (ce != cudaSuccess) return cuda_fail(ce, "k_scatter");
    }
    if (dec_mid) {
        moqe_status s2 = ensure_dec_workspace(b);
        if (s2 != MOQE_OK) return s2;
        KernelTimer kt(b, 2, st);
        ce = launch_dec_prep(b->bits, h, h_dtype == MOQE_F16, t, int(b->d), b->E, b->Kp1, eff_path, gemv_max, P,
                             w.d_units, w.d_nunits, w.d_xperm, b->Kp1 * 2 + 16, st);
        if (ce != cudaSuccess) return cuda_fail(ce, "k_dec_prep");
        DecArgs a{};
        a.h = h;
        a.h_f16 = h_dtype == MOQE_F16;
        a.T = int(t);
        a.d = int(b->d);
        a.E = b->E;
        a.topk = 1;
        a.bits = b->bits;
        a.units = w.d_units;
        a.n_units = w.d_nunits;
        a.perm_token = P.perm_token;
        a.perm_gate = P.perm_gate;
        a.row_of = P.inv_pos;
        a.xperm = w.d_xperm;
        a.xpitch = b->Kp1 * 2 + 16;
        a.Kp1 = b->Kp1;
        a.Np1 = b->Np1;
        a.Np2 = b->Np2;
        a.S = b->Np1 / 64;
        a.wdec = b->wdec;
        a.wdec_stride = b->wdec_stride;
        a.slice_bytes = b->dec_slice;
        a.s1 = b->s1;
        a.b1 = b->b1;
        a.s2 = b->s2;
        a.b2 = b->b2;
        a.acc = w.d_acc;
        a.unit_done = w.d_unit_done;
        a.ybuf = w.d_ybuf;
        a.tok_cnt = w.d_tok_cnt;
        a.out = out;
        a.out_f16 = out_dtype == MOQE_F16;
        a.trace = b->trace;
        a.fused = 0;
        a.plan_ready = 1;
        a.route_cluster = 1;
        ce = launch_dec(b->bits, a, st, b->num_sms);
        if (ce != cudaSuccess) return cuda_fail(ce, "k_dec (mid)");
    } else if (need_gemv) {
        GemvArgs g{h, h_dtype == MOQE_F16, t, int(b->d), int(b->f), top_k, b->E, b->w1, b->w2,
                   b->w1_stride, b->w2_stride, b->s1, b->s2, b->b1, b->b2, b->Kp1, b->Np1, b->Kp2, b->Np2,
                   out, out_dtype == MOQE_F16, acc, w.xr, gemv_chunks(b->Kp1), w.xb, b->smax1, b->bmax1, b->trace, gemv_dbg(), self_plan ? 1 : 0,
                   self_plan && gemv_fused() ? w.ready : nullptr};
        KernelTimer kt(b, 2, st);
        ce = launch_gemv(b->bits, g, P, st, b->num_sms);
        if (ce != cudaSuccess) return cuda_fail(ce, "k_ffn_gemv");
    }
    if (need_gemm) {
        GemmArgs g{w.x_perm, w.mid, b->w1, b->w2, b->w1_stride, b->w2_stride, b->s1, b->s2, b->b1, b->b2,
                   b->Kp1, b->Np1, b->Kp2, b->Np2, w.cap_rows, int(b->d), out, out_dtype == MOQE_F16, acc, b->log};
        {
            KernelTimer kt(b, 3, st);
            ce = launch_gemm(b->bits, 1, g, P, st, b->num_sms);
        }
        if (ce != cudaSuccess) return cuda_fail(ce, "k_ffn_gemm fc1");
        {
            KernelTimer kt(b, 4, st);
            ce = launch_gemm(b->bits, 2, g, P, st, b->num_sms);
        }
        if (ce != cudaSuccess) return cuda_fail(ce, "k_ffn_gemm fc2");
    }
    if (top_k == 2 && out_dtype == MOQE_F16) {
        const int64_t n = t * b->d;
        KernelTimer kt(b, 5, st);
        k_f32_to_f16<<<unsigned((n + 255) / 256), 256, 0, st>>>(acc, static_cast<__half*>(out), n);
        MOQE_CHECK_LAUNCH("k_f32_to_f16");
    }
    return MOQE_OK;
}
}  // namespace

moqe_status moqe_gpu_moe_forward(moqe_bank_t b, const void* h, moqe_dtype h_dtype, int64_t t,
                                 const float* wg, int top_k, void* out, moqe_dtype out_dtype,
                                 int32_t* expert_out, float* gate_out, moqe_path path, void* stream) {
    return forward_impl(b, h, h_dtype, t, wg, top_k, out, out_dtype, expert_out, gate_out, path, stream, nullptr,
                        nullptr);
}

moqe_status moqe_gpu_expert_ffn(moqe_bank_t b, const void* x, moqe_dtype x_dtype, int64_t rows,
                                const int32_t* expert, const float* gate, void* out, moqe_dtype out_dtype,
                                moqe_path path, void* stream) {
    if (!expert || !gate) return fail(MOQE_INVALID_ARGUMENT, "expert_ffn: null expert ids / gates");
    return forward_impl(b, x, x_dtype, rows, nullptr, 1, out, out_dtype, nullptr, nullptr, path, stream, expert,
                        gate);
}

moqe_status moqe_gpu_bank_trace(moqe_bank_t b, int enable) {
    if (!b) return fail(MOQE_INVALID_ARGUMENT, "trace: null bank");
    MOQE_CUDA(cudaDeviceSynchronize());
    cudaFree(b->trace);
    b->trace = nullptr;
    if (enable) {
        const size_t bytes = (size_t(b->num_sms) * kTraceCap * 2 + kTraceRouteCtas * 16) * sizeof(unsigned long long);
        MOQE_CUDA(cudaMalloc(&b->trace, bytes));
        MOQE_CUDA(cudaMemset(b->trace, 0, bytes));
    }
    return MOQE_OK;
}

int64_t moqe_gpu_bank_trace_read(moqe_bank_t b, uint64_t* out, int64_t cap) {
    if (!b || !b->trace) return -1;
    const int64_t n = int64_t(b->num_sms) * kTraceCap * 2 + kTraceRouteCtas * 16;
    if (out) {
        if (cudaDeviceSynchronize() != cudaSuccess) return -1;
        if (cudaMemcpy(out, b->trace, sizeof(uint64_t) * std::min(n, cap), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
        cudaMemset(b->trace, 0, sizeof(uint64_t) * n);
    }
    return n;
}

moqe_status moqe_gpu_bank_span(moqe_bank_t b, int enable) {
    if (!b) return fail(MOQE_INVALID_ARGUMENT, "span: null bank");
    b->span_on = enable != 0;
    return MOQE_OK;
}

moqe_status moqe_gpu_bank_span_read(moqe_bank_t b, double* total_us, int64_t* launches) {
    if (!b) return fail(MOQE_INVALID_ARGUMENT, "span: null bank");
    MOQE_CUDA(cudaDeviceSynchronize());
    DecSpan sp[2];
    MOQE_CUDA(cudaMemcpy(sp, b->spans, sizeof(sp), cudaMemcpyDeviceToHost));
    for (int k = 0; k < 2; ++k) {
        if (total_us) total_us[k] = double(sp[k].total_ns) * 1e-3;
        if (launches) launches[k] = int64_t(sp[k].count);
        sp[k].total_ns = sp[k].count = 0;
        sp[k].start_min = ~0ull;
        sp[k].ticket = 0;
    }
    MOQE_CUDA(cudaMemcpy(b->spans, sp, sizeof(sp), cudaMemcpyHostToDevice));
    return MOQE_OK;
}

moqe_status moqe_gpu_bank_profile(moqe_bank_t b, int enable) {
    if (!b) return fail(MOQE_INVALID_ARGUMENT, "profile: null bank");
    b->prof = enable != 0;
    return MOQE_OK;
}

moqe_status moqe_gpu_bank_profile_read(moqe_bank_t b, double* ms, int64_t* launches, int keep) {
    if (!b) return fail(MOQE_INVALID_ARGUMENT, "profile: null bank");
    MOQE_CUDA(cudaDeviceSynchronize());
    for (auto& ku : b->ev_used) {
        float t = 0.f;
        MOQE_CUDA(cudaEventElapsedTime(&t, b->ev_pool[ku.second].first, b->ev_pool[ku.second].second));
        b->prof_ms[ku.first] += t;
        b->prof_n[ku.first] += 1;
    }
    if (!keep) b->ev_used.clear();
    for (int k = 0; k < MOQE_PROFILE_KINDS; ++k) {
        if (ms) ms[k] = b->prof_ms[k];
        if (launches) launches[k] = b->prof_n[k];
        b->prof_ms[k] = 0;
        b->prof_n[k] = 0;
    }
    return MOQE_OK;
}

moqe_status moqe_gpu_moe_forward_host(moqe_bank_t b, const void* h_host, moqe_dtype h_dtype, int64_t t,
                                      int top_k, void* out_host, moqe_dtype out_dtype, void* stream) {
    if (!b) return fail(MOQE_INVALID_ARGUMENT, "moe_ffn_forward: empty expert bank");
    if (t < 0) return fail(MOQE_INVALID_ARGUMENT, "moe_ffn_forward: negative token count");
    if (t == 0) return MOQE_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t hb = t * b->d * (h_dtype == MOQE_F16 ? 2 : 4);
    const int64_t ob = t * b->d * (out_dtype == MOQE_F16 ? 2 : 4);
    const int64_t need = std::max(hb, ob);
    if (need > b->host_cap) {
        MOQE_CUDA(cudaDeviceSynchronize());
        cudaFree(b->h_dev);
        cudaFree(b->o_dev);
        b->h_dev = b->o_dev = nullptr;
        MOQE_CUDA(cudaMalloc(&b->h_dev, need));
        MOQE_CUDA(cudaMalloc(&b->o_dev, need));
        b->host_cap = need;
    }
    // Pinned (page-locked, mapped) output buffer on the decode path: the kernel's finishers store
    // the rows straight into host memory (posted writes over the host link, overlapped with the
    // kernel's tail), which removes the D2H copy and its launch from the call.
    void* out_dev = nullptr;
    if (b->wg && dec_path_taken(b, t, top_k, MOQE_PATH_AUTO)) {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, out_host) == cudaSuccess && pa.type == cudaMemoryTypeHost)
            out_dev = pa.devicePointer;
        (void)cudaGetLastError();  // pageable memory: not an error, just no direct path
    }
    MOQE_CUDA(cudaMemcpyAsync(b->h_dev, h_host, hb, cudaMemcpyHostToDevice, st));
    moqe_status s = moqe_gpu_moe_forward(b, b->h_dev, h_dtype, t, nullptr, top_k, out_dev ? out_dev : b->o_dev,
                                         out_dtype, nullptr, nullptr, MOQE_PATH_AUTO, st);
    if (s != MOQE_OK) return s;
    if (!out_dev) MOQE_CUDA(cudaMemcpyAsync(out_host, b->o_dev, ob, cudaMemcpyDeviceToHost, st));
    MOQE_CUDA(cudaStreamSynchronize(st));
    return MOQE_OK;
}

moqe_status moqe_gpu_route(const void* h, moqe_dtype h_dtype, int64_t t, int64_t d, const float* wg,
                           int n_experts, int top_k, int32_t* expert, float* gate, void* stream) {
    if (!wg) return fail(MOQE_INVALID_ARGUMENT, "top1_route: no gate weights");
    if (n_experts <= 0 || n_experts > 256) return fail(MOQE_INVALID_ARGUMENT, "route: bad expert count");
    if (top_k != 1 && top_k != 2) return fail(MOQE_INVALID_ARGUMENT, "route: top_k must be 1 or 2");
    if (top_k == 2 && n_experts < 2) return fail(MOQE_INVALID_ARGUMENT, "route: top-2 needs >= 2 experts");
    if (t < 0 || d <= 0) return fail(MOQE_INVALID_ARGUMENT, "matmul: shape mismatch");
    if (t == 0) return MOQE_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int E = n_experts;
    const int64_t R = t * top_k;
    const int64_t nctas = (t + route_tokens_per_cta(t) - 1) / route_tokens_per_cta(t);
    int64_t bytes = 0;
    auto sz = [&](int64_t n) { int64_t r = bytes; bytes += round_up(4 * std::max<int64_t>(n, 1), 256); return r; };
    const int64_t o_lrank = sz(R), o_cta = sz(nctas * E), o_counts = sz(E), o_off = sz(E + 1),
                  o_pt = sz(R), o_pg = sz(R), o_inv = sz(R), o_gl = sz(E), o_ml = sz(E), o_ts = sz(E + 1),
                  o_meta = sz(8), o_tk = sz(8), o_done = sz(E), o_log = sz(t * E), o_gt = sz(4 * (E + 1));
    char* blk = nullptr;
    MOQE_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&blk), bytes, st));
    MOQE_CUDA(cudaMemsetAsync(blk, 0, bytes, st));
    Plan P{};
    P.expert = expert;
    P.gate = gate;
    P.lrank = reinterpret_cast<int32_t*>(blk + o_lrank);
    P.cta_counts = reinterpret_cast<int32_t*>(blk + o_cta);
    P.counts = reinterpret_cast<int32_t*>(blk + o_counts);
    P.offsets = reinterpret_cast<int32_t*>(blk + o_off);
    P.perm_token = reinterpret_cast<int32_t*>(blk + o_pt);
    P.perm_gate = reinterpret_cast<float*>(blk + o_pg);
    P.inv_pos = reinterpret_cast<int32_t*>(blk + o_inv);
    P.gemv_list = reinterpret_cast<int32_t*>(blk + o_gl);
    P.gemm_list = reinterpret_cast<int32_t*>(blk + o_ml);
    P.gemm_tile_start = reinterpret_cast<int32_t*>(blk + o_ts);
    P.meta = reinterpret_cast<int32_t*>(blk + o_meta);
    P.tickets = reinterpret_cast<unsigned*>(blk + o_tk);
    P.done = reinterpret_cast<unsigned*>(blk + o_done);
    P.logits = reinterpret_cast<float*>(blk + o_log);
    P.gtab = reinterpret_cast<int4*>(blk + o_gt);
    RouteArgs ra{h, h_dtype == MOQE_F16, t, int(d), wg, E, top_k, 0, 0, 128, nullptr};
    cudaError_t ce = launch_route(ra, P, st);
    cudaFreeAsync(blk, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "k_route");
    return MOQE_OK;
}

}  // extern "C"
