// ep.cu — expert-parallel dispatch / combine (BASELINE config 4).
//
// The reference is single-process; its layer gathers the rows routed to each
// expert in ascending token order (proj/src/model.cpp:360-364) and scatters the gate-weighted
// results back (model.cpp:387-390). Sharded over G ranks, the same two steps become:
//   dispatch: (token, slot) assignments ordered by owner rank, stable in flat order t*k+s,
//             packed as [row fp16 | owner-local expert id i32 | gate f32] records (the
//             all_to_all payload) + per-rank send counts + each assignment's record position;
//   combine:  out[t] = 0 + back[pos(t,0)] (+ back[pos(t,1)]), slot order, fp32.
// These replace torch.sort / bincount / index_select / index_add_ in ep.py on the GPU path.
//
// k_ep_plan is one CTA: per 1024-assignment chunk, a ballot rank per owner rank gives each
// assignment its rank inside its destination (stable), the chunk's per-rank totals advance
// running bases; a second pass adds the exclusive offsets of the destinations. Assignments
// are T*k <= a few 10^4, so one CTA is a few us and needs no grid-wide sync.
#include <cuda_fp16.h>

#include "kernels.cuh"

namespace moqe_gpu {

namespace {
constexpr int kEpThreads = 1024;
constexpr int kEpWarps = kEpThreads / 32;
constexpr int kEpMaxWorld = 32;

__global__ void __launch_bounds__(kEpThreads) k_ep_plan(const int32_t* __restrict__ expert, int64_t n,
                                                        int per, int world, int32_t* __restrict__ pos,
                                                        int64_t* __restrict__ send_counts,
                                                        int32_t* __restrict__ err) {
    __shared__ int wcnt[kEpMaxWorld][kEpWarps];
    __shared__ int base[kEpMaxWorld];
    const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
    const unsigned lt = (1u << l) - 1u;
    if (tid < kEpMaxWorld) base[tid] = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < n; c0 += kEpThreads) {
        const int64_t i = c0 + tid;
        int g = -1;
        if (i < n) {
            const int e = expert[i];
            g = e / per;
            if (e < 0 || g >= world) {
                atomicExch(err, 1);
                g = -1;
            }
        }
        int rank = 0;
        for (int r = 0; r < world; ++r) {
            const unsigned b = __ballot_sync(0xffffffffu, g == r);
            if (g == r) rank = __popc(b & lt);
            if (l == 0) wcnt[r][w] = __popc(b);
        }
        __syncthreads();
        // warp r: exclusive scan of destination r's per-warp counts (in place) + its total
        if (w < world) {
            const int v = wcnt[w][l];
            int s = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, s, o);
                if (l >= o) s += u;
            }
            wcnt[w][l] = s - v + base[w];
            __syncwarp();
            if (l == 31) base[w] += s;
        }
        __syncthreads();
        if (g >= 0) pos[i] = wcnt[g][w] + rank;
        __syncthreads();
    }
    // exclusive offsets of the destinations (rank order)
    __shared__ int off[kEpMaxWorld];
    if (tid == 0) {
        int s = 0;
        for (int r = 0; r < world; ++r) {
            off[r] = s;
            s += base[r];
            send_counts[r] = base[r];
        }
    }
    __syncthreads();
    for (int64_t i = tid; i < n; i += kEpThreads) {
        const int e = expert[i];
        const int g = e / per;
        if (e >= 0 && g < world) pos[i] += off[g];
    }
}

// one warp per assignment: the token row (8-byte copies when d % 4 == 0) + metadata
__global__ void k_ep_pack(const __half* __restrict__ h, const int32_t* __restrict__ expert,
                          const float* __restrict__ gate, const int32_t* __restrict__ pos, int64_t n, int k,
                          int d, int per, int world, __half* __restrict__ rec) {
    const int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int l = threadIdx.x & 31;
    if (i >= n) return;
    const int64_t t = i / k;
    const int e = expert[i];
    if (e < 0 || e / per >= world) return;  // flagged by k_ep_plan
    __half* dst = rec + int64_t(pos[i]) * (d + 4);
    const __half* src = h + t * d;
    if ((d & 3) == 0) {  // record stride (d + 4) * 2 bytes: 8-byte aligned, not 16
        const int nv = d >> 2;
        for (int j = l; j < nv; j += 32)
            reinterpret_cast<uint2*>(dst)[j] = __ldg(reinterpret_cast<const uint2*>(src) + j);
    } else {
        for (int j = l; j < d; j += 32) dst[j] = src[j];
    }
    if (l == 0) {
        int32_t* meta = reinterpret_cast<int32_t*>(dst + d);  // d + 4 fp16 slots: 4-byte aligned (d even)
        meta[0] = e % per;
        meta[1] = __float_as_int(gate[i]);
    }
}

// 4 channels per thread when d % 4 == 0 (8-byte f16 / 16-byte f32 loads, 16-byte stores)
template <bool kF16, int V>
__global__ void k_ep_combine(const void* __restrict__ back, const int32_t* __restrict__ pos, int64_t t, int k,
                             int d, float* __restrict__ out) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int dv = d / V;
    if (idx >= t * dv) return;
    const int64_t tok = idx / dv;
    const int c = int(idx - tok * dv) * V;
    float s[V];
#pragma unroll
    for (int v = 0; v < V; ++v) s[v] = 0.0f;  // index_add_ onto zeros: 0 + a (+ b), slot order
    for (int j = 0; j < k; ++j) {
        const int64_t r = __ldg(pos + tok * k + j);
        if constexpr (V == 4) {
            if constexpr (kF16) {
                const uint2 q = __ldg(reinterpret_cast<const uint2*>(static_cast<const __half*>(back) + r * d + c));
                const float2 lo = __half22float2(*reinterpret_cast<const __half2*>(&q.x));
                const float2 hi = __half22float2(*reinterpret_cast<const __half2*>(&q.y));
                s[0] += lo.x; s[1] += lo.y; s[2] += hi.x; s[3] += hi.y;
            } else {
                const float4 q = __ldg(reinterpret_cast<const float4*>(static_cast<const float*>(back) + r * d + c));
                s[0] += q.x; s[1] += q.y; s[2] += q.z; s[3] += q.w;
            }
        } else {
            if constexpr (kF16)
                s[0] += __half2float(static_cast<const __half*>(back)[r * d + c]);
            else
                s[0] += static_cast<const float*>(back)[r * d + c];
        }
    }
    if constexpr (V == 4)
        __stcs(reinterpret_cast<float4*>(out + tok * d + c), make_float4(s[0], s[1], s[2], s[3]));
    else
        out[tok * d + c] = s[0];
}
}  // namespace

}  // namespace moqe_gpu

using namespace moqe_gpu;

extern "C" moqe_status moqe_gpu_ep_dispatch(const void* h, int64_t t, int64_t d, const int32_t* expert,
                                            const float* gate, int top_k, int n_experts, int world,
                                            void* records, int32_t* pos, int64_t* send_counts,
                                            int32_t* err, void* stream) {
    if (t < 0 || d <= 0 || (d & 1) || top_k < 1 || top_k > 2)
        return fail(MOQE_INVALID_ARGUMENT, "ep_dispatch: bad shape (d even, top_k 1 or 2)");
    if (world < 1 || world > kEpMaxWorld || n_experts < world || n_experts % world)
        return fail(MOQE_INVALID_ARGUMENT, "ep_dispatch: experts must shard evenly over 1..32 ranks");
    if (!send_counts || !err || (t > 0 && (!h || !expert || !gate || !records || !pos)))
        return fail(MOQE_INVALID_ARGUMENT, "ep_dispatch: null buffer");
    if (t * top_k > 0x7fffffff || d > 0x7fffffff) return fail(MOQE_INVALID_ARGUMENT, "ep_dispatch: too large");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t n = t * top_k;
    const int per = n_experts / world;
    cudaMemsetAsync(err, 0, sizeof(int32_t), st);
    k_ep_plan<<<1, kEpThreads, 0, st>>>(expert, n, per, world, pos, send_counts, err);
    MOQE_CHECK_LAUNCH("k_ep_plan");
    if (n == 0) return MOQE_OK;
    const int64_t warps = n, per_cta = 8;
    k_ep_pack<<<unsigned((warps + per_cta - 1) / per_cta), unsigned(per_cta * 32), 0, st>>>(
        static_cast<const __half*>(h), expert, gate, pos, n, top_k, int(d), per, world, static_cast<__half*>(records));
    MOQE_CHECK_LAUNCH("k_ep_pack");
    return MOQE_OK;
}

extern "C" moqe_status moqe_gpu_ep_combine(const void* back, moqe_dtype back_dtype, const int32_t* pos, int64_t t,
                                           int top_k, int64_t d, float* out, void* stream) {
    if (t < 0 || d <= 0 || top_k < 1 || top_k > 2) return fail(MOQE_INVALID_ARGUMENT, "ep_combine: bad shape");
    if (back_dtype != MOQE_F32 && back_dtype != MOQE_F16) return fail(MOQE_INVALID_ARGUMENT, "ep_combine: bad dtype");
    if (t == 0) return MOQE_OK;
    if (!back || !pos || !out) return fail(MOQE_INVALID_ARGUMENT, "ep_combine: null buffer");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool v4 = (d & 3) == 0;
    const int64_t total = v4 ? t * (d / 4) : t * d;
    const unsigned blocks = unsigned((total + 255) / 256);
    if (back_dtype == MOQE_F16) {
        if (v4) k_ep_combine<true, 4><<<blocks, 256, 0, st>>>(back, pos, t, top_k, int(d), out);
        else k_ep_combine<true, 1><<<blocks, 256, 0, st>>>(back, pos, t, top_k, int(d), out);
    } else {
        if (v4) k_ep_combine<false, 4><<<blocks, 256, 0, st>>>(back, pos, t, top_k, int(d), out);
        else k_ep_combine<false, 1><<<blocks, 256, 0, st>>>(back, pos, t, top_k, int(d), out);
    }
    MOQE_CHECK_LAUNCH("k_ep_combine");
    return MOQE_OK;
}
