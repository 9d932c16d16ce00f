// probe_route_loop.cu — the decode router's exact chain loop in isolation: 4 token
// warps (lane = expert), Wg rows [128][32] fp32 in smem, the token row in smem,
// operand blocks of BK rows loaded ahead of the BK-step FMUL + predicated FADD chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_route_loop tools/probe_route_loop.cu
#include <cstdio>
constexpr int BK = 16, E = 32, ROWS = 1024;
__device__ __forceinline__ void ld(const float* hc, const float* wb, int q0, float (&x)[BK], float (&w)[BK]) {
#pragma unroll
    for (int u = 0; u < BK; u += 4) {
        const float4 t4 = *reinterpret_cast<const float4*>(hc + q0 + u);
        x[u] = t4.x; x[u + 1] = t4.y; x[u + 2] = t4.z; x[u + 3] = t4.w;
    }
#pragma unroll
    for (int u = 0; u < BK; ++u) w[u] = wb[(q0 + u) * E];
}
__device__ __forceinline__ void run(float& acc, const float (&x)[BK], const float (&w)[BK]) {
#pragma unroll
    for (int u = 0; u < BK; ++u) {
        const float pr = __fmul_rn(x[u], w[u]);
        if (x[u] != 0.0f) acc = __fadd_rn(acc, pr);
    }
}
template <int V>
__global__ void k(float* out, long long* cyc) {
    extern __shared__ __align__(16) float sm[];
    float* W = sm;                 // [ROWS][32]
    float* H = sm + ROWS * E;      // [4][ROWS]
    for (int i = threadIdx.x; i < ROWS * E + 4 * ROWS; i += blockDim.x) sm[i] = (i % 7) ? 0.001f * (i % 97) : 0.f;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* hc = H + warp * ROWS;
    const float* wb = W + lane;
    float acc = 0.f;
    long long t0 = clock64();
    if (V == 0) {
        float xa[BK], wa[BK], xb[BK], wbk[BK];
        ld(hc, wb, 0, xa, wa);
        for (int q = 0; q + 2 * BK <= ROWS; q += 2 * BK) {
            ld(hc, wb, q + BK, xb, wbk);
            run(acc, xa, wa);
            ld(hc, wb, min(q + 2 * BK, ROWS - BK), xa, wa);
            run(acc, xb, wbk);
        }
    } else if (V == 2) {  // the kernel's structure: 8 chunks of 128 rows, the pipeline restarts per chunk
        for (int c = 0; c < ROWS / 128; ++c) {
            const float* wc = wb + c * 128 * E;
            const float* hcc = hc + c * 128;
            float xa[BK], wa[BK], xb[BK], wbk[BK];
            ld(hcc, wc, 0, xa, wa);
            for (int q = 0; q + 2 * BK <= 128; q += 2 * BK) {
                ld(hcc, wc, q + BK, xb, wbk);
                run(acc, xa, wa);
                ld(hcc, wc, min(q + 2 * BK, 128 - BK), xa, wa);
                run(acc, xb, wbk);
            }
            __syncwarp();
        }
    } else {  // deeper: 4 blocks in flight
        float x0[BK], w0[BK], x1[BK], w1[BK], x2[BK], w2[BK], x3[BK], w3[BK];
        ld(hc, wb, 0, x0, w0); ld(hc, wb, BK, x1, w1); ld(hc, wb, 2 * BK, x2, w2);
        for (int q = 0; q + 4 * BK <= ROWS; q += 4 * BK) {
            ld(hc, wb, min(q + 3 * BK, ROWS - BK), x3, w3);
            run(acc, x0, w0);
            ld(hc, wb, min(q + 4 * BK, ROWS - BK), x0, w0);
            run(acc, x1, w1);
            ld(hc, wb, min(q + 5 * BK, ROWS - BK), x1, w1);
            run(acc, x2, w2);
            ld(hc, wb, min(q + 6 * BK, ROWS - BK), x2, w2);
            run(acc, x3, w3);
        }
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[V] = t1 - t0;
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 1024 * 4); cudaMalloc(&c, 64);
    const int smem = (ROWS * E + 4 * ROWS) * 4;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
        k<0><<<1, 128, smem>>>(o, c); k<1><<<1, 128, smem>>>(o, c); k<2><<<1, 128, smem>>>(o, c);
        k<0><<<1, 32, smem>>>(o, c + 4);
    }
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("ping-pong (router): %.2f cycles/step\n4-deep:             %.2f cycles/step\nchunked (kernel):   %.2f cycles/step\n1 warp ping-pong:   %.2f cycles/step\n",
           double(h[0]) / ROWS, double(h[1]) / ROWS, double(h[2]) / ROWS, double(h[4]) / ROWS);
    return 0;
}
