// Micro-probe: latency of a dependent fp32 add chain (the exact router order) on B200.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_chain(const float* __restrict__ w, int n, float* out, long long* cyc) {
    extern __shared__ float s[];
    const int ld = n + 4;  // transposed rows, padded
    for (int i = threadIdx.x; i < 32 * ld + n; i += blockDim.x) s[i] = w[i % 4096];
    __syncthreads();
    const float* hs = s + 32 * ld;
    const float* wt = s + threadIdx.x * ld;
    float acc = 0.f;
    float r0 = w[threadIdx.x], r1 = w[threadIdx.x + 32];
    const long long t0 = clock64();
    if (MODE == 0) {  // register-only dependent chain (FMUL off-chain)
#pragma unroll 16
        for (int k = 0; k < n; ++k) { acc = __fadd_rn(acc, __fmul_rn(r0, r1)); r0 = __fadd_rn(r0, 1.0f); }
    } else if (MODE == 1) {  // transposed Wg + broadcast h, both as LDS.128, predicated skip
#pragma unroll 4
        for (int k = 0; k < n; k += 4) {
            const float4 a = *reinterpret_cast<const float4*>(hs + k);
            const float4 b = *reinterpret_cast<const float4*>(wt + k);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float pr = __fmul_rn(av[u], bv[u]);
                if (av[u] != 0.0f) acc = __fadd_rn(acc, pr);
            }
        }
    } else {  // same, 16-wide register double buffer
        float4 a[4], b[4];
        for (int u = 0; u < 4; ++u) { a[u] = *reinterpret_cast<const float4*>(hs + 4 * u); b[u] = *reinterpret_cast<const float4*>(wt + 4 * u); }
        for (int k = 0; k < n; k += 16) {
            float4 an[4], bn[4];
            const int kn = k + 16 < n ? k + 16 : k;
#pragma unroll
            for (int u = 0; u < 4; ++u) { an[u] = *reinterpret_cast<const float4*>(hs + kn + 4 * u); bn[u] = *reinterpret_cast<const float4*>(wt + kn + 4 * u); }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float av[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, bv[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const float pr = __fmul_rn(av[v], bv[v]);
                    if (av[v] != 0.0f) acc = __fadd_rn(acc, pr);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) { a[u] = an[u]; b[u] = bn[u]; }
        }
    }
    const long long t1 = clock64();
    out[threadIdx.x] = acc + r0;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    const int n = 1024;
    float *w, *o; long long* c;
    cudaMalloc(&w, 4096 * 4); cudaMemset(w, 0x3f, 4096 * 4);
    cudaMalloc(&o, 128 * 4); cudaMalloc(&c, 8);
    const int sm = (32 * (n + 4) + n) * 4;
    cudaFuncSetAttribute(k_chain<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_chain<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_chain<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    const char* nm[3] = {"register chain", "LDS.128 both, unroll 4", "LDS.128 both, 16-wide double buffer"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int it = 0; it < 2; ++it) {
            if (mode == 0) k_chain<0><<<1, 32, sm>>>(w, n, o, c);
            if (mode == 1) k_chain<1><<<1, 32, sm>>>(w, n, o, c);
            if (mode == 2) k_chain<2><<<1, 32, sm>>>(w, n, o, c);
        }
        long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
        printf("mode %d (%s): %lld cycles = %.2f cyc/k\n", mode, nm[mode], cy, double(cy) / n);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
