// Cold instruction-fetch cost: a straight-line block of N independent FFMAs run twice in one
// launch (the second pass hits the instruction caches). Prints cycles per instruction per pass.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_icache tools/probe_icache.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__device__ __forceinline__ void block(float (&v)[8], float a, float b) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i & 7] = fmaf(v[i & 7], a, b);
}

template <int N>
__global__ void k(float* out, long long* cyc, float a, float b) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
    long long t[3];
#pragma unroll 1
    for (int p = 0; p < 2; ++p) {
        t[p] = clock64();
        block<N>(v, a, b);
        __syncwarp();
    }
    t[2] = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) {
        cyc[blockIdx.x * 2] = t[1] - t[0];
        cyc[blockIdx.x * 2 + 1] = t[2] - t[1];
    }
}

template <int N>
void run(int warps) {
    float* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 2 * 8);
    long long h[296];
    for (int rep = 0; rep < 3; ++rep) {
        k<N><<<148, warps * 32>>>(out, cyc, 1.0001f, 0.5f);
        cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c0 = 0, c1 = 0;
    for (int i = 0; i < 148; ++i) { c0 += h[2 * i]; c1 += h[2 * i + 1]; }
    printf("N=%5d warps=%2d  pass0 %.2f cyc/instr  pass1 %.2f cyc/instr  (%.0f / %.0f cycles)\n", N, warps,
           c0 / 148 / N, c1 / 148 / N, c0 / 148, c1 / 148);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {1, 4, 16}) {
        run<256>(w);
        run<1024>(w);
        run<4096>(w);
    }
    return 0;
}
