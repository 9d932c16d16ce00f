// probe_fadd_chain.cu — cycles per step of a dependent fp32 add chain (the router's
// exact sequential sum): plain FADD, predicated FADD, FMUL+FADD, with/without FTZ.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_fadd_chain tools/probe_fadd_chain.cu
#include <cstdio>
template <int MODE>
__global__ void k(const float* x, const float* w, float* out, long long* cyc, int n) {
    __shared__ float sx[1024], sw[1024];
    for (int i = threadIdx.x; i < n; i += blockDim.x) { sx[i] = x[i]; sw[i] = w[i]; }
    __syncthreads();
    float acc = 0.f;
    long long t0 = clock64();
#pragma unroll 16
    for (int k = 0; k < n; ++k) {
        const float a = sx[k], b = sw[(k + threadIdx.x) & 1023];
        if (MODE == 0) acc = __fadd_rn(acc, b);
        if (MODE == 1) { const float p = __fmul_rn(a, b); acc = __fadd_rn(acc, p); }
        if (MODE == 2) { const float p = __fmul_rn(a, b); if (a != 0.f) acc = __fadd_rn(acc, p); }
        if (MODE == 3) { const float p = a * b; acc = acc + p; }  // (ffma contraction allowed)
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[MODE] = t1 - t0;
}
int main() {
    const int n = 1024;
    float *x, *w, *o; long long* c;
    cudaMalloc(&x, n * 4); cudaMalloc(&w, n * 4); cudaMalloc(&o, 128 * 4); cudaMalloc(&c, 64);
    float hx[n]; for (int i = 0; i < n; ++i) hx[i] = (i % 7) ? 0.5f + i * 1e-3f : 0.f;
    cudaMemcpy(x, hx, n * 4, cudaMemcpyHostToDevice); cudaMemcpy(w, hx, n * 4, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) { k<0><<<1, 32>>>(x, w, o, c, n); k<1><<<1, 32>>>(x, w, o, c, n); k<2><<<1, 32>>>(x, w, o, c, n); k<3><<<1, 32>>>(x, w, o, c, n); }
    long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    const char* nm[4] = {"fadd chain", "fmul+fadd", "fmul+pred fadd (router)", "ffma (contracted)"};
    for (int i = 0; i < 4; ++i) printf("%-26s %.2f cycles/step\n", nm[i], double(h[i]) / n);
    return 0;
}
