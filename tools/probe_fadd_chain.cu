// probe_fadd_chain.cu — cycles per step of a dependent fp32 add chain (the router's
// exact sequential sum), operands in registers (no loads in the loop):
// plain FADD, FMUL+FADD, FMUL + predicated FADD (the router), and with 2 chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_fadd_chain tools/probe_fadd_chain.cu
#include <cstdio>
template <int MODE>
__global__ void k(float seed, float* out, long long* cyc, int reps) {
    float x[16], w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { x[i] = (i % 5) ? seed + i * 0.01f : 0.f; w[i] = seed * (i + 1) * 0.003f; }
    float acc = 0.f, acc2 = 0.f;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) acc = __fadd_rn(acc, w[i]);
            if (MODE == 1) { const float p = __fmul_rn(x[i], w[i]); acc = __fadd_rn(acc, p); }
            if (MODE == 2) { const float p = __fmul_rn(x[i], w[i]); if (x[i] != 0.f) acc = __fadd_rn(acc, p); }
            if (MODE == 3) {  // two independent chains (two experts per lane)
                const float p = __fmul_rn(x[i], w[i]), q = __fmul_rn(x[i], w[15 - i]);
                if (x[i] != 0.f) { acc = __fadd_rn(acc, p); acc2 = __fadd_rn(acc2, q); }
            }
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = __fadd_rn(w[i], 1e-7f);  // keep the loop from folding
    }
    long long t1 = clock64();
    out[threadIdx.x] = acc + acc2;
    if (threadIdx.x == 0) cyc[MODE] = t1 - t0;
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 128 * 4); cudaMalloc(&c, 64);
    const int reps = 64;
    for (int rep = 0; rep < 2; ++rep) { k<0><<<1, 32>>>(0.5f, o, c, reps); k<1><<<1, 32>>>(0.5f, o, c, reps); k<2><<<1, 32>>>(0.5f, o, c, reps); k<3><<<1, 32>>>(0.5f, o, c, reps); }
    long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    const char* nm[4] = {"fadd chain", "fmul+fadd", "fmul+pred fadd (router)", "2 chains fmul+pred fadd"};
    for (int i = 0; i < 4; ++i) printf("%-26s %.2f cycles/step (incl. 1 extra FADD per step for w)\n", nm[i], double(h[i]) / (reps * 16));
    return 0;
}
