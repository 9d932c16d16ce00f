// probe_unit_mma.cu — the decode consumer's compute in isolation: 8 warps, each runs
// the int3 unit loop (LOP3 unpack of 4 stages + IMMA against B words) over smem data,
// NT = 1; cycles per unit per CTA. Variants: the kernel's loop vs. software-pipelined.
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2310_02410_b200/csrc -o tools/probe_unit_mma tools/probe_unit_mma.cu
#include <cstdio>
#include "frag.cuh"
using namespace moqe_gpu;
constexpr int BITS = 3, F = Frag<3>::F, G = Frag<3>::G, US = 4, TB = 3072, SB = 2 * TB;

template <int V>
__global__ void k(int nunits, int* out, long long* cyc) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* U = sm;               // one unit: 4 stages x 2 tiles (24 KB)
    uint8_t* Bw = sm + US * SB;    // B words: 8 stages x F x 32 lanes x 8 B
    for (int i = threadIdx.x; i < (US * SB + 8 * F * 256) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
    const int r0 = 16 * warp + gq;
    const uint8_t* bp = Bw + lane * 8;
    int acc[G][4] = {};
    long long t0 = clock64();
    for (int u = 0; u < nunits; ++u) {
        if (V == 0) {
            uint32_t a[US][F][4];
            uint2 b[US][F];
#pragma unroll
            for (int s = 0; s < US; ++s) {
                Frag<3>::load(U + s * SB, U + s * SB + TB, r0, tq, a[s]);
#pragma unroll
                for (int f = 0; f < F; ++f) b[s][f] = *reinterpret_cast<const uint2*>(bp + (s * F + f) * 256);
            }
#pragma unroll
            for (int s = 0; s < US; ++s)
#pragma unroll
                for (int f = 0; f < F; ++f) imma(acc[Frag<3>::grp(f)], a[s][f], b[s][f].x, b[s][f].y);
        } else {
#pragma unroll 1
            for (int s = 0; s < US; ++s) {
                uint32_t a[F][4];
                Frag<3>::load(U + s * SB, U + s * SB + TB, r0, tq, a);
#pragma unroll
                for (int f = 0; f < F; ++f) {
                    const uint2 b = *reinterpret_cast<const uint2*>(bp + (s * F + f) * 256);
                    imma(acc[Frag<3>::grp(f)], a[f], b.x, b.y);
                }
            }
        }
        asm volatile("" ::: "memory");
    }
    long long t1 = clock64();
    int s = 0;
    for (int g = 0; g < G; ++g) s += acc[g][0] + acc[g][1] + acc[g][2] + acc[g][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    int* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8);
    const int smem = US * SB + 8 * F * 256, n = 256;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int v = 0; v < 2; ++v) {
        for (int rep = 0; rep < 2; ++rep) {
            if (v == 0) k<0><<<148, 256, smem>>>(n, o, c); else k<1><<<148, 256, smem>>>(n, o, c);
        }
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("variant %d: %.0f cycles per unit (4 stages, 128 ch x 512 k, int3, NT=1) = %.3f us at 1.965 GHz; %s\n", v,
               double(h) / n, double(h) / n / 1965.0, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
