// probe_hmma_lat.cu — dependent-chain latency of mma.sync m16n8k16 (f16 -> f32) on B200, and
// the rate of one warp per SMSP running C independent chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_hmma_lat tools/probe_hmma_lat.cu
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ void hmma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int C>
__global__ void k(int n, float* out, long long* cyc) {
    float acc[C][4] = {};
    uint32_t a = 0x3c003c00u ^ (threadIdx.x & 7), b = 0x3c003c00u;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < C; ++j) hmma(acc[j], a + j, a ^ j, a + 2 * j, a ^ (3 * j), b + j, b ^ j);
    }
    long long t1 = clock64();
    float s = 0;
    for (int j = 0; j < C; ++j) s += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int C>
void run(int warps, float* o, long long* c) {
    const int n = 512;
    k<C><<<148, warps * 32>>>(n, o, c);
    k<C><<<148, warps * 32>>>(n, o, c);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%2d warps/SM, %d chains/warp: %.1f cycles per HMMA step per warp\n", warps, C, double(h) / (double(n) * C));
}
int main() {
    float* o;
    long long* c;
    cudaMalloc(&o, 1 << 20);
    cudaMalloc(&c, 8);
    run<1>(1, o, c);
    run<1>(4, o, c);
    run<2>(4, o, c);
    run<4>(4, o, c);
    run<8>(4, o, c);
    run<1>(12, o, c);
    run<2>(12, o, c);
    return 0;
}
