// probe_hmma_rate.cu — mma.sync.m16n8k16 f16 x f16 -> f32 throughput on B200: cycles per HMMA
// per SM sub-partition for W warps per SMSP, 8 independent accumulators per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_hmma_rate tools/probe_hmma_rate.cu
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ void hmma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__global__ void k(int n, float* out, long long* cyc) {
    float acc[8][4] = {};
    uint32_t a = 0x3c003c00u ^ (threadIdx.x & 7), b = 0x3c003c00u;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) hmma(acc[j], a + j, a ^ j, a + 2 * j, a ^ (3 * j), b + j, b ^ j);
    }
    long long t1 = clock64();
    float s = 0;
    for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1] + acc[j][2] + acc[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    float* o;
    long long* c;
    cudaMalloc(&o, 1 << 20);
    cudaMalloc(&c, 8);
    const int n = 256;
    for (int warps : {4, 8, 16, 32}) {
        k<<<148, warps * 32>>>(n, o, c);
        k<<<148, warps * 32>>>(n, o, c);
        long long h;
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        const double per_smsp = double(n) * 8 * (warps / 4);
        printf("%2d warps/SM (%d per SMSP): %.1f cycles per HMMA.16816 per SMSP  (%.0f fp16 MAC/clk/SM)\n", warps,
               warps / 4, double(h) / per_smsp, 4 * 2048.0 * per_smsp / double(h));
    }
    return 0;
}
