// probe_alu_rate.cu — issue rate of LOP3 / PRMT / SHF / HFMA2 / IMAD per SM sub-partition on B200
// (16 warps per SM, 8 independent streams per thread).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_alu_rate tools/probe_alu_rate.cu
#include <cstdint>
#include <cstdio>
template <int OP>
__global__ void k(int n, uint32_t* out, long long* cyc) {
    uint32_t v[8];
    for (int j = 0; j < 8; ++j) v[j] = threadIdx.x * 0x9E3779B9u + j;
    const uint32_t m = 0x00070007u ^ threadIdx.x, c = 0x64006400u;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[j]) : "r"(m), "r"(c));
            if (OP == 1) asm volatile("prmt.b32 %0, %0, %1, 0x4140;" : "+r"(v[j]) : "r"(c));
            if (OP == 2) asm volatile("shf.r.wrap.b32 %0, %0, %0, 3;" : "+r"(v[j]));
            if (OP == 3) asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(v[j]) : "r"(m), "r"(c));
            if (OP == 4) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[j]) : "r"(m), "r"(c));
            if (OP == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(v[j]) : "r"(m));
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
    for (int j = 0; j < 8; ++j) s ^= v[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int OP>
void run(const char* name, uint32_t* o, long long* c) {
    const int n = 1024, warps = 16;
    k<OP><<<148, warps * 32>>>(n, o, c);
    k<OP><<<148, warps * 32>>>(n, o, c);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-6s %.2f cycles per warp-instruction per SMSP\n", name, double(h) / (double(n) * 8 * (warps / 4)));
}
int main() {
    uint32_t* o;
    long long* c;
    cudaMalloc(&o, 1 << 22);
    cudaMalloc(&c, 8);
    run<0>("LOP3", o, c);
    run<1>("PRMT", o, c);
    run<2>("SHF", o, c);
    run<3>("HFMA2", o, c);
    run<4>("IMAD", o, c);
    run<5>("IADD", o, c);
    return 0;
}
