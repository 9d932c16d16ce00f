// Micro-probe: legacy mma.sync throughput on B200 (IMMA u8.s8 m16n8k32 vs HMMA f16 m16n8k16).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

template <int KIND>
__global__ void k_mma(int iters, int* out) {
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55, b1 = a0 ^ 0x33;
    int acc[4][4] = {};
    float facc[4][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (KIND == 0) {
                asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+r"(acc[j][0]), "+r"(acc[j][1]), "+r"(acc[j][2]), "+r"(acc[j][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            } else {
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(facc[j][0]), "+f"(facc[j][1]), "+f"(facc[j][2]), "+f"(facc[j][3])
                             : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            }
        }
    }
    int s = 0;
    for (int j = 0; j < 4; ++j) for (int q = 0; q < 4; ++q) s += acc[j][q] + int(facc[j][q]);
    if (s == 0x12345) out[0] = s;
}

int main() {
    int* d; cudaMalloc(&d, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int kind = 0; kind < 2; ++kind) {
        for (int wps : {4, 8, 16}) {
            const int iters = 4096;
            auto run = [&]() { if (kind == 0) k_mma<0><<<sms, wps * 32>>>(iters, d); else k_mma<1><<<sms, wps * 32>>>(iters, d); };
            run(); cudaDeviceSynchronize();
            cudaEventRecord(a); run(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double n_mma = double(sms) * wps * iters * 4;
            double per_sm_per_us = n_mma / sms / (ms * 1e3);
            double ops = n_mma * (kind == 0 ? 2.0 * 16 * 8 * 32 : 2.0 * 16 * 8 * 16);
            printf("%s warps/SM=%2d: %.3f ms, %.1f mma/SM/us, %.1f T(FL)OPS, %.3f mma/SM/cycle@%dMHz\n",
                   kind == 0 ? "IMMA m16n8k32 u8s8" : "HMMA m16n8k16 f16 ", wps, ms, per_sm_per_us, ops / (ms * 1e-3) / 1e12,
                   per_sm_per_us / (clk / 1000.0), clk / 1000);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
