// Micro-probe: TMA bulk-copy (cp.async.bulk) streaming bandwidth per chip, 1 CTA/SM,
// a smem ring of NST slots; consumer warps only wait/release. Varies copy size,
// ring bytes, number of issuing threads (lanes of the producer warp), cache hint.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#include "../paper_2310_02410_b200/csrc/ptx.cuh"

using namespace moqe_gpu;

__global__ void __launch_bounds__(160, 1) k_stream(const uint8_t* src, int64_t bytes_per_cta, int copy, int nst,
                                                   int issuers, int hint, int* out, unsigned long long* span) {
    if (threadIdx.x == 0 && span) span[2 * blockIdx.x] = gtime_ns();
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(nst) * copy);
    uint64_t* empty = full + nst;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const int64_t n = bytes_per_cta / copy;
    const uint8_t* base = src + int64_t(blockIdx.x) * bytes_per_cta;
    if (warp == 4) {
        const uint64_t pol = policy_evict_first();
        // lane i issues copies i, i + issuers, ... (slot = copy index % nst)
        if (lane < issuers) {
            for (int64_t c = lane; c < n; c += issuers) {
                const int s = int(c % nst);
                const int ph = int((c / nst) & 1);
                if (c >= nst) mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], copy);
                if (hint) bulk_g2s_hint(sm + size_t(s) * copy, base + c * copy, copy, &full[s], pol);
                else bulk_g2s(sm + size_t(s) * copy, base + c * copy, copy, &full[s]);
            }
        }
        return;
    }
    int acc = 0;
    if (warp > 0) return;  // one consumer warp suffices to wait / release (count 4 below)
    for (int64_t c = 0; c < n; ++c) {
        const int s = int(c % nst);
        mbar_wait(&full[s], int((c / nst) & 1));
        acc += sm[size_t(s) * copy + lane];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678) out[0] = acc;
    __syncwarp();
    if (threadIdx.x == 0 && span) span[2 * blockIdx.x + 1] = gtime_ns();
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t per_cta = 8ll << 20;  // 8 MB per CTA -> 1.2 GB total (>> L2)
    uint8_t* src; cudaMalloc(&src, per_cta * sms); cudaMemset(src, 1, per_cta * sms);
    int* out; cudaMalloc(&out, 4);
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    struct Cfg { int copy, ring_kb, issuers, hint; };
    Cfg cfgs[] = {{1536, 128, 1, 1}, {1536, 128, 4, 1}, {4096, 128, 1, 1}, {6144, 120, 1, 1}, {6144, 120, 1, 0},
                  {6144, 120, 4, 1}, {16384, 128, 1, 1}, {16384, 192, 1, 1}, {32768, 192, 1, 1}, {6144, 48, 1, 1},
                  {6144, 192, 2, 1}};
    for (auto c : cfgs) {
        const int nst = c.ring_kb * 1024 / c.copy;
        const size_t smem = size_t(nst) * c.copy + 2 * nst * 8;
        k_stream<<<sms, 160, smem>>>(src, per_cta, c.copy, nst, c.issuers, c.hint, out, nullptr);
        cudaEventRecord(a);
        k_stream<<<sms, 160, smem>>>(src, per_cta, c.copy, nst, c.issuers, c.hint, out, nullptr);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("copy %6d B ring %3d KB (%2d slots) issuers %d hint %d: %7.1f GB/s\n", c.copy, c.ring_kb, nst, c.issuers,
               c.hint, double(per_cta) * sms / (ms * 1e-3) / 1e9);
    }
    // short streams (the decode GEMV's per-CTA volume): in-kernel span (first start .. last end)
    unsigned long long* span; cudaMalloc(&span, sms * 16);
    struct S { int copy, nst, units; };
    S ss[] = {{24576, 6, 7}, {24576, 6, 28}, {24576, 6, 112}, {16384, 8, 10}, {49152, 3, 4}, {24576, 4, 7}};
    for (auto c : ss) {
        const size_t smem = size_t(c.nst) * c.copy + 2 * c.nst * 8;
        const int64_t per = int64_t(c.copy) * c.units;
        for (int rep = 0; rep < 3; ++rep) {
            // rotate the source so every run reads cold data
            k_stream<<<sms, 160, smem>>>(src + int64_t(rep) * per * sms, per, c.copy, c.nst, 1, 1, out, span);
        }
        cudaDeviceSynchronize();
        unsigned long long h[2 * 160];
        cudaMemcpy(h, span, sms * 16, cudaMemcpyDeviceToHost);
        unsigned long long lo = ~0ull, hi = 0; double mean = 0;
        for (int i = 0; i < sms; ++i) { lo = h[2 * i] < lo ? h[2 * i] : lo; hi = h[2 * i + 1] > hi ? h[2 * i + 1] : hi; mean += double(h[2 * i + 1] - h[2 * i]); }
        printf("short: copy %6d x %3d units (%4lld KB/CTA), ring %d: span %.2f us, mean CTA %.2f us -> %.0f GB/s\n", c.copy,
               c.units, (long long)(per >> 10), c.nst, (hi - lo) / 1e3, mean / sms / 1e3, double(per) * sms / double(hi - lo));
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
