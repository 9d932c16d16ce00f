// Micro-probe: TMA weight streaming (copy units of US stages) + the decode IMMA
// mainloop on the landed data, 1 CTA/SM, 8 consumer warps (16 rows each), no
// epilogue, no B traffic beyond a fixed fragment buffer. Reports chip GB/s.
#include <cstdio>
#include "../paper_2310_02410_b200/csrc/frag.cuh"
#include "../paper_2310_02410_b200/csrc/common.cuh"

using namespace moqe_gpu;

template <int BITS, int NT>
__global__ void __launch_bounds__(288, 1) k_sm(const uint8_t* src, int64_t bytes_per_cta, int unit, int nu, int* out) {
    using FR = Frag<BITS>;
    constexpr int F = FR::F, G = FR::G, TB = tile_bytes(BITS), SB = 2 * TB;
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* bb = sm + size_t(nu) * unit;  // fragments: 8 stages
    uint64_t* full = reinterpret_cast<uint64_t*>(bb + 8 * F * NT * 256);
    uint64_t* empty = full + nu;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8 * F * NT * 256 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bb)[i] = i * 2654435761u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nu; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 8); }
        fence_barrier_init();
    }
    __syncthreads();
    const int64_t n = bytes_per_cta / unit;
    const uint8_t* base = src + int64_t(blockIdx.x) * bytes_per_cta;
    if (warp == 8) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int64_t c = 0; c < n; ++c) {
                const int s = int(c % nu);
                if (c >= nu) mbar_wait(&empty[s], int(((c / nu) & 1) ^ 1));
                mbar_arrive_expect_tx(&full[s], unit);
                bulk_g2s_hint(sm + size_t(s) * unit, base + c * unit, unit, &full[s], pol);
            }
        }
        return;
    }
    int acc[G][NT][4] = {};
    const int us = unit / SB;
    for (int64_t c = 0; c < n; ++c) {
        const int s = int(c % nu);
        mbar_wait(&full[s], int((c / nu) & 1));
        const uint8_t* U = sm + size_t(s) * unit;
        for (int st = 0; st < us; ++st) {
            uint32_t a[F][4];
            FR::load(U + st * SB, U + st * SB + TB, 16 * warp + (lane >> 2), lane & 3, a);
            const uint8_t* bs = bb + size_t((int(c * us + st) & 7) * F) * NT * 256 + lane * 8;
#pragma unroll
            for (int f = 0; f < F; ++f)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    const uint2 b = *reinterpret_cast<const uint2*>(bs + (f * NT + j) * 256);
                    imma(acc[FR::grp(f)][j], a[f], b.x, b.y);
                }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    int t = 0;
    for (int q = 0; q < G; ++q) for (int j = 0; j < NT; ++j) for (int i = 0; i < 4; ++i) t += acc[q][j][i];
    if (t == 0x12345678) out[0] = t;
}

template <int BITS, int NT>
void run(const uint8_t* src, int64_t per_cta, int sms, int us, int ring_kb, int* out) {
    const int unit = us * 2 * tile_bytes(BITS);
    const int nu = ring_kb * 1024 / unit;
    const size_t smem = size_t(nu) * unit + 8 * Frag<BITS>::F * NT * 256 + 2 * nu * 8;
    cudaFuncSetAttribute(k_sm<BITS, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int64_t pc = per_cta / unit * unit;
    k_sm<BITS, NT><<<sms, 288, smem>>>(src, pc, unit, nu, out);
    cudaEventRecord(a);
    k_sm<BITS, NT><<<sms, 288, smem>>>(src, pc, unit, nu, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("int%d NT=%d unit %2d stages (%6d B) ring %3d KB: %7.1f GB/s  %s\n", BITS, NT, us, unit, ring_kb,
           double(pc) * sms / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t per_cta = 8ll << 20;
    uint8_t* src; cudaMalloc(&src, per_cta * sms); cudaMemset(src, 0x5a, per_cta * sms);
    int* out; cudaMalloc(&out, 4);
    run<3, 1>(src, per_cta, sms, 1, 96, out);
    run<3, 1>(src, per_cta, sms, 4, 96, out);
    run<3, 1>(src, per_cta, sms, 4, 144, out);
    run<3, 1>(src, per_cta, sms, 8, 144, out);
    run<3, 2>(src, per_cta, sms, 4, 144, out);
    run<2, 1>(src, per_cta, sms, 4, 96, out);
    run<2, 1>(src, per_cta, sms, 8, 144, out);
    run<4, 1>(src, per_cta, sms, 4, 144, out);
    run<8, 1>(src, per_cta, sms, 2, 144, out);
}
