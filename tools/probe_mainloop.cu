// Micro-probe: the decode GEMV's per-stage compute (Frag<BITS>::load + IMMAs) on resident
// shared memory, no barriers: cycles per 128-k stage per warp, 8 warps per CTA, 1 CTA/SM.
#include "../paper_2310_02410_b200/csrc/ffn_gemv.cu"
// WARPS consumer warps, each BLK m16 blocks (WARPS * BLK * 16 = 128 channels)

namespace moqe_gpu {
template <int BITS, int NT, int WARPS>
__global__ void __launch_bounds__(256, 1) k_probe(int iters, int* out, long long* cyc) {
    constexpr int BLK = 8 / WARPS;
    using Cfg = GemvCfg<BITS>;
    using FR = Frag<BITS>;
    constexpr int F = FR::F, G = FR::G;
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* ring = sm;                      // 8 stages
    uint8_t* bb = sm + 8 * Cfg::SB;          // fragments for 8 stages
    for (int i = threadIdx.x; i < (8 * Cfg::SB + 8 * F * NT * 256) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tq = lane & 3, r0 = 16 * BLK * warp + (lane >> 2);
    int acc[BLK][G][kMaxNT][4] = {};
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll 2
        for (int s = 0; s < 8; ++s) {
            const uint8_t* T0 = ring + s * Cfg::SB;
            uint32_t a[BLK][F][4];
#pragma unroll
            for (int bk = 0; bk < BLK; ++bk) FR::load(T0, T0 + Cfg::TB, r0 + 16 * bk, tq, a[bk]);
            const uint8_t* bs = bb + size_t(s * F) * NT * 256 + lane * 8;
#pragma unroll
            for (int f = 0; f < F; ++f)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    const uint2 b = *reinterpret_cast<const uint2*>(bs + (f * NT + j) * 256);
#pragma unroll
                    for (int bk = 0; bk < BLK; ++bk) imma(acc[bk][FR::grp(f)][j], a[bk][f], b.x, b.y);
                }
        }
    }
    const long long t1 = clock64();
    int s = 0;
    for (int bk = 0; bk < BLK; ++bk) for (int q = 0; q < G; ++q) for (int j = 0; j < NT; ++j) for (int i = 0; i < 4; ++i) s += acc[bk][q][j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
}  // namespace moqe_gpu

using namespace moqe_gpu;
template <int BITS, int NT, int WARPS>
void run(int* o, long long* c) {
    using Cfg = GemvCfg<BITS>;
    const int smem = 8 * Cfg::SB + 8 * Frag<BITS>::F * NT * 256;
    cudaFuncSetAttribute(k_probe<BITS, NT, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 200;
    k_probe<BITS, NT, WARPS><<<148, WARPS * 32, smem>>>(iters, o, c);
    k_probe<BITS, NT, WARPS><<<148, WARPS * 32, smem>>>(iters, o, c);
    long long cy; cudaDeviceSynchronize(); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    const double per_stage = double(cy) / (iters * 8);
    const double bytes_per_cycle = Cfg::SB / per_stage;  // per SM (8 warps cover the 128-channel stage)
    printf("warps=%d int%d NT=%d: %.1f cycles/stage -> %.1f B/cycle/SM = %.0f GB/s chip @1.9GHz\n", WARPS, BITS, NT, per_stage,
           bytes_per_cycle, bytes_per_cycle * 148 * 1.9);
}
int main() {
    int* o; long long* c;
    cudaMalloc(&o, 148 * 256 * 4); cudaMalloc(&c, 8);
    run<2, 1, 8>(o, c); run<3, 1, 8>(o, c); run<3, 2, 8>(o, c);
    run<2, 1, 4>(o, c); run<3, 1, 4>(o, c); run<3, 2, 4>(o, c); run<4, 1, 4>(o, c); run<8, 1, 4>(o, c);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
