// probe_umma_i8.cu — checks the decode tcgen05 building blocks on the GPU:
// kind::i8 MMA (u8 A from TMEM via tcgen05.st, s8 B from smem in the K-major
// no-swizzle canonical layout, s32 D in TMEM), M=128, N=16, K=32, against a CPU
// reference. Tries both readings of the descriptor's LBO/SBO fields.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_umma_i8 tools/probe_umma_i8.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void k_probe(const uint8_t* A, const int8_t* B, int* D, int lbo, int sbo, int n) {
    __shared__ __align__(1024) uint8_t sb[16 * 32];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, m = threadIdx.x;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // B canonical: element (col c, k) at (c/8)*sbo + (k/16)*lbo + (c%8)*16 + k%16
    for (int i = threadIdx.x; i < n * 32; i += blockDim.x) {
        const int c = i / 32, k = i % 32;
        sb[(c / 8) * sbo + (k / 16) * lbo + (c % 8) * 16 + (k % 16)] = uint8_t(B[c * 32 + k]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = s_tmem;
    // A row m: 32 bytes -> TMEM lane m, columns 0..7 (k = 4c + byte)
    uint32_t r[8];
    for (int c = 0; c < 8; ++c) {
        uint32_t w = 0;
        for (int b = 0; b < 4; ++b) w |= uint32_t(A[m * 32 + 4 * c + b]) << (8 * b);
        r[c] = w;
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tm + ((32u * warp) << 16)),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint64_t desc = 0;
        desc |= uint64_t((smem_u32(sb) >> 4) & 0x3FFFu);
        desc |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
        desc |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
        desc |= uint64_t(1) << 46;  // sm_100 descriptor version, no swizzle
        const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 64),
                     "r"(tm), "l"(desc), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    }
    // wait for the MMA
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t v[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(tm + 64 + ((32u * warp) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int c = 0; c < n; ++c) D[m * 16 + c] = int(v[c]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128));
}

int main() {
    const int n = 16;
    std::vector<uint8_t> A(128 * 32);
    std::vector<int8_t> B(16 * 32);
    srand(7);
    for (auto& a : A) a = uint8_t(rand() & 0xff);
    for (auto& b : B) b = int8_t((rand() & 0xff) - 128);
    std::vector<int> ref(128 * 16, 0);
    for (int m = 0; m < 128; ++m)
        for (int c = 0; c < n; ++c) {
            int s = 0;
            for (int k = 0; k < 32; ++k) s += int(A[m * 32 + k]) * int(B[c * 32 + k]);
            ref[m * 16 + c] = s;
        }
    uint8_t* dA;
    int8_t* dB;
    int* dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dD, 128 * 16 * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    const int cfg[2][2] = {{128, 256}, {256, 128}};
    for (auto& c : cfg) {
        cudaMemset(dD, 0, 128 * 16 * 4);
        k_probe<<<1, 128>>>(dA, dB, dD, c[0], c[1], n);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<int> got(128 * 16);
        cudaMemcpy(got.data(), dD, got.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < 128 * 16; ++i) bad += got[i] != ref[i];
        printf("LBO=%d SBO=%d: %s, mismatches %d / %d (got[0]=%d ref[0]=%d got[17]=%d ref[17]=%d)\n", c[0], c[1],
               cudaGetErrorString(e), bad, 128 * 16, got[0], ref[0], got[17], ref[17]);
    }
    return 0;
}
