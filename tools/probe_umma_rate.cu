// probe_umma_rate.cu — issue rate of tcgen05.mma.kind::i8 (and kind::f16 for
// reference), M = 128, for several N, A from TMEM (ts) or smem (ss), with
// independent vs. chained accumulators. One CTA; cycles per MMA from clock64
// around NMMA back-to-back issues + commit wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/probe_umma_rate tools/probe_umma_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
    return uint64_t((a >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) | (uint64_t((sbo >> 4) & 0x3FFFu) << 32) |
           (uint64_t(1) << 46);
}

template <int KIND, bool TS>  // KIND 0 = i8, 1 = f16
__global__ void k_rate(int n, int nd, int nmma, long long* out) {
    __shared__ __align__(1024) uint8_t sa[128 * 64];
    __shared__ __align__(1024) uint8_t sb[256 * 64];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) sa[i] = uint8_t(i * 7);
    for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) sb[i] = uint8_t(i * 3);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = s_tmem;
    if (threadIdx.x == 0) {
        const uint32_t idesc = KIND == 0 ? ((2u << 4) | (1u << 10) | (uint32_t(n >> 3) << 17) | (8u << 24))
                                         : ((1u << 4) | (uint32_t(n >> 3) << 17) | (8u << 24));
        const uint64_t bd = desc(smem_u32(sb), 128, 256);
        const uint64_t ad = desc(smem_u32(sa), 128, 256);
        long long t0 = clock64();
        for (int i = 0; i < nmma; ++i) {
            const uint32_t d = tm + 256 + (i % nd) * 32;  // nd independent accumulators
            if (TS) {
                if (KIND == 0)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                                 ::"r"(d), "r"(tm), "l"(bd), "r"(idesc), "r"(1));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                                 ::"r"(d), "r"(tm), "l"(bd), "r"(idesc), "r"(1));
            } else {
                if (KIND == 0)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
            }
        }
        long long t1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
        long long t2 = clock64();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

template <int KIND, bool TS>
void run(const char* name, int n, int nd) {
    long long* d;
    cudaMalloc(&d, 16);
    const int nmma = 512;
    k_rate<KIND, TS><<<1, 128>>>(n, nd, nmma, d);  // warm
    k_rate<KIND, TS><<<1, 128>>>(n, nd, nmma, d);
    long long h[2];
    cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-10s N=%3d indep=%d: issue %.1f cyc/mma, complete %.1f cyc/mma  (%s)\n", name, n, nd, double(h[0]) / nmma,
           double(h[1]) / nmma, cudaGetErrorString(e));
    cudaFree(d);
}


// whole warp runs the loop (operands warp-uniform); elect.sync picks the issuing lane
__global__ void k_rate_warp(int n, int nd, int nmma, long long* out) {
    __shared__ __align__(1024) uint8_t sb[256 * 64];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) sb[i] = uint8_t(i * 3);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = s_tmem;
    if (warp == 0) {
        const uint32_t idesc = (2u << 4) | (1u << 10) | (uint32_t(n >> 3) << 17) | (8u << 24);
        const uint64_t bd = desc(smem_u32(sb), 128, 256);
        long long t0 = clock64();
        for (int i = 0; i < nmma; ++i) {
            const uint32_t d = tm + 256 + (i % nd) * 32;
            asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                         "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                         ::"r"(d), "r"(tm), "l"(bd), "r"(idesc), "r"(1));
        }
        long long t1 = clock64();
        if ((threadIdx.x & 31) == 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
        long long t2 = clock64();
        if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}
void run_warp(int n, int nd) {
    long long* d;
    cudaMalloc(&d, 16);
    const int nmma = 512;
    k_rate_warp<<<1, 128>>>(n, nd, nmma, d);
    k_rate_warp<<<1, 128>>>(n, nd, nmma, d);
    long long h[2];
    cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("i8 ts warp N=%3d indep=%d: issue %.1f cyc/mma, complete %.1f cyc/mma  (%s)\\n", n, nd, double(h[0]) / nmma,
           double(h[1]) / nmma, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    for (int n : {8, 16, 64, 256}) run_warp(n, n <= 16 ? 8 : n == 64 ? 4 : 1);
    for (int n : {8, 16, 64, 256}) {
        const int nd = n <= 16 ? 8 : n == 64 ? 4 : 1;
        run<0, true>("i8 ts", n, nd);
        run<0, false>("i8 ss", n, nd);
        run<1, true>("f16 ts", n, nd);
        run<1, false>("f16 ss", n, nd);
    }
    run<0, true>("i8 ts", 8, 1);
    run<0, false>("i8 ss", 8, 1);
    return 0;
}
