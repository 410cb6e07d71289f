// Microbenchmark: cycles per tcgen05.mma (M=128, N=128, K=16, bf16 -> fp32) for the
// operand modes the attention kernel uses.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int amn, int bmn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__global__ void bench(long long *out, int mode, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    sb = (sb + 1023) & ~1023u;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t *)sm)[i] = 0;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tm = slot;
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t acc = i > 0;
            if (mode == 0) {        // SS, A K-major, B K-major (QK^T)
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                             ::"r"(tm), "l"(desc(sb + (i & 3) * 32, 16, 1024)), "l"(desc(sb + 32768 + (i & 3) * 32, 16, 1024)), "r"(idesc(128, 128, 0, 0)), "r"(acc));
            } else if (mode == 1) { // TS, A in TMEM, B MN-major (P V)
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                             ::"r"(tm + 128), "r"(tm + (i & 7) * 8), "l"(desc(sb + 32768 + (i & 7) * 2048, 16384, 1024)), "r"(idesc(128, 128, 0, 1)), "r"(acc));
            } else if (mode == 3) { // TS, B MN-major, N-atoms adjacent (LBO 1 KB, SBO 2 KB)
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                             ::"r"(tm + 128), "r"(tm + (i & 7) * 8), "l"(desc(sb + 32768 + (i & 7) * 4096, 1024, 2048)), "r"(idesc(128, 128, 0, 1)), "r"(acc));
            } else if (mode == 4) { // TS, B K-major
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                             ::"r"(tm + 128), "r"(tm + (i & 7) * 8), "l"(desc(sb + 32768 + (i & 3) * 32, 16, 1024)), "r"(idesc(128, 128, 0, 0)), "r"(acc));
            } else if (mode == 5) { // SS, A K-major, B K-major, N=256
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                             ::"r"(tm), "l"(desc(sb + (i & 3) * 32, 16, 1024)), "l"(desc(sb + 32768 + (i & 3) * 32, 16, 1024)), "r"(idesc(128, 256, 0, 0)), "r"(acc));
            } else if (mode == 6) { // TS, B MN-major, N = 64 (one atom)
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                             ::"r"(tm + 128), "r"(tm + (i & 7) * 8), "l"(desc(sb + 32768 + (i & 7) * 2048, 16384, 1024)), "r"(idesc(128, 64, 0, 1)), "r"(acc));
            } else {                // SS, B MN-major
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                             ::"r"(tm + 256), "l"(desc(sb + (i & 3) * 32, 16, 1024)), "l"(desc(sb + 32768 + (i & 7) * 2048, 16384, 1024)), "r"(idesc(128, 128, 0, 1)), "r"(acc));
            }
        }
        long long t1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @!P1 bra W;}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        long long t2 = clock64();
        out[blockIdx.x * 2] = t1 - t0;
        out[blockIdx.x * 2 + 1] = t2 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
    long long *d;
    cudaMalloc(&d, 148 * 2 * 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    const char *names[7] = {"SS K/K (QK)", "TS A=tmem B=MN (PV)", "SS B=MN", "TS B=MN lbo1K sbo2K", "TS B=K-major", "SS K/K N=256", "TS B=MN N=64"};
    for (int mode = 0; mode < 7; ++mode)
        for (int grid : {148}) {
            int iters = 4096;
            bench<<<grid, 128, 100000>>>(d, mode, iters);
            cudaDeviceSynchronize();
            long long h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            printf("%-22s grid %3d: issue %.1f cyc/mma, complete %.1f cyc/mma  (%s)\n", names[mode], grid, (double)h[0] / iters,
                   (double)h[1] / iters, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
