// Microbenchmark: cycles per tcgen05.mma (M=128, K=16, bf16 -> fp32) for operand modes.
// Warp-uniform issue (elect.sync), unrolled, precomputed descriptors.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int amn, int bmn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ bool elect() {
    uint32_t p;
    asm volatile("{.reg .pred P; elect.sync _|P, 0xffffffff; selp.b32 %0, 1, 0, P;}" : "=r"(p));
    return p;
}
template <int MODE>
__global__ void bench(long long *out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    sb = (sb + 1023) & ~1023u;
    for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) ((uint32_t *)sm)[i] = 0;
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
    const uint32_t tm = slot;
    if (MODE == 7 && threadIdx.x >= 32) {   // TMEM traffic from the other warps (softmax-like ld/st)
        const int w = threadIdx.x >> 5;
        const uint32_t ta = tm + 384 + ((uint32_t)(w * 32) << 16);
        uint32_t r[32];
        for (int k = 0; k < iters / 16; ++k) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                           "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                         : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                         :: "r"(ta + 32), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
                            "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
            asm volatile("tcgen05.wait::st.sync.aligned;");
        }
    }
    if (threadIdx.x < 32) {
        const uint64_t dA = desc(sb, 16, 1024, 2);
        const uint64_t dB_k128 = desc(sb + 32768, 16, 1024, 2);
        const uint64_t dB_mn = desc(sb + 32768, 16384, 1024, 2);
        const uint64_t dB_k32 = desc(sb + 32768, 16, 256, 6);
        long long t0 = clock64();
        for (int i = 0; i < iters; i += 8) {
            if (elect()) {
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const uint32_t acc = (i + ks) > 0;
                    if (MODE == 0)  // SS, A K-major SW128, B K-major SW128 (Q K^T)
                        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                                     ::"r"(tm), "l"(dA + (((ks / 4) * 16384 + (ks % 4) * 32) >> 4)), "l"(dB_k128 + (((ks / 4) * 16384 + (ks % 4) * 32) >> 4)), "r"(idesc(128, 128, 0, 0)), "r"(acc));
                    if (MODE == 1)  // TS, B MN-major SW128 (P V, current)
                        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                                     ::"r"(tm + 128), "r"(tm + ks * 8), "l"(dB_mn + ((ks * 2048) >> 4)), "r"(idesc(128, 128, 0, 1)), "r"(acc));
                    if (MODE == 2)  // TS, B K-major SW128
                        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                                     ::"r"(tm + 128), "r"(tm + ks * 8), "l"(dB_k128 + (((ks / 4) * 16384 + (ks % 4) * 32) >> 4)), "r"(idesc(128, 128, 0, 0)), "r"(acc));
                    if (MODE == 3)  // TS, B K-major SW32 (V^T per 16-key block: one block per k-step)
                        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                                     ::"r"(tm + 128), "r"(tm + ks * 8), "l"(dB_k32 + ((ks * 4096) >> 4)), "r"(idesc(128, 128, 0, 0)), "r"(acc));
                    if (MODE == 4)  // SS, A K-major, B MN-major SW128
                        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                                     ::"r"(tm + 256), "l"(dA + (((ks / 4) * 16384 + (ks % 4) * 32) >> 4)), "l"(dB_mn + ((ks * 2048) >> 4)), "r"(idesc(128, 128, 0, 1)), "r"(acc));
                    if (MODE == 6 || MODE == 7) {  // alternate: 8 x QK (SS, K-major B) then 8 x PV (TS, MN-major B)
                        if (((i / 8) & 1) == 0)
                            asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                                         ::"r"(tm + 256), "l"(dA + (((ks / 4) * 16384 + (ks % 4) * 32) >> 4)), "l"(dB_k128 + (((ks / 4) * 16384 + (ks % 4) * 32) >> 4)), "r"(idesc(128, 128, 0, 0)), "r"(acc));
                        else
                            asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                                         ::"r"(tm + 128), "r"(tm + ks * 8), "l"(dB_mn + ((ks * 2048) >> 4)), "r"(idesc(128, 128, 0, 1)), "r"(acc));
                    }
                    if (MODE == 8 || MODE == 9 || MODE == 10) {  // SS, N = 80 / 64 / 96 (narrow KV tiles)
                        constexpr int NN = MODE == 8 ? 80 : MODE == 9 ? 64 : 96;
                        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                                     ::"r"(tm), "l"(dA + (((ks / 4) * 16384 + (ks % 4) * 32) >> 4)), "l"(dB_k128 + (((ks / 4) * 16384 + (ks % 4) * 32) >> 4)), "r"(idesc(128, NN, 0, 0)), "r"(acc));
                    }
                    if (MODE == 5)  // SS, N=256 (both Q tiles' PV in one, if V were the A operand)
                        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                                     ::"r"(tm), "l"(dA + (((ks / 4) * 16384 + (ks % 4) * 32) >> 4)), "l"(dB_k128 + (((ks / 4) * 16384 + (ks % 4) * 32) >> 4)), "r"(idesc(128, 256, 0, 0)), "r"(acc));
                }
            }
            __syncwarp();
        }
        long long t1 = clock64();
        if (elect()) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        }
        __syncwarp();
        asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @!P1 bra W;}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        long long t2 = clock64();
        if (threadIdx.x == 0) {
            out[blockIdx.x * 2] = t1 - t0;
            out[blockIdx.x * 2 + 1] = t2 - t0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
template <int MODE>
void run(const char *name, long long *d) {
    cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    const int iters = 8192;
    bench<MODE><<<148, 128, 100000>>>(d, iters);
    bench<MODE><<<148, 128, 100000>>>(d, iters);
    cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-34s issue %.1f cyc/mma, complete %.1f cyc/mma (%s)\n", name, (double)h[0] / iters, (double)h[1] / iters,
           cudaGetErrorString(cudaGetLastError()));
}
int main() {
    long long *d;
    cudaMalloc(&d, 148 * 2 * 8);
    run<0>("SS A=K128 B=K128 N128 (QK)", d);
    run<1>("TS B=MN128 N128 (PV now)", d);
    run<2>("TS B=K128 N128", d);
    run<3>("TS B=K32 N128 (V^T blocks)", d);
    run<4>("SS B=MN128 N128", d);
    run<5>("SS A=K128 B=K128 N256", d);
    run<8>("SS N80", d);
    run<9>("SS N64", d);
    run<10>("SS N96", d);
    run<6>("alternate 8 QK (SS) / 8 PV (TS)", d);
    run<7>("alternate + TMEM ld/st traffic", d);
    return 0;
}
