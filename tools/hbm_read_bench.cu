// HBM read ceiling on B200: stream N bytes (>> L2) with (a) 16-byte ld.global.v4
// loads, (b) cp.async.bulk (1-D TMA) of 4 KB chunks into a shared-memory ring
// with mbarriers -- the two ways split-K could fetch (block, head) KV runs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_read_bench tools/hbm_read_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ld_kernel(const uint4 *__restrict__ p, int64_t n16, unsigned *out) {
    uint32_t acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride), d = __ldcs(p + i + 3 * stride);
        acc ^= a.x ^ b.y ^ c.z ^ d.w;
    }
    for (; i < n16; i += stride) acc ^= __ldcs(p + i).x;
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int CHUNK>
__global__ void bulk_kernel(const uint8_t *__restrict__ p, int64_t nchunks, unsigned *out,
                            const int32_t *__restrict__ perm = nullptr) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[STAGES];
    uint8_t *buf = sm;
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    __syncthreads();
    // chunks of this CTA: blockIdx.x, +gridDim.x, ...
    const int64_t first = blockIdx.x, step = gridDim.x;
    const int64_t mine = first < nchunks ? (nchunks - 1 - first) / step + 1 : 0;
    auto issue = [&](int64_t k) {
        const int s = (int)(k % STAGES);
        const uint32_t b = su32(&bar[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(buf + s * CHUNK)),
                     "l"(p + (int64_t)(perm ? perm[first + k * step] : (first + k * step)) * CHUNK), "r"(CHUNK), "r"(b)
                     : "memory");
    };
    uint32_t acc = 0;
    if (threadIdx.x == 0)
        for (int64_t k = 0; k < STAGES - 1 && k < mine; ++k) issue(k);
    for (int64_t k = 0; k < mine; ++k) {
        if (threadIdx.x == 0 && k + STAGES - 1 < mine) issue(k + STAGES - 1);
        const int s = (int)(k % STAGES);
        const uint32_t b = su32(&bar[s]), ph = (uint32_t)((k / STAGES) & 1);
        asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(b), "r"(ph)
                     : "memory");
        acc ^= reinterpret_cast<const uint32_t *>(buf + s * CHUNK)[threadIdx.x];
        __syncthreads();   // slot consumed before it is refilled
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const size_t bytes = 4ull << 30;
    uint8_t *p;
    unsigned *o;
    cudaMalloc(&p, bytes);
    cudaMalloc(&o, 4);
    cudaMemset(p, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 148;
    auto timeit = [&](const char *name, auto launch) {
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r) best = ms < best ? ms : best;
        }
        printf("%-40s %.1f GB/s (%s)\n", name, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    for (int bpsm : {2, 4, 8})
        timeit(bpsm == 2 ? "ld.v4 256thr x 2/SM" : bpsm == 4 ? "ld.v4 256thr x 4/SM" : "ld.v4 256thr x 8/SM",
               [&] { ld_kernel<<<sms * bpsm, 256>>>((const uint4 *)p, bytes / 16, o); });
    constexpr int C = 4096;
    {
        constexpr int S = 8;
        cudaFuncSetAttribute(bulk_kernel<S, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * C);
        timeit("bulk 4KB x 8 stages, 4 CTA/SM", [&] { bulk_kernel<S, C><<<sms * 4, 128, S * C>>>(p, bytes / C, o); });
        timeit("bulk 4KB x 8 stages, 8 CTA/SM", [&] { bulk_kernel<S, C><<<sms * 8, 128, S * C>>>(p, bytes / C, o); });
    }
    {
        constexpr int S = 16;
        cudaFuncSetAttribute(bulk_kernel<S, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * C);
        timeit("bulk 4KB x 16 stages, 2 CTA/SM", [&] { bulk_kernel<S, C><<<sms * 2, 128, S * C>>>(p, bytes / C, o); });
        timeit("bulk 4KB x 16 stages, 3 CTA/SM", [&] { bulk_kernel<S, C><<<sms * 3, 128, S * C>>>(p, bytes / C, o); });
    }
    {   // the paged pool's access pattern: 4 KB (block, head) runs in a random order
        constexpr int S = 8;
        const int64_t n = bytes / C;
        int32_t *hperm = (int32_t *)malloc(n * 4), *dperm;
        for (int64_t i = 0; i < n; ++i) hperm[i] = (int32_t)i;
        uint64_t x = 88172645463325252ull;
        for (int64_t i = n - 1; i > 0; --i) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            const int64_t j = (int64_t)(x % (uint64_t)(i + 1));
            const int32_t t = hperm[i]; hperm[i] = hperm[j]; hperm[j] = t;
        }
        cudaMalloc(&dperm, n * 4);
        cudaMemcpy(dperm, hperm, n * 4, cudaMemcpyHostToDevice);
        timeit("bulk 4KB x 8 stages, 4 CTA/SM, RANDOM", [&] { bulk_kernel<S, C><<<sms * 4, 128, S * C>>>(p, n, o, dperm); });
        timeit("bulk 4KB x 8 stages, 6 CTA/SM, RANDOM", [&] { bulk_kernel<S, C><<<sms * 6, 128, S * C>>>(p, n, o, dperm); });
    }
    {
        constexpr int S = 32;
        cudaFuncSetAttribute(bulk_kernel<S, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * C);
        timeit("bulk 4KB x 32 stages, 1 CTA/SM", [&] { bulk_kernel<S, C><<<sms * 1, 128, S * C>>>(p, bytes / C, o); });
    }
    return 0;
}
