// MUFU throughput: ex2.approx.f32 vs ex2.approx.ftz.bf16x2 (values per SM per clock).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mufu_bench tools/mufu_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float *out, int iters, long long *cyc) {
    uint32_t r[8];
    float f[8];
    for (int i = 0; i < 8; ++i) {
        f[i] = -0.001f * (threadIdx.x + i);
        __nv_bfloat162 b = __floats2bfloat162_rn(f[i], f[i] * 0.5f);
        r[i] = *reinterpret_cast<uint32_t *>(&b);
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
            else asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r[i]));
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += f[i] + __uint_as_float(r[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    float *out;
    long long *cyc, h;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 8);
    const int iters = 4096;
    for (int mode = 0; mode < 2; ++mode)
        for (int threads : {128, 256, 512, 1024}) {
            for (int rep = 0; rep < 2; ++rep) {
                if (mode == 0) k<0><<<148, threads>>>(out, iters, cyc);
                else k<1><<<148, threads>>>(out, iters, cyc);
            }
            cudaDeviceSynchronize();
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            double instr = (double)threads * iters * 8;   // thread-instructions per SM
            printf("%s threads/SM %4d: %.2f thread-instr/clk/SM (%.2f values/clk/SM)\n",
                   mode ? "ex2 bf16x2" : "ex2 f32   ", threads, instr / h, instr / h * (mode ? 2 : 1));
        }
    return 0;
}
