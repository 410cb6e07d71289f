// Per-SM issue throughput of the softmax's instruction mix on sm_100a (thread-instructions
// per clock per SM): MUFU.EX2, F2FP (bf16x2 pack), FFMA2 / FADD2 (f32x2), FMNMX3, and the
// per-pair pattern of the tcgen05 softmax (FFMA2 + 2 EX2 + FADD2 + F2FP).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_bench tools/pipe_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }

template <int MODE>
__global__ void k(float *out, int iters, long long *cyc) {
    float f[8];
    uint64_t d[8];
    uint32_t u[8];
    for (int i = 0; i < 8; ++i) {
        f[i] = -0.001f * (threadIdx.x + i);
        d[i] = pk(f[i], f[i] * 0.5f);
        u[i] = i;
    }
    const uint64_t c2 = pk(0.999f, 0.998f), a2 = pk(-0.001f, 0.002f);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
            if (MODE == 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "+r"(u[i]) : "f"(f[i]), "f"(f[(i + 1) & 7]));
            if (MODE == 2) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(d[i]) : "l"(c2), "l"(a2));
            if (MODE == 3) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(d[i]) : "l"(a2));
            if (MODE == 4) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(f[(i + 1) & 7]), "f"(f[(i + 2) & 7]));
            if (MODE == 5) {   // softmax pair: x2 = s2*c + a; e0 = ex2(x.lo); e1 = ex2(x.hi); sum += (e0,e1); pack
                uint64_t x;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(x) : "l"(d[i]), "l"(c2), "l"(a2));
                float x0, x1;
                asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(x0), "=f"(x1) : "l"(x));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
                uint64_t e = pk(x0, x1);
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(d[(i + 4) & 7]) : "l"(e));
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "+r"(u[i]) : "f"(x1), "f"(x0));
            }
            if (MODE == 6) {   // the same without the pack
                uint64_t x;
                asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(x) : "l"(d[i]), "l"(c2), "l"(a2));
                float x0, x1;
                asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(x0), "=f"(x1) : "l"(x));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
                uint64_t e = pk(x0, x1);
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(d[(i + 4) & 7]) : "l"(e));
            }
            if (MODE == 7) {   // ex2 + pack only
                float x0 = f[i], x1 = f[(i + 3) & 7];
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "+r"(u[i]) : "f"(x1), "f"(x0));
                f[i] = x0 * 0.5f;
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += f[i] + __uint_as_float(u[i]) + __uint_as_float((uint32_t)d[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void run(const char *name, int per_iter, float *out, long long *cyc) {
    const int iters = 2048;
    for (int threads : {128, 256, 512}) {
        long long h;
        for (int rep = 0; rep < 2; ++rep) k<MODE><<<148, threads>>>(out, iters, cyc);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        const double units = (double)threads * iters * 8;   // per SM
        printf("%-28s threads/SM %4d: %6.2f units/clk/SM  (%d instr per unit)\n", name, threads, units / h, per_iter);
    }
}

int main() {
    float *out;
    long long *cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 8);
    run<0>("ex2.f32 (values)", 1, out, cyc);
    run<1>("cvt bf16x2 pack", 1, out, cyc);
    run<2>("fma.f32x2 (pairs)", 1, out, cyc);
    run<3>("add.f32x2 (pairs)", 1, out, cyc);
    run<4>("max3.f32", 1, out, cyc);
    run<5>("softmax pair (pairs)", 5, out, cyc);
    run<6>("softmax pair, no pack", 4, out, cyc);
    run<7>("2 ex2 + pack (pairs)", 3, out, cyc);
    return 0;
}
