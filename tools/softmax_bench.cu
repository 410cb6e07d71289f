// The tcgen05 kernel's per-tile softmax body in isolation (S row in registers, no TMEM):
// cycles per 128-key row per thread, one warp per SMSP (128 threads / CTA, 1 CTA / SM),
// for code-shape variants (template MODE).  Shows what the SMSP sustains on this mix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/softmax_bench tools/softmax_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t f2pack(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void f2unpack(uint64_t v, float &a, float &b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { uint64_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pack2(float lo, float hi) { __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi); return *reinterpret_cast<uint32_t *>(&v); }
__device__ __forceinline__ void exp2_poly2(uint64_t x2, float &a, float &b) {
    float x0, x1;
    f2unpack(x2, x0, x1);
    x2 = f2pack(fmaxf(x0, -126.0f), fmaxf(x1, -126.0f));
    const uint64_t t = fadd2(x2, f2pack(12582912.0f, 12582912.0f));
    const uint64_t r = fadd2(t, f2pack(-12582912.0f, -12582912.0f));
    const uint64_t f = ffma2(r, f2pack(-1.0f, -1.0f), x2);
    uint64_t q = ffma2(f2pack(0.05502927f, 0.05502927f), f, f2pack(0.24225698f, 0.24225698f));
    q = ffma2(q, f, f2pack(0.69325305f, 0.69325305f));
    q = ffma2(q, f, f2pack(0.99995134f, 0.99995134f));
    float q0, q1, t0, t1;
    f2unpack(q, q0, q1);
    f2unpack(t, t0, t1);
    a = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
    b = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

// MODE bits: 1 = 1/4 of the pairs on the polynomial (else all MUFU), 2 = compute the row max,
// 4 = 4 sum accumulators (else 2), 8 = 3/8 polynomial, 16 = half row (64 keys)
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(const float *in, uint32_t *out, float *lsum, int iters, long long *cyc) {
    constexpr int NC = (MODE & 16) ? 32 : 64;   // pairs per row
    uint32_t sr[2 * NC];
    for (int c = 0; c < 2 * NC; ++c) sr[c] = __float_as_uint(in[(threadIdx.x * 7 + c) & 1023]);
    float m_used = 3.0f, l_sum = 0.f;
    const float sc = 0.12f;
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE & 2) {
            float mx[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) mx[e] = __uint_as_float(sr[e]);
#pragma unroll
            for (int c = 8; c < 2 * NC; ++c) mx[c & 7] = fmaxf(mx[c & 7], __uint_as_float(sr[c]));
            const float mt = sc * fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
            if (mt > m_used + 8.f) m_used = mt;
        }
        const uint64_t sc2 = f2pack(sc, sc), nref2 = f2pack(-m_used, -m_used);
        constexpr int NA = (MODE & 4) ? 4 : 2;
        uint64_t ls2[NA];
#pragma unroll
        for (int a = 0; a < NA; ++a) ls2[a] = 0ull;
        uint32_t pk[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const uint64_t x2 = (MODE & 128) ? f2pack(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1]))
                                             : ffma2(f2pack(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), sc2, nref2);
            float a, b;
            const bool poly = (MODE & 8) ? ((0x49 >> (c & 7)) & 1) : ((MODE & 1) && ((0x88 >> (c & 7)) & 1));
            if (poly) {
                exp2_poly2(x2, a, b);
            } else {
                float x0, x1;
                f2unpack(x2, x0, x1);
                a = ex2(x0);
                b = ex2(x1);
            }
            if (!(MODE & 32)) ls2[c % NA] = fadd2(ls2[c % NA], f2pack(a, b));
            if (MODE & 64) pk[c] = __float_as_uint(a) ^ __float_as_uint(b);
            else pk[c] = pack2(a, b);
        }
        float l = 0.f;
#pragma unroll
        for (int a = 0; a < NA; ++a) { float x, y; f2unpack(ls2[a], x, y); l += x + y; }
        l_sum += l;
#pragma unroll
        for (int c = 0; c < NC; ++c) acc ^= pk[c];
        // next "tile": perturb S a little (keeps values live, defeats hoisting)
#pragma unroll
        for (int c = 0; c < 2 * NC; ++c) sr[c] ^= (acc & 1);
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    lsum[blockIdx.x * blockDim.x + threadIdx.x] = l_sum + m_used;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void run(const char *name, float *in, uint32_t *out, float *ls, long long *cyc, int threads = 128) {
    const int iters = 512;
    long long h;
    for (int rep = 0; rep < 2; ++rep) k<MODE><<<148, threads>>>(in, out, ls, iters, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const int keys = (MODE & 16) ? 64 : 128;
    printf("%-44s %s: %7.1f cycles per %d-key row per warp (%d threads/CTA)\n", name, cudaGetErrorString(e),
           (double)h / iters, keys, threads);
}

int main() {
    float *in;
    uint32_t *out;
    float *ls;
    long long *cyc;
    cudaMalloc(&in, 4096 * 4);
    cudaMemset(in, 0, 4096 * 4);
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&ls, 148 * 1024 * 4);
    cudaMalloc(&cyc, 8);
    run<32>("all MUFU, no max, no row sum", in, out, ls, cyc);
    run<64>("all MUFU, no max, no bf16 pack", in, out, ls, cyc);
    run<96>("all MUFU, no max, no sum, no pack", in, out, ls, cyc);
    run<224>("MUFU only (no scale FFMA2, sum, pack)", in, out, ls, cyc);
    run<33>("1/4 poly, no max, no row sum", in, out, ls, cyc);
    run<35>("1/4 poly + max, no row sum", in, out, ls, cyc);
#ifndef ONLY_HALF
    run<0>("all MUFU, no max", in, out, ls, cyc);
    run<1>("1/4 poly, no max", in, out, ls, cyc);
    run<3>("1/4 poly + max (kernel's mix)", in, out, ls, cyc);
    run<2>("all MUFU + max", in, out, ls, cyc);
    run<7>("1/4 poly + max, 4 sum accumulators", in, out, ls, cyc);
    run<10>("3/8 poly + max", in, out, ls, cyc);
    run<3>("1/4 poly + max, 2 warps per SMSP", in, out, ls, cyc, 256);
    run<0>("all MUFU, no max, 2 warps per SMSP", in, out, ls, cyc, 256);
#endif
    run<19>("half row: 1/4 poly + max", in, out, ls, cyc);
    run<19>("half row: 1/4 poly + max, 2 warps per SMSP", in, out, ls, cyc, 256);
    return 0;
}
