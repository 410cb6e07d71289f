// gemm.cu -- TP-native attention epilogue: the output
// projection of a tensor-parallel attention layer fused with its
// reduce-scatter over NVLink peer memory.
//
// Rank r holds the heads [r H/G, (r+1) H/G) and the matching rows of the
// output projection W_o, so its contribution is the partial product
//   Y_r = O_r W_r,   O_r [T][K] bf16 (K = H/G * d), W_r [K][N] bf16 (N = hidden)
// and the layer output is Y = sum_r Y_r, reduce-scattered by tokens: rank o
// keeps rows [o T / G, (o+1) T / G).  One persistent tcgen05 kernel computes
// Y_r in 128 x 256 (or 128 x 128) tiles (TMA -> smem ring -> tcgen05.mma, fp32 accumulators
// double-buffered in TMEM) and its epilogue stores every finished row, as
// bf16, straight into the receive slot [r] of the rank owning that row (a
// CUDA-IPC peer window), so the transfer overlaps the GEMM tile by tile.  A
// flag barrier and a small fp32 reduction over the G slots finish the step.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "hg_internal.h"
#include "tc_ptx.cuh"

namespace hg {

namespace {
constexpr int kBM = 128, kBK = 64;
constexpr int kGemmThreads = 192;   // warp 0 TMA, warp 1 MMA + TMEM, warps 2-5 epilogue
constexpr int kATile = kBM * kBK * 2;            // 16 KB, K-major SW128 ([128 rows][64 K])
constexpr int kBChunk = kBK * 64 * 2;            // 8 KB: [64 K rows][64 N cols], N-major SW128
// Tile width BN = 256 (or 128 when N is not a multiple of 256); the smem ring
// takes as many stages as fit.
template <int BN>
struct GemmCfg {
    static constexpr int kBTile = (BN / 64) * kBChunk;
    static constexpr int kStage = kATile + kBTile;
    static constexpr int kStages = BN == 256 ? 4 : 6;
    static constexpr int kBarOff = kStages * kStage;   // barriers: full[S], empty[S], accfull[2], accempty[2]
    static constexpr int kSmem = kBarOff + 256 + 1024;
    static constexpr int kTmemCols = 2 * BN;            // double-buffered fp32 accumulators
};

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeFn)p;
        else
            cudaGetLastError();
    }
    return fn;
}
}  // namespace

struct ProjParams {
    int M, N, K;            // Y_r [M][N] = O_r [M][K] . W_r [K][N]
    int G, rank;
    int rows_max;           // receive slot rows (ceil(M / G))
    uint16_t *dst[kMaxOuts];  // rank o's receive buffer [G][rows_max][N] (G == 1: Y itself, rows_max = M)
};

template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    out_proj_kernel(const ProjParams p, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB) {
    using C = GemmCfg<BN>;
    constexpr int kStages = C::kStages, kStage = C::kStage, kBarOff = C::kBarOff, kBN = BN;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t sbase = (su32(smem_raw) + 1023) & ~1023u;
    const uint32_t bars = sbase + kBarOff;
    uint32_t *tmem_slot = (uint32_t *)(smem_raw + (sbase - su32(smem_raw)) + kBarOff + 128);
    auto full = [&](int s) { return bars + 8u * s; };
    auto empty = [&](int s) { return bars + 8u * (kStages + s); };
    auto accfull = [&](int a) { return bars + 8u * (2 * kStages + a); };
    auto accempty = [&](int a) { return bars + 8u * (2 * kStages + 2 + a); };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int MT = (p.M + kBM - 1) / kBM, NT = p.N / kBN, KB = p.K / kBK;
    const int ntiles = MT * NT;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full(s), 1);
            mbar_init(empty(s), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(accfull(a), 1);
            mbar_init(accempty(a), 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 1) {   // accumulators: tile buffer a at TMEM columns [BN a, BN a + BN)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                     "n"(C::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // tiles in N-column-major order: the CTAs of a wave share W's columns through L2
    if (warp == 0) {
        if (lane == 0) {
            int64_t it = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                const int mt = tile % MT, nt = tile / MT;
                for (int kb = 0; kb < KB; ++kb, ++it) {
                    const int s = (int)(it % kStages);
                    if (it >= kStages) mbar_wait(empty(s), ((it / kStages) - 1) & 1);
                    const uint32_t a = sbase + s * kStage, b = a + kATile;
                    mbar_expect_tx(full(s), kStage);
                    tma_load_2d(a, &tmA, kb * kBK, mt * kBM, full(s));
#pragma unroll
                    for (int c = 0; c < kBN / 64; ++c) tma_load_2d(b + c * kBChunk, &tmB, nt * kBN + c * 64, kb * kBK, full(s));
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_bf16(kBM, kBN, 0, 1);   // A K-major, B N-major
        int64_t it = 0;
        int n = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++n) {
            const int acc = n & 1;
            if (n >= 2) {
                mbar_wait(accempty(acc), ((n >> 1) - 1) & 1);
                tc_fence_after();
            }
            const uint32_t td = tmem + BN * acc;
            for (int kb = 0; kb < KB; ++kb, ++it) {
                const int s = (int)(it % kStages);
                mbar_wait(full(s), (it / kStages) & 1);
                tc_fence_after();
                const uint32_t a = sbase + s * kStage, b = a + kATile;
                const uint64_t da = smem_desc(a, 16, 1024), db = smem_desc(b, kBChunk, 1024);
                if (elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < kBK / 16; ++ks)   // 16 K-elements: 32 B along a SW128 row of A, 16 rows of B
                        umma_bf16(td, da + (uint64_t)((ks * 32) >> 4), db + (uint64_t)((ks * 2048) >> 4), idesc,
                                  (kb > 0 || ks > 0));
                    umma_commit(empty(s));
                    if (kb == KB - 1) umma_commit(accfull(acc));
                }
                __syncwarp();
            }
        }
    } else {
        // epilogue: thread <-> TMEM lane <-> tile row
        const int q = warp & 3;                  // TMEM lane quadrant this warp may access
        const int row = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        int n = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++n) {
            const int mt = tile % MT, nt = tile / MT;
            const int acc = n & 1;
            mbar_wait(accfull(acc), (n >> 1) & 1);
            tc_fence_after();
            const int m = mt * kBM + row;
            // owner rank of row m: shards [o M / G, (o+1) M / G)
            int o = 0;
            while (o + 1 < p.G && ((o + 1) * p.M) / p.G <= m) ++o;
            const int lr = m - (o * p.M) / p.G;
            uint16_t *dst = p.dst[o] + ((int64_t)p.rank * p.rows_max + lr) * p.N + nt * kBN;
#pragma unroll 1
            for (int c = 0; c < kBN / 32; ++c) {
                uint32_t v[32];
                TMEM_LD32(tmem + BN * acc + lane_base + c * 32, v);
                tmem_wait_ld();
                if (m < p.M) {
                    uint4 *d4 = reinterpret_cast<uint4 *>(dst + c * 32);
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        d4[e] = make_uint4(pack2(__uint_as_float(v[8 * e + 0]), __uint_as_float(v[8 * e + 1])),
                                           pack2(__uint_as_float(v[8 * e + 2]), __uint_as_float(v[8 * e + 3])),
                                           pack2(__uint_as_float(v[8 * e + 4]), __uint_as_float(v[8 * e + 5])),
                                           pack2(__uint_as_float(v[8 * e + 6]), __uint_as_float(v[8 * e + 7])));
                }
            }
            tc_fence_before();
            mbar_arrive(accempty(acc));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(C::kTmemCols));
    }
}

// y[lr][n] = sum over the G slots of recv[s][lr][n] (fp32), for this rank's rows
__global__ void rs_reduce_kernel(const uint16_t *__restrict__ recv, uint16_t *__restrict__ y, int rows, int rows_max,
                                 int N, int G) {
    const int64_t total = (int64_t)rows * N / 8;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = (i * 8) / N, c = (i * 8) % N;
        float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int s = 0; s < G; ++s) {
            const uint4 v = *reinterpret_cast<const uint4 *>(recv + ((int64_t)s * rows_max + r) * N + c);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&w[e]));
                a[2 * e] += f.x;
                a[2 * e + 1] += f.y;
            }
        }
        *reinterpret_cast<uint4 *>(y + r * N + c) =
            make_uint4(pack2(a[0], a[1]), pack2(a[2], a[3]), pack2(a[4], a[5]), pack2(a[6], a[7]));
    }
}

hg_status launch_out_proj(const uint16_t *o, const uint16_t *w, int M, int N, int K, int G, int rank, int rows_max,
                          uint16_t *const *dst, void *stream) {
    EncodeFn enc = encode_fn();
    if (!enc) return fail(HG_E_UNSUPPORTED, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap ta, tb;
    {   // A = O [M][K], box [128 rows][64 K]
        cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
        cuuint64_t strides[1] = {(cuuint64_t)K * 2};
        cuuint32_t box[2] = {64, kBM}, es[2] = {1, 1};
        if (enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void *)o, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return fail(HG_E_INVALID, "out-proj: A tensor map (M %d, K %d)", M, K);
    }
    {   // B = W [K][N], box [64 K rows][64 N cols]
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K};
        cuuint64_t strides[1] = {(cuuint64_t)N * 2};
        cuuint32_t box[2] = {64, kBK}, es[2] = {1, 1};
        if (enc(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void *)w, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return fail(HG_E_INVALID, "out-proj: B tensor map (K %d, N %d)", K, N);
    }
    ProjParams p{};
    p.M = M;
    p.N = N;
    p.K = K;
    p.G = G;
    p.rank = rank;
    p.rows_max = rows_max;
    for (int k = 0; k < G; ++k) p.dst[k] = dst[k];
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int mt = (M + kBM - 1) / kBM;
    // 128 x 256 tiles whenever N allows: measured faster than 128 x 128 even where
    // the narrow tiles fill the last wave better (768x8192x8192: 101 vs 112 us)
    const bool wide = N % 256 == 0;
    cudaError_t e;
    if (wide) {
        static bool attr = false;
        if (!attr) {
            e = cudaFuncSetAttribute(out_proj_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     GemmCfg<256>::kSmem);
            if (e != cudaSuccess) return fail(HG_E_CUDA, "out-proj smem attribute: %s", cudaGetErrorString(e));
            attr = true;
        }
        const int tiles = mt * (N / 256);
        out_proj_kernel<256><<<std::min(tiles, sms), kGemmThreads, GemmCfg<256>::kSmem, (cudaStream_t)stream>>>(p, ta, tb);
    } else {
        static bool attr = false;
        if (!attr) {
            e = cudaFuncSetAttribute(out_proj_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     GemmCfg<128>::kSmem);
            if (e != cudaSuccess) return fail(HG_E_CUDA, "out-proj smem attribute: %s", cudaGetErrorString(e));
            attr = true;
        }
        const int tiles = mt * (N / 128);
        out_proj_kernel<128><<<std::min(tiles, sms), kGemmThreads, GemmCfg<128>::kSmem, (cudaStream_t)stream>>>(p, ta, tb);
    }
    e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "out-proj launch: %s", cudaGetErrorString(e));
}

hg_status launch_rs_reduce(const uint16_t *recv, uint16_t *y, int rows, int rows_max, int N, int G, void *stream) {
    if (rows <= 0) return HG_OK;
    const int64_t total = (int64_t)rows * N / 8;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
    rs_reduce_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(recv, y, rows, rows_max, N, G);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "reduce launch: %s", cudaGetErrorString(e));
}

}  // namespace hg
