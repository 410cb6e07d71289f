// tc_attn.cu -- tcgen05 / TMEM / TMA flash-attention tiles for sm_100a.
//
// One CTA computes one TcItem: 128 stacked query rows (token x q-head of one
// GQA group, or the decode rows of every member of a shared-prefix group, the
// Hydragen-style stacking of SURVEY §8(a) a.4) against the keys [k0, k1) of one
// block table, in KV tiles of 128 keys:
//
//   S   = Q K^T        tcgen05.mma kind::f16, M=128 N=128 K=16 x (D/16), A/B from
//                      smem (K-major, 128B swizzle), fp32 accumulator in TMEM
//   P   = exp2(S*c - m) softmax warps: tcgen05.ld S row -> registers, online
//                      max with lazy (threshold 2^8) rescaling, P -> smem bf16
//   O  += P V          tcgen05.mma M=128 N=D K=16 x 8, A=P (K-major), B=V
//                      (MN-major, 128B swizzle), fp32 accumulator in TMEM
//
// K/V tiles are staged by TMA from the paged pool: each 16-token block of one
// KV head is a [16][64] box per 64-column half (2 KB), eight blocks per tile,
// double buffered.  Warp roles (192 threads): warps 0-3 softmax / epilogue
// (thread i <-> TMEM lane i <-> tile row i), warp 4 TMA producer, warp 5 MMA
// issuer + TMEM allocator.  Synchronisation is mbarrier-only.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "hg_internal.h"

struct hg_kv_pool;

namespace hg {

const hg_kv_pool_desc &pool_desc(hg_kv_pool *p);
void *pool_tmap_k(hg_kv_pool *p);
void *pool_tmap_v(hg_kv_pool *p);

// ---------------------------------------------------------------------------
// host: TMA descriptors over the pool, viewed as [N_blk * H_kv * B rows][D]
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
        else
            cudaGetLastError();
    }
    return fn;
}

bool make_tensor_maps(hg_kv_pool *pool) {
    const hg_kv_pool_desc &d = pool_desc(pool);
    if (!tc_supported(d.head_dim)) return false;
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)d.head_dim, (cuuint64_t)d.num_blocks * d.num_kv_heads * d.block_size};
    cuuint64_t strides[1] = {(cuuint64_t)d.head_dim * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)kBlock};
    cuuint32_t estr[2] = {1, 1};
    void *bufs[2] = {d.k_cache, d.v_cache};
    void *maps[2] = {pool_tmap_k(pool), pool_tmap_v(pool)};
    for (int k = 0; k < 2; ++k) {
        CUresult r = enc((CUtensorMap *)maps[k], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, bufs[k], dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return false;
    }
    return true;
}

int tc_supported(int d) { return d == 128 || d == 64; }

// ---------------------------------------------------------------------------
// device helpers (PTX)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void *tmap, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// UMMA shared-memory descriptor (sm_100): start>>4 [0,14), LBO>>4 [16,30),
// SBO>>4 [32,46), version 1 at [46,48), layout type at [61,64) (2 = 128B swizzle).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor, kind::f16: D fp32 (bits 4-5 = 1), A/B bf16 (7-9, 10-12 = 1),
// a_major bit 15, b_major bit 16 (1 = MN-major), N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
                 : "memory");
}

#define TMEM_LD32(taddr, r)                                                                                        \
    asm volatile(                                                                                                  \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"   \
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                                       \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),          \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),    \
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),  \
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])   \
        : "r"(taddr))
#define TMEM_ST32(taddr, r)                                                                                        \
    asm volatile(                                                                                                  \
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"    \
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),                        \
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),        \
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), \
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]),           \
        "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]))
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&v);
}

// ---------------------------------------------------------------------------
// kernel
// ---------------------------------------------------------------------------
constexpr int kTcThreads = 192;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: P values stay <= 2^8 between rescales

template <int D>
struct TcSmem {
    static constexpr int NH = D / 64;                  // 64-column (128 B) halves of a row
    static constexpr int kHalf = kTcRows * 128;        // one [128][64] bf16 half tile = 16 KB
    static constexpr int kQ = NH * kHalf;
    static constexpr int kKV = NH * kHalf;             // one K (or V) tile of 128 keys
    static constexpr int kP = 2 * kHalf;               // P: 128 rows x 128 keys
    static constexpr int oQ = 0;
    static constexpr int oK = oQ + kQ;                 // 2 stages
    static constexpr int oV = oK + 2 * kKV;            // 2 stages
    static constexpr int oP = oV + 2 * kKV;
    static constexpr int oBar = oP + kP;
    static constexpr int kBytes = oBar + 256 + 1024;   // barriers + alignment slack
};

enum { BAR_KFULL = 0, BAR_VFULL = 2, BAR_KVEMPTY = 4, BAR_SFULL = 6, BAR_SFREE = 7, BAR_PFULL = 8, BAR_ODONE = 9,
       BAR_QREADY = 10, BAR_N = 11 };

template <int D>
__global__ void __launch_bounds__(kTcThreads, 1)
tc_attn_kernel(const AttnParams p, const __grid_constant__ CUtensorMap tmap_k,
               const __grid_constant__ CUtensorMap tmap_v) {
    using L = TcSmem<D>;
    constexpr int NH = L::NH;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t sbase = su32(smem);
    const uint32_t sQ = sbase + L::oQ, sK = sbase + L::oK, sV = sbase + L::oV, sP = sbase + L::oP;
    const uint32_t bars = sbase + L::oBar;
    uint32_t *tmem_slot = (uint32_t *)(smem + L::oBar + BAR_N * 8);
    auto bar = [&](int i) { return bars + 8u * i; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const TcItem it = p.tc[blockIdx.x];
    const int nkt = (it.k1 - it.k0 + kTcKeys - 1) / kTcKeys;

    if (threadIdx.x == 0) {
        mbar_init(bar(BAR_KFULL), 1);
        mbar_init(bar(BAR_KFULL + 1), 1);
        mbar_init(bar(BAR_VFULL), 1);
        mbar_init(bar(BAR_VFULL + 1), 1);
        mbar_init(bar(BAR_KVEMPTY), 1);
        mbar_init(bar(BAR_KVEMPTY + 1), 1);
        mbar_init(bar(BAR_SFULL), 1);
        mbar_init(bar(BAR_SFREE), 128);
        mbar_init(bar(BAR_PFULL), 128);
        mbar_init(bar(BAR_ODONE), 1);
        mbar_init(bar(BAR_QREADY), 128);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 5) {  // TMEM: S [0,128) + O [128, 128+D) fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(su32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS = tmem, tO = tmem + 128;

    if (warp == 4) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const int32_t *bt = p.bt_flat + it.bt_off;
            const int kb0 = it.k0 / kBlock;
            const int kb_last = (it.k1 - 1) / kBlock;
            for (int j = 0; j < nkt; ++j) {
                const int s = j & 1;
                if (j >= 2) mbar_wait(bar(BAR_KVEMPTY + s), ((j - 2) >> 1) & 1);
                const uint32_t dk = sK + s * L::kKV, dv = sV + s * L::kKV;
                mbar_expect_tx(bar(BAR_KFULL + s), L::kKV);
#pragma unroll 1
                for (int b = 0; b < 8; ++b) {
                    int kb = kb0 + j * 8 + b;
                    kb = kb <= kb_last ? kb : kb0;  // rows past k1 are masked; keep the data finite
                    const int row = (bt[kb] * p.H_kv + it.g) * kBlock;
#pragma unroll
                    for (int h = 0; h < NH; ++h)
                        tma_load_2d(dk + h * L::kHalf + b * (kBlock * 128), &tmap_k, h * 64, row, bar(BAR_KFULL + s));
                }
                mbar_expect_tx(bar(BAR_VFULL + s), L::kKV);
#pragma unroll 1
                for (int b = 0; b < 8; ++b) {
                    int kb = kb0 + j * 8 + b;
                    kb = kb <= kb_last ? kb : kb0;
                    const int row = (bt[kb] * p.H_kv + it.g) * kBlock;
#pragma unroll
                    for (int h = 0; h < NH; ++h)
                        tma_load_2d(dv + h * L::kHalf + b * (kBlock * 128), &tmap_v, h * 64, row, bar(BAR_VFULL + s));
                }
            }
        }
    } else if (warp == 5) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);  // S = Q K^T: A, B K-major
            constexpr uint32_t idO = idesc_bf16(128, D, 0, 1);    // O += P V: A K-major, B (V) MN-major
            mbar_wait(bar(BAR_QREADY), 0);
            auto issue_qk = [&](int j) {
                const int s = j & 1;
                mbar_wait(bar(BAR_KFULL + s), (j >> 1) & 1);
                if (j > 0) mbar_wait(bar(BAR_SFREE), (j - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int ks = 0; ks < D / 16; ++ks) {
                    const uint32_t off = (ks / 4) * L::kHalf + (ks % 4) * 32;
                    umma_bf16(tS, smem_desc(sQ + off, 16, 1024), smem_desc(sK + s * L::kKV + off, 16, 1024), idS,
                              ks > 0);
                }
                umma_commit(bar(BAR_SFULL));
            };
            issue_qk(0);
            for (int j = 0; j < nkt; ++j) {
                if (j + 1 < nkt) issue_qk(j + 1);
                const int s = j & 1;
                mbar_wait(bar(BAR_PFULL), j & 1);
                mbar_wait(bar(BAR_VFULL + s), (j >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int ks = 0; ks < kTcKeys / 16; ++ks) {
                    const uint32_t aoff = (ks / 4) * L::kHalf + (ks % 4) * 32;   // P: K-major, keys along K
                    const uint32_t boff = ks * 2048;                             // V: 16 keys = 2 x 8-row groups
                    umma_bf16(tO, smem_desc(sP + aoff, 16, 1024), smem_desc(sV + s * L::kKV + boff, L::kHalf, 1024),
                              idO, (j > 0 || ks > 0));
                }
                umma_commit(bar(BAR_KVEMPTY + s));
                umma_commit(bar(BAR_ODONE));
            }
        }
    } else {
        // ===================== softmax / correction / epilogue (warps 0-3) =====================
        const int r = threadIdx.x;  // tile row == TMEM lane
        const bool valid = r < it.nrows;
        struct { int t, h, lim; } row{0, 0, 0};
        if (valid) {
            const int x = it.hl0 + r, j = x / p.G_q;
            row.h = it.g * p.G_q + (x - j * p.G_q);
            if (it.mode == 0) {
                row.t = it.t0 + j;
                row.lim = it.pos0 + j + 1;
            } else {
                row.t = p.tc_tok[it.t0 + j];
                row.lim = it.k1;
            }
        }
        // Q row -> smem, K-major 128B swizzle: half h, row r at h*16K + r*128, chunk c at (c ^ (r&7))*16
        {
            const uint4 *src = reinterpret_cast<const uint4 *>(p.q + ((int64_t)row.t * p.H_q + row.h) * D);
#pragma unroll
            for (int c = 0; c < D / 8; ++c) {
                uint4 v = valid ? src[c] : make_uint4(0, 0, 0, 0);
                const int h = c >> 3, cc = c & 7;
                *reinterpret_cast<uint4 *>(smem + L::oQ + h * L::kHalf + r * 128 + ((cc ^ (r & 7)) << 4)) = v;
            }
            fence_async_smem();
            mbar_arrive(bar(BAR_QREADY));
        }
        const int lim = valid ? row.lim : 0;
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        float m_used = -CUDART_INF_F;  // reference max (log2 domain) of the exponentials
        float l_sum = 0.f;
        for (int j = 0; j < nkt; ++j) {
            mbar_wait(bar(BAR_SFULL), j & 1);
            tc_fence_after();
            uint32_t sr[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) TMEM_LD32(tS + lane_base + c * 32, (&sr[c * 32]));
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(bar(BAR_SFREE));
            const int kbase = it.k0 + j * kTcKeys;
            float mt = -CUDART_INF_F;
#pragma unroll
            for (int c = 0; c < 128; ++c) {
                float x = (kbase + c < lim) ? __uint_as_float(sr[c]) * p.scale_log2 : -CUDART_INF_F;
                sr[c] = __float_as_uint(x);
                mt = fmaxf(mt, x);
            }
            // lazy rescaling: move the reference only when the row max grew by > 2^8
            const bool bump = mt > m_used + kRescaleThreshold;
            float alpha = 1.f;
            if (bump) {
                alpha = (m_used == -CUDART_INF_F) ? 0.f : ex2(m_used - mt);
                m_used = mt;
            }
            const float ref = (m_used == -CUDART_INF_F) ? 0.f : m_used;
            float ls = 0.f;
            uint32_t pk[64];
#pragma unroll
            for (int c = 0; c < 64; ++c) {
                const float a = ex2(__uint_as_float(sr[2 * c]) - ref);
                const float b = ex2(__uint_as_float(sr[2 * c + 1]) - ref);
                ls += a + b;
                pk[c] = pack2(a, b);
            }
            l_sum = l_sum * alpha + ls;
            if (j > 0) {
                mbar_wait(bar(BAR_ODONE), (j - 1) & 1);  // PV_{j-1} done: P smem free, O stable
                tc_fence_after();
            }
            // P row -> smem (K-major 128B swizzle; keys 0-63 in half 0, 64-127 in half 1)
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const int h = c >> 3, cc = c & 7;
                *reinterpret_cast<uint4 *>(smem + L::oP + h * L::kHalf + r * 128 + ((cc ^ (r & 7)) << 4)) =
                    make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
            }
            fence_async_smem();
            if (j > 0 && __any_sync(0xffffffffu, bump)) {
                uint32_t orr[32];
#pragma unroll 1
                for (int c = 0; c < D / 32; ++c) {
                    TMEM_LD32(tO + lane_base + c * 32, orr);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; ++e) orr[e] = __float_as_uint(__uint_as_float(orr[e]) * alpha);
                    TMEM_ST32(tO + lane_base + c * 32, orr);
                }
                tmem_wait_st();
            }
            tc_fence_before();
            mbar_arrive(bar(BAR_PFULL));
        }
        // ---- epilogue ----
        mbar_wait(bar(BAR_ODONE), (nkt - 1) & 1);
        tc_fence_after();
        const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
        const float lse2 = l_sum > 0.f ? m_used + __log2f(l_sum) : -CUDART_INF_F;
        const int G = p.G_q;
        const int base = (valid && it.part >= 0) ? p.comb_base[(int64_t)row.t * p.H_kv + it.g] : -1;
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
            uint32_t orr[32];
            TMEM_LD32(tO + lane_base + c * 32, orr);
            tmem_wait_ld();
            if (!valid) continue;
            if (it.part < 0) {
                uint4 *dst = reinterpret_cast<uint4 *>(p.out + ((int64_t)row.t * p.H_q + row.h) * D + c * 32);
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    dst[e] = make_uint4(pack2(__uint_as_float(orr[8 * e + 0]) * inv, __uint_as_float(orr[8 * e + 1]) * inv),
                                        pack2(__uint_as_float(orr[8 * e + 2]) * inv, __uint_as_float(orr[8 * e + 3]) * inv),
                                        pack2(__uint_as_float(orr[8 * e + 4]) * inv, __uint_as_float(orr[8 * e + 5]) * inv),
                                        pack2(__uint_as_float(orr[8 * e + 6]) * inv, __uint_as_float(orr[8 * e + 7]) * inv));
            } else {
                const int64_t slot = base + (int64_t)it.part * G + (row.h % G);
                float4 *dst = reinterpret_cast<float4 *>(p.part_o + slot * D + c * 32);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    dst[e] = make_float4(__uint_as_float(orr[4 * e]) * inv, __uint_as_float(orr[4 * e + 1]) * inv,
                                         __uint_as_float(orr[4 * e + 2]) * inv, __uint_as_float(orr[4 * e + 3]) * inv);
            }
        }
        if (valid) {
            if (it.part < 0) {
                if (p.lse) p.lse[(int64_t)row.t * p.H_q + row.h] = lse2 * 0.69314718055994531f;
            } else {
                p.part_lse[base + (int64_t)it.part * G + (row.h % G)] = lse2;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
    }
}

template <int D>
static hg_status launch_tc_d(const AttnParams &p, const void *tk, const void *tv, cudaStream_t st) {
    constexpr int bytes = TcSmem<D>::kBytes;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(tc_attn_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return fail(HG_E_CUDA, "tc smem attribute: %s", cudaGetErrorString(e));
        attr = true;
    }
    tc_attn_kernel<D><<<p.n_tc, kTcThreads, bytes, st>>>(p, *(const CUtensorMap *)tk, *(const CUtensorMap *)tv);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "tcgen05 launch: %s", cudaGetErrorString(e));
}

hg_status launch_tc(const AttnParams &p, const void *tk, const void *tv, void *stream) {
    if (p.n_tc == 0) return HG_OK;
    if (p.d == 128) return launch_tc_d<128>(p, tk, tv, (cudaStream_t)stream);
    if (p.d == 64) return launch_tc_d<64>(p, tk, tv, (cudaStream_t)stream);
    return fail(HG_E_UNSUPPORTED, "tcgen05 head_dim %d", p.d);
}

}  // namespace hg
