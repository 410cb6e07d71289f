// tc_attn.cu -- tcgen05 / TMEM / TMA flash-attention tiles for sm_100a.
//
// One CTA computes one TcItem: up to 256 stacked query rows (token x q-head of
// one GQA group, or the decode rows of every member of a shared-prefix group:
// the Hydragen-style stacking of SURVEY §8(a) a.4), as two 128-row Q tiles,
// against the keys [k0, k1) of one block table, in KV tiles of 128 keys:
//
//   S   = Q K^T        tcgen05.mma kind::f16, M=128 N=128 K=16 x (D/16), A/B from
//                      smem (K-major, 128B swizzle), fp32 accumulator in TMEM
//   P   = exp2(S*c - m) softmax warps: tcgen05.ld S row -> registers, online
//                      max with lazy (threshold 2^8) rescaling, exp2 on MUFU with
//                      1/4 on the FMA pipe (polynomial), P -> TMEM (bf16 pairs)
//   O  += P V          tcgen05.mma M=128 N=D K=16 x 8, A=P from TMEM, B=V from
//                      smem (MN-major, 128B swizzle), fp32 accumulator in TMEM
//
// K/V tiles are staged by TMA from the paged pool: each 16-token block of one
// KV head is a [16][64] box per 64-column half (2 KB), eight blocks per tile,
// K in a 3-deep ring and V in a 2-deep ring, shared by both Q tiles.  Warp
// roles (384 threads): warps 0-3 / 4-7 softmax + epilogue of Q tile 0 / 1
// (thread <-> TMEM lane <-> row, setmaxnreg 200), warp 8 the K TMA producer,
// warp 10 the V TMA producer, warp 9 MMA issuer + TMEM allocator (all 512
// columns), warp 11 the fused step's background append (else idle); warps
// 8-11 drop to 104 registers.  Synchronisation is mbarrier-only.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "hg_internal.h"
#include "tc_ptx.cuh"

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
// kernel
// ---------------------------------------------------------------------------
constexpr int kTcThreads = 384;
// Register split between the warpgroups (setmaxnreg; 2 x 128 x SOFTMAX + 128 x WG2 <= 384 x 168,
// the launch allocation).  200 / 104: neither the softmax loop nor the MMA issuer spills.
#ifndef HG_TC_REG_SOFTMAX
#define HG_TC_REG_SOFTMAX 200
#endif
#ifndef HG_TC_REG_WG2
#define HG_TC_REG_WG2 104
#endif
static_assert(2 * 128 * HG_TC_REG_SOFTMAX + 128 * HG_TC_REG_WG2 <= 384 * 168, "register split exceeds the launch allocation");  // WG0/WG1: softmax of Q tile 0/1; WG2: warp 8 TMA, warp 9 MMA, 10-11 idle
constexpr float kRescaleThreshold = 8.0f;  // log2 units: P values stay <= 2^8 between rescales

// 2^x on the FMA/ALU pipes (offloads the MUFU unit): x = n + f, n = rint(x)
// by the 1.5*2^23 magic add, f in [-0.5, 0.5], 2^f by a degree-3 polynomial
// (max rel. error 1.4e-4, far below bf16's 3.9e-3 rounding of P).
__device__ __forceinline__ float exp2_poly(float x) {
    x = fmaxf(x, -126.0f);
    const float t = x + 12582912.0f;
    const float f = x - (t - 12582912.0f);
    const int n = __float_as_int(t) - 0x4B400000;
    float q = fmaf(0.05502927f, f, 0.24225698f);
    q = fmaf(q, f, 0.69325305f);
    q = fmaf(q, f, 0.99995134f);
    return __int_as_float(__float_as_int(q) + (n << 23));
}

// Packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2): two lanes of the softmax per instruction.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float &a, float &b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// Which exp2 pairs (bit c & 7 of the 128-key row's pair index c) go to the FMA-pipe
// polynomial instead of MUFU.EX2: 0x88 = one in four.
#ifndef HG_POLY_MASK
#define HG_POLY_MASK 0x88
#endif

// exp2_poly on a pair: 2 FMNMX + 3 FADD2/FFMA2 + 3 FFMA2 + 2 IMAD for two values.
// The exponent add folds (bits(t) - 0x4B400000) << 23 into bits(t) << 23 (the
// constant vanishes mod 2^32).
__device__ __forceinline__ void exp2_poly2(uint64_t x2, float &a, float &b) {
    float x0, x1;
    f2unpack(x2, x0, x1);
    x2 = f2pack(fmaxf(x0, -126.0f), fmaxf(x1, -126.0f));
    const uint64_t magic = f2pack(12582912.0f, 12582912.0f);
    const uint64_t t = fadd2(x2, magic);
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

// Two 128-row Q tiles per CTA (FA4-style ping-pong) share every K/V tile, so a
// KV byte staged from L2 feeds 256 query rows; P never leaves TMEM: softmax
// overwrites S's first 64 columns with packed bf16 P and PV is a TS-MMA (A from
// TMEM).  tcgen05 ops issued by one thread complete in order and a commit
// covers all prior ops, so "S(j+1) full" also means "PV(j) done": the S-free
// and O-stable handshakes of a one-tile design disappear.
template <int D>
struct TcSmem {
    static constexpr int NH = D / 64;                  // 64-column (128 B) halves of a row
    static constexpr int kHalf = kTcRows * 128;        // one [128][64] bf16 half tile = 16 KB
    static constexpr int kQ = NH * kHalf;              // one 128-row Q tile
    static constexpr int kKV = NH * kHalf;             // one K (or V) tile of 128 keys
    static constexpr int kKStages = 3;                 // K ring: freed as soon as both QKs read it
    static constexpr int kVStages = 2;                 // V ring: freed after both PVs
    static constexpr int oQ = 0;                       // 2 Q tiles
    static constexpr int oK = oQ + 2 * kQ;
    static constexpr int oV = oK + kKStages * kKV;
    static constexpr int oBar = oV + kVStages * kKV;
    static constexpr int kBytes = oBar + 256 + 1024;   // barriers + alignment slack
};

enum { BAR_KFULL = 0, BAR_KEMPTY = 3, BAR_VFULL = 6, BAR_VEMPTY = 8, BAR_SFULL = 10, BAR_PFULL = 12, BAR_ODONE = 14,
       BAR_QREADY = 15, BAR_PHALF = 16, BAR_OFREE = 18, BAR_ODONE1 = 19, BAR_N = 20 };
// O of Q tile t final: BAR_ODONE (t = 0; committed right after tile 0's last PV, so its
// epilogue overlaps tile 1's last step) / BAR_ODONE1 (t = 1; at the item's end)

__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                             uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

template <int D>
__global__ void __launch_bounds__(kTcThreads, 1)
tc_attn_kernel(const AttnParams p, const __grid_constant__ CUtensorMap tmap_k,
               const __grid_constant__ CUtensorMap tmap_v) {
    using L = TcSmem<D>;
    constexpr int NH = L::NH;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const uint32_t sbase = su32(smem);
    const uint32_t sQ = sbase + L::oQ, sK = sbase + L::oK, sV = sbase + L::oV;
    const uint32_t bars = sbase + L::oBar;
    uint32_t *tmem_slot = (uint32_t *)(smem + L::oBar + BAR_N * 8);
    const uint32_t s_zero = sbase + L::oBar + BAR_N * 8 + 8;   // a 0.0f word (scheduling fence, see softmax)
    auto bar = [&](int i) { return bars + 8u * i; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // Persistent: CTA b processes items [tc_off[b], tc_off[b+1]) (greedy LPT
    // assignment by the planner).  Every role walks the same item sequence;
    // barrier phases come from running counters, so the pipelines never drain
    // between items.
    long long *tr = (blockIdx.x == 0) ? p.trace : nullptr;   // debug timeline of CTA 0's first item (NULL: off)
    long long *trc = p.trace ? p.trace + 4096 + 4 * blockIdx.x : nullptr;   // per-CTA start / end (clock, ns)
    if (trc && threadIdx.x == 0) {
        trc[0] = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(trc[2]));
    }
    const int it_begin = p.tc_off[blockIdx.x], it_end = p.tc_off[blockIdx.x + 1];
    auto nkt_of = [&](const TcItem &it) { return (it.k1 - it.k0 + kTcKeys - 1) / kTcKeys; };
    auto ntiles_of = [&](const TcItem &it) { return it.nrows > kTcRows ? 2 : 1; };
    // KV tiles Q tile t of a prefill item needs: up to the causal limit of its last
    // row (tile 0 of a 256-row item stops one tile before tile 1 -- its last tile
    // would be fully masked).  The last Q tile needs them all; prefix nodes too.
    auto nkt_tile = [&](const TcItem &it, int t) {
        const int nkt = nkt_of(it);
        if (it.mode != 0 || t == ntiles_of(it) - 1) return nkt;
        const int x_last = it.hl0 + min(kTcRows * (t + 1), it.nrows) - 1;
        const int lim = min(it.k1, it.pos0 + x_last / p.G_q + 1);
        const int n = (lim - it.k0 + kTcKeys - 1) / kTcKeys;
        return n < 1 ? 1 : (n > nkt ? nkt : n);
    };

    if (threadIdx.x == 0) {
        for (int i = 0; i < L::kKStages; ++i) {
            mbar_init(bar(BAR_KFULL + i), 1);
            mbar_init(bar(BAR_KEMPTY + i), 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar(BAR_VFULL + i), 1);
            mbar_init(bar(BAR_VEMPTY + i), 1);
            mbar_init(bar(BAR_SFULL + i), 1);
            mbar_init(bar(BAR_PFULL + i), 128);
            mbar_init(bar(BAR_PHALF + i), 128);
        }
        mbar_init(bar(BAR_ODONE), 1);
        mbar_init(bar(BAR_ODONE1), 1);
        mbar_init(bar(BAR_QREADY), 256);
        mbar_init(bar(BAR_OFREE), 256);
        asm volatile("st.shared.u32 [%0], 0;\n" ::"r"(s_zero) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 9) {  // TMEM: tile t: S/P at [256 t, 256 t + 128), O at [256 t + 128, 256 t + 128 + D)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (p.app_T > 0 && !p.app_bg) {
        // ---- fused append: this CTA's share of the call's new tokens -> paged cache ----
        // (all 384 threads, 16-byte vectors; the slot of token t from the descriptors)
        const int t0 = (int)((int64_t)p.app_T * blockIdx.x / gridDim.x);
        const int t1 = (int)((int64_t)p.app_T * (blockIdx.x + 1) / gridDim.x);
        constexpr int cpr = D / 8;                   // uint4 chunks per head row
        const int row = p.H_kv * cpr;                // uint4 chunks per token (all KV heads)
        const uint4 *kn = reinterpret_cast<const uint4 *>(p.k_new) + (int64_t)t0 * row;
        const uint4 *vn = reinterpret_cast<const uint4 *>(p.v_new) + (int64_t)t0 * row;
        uint4 *kc = reinterpret_cast<uint4 *>(const_cast<uint16_t *>(p.k_cache));
        uint4 *vc = reinterpret_cast<uint4 *>(const_cast<uint16_t *>(p.v_cache));
        // 1) each token's cache row base (the token -> request -> block id chain, once
        //    per token) into smem; the K ring is unused until the producers start
        int64_t *s_base = reinterpret_cast<int64_t *>(smem + L::oK);
        const int ntok = t1 - t0;
        for (int i = threadIdx.x; i < ntok; i += kTcThreads) {
            const int t = t0 + i;
            const ReqDev rq = p.reqs[p.tok[t].req];
            const int pos = rq.c + (t - rq.cu_q);
            const int64_t blk = p.bt_flat[rq.bt_off + pos / kBlock];
            s_base[i] = (blk * p.H_kv * kBlock + pos % kBlock) * cpr;   // + g * kBlock * cpr + chunk
        }
        __syncthreads();
        // 2) the copy: 8 K and 8 V 16-byte loads in flight per thread before the stores
        constexpr int U = 8;
        const int64_t n = (int64_t)ntok * row;
        for (int64_t b0 = threadIdx.x; b0 < n; b0 += (int64_t)kTcThreads * U) {
            uint4 kv[U], vv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t idx = b0 + (int64_t)u * kTcThreads;
                if (idx < n) {
                    kv[u] = kn[idx];
                    vv[u] = vn[idx];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t idx = b0 + (int64_t)u * kTcThreads;
                if (idx < n) {
                    const int i = (int)(idx / row), e = (int)(idx - (int64_t)i * row);
                    const int g = e / cpr, ch = e % cpr;
                    const int64_t dst = s_base[i] + (int64_t)g * kBlock * cpr + ch;
                    kc[dst] = kv[u];
                    vc[dst] = vv[u];
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {   // release: this share is in global memory
            __threadfence();
            atomicAdd(p.app_cnt, 1ull);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // register rebalance between warpgroups (setmaxnreg at the head of each role):
    // producers need few registers, a softmax thread holds a 128-column S row
    if (warp >= 8) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(HG_TC_REG_WG2) : "memory");
    if (warp == 11 && p.app_T > 0 && p.app_bg) {
        // ===================== background append (warp 11) =====================
        // request by request in need order, this CTA's slice of each request's new
        // tokens (the block chain once per token), 8 K and 8 V 16-byte loads in flight
        // per lane; one count per (request, CTA) when the slice is in the cache
        constexpr int cpr = D / 8;
        const int row = p.H_kv * cpr;
        const uint4 *kn = reinterpret_cast<const uint4 *>(p.k_new), *vn = reinterpret_cast<const uint4 *>(p.v_new);
        uint4 *kc = reinterpret_cast<uint4 *>(const_cast<uint16_t *>(p.k_cache));
        uint4 *vc = reinterpret_cast<uint4 *>(const_cast<uint16_t *>(p.v_cache));
        constexpr int U = 8;
        for (int r = p.app_head; r >= 0;) {
            const ReqDev rq = p.reqs[r];
            const int a0 = rq.cu_q + (int)((int64_t)rq.n * blockIdx.x / gridDim.x);
            const int a1 = rq.cu_q + (int)((int64_t)rq.n * (blockIdx.x + 1) / gridDim.x);
            for (int t = a0; t < a1; ++t) {
                const int pos = rq.c + (t - rq.cu_q);
                const int64_t base = ((int64_t)p.bt_flat[rq.bt_off + pos / kBlock] * p.H_kv * kBlock + pos % kBlock) * cpr;
                const int64_t src = (int64_t)t * row;
                for (int e0 = lane; e0 < row; e0 += 32 * U) {
                    uint4 kv[U], vv[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int e = e0 + 32 * u;
                        if (e < row) {
                            kv[u] = kn[src + e];
                            vv[u] = vn[src + e];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int e = e0 + 32 * u;
                        if (e < row) {
                            const int g = e / cpr, ch = e % cpr;
                            const int64_t dst = base + (int64_t)g * kBlock * cpr + ch;
                            kc[dst] = kv[u];
                            vc[dst] = vv[u];
                        }
                    }
                }
            }
            __threadfence();   // every lane's stores, then one release count per (request, CTA)
            __syncwarp();
            if (lane == 0) atomicAdd(p.app_req_cnt + r, 1ull);
            r = rq.app_next;
        }
    } else if (warp == 8 || warp == 10) {
        // ===================== TMA producers: warp 8 streams K, warp 10 streams V =====================
        // (separate threads so a V slot that is still busy never delays the next K load)
        if (lane == 0) {
            int64_t gn = 0;   // K (or V) tiles loaded by this CTA so far
            bool appended = p.app_T == 0;   // every CTA's share of the fused append is in the cache
            for (int item = it_begin; item < it_end; ++item) {
                const TcItem it = p.tc[item];
                if (p.app_bg) appended = p.app_T == 0;   // background mode: waited per item's request
                const int nkt = nkt_of(it);
                const int32_t *bt = p.bt_flat + it.bt_off;
                const int kb0 = it.k0 / kBlock;
                const int kb_last = (it.k1 - 1) / kBlock;
                for (int j = 0; j < nkt; ++j, ++gn) {
                    if (!appended && it.k0 + (j + 1) * kTcKeys > it.cnew) {
                        // the tile holds keys this call appends: wait for every CTA's share
                        // prologue mode: every CTA's share (global count); background mode:
                        // every slice of this item's request (a prefill item's rows are one request)
                        const unsigned long long *cnt = p.app_cnt;
                        unsigned long long tgt = p.app_target;
                        if (p.app_bg) {
                            const int rq = p.tok[it.t0].req;
                            cnt = p.app_req_cnt + rq;
                            tgt = p.reqs[rq].app_tgt;
                        }
                        unsigned long long c;
                        for (;;) {
                            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(c) : "l"(cnt) : "memory");
                            if (c >= tgt) break;
                            __nanosleep(64);
                        }
                        asm volatile("fence.proxy.async.global;\n" ::: "memory");   // before the TMA reads
                        appended = true;
                    }
                    int rows[8];
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        int kb = kb0 + j * 8 + b;
                        kb = kb <= kb_last ? kb : kb0;  // rows past k1 are masked; keep the data finite
                        rows[b] = (bt[kb] * p.H_kv + it.g) * kBlock;
                    }
                    uint32_t dst, fb;
                    const CUtensorMap *tm;
                    if (warp == 8) {
                        const int st = (int)(gn % L::kKStages);
                        if (gn >= L::kKStages) mbar_wait(bar(BAR_KEMPTY + st), ((gn / L::kKStages) - 1) & 1);
                        if (tr && item == it_begin && j < 64) tr[1024 + 2 * j] = clock64();
                        dst = sK + st * L::kKV;
                        fb = bar(BAR_KFULL + st);
                        tm = &tmap_k;
                    } else {
                        const int st = (int)(gn & 1);
                        if (gn >= 2) mbar_wait(bar(BAR_VEMPTY + st), ((gn >> 1) - 1) & 1);
                        dst = sV + st * L::kKV;
                        fb = bar(BAR_VFULL + st);
                        tm = &tmap_v;
                    }
#ifdef HG_TC_NOLOAD   // A/B: after the rings' first fill, no K/V traffic (stale tiles; timing only)
                    if (gn >= L::kKStages) { mbar_arrive(fb); continue; }
#endif
                    mbar_expect_tx(fb, L::kKV);
#pragma unroll
                    for (int b = 0; b < 8; ++b)
#pragma unroll
                        for (int h = 0; h < NH; ++h)
                            tma_load_2d(dst + h * L::kHalf + b * (kBlock * 128), tm, h * 64, rows[b], fb);
                }
            }
        }
    } else if (warp == 9) {
        // ===================== MMA issuer =====================
        // The whole warp runs the control flow (warp-uniform: descriptors live in
        // uniform registers, no per-MMA register->uniform moves); one elected lane
        // issues each tcgen05 instruction.  Descriptors are built once and advanced
        // by compile-time offsets (start address field counts 16-byte units).
        constexpr uint32_t idS = idesc_bf16(128, 128, 0, 0);  // S = Q K^T: A, B K-major (smem)
        constexpr uint32_t idO = idesc_bf16(128, D, 0, 1);    // O += P V: A (P) in TMEM, B (V) MN-major
        const uint64_t dQ0 = smem_desc(sQ, 16, 1024);
        const uint64_t dK0 = smem_desc(sK, 16, 1024);
        const uint64_t dV0 = smem_desc(sV, L::kHalf, 1024);
        int64_t gk = 0, gv = 0;          // K / V tiles consumed so far
        int ps[2] = {0, 0};              // P steps consumed per Q tile
        int n_item = 0;
        for (int item = it_begin; item < it_end; ++item, ++n_item) {
            const TcItem it = p.tc[item];
            const int nkt = nkt_of(it), ntiles = ntiles_of(it);
            const int nkt0 = nkt_tile(it, 0);   // tile 0's steps (tile 1, if any, takes all nkt)
            const bool trace = tr && item == it_begin;
            auto issue_qk = [&](int t, int64_t kt, bool last_tile) {
                const uint32_t tS = tmem + 256 * t;
                const uint64_t dq = dQ0 + (uint64_t)((t * L::kQ) >> 4);
                const uint64_t dk = dK0 + (uint64_t)(((kt % L::kKStages) * L::kKV) >> 4);
                if (elect_one()) {
#pragma unroll
                    for (int ks = 0; ks < D / 16; ++ks) {
                        constexpr int kh = L::kHalf;
                        const uint32_t off = ((ks / 4) * kh + (ks % 4) * 32) >> 4;
                        umma_bf16(tS, dq + off, dk + off, idS, ks > 0);
                    }
                    umma_commit(bar(BAR_SFULL + t));
                    if (last_tile) umma_commit(bar(BAR_KEMPTY + kt % L::kKStages));  // every QK read K(kt)
                }
                __syncwarp();
            };
            mbar_wait(bar(BAR_QREADY), n_item & 1);
            mbar_wait(bar(BAR_KFULL + gk % L::kKStages), (gk / L::kKStages) & 1);
            tc_fence_after();
            for (int t = 0; t < ntiles; ++t) issue_qk(t, gk, t == ntiles - 1);
            if (n_item > 0) {   // the previous item's epilogue has read O out of TMEM
                mbar_wait(bar(BAR_OFREE), (n_item - 1) & 1);
                tc_fence_after();
            }
            for (int j = 0; j < nkt; ++j, ++gk, ++gv) {
                const int s = (int)(gv & 1);
                const uint64_t dv = dV0 + (uint64_t)((s * L::kKV) >> 4);
                bool kfull_next = false;   // K(j + 1) waited for (before the first QK of step j + 1)
                for (int t = 0; t < ntiles; ++t) {
                    if (t == 0 && j >= nkt0) continue;   // tile 0 is past its causal range
                    // PV in two halves: keys 0-63 as soon as the softmax has written them
                    mbar_wait(bar(BAR_PHALF + t), ps[t] & 1);
                    if (trace && j < 64 && lane == 0) tr[8 * j + 2 * t] = clock64();
                    if (t == 0 || j >= nkt0) mbar_wait(bar(BAR_VFULL + s), (gv >> 1) & 1);   // first tile of the step
                    tc_fence_after();
                    const uint32_t tS = tmem + 256 * t, tO = tS + 128;
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        if (half == 1) {
                            mbar_wait(bar(BAR_PFULL + t), ps[t] & 1);
                            tc_fence_after();
                        }
                        if (elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < kTcKeys / 32; ++kk) {   // P: 16 keys = 8 packed columns per k-step
                                const int ks = half * (kTcKeys / 32) + kk;
                                umma_bf16_ts(tO, tS + ks * 8, dv + (uint64_t)((ks * 2048) >> 4), idO,
                                             (j > 0 || ks > 0));
                            }
                        }
                        __syncwarp();
                    }
                    ++ps[t];
                    if (t == 0 && j == nkt0 - 1 && elect_one()) umma_commit(bar(BAR_ODONE));   // tile 0's O final
                    __syncwarp();
                    if (j + 1 < (t == 0 ? nkt0 : nkt)) {
                        if (!kfull_next) {
                            mbar_wait(bar(BAR_KFULL + (gk + 1) % L::kKStages), ((gk + 1) / L::kKStages) & 1);
                            tc_fence_after();
                            kfull_next = true;
                        }
                        issue_qk(t, gk + 1, t == ntiles - 1);   // in order after PV(t, j): S/P of tile t is free
                    }
                    if (trace && j < 64 && lane == 0) tr[8 * j + 2 * t + 1] = clock64();
                }
                if (elect_one()) umma_commit(bar(BAR_VEMPTY + s));   // every PV read V(j)
                __syncwarp();
            }
            if (elect_one()) umma_commit(bar(BAR_ODONE1));   // tile 1's O (and every MMA of the item) final
            __syncwarp();
        }
    } else if (warp < 8) {
        // ===================== softmax / correction / epilogue (warps 0-7) =====================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(HG_TC_REG_SOFTMAX) : "memory");
        const int t = warp >> 2;             // Q tile of this warpgroup
        const int r = threadIdx.x & 127;     // row in the tile == TMEM lane
        const int rr = t * kTcRows + r;      // stacked row of the item
        const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + 256 * t + lane_base, tO = tS + 128;
        const float sc = p.scale_log2;
        int ss = 0;                          // S steps consumed by this Q tile
        int n_item = 0;
        for (int item = it_begin; item < it_end; ++item, ++n_item) {
            const TcItem it = p.tc[item];
            const int ntiles = ntiles_of(it);
            const int nkt = t < ntiles ? nkt_tile(it, t) : 0;   // this Q tile's KV steps
            const bool trace = tr && item == it_begin;
            const bool valid = rr < it.nrows;
            struct { int t, h, lim; } row{0, 0, 0};
            if (valid) {
                const int x = it.hl0 + rr, j = x / p.G_q;
                row.h = it.g * p.G_q + (x - j * p.G_q);
                if (it.mode == 0) {
                    row.t = it.t0 + j;
                    row.lim = it.pos0 + j + 1;
                } else {
                    row.t = p.tc_tok[it.t0 + j];
                    row.lim = it.k1;
                }
            }
            // Q row -> smem, K-major 128B swizzle: half h, row r at h*16K + r*128, chunk c at (c ^ (r&7))*16.
            // The previous item's QKs are complete: this warpgroup waited its ODONE.
            if (t < ntiles) {
                HG_DCHECK(!valid || (row.t >= 0 && row.t < p.T && row.h < p.H_q));
                const uint4 *src = reinterpret_cast<const uint4 *>(p.q + ((int64_t)row.t * p.H_q + row.h) * D);
                const uint32_t qb = sQ + t * L::kQ + r * 128;
#pragma unroll
                for (int c = 0; c < D / 8; ++c) {
                    const uint4 v = valid ? src[c] : make_uint4(0, 0, 0, 0);
                    sts128(qb + (c >> 3) * L::kHalf + (((c & 7) ^ (r & 7)) << 4), v);
                }
                fence_async_smem();
            }
            mbar_arrive(bar(BAR_QREADY));
            if (t < ntiles) {
                const int lim = valid ? row.lim : 0;
                float m_used = -CUDART_INF_F;  // reference max (log2 domain) of the exponentials
                float l_sum = 0.f;
                for (int j = 0; j < nkt; ++j, ++ss) {
                    mbar_wait(bar(BAR_SFULL + t), ss & 1);   // QK(t, j) and everything before it (PV(t, j-1)) done
                    if (trace && r == 0 && j < 64) tr[512 + 256 * t + 2 * j] = clock64();
                    tc_fence_after();
#ifdef HG_TC_NOSOFTMAX   // A/B: no softmax work at all (the MMA + TMA pipeline alone; output wrong)
                    mbar_arrive(bar(BAR_PHALF + t));
                    mbar_arrive(bar(BAR_PFULL + t));
                    continue;
#endif
                    uint32_t sr[128];
#pragma unroll
                    for (int c = 0; c < 4; ++c) TMEM_LD32(tS + c * 32, (&sr[c * 32]));
                    tmem_wait_ld();
                    if (trace && r == 0 && j < 64) tr[2048 + 512 * t + 8 * j + 0] = clock64();
                    const int kbase = it.k0 + j * kTcKeys;
                    // diagonal / tail tile: mask keys >= lim.  The branch is made
                    // warp-uniform so full tiles skip the (if-converted) mask body.
                    const int nvalid = lim - kbase;
                    if (__any_sync(0xffffffffu, nvalid < kTcKeys)) {
#pragma unroll
                        for (int c = 0; c < 128; ++c)
                            if (c >= nvalid) sr[c] = __float_as_uint(-CUDART_INF_F);
                    }
                    float mx[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) mx[e] = __uint_as_float(sr[e]);
#pragma unroll
                    for (int c = 8; c < 128; ++c) mx[c & 7] = fmaxf(mx[c & 7], __uint_as_float(sr[c]));
                    const float mraw = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                             fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
                    const float mt = mraw * sc;   // scale > 0: max commutes with scaling
                    // lazy rescaling: move the reference only when the row max grew by > 2^8
                    const bool bump = mt > m_used + kRescaleThreshold;
                    float alpha = 1.f;
                    if (bump) {
                        alpha = (m_used == -CUDART_INF_F) ? 0.f : ex2(m_used - mt);
                        m_used = mt;
                    }
                    if (j > 0 && __any_sync(0xffffffffu, bump)) {  // O(t) is stable: PV(t, j-1) completed
                        uint32_t orr[32];
#pragma unroll 1
                        for (int c = 0; c < D / 32; ++c) {
                            TMEM_LD32(tO + c * 32, orr);
                            tmem_wait_ld();
#pragma unroll
                            for (int e = 0; e < 32; ++e) orr[e] = __float_as_uint(__uint_as_float(orr[e]) * alpha);
                            TMEM_ST32(tO + c * 32, orr);
                        }
                    }
                    if (trace && r == 0 && j < 64) tr[2048 + 512 * t + 8 * j + 1] = clock64();
                    const float nref = (m_used == -CUDART_INF_F) ? 0.f : -m_used;
                    const uint64_t sc2 = f2pack(sc, sc);
                    uint64_t nref2 = f2pack(nref, nref);
                    uint64_t ls2[2] = {0ull, 0ull};
                    uint32_t pk[64];
#pragma unroll
                    for (int c = 0; c < 64; ++c) {
                        if (c == 32) {   // first half of P (keys 0-63) -> TMEM: the MMA can start PV on it
                            if (trace && r == 0 && j < 64) tr[2048 + 512 * t + 8 * j + 2] = clock64();
                            TMEM_ST32(tS, pk);
                            tmem_wait_st();
                            tc_fence_before();
                            mbar_arrive(bar(BAR_PHALF + t));
                            if (trace && r == 0 && j < 64) tr[2048 + 512 * t + 8 * j + 3] = clock64();
                            // keep the second half's exponentials after this point: otherwise
                            // ptxas hoists nearly all MUFU work above the first store and the PV
                            // of keys 0-63 cannot start until the whole row is done.  The second
                            // half's offset comes from a volatile load of a 0.0f word, ordered
                            // after the arrive.
                            float zero;
                            asm volatile("ld.volatile.shared.f32 %0, [%1];\n" : "=f"(zero) : "r"(s_zero) : "memory");
                            nref2 = f2pack(nref + zero, nref + zero);
                        }
                        const uint64_t x2 = ffma2(f2pack(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])),
                                                  sc2, nref2);
                        float a, b;
                        if ((HG_POLY_MASK >> (c & 7)) & 1) {   // pairs on the FMA pipe, the rest on MUFU (FA4-style offload)
                            exp2_poly2(x2, a, b);
                        } else {
                            float x0, x1;
                            f2unpack(x2, x0, x1);
                            a = ex2(x0);
                            b = ex2(x1);
                        }
                        const uint64_t ab = f2pack(a, b);
                        ls2[c & 1] = fadd2(ls2[c & 1], ab);
                        pk[c] = pack2(a, b);
                    }
                    float l0, l1, l2, l3;
                    f2unpack(ls2[0], l0, l1);
                    f2unpack(ls2[1], l2, l3);
                    l_sum = l_sum * alpha + ((l0 + l1) + (l2 + l3));
                    // second half of P (bf16 pairs, keys 64-127) over S's columns 32-63 of this lane
                    TMEM_ST32(tS + 32, (&pk[32]));
                    tmem_wait_st();
                    tc_fence_before();
                    mbar_arrive(bar(BAR_PFULL + t));
                    if (trace && r == 0 && j < 64) tr[512 + 256 * t + 2 * j + 1] = clock64();
                }
                // ---- epilogue ----
                mbar_wait(bar(t == 0 ? BAR_ODONE : BAR_ODONE1), n_item & 1);
                tc_fence_after();
                const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
                const float lse2 = l_sum > 0.f ? m_used + __log2f(l_sum) : -CUDART_INF_F;
                const int G = p.G_q;
                int base = -1;
                if (valid && it.part >= 0) {
                    const TokDev tk = p.tok[row.t];
                    base = tk.base + it.g * tk.nparts * G;   // + part * G + hl below
                }
#pragma unroll 1
                for (int c = 0; c < D / 32; ++c) {
                    uint32_t orr[32];
                    TMEM_LD32(tO + c * 32, orr);
                    tmem_wait_ld();
                    if (c == D / 32 - 1) {   // O fully read: the next item's PV may overwrite it
                        tc_fence_before();
                        mbar_arrive(bar(BAR_OFREE));
                    }
                    if (!valid) continue;
                    if (it.part < 0) {
                        const int64_t off = (int64_t)row.t * p.out_ld + (int64_t)row.h * D + c * 32;
                        uint4 v[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            v[e] = make_uint4(
                                pack2(__uint_as_float(orr[8 * e + 0]) * inv, __uint_as_float(orr[8 * e + 1]) * inv),
                                pack2(__uint_as_float(orr[8 * e + 2]) * inv, __uint_as_float(orr[8 * e + 3]) * inv),
                                pack2(__uint_as_float(orr[8 * e + 4]) * inv, __uint_as_float(orr[8 * e + 5]) * inv),
                                pack2(__uint_as_float(orr[8 * e + 6]) * inv, __uint_as_float(orr[8 * e + 7]) * inv));
                        for (int k = 0; k < p.n_out; ++k) {
                            uint4 *dst = reinterpret_cast<uint4 *>(p.outs[k] + off);
#pragma unroll
                            for (int e = 0; e < 4; ++e) dst[e] = v[e];
                        }
                    } else {
                        const int64_t slot = base + (int64_t)it.part * G + (row.h % G);
                        HG_DCHECK(slot >= 0 && slot < p.n_slots);
                        float4 *dst = reinterpret_cast<float4 *>(p.part_o + slot * D + c * 32);
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            dst[e] = make_float4(__uint_as_float(orr[4 * e]) * inv, __uint_as_float(orr[4 * e + 1]) * inv,
                                                 __uint_as_float(orr[4 * e + 2]) * inv,
                                                 __uint_as_float(orr[4 * e + 3]) * inv);
                    }
                }
                if (valid) {
                    if (it.part < 0) {
                        if (p.lse) p.lse[(int64_t)row.t * p.H_q + row.h] = lse2 * 0.69314718055994531f;
                    } else {
                        p.part_lse[base + (int64_t)it.part * G + (row.h % G)] = lse2;
                    }
                }
            } else {
                // an unused Q tile holds no O; stay in step with the item (QREADY / OFREE
                // phases must not mix arrivals of different items)
                mbar_wait(bar(t == 0 ? BAR_ODONE : BAR_ODONE1), n_item & 1);
                mbar_arrive(bar(BAR_OFREE));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (trc && threadIdx.x == 0) {
        trc[1] = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(trc[3]));
    }
    if (warp == 9) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
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
    const int grid = std::max(1, std::min(p.n_tc, p.tc_ctas > 0 ? p.tc_ctas : p.n_tc));
    tc_attn_kernel<D><<<grid, kTcThreads, bytes, st>>>(p, *(const CUtensorMap *)tk, *(const CUtensorMap *)tv);
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
