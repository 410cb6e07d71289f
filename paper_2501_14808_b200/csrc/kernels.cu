// kernels.cu -- sm_100a kernels of the HBM-bound half of the hot path:
//   append_kernel   a.3  paged KV write (16-byte vector copies)
//   splitk_kernel   a.6  split-K attention for decode rows (and small row groups):
//                        per (request, KV head, key range) item, up to 16 stacked
//                        query rows (token x q-head of one GQA group) against
//                        paged KV blocks streamed by cp.async with 16-byte
//                        coalesced loads; QK^T and PV on mma.sync m16n8k16
//                        (bf16 in, fp32 accumulate) because GQA decode is
//                        G_q FLOP/B and CUDA-core FMA cannot keep up with HBM
//                        at G_q >= 4; warp-shuffle online
//                        softmax; 4 warps split the item's blocks and merge
//                        through shared memory.
//   combine_kernel  a.7  log-sum-exp merge of split / prefix partials.
#include <cstring>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "hg_internal.h"

namespace hg {

// ----------------------------------------------------------------------------
// a.3 append: K[slot] = K_new[t], V[slot] = V_new[t] for every KV head.
// ----------------------------------------------------------------------------
__global__ void append_kernel(const uint4 *__restrict__ k_new, const uint4 *__restrict__ v_new,
                              uint4 *__restrict__ k_cache, uint4 *__restrict__ v_cache,
                              const int64_t *__restrict__ slot, int T, int H_kv, int chunks_per_row) {
    // one 16-byte chunk of K and of V per thread; rows = (t, g)
    const int64_t total = (int64_t)T * H_kv * chunks_per_row;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = idx / chunks_per_row;
        const int ch = (int)(idx % chunks_per_row);
        const int64_t t = row / H_kv;
        const int g = (int)(row % H_kv);
        const int64_t s = slot[t];
        const int64_t blk = s / kBlock, off = s % kBlock;
        const int64_t dst = ((blk * H_kv + g) * kBlock + off) * chunks_per_row + ch;
        k_cache[dst] = k_new[idx];
        v_cache[dst] = v_new[idx];
    }
}

hg_status launch_append(const uint16_t *k_new, const uint16_t *v_new, uint16_t *k_cache,
                        uint16_t *v_cache, const int64_t *slot, int T, int H_kv, int d, void *stream) {
    if (T == 0) return HG_OK;
    const int cpr = d / 8;
    const int64_t total = (int64_t)T * H_kv * cpr;
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((total + threads - 1) / threads, 148 * 16);
    append_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(
        (const uint4 *)k_new, (const uint4 *)v_new, (uint4 *)k_cache, (uint4 *)v_cache, slot, T, H_kv, cpr);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "append launch: %s", cudaGetErrorString(e));
}

// Fused-step append: the slot of token t is derived on the device from the
// attention descriptors (owning request, cached length, flattened block ids).
// One CTA per token: the slot is computed once, then every (KV head, 16-byte
// chunk) of K and V is moved with all loads issued before the stores.
// Peer-window barrier body (see peer_barrier_kernel below): thread k < world
// publishes `epoch` into rank k's slot [rank] and waits for rank k's arrival in
// the local slot [k]; traps after ~30 s.
__device__ __forceinline__ void peer_barrier_body(unsigned long long *const *flags, unsigned long long *mine,
                                                  int rank, int world, unsigned long long epoch, int k) {
    if (k >= world) return;
    asm volatile("fence.acq_rel.sys;\n" ::: "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(flags[k] + rank), "l"(epoch) : "memory");
    unsigned long long t0, now, v;
    asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t0));
    for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(mine + k) : "memory");
        if (v >= epoch) break;
        asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(now));
        if (now - t0 > 30000000000ull) __trap();
        __nanosleep(256);
    }
}

template <int PER>   // uint4 chunks of K (and of V) per thread
__global__ void __launch_bounds__(256) append_dev_kernel(const uint4 *__restrict__ k_new,
                                                         const uint4 *__restrict__ v_new, uint4 *__restrict__ k_cache,
                                                         uint4 *__restrict__ v_cache, const AttnParams p,
                                                         int chunks_per_row, int wave) {
    const int t = blockIdx.x;
    // sharded fused step: CTA 0's first warp also runs the peer-window entry
    // barrier (the kernels after this one are the first to write peer windows)
    if (p.bar_world > 0 && t == 0 && threadIdx.x < 32)
        peer_barrier_body(p.bar_flags, p.bar_mine, p.bar_rank, p.bar_world, p.bar_epoch, threadIdx.x);
    const int row_chunks = p.H_kv * chunks_per_row;   // uint4 chunks of one token's K (or V)
    const int64_t src0 = (int64_t)t * row_chunks;
    // the first batch of this token's K/V loads goes out before the descriptor
    // chain (token -> request -> block id) it does not depend on
    uint4 kv[2 * PER];
    int idx[PER];
    if (wave < 0) {
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            idx[e] = threadIdx.x + e * 256;
            if (idx[e] < row_chunks) {
                kv[e] = k_new[src0 + idx[e]];
                kv[PER + e] = v_new[src0 + idx[e]];
            }
        }
    }
    const TokDev tk = p.tok[t];
    if (wave >= 0 && tk.wave != wave) return;   // pipelined host step: this token's inputs arrive in the other wave
    const ReqDev rq = p.reqs[tk.req];
    const int pos = rq.c + (t - rq.cu_q);
    const int64_t blk = p.bt_flat[rq.bt_off + pos / kBlock];
    for (int base = 0; base < row_chunks; base += 256 * PER) {
        if (base > 0 || wave >= 0) {
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                idx[e] = base + threadIdx.x + e * 256;
                if (idx[e] < row_chunks) {
                    kv[e] = k_new[src0 + idx[e]];
                    kv[PER + e] = v_new[src0 + idx[e]];
                }
            }
        }
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            if (idx[e] < row_chunks) {
                const int g = idx[e] / chunks_per_row, ch = idx[e] - g * chunks_per_row;
                const int64_t dst = ((blk * p.H_kv + g) * kBlock + pos % kBlock) * chunks_per_row + ch;
                k_cache[dst] = kv[e];
                v_cache[dst] = kv[PER + e];
            }
        }
    }
}

// Fused-step append with the token slots in the kernel parameters (no
// dependency on the descriptor upload, so it runs while that copy is in
// flight).  One CTA per token, K/V loads issued before the stores.
template <int NS>
struct SlotParams {
    int64_t slot[NS];
};

struct BarrierArgs {   // peer-window entry barrier carried by the append (world = 0: none)
    unsigned long long *flags[kMaxOuts];
    unsigned long long *mine;
    int rank, world;
    unsigned long long epoch;
    unsigned long long *done;   // non-NULL: every CTA counts itself here after its stores
};

template <int PER, int NS>
__global__ void __launch_bounds__(256) append_param_kernel(const uint4 *__restrict__ k_new,
                                                           const uint4 *__restrict__ v_new,
                                                           uint4 *__restrict__ k_cache, uint4 *__restrict__ v_cache,
                                                           const __grid_constant__ SlotParams<NS> sp, int H_kv,
                                                           int chunks_per_row, const BarrierArgs ba) {
    const int t = blockIdx.x;
    if (ba.world > 0 && t == 0 && threadIdx.x < 32)
        peer_barrier_body(ba.flags, ba.mine, ba.rank, ba.world, ba.epoch, threadIdx.x);
    const int row_chunks = H_kv * chunks_per_row;
    const int64_t src0 = (int64_t)t * row_chunks;
    const int64_t s = sp.slot[t];
    const int64_t blk = s / kBlock, pos = s % kBlock;
    for (int base = 0; base < row_chunks; base += 256 * PER) {
        uint4 kv[2 * PER];
        int idx[PER];
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            idx[e] = base + threadIdx.x + e * 256;
            if (idx[e] < row_chunks) {
                kv[e] = k_new[src0 + idx[e]];
                kv[PER + e] = v_new[src0 + idx[e]];
            }
        }
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            if (idx[e] < row_chunks) {
                const int g = idx[e] / chunks_per_row, ch = idx[e] - g * chunks_per_row;
                const int64_t dst = ((blk * H_kv + g) * kBlock + pos) * chunks_per_row + ch;
                k_cache[dst] = kv[e];
                v_cache[dst] = kv[PER + e];
            }
        }
    }
    if (ba.done) {   // a later kernel on another stream waits for the count (no stream join)
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(ba.done, 1ull);
        }
    }
}

template <int NS>
static void launch_append_param_ns(const uint4 *kn, const uint4 *vn, uint4 *kc, uint4 *vc, const int64_t *slots,
                                   int T, int H_kv, int cpr, const BarrierArgs &ba, cudaStream_t st) {
    SlotParams<NS> sp;
    memcpy(sp.slot, slots, sizeof(int64_t) * (size_t)T);
    const int per = (H_kv * cpr + 255) / 256;
    if (per <= 1) append_param_kernel<1, NS><<<T, 256, 0, st>>>(kn, vn, kc, vc, sp, H_kv, cpr, ba);
    else if (per <= 2) append_param_kernel<2, NS><<<T, 256, 0, st>>>(kn, vn, kc, vc, sp, H_kv, cpr, ba);
    else if (per <= 4) append_param_kernel<4, NS><<<T, 256, 0, st>>>(kn, vn, kc, vc, sp, H_kv, cpr, ba);
    else append_param_kernel<8, NS><<<T, 256, 0, st>>>(kn, vn, kc, vc, sp, H_kv, cpr, ba);
}

hg_status launch_append_param(const uint16_t *k_new, const uint16_t *v_new, uint16_t *k_cache, uint16_t *v_cache,
                              const int64_t *slots_host, int T, int H_kv, int d, void *stream,
                              const AttnParams *bar) {
    BarrierArgs ba{};
    if (bar && bar->bar_world > 0) {
        for (int k = 0; k < bar->bar_world; ++k) ba.flags[k] = bar->bar_flags[k];
        ba.mine = bar->bar_mine;
        ba.rank = bar->bar_rank;
        ba.world = bar->bar_world;
        ba.epoch = bar->bar_epoch;
    }
    if (bar) ba.done = bar->app_cnt;
    if (T == 0) return HG_OK;
    if (T > kParamSlots) return fail(HG_E_INVALID, "append_param: T %d > %d", T, kParamSlots);
    auto *kn = (const uint4 *)k_new, *vn = (const uint4 *)v_new;
    auto *kc = (uint4 *)k_cache, *vc = (uint4 *)v_cache;
    cudaStream_t st = (cudaStream_t)stream;
    if (T <= 1024) launch_append_param_ns<1024>(kn, vn, kc, vc, slots_host, T, H_kv, d / 8, ba, st);
    else launch_append_param_ns<kParamSlots>(kn, vn, kc, vc, slots_host, T, H_kv, d / 8, ba, st);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "append launch: %s", cudaGetErrorString(e));
}

hg_status launch_append_dev(const AttnParams &p, const uint16_t *k_new, const uint16_t *v_new, int T, void *stream,
                            int wave) {
    if (T == 0) return HG_OK;
    const int cpr = p.d / 8;
    const int row_chunks = p.H_kv * cpr;
    const int per = (row_chunks + 255) / 256;
    auto *kn = (const uint4 *)k_new, *vn = (const uint4 *)v_new;
    auto *kc = (uint4 *)p.k_cache, *vc = (uint4 *)p.v_cache;
    cudaStream_t st = (cudaStream_t)stream;
    if (per <= 1) append_dev_kernel<1><<<T, 256, 0, st>>>(kn, vn, kc, vc, p, cpr, wave);
    else if (per <= 2) append_dev_kernel<2><<<T, 256, 0, st>>>(kn, vn, kc, vc, p, cpr, wave);
    else if (per <= 4) append_dev_kernel<4><<<T, 256, 0, st>>>(kn, vn, kc, vc, p, cpr, wave);
    else append_dev_kernel<8><<<T, 256, 0, st>>>(kn, vn, kc, vc, p, cpr, wave);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "append launch: %s", cudaGetErrorString(e));
}

// ----------------------------------------------------------------------------
// PTX helpers
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
// 16 bytes, or 16 zero bytes when !valid (src-size 0: nothing is read from src)
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
// D = A * B + D, m16n8k16, bf16 inputs, fp32 accumulators
__device__ __forceinline__ void mma_bf16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&v);
}
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
    return y;
}

// Byte offset of 16-byte chunk `ch` of row `row` in a [rows][D] bf16 tile whose
// chunks are XOR-swizzled by (row & 7): ldmatrix of 8 rows at one chunk index
// then touches 8 distinct bank groups.
template <int D>
__device__ __forceinline__ uint32_t swz(int row, int ch) {
    return (uint32_t)(row * D * 2 + ((ch ^ (row & 7)) << 4));
}

// ----------------------------------------------------------------------------
// NEXT-4 prologue: append + rotary position embedding (include/hygen.h hg_rope).
// One CTA per token: the R/2 (cos, sin) of its position are computed once in
// fp64 into shared memory; each thread then rotates a pair of 16-byte chunks
// (dims [8c, 8c+8) and [8c + R/2, 8c + R/2 + 8)) of one head in fp32 and
// rounds to bf16.  Dims >= R and V are copied.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void rope_chunk(uint4 &lo, uint4 &hi, const float2 *cs) {
    uint32_t *a = reinterpret_cast<uint32_t *>(&lo), *b = reinterpret_cast<uint32_t *>(&hi);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&a[e]));
        const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&b[e]));
        const float2 c0 = cs[2 * e], c1 = cs[2 * e + 1];
        a[e] = pack_bf16(x.x * c0.x - y.x * c0.y, x.y * c1.x - y.y * c1.y);
        b[e] = pack_bf16(y.x * c0.x + x.x * c0.y, y.y * c1.x + x.y * c1.y);
    }
}

template <bool DESC>
__global__ void __launch_bounds__(256) rope_append_kernel(const uint4 *__restrict__ k_new,
                                                          const uint4 *__restrict__ v_new, uint4 *__restrict__ k_cache,
                                                          uint4 *__restrict__ v_cache, const AttnParams p,
                                                          const int64_t *__restrict__ slot_arr,
                                                          const int32_t *__restrict__ pos_arr,
                                                          const uint4 *__restrict__ q_src, uint4 *__restrict__ q_dst,
                                                          int H_q, int H_kv, int cpr, double theta, int rot) {
    __shared__ float2 cs[128];
    const int t = blockIdx.x;
    int64_t blk, off;
    int pos;
    if (DESC) {
        const ReqDev rq = p.reqs[p.tok[t].req];
        pos = rq.c + (t - rq.cu_q);
        blk = p.bt_flat[rq.bt_off + pos / kBlock];
        off = pos % kBlock;
    } else {
        const int64_t sl = slot_arr[t];
        blk = sl / kBlock;
        off = sl % kBlock;
        pos = pos_arr[t];
    }
    const int half = rot / 2, hc = half / 8;
    for (int i = threadIdx.x; i < half; i += blockDim.x) {
        double sv, cv;
        sincos((double)pos * pow(theta, -2.0 * i / rot), &sv, &cv);
        cs[i] = make_float2((float)cv, (float)sv);
    }
    __syncthreads();
    const int units = cpr - hc;   // per head: hc rotated chunk pairs + the unrotated chunks
    for (int u = threadIdx.x; u < H_kv * units; u += blockDim.x) {
        const int g = u / units, c = u - g * units;
        const int64_t src = ((int64_t)t * H_kv + g) * cpr;
        const int64_t dst = ((blk * H_kv + g) * kBlock + off) * cpr;
        if (c < hc) {
            uint4 lo = k_new[src + c], hi = k_new[src + c + hc];
            const uint4 vl = v_new[src + c], vh = v_new[src + c + hc];
            rope_chunk(lo, hi, cs + 8 * c);
            k_cache[dst + c] = lo;
            k_cache[dst + c + hc] = hi;
            v_cache[dst + c] = vl;
            v_cache[dst + c + hc] = vh;
        } else {
            const int cc = c + hc;
            k_cache[dst + cc] = k_new[src + cc];
            v_cache[dst + cc] = v_new[src + cc];
        }
    }
    if (q_dst) {
        for (int u = threadIdx.x; u < H_q * units; u += blockDim.x) {
            const int h = u / units, c = u - h * units;
            const int64_t base = ((int64_t)t * H_q + h) * cpr;
            if (c < hc) {
                uint4 lo = q_src[base + c], hi = q_src[base + c + hc];
                rope_chunk(lo, hi, cs + 8 * c);
                q_dst[base + c] = lo;
                q_dst[base + c + hc] = hi;
            } else {
                q_dst[base + c + hc] = q_src[base + c + hc];
            }
        }
    }
}

hg_status launch_rope_append_dev(const AttnParams &p, const uint16_t *k_new, const uint16_t *v_new,
                                 const uint16_t *q_src, uint16_t *q_dst, int T, const RopeArgs &r, void *stream) {
    if (T == 0) return HG_OK;
    rope_append_kernel<true><<<T, 256, 0, (cudaStream_t)stream>>>(
        (const uint4 *)k_new, (const uint4 *)v_new, (uint4 *)p.k_cache, (uint4 *)p.v_cache, p, nullptr, nullptr,
        (const uint4 *)q_src, (uint4 *)q_dst, p.H_q, p.H_kv, p.d / 8, r.theta, r.rot);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "rope append launch: %s", cudaGetErrorString(e));
}

hg_status launch_rope_append(const uint16_t *k_new, const uint16_t *v_new, uint16_t *k_cache, uint16_t *v_cache,
                             const int64_t *slot, const int32_t *pos, int T, int H_kv, int d, const RopeArgs &r,
                             void *stream) {
    if (T == 0) return HG_OK;
    AttnParams p{};
    rope_append_kernel<false><<<T, 256, 0, (cudaStream_t)stream>>>(
        (const uint4 *)k_new, (const uint4 *)v_new, (uint4 *)k_cache, (uint4 *)v_cache, p, slot, pos, nullptr,
        nullptr, 0, H_kv, d / 8, r.theta, r.rot);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "rope append launch: %s", cudaGetErrorString(e));
}

// ----------------------------------------------------------------------------
// a.6 split-K attention item kernel
// ----------------------------------------------------------------------------
#ifndef HG_SK_WARPS
#define HG_SK_WARPS 4
#endif
#ifndef HG_SK_STAGES
#define HG_SK_STAGES 2
#endif
constexpr int kSkWarps = HG_SK_WARPS;    // warps per split-K CTA (each streams its own blocks)
constexpr int kSkStages = HG_SK_STAGES;  // cp.async stages per warp (one 16-token K+V block each)

template <int D>
struct SkSmem {
    static constexpr int kTile = kBlock * D * 2;            // one K (or V) block tile, bytes
    static constexpr int kStage = 2 * kTile;                 // K + V
    static constexpr int kWarp = kSkStages * kStage;
    static constexpr int kQ = kSkRows * D * 2;
    static constexpr int kMS = D + 4;                         // merge row stride (floats): rotates rows by 4 banks
    static constexpr int kMerge = kSkWarps * (kSkRows * kMS + 2 * kSkRows) * 4;
    static constexpr int kMain = kSkWarps * kWarp;
    static constexpr int kBytes = kQ + (kMain > kMerge ? kMain : kMerge);
};

// Sharded step: split-K's first store into a peer window waits until this call's
// entry barrier is through -- either the barrier kernel ahead of it (programmatic
// dependency, bar_pdl) or the barrier run by split-K's own first CTA (entry_word).
__device__ __forceinline__ void wait_entry(const AttnParams &p) {
    if (p.bar_pdl) asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (p.entry_word) {
        unsigned int c;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(c) : "l"(p.entry_word + 1) : "memory");
            if (c) break;
            __nanosleep(128);
        }
    }
}

// a.7 merge of one row's partials: O = sum_s 2^{lse_s - LSE} o_s, LSE = log2 sum_s 2^{lse_s}
// One merged row (token t, KV head g, q-head-in-group hl) by one warp.  Shared by
// the combine kernel and split-K's in-kernel merge (AttnParams.sk_cnt), so the two
// give bit-identical rows.  Partials are read through L2 (ld.global.cg): inside
// split-K they were written by other SMs during this grid.
template <int D>
__device__ __forceinline__ void combine_row(const AttnParams &p, const int t, const int g, const int hl,
                                            const int lane) {
    const int G = p.G_q;
    const TokDev tk = p.tok[t];
    const int64_t base = tk.base + (int64_t)g * tk.nparts * G;
    HG_DCHECK(t >= 0 && t < p.T && tk.nparts >= 1 && tk.base >= 0 && g < p.H_kv && hl < G);
    HG_DCHECK(base + (int64_t)(tk.nparts - 1) * G + hl < p.n_slots);
    // the parts' LSEs are loaded once, lane s holding parts s, s + 32, ...; max and
    // sum by warp shuffles (no chain of dependent loads per part)
    float lv[2];
    float M = -CUDART_INF_F;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int sidx = lane + 32 * k;
        lv[k] = sidx < tk.nparts ? __ldcg(p.part_lse + base + (int64_t)sidx * G + hl) : -CUDART_INF_F;
        M = fmaxf(M, lv[k]);
    }
    for (int sidx = lane + 64; sidx < tk.nparts; sidx += 32) M = fmaxf(M, __ldcg(p.part_lse + base + (int64_t)sidx * G + hl));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    const float ref = (M == -CUDART_INF_F) ? 0.f : M;
    float wl[2], L = 0.f;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        wl[k] = fast_exp2(lv[k] - ref);   // 0 for missing / empty parts
        L += wl[k];
    }
    for (int sidx = lane + 64; sidx < tk.nparts; sidx += 32)
        L += fast_exp2(__ldcg(p.part_lse + base + (int64_t)sidx * G + hl) - ref);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    const float inv = L > 0.f ? 1.f / L : 0.f;
    constexpr int PER = D / 32;
    float acc[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = 0.f;
#pragma unroll 4
    for (int sidx = 0; sidx < tk.nparts; ++sidx) {
        const int64_t slot = base + (int64_t)sidx * G + hl;
        const float w = (sidx < 64 ? __shfl_sync(0xffffffffu, wl[sidx >> 5], sidx & 31)
                                   : fast_exp2(__ldcg(p.part_lse + slot) - ref)) * inv;
        const float *src = p.part_o + slot * D + lane * PER;
#pragma unroll
        for (int e = 0; e < PER; e += 2) {
            float2 v = __ldcg(reinterpret_cast<const float2 *>(src + e));
            acc[e] += w * v.x;
            acc[e + 1] += w * v.y;
        }
    }
    const int h = g * G + hl;
    const int64_t off = (int64_t)t * p.out_ld + (int64_t)h * D + lane * PER;
    uint32_t pk[PER / 2];
#pragma unroll
    for (int e = 0; e < PER; e += 2) pk[e / 2] = pack_bf16(acc[e], acc[e + 1]);
    for (int k = 0; k < p.n_out; ++k) {
#pragma unroll
        for (int e = 0; e < PER / 2; ++e) reinterpret_cast<uint32_t *>(p.outs[k] + off)[e] = pk[e];
    }
    if (p.lse && lane == 0)
        p.lse[(int64_t)t * p.H_q + h] = (L > 0.f ? ref + __log2f(L) : -CUDART_INF_F) * 0.69314718055994531f;
}

// One split-K item (a piece of one row chunk's keys for KV head g) by the whole CTA.
template <int D>
__device__ __forceinline__ void splitk_item(const AttnParams &p, const SkItem it, const int g, uint8_t *smem) {
    constexpr int NCH = D / 8;   // 16-byte chunks per row
    constexpr int NKS = D / 16;  // k-steps over the head dim
    constexpr int NNT = D / 8;   // n-tiles over the head dim (PV)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const ReqDev rq = p.reqs[it.req];
    const int G = p.G_q;
    const int nrows = it.nrows;   // stacked rows x = hl0 + r: token j0 + x / G, q head g*G + x % G
    uint8_t *sQ = smem;
    uint8_t *sKV = smem + SkSmem<D>::kQ;

    // per-row causal limit (exclusive), rows this lane owns: r0 = lane/4, r1 = r0 + 8
    const int ra = lane >> 2, rb = ra + 8;
    auto row_lim = [&](int r) -> int {
        if (r >= nrows) return 0;
        if (it.mode) return it.k1;   // a prefix node: every member sees all of its keys
        const int lim = rq.c + it.j0 + (it.hl0 + r) / G + 1;
        return lim < it.k1 ? lim : it.k1;
    };
    const int lim_a = row_lim(ra), lim_b = row_lim(rb);

    // ---- this warp's blocks ----------------------------------------------------
    const int kb0 = it.k0 / kBlock;
    const int kb_end = (it.k1 + kBlock - 1) / kBlock;
    const int nblk_w = (kb_end - kb0 - warp + kSkWarps - 1) / kSkWarps;  // may be <= 0
    const int32_t *bt = p.bt_flat + rq.bt_off;
    uint8_t *sW = sKV + warp * SkSmem<D>::kWarp;
    const uint32_t sW_u = smem_u32(sW);
    const int64_t head_stride = (int64_t)kBlock * D;            // elements per (block, head)
    auto issue = [&](int bi, int stage) {
        const int kb = kb0 + warp + bi * kSkWarps;
        const int64_t base = ((int64_t)bt[kb] * p.H_kv + g) * head_stride;
        const uint16_t *gk = p.k_cache + base;
        const uint16_t *gv = p.v_cache + base;
        const uint32_t dk = sW_u + stage * SkSmem<D>::kStage;
        const uint32_t dv = dk + SkSmem<D>::kTile;
        if (p.k_new && (kb + 1) * kBlock > rq.c) {
            // the block holds this call's new tokens: read them from the step's inputs
            // (the append writing them into the cache runs beside this kernel)
#pragma unroll
            for (int i = 0; i < kBlock * NCH / 32; ++i) {
                const int id = lane + 32 * i;
                const int r = id / NCH, ch = id % NCH;
                const int pos = kb * kBlock + r;
                const uint16_t *sk = gk + r * D + ch * 8, *sv = gv + r * D + ch * 8;
                if (pos >= rq.c && pos < rq.c + rq.n) {
                    const int64_t off = ((int64_t)(rq.cu_q + pos - rq.c) * p.H_kv + g) * D + ch * 8;
                    sk = p.k_new + off;
                    sv = p.v_new + off;
                }
                cp_async16(dk + swz<D>(r, ch), sk);
                cp_async16(dv + swz<D>(r, ch), sv);
            }
            return;
        }
#pragma unroll
        for (int i = 0; i < kBlock * NCH / 32; ++i) {
            const int id = lane + 32 * i;
            const int r = id / NCH, ch = id % NCH;
            cp_async16(dk + swz<D>(r, ch), gk + r * D + ch * 8);
            cp_async16(dv + swz<D>(r, ch), gv + r * D + ch * 8);
        }
    };
    // ---- Q tile (16 rows, zero padded) -> smem (swizzled), asynchronously: its
    // loads are in flight together with the first K/V blocks' (one cp.async group
    // ahead of the prologue's), so an item's start-up pays one memory latency
    const uint32_t sQ_w = smem_u32(sQ);
    for (int idx = threadIdx.x; idx < kSkRows * NCH; idx += blockDim.x) {
        const int r = idx / NCH, ch = idx % NCH;
        const uint16_t *src = p.q;
        if (r < nrows) {
            const int x = it.hl0 + r;
            const int t = it.mode ? p.tc_tok[it.j0 + x / G] : rq.cu_q + it.j0 + x / G;
            const int h = g * G + x % G;
            HG_DCHECK(t >= 0 && t < p.T && h < p.H_q);
            src = p.q + ((int64_t)t * p.H_q + h) * D + ch * 8;
        }
        cp_async16_zfill(sQ_w + swz<D>(r, ch), src, r < nrows);
    }
    cp_async_commit();
#pragma unroll
    for (int b = 0; b < kSkStages - 1; ++b) {   // prologue: blocks 0 .. S-2 in flight
        if (b < nblk_w) issue(b, b);
        cp_async_commit();
    }
    cp_async_wait<kSkStages - 1>();   // the Q group (the prologue's blocks may still be in flight)
    __syncthreads();  // Q tile visible

    // Q A-fragments (all warps hold the same 16 x D tile)
    uint32_t qa[NKS][4];
    {
        const uint32_t sQ_u = smem_u32(sQ);
#pragma unroll
        for (int ks = 0; ks < NKS; ++ks) {
            const int r = lane & 15;
            const int ch = 2 * ks + (lane >> 4);
            ldsm_x4(sQ_u + swz<D>(r, ch), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
        }
    }

    float o[NNT][4];
#pragma unroll
    for (int nt = 0; nt < NNT; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float m_a = -CUDART_INF_F, m_b = -CUDART_INF_F;  // running max (log2 domain)
    float l_a = 0.f, l_b = 0.f;                      // per-lane partial sums

    for (int bi = 0; bi < nblk_w; ++bi) {
        const int stage = bi % kSkStages;
        if (bi + kSkStages - 1 < nblk_w) issue(bi + kSkStages - 1, (bi + kSkStages - 1) % kSkStages);
        cp_async_commit();
        cp_async_wait<kSkStages - 1>();
        __syncwarp();
        const uint32_t sk = sW_u + stage * SkSmem<D>::kStage;
        const uint32_t sv = sk + SkSmem<D>::kTile;
        // ---- S = Q K^T (16 rows x 16 keys) ----
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < NKS; ++ks) {
            uint32_t b0, b1, b2, b3;
            const int key = (lane & 7) + ((lane >> 4) << 3);
            const int ch = 2 * ks + ((lane >> 3) & 1);
            ldsm_x4(sk + swz<D>(key, ch), b0, b1, b2, b3);
            mma_bf16(s0, qa[ks], b0, b1);
            mma_bf16(s1, qa[ks], b2, b3);
        }
        // ---- mask + online softmax (rows ra, rb; cols 2*(lane&3)+{0,1} (+8)) ----
        const int kbase = (kb0 + warp + bi * kSkWarps) * kBlock;
        const int c0 = kbase + 2 * (lane & 3);
        float x[8];
        x[0] = (c0 < lim_a) ? s0[0] * p.scale_log2 : -CUDART_INF_F;
        x[1] = (c0 + 1 < lim_a) ? s0[1] * p.scale_log2 : -CUDART_INF_F;
        x[2] = (c0 < lim_b) ? s0[2] * p.scale_log2 : -CUDART_INF_F;
        x[3] = (c0 + 1 < lim_b) ? s0[3] * p.scale_log2 : -CUDART_INF_F;
        x[4] = (c0 + 8 < lim_a) ? s1[0] * p.scale_log2 : -CUDART_INF_F;
        x[5] = (c0 + 9 < lim_a) ? s1[1] * p.scale_log2 : -CUDART_INF_F;
        x[6] = (c0 + 8 < lim_b) ? s1[2] * p.scale_log2 : -CUDART_INF_F;
        x[7] = (c0 + 9 < lim_b) ? s1[3] * p.scale_log2 : -CUDART_INF_F;
        float mxa = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[4], x[5]));
        float mxb = fmaxf(fmaxf(x[2], x[3]), fmaxf(x[6], x[7]));
        mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 1));
        mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 2));
        mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 1));
        mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 2));
        const float mna = fmaxf(m_a, mxa), mnb = fmaxf(m_b, mxb);
        const float refa = (mna == -CUDART_INF_F) ? 0.f : mna;
        const float refb = (mnb == -CUDART_INF_F) ? 0.f : mnb;
        const float alpha_a = fast_exp2(m_a - refa), alpha_b = fast_exp2(m_b - refb);
        m_a = mna;
        m_b = mnb;
        float pr[8];
        pr[0] = fast_exp2(x[0] - refa); pr[1] = fast_exp2(x[1] - refa);
        pr[2] = fast_exp2(x[2] - refb); pr[3] = fast_exp2(x[3] - refb);
        pr[4] = fast_exp2(x[4] - refa); pr[5] = fast_exp2(x[5] - refa);
        pr[6] = fast_exp2(x[6] - refb); pr[7] = fast_exp2(x[7] - refb);
        l_a = l_a * alpha_a + (pr[0] + pr[1] + pr[4] + pr[5]);
        l_b = l_b * alpha_b + (pr[2] + pr[3] + pr[6] + pr[7]);
        if (__any_sync(0xffffffffu, alpha_a != 1.f || alpha_b != 1.f)) {
#pragma unroll
            for (int nt = 0; nt < NNT; ++nt) {
                o[nt][0] *= alpha_a; o[nt][1] *= alpha_a;
                o[nt][2] *= alpha_b; o[nt][3] *= alpha_b;
            }
        }
        // P as the A operand (16 x 16 keys): a0=(ra, k0..1) a1=(rb, k0..1) a2=(ra, k8..9) a3=(rb, k8..9)
        uint32_t pa[4];
        pa[0] = pack_bf16(pr[0], pr[1]);
        pa[1] = pack_bf16(pr[2], pr[3]);
        pa[2] = pack_bf16(pr[4], pr[5]);
        pa[3] = pack_bf16(pr[6], pr[7]);
        // ---- O += P V ----
#pragma unroll
        for (int c2 = 0; c2 < NNT / 2; ++c2) {
            uint32_t b0, b1, b2, b3;
            const int key = (lane & 7) + (((lane >> 3) & 1) << 3);
            const int ch = 2 * c2 + (lane >> 4);
            ldsm_x4_t(sv + swz<D>(key, ch), b0, b1, b2, b3);
            mma_bf16(o[2 * c2], pa, b0, b1);
            mma_bf16(o[2 * c2 + 1], pa, b2, b3);
        }
        __syncwarp();
    }
    cp_async_wait<0>();
    // ---- reduce l over the quad, then merge the 4 warps through smem ----------
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
    __syncthreads();  // all warps done with their KV stages
    // [warp][16][MS] (row stride D + 4 floats: the fragment stores' 8 rows and the
    // merge's 4 rows per quarter-warp land on distinct banks), then [warp][16][2]
    constexpr int MS = SkSmem<D>::kMS;
    float *mo = reinterpret_cast<float *>(sKV);
    float *mml = mo + kSkWarps * kSkRows * MS;
    {
        float *ow = mo + warp * kSkRows * MS;
        const int cc = 2 * (lane & 3);
#pragma unroll
        for (int nt = 0; nt < NNT; ++nt) {
            *reinterpret_cast<float2 *>(ow + ra * MS + nt * 8 + cc) = make_float2(o[nt][0], o[nt][1]);
            *reinterpret_cast<float2 *>(ow + rb * MS + nt * 8 + cc) = make_float2(o[nt][2], o[nt][3]);
        }
        if ((lane & 3) == 0) {
            mml[(warp * kSkRows + ra) * 2 + 0] = m_a;
            mml[(warp * kSkRows + ra) * 2 + 1] = l_a;
            mml[(warp * kSkRows + rb) * 2 + 0] = m_b;
            mml[(warp * kSkRows + rb) * 2 + 1] = l_b;
        }
    }
    __syncthreads();
    // 128 threads: thread -> (row r = tid / 8, columns 4 part8 + 32 k + [0, 4) for k < D/32:
    // a quarter-warp reads one row's 128 contiguous bytes per k, conflict-free)
    {
        const int r = threadIdx.x >> 3;
        const int part8 = threadIdx.x & 7;
        if (r < nrows) {
            float M = -CUDART_INF_F;
#pragma unroll
            for (int w = 0; w < kSkWarps; ++w) M = fmaxf(M, mml[(w * kSkRows + r) * 2]);
            const float ref = (M == -CUDART_INF_F) ? 0.f : M;
            float f[kSkWarps], L = 0.f;
#pragma unroll
            for (int w = 0; w < kSkWarps; ++w) {
                f[w] = fast_exp2(mml[(w * kSkRows + r) * 2] - ref);
                L += f[w] * mml[(w * kSkRows + r) * 2 + 1];
            }
            const float inv = L > 0.f ? 1.f / L : 0.f;
            const int x = it.hl0 + r;
            const int t = it.mode ? p.tc_tok[it.j0 + x / G] : rq.cu_q + it.j0 + x / G;
            const int h = g * G + x % G;
            int base = -1;
            if (it.part >= 0) {
                const TokDev tk = p.tok[t];
                base = tk.base + g * tk.nparts * G;
            }
            constexpr int PER = D / 8;
            float acc[PER];
#pragma unroll
            for (int e = 0; e < PER; ++e) acc[e] = 0.f;
#pragma unroll
            for (int w = 0; w < kSkWarps; ++w) {
                const float fw = f[w] * inv;
                const float *src = mo + (w * kSkRows + r) * MS + part8 * 4;
#pragma unroll
                for (int k = 0; k < PER / 4; ++k) {
                    const float4 v = *reinterpret_cast<const float4 *>(src + 32 * k);
                    acc[4 * k] += fw * v.x;
                    acc[4 * k + 1] += fw * v.y;
                    acc[4 * k + 2] += fw * v.z;
                    acc[4 * k + 3] += fw * v.w;
                }
            }
            const float lse2 = (L > 0.f) ? ref + __log2f(L) : -CUDART_INF_F;
            if (base < 0) {
                // sharded call: the entry barrier kernel ahead of this grid (programmatic
                // dependency) must be through before the first store into a peer's window
                wait_entry(p);
                const int64_t off = (int64_t)t * p.out_ld + (int64_t)h * D + part8 * 4;
#pragma unroll
                for (int k = 0; k < PER / 4; ++k) {
                    uint2 v;
                    v.x = pack_bf16(acc[4 * k + 0], acc[4 * k + 1]);
                    v.y = pack_bf16(acc[4 * k + 2], acc[4 * k + 3]);
                    for (int o2 = 0; o2 < p.n_out; ++o2) *reinterpret_cast<uint2 *>(p.outs[o2] + off + 32 * k) = v;
                }
                if (p.lse && part8 == 0) p.lse[(int64_t)t * p.H_q + h] = lse2 * 0.69314718055994531f;
            } else {
                const int64_t slot = base + (int64_t)it.part * G + (x % G);
                HG_DCHECK(slot >= 0 && slot < p.n_slots && it.part < p.tok[t].nparts);
                float *dst = p.part_o + slot * D + part8 * 4;
#pragma unroll
                for (int k = 0; k < PER / 4; ++k)
                    *reinterpret_cast<float4 *>(dst + 32 * k) =
                        make_float4(acc[4 * k], acc[4 * k + 1], acc[4 * k + 2], acc[4 * k + 3]);
                if (part8 == 0) p.part_lse[slot] = lse2;
            }
        }
    }
    // ---- in-kernel merge (no combine kernel; every partial comes from this grid) ----
    // Each token this item wrote partials for counts one arrival per (token, KV head);
    // the CTA bringing the count to nparts x (head chunks) merges the token's G rows.
    // Release: every writer fences, then the CTA barrier, then the counting atomics
    // (the threadFenceReduction pattern); acquire: a fence after the winning atomic,
    // partials read through L2.
    if (p.sk_cnt && it.part >= 0) {
        __shared__ uint32_t s_win;
        __threadfence();
        if (threadIdx.x == 0) s_win = 0;
        __syncthreads();
        const int u0 = it.hl0 / G, u1 = (it.hl0 + nrows - 1) / G;   // local token range of the rows
        const int nu = u1 - u0 + 1;                                // <= 16
        if ((int)threadIdx.x < nu) {
            const int u = u0 + threadIdx.x;
            const int t = it.mode ? p.tc_tok[it.j0 + u] : rq.cu_q + it.j0 + u;
            const int need = p.tok[t].nparts * (G > kSkRows ? (G + kSkRows - 1) / kSkRows : 1);
            const unsigned old = atomicAdd(p.sk_cnt + (int64_t)t * p.H_kv + g, 1u);
            HG_DCHECK(old < (unsigned)need);   // no more arrivals than the token has parts
            if (old == (unsigned)need - 1) atomicOr(&s_win, 1u << threadIdx.x);
        }
        __syncthreads();
        uint32_t win = s_win;
        if (win) {
            __threadfence();
            wait_entry(p);   // peer-window stores follow
            // rows (u, hl) of the winning tokens, one warp each
            const int nw = __popc(win);
            for (int k = warp; k < nw * G; k += kSkWarps) {
                uint32_t m = win;
                for (int z = k / G; z > 0; --z) m &= m - 1;
                const int u = u0 + __ffs(m) - 1;
                const int t = it.mode ? p.tc_tok[it.j0 + u] : rq.cu_q + it.j0 + u;
                combine_row<D>(p, t, g, k % G, lane);
            }
        }
    }
}

// Persistent split-K grid: CTA (b, g) runs the items [sk_off[b], sk_off[b+1]) for
// KV head g (stream-K plans give every CTA the same number of KV blocks).
template <int D>
#ifndef HG_SK_MIN_CTAS
#define HG_SK_MIN_CTAS 3
#endif
__global__ void __launch_bounds__(kSkWarps * 32, HG_SK_MIN_CTAS)   // 3 CTAs per SM: <= 170 registers
splitk_kernel(const AttnParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    // the combine kernel behind this one (programmatic dependent launch) may be
    // scheduled as soon as every CTA of this grid has started; it waits for this
    // grid's completion in griddepcontrol.wait
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int g = blockIdx.y;   // KV head
    const int i0 = p.sk_off[blockIdx.x], i1 = p.sk_off[blockIdx.x + 1];
    if (p.entry_word && threadIdx.x < 32) {
        // folded entry barrier: the first CTA to start (so one that is resident) runs the
        // peer-window flag barrier and publishes its passage; every CTA waits for that
        // only before its first peer-window store (wait_entry)
        unsigned int first = 0;
        if (threadIdx.x == 0) first = atomicAdd(p.entry_word, 1u) == 0;
        if (__shfl_sync(0xffffffffu, first, 0)) {
            peer_barrier_body(p.bar_flags, p.bar_mine, p.bar_rank, p.bar_world, p.bar_epoch, threadIdx.x);
            __syncwarp();
            if (threadIdx.x == 0) {
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], 1;\n" ::"l"(p.entry_word + 1) : "memory");
            }
        }
    }
    long long *tr = p.sk_trace ? p.sk_trace + 2 * ((int64_t)g * gridDim.x + blockIdx.x) : nullptr;
    if (tr && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(tr[0]));
    for (int i = i0; i < i1; ++i) {
        if (i > i0) __syncthreads();   // the previous item's merge has read its smem
        splitk_item<D>(p, p.sk[i], g, smem);
    }
    if (tr) {
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(tr[1]));
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;\n" : "=r"(smid));
            p.sk_trace[2 * (int64_t)gridDim.x * gridDim.y + (int64_t)g * gridDim.x + blockIdx.x] = smid;
        }
    }
    // this grid completes only after the entry barrier ahead of it: the combine behind
    // it (which waits for this grid) stores into peers' windows only after the barrier
    if (p.bar_pdl || p.entry_word) {
        if (threadIdx.x == 0) wait_entry(p);
        __syncthreads();
    }
    if (p.exit_epoch) {
        // folded exit barrier: every CTA releases its stores at GPU scope and takes a
        // ticket; the last one (acquire) waits for the side-stream append's count, then
        // runs the flag barrier, whose system-scope release is cumulative over every
        // store it has observed
        __shared__ int s_last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned tk = atomicAdd(p.exit_ticket, 1u);
            HG_DCHECK(tk < gridDim.x * gridDim.y);
            s_last = tk == gridDim.x * gridDim.y - 1;
        }
        __syncthreads();
        if (s_last && threadIdx.x < 32) {
            __threadfence();
            if (p.exit_wait_cnt && threadIdx.x == 0) {
                unsigned long long c;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(c) : "l"(p.exit_wait_cnt) : "memory");
                    if (c >= p.exit_wait_target) break;
                    __nanosleep(64);
                }
            }
            __syncwarp();
            peer_barrier_body(p.bar_flags, p.bar_mine, p.bar_rank, p.bar_world, p.exit_epoch, threadIdx.x);
        }
    }
}

// Launch with the programmatic-stream-serialization attribute (pdl = true): the
// kernel may start before the previous kernel in the stream has finished; it
// must execute griddepcontrol.wait before touching that kernel's results.
template <typename... Args>
static cudaError_t launch_maybe_pdl(void (*kern)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                    bool pdl, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int D>
static hg_status launch_splitk_d(const AttnParams &p, cudaStream_t st) {
    constexpr int bytes = SkSmem<D>::kBytes;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(splitk_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        attr = true;
    }
    cudaError_t e = launch_maybe_pdl(splitk_kernel<D>, dim3(p.sk_ctas, p.H_kv), dim3(kSkWarps * 32), (size_t)bytes, st,
                                     p.bar_pdl != 0, p);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "split-K launch: %s", cudaGetErrorString(e));
}

hg_status launch_splitk(const AttnParams &p, void *stream) {
    if (p.n_sk == 0) return HG_OK;
    if (p.d == 128) return launch_splitk_d<128>(p, (cudaStream_t)stream);
    if (p.d == 64) return launch_splitk_d<64>(p, (cudaStream_t)stream);
    return fail(HG_E_UNSUPPORTED, "head_dim %d", p.d);
}

// ----------------------------------------------------------------------------
// a.7 combine: O = sum_s 2^{lse_s - LSE} o_s, LSE = log2 sum_s 2^{lse_s}
// one warp per (merged token, KV head, q-head-in-group)
// ----------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) combine_kernel(const AttnParams p) {
    // launched as a programmatic dependent of split-K: resident early, reads the
    // partials only once that grid has completed and its writes are visible
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int G = p.G_q;
    if (wid >= (int64_t)p.n_comb * p.H_kv * G) return;
    const int t = p.comb[wid / (p.H_kv * G)];
    const int rem = (int)(wid % (p.H_kv * G));
    combine_row<D>(p, t, rem / G, rem % G, lane);
}

hg_status launch_combine(const AttnParams &p, void *stream, bool pdl) {
    if (p.n_comb == 0) return HG_OK;
    const int64_t warps = (int64_t)p.n_comb * p.H_kv * p.G_q;
    const int blocks = (int)((warps * 32 + 255) / 256);
    cudaError_t e;
    if (p.d == 128) e = launch_maybe_pdl(combine_kernel<128>, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, pdl, p);
    else if (p.d == 64) e = launch_maybe_pdl(combine_kernel<64>, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, pdl, p);
    else return fail(HG_E_UNSUPPORTED, "head_dim %d", p.d);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "combine launch: %s", cudaGetErrorString(e));
}

}  // namespace hg

namespace hg {
// [G][T][E] -> [T][G][E] (E = H_q/G * d bf16 elements), 16-byte chunks.
__global__ void gather_transpose_kernel(const uint4 *__restrict__ src, uint4 *__restrict__ dst, int G, int T,
                                        int chunks) {
    const int64_t total = (int64_t)G * T * chunks;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % chunks);
        const int64_t rt = i / chunks;
        const int t = (int)(rt % T);
        const int r = (int)(rt / T);
        dst[((int64_t)t * G + r) * chunks + c] = src[i];
    }
}

hg_status launch_gather_transpose(const uint16_t *src, uint16_t *dst, int G, int T, int row_elems, void *stream) {
    const int chunks = row_elems / 8;
    const int64_t total = (int64_t)G * T * chunks;
    if (total == 0) return HG_OK;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
    gather_transpose_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((const uint4 *)src, (uint4 *)dst, G, T, chunks);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "transpose launch: %s", cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// Peer-window barrier.  Thread k (< world) publishes `epoch`
// into rank k's flag slot [rank] with a system-scope release store, then waits
// (acquire) until rank k's own arrival shows up in the local slot [k].  Flags
// only grow, so no reset is needed.  Kernels earlier in the stream have
// completed, so their peer stores precede the release.  A peer that never
// arrives is a broken job: after ~30 s the kernel traps (sticky HG_E_CUDA)
// instead of hanging the GPU.
// ---------------------------------------------------------------------------
struct PeerFlags {
    unsigned long long *flags[kMaxOuts];  // flags[k]: rank k's flag array (peer mapping)
};

__global__ void peer_barrier_kernel(PeerFlags pf, unsigned long long *mine, int rank, int world,
                                    unsigned long long epoch, const unsigned long long *wait_cnt,
                                    unsigned long long wait_target) {
    // as a programmatic dependent of the attention's last kernel: resident early,
    // the barrier starts once that kernel's peer stores are complete
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (wait_cnt) {   // the call's side-stream append has counted every CTA (long done by now)
        unsigned long long c;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(c) : "l"(wait_cnt) : "memory");
            if (c >= wait_target) break;
            __nanosleep(64);
        }
    }
    // as the entry barrier: the attention grid behind it may launch at once (it waits
    // for this grid in griddepcontrol.wait before its first peer-window store)
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    peer_barrier_body(pf.flags, mine, rank, world, epoch, threadIdx.x);
}

hg_status launch_peer_barrier(unsigned long long *const *flags, unsigned long long *mine, int rank, int world,
                              unsigned long long epoch, void *stream, bool pdl, const unsigned long long *wait_cnt,
                              unsigned long long wait_target) {
    PeerFlags pf{};
    for (int k = 0; k < world; ++k) pf.flags[k] = flags[k];
    cudaError_t e = launch_maybe_pdl(peer_barrier_kernel, dim3(1), dim3(32), 0, (cudaStream_t)stream, pdl, pf, mine,
                                     rank, world, epoch, wait_cnt, wait_target);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e == cudaSuccess ? HG_OK : fail(HG_E_CUDA, "peer barrier launch: %s", cudaGetErrorString(e));
}
}  // namespace hg
