/*
 * oracle.c -- plain, slow, fp64 CPU oracle for one hybrid serving iteration's
 * attention over a paged KV cache.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header or constant with paper_2501_14808_b200/ (the product).
 *
 * What it follows (PAPER.md = P):
 *   - A batch is a set of requests, each contributing l new tokens this
 *     iteration (Alg. 1 tuples (r, l, t_req)); chunked-prefill
 *     rows and decode rows are "processed together within a single
 *     iteration".  Request i has c_i cached tokens and n_i new tokens.
 *   - KV memory is counted in blocks, GET_NUM_BLOCKS(l); the cache
 *     is paged: position p of request i lives in physical block
 *     bt[i][p / B] at offset p % B.
 *   - The cost the predictor models is attention's: "quadratic complexity due
 *     to attention" for prefill, "linear scaling" for decode.
 *     The paper never writes the attention formula; we take the standard
 *     scaled-dot-product attention with causal masking aligned to the
 *     request's absolute positions (readings R1-R4):
 *
 *       for row j of request i (absolute position c_i + j), q-head h,
 *       KV head g = floor(h / (H_q / H_kv)):
 *         s_p = (sum_k Q[t][h][k] * K_i(p)[g][k]) / sqrt(d),  p = 0 .. c_i+j
 *         m   = max_p s_p,  w_p = exp(s_p - m),  l = sum_p w_p
 *         O[t][h] = sum_p w_p * V_i(p)[g] / l,  LSE[t][h] = m + ln l
 *
 *     summed in increasing p and increasing k, all in fp64 (bf16 -> fp64 is
 *     exact).  oracle_attention_range restricts p to [lo, hi) and returns the
 *     partial (o, m, l) triple used to pin split-K / prefix merging.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC oracle.c -o liboracle.so -lm
 * (no -ffast-math: the order of operations above is the specification).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static double bf16_to_f64(uint16_t b) {
    uint32_t u = ((uint32_t)b) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

/* Append: token j of request i goes to position c_i + j.
 * Pure copy of bf16 bits.  Returns 0, or -1 if a block id is out of range. */
int oracle_append(uint16_t *Kc, uint16_t *Vc, int64_t num_blocks, int H_kv, int B, int d,
                  int R, const int32_t *bt, int W, const int32_t *c, const int32_t *n,
                  const uint16_t *Knew, const uint16_t *Vnew) {
    int64_t t = 0;
    for (int i = 0; i < R; ++i) {
        for (int j = 0; j < n[i]; ++j, ++t) {
            int64_t p = (int64_t)c[i] + j;
            int64_t col = p / B;
            if (col >= W) return -1;
            int64_t b = bt[(int64_t)i * W + col];
            if (b < 0 || b >= num_blocks) return -1;
            int64_t o = p % B;
            for (int g = 0; g < H_kv; ++g) {
                int64_t dst = ((b * H_kv + g) * B + o) * d;
                int64_t src = (t * H_kv + g) * (int64_t)d;
                memcpy(Kc + dst, Knew + src, (size_t)d * sizeof(uint16_t));
                memcpy(Vc + dst, Vnew + src, (size_t)d * sizeof(uint16_t));
            }
        }
    }
    return 0;
}

/* Attention over keys p in [lo, min(hi, c_i + j + 1)) for the selected
 * requests (req_sel == NULL: all).  Outputs, indexed by the batch token t:
 *   out [T][H_q][d]  o = sum w_p v_p / l   (0 when the range is empty)
 *   mx  [T][H_q]     m (or -inf)
 *   sm  [T][H_q]     l (or 0)
 *   lse [T][H_q]     m + ln l (or -inf)
 * Any of mx/sm/lse may be NULL.  hi < 0 means "no upper cap".
 * Returns 0, or -1 on an invalid block id / shape. */
int oracle_attention_range(const uint16_t *Kc, const uint16_t *Vc, int64_t num_blocks,
                           int H_kv, int B, int d, int R, const int32_t *bt, int W,
                           const int32_t *c, const int32_t *n, const uint16_t *Q, int H_q,
                           const int32_t *req_sel, int n_sel, int64_t lo, int64_t hi,
                           double *out, double *mx, double *sm, double *lse) {
    if (H_kv <= 0 || H_q % H_kv != 0) return -1;
    int G = H_q / H_kv;
    int64_t *cu = (int64_t *)malloc(sizeof(int64_t) * (size_t)(R + 1));
    cu[0] = 0;
    for (int i = 0; i < R; ++i) cu[i + 1] = cu[i] + n[i];
    int nreq = req_sel ? n_sel : R;
    /* flatten (request, row) pairs of the selection */
    int64_t rows = 0;
    for (int k = 0; k < nreq; ++k) rows += n[req_sel ? req_sel[k] : k];
    int64_t *row_i = (int64_t *)malloc(sizeof(int64_t) * (size_t)(rows > 0 ? rows : 1));
    int64_t *row_j = (int64_t *)malloc(sizeof(int64_t) * (size_t)(rows > 0 ? rows : 1));
    int64_t r = 0;
    for (int k = 0; k < nreq; ++k) {
        int i = req_sel ? req_sel[k] : k;
        for (int j = 0; j < n[i]; ++j, ++r) { row_i[r] = i; row_j[r] = j; }
    }
    int bad = 0;
    const double inv_sqrt_d = 1.0 / sqrt((double)d);
    int64_t total = rows * H_q;
#pragma omp parallel for schedule(dynamic, 4) reduction(|| : bad)
    for (int64_t w = 0; w < total; ++w) {
        int64_t rr = w / H_q;
        int h = (int)(w % H_q);
        int64_t i = row_i[rr], j = row_j[rr];
        int64_t t = cu[i] + j;
        int g = h / G;
        int64_t kend = (int64_t)c[i] + j + 1;          /* causal: keys 0 .. c_i + j */
        if (hi >= 0 && hi < kend) kend = hi;
        int64_t kbeg = lo > 0 ? lo : 0;
        int64_t L = kend - kbeg;
        double *o = out + (t * H_q + h) * (int64_t)d;
        for (int k = 0; k < d; ++k) o[k] = 0.0;
        if (L <= 0) {
            if (mx) mx[t * H_q + h] = -INFINITY;
            if (sm) sm[t * H_q + h] = 0.0;
            if (lse) lse[t * H_q + h] = -INFINITY;
            continue;
        }
        double *q = (double *)malloc(sizeof(double) * (size_t)d);
        double *s = (double *)malloc(sizeof(double) * (size_t)L);
        const uint16_t *qb = Q + (t * H_q + h) * (int64_t)d;
        for (int k = 0; k < d; ++k) q[k] = bf16_to_f64(qb[k]);
        double m = -INFINITY;
        for (int64_t p = kbeg; p < kend; ++p) {
            int64_t col = p / B;
            int64_t b = col < W ? bt[i * W + col] : -1;
            if (b < 0 || b >= num_blocks) { bad = 1; s[p - kbeg] = 0.0; continue; }
            const uint16_t *kr = Kc + ((b * H_kv + g) * B + p % B) * (int64_t)d;
            double acc = 0.0;
            for (int k = 0; k < d; ++k) acc += q[k] * bf16_to_f64(kr[k]);
            s[p - kbeg] = acc * inv_sqrt_d;
            if (s[p - kbeg] > m) m = s[p - kbeg];
        }
        double l = 0.0;
        for (int64_t p = kbeg; p < kend; ++p) {
            double wp = exp(s[p - kbeg] - m);
            s[p - kbeg] = wp;
            l += wp;
        }
        for (int64_t p = kbeg; p < kend; ++p) {
            int64_t col = p / B;
            int64_t b = col < W ? bt[i * W + col] : -1;
            if (b < 0 || b >= num_blocks) continue;
            const uint16_t *vr = Vc + ((b * H_kv + g) * B + p % B) * (int64_t)d;
            double wp = s[p - kbeg];
            for (int k = 0; k < d; ++k) o[k] += wp * bf16_to_f64(vr[k]);
        }
        for (int k = 0; k < d; ++k) o[k] /= l;
        if (mx) mx[t * H_q + h] = m;
        if (sm) sm[t * H_q + h] = l;
        if (lse) lse[t * H_q + h] = m + log(l);
        free(q);
        free(s);
    }
    free(cu);
    free(row_i);
    free(row_j);
    return bad ? -1 : 0;
}

/* Full attention (all keys 0 .. c_i + j). */
int oracle_attention(const uint16_t *Kc, const uint16_t *Vc, int64_t num_blocks, int H_kv, int B,
                     int d, int R, const int32_t *bt, int W, const int32_t *c, const int32_t *n,
                     const uint16_t *Q, int H_q, const int32_t *req_sel, int n_sel, double *out,
                     double *lse) {
    return oracle_attention_range(Kc, Vc, num_blocks, H_kv, B, d, R, bt, W, c, n, Q, H_q, req_sel,
                                  n_sel, 0, -1, out, NULL, NULL, lse);
}

/* Thread count for the following parallel regions (the host's cores: SURVEY
 * §8(d)); overrides OMP_NUM_THREADS, which torchrun pins to 1. */
void oracle_set_num_threads(int nt) {
#ifdef _OPENMP
    if (nt > 0) omp_set_num_threads(nt);
#else
    (void)nt;
#endif
}

int oracle_num_threads(void) {
    int nt = 1;
#ifdef _OPENMP
#pragma omp parallel
    {
#pragma omp single
        nt = omp_get_num_threads();
    }
#endif
    return nt;
}
