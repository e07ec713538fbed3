/*
 * tg_oracle.c — CPU oracle for the Tarragon MoE-layer round trip.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA product path
 * (paper_2601_01310_b200/csrc); neither includes or links the other.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   out[t] = sum_{e in TopK(t)} w_{t,e} * FFN_e(x_t)   (+ FFN_sh(x_t))
 *   "a gating network that selects only the top-k experts for each token ...
 *    the resulting expert outputs are aggregated via a weighted sum using the
 *    gating weights"                                        (§2.1)
 * plus the routing that the method uses to reach it: the Expert Routing Table
 * (ERT) lookup that maps an expert to its first healthy candidate EW, i.e. a
 * primary or a shadow replica (§4.2, §5.1
 * §5.3), and the layer-wise per-(expert) batching permutation on the EWs
 * (§2.2.1).  Every step below is written in the paper's order; the
 * readings of points the paper leaves open are listed in DESIGN.md §3 and
 * referenced here as "R#n".
 *
 * Precision: floating-point arithmetic is fp64 (the paper fixes none).  The
 * method's storage formats are kept: x, weights, h, y and out are bf16
 * (R#7: the paper's AW<->EW volume V = 2*Top_k*N_hidden*S_elem with
 * S_elem = 2 B, App. C), router logits and gate weights are fp32
 * ("fp32 top-k gating", BASELINE.json north_star).  Rounding to bf16 is
 * round-to-nearest-even of the fp64 value (orc_bf16_from_f64), implemented
 * here from the IEEE-754 definition.
 *
 * Parity pins (tests/test_oracle_pins.py): hand-computed worked example
 * (tests/golden/worked_example.json), brute-force top-k with forced ties,
 * dense special cases against torch fp64, exhaustive bf16 rounding against
 * torch, invariants.  Unpinned: none of the functions below.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ERR_INVALID (-1)
#define ORC_ERR_NO_ROUTE (-2)
#define ORC_MAX_K 64

/* ------------------------------------------------------------------ bf16 */

/* bf16 bits -> exact double (bf16 is the top half of an IEEE binary32). */
static double orc_bf16_to_f64(uint16_t b) {
    uint32_t u = ((uint32_t)b) << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* Round an fp64 value to the nearest bf16 (ties to even), directly from the
 * binary64 encoding: bf16 has 8 significant bits and the binary32 exponent
 * range (normals and subnormals).  Overflow goes to +-inf; NaN stays NaN. */
uint16_t orc_bf16_from_f64(double v) {
    uint64_t u;
    memcpy(&u, &v, 8);
    uint16_t sign = (uint16_t)((u >> 48) & 0x8000u);
    int e = (int)((u >> 52) & 0x7FF);
    uint64_t m = u & 0x000FFFFFFFFFFFFFull;
    if (e == 0x7FF) return m ? (uint16_t)(sign | 0x7FC0u) : (uint16_t)(sign | 0x7F80u);
    if (e == 0 && m == 0) return sign;
    /* value = 1.m * 2^(e-1023) for normals; fp64 subnormals are far below bf16 range */
    if (e == 0) return sign; /* |v| < 2^-1022: rounds to zero in bf16 */
    int exp2 = e - 1023;                      /* unbiased exponent */
    uint64_t sig = (1ull << 52) | m;          /* 53-bit significand */
    /* bf16 normal: exponent in [-126, 127], 8 significant bits.
     * bf16 subnormal: quantum 2^-133.  Quantum of the target format: */
    int q = (exp2 >= -126) ? (exp2 - 7) : -133;   /* value of one ulp: 2^q */
    /* number of ulps = sig * 2^(exp2-52) / 2^q = sig >> (52 - exp2 + q) */
    int shift = 52 - exp2 + q;                /* 45 for normals, >= 46 below */
    if (shift >= 55) return sign;             /* |v| < half a quantum: rounds to zero */
    uint64_t n = sig >> shift;
    uint64_t rem = sig & ((1ull << shift) - 1);
    uint64_t half = 1ull << (shift - 1);
    if (rem > half || (rem == half && (n & 1))) n += 1;
    /* n ulps of 2^q.  Re-encode. */
    if (exp2 >= -126) {
        /* n in [128, 256]; 256 means carry into the next binade */
        int be = exp2 + 127;
        if (n == 256) { n = 128; be += 1; }
        if (be >= 255) return (uint16_t)(sign | 0x7F80u);
        return (uint16_t)(sign | (uint16_t)(be << 7) | (uint16_t)(n & 0x7F));
    } else {
        /* subnormal: n in [0, 128]; 128 becomes the smallest normal (exp field 1) */
        return (uint16_t)(sign | (uint16_t)n);
    }
}

void orc_bf16_from_f64_array(const double *v, uint16_t *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_bf16_from_f64(v[i]);
}

/* fp32 inputs, for the exhaustive pin: every binary32 is exact in binary64. */
void orc_bf16_from_f32_array(const float *v, uint16_t *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_bf16_from_f64((double)v[i]);
}

/* ---------------------------------------------------------- O1 router */

/* O1  l[t][e] = fp32( sum_i x[t][i] * Wg[e][i] )  — accumulated in fp64,
 * rounded once to fp32.  "gating network" (§2.1); R#1: linear router,
 * no bias; "fp32 top-k gating" (north_star). */
void orc_router(const uint16_t *x, const uint16_t *wg, int T, int d, int E, float *logits) {
    for (int t = 0; t < T; ++t)
        for (int e = 0; e < E; ++e) {
            double acc = 0.0;
            for (int i = 0; i < d; ++i)
                acc += orc_bf16_to_f64(x[(int64_t)t * d + i]) * orc_bf16_to_f64(wg[(int64_t)e * d + i]);
            logits[(int64_t)t * E + e] = (float)acc;
        }
}

/* O1 before its fp32 rounding (parity tests): l_exact[t][e] in fp64 and
 * s[t][e] = sum_i |x Wg| (the scale of a floating-point evaluation's error). */
void orc_router_f64(const uint16_t *x, const uint16_t *wg, int T, int d, int E, double *l, double *s) {
    for (int t = 0; t < T; ++t)
        for (int e = 0; e < E; ++e) {
            double acc = 0.0, sa = 0.0;
            for (int i = 0; i < d; ++i) {
                double p = orc_bf16_to_f64(x[(int64_t)t * d + i]) * orc_bf16_to_f64(wg[(int64_t)e * d + i]);
                acc += p;
                sa += fabs(p);
            }
            l[(int64_t)t * E + e] = acc;
            s[(int64_t)t * E + e] = sa;
        }
}


/* ---------------------------------------------------- O2/O3 top-k, softmax */

/* O2  S_t = the k experts first in the order (−l, e) ascending, i.e. largest
 *     logit first, equal logits broken by lowest expert id (R#3).  Slots j
 *     are the selected ids in ascending id order (R#4).
 *     gap_t = l_(k) − l_(k+1) in that order; +inf if k == E (there is no
 *     (k+1)-th logit, so no selection can flip: the near-tie rule of the
 *     north_star, "the k-th and (k+1)-th gate logits differ by less than
 *     1e-5", never applies).
 * O3  w_j = exp(l_j − m) / sum_j' exp(l_j' − m), m = max selected logit,
 *     computed in fp64 from the fp32 logits and rounded once to fp32
 *     (R#1/R#2: softmax over the k selected logits = renormalised top-k).
 * Returns ORC_OK. */
/* O3' (gate_mode 1, NEXT-3b: the public DS-V2-Lite / Qwen1.5-MoE routers,
 *     norm_topk_prob = false; R#2 variant): softmax over ALL E
 *     logits, the k selected weights are NOT renormalised:
 *     w_j = exp(l_j − M) / sum_{e<E} exp(l_e − M), M = max over all E, fp64.
 *     Selection (O2) is unchanged. */
int orc_select_mode(const float *logits, int T, int E, int k, int mode, int32_t *idx, float *w, float *gap);

int orc_select(const float *logits, int T, int E, int k, int32_t *idx, float *w, float *gap) {
    return orc_select_mode(logits, T, E, k, 0, idx, w, gap);
}

int orc_select_mode(const float *logits, int T, int E, int k, int mode, int32_t *idx, float *w, float *gap) {
    if (k < 1 || k > E || k > ORC_MAX_K || mode < 0 || mode > 1) return ORC_ERR_INVALID;
    int *order = (int *)malloc(sizeof(int) * E);
    int *sel = (int *)malloc(sizeof(int) * k);
    for (int t = 0; t < T; ++t) {
        const float *l = logits + (int64_t)t * E;
        /* selection sort of the first k+1 positions by key (−l, e) */
        for (int e = 0; e < E; ++e) order[e] = e;
        int lim = (k < E) ? k + 1 : k;
        for (int p = 0; p < lim; ++p) {
            int best = p;
            for (int q = p + 1; q < E; ++q) {
                float lq = l[order[q]], lb = l[order[best]];
                /* float compare: -0 == +0 is a tie */
                if (lq > lb || (lq == lb && order[q] < order[best])) best = q;
            }
            int tmp = order[p]; order[p] = order[best]; order[best] = tmp;
        }
        if (gap) gap[t] = (k < E) ? (l[order[k - 1]] - l[order[k]]) : INFINITY;
        /* ascending expert id within the selected set */
        for (int j = 0; j < k; ++j) sel[j] = order[j];
        for (int a = 1; a < k; ++a) {
            int v = sel[a], b = a - 1;
            while (b >= 0 && sel[b] > v) { sel[b + 1] = sel[b]; --b; }
            sel[b + 1] = v;
        }
        double m = -INFINITY;
        for (int j = 0; j < k; ++j) if ((double)l[sel[j]] > m) m = (double)l[sel[j]];
        double z[ORC_MAX_K];
        double Z = 0.0;
        for (int j = 0; j < k; ++j) { z[j] = exp((double)l[sel[j]] - m); Z += z[j]; }
        if (mode == 1) {  /* full softmax denominator; the max over all E is the max selected */
            Z = 0.0;
            for (int e = 0; e < E; ++e) Z += exp((double)l[e] - m);
        }
        for (int j = 0; j < k; ++j) {
            idx[(int64_t)t * k + j] = sel[j];
            w[(int64_t)t * k + j] = (float)(z[j] / Z);
        }
    }
    free(order);
    free(sel);
    return ORC_OK;
}

/* ------------------------------------------------------------ O4 resolve */

/* O4  ERT lookup with masked-EW redirect (§4.2; §5.1):
 *     (ew_e, slot_e) = first candidate (ew, slot) of cand[e][0..C) with
 *     ew >= 0 and !mask[ew] (R#8, "first healthy").
 *     rank_e = ew_rank[ew_e]; bank_e = ew_slot_base[ew_e] + slot_e.
 *     Experts with no live candidate get rank_e = bank_e = -1.
 * Returns ORC_OK, or ORC_ERR_NO_ROUTE if some expert has none (R#9). */
int orc_resolve(int E, int C, const int32_t *cand, const int32_t *ew_rank,
                const int32_t *ew_slot_base, const uint8_t *mask,
                int32_t *rank_e, int32_t *bank_e) {
    int rc = ORC_OK;
    for (int e = 0; e < E; ++e) {
        rank_e[e] = -1; bank_e[e] = -1;
        for (int c = 0; c < C; ++c) {
            int ew = cand[((int64_t)e * C + c) * 2 + 0];
            int sl = cand[((int64_t)e * C + c) * 2 + 1];
            if (ew < 0) continue;
            if (mask[ew]) continue;
            rank_e[e] = ew_rank[ew];
            bank_e[e] = ew_slot_base[ew] + sl;
            break;
        }
        if (rank_e[e] < 0) rc = ORC_ERR_NO_ROUTE;
    }
    return rc;
}

/* --------------------------------------------------------- O5 permutation */

/* O5  Layer-wise batching per (EW, expert) (§2.2.1): a stable counting
 *     sort of all pairs (t, j), visited in (global t, j) order, by key
 *     (rank_e, bank_e) of e = idx[t][j].  On rank q the receive buffer holds
 *     bank slots in ascending order; inside a slot, rows are in ascending
 *     global t (R#12: tokens are split contiguously over ranks, so source
 *     rank then local t == global t).
 *     dst_pos(t,j) = (rows of lower slots on that rank) + (rank of t in slot).
 *     counts[q][s] = rows of bank slot s on rank q (S_max slots per rank).
 * Returns ORC_OK, or ORC_ERR_NO_ROUTE if a selected expert is unroutable. */
int orc_permute(int T, int k, const int32_t *idx, const int32_t *rank_e, const int32_t *bank_e,
                int G, int S_max, int32_t *dst_rank, int32_t *dst_slot, int32_t *dst_pos,
                int32_t *counts) {
    memset(counts, 0, sizeof(int32_t) * (size_t)G * S_max);
    for (int64_t p = 0; p < (int64_t)T * k; ++p) {
        int e = idx[p];
        if (rank_e[e] < 0) return ORC_ERR_NO_ROUTE;
        if (rank_e[e] >= G || bank_e[e] >= S_max) return ORC_ERR_INVALID;
        counts[rank_e[e] * S_max + bank_e[e]] += 1;
    }
    int32_t *base = (int32_t *)malloc(sizeof(int32_t) * (size_t)G * S_max);
    for (int q = 0; q < G; ++q) {
        int32_t run = 0;
        for (int s = 0; s < S_max; ++s) { base[q * S_max + s] = run; run += counts[q * S_max + s]; }
    }
    for (int t = 0; t < T; ++t)
        for (int j = 0; j < k; ++j) {
            int64_t p = (int64_t)t * k + j;
            int e = idx[p];
            int q = rank_e[e], s = bank_e[e];
            dst_rank[p] = q;
            dst_slot[p] = s;
            dst_pos[p] = base[q * S_max + s]++;
        }
    free(base);
    return ORC_OK;
}

/* ------------------------------------------------------------ O6/O7 FFN */

/* O6  Expert FFN, SwiGLU form (R#6; Mixtral w1/w3/w2), §2.1
 *     "experts are stateless FFNs with fixed weights":
 *       a1[f] = sum_i x[i] W1[f][i],  a3[f] = sum_i x[i] W3[f][i]   (fp64)
 *       h[f]  = bf16( silu(a1[f]) * a3[f] ),  silu(a) = a / (1 + exp(−a))
 *       y[c]  = bf16( sum_f h[f] W2[c][f] )                          (fp64)
 *     W1, W3: [F][d] row-major; W2: [d][F] row-major.
 * The two halves are exported separately (O6a, O6b) with their values BEFORE
 * the bf16 storage rounding, so that the parity tests can check each storage
 * point of the GPU path against the exact value computed from the GPU's own
 * inputs to that stage (R#21).  s* = sums of |terms|: the scale of
 * the accumulation error of a floating-point evaluation of the same sum. */

/* O6a  one token row x [d]: h_exact[f] = silu(a1[f]) * a3[f] in fp64 (not
 *      rounded); a1, a3, s1 = sum_i |x W1|, s3 = sum_i |x W3| (may be NULL). */
void orc_ffn_h_f64(const uint16_t *x, int d, int F, const uint16_t *W1, const uint16_t *W3,
                   double *h, double *a1o, double *a3o, double *s1o, double *s3o) {
    for (int f = 0; f < F; ++f) {
        double a1 = 0.0, a3 = 0.0, s1 = 0.0, s3 = 0.0;
        const uint16_t *r1 = W1 + (int64_t)f * d, *r3 = W3 + (int64_t)f * d;
        for (int i = 0; i < d; ++i) {
            double xi = orc_bf16_to_f64(x[i]);
            double p1 = xi * orc_bf16_to_f64(r1[i]), p3 = xi * orc_bf16_to_f64(r3[i]);
            a1 += p1;
            a3 += p3;
            s1 += fabs(p1);
            s3 += fabs(p3);
        }
        double silu = a1 / (1.0 + exp(-a1));
        h[f] = silu * a3;
        if (a1o) a1o[f] = a1;
        if (a3o) a3o[f] = a3;
        if (s1o) s1o[f] = s1;
        if (s3o) s3o[f] = s3;
    }
}

/* O6b  from the stored (bf16) h [F]: y_exact[c] = sum_f h[f] W2[c][f] in fp64
 *      (not rounded); s[c] = sum_f |h[f] W2[c][f]| (may be NULL). */
void orc_ffn_y_f64(const uint16_t *h, int d, int F, const uint16_t *W2, double *y, double *s) {
    for (int c = 0; c < d; ++c) {
        double acc = 0.0, sa = 0.0;
        const uint16_t *r2 = W2 + (int64_t)c * F;
        for (int f = 0; f < F; ++f) {
            double p = orc_bf16_to_f64(h[f]) * orc_bf16_to_f64(r2[f]);
            acc += p;
            sa += fabs(p);
        }
        y[c] = acc;
        if (s) s[c] = sa;
    }
}

/* O6 = O6a, bf16 storage of h, O6b, bf16 storage of y.  y_exact (optional):
 * y before its rounding.  hwork: [F] doubles, hbf: [F] bf16 scratch. */
static void orc_ffn(const uint16_t *x, int d, int F, const uint16_t *W1, const uint16_t *W3,
                    const uint16_t *W2, double *hwork, uint16_t *hbf, double *ywork, uint16_t *y) {
    orc_ffn_h_f64(x, d, F, W1, W3, hwork, NULL, NULL, NULL, NULL);
    for (int f = 0; f < F; ++f) hbf[f] = orc_bf16_from_f64(hwork[f]);
    orc_ffn_y_f64(hbf, d, F, W2, ywork, NULL);
    for (int c = 0; c < d; ++c) y[c] = orc_bf16_from_f64(ywork[c]);
}

/* Batched O6a / O6b over n rows that share one expert's weights (parity
 * tests; OpenMP over rows only, the arithmetic per row is unchanged).
 *   rows_x [n][d] bf16 -> h [n][F] fp64 (+ a1, a3, s1, s3 [n][F], optional)
 *   rows_h [n][F] bf16 -> y [n][d] fp64 (+ s [n][d], optional)           */
void orc_stage_h(const uint16_t *rows_x, int n, int d, int F, const uint16_t *W1, const uint16_t *W3,
                 double *h, double *a1, double *a3, double *s1, double *s3, int n_threads) {
#ifdef _OPENMP
    if (n_threads < 1) n_threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads)
#endif
    for (int r = 0; r < n; ++r) {
        const int64_t o = (int64_t)r * F;
        orc_ffn_h_f64(rows_x + (int64_t)r * d, d, F, W1, W3, h + o, a1 ? a1 + o : NULL, a3 ? a3 + o : NULL,
                      s1 ? s1 + o : NULL, s3 ? s3 + o : NULL);
    }
}

void orc_stage_y(const uint16_t *rows_h, int n, int d, int F, const uint16_t *W2, double *y, double *s,
                 int n_threads) {
#ifdef _OPENMP
    if (n_threads < 1) n_threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads)
#endif
    for (int r = 0; r < n; ++r)
        orc_ffn_y_f64(rows_h + (int64_t)r * F, d, F, W2, y + (int64_t)r * d, s ? s + (int64_t)r * d : NULL);
}

/* -------------------------------------------------------- O8 combine */

/* O8  one token: out_exact[c] = sum_j w_j * y_j[c] (+ sg * y_sh[c]) in fp64, j in
 *     order, before the bf16 storage rounding of out ("aggregated via a
 *     weighted sum using the gating weights"; R#5 on the AW; R#16 shared expert
 *     with weight 1, or sg = sigmoid gate, O7').  y [k][d] and y_sh [d] bf16
 *     (y_sh may be NULL); s[c] = sum of |terms| (may be NULL). */
void orc_combine_f64(int d, int k, const float *w, const uint16_t *y, const uint16_t *ysh, double sg,
                     double *out, double *s) {
    for (int c = 0; c < d; ++c) {
        double acc = 0.0, sa = 0.0;
        for (int j = 0; j < k; ++j) {
            double p = (double)w[j] * orc_bf16_to_f64(y[(int64_t)j * d + c]);
            acc += p;
            sa += fabs(p);
        }
        if (ysh) {
            double p = sg * orc_bf16_to_f64(ysh[c]);
            acc += p;
            sa += fabs(p);
        }
        out[c] = acc;
        if (s) s[c] = sa;
    }
}

/* Batched O8 over n tokens (parity tests): w [n][k], y [n][k][d], ysh [n][d]
 * (or NULL), sg [n] (or NULL = weight 1) -> out [n][d], s [n][d] (optional). */
void orc_stage_combine(int n, int d, int k, const float *w, const uint16_t *y, const uint16_t *ysh,
                       const float *sg, double *out, double *s) {
    for (int t = 0; t < n; ++t)
        orc_combine_f64(d, k, w + (int64_t)t * k, y + (int64_t)t * k * d, ysh ? ysh + (int64_t)t * d : NULL,
                        sg ? (double)sg[t] : 1.0, out + (int64_t)t * d, s ? s + (int64_t)t * d : NULL);
}

/* O7' shared-expert gate (NEXT-3b: Qwen1.5-MoE shared_expert_gate, DESIGN.md
 *     R#17 variant): g_t = fp32( sum_i x[t][i] wsg[i] ) accumulated in fp64,
 *     s_t = fp32( 1 / (1 + exp(-g_t)) ) in fp64; the shared expert's output is
 *     added with weight s_t instead of 1. */
void orc_shared_gate(const uint16_t *x, const uint16_t *wsg, int T, int d, float *s_out) {
    for (int t = 0; t < T; ++t) {
        double acc = 0.0;
        for (int i = 0; i < d; ++i) acc += orc_bf16_to_f64(x[(int64_t)t * d + i]) * orc_bf16_to_f64(wsg[i]);
        float g = (float)acc;
        s_out[t] = (float)(1.0 / (1.0 + exp(-(double)g)));
    }
}

/* O6-O8 for a list of tokens.
 *   For token t (global index tokens[n]) and its k selected experts idx[t][j]
 *   with weights w[t][j]:  y_j = FFN_{e_j}(x_t)  (O6);  y_sh = FFN_sh(x_t) if
 *   F_sh > 0 (O7, R#16: shared expert added with weight 1, or sgate[t], O7');
 *   out[n][c] = bf16( sum_j w_j * y_j[c]  (+ y_sh[c]) )   in fp64, j order
 *   (O8, "aggregated via a weighted sum using the gating weights").
 *   The FFN of a pair depends only on (x_t, expert weights): which EW or
 *   slot serves it never enters (§5.1, stateless replay).
 * w1/w3/w2: arrays of E pointers to the per-expert matrices.
 * sgate (optional, [T] fp32): weight of the shared expert per token; NULL = 1.
 * y_out (optional): [n_tokens][k][d] bf16 per-pair expert outputs.
 * ysh_out (optional): [n_tokens][d] bf16 shared-expert outputs.
 * out_f64 (optional): [n_tokens][d] out before its bf16 rounding (O8 exact).
 * n_threads > 1 parallelises over tokens only (arithmetic per token unchanged). */
int orc_moe_tokens3(int d, int E, int k, int F, int F_sh,
                    const uint16_t *x, const int32_t *idx, const float *w,
                    const uint16_t *const *w1, const uint16_t *const *w3, const uint16_t *const *w2,
                    const uint16_t *w1s, const uint16_t *w3s, const uint16_t *w2s, const float *sgate,
                    const int32_t *tokens, int n_tokens, uint16_t *out, uint16_t *y_out,
                    int n_threads, uint16_t *ysh_out, double *out_f64) {
    if (k < 1 || k > E || d < 1 || F < 1) return ORC_ERR_INVALID;
    int Fmax = F > F_sh ? F : F_sh;
    int bad = 0;
#ifdef _OPENMP
    if (n_threads < 1) n_threads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads)
#endif
    for (int n = 0; n < n_tokens; ++n) {
        double *hwork = (double *)malloc(sizeof(double) * (size_t)Fmax);
        uint16_t *hbf = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)Fmax);
        double *work = (double *)malloc(sizeof(double) * (size_t)d);
        uint16_t *y = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)d * (k + 1));
        int t = tokens ? tokens[n] : n;
        const uint16_t *xt = x + (int64_t)t * d;
        for (int j = 0; j < k; ++j) {
            int e = idx[(int64_t)t * k + j];
            if (e < 0 || e >= E) { bad = 1; continue; }
            orc_ffn(xt, d, F, w1[e], w3[e], w2[e], hwork, hbf, work, y + (int64_t)j * d);
            if (y_out) memcpy(y_out + ((int64_t)n * k + j) * d, y + (int64_t)j * d, sizeof(uint16_t) * d);
        }
        if (F_sh > 0) {
            orc_ffn(xt, d, F_sh, w1s, w3s, w2s, hwork, hbf, work, y + (int64_t)k * d);
            if (ysh_out) memcpy(ysh_out + (int64_t)n * d, y + (int64_t)k * d, sizeof(uint16_t) * d);
        }
        orc_combine_f64(d, k, w + (int64_t)t * k, y, F_sh > 0 ? y + (int64_t)k * d : NULL,
                        sgate ? (double)sgate[t] : 1.0, work, NULL);
        for (int c = 0; c < d; ++c) out[(int64_t)n * d + c] = orc_bf16_from_f64(work[c]);
        if (out_f64) memcpy(out_f64 + (int64_t)n * d, work, sizeof(double) * d);
        free(hwork);
        free(hbf);
        free(work);
        free(y);
    }
    return bad ? ORC_ERR_INVALID : ORC_OK;
}

int orc_moe_tokens2(int d, int E, int k, int F, int F_sh,
                    const uint16_t *x, const int32_t *idx, const float *w,
                    const uint16_t *const *w1, const uint16_t *const *w3, const uint16_t *const *w2,
                    const uint16_t *w1s, const uint16_t *w3s, const uint16_t *w2s, const float *sgate,
                    const int32_t *tokens, int n_tokens, uint16_t *out, uint16_t *y_out,
                    int n_threads, uint16_t *ysh_out) {
    return orc_moe_tokens3(d, E, k, F, F_sh, x, idx, w, w1, w3, w2, w1s, w3s, w2s, sgate, tokens, n_tokens,
                           out, y_out, n_threads, ysh_out, NULL);
}

int orc_moe_tokens(int d, int E, int k, int F, int F_sh,
                   const uint16_t *x, const int32_t *idx, const float *w,
                   const uint16_t *const *w1, const uint16_t *const *w3, const uint16_t *const *w2,
                   const uint16_t *w1s, const uint16_t *w3s, const uint16_t *w2s,
                   const int32_t *tokens, int n_tokens, uint16_t *out, uint16_t *y_out,
                   int n_threads) {
    return orc_moe_tokens3(d, E, k, F, F_sh, x, idx, w, w1, w3, w2, w1s, w3s, w2s, NULL, tokens, n_tokens,
                           out, y_out, n_threads, NULL, NULL);
}

int orc_version(void) { return 1; }
