/*
 * oracle/sfa_oracle.c -- plain, slow, fp64 CPU oracle for Sparse Feature Attention (SFA).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2603_22300_b200/) never imports, links or executes anything here, and this
 * file shares no source, header, table or helper with the CUDA path.
 *
 * Citation convention: "P:Lnnn" is /root/reference/PAPER.md line nnn (section / equation
 * named beside it); "S:Lnnn" is SPEC.md.  Readings of gaps are numbered A1..A21 as in
 * DESIGN.md section "Readings".
 *
 * What is computed (the plain definitions, written out, no blocking / fusion / reordering):
 *
 *   ref_topk_codes   Eq. (topk_QK) + the Topk_k definition, P:L83-94 (Sec. 3.1):
 *                    keep the k entries of largest |x_u|, sign kept.  Ties -> lower index
 *                    (A2), output indices ascending (A4), exactly k entries always (A8).
 *                    Ranking uses fabs() of the value widened to double: the real-number
 *                    magnitude, not a bit trick.
 *
 *   ref_attn_fwd     P:L97-101 (Sec. 3.1, "Attention scores are then computed as
 *                    S = Q~ K~^T", Eq. s_ij) and P:L43-50 (Sec. 2, P = softmax(S (.) M),
 *                    O = P V), on the DECOMPRESSED codes:
 *                      q~_i = densify(q codes of row i)      (d doubles, zeros elsewhere)
 *                      s_ij = scale * sum_{u<d} q~_iu k~_ju  (= sum over the support overlap;
 *                                                             0 when the supports are disjoint, A1/R1)
 *                      allowed(i,j) = !causal || j <= q_pos0 + i            (A9)
 *                      m_i = max_j s_ij ; l_i = sum_j exp(s_ij - m_i)
 *                      O_i = sum_j exp(s_ij - m_i) V_j / l_i ; LSE_i = m_i + log(l_i)  (A11)
 *                    two passes over the materialised row, fp64 throughout.
 *                    Rows with no allowed key: O_i = 0, LSE_i = -inf (A10).
 *
 *   ref_scores_row   the s_ij of one row (for the "rows of P sum to 1" pin).
 *
 *   ref_edge_count   E = sum_i sum_{allowed j} |S_i (intersect) S_j|  -- the number of
 *                    structural intersections ("Efficiency analysis"),
 *                    counted pair by pair.
 *
 * Pins (tests/test_oracle_topk.py, tests/test_oracle_attn.py, tests/test_accounting.py; -m "not gpu") tie every function above to
 * something other than itself: brute-force subset enumeration and the SPEC vectors for
 * top-k; torch's fp64 scaled_dot_product_attention at k = d; closed forms (n = 1,
 * disjoint supports, Q = K = V = I); causality perturbation; row sums of P; the hand
 * example 6/sqrt(4) = 3.0; prefix-count edge formula and the balanced-support closed
 * form n^2 k^2 / d.
 *
 * Dtypes: 0 = fp32, 1 = bf16 (IEEE bit patterns, widened exactly to double).
 * Layouts (row-major, last index fastest):
 *   x      [rows][d]          q_idx/q_val [B][H][n_q][k]     k_idx/k_val [B][H_kv][n_kv][k]
 *   v      [B][H_kv][n_kv][d_v]                              o [nsel][d_v] fp64, lse [nsel] fp64
 * GQA: query head h reads kv head h / (H / H_kv) (A15).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORACLE_OK = 0, ORACLE_INVALID_ARGUMENT = 1, ORACLE_INVALID_INPUT = 2 };

/* ---- value widening (exact) ------------------------------------------------------ */
static double widen(const void *base, int dtype, int64_t i) {
    if (dtype == 0) {
        float f;
        memcpy(&f, (const char *)base + 4 * i, 4);
        return (double)f;
    } else {
        uint16_t h;
        uint32_t u;
        float f;
        memcpy(&h, (const char *)base + 2 * i, 2);
        u = ((uint32_t)h) << 16; /* bf16 is the top half of an fp32 */
        memcpy(&f, &u, 4);
        return (double)f;
    }
}

static void copy_elem(void *dst, int64_t di, const void *src, int64_t si, int dtype) {
    size_t s = dtype == 0 ? 4 : 2;
    memcpy((char *)dst + s * di, (const char *)src + s * si, s);
}

/* ---- Top-k codes: P:L83-94 --------------------------------------------------------- */
/* Selection of the k largest |x_u|: repeatedly take the not-yet-chosen entry with the
 * largest magnitude, the lower index winning a tie (A2).  O(k d) per row. */
int ref_topk_codes(const void *x, int dtype, int64_t rows, int d, int k, uint8_t *idx, void *val) {
    if (d < 1 || d > 256 || k < 1 || k > d || rows < 0 || (dtype != 0 && dtype != 1))
        return ORACLE_INVALID_ARGUMENT;
    char chosen[256];
    int sel[256];
    for (int64_t r = 0; r < rows; ++r) {
        for (int u = 0; u < d; ++u)
            if (!isfinite(widen(x, dtype, r * d + u))) return ORACLE_INVALID_INPUT; /* A14 */
        memset(chosen, 0, sizeof chosen);
        for (int t = 0; t < k; ++t) {
            int best = -1;
            double bestmag = -1.0;
            for (int u = 0; u < d; ++u) {
                if (chosen[u]) continue;
                double m = fabs(widen(x, dtype, r * d + u));
                if (m > bestmag) { /* strict: an equal magnitude at a higher index never wins */
                    bestmag = m;
                    best = u;
                }
            }
            chosen[best] = 1;
        }
        /* emit ascending feature index (A4), values bit-copied (A7) */
        int t = 0;
        for (int u = 0; u < d; ++u)
            if (chosen[u]) sel[t++] = u;
        for (t = 0; t < k; ++t) {
            idx[r * k + t] = (uint8_t)sel[t];
            copy_elem(val, r * k + t, x, r * d + sel[t], dtype);
        }
    }
    return ORACLE_OK;
}

/* ---- attention on the decompressed codes: P:L97-101, P:L43-50 ---------------------- */
typedef struct {
    int B, H, H_kv, d, k, d_v, causal, dtype;
    int64_t n_q, n_kv, q_pos0;
    double scale;
    const uint8_t *q_idx, *k_idx;
    const void *q_val, *k_val, *v;
    const int64_t *sel; /* nullable: flat row ids into [B][H][n_q] */
    int64_t nsel;
    double *o, *lse;
    int64_t next; /* work cursor (guarded by mu) */
    pthread_mutex_t mu;
    int status;
} attn_job;

static void densify(const uint8_t *idx, const void *val, int dtype, int64_t row, int k, int d, double *out) {
    for (int u = 0; u < d; ++u) out[u] = 0.0;
    for (int t = 0; t < k; ++t) out[idx[row * k + t]] = widen(val, dtype, row * k + t);
}

static void attn_one_row(attn_job *J, int64_t flat, double *o, double *lse, double *qd, double *kd, double *s) {
    int64_t i = flat % J->n_q;
    int64_t bh = flat / J->n_q;
    int h = (int)(bh % J->H), b = (int)(bh / J->H);
    int g = h / (J->H / J->H_kv); /* A15 */
    int64_t kvrow0 = ((int64_t)b * J->H_kv + g) * J->n_kv;
    int64_t jmax = J->n_kv - 1;
    if (J->causal && J->q_pos0 + i < jmax) jmax = J->q_pos0 + i; /* A9 */
    for (int c = 0; c < J->d_v; ++c) o[c] = 0.0;
    if (jmax < 0) { /* A10 */
        *lse = -INFINITY;
        return;
    }
    densify(J->q_idx, J->q_val, J->dtype, flat, J->k, J->d, qd);
    double m = -INFINITY;
    for (int64_t j = 0; j <= jmax; ++j) {
        densify(J->k_idx, J->k_val, J->dtype, kvrow0 + j, J->k, J->d, kd);
        double acc = 0.0;
        for (int u = 0; u < J->d; ++u) acc += qd[u] * kd[u];
        s[j] = J->scale * acc; /* A5/A17: scale applied after the sum */
        if (s[j] > m) m = s[j];
    }
    double l = 0.0;
    for (int64_t j = 0; j <= jmax; ++j) {
        double p = exp(s[j] - m);
        l += p;
        for (int c = 0; c < J->d_v; ++c) o[c] += p * widen(J->v, J->dtype, (kvrow0 + j) * J->d_v + c);
    }
    for (int c = 0; c < J->d_v; ++c) o[c] /= l;
    *lse = m + log(l);
}

static void *attn_worker(void *arg) {
    attn_job *J = (attn_job *)arg;
    double *qd = malloc(sizeof(double) * J->d), *kd = malloc(sizeof(double) * J->d);
    double *s = malloc(sizeof(double) * (size_t)(J->n_kv > 0 ? J->n_kv : 1));
    if (!qd || !kd || !s) {
        pthread_mutex_lock(&J->mu);
        J->status = ORACLE_INVALID_ARGUMENT;
        pthread_mutex_unlock(&J->mu);
    } else {
        for (;;) {
            pthread_mutex_lock(&J->mu);
            int64_t r = J->next;
            J->next += 16;
            pthread_mutex_unlock(&J->mu);
            if (r >= J->nsel) break;
            int64_t r1 = r + 16 < J->nsel ? r + 16 : J->nsel;
            for (; r < r1; ++r) {
                int64_t flat = J->sel ? J->sel[r] : r;
                attn_one_row(J, flat, J->o + r * J->d_v, J->lse + r, qd, kd, s);
            }
        }
    }
    free(qd);
    free(kd);
    free(s);
    return NULL;
}

int ref_attn_fwd(int B, int H, int H_kv, int d, int k, int d_v, int64_t n_q, int64_t n_kv, int64_t q_pos0,
                 int causal, double scale, int dtype, const uint8_t *q_idx, const void *q_val,
                 const uint8_t *k_idx, const void *k_val, const void *v, const int64_t *sel, int64_t nsel,
                 double *o, double *lse, int threads) {
    if (B < 1 || H < 1 || H_kv < 1 || H % H_kv || d < 1 || d > 256 || k < 1 || k > d || d_v < 1 || n_q < 0 ||
        n_kv < 0 || (dtype != 0 && dtype != 1) || !(scale > 0) || !isfinite(scale))
        return ORACLE_INVALID_ARGUMENT;
    attn_job J;
    memset(&J, 0, sizeof J);
    J.B = B; J.H = H; J.H_kv = H_kv; J.d = d; J.k = k; J.d_v = d_v; J.causal = causal; J.dtype = dtype;
    J.n_q = n_q; J.n_kv = n_kv; J.q_pos0 = q_pos0; J.scale = scale;
    J.q_idx = q_idx; J.k_idx = k_idx; J.q_val = q_val; J.k_val = k_val; J.v = v;
    J.sel = sel;
    J.nsel = sel ? nsel : (int64_t)B * H * n_q;
    J.o = o; J.lse = lse;
    pthread_mutex_init(&J.mu, NULL);
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, attn_worker, &J);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    pthread_mutex_destroy(&J.mu);
    return J.status;
}

/* s_ij for j = 0..n_kv-1 of one query row (flat id into [B][H][n_q]); masked keys get -inf. */
int ref_scores_row(int B, int H, int H_kv, int d, int k, int64_t n_q, int64_t n_kv, int64_t q_pos0, int causal,
                   double scale, int dtype, const uint8_t *q_idx, const void *q_val, const uint8_t *k_idx,
                   const void *k_val, int64_t flat, double *s_out) {
    if (B < 1 || H < 1 || H_kv < 1 || H % H_kv || k < 1 || k > d || d > 256) return ORACLE_INVALID_ARGUMENT;
    double qd[256], kd[256];
    int64_t i = flat % n_q, bh = flat / n_q;
    int h = (int)(bh % H), b = (int)(bh / H), g = h / (H / H_kv);
    int64_t kvrow0 = ((int64_t)b * H_kv + g) * n_kv;
    densify(q_idx, q_val, dtype, flat, k, d, qd);
    for (int64_t j = 0; j < n_kv; ++j) {
        if (causal && j > q_pos0 + i) {
            s_out[j] = -INFINITY;
            continue;
        }
        densify(k_idx, k_val, dtype, kvrow0 + j, k, d, kd);
        double acc = 0.0;
        for (int u = 0; u < d; ++u) acc += qd[u] * kd[u];
        s_out[j] = scale * acc;
    }
    return ORACLE_OK;
}

/* E = number of (query i, allowed key j, feature u) with u in S_i and u in S_j. */
int64_t ref_edge_count(int B, int H, int H_kv, int k, int64_t n_q, int64_t n_kv, int64_t q_pos0, int causal,
                       const uint8_t *q_idx, const uint8_t *k_idx) {
    int64_t E = 0;
    for (int b = 0; b < B; ++b)
        for (int h = 0; h < H; ++h) {
            int g = h / (H / H_kv);
            for (int64_t i = 0; i < n_q; ++i) {
                const uint8_t *qi = q_idx + (((int64_t)b * H + h) * n_q + i) * k;
                int64_t jmax = n_kv - 1;
                if (causal && q_pos0 + i < jmax) jmax = q_pos0 + i;
                for (int64_t j = 0; j <= jmax; ++j) {
                    const uint8_t *kj = k_idx + (((int64_t)b * H_kv + g) * n_kv + j) * k;
                    for (int a = 0; a < k; ++a)
                        for (int c = 0; c < k; ++c) E += (qi[a] == kj[c]);
                }
            }
        }
    return E;
}
