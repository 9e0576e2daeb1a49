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
 *                    edges_only = 1 (reading A1/R2; "Traversing active
 *                    coordinates yields only the nonzero attention edges", P:L122 O(E + E d_v)):
 *                    a pair (i, j) is kept only if it is allowed AND the supports intersect,
 *                      edge(i,j) = exists t, t' : q_idx[i][t] == k_idx[j][t']
 *                    (index equality; zero-valued selected entries count as support, A8); the
 *                    softmax runs over the edges only; a row with no edge gets O = 0, LSE = -inf
 *                    (as A10).
 *
 *                    window = w > 0 (composition with token sparsity: the causal
 *                    sliding window of Longformer/Mistral-style local attention, "SFA is
 *                    orthogonal to token-level sparsity"): key j is allowed only if, in addition,
 *                      j > q_pos0 + i - w          (the last w positions up to and including i)
 *                    Rows with no allowed key: O = 0, LSE = -inf (A10).
 *
 *                    block_sel (composition with block-level token selection: NSA-style
 *                    "select the key blocks each query block attends"): with blocks of
 *                    128 positions, key j is allowed only if, in addition, its block j / 128 appears in
 *                    the list block_sel[b][g][i / 128][0 .. max_sel) of the row's (batch, kv head, local
 *                    query block); entries < 0 are padding.  Rows with no allowed key: O = 0, LSE = -inf.
 *
 *   ref_scores_row   the s_ij of one row (for the "rows of P sum to 1" pin).
 *
 *   ref_attn_bwd     the backward pass of ref_attn_fwd with the straight-through rule
 *                    (Sec. 3.1 "Backward computation", Eq. topk_grad: gradients
 *                    flow only through the selected coordinates), given the upstream dO:
 *                      P_ij = exp(s_ij - LSE_i) (s, LSE recomputed as in ref_attn_fwd)
 *                      O_i = sum_j P_ij V_j ;  D_i = sum_c dO_ic O_ic
 *                      dP_ij = sum_c dO_ic V_jc ;  dS_ij = P_ij (dP_ij - D_i)   (softmax Jacobian)
 *                      dV_j  = sum_{h in group} sum_i P_ij dO_i                 (A15: GQA heads add)
 *                      dq~_iu = scale sum_j dS_ij k~_ju ;  dk~_ju = scale sum_{h,i} dS_ij q~_iu
 *                      dq_val[i][t] = dq~_{i, q_idx[i][t]} ; dk_val[j][t] = dk~_{j, k_idx[j][t]}
 *                    (the gradient w.r.t. the code values; the dense dQ / dK of Eq. topk_grad are
 *                    these scattered to the support, zero elsewhere).  Materialised rows, fp64.
 *                    Optional companions (tests' componentwise error bounds, A24):
 *                      bv[j][c] = sum_i P_ij |dO_ic|
 *                      bq[i][t] = scale sum_j P_ij (|dP_ij| + |D_i| + sum_c |dO_ic|(|O_ic| + 1)) |k~_ju|
 *                      bk[j][t] = the same with q~ in place of k~ (summed over the group's heads)
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
 * Dtypes: 0 = fp32, 1 = bf16 (IEEE bit patterns, widened exactly to double), 2 = fp64 (gradient pins).
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
    if (dtype == 2) { /* fp64 values: only for the finite-difference pins of ref_attn_bwd */
        double x;
        memcpy(&x, (const char *)base + 8 * i, 8);
        return x;
    }
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
    size_t s = dtype == 2 ? 8 : (dtype == 0 ? 4 : 2);
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
    int B, H, H_kv, d, k, d_v, causal, dtype, edges_only;
    int64_t n_q, n_kv, q_pos0, window;
    const int32_t *bsel; /* nullable: [B][H_kv][ceil(n_q/128)][max_sel] key-block lists */
    int max_sel;
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

/* R2 (edges_only): do the supports of query row qrow and key row krow share a feature index? */
static int supports_intersect(const uint8_t *q_idx, int64_t qrow, const uint8_t *k_idx, int64_t krow, int k) {
    for (int t = 0; t < k; ++t)
        for (int u = 0; u < k; ++u)
            if (q_idx[qrow * k + t] == k_idx[krow * k + u]) return 1;
    return 0;
}

/* block selection: is key j's block in the list of (b, g, query block of local row i)? */
static int block_selected(const attn_job *J, int b, int g, int64_t i, int64_t j) {
    int64_t nqb = (J->n_q + 127) / 128;
    const int32_t *L = J->bsel + (((int64_t)b * J->H_kv + g) * nqb + i / 128) * J->max_sel;
    for (int t = 0; t < J->max_sel; ++t)
        if (L[t] >= 0 && (int64_t)L[t] == j / 128) return 1;
    return 0;
}

static void attn_one_row(attn_job *J, int64_t flat, double *o, double *lse, double *qd, double *kd, double *s) {
    int64_t i = flat % J->n_q;
    int64_t bh = flat / J->n_q;
    int h = (int)(bh % J->H), b = (int)(bh / J->H);
    int g = h / (J->H / J->H_kv); /* A15 */
    int64_t kvrow0 = ((int64_t)b * J->H_kv + g) * J->n_kv;
    int64_t jmax = J->n_kv - 1;
    if (J->causal && J->q_pos0 + i < jmax) jmax = J->q_pos0 + i; /* A9 */
    int64_t jmin = 0;
    if (J->window > 0 && J->q_pos0 + i - J->window + 1 > jmin) jmin = J->q_pos0 + i - J->window + 1; /* N4 window */
    for (int c = 0; c < J->d_v; ++c) o[c] = 0.0;
    if (jmax < jmin) { /* A10 */
        *lse = -INFINITY;
        return;
    }
    densify(J->q_idx, J->q_val, J->dtype, flat, J->k, J->d, qd);
    double m = -INFINITY;
    for (int64_t j = 0; j <= jmax; ++j) {
        if (j < jmin || (J->edges_only && !supports_intersect(J->q_idx, flat, J->k_idx, kvrow0 + j, J->k)) ||
            (J->bsel && !block_selected(J, b, g, i, j))) {
            s[j] = -INFINITY; /* R2: not an edge / block not selected -> excluded from the softmax */
            continue;
        }
        densify(J->k_idx, J->k_val, J->dtype, kvrow0 + j, J->k, J->d, kd);
        double acc = 0.0;
        for (int u = 0; u < J->d; ++u) acc += qd[u] * kd[u];
        s[j] = J->scale * acc; /* A5/A17: scale applied after the sum */
        if (s[j] > m) m = s[j];
    }
    if (m == -INFINITY) { /* R2 / block selection: no allowed key in the row (as A10) */
        *lse = -INFINITY;
        return;
    }
    double l = 0.0;
    for (int64_t j = 0; j <= jmax; ++j) {
        if (s[j] == -INFINITY) continue;
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

int ref_attn_fwd_ex(int B, int H, int H_kv, int d, int k, int d_v, int64_t n_q, int64_t n_kv, int64_t q_pos0,
                    int causal, double scale, int dtype, const uint8_t *q_idx, const void *q_val,
                    const uint8_t *k_idx, const void *k_val, const void *v, const int64_t *sel, int64_t nsel,
                    double *o, double *lse, int threads, int edges_only, int64_t window, const int32_t *bsel,
                    int max_sel) {
    if (window < 0 || (bsel && max_sel < 1)) return ORACLE_INVALID_ARGUMENT;
    if (B < 1 || H < 1 || H_kv < 1 || H % H_kv || d < 1 || d > 256 || k < 1 || k > d || d_v < 1 || n_q < 0 ||
        n_kv < 0 || dtype < 0 || dtype > 2 || !(scale > 0) || !isfinite(scale))
        return ORACLE_INVALID_ARGUMENT;
    attn_job J;
    memset(&J, 0, sizeof J);
    J.B = B; J.H = H; J.H_kv = H_kv; J.d = d; J.k = k; J.d_v = d_v; J.causal = causal; J.dtype = dtype;
    J.n_q = n_q; J.n_kv = n_kv; J.q_pos0 = q_pos0; J.scale = scale;
    J.edges_only = edges_only != 0;
    J.window = window;
    J.bsel = bsel;
    J.max_sel = max_sel;
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

int ref_attn_fwd(int B, int H, int H_kv, int d, int k, int d_v, int64_t n_q, int64_t n_kv, int64_t q_pos0,
                 int causal, double scale, int dtype, const uint8_t *q_idx, const void *q_val,
                 const uint8_t *k_idx, const void *k_val, const void *v, const int64_t *sel, int64_t nsel,
                 double *o, double *lse, int threads) {
    return ref_attn_fwd_ex(B, H, H_kv, d, k, d_v, n_q, n_kv, q_pos0, causal, scale, dtype, q_idx, q_val, k_idx,
                           k_val, v, sel, nsel, o, lse, threads, 0, 0, NULL, 0);
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

/* ---- backward with the straight-through rule: P:L103-112 ----------------------------- */
typedef struct {
    int B, H, H_kv, d, k, d_v, causal, dtype;
    int64_t n_q, n_kv, q_pos0;
    double scale;
    const uint8_t *q_idx, *k_idx;
    const void *q_val, *k_val, *v;
    const double *dO;                 /* [B][H][n_q][d_v] fp64 */
    double *dq, *dk, *dv;             /* [B][H][n_q][k], [B][H_kv][n_kv][k], [B][H_kv][n_kv][d_v] */
    double *bq, *bk, *bv;             /* nullable bounds, same shapes */
    int64_t next;                     /* work cursor over (b, kv head) groups */
    pthread_mutex_t mu;
    int status;
} bwd_job;

/* one (b, kv head g): all R query heads of the group, so dK~ / dV of the group are owned here */
static int bwd_group(bwd_job *J, int b, int g) {
    const int R = J->H / J->H_kv, d = J->d, k = J->k, dv = J->d_v;
    const int64_t nq = J->n_q, nkv = J->n_kv;
    const int64_t kvrow0 = ((int64_t)b * J->H_kv + g) * nkv;
    double *kd = malloc(sizeof(double) * (size_t)(nkv > 0 ? nkv : 1) * d);   /* k~ rows of the group */
    double *dkd = calloc((size_t)(nkv > 0 ? nkv : 1) * d, sizeof(double));  /* dk~ */
    double *bkd = calloc((size_t)(nkv > 0 ? nkv : 1) * d, sizeof(double));
    double *vv = malloc(sizeof(double) * (size_t)(nkv > 0 ? nkv : 1) * dv);
    double *s = malloc(sizeof(double) * (size_t)(nkv > 0 ? nkv : 1));
    double *qd = malloc(sizeof(double) * d), *dqd = malloc(sizeof(double) * d), *bqd = malloc(sizeof(double) * d);
    double *o = malloc(sizeof(double) * dv);
    if (!kd || !dkd || !bkd || !vv || !s || !qd || !dqd || !bqd || !o) {
        free(kd); free(dkd); free(bkd); free(vv); free(s); free(qd); free(dqd); free(bqd); free(o);
        return ORACLE_INVALID_ARGUMENT;
    }
    for (int64_t j = 0; j < nkv; ++j) {
        densify(J->k_idx, J->k_val, J->dtype, kvrow0 + j, k, d, kd + j * d);
        for (int c = 0; c < dv; ++c) vv[j * dv + c] = widen(J->v, J->dtype, (kvrow0 + j) * dv + c);
    }
    double *dvg = J->dv + kvrow0 * dv; /* zero-initialised by the caller */
    double *bvg = J->bv ? J->bv + kvrow0 * dv : NULL;
    for (int r = 0; r < R; ++r) {
        const int h = g * R + r;
        for (int64_t i = 0; i < nq; ++i) {
            const int64_t flat = ((int64_t)b * J->H + h) * nq + i;
            int64_t jmax = nkv - 1;
            if (J->causal && J->q_pos0 + i < jmax) jmax = J->q_pos0 + i; /* A9 */
            for (int t = 0; t < k; ++t) {
                J->dq[flat * k + t] = 0.0;
                if (J->bq) J->bq[flat * k + t] = 0.0;
            }
            if (jmax < 0) continue; /* A10: no allowed key, no gradient */
            densify(J->q_idx, J->q_val, J->dtype, flat, k, d, qd);
            const double *dO = J->dO + flat * dv;
            /* forward again: s, LSE, O (two passes, as ref_attn_fwd) */
            double m = -INFINITY;
            for (int64_t j = 0; j <= jmax; ++j) {
                double acc = 0.0;
                for (int u = 0; u < d; ++u) acc += qd[u] * kd[j * d + u];
                s[j] = J->scale * acc;
                if (s[j] > m) m = s[j];
            }
            double l = 0.0;
            for (int64_t j = 0; j <= jmax; ++j) l += exp(s[j] - m);
            const double lse = m + log(l);
            for (int c = 0; c < dv; ++c) o[c] = 0.0;
            for (int64_t j = 0; j <= jmax; ++j) {
                const double p = exp(s[j] - lse);
                for (int c = 0; c < dv; ++c) o[c] += p * vv[j * dv + c];
            }
            double D = 0.0, E = 0.0;
            for (int c = 0; c < dv; ++c) {
                D += dO[c] * o[c];
                E += fabs(dO[c]) * (fabs(o[c]) + 1.0);
            }
            for (int u = 0; u < d; ++u) {
                dqd[u] = 0.0;
                bqd[u] = 0.0;
            }
            for (int64_t j = 0; j <= jmax; ++j) {
                const double p = exp(s[j] - lse);
                double dp = 0.0;
                for (int c = 0; c < dv; ++c) dp += dO[c] * vv[j * dv + c];
                const double ds = p * (dp - D);
                const double w = p * (fabs(dp) + fabs(D) + E);
                for (int c = 0; c < dv; ++c) {
                    dvg[j * dv + c] += p * dO[c];
                    if (bvg) bvg[j * dv + c] += p * fabs(dO[c]);
                }
                for (int u = 0; u < d; ++u) {
                    dqd[u] += J->scale * ds * kd[j * d + u];
                    bqd[u] += J->scale * w * fabs(kd[j * d + u]);
                    dkd[j * d + u] += J->scale * ds * qd[u];
                    bkd[j * d + u] += J->scale * w * fabs(qd[u]);
                }
            }
            for (int t = 0; t < k; ++t) { /* Eq. topk_grad: the selected coordinates only */
                const int u = J->q_idx[flat * k + t];
                J->dq[flat * k + t] = dqd[u];
                if (J->bq) J->bq[flat * k + t] = bqd[u];
            }
        }
    }
    for (int64_t j = 0; j < nkv; ++j)
        for (int t = 0; t < k; ++t) {
            const int u = J->k_idx[(kvrow0 + j) * k + t];
            J->dk[(kvrow0 + j) * k + t] = dkd[j * d + u];
            if (J->bk) J->bk[(kvrow0 + j) * k + t] = bkd[j * d + u];
        }
    free(kd); free(dkd); free(bkd); free(vv); free(s); free(qd); free(dqd); free(bqd); free(o);
    return ORACLE_OK;
}

static void *bwd_worker(void *arg) {
    bwd_job *J = (bwd_job *)arg;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int64_t w = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (w >= (int64_t)J->B * J->H_kv) break;
        int st = bwd_group(J, (int)(w / J->H_kv), (int)(w % J->H_kv));
        if (st) {
            pthread_mutex_lock(&J->mu);
            J->status = st;
            pthread_mutex_unlock(&J->mu);
        }
    }
    return NULL;
}

int ref_attn_bwd(int B, int H, int H_kv, int d, int k, int d_v, int64_t n_q, int64_t n_kv, int64_t q_pos0,
                 int causal, double scale, int dtype, const uint8_t *q_idx, const void *q_val, const uint8_t *k_idx,
                 const void *k_val, const void *v, const double *dO, double *dq, double *dk, double *dv, double *bq,
                 double *bk, double *bv, int threads) {
    if (B < 1 || H < 1 || H_kv < 1 || H % H_kv || d < 1 || d > 256 || k < 1 || k > d || d_v < 1 || n_q < 0 ||
        n_kv < 0 || dtype < 0 || dtype > 2 || !(scale > 0) || !isfinite(scale))
        return ORACLE_INVALID_ARGUMENT;
    bwd_job J;
    memset(&J, 0, sizeof J);
    J.B = B; J.H = H; J.H_kv = H_kv; J.d = d; J.k = k; J.d_v = d_v; J.causal = causal; J.dtype = dtype;
    J.n_q = n_q; J.n_kv = n_kv; J.q_pos0 = q_pos0; J.scale = scale;
    J.q_idx = q_idx; J.k_idx = k_idx; J.q_val = q_val; J.k_val = k_val; J.v = v; J.dO = dO;
    J.dq = dq; J.dk = dk; J.dv = dv; J.bq = bq; J.bk = bk; J.bv = bv;
    memset(dv, 0, sizeof(double) * (size_t)B * H_kv * n_kv * d_v);
    if (bv) memset(bv, 0, sizeof(double) * (size_t)B * H_kv * n_kv * d_v);
    pthread_mutex_init(&J.mu, NULL);
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, bwd_worker, &J);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    pthread_mutex_destroy(&J.mu);
    return J.status;
}
