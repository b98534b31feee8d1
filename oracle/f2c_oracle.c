/*
 * f2c_oracle.c -- plain, slow, obviously-correct CPU oracle for the F2C DCP head.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2105_10375_b200/) never links, imports or calls it, and shares no code,
 * header, table or constant with it.
 *
 * Everything is fp64, single-threaded, written in the paper's order and notation.
 * Inputs are the same dtype-rounded bytes the GPU consumes (bf16 bit patterns or
 * fp32), upcast exactly to double.  Compile with -O2 -ffp-contract=off.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / equation named
 * alongside); S:n = SPEC.md line n; D-n = reading n of DESIGN.md section 3.
 *
 *   orc_enqueue      Eq. 7 + Algorithm 1: ring of C slots.
 *   orc_loss         Eq. 6 split, Eq. 8 logits (K=1),
 *                    Eq. 9 CE with scale s and cosine margin m (D3),
 *                    L_cos (mean reduction D10), L_total,
 *                    gradient w.r.t. the raw P-Net features (D12).
 *   orc_loss_rows    the same definition, evaluated for a subset of rows only
 *                    (the global normalisers N_pos, N_neg, C_occ and mu are still
 *                    computed from the whole batch / pool).
 *   orc_enqueue_refresh
 *                    NEXT-3: SPEC's refresh-in-place insert (reading R7).
 *   orc_ema          G-Net moving average phi <- m*phi + (1-m)*theta.
 *   orc_loss_k / orc_loss_rows_k
 *                    the pool with K features per slot ("C x K x D"):
 *                    logits use T_bar_c = (1/K) sum_k T[c,k] (Eq. 8 "(1/K) sum_k <F_p, T[:,k,:]>",
 *                    P:155-159); for K >= 2 the L_cos term uses the true cosine
 *                    <x_hat, T_bar_c> / ||T_bar_c|| ("phi ... cosine similarity",
 *                    "T_bar ... average along the axis of K"; reading R4), a zero-norm
 *                    center contributing 0.  K = 1 is exactly orc_loss.
 *   orc_loss_v / orc_loss_rows_v
 *                    NEXT-3 variants of the L_cos term (the paper leaves the reduction of
 *                    phi over the pool unstated; SPEC's open questions S:399,
 *                    S:426): phi_mode 0 = mean over the occupied centers (D10,
 *                    default), 1 = sum, 2 = max (hardest negative, first slot on ties);
 *                    hinge = 1 penalises only positive similarity, max(0, cos); and the
 *                    weight lambda on L_cos (L_total = L_ce + lambda L_cos).
 *                    flags bit 0 = hinge; bit 1 = exclude stale self-duplicates: an in-pool
 *                    row's softmax runs over the occupied slots minus the OLDER slots that
 *                    carry its own label (D8 keeps them as ordinary denominator terms).
 *                    orc_loss_k is orc_loss_v with (mean, no hinge, lambda = 1).
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py
 * (pins P1-P8 of DESIGN.md section 4).  The semantics choices D3 (margin form),
 * D8 (newest duplicate is the target) and D10 (mean reduction of phi) have no
 * paper-printed numbers; they are pinned only by closed forms derived from those
 * readings ("parity unpinned" with respect to the paper for those choices).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ESHAPE 2
#define ORC_ECAPACITY 3
#define ORC_EPAIRING 4
#define ORC_EZERO 5

/* ---- dtype upcast: 0 = bf16 (uint16 bit pattern), 1 = fp32 ------------------ */
static double orc_elem(const void *base, int dtype, int64_t idx) {
    if (dtype == 0) {
        uint16_t h = ((const uint16_t *)base)[idx];
        uint32_t w = ((uint32_t)h) << 16;
        float f;
        memcpy(&f, &w, sizeof f);
        return (double)f;
    }
    return (double)((const float *)base)[idx];
}

static size_t orc_esize(int dtype) { return dtype == 0 ? 2u : 4u; }

/* ---- Eq. 7 / Algorithm 1 ------------------------------------------------------
 * T[C][d] (raw dtype bytes), lab[C], *E = rows ever enqueued, *M_last = size of
 * the last block.  While E < C this is Algorithm 1's sequential fill of the
 * unoccupied positions; afterwards it overwrites the oldest rows, which
 * is Eq. 7's shift up to relabelling of positions (D6, D7). */
int orc_enqueue(int64_t C, int32_t d, int32_t dtype, void *T, int64_t *lab, int64_t *E,
                int64_t *M_last, const void *G, const int64_t *y, int64_t M) {
    if (C < 1 || d < 1 || (dtype != 0 && dtype != 1)) return ORC_EINVAL;
    if (M < 1 || M > C) return ORC_ECAPACITY;
    for (int64_t j = 0; j < M; ++j)
        if (y[j] < 0) return ORC_EINVAL;
    size_t rb = (size_t)d * orc_esize(dtype);
    for (int64_t j = 0; j < M; ++j) {
        int64_t c = (*E + j) % C;
        memcpy((char *)T + (size_t)c * rb, (const char *)G + (size_t)j * rb, rb);
        lab[c] = y[j];
    }
    *E += M;
    *M_last = M;
    return ORC_OK;
}

/* global write index of the current content of slot c (c < min(E, C)) */
static int64_t orc_seq(int64_t c, int64_t C, int64_t E) { return c + C * ((E - 1 - c) / C); }

/* ---- NEXT-3: refresh-in-place enqueue (reading R7) ----------
 * SPEC's insert_batch: "If an id is already resident, its features are overwritten in place
 * and its queue position is unchanged"; new ids take the next positions of the ring,
 * evicting the oldest (Alg. 1 / Eq. 7 for them).  Reading R7 for the one case SPEC leaves
 * open -- a resident id whose slot is among those this block's new rows evict -- keeps
 * every block id resident after the call: such a row is appended as a new one.
 *   1. y_j >= 0 and pairwise distinct within the block ("duplicate ids ... input error");
 *   2. res(j) = the newest occupied slot with label y_j (D8) and sigma_j its write index,
 *      or none;
 *   3. appending n rows overwrites the contents with write index < E + n - C; so
 *      n = the smallest n >= n0 = #{j : no res(j)} with
 *      n = n0 + #{j : res(j) exists, sigma_j < E + n - C}   (iterated from n0; monotone);
 *   4. rows with no res(j), or whose res(j) is overwritten (step 3), are appended in block
 *      order: k-th such row -> slot (E + k) mod C, write index E + k;
 *   5. every other row overwrites the features of slot res(j) (label and age unchanged);
 *   6. E += n; blk_seq[j] = write index of the slot now holding row j. */
int orc_enqueue_refresh(int64_t C, int32_t d, int32_t dtype, void *T, int64_t *lab, int64_t *E,
                        int64_t *M_last, const void *G, const int64_t *y, int64_t M,
                        int64_t *blk_seq) {
    if (C < 1 || d < 1 || (dtype != 0 && dtype != 1)) return ORC_EINVAL;
    if (M < 1 || M > C) return ORC_ECAPACITY;
    for (int64_t j = 0; j < M; ++j) {
        if (y[j] < 0) return ORC_EINVAL;
        for (int64_t i = 0; i < j; ++i)
            if (y[i] == y[j]) return ORC_EINVAL;
    }
    const int64_t Ec = *E, C_occ = Ec < C ? Ec : C;
    int64_t *sigma = (int64_t *)malloc((size_t)M * sizeof(int64_t));
    if (!sigma) return ORC_EINVAL;
    for (int64_t j = 0; j < M; ++j) {  /* step 2 */
        sigma[j] = -1;
        for (int64_t c = 0; c < C_occ; ++c)
            if (lab[c] == y[j] && orc_seq(c, C, Ec) > sigma[j]) sigma[j] = orc_seq(c, C, Ec);
    }
    int64_t n0 = 0;
    for (int64_t j = 0; j < M; ++j) n0 += sigma[j] < 0;
    int64_t n = n0;
    for (;;) {  /* step 3 */
        int64_t f = n0;
        for (int64_t j = 0; j < M; ++j) f += sigma[j] >= 0 && sigma[j] < Ec + n - C;
        if (f == n) break;
        n = f;
    }
    size_t rb = (size_t)d * orc_esize(dtype);
    int64_t k = 0;
    for (int64_t j = 0; j < M; ++j) {  /* steps 4, 5 */
        int64_t w;
        if (sigma[j] < 0 || sigma[j] < Ec + n - C) w = Ec + k++;
        else w = sigma[j];
        int64_t c = w % C;
        memcpy((char *)T + (size_t)c * rb, (const char *)G + (size_t)j * rb, rb);
        lab[c] = y[j];
        blk_seq[j] = w;
    }
    free(sigma);
    *E = Ec + n;  /* step 6 */
    *M_last = M;
    return ORC_OK;
}

/* ---- shared pieces of the loss definition ------------------------------------ */
typedef struct {
    int64_t C, N, E, M_last, C_occ;
    int32_t d, dtype, K;
    const void *T;
    const int64_t *lab;
    const void *X;
    const int64_t *y;
    double s, m;
    /* derived */
    double *n;     /* [N] row norms ||x_i|| */
    int64_t *t;    /* [N] target slot or -1 (Eq. 6 split) */
    int64_t N_pos, N_neg;
    double *mu;    /* [d] sum over occupied slots of T_c */
    /* NEXT-3 variants of L_cos */
    int32_t phi_mode, hinge, excl_dup;
    double lam;
} orc_ctx;

/* T_bar[c][k] = (1/K) sum_kk T[c][kk][k]  (Eq. 8's average over the K axis) */
static double orc_tbar(const orc_ctx *q, int64_t c, int32_t k) {
    if (q->K == 1) return orc_elem(q->T, q->dtype, c * q->d + k);
    double acc = 0.0;
    for (int32_t kk = 0; kk < q->K; ++kk) acc += orc_elem(q->T, q->dtype, (c * q->K + kk) * q->d + k);
    return acc / (double)q->K;
}

/* ||T_bar_c|| for the true cosine of L_cos (K >= 2); 1 for K = 1 (rows as stored, D2) */
static double orc_tbar_norm(const orc_ctx *q, int64_t c) {
    if (q->K == 1) return 1.0;
    double ss = 0.0;
    for (int32_t k = 0; k < q->d; ++k) {
        double v = orc_tbar(q, c, k);
        ss += v * v;
    }
    return sqrt(ss);
}

/* step 1-4 of the definition: norms, targets, split, mu */
static int orc_prepare(orc_ctx *q, const int32_t *pairing) {
    int64_t N = q->N, C = q->C;
    int32_t d = q->d;
    q->C_occ = q->E < C ? q->E : C;
    for (int64_t i = 0; i < N; ++i) {
        double ss = 0.0;
        for (int32_t k = 0; k < d; ++k) {
            double v = orc_elem(q->X, q->dtype, i * d + k);
            ss += v * v;
        }
        q->n[i] = sqrt(ss);
        if (!(q->n[i] > 0.0)) return ORC_EZERO;
    }
    q->N_pos = 0;
    for (int64_t i = 0; i < N; ++i) {
        int64_t best = -1, best_seq = -1;
        for (int64_t c = 0; c < q->C_occ; ++c) {
            if (q->lab[c] != q->y[i]) continue;
            int64_t sq = orc_seq(c, C, q->E);
            if (sq > best_seq) { best_seq = sq; best = c; }
        }
        q->t[i] = best;
        if (pairing && pairing[i] >= 0) {
            int64_t want = (q->E - q->M_last + pairing[i]) % C;
            if (pairing[i] >= q->M_last || best != want) return ORC_EPAIRING;
        }
        if (best >= 0) q->N_pos++;
    }
    q->N_neg = N - q->N_pos;
    for (int32_t k = 0; k < d; ++k) q->mu[k] = 0.0;
    for (int64_t c = 0; c < q->C_occ; ++c)
        for (int32_t k = 0; k < d; ++k) q->mu[k] += orc_tbar(q, c, k);
    return ORC_OK;
}

/* per-row loss contribution and gradient (steps 5-9 of the definition).
 * Writes ell (CE term, in-pool rows) or phi (cosine term, out-of-pool rows),
 * lse, the gradient dx_i (raw x) and optionally p_i[c] and accumulates dT. */
static void orc_row(const orc_ctx *q, int64_t i, double *ell, double *phi, double *lse,
                    double *dx, double *prow, double *dT, double *cos_buf, double *g) {
    int32_t d = q->d;
    int64_t Co = q->C_occ;
    double inv_n = 1.0 / q->n[i];
    /* x_hat */
    for (int32_t k = 0; k < d; ++k) g[k] = 0.0;
    for (int64_t c = 0; c < Co; ++c) {
        double dot = 0.0;
        for (int32_t k = 0; k < d; ++k)
            dot += orc_elem(q->X, q->dtype, i * d + k) * inv_n * orc_tbar(q, c, k);
        cos_buf[c] = dot; /* Eq. 8: (1/K) sum_k <F_p, T[c,k]> on the normalised feature */
    }
    *ell = 0.0;
    *phi = 0.0;
    *lse = 0.0;
    if (q->t[i] >= 0) {
        /* Eq. 9 with z_ic = s*cos_ic and the target logit s*(cos_it - m)  (D3) */
        int64_t t = q->t[i];
        double zmax = -INFINITY;
        for (int64_t c = 0; c < Co; ++c) {
            if (q->excl_dup && c != t && q->lab[c] == q->y[i]) continue; /* stale self-duplicate */
            double z = q->s * cos_buf[c] - (c == t ? q->s * q->m : 0.0);
            if (z > zmax) zmax = z;
        }
        double sum = 0.0;
        for (int64_t c = 0; c < Co; ++c) {
            if (q->excl_dup && c != t && q->lab[c] == q->y[i]) continue;
            double z = q->s * cos_buf[c] - (c == t ? q->s * q->m : 0.0);
            sum += exp(z - zmax);
        }
        double L = zmax + log(sum);
        *lse = L;
        *ell = L - (q->s * cos_buf[t] - q->s * q->m);
        double w = q->s / (double)q->N_pos;
        for (int64_t c = 0; c < Co; ++c) {
            if (q->excl_dup && c != t && q->lab[c] == q->y[i]) {
                if (prow) prow[c] = 0.0;
                continue;
            }
            double z = q->s * cos_buf[c] - (c == t ? q->s * q->m : 0.0);
            double p = exp(z - L);
            if (prow) prow[c] = p;
            double gc = w * (p - (c == t ? 1.0 : 0.0)); /* dL/dz * dz/dcos */
            for (int32_t k = 0; k < d; ++k) g[k] += gc * orc_tbar(q, c, k);
            if (dT)
                for (int32_t k = 0; k < d; ++k)
                    dT[c * d + k] += gc * orc_elem(q->X, q->dtype, i * d + k) * inv_n;
        }
    } else {
        /* L_cos: phi_i = R_c h(cos(x_i, T_bar_c)) over the occupied centers with a
         * nonzero T_bar, R = mean (D10) / sum / max, h = identity or the hinge
         * max(0, .) (NEXT-3); cos is the true cosine <x_hat, T_bar_c>/||T_bar_c|| (R4).
         * Gradient: (lambda / N_neg) dphi/dx_hat (P:167 normaliser 1/(M-I)). */
        if (Co > 0) {
            double acc = 0.0, best = -INFINITY;
            int64_t cbest = -1;
            for (int64_t c = 0; c < Co; ++c) {
                double tn = orc_tbar_norm(q, c);
                if (!(tn > 0.0)) continue;
                double cs = cos_buf[c] / tn;
                if (q->phi_mode == 2) {
                    if (cs > best) { best = cs; cbest = c; }
                } else {
                    acc += q->hinge ? (cs > 0.0 ? cs : 0.0) : cs;
                }
            }
            double w = q->lam / (double)q->N_neg;  /* dL/dphi_i */
            if (q->phi_mode == 0) { *phi = acc / (double)Co; w /= (double)Co; }
            else if (q->phi_mode == 1) { *phi = acc; }
            else { *phi = cbest < 0 ? 0.0 : (q->hinge && best <= 0.0 ? 0.0 : best); }
            for (int64_t c = 0; c < Co; ++c) {
                double tn = orc_tbar_norm(q, c);
                if (!(tn > 0.0)) continue;
                double cs = cos_buf[c] / tn;
                double hp;  /* dphi_i / dcos_c (before the reduction weight w) */
                if (q->phi_mode == 2) hp = (c == cbest && !(q->hinge && cs <= 0.0)) ? 1.0 : 0.0;
                else hp = q->hinge ? (cs > 0.0 ? 1.0 : 0.0) : 1.0;
                if (hp == 0.0) continue;
                double wc = w * hp / tn;
                for (int32_t k = 0; k < d; ++k) g[k] += wc * orc_tbar(q, c, k);
                if (dT)
                    for (int32_t k = 0; k < d; ++k)
                        dT[c * d + k] += wc * orc_elem(q->X, q->dtype, i * d + k) * inv_n;
            }
        }
    }
    /* normalisation Jacobian: dL/dx = (I - x_hat x_hat^T) g / ||x||  (D12) */
    double gx = 0.0;
    for (int32_t k = 0; k < d; ++k) gx += g[k] * orc_elem(q->X, q->dtype, i * d + k) * inv_n;
    for (int32_t k = 0; k < d; ++k) {
        double xh = orc_elem(q->X, q->dtype, i * d + k) * inv_n;
        dx[k] = (g[k] - gx * xh) * inv_n;
    }
}

/* Full definition over all N rows.
 * out3 = {L, L_ce, L_cos}; dx [N*d]; lse [N] (0 for out-of-pool rows); tslot [N];
 * phi [N] (0 for in-pool rows); ell [N] (0 for out-of-pool rows);
 * counts = {N_pos, N_neg, C_occ}; P [N * C_occ] or NULL; dT [C * d] or NULL. */
int orc_loss_v(int64_t C, int32_t K, int32_t d, int32_t dtype, const void *T, const int64_t *lab,
               int64_t E, int64_t M_last, int64_t N, const void *X, const int64_t *y,
               const int32_t *pairing, double s, double m, int32_t phi_mode, int32_t flags,
               double lam, double *out3, double *dx, double *lse, int64_t *tslot, double *phi,
               double *ell, int64_t *counts, double *P, double *dT) {
    if (C < 1 || d < 1 || K < 1 || N < 0 || (dtype != 0 && dtype != 1)) return ORC_EINVAL;
    if (!(s > 0.0) || !isfinite(m)) return ORC_EINVAL;
    if (phi_mode < 0 || phi_mode > 2 || flags < 0 || flags > 3 || !isfinite(lam)) return ORC_EINVAL;
    if (dT && K != 1) return ORC_EINVAL;
    orc_ctx q = {0};
    q.C = C; q.N = N; q.E = E; q.M_last = M_last; q.d = d; q.dtype = dtype; q.K = K;
    q.T = T; q.lab = lab; q.X = X; q.y = y; q.s = s; q.m = m;
    q.phi_mode = phi_mode; q.hinge = flags & 1; q.excl_dup = (flags >> 1) & 1; q.lam = lam;
    q.n = (double *)calloc((size_t)(N > 0 ? N : 1), sizeof(double));
    q.t = (int64_t *)calloc((size_t)(N > 0 ? N : 1), sizeof(int64_t));
    q.mu = (double *)calloc((size_t)d, sizeof(double));
    int64_t Cmax = C;
    double *cos_buf = (double *)calloc((size_t)Cmax, sizeof(double));
    double *g = (double *)calloc((size_t)d, sizeof(double));
    int rc = orc_prepare(&q, pairing);
    if (rc == ORC_OK) {
        if (dT) memset(dT, 0, (size_t)C * d * sizeof(double));
        double sce = 0.0, scos = 0.0;
        for (int64_t i = 0; i < N; ++i) {
            double e, f, l;
            orc_row(&q, i, &e, &f, &l, dx + i * d, P ? P + i * q.C_occ : NULL, dT, cos_buf, g);
            lse[i] = l; phi[i] = f; ell[i] = e; tslot[i] = q.t[i];
            sce += e;
            scos += f;
        }
        double Lce = q.N_pos > 0 ? sce / (double)q.N_pos : 0.0;  /* 1/I */
        double Lcos = q.N_neg > 0 ? scos / (double)q.N_neg : 0.0; /* 1/(M-I) */
        out3[0] = Lce + lam * Lcos; /* L_total = L_ce + L_cos; lambda: S:408 */
        out3[1] = Lce;
        out3[2] = Lcos;
        counts[0] = q.N_pos; counts[1] = q.N_neg; counts[2] = q.C_occ;
    }
    free(q.n); free(q.t); free(q.mu); free(cos_buf); free(g);
    return rc;
}

int orc_loss_k(int64_t C, int32_t K, int32_t d, int32_t dtype, const void *T, const int64_t *lab,
               int64_t E, int64_t M_last, int64_t N, const void *X, const int64_t *y,
               const int32_t *pairing, double s, double m, double *out3, double *dx, double *lse,
               int64_t *tslot, double *phi, double *ell, int64_t *counts, double *P, double *dT) {
    return orc_loss_v(C, K, d, dtype, T, lab, E, M_last, N, X, y, pairing, s, m, 0, 0, 1.0, out3, dx,
                      lse, tslot, phi, ell, counts, P, dT);
}

int orc_loss(int64_t C, int32_t d, int32_t dtype, const void *T, const int64_t *lab, int64_t E,
             int64_t M_last, int64_t N, const void *X, const int64_t *y, const int32_t *pairing,
             double s, double m, double *out3, double *dx, double *lse, int64_t *tslot, double *phi,
             double *ell, int64_t *counts, double *P, double *dT) {
    return orc_loss_k(C, 1, d, dtype, T, lab, E, M_last, N, X, y, pairing, s, m, out3, dx, lse, tslot,
                      phi, ell, counts, P, dT);
}

/* Same definition for a subset of rows (for configurations too large for the
 * full O(N*C*d) evaluation).  Normalisers are global.  Outputs are per selected
 * row: dx [nsel*d], lse, tslot, phi, ell. counts = {N_pos, N_neg, C_occ}. */
int orc_loss_rows_v(int64_t C, int32_t K, int32_t d, int32_t dtype, const void *T,
                    const int64_t *lab, int64_t E, int64_t M_last, int64_t N, const void *X,
                    const int64_t *y, const int32_t *pairing, double s, double m, int32_t phi_mode,
                    int32_t flags, double lam, int64_t nsel, const int64_t *rows, double *dx,
                    double *lse, int64_t *tslot, double *phi, double *ell, int64_t *counts,
                    double *mu_out) {
    if (C < 1 || d < 1 || K < 1 || N < 0 || (dtype != 0 && dtype != 1)) return ORC_EINVAL;
    if (phi_mode < 0 || phi_mode > 2 || flags < 0 || flags > 3 || !isfinite(lam)) return ORC_EINVAL;
    orc_ctx q = {0};
    q.C = C; q.N = N; q.E = E; q.M_last = M_last; q.d = d; q.dtype = dtype; q.K = K;
    q.T = T; q.lab = lab; q.X = X; q.y = y; q.s = s; q.m = m;
    q.phi_mode = phi_mode; q.hinge = flags & 1; q.excl_dup = (flags >> 1) & 1; q.lam = lam;
    q.n = (double *)calloc((size_t)(N > 0 ? N : 1), sizeof(double));
    q.t = (int64_t *)calloc((size_t)(N > 0 ? N : 1), sizeof(int64_t));
    q.mu = (double *)calloc((size_t)d, sizeof(double));
    double *cos_buf = (double *)calloc((size_t)C, sizeof(double));
    double *g = (double *)calloc((size_t)d, sizeof(double));
    int rc = orc_prepare(&q, pairing);
    if (rc == ORC_OK) {
        for (int64_t k = 0; k < nsel; ++k) {
            int64_t i = rows[k];
            double e, f, l;
            orc_row(&q, i, &e, &f, &l, dx + k * d, NULL, NULL, cos_buf, g);
            lse[k] = l; phi[k] = f; ell[k] = e; tslot[k] = q.t[i];
        }
        counts[0] = q.N_pos; counts[1] = q.N_neg; counts[2] = q.C_occ;
        if (mu_out) memcpy(mu_out, q.mu, (size_t)d * sizeof(double));
    }
    free(q.n); free(q.t); free(q.mu); free(cos_buf); free(g);
    return rc;
}

int orc_loss_rows_k(int64_t C, int32_t K, int32_t d, int32_t dtype, const void *T,
                    const int64_t *lab, int64_t E, int64_t M_last, int64_t N, const void *X,
                    const int64_t *y, const int32_t *pairing, double s, double m, int64_t nsel,
                    const int64_t *rows, double *dx, double *lse, int64_t *tslot, double *phi,
                    double *ell, int64_t *counts, double *mu_out) {
    return orc_loss_rows_v(C, K, d, dtype, T, lab, E, M_last, N, X, y, pairing, s, m, 0, 0, 1.0, nsel,
                           rows, dx, lse, tslot, phi, ell, counts, mu_out);
}

int orc_loss_rows(int64_t C, int32_t d, int32_t dtype, const void *T, const int64_t *lab,
                  int64_t E, int64_t M_last, int64_t N, const void *X, const int64_t *y,
                  const int32_t *pairing, double s, double m, int64_t nsel, const int64_t *rows,
                  double *dx, double *lse, int64_t *tslot, double *phi, double *ell,
                  int64_t *counts, double *mu_out) {
    return orc_loss_rows_k(C, 1, d, dtype, T, lab, E, M_last, N, X, y, pairing, s, m, nsel, rows, dx,
                           lse, tslot, phi, ell, counts, mu_out);
}

/* G-Net moving average: g <- m*g + (1-m)*p, evaluated in fp64
 * exactly in that order, rounded to nearest-even fp32 (D17). */
int orc_ema(const float *p, float *g, int64_t n, double momentum) {
    if (n < 0 || !(momentum >= 0.0 && momentum <= 1.0)) return ORC_EINVAL;
    for (int64_t k = 0; k < n; ++k) {
        double a = momentum * (double)g[k];
        double b = (1.0 - momentum) * (double)p[k];
        g[k] = (float)(a + b);
    }
    return ORC_OK;
}
