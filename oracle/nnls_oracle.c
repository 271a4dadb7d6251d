/*
 * oracle/nnls_oracle.c -- CPU restatement of the reference's compiled shard
 * kernels (nmfkit/kernels.py), in plain C.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
 * baseline / `--impl reference` arm may load it.  The product package
 * (paper_1506_08938_b200/) never links, imports or calls anything here.
 *
 * Pinned against the reference: tests/golden/make_golden.py runs the
 * reference's numba kernels on seeded batches and commits their outputs;
 * tests/test_oracle_golden.py checks this file reproduces them bit for bit.
 *
 * Build: see oracle/Makefile.  MUST be compiled with -ffp-contract=off and
 * without -ffast-math: numba (fastmath=False) never fuses a multiply and an
 * add, so bit parity requires that every product is rounded before the sum.
 *
 * Array conventions follow kernels.py:9-15 (all C-contiguous, float64,
 * int64 indices, uint8 bool mask):
 *   G  (n, r)   FT (m, r)   YT (n, r)   HP (r, r)   VT (m, n)   Qa (ra, ra)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define FAIL_NONE (-1)      /* kernels.py:27 */
#define FASTBREAK_BLOCK 32  /* kernels.py:35 */

/* Python's builtin max(a, b): b only when strictly greater (kernels.py:117). */
static inline double py_max(double a, double b) { return (b > a) ? b : a; }

/* kernels.py:153-175 (_take_step): projected step y -> [y - alpha d]+,
 * fills ynew, delta, qd = Q delta; returns the exact objective change. */
static double take_step(const double *Q, int64_t r, const double *y,
                        const double *grad, const double *d, double alpha,
                        double *ynew, double *delta, double *qd) {
    for (int64_t i = 0; i < r; ++i) {
        double v = y[i] - alpha * d[i];
        if (v < 0.0) v = 0.0;
        ynew[i] = v;
        delta[i] = v - y[i];
        qd[i] = 0.0;
    }
    for (int64_t j = 0; j < r; ++j) {
        double dj = delta[j];
        if (dj != 0.0) {
            for (int64_t i = 0; i < r; ++i) qd[i] += Q[i * r + j] * dj;
        }
    }
    double df = 0.0;
    for (int64_t i = 0; i < r; ++i) df += grad[i] * delta[i] + 0.5 * delta[i] * qd[i];
    return df;
}

/* kernels.py:38-150 (_solve_rescaled).  Returns iterations (negated on a
 * NaN/Inf), writes initial and final squared passive-gradient norms. */
int64_t oracle_solve_rescaled(const double *Q, int64_t r, double *y, double *grad,
                              double eps, double max_stop, int64_t max_inner,
                              double *d, double *ynew, double *delta, double *qd,
                              double *norm0_out, double *normk_out) {
    double norm0 = 0.0;
    for (int64_t i = 0; i < r; ++i)
        if (y[i] > 0.0 || grad[i] < 0.0) norm0 += grad[i] * grad[i];
    if (norm0 <= 0.0) {
        *norm0_out = norm0;
        *normk_out = norm0;
        return 0;
    }
    double threshold = eps * norm0;
    double norm_k = norm0;
    int64_t iterations = 0;
    while (iterations < max_inner) {
        int moved = 0;
        /* exact line search over the passive set (kernels.py:57-103) */
        double nsq = 0.0;
        for (int64_t i = 0; i < r; ++i) {
            if (y[i] > 0.0 || grad[i] < 0.0) {
                d[i] = grad[i];
                nsq += d[i] * d[i];
            } else {
                d[i] = 0.0;
            }
        }
        if (nsq > 0.0) {
            double curv = 0.0;
            for (int64_t i = 0; i < r; ++i) {
                double acc = 0.0;
                for (int64_t j = 0; j < r; ++j) acc += Q[i * r + j] * d[j];
                qd[i] = acc;
                curv += d[i] * acc;
            }
            double alpha = (curv > 0.0) ? nsq / curv : 1.0;
            int clamped = 0;
            for (int64_t i = 0; i < r; ++i) {
                double v = y[i] - alpha * d[i];
                if (v < 0.0) {
                    clamped = 1;
                    v = 0.0;
                }
                ynew[i] = v;
                delta[i] = v - y[i];
            }
            if (!clamped) {
                /* the free step: Q delta = -alpha Q d (kernels.py:82-88);
                 * df is computed there but never read on this branch */
                for (int64_t i = 0; i < r; ++i) qd[i] = -alpha * qd[i];
            } else {
                double df = take_step(Q, r, y, grad, d, alpha, ynew, delta, qd);
                if (df > 0.0) {
                    double alpha_bp = INFINITY;
                    for (int64_t i = 0; i < r; ++i) {
                        if (d[i] > 0.0 && y[i] > 0.0) {
                            double c = y[i] / d[i];
                            if (c < alpha_bp) alpha_bp = c;
                        }
                    }
                    if (alpha_bp < alpha)
                        take_step(Q, r, y, grad, d, alpha_bp, ynew, delta, qd);
                }
            }
            for (int64_t i = 0; i < r; ++i) {
                if (delta[i] != 0.0) moved = 1;
                y[i] = ynew[i];
                grad[i] += qd[i];
            }
        }
        /* greedy coordinate descent, r updates, gradient update of the chosen
         * coordinate fused into the next scan (kernels.py:104-132) */
        int64_t pending_p = -1;
        double pending_dx = 0.0;
        for (int64_t s = 0; s < r; ++s) {
            double best = 0.0;
            int64_t p = -1;
            double best_dx = 0.0;
            for (int64_t i = 0; i < r; ++i) {
                double gi = grad[i];
                if (pending_p >= 0) {
                    gi += Q[i * r + pending_p] * pending_dx;
                    grad[i] = gi;
                }
                double dxi = py_max(y[i] - gi, 0.0) - y[i];
                double dec = fabs(gi * dxi + 0.5 * dxi * dxi);
                if (dec > best) {
                    best = dec;
                    p = i;
                    best_dx = dxi;
                }
            }
            pending_p = -1;
            if (p < 0) break;
            y[p] += best_dx;
            moved = 1;
            pending_p = p;
            pending_dx = best_dx;
        }
        if (pending_p >= 0)
            for (int64_t i = 0; i < r; ++i) grad[i] += Q[i * r + pending_p] * pending_dx;
        iterations += 1;
        for (int64_t i = 0; i < r; ++i) {
            if (!(isfinite(y[i]) && isfinite(grad[i]))) {
                *norm0_out = norm0;
                *normk_out = NAN;
                return -iterations;
            }
        }
        norm_k = 0.0;
        for (int64_t i = 0; i < r; ++i)
            if (y[i] > 0.0 || grad[i] < 0.0) norm_k += grad[i] * grad[i];
        if (norm_k <= threshold || norm_k <= max_stop) break;
        if (!moved) break; /* stagnation (kernels.py:147-149) */
    }
    *norm0_out = norm0;
    *normk_out = norm_k;
    return iterations;
}

/* Scratch for one shard call: the dozen length-r vectors of kernels.py:234-243. */
typedef struct {
    double *hbuf, *x_full, *warm, *y, *grad, *q, *d, *ynew, *delta, *qd;
} scratch_t;

static int scratch_alloc(scratch_t *s, int64_t r_full, int64_t ra) {
    int64_t rf = r_full > 0 ? r_full : 1, rr = ra > 0 ? ra : 1;
    double *block = (double *)calloc((size_t)(3 * rf + 7 * rr), sizeof(double));
    if (!block) return -1;
    s->hbuf = block;
    s->x_full = block + rf;
    s->warm = block + 2 * rf;
    s->y = block + 3 * rf;
    s->grad = s->y + rr;
    s->q = s->grad + rr;
    s->d = s->q + rr;
    s->ynew = s->d + rr;
    s->delta = s->ynew + rr;
    s->qd = s->delta + rr;
    return 0;
}

/* kernels.py:178-220 (_coefficient_solve).  Returns iterations, or < 0 on a
 * NaN inside the solve / an unbounded frozen dimension. */
int64_t oracle_coefficient_solve(const double *hbuf, int64_t r_full, const int64_t *act_idx,
                                 int64_t ra, const uint8_t *active, const double *scale_a,
                                 const double *Qa, const double *warm, double eps,
                                 double max_stop, int64_t max_inner, double *x_full,
                                 double *normk_out, double *work /* 7*ra */) {
    double *y = work, *grad = work + ra, *q = work + 2 * ra, *d = work + 3 * ra;
    double *ynew = work + 4 * ra, *delta = work + 5 * ra, *qd = work + 6 * ra;
    int all_nonneg = 1;
    for (int64_t i = 0; i < r_full; ++i) {
        if (hbuf[i] < 0.0) {
            all_nonneg = 0;
            break;
        }
    }
    if (all_nonneg) {
        for (int64_t i = 0; i < r_full; ++i) x_full[i] = 0.0;
        *normk_out = 0.0;
        return 0;
    }
    for (int64_t i = 0; i < r_full; ++i) {
        if (!active[i] && hbuf[i] < 0.0) {
            *normk_out = NAN;
            return -1;
        }
    }
    for (int64_t k = 0; k < ra; ++k) {
        int64_t i = act_idx[k];
        q[k] = hbuf[i] / scale_a[k];
        y[k] = warm[i] * scale_a[k];
    }
    for (int64_t k = 0; k < ra; ++k) {
        double acc = q[k];
        for (int64_t j = 0; j < ra; ++j) acc += Qa[k * ra + j] * y[j];
        grad[k] = acc;
    }
    double n0, nk;
    int64_t iters = oracle_solve_rescaled(Qa, ra, y, grad, eps, max_stop, max_inner, d, ynew,
                                          delta, qd, &n0, &nk);
    if (iters < 0) {
        *normk_out = NAN;
        return iters;
    }
    for (int64_t i = 0; i < r_full; ++i) x_full[i] = 0.0;
    for (int64_t k = 0; k < ra; ++k) x_full[act_idx[k]] = y[k] / scale_a[k];
    *normk_out = nk;
    return iters;
}

/* Common tail of the three shard loops: solve, fast-break bookkeeping.
 * Returns 0 or -1 (failure). */
static int solve_one(scratch_t *s, int64_t r_full, const int64_t *act_idx, int64_t ra,
                     const uint8_t *active, const double *scale_a, const double *Qa, double eps,
                     double *max_stop, int64_t max_inner, int64_t *inner_total) {
    double nk;
    int64_t iters = oracle_coefficient_solve(s->hbuf, r_full, act_idx, ra, active, scale_a, Qa,
                                             s->warm, eps, *max_stop, max_inner, s->x_full, &nk,
                                             s->y);
    if (iters < 0) return -1;
    *inner_total += iters;
    if (nk > *max_stop) *max_stop = nk; /* kernels.py:266-267 */
    return 0;
}

/* kernels.py:223-281 (estep_sparse).  Returns the failing column or -1. */
int64_t oracle_estep_sparse(const int64_t *indptr, const int64_t *rowidx, const double *vals,
                            int64_t col_lo, int64_t col_hi, const double *G, int64_t r_full,
                            const double *Qa, const double *scale_a, const int64_t *act_idx,
                            int64_t ra, const uint8_t *active, double mu1, double eps,
                            int64_t max_inner, double max_stop0, double *FT, double *YT,
                            double *HP, int64_t *inner_total_out, double *max_stop_out) {
    scratch_t s;
    if (scratch_alloc(&s, r_full, ra)) return -2;
    int64_t inner_total = 0, fail = FAIL_NONE;
    double max_stop = max_stop0;
    for (int64_t col = col_lo; col < col_hi; ++col) {
        if (col % FASTBREAK_BLOCK == 0) max_stop = 0.0;
        int64_t p0 = indptr[col], p1 = indptr[col + 1];
        for (int64_t i = 0; i < r_full; ++i) {
            s.hbuf[i] = mu1;
            s.warm[i] = FT[col * r_full + i];
        }
        for (int64_t t = p0; t < p1; ++t) {
            const double *grow = G + rowidx[t] * r_full;
            double v = vals[t];
            for (int64_t i = 0; i < r_full; ++i) s.hbuf[i] -= grow[i] * v;
        }
        if (solve_one(&s, r_full, act_idx, ra, active, scale_a, Qa, eps, &max_stop, max_inner,
                      &inner_total)) {
            fail = col;
            break;
        }
        for (int64_t i = 0; i < r_full; ++i) FT[col * r_full + i] = s.x_full[i];
        for (int64_t t = p0; t < p1; ++t) {
            double *yrow = YT + rowidx[t] * r_full;
            double v = vals[t];
            for (int64_t i = 0; i < r_full; ++i) yrow[i] += s.x_full[i] * v;
        }
        /* upper triangle only; mirrored once per shard by the caller */
        for (int64_t a = 0; a < r_full; ++a) {
            double xa = s.x_full[a];
            if (xa != 0.0)
                for (int64_t b = a; b < r_full; ++b) HP[a * r_full + b] += xa * s.x_full[b];
        }
    }
    free(s.hbuf);
    *inner_total_out = inner_total;
    *max_stop_out = max_stop;
    return fail;
}

/* kernels.py:284-336 (estep_dense): VT is (m, n) C-contiguous. */
int64_t oracle_estep_dense(const double *VT, int64_t n, int64_t col_lo, int64_t col_hi,
                           const double *G, int64_t r_full, const double *Qa,
                           const double *scale_a, const int64_t *act_idx, int64_t ra,
                           const uint8_t *active, double mu1, double eps, int64_t max_inner,
                           double max_stop0, double *FT, double *YT, double *HP,
                           int64_t *inner_total_out, double *max_stop_out) {
    scratch_t s;
    if (scratch_alloc(&s, r_full, ra)) return -2;
    int64_t inner_total = 0, fail = FAIL_NONE;
    double max_stop = max_stop0;
    for (int64_t col = col_lo; col < col_hi; ++col) {
        if (col % FASTBREAK_BLOCK == 0) max_stop = 0.0;
        const double *vcol = VT + col * n;
        for (int64_t i = 0; i < r_full; ++i) {
            s.hbuf[i] = mu1;
            s.warm[i] = FT[col * r_full + i];
        }
        for (int64_t row = 0; row < n; ++row) {
            double v = vcol[row];
            if (v != 0.0) {
                const double *grow = G + row * r_full;
                for (int64_t i = 0; i < r_full; ++i) s.hbuf[i] -= grow[i] * v;
            }
        }
        if (solve_one(&s, r_full, act_idx, ra, active, scale_a, Qa, eps, &max_stop, max_inner,
                      &inner_total)) {
            fail = col;
            break;
        }
        for (int64_t i = 0; i < r_full; ++i) FT[col * r_full + i] = s.x_full[i];
        for (int64_t row = 0; row < n; ++row) {
            double v = vcol[row];
            if (v != 0.0) {
                double *yrow = YT + row * r_full;
                for (int64_t i = 0; i < r_full; ++i) yrow[i] += s.x_full[i] * v;
            }
        }
        for (int64_t a = 0; a < r_full; ++a) {
            double xa = s.x_full[a];
            if (xa != 0.0)
                for (int64_t b = a; b < r_full; ++b) HP[a * r_full + b] += xa * s.x_full[b];
        }
    }
    free(s.hbuf);
    *inner_total_out = inner_total;
    *max_stop_out = max_stop;
    return fail;
}

/* kernels.py:339-378 (mstep_rows): solves rows [row_lo, row_hi) of G. */
int64_t oracle_mstep_rows(const double *YT, int64_t row_lo, int64_t row_hi, const double *Qa,
                          const double *scale_a, const int64_t *act_idx, int64_t ra,
                          const uint8_t *active, double beta1, double eps, int64_t max_inner,
                          double max_stop0, double *G, int64_t r_full, int64_t *inner_total_out,
                          double *max_stop_out) {
    scratch_t s;
    if (scratch_alloc(&s, r_full, ra)) return -2;
    int64_t inner_total = 0, fail = FAIL_NONE;
    double max_stop = max_stop0;
    for (int64_t row = row_lo; row < row_hi; ++row) {
        if (row % FASTBREAK_BLOCK == 0) max_stop = 0.0;
        for (int64_t i = 0; i < r_full; ++i) {
            s.hbuf[i] = beta1 - YT[row * r_full + i];
            s.warm[i] = G[row * r_full + i];
        }
        if (solve_one(&s, r_full, act_idx, ra, active, scale_a, Qa, eps, &max_stop, max_inner,
                      &inner_total)) {
            fail = row;
            break;
        }
        for (int64_t i = 0; i < r_full; ++i) G[row * r_full + i] = s.x_full[i];
    }
    free(s.hbuf);
    *inner_total_out = inner_total;
    *max_stop_out = max_stop;
    return fail;
}

/* Sparse objective cross term sum_nnz v * <G[row,:], FT[col,:]> for columns
 * [col_lo, col_hi): the formula of matrix.py:246-250 evaluated as an nnz loop
 * (no nnz x r temporaries), used only where the reference's own gathers would
 * not fit in memory.  Plain sequential fp64 sums. */
double oracle_sparse_cross(const int64_t *indptr, const int64_t *rowidx, const double *vals,
                           int64_t col_lo, int64_t col_hi, const double *G, const double *FT,
                           int64_t r) {
    double cross = 0.0;
    for (int64_t col = col_lo; col < col_hi; ++col) {
        const double *f = FT + col * r;
        for (int64_t t = indptr[col]; t < indptr[col + 1]; ++t) {
            const double *g = G + rowidx[t] * r;
            double dot = 0.0;
            for (int64_t i = 0; i < r; ++i) dot += g[i] * f[i];
            cross += dot * vals[t];
        }
    }
    return cross;
}
