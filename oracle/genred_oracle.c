/*
 * genred_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the Genred hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or helper with
 * the CUDA path (paper_2004_11127_b200/csrc); neither side includes or links the other.
 *
 * What it computes is Eq. (1) of the paper (Sec. 2):
 *
 *        a_i = Reduction_{j=1..N} F(p, x_i, y_j),   i = 1..M
 *
 * written out as the plain definition, one row at a time, in fp64 on fp64 inputs (the Python
 * wrapper widens the fp32 inputs exactly).  No tiling, no fusion, no reordering: a double loop.
 * Sums use Neumaier compensated summation so the oracle's own rounding (~1e-16 of sum|terms|)
 * is negligible against every tolerance.  libm exp/log, compiled without -ffast-math.
 *
 * Functions and the passages they follow (readings R1..R18 are listed in DESIGN.md Sec. 3):
 *   oracle_gauss_sum    O1  F = exp(-|x_i-y_j|^2/sigma^2) * b_j           PAPER.md:166-167, 182 (R1)
 *   oracle_gauss_gradx  O2  G_i = sum_j (-2/sigma^2)(x_i-y_j) e_ij <b_j,g_i>  PAPER.md:141-147, 168 (R10)
 *   oracle_lse          O3  F = -|x_i-y_j|^2/eps + h_j ; a_i = m_i + log sum_j exp(F_ij - m_i)
 *   oracle_lse_cond         the metric's conditioning of O3 (reading R6b)
 *   oracle_gauss_cond       the metric's conditioning of O1 / O2 (reading R4c)
 *   oracle_softmax_cond     the metric's conditioning of O6 (reading R4c)
 *                                                                          PAPER.md:85, 134 (R5)
 *   oracle_argkmin      O4  K smallest (|x_i-y_j|^2, j) in lexicographic order   PAPER.md:85, 134 (R7-R9)
 *   oracle_sqdist_sum   O5  sum_j |x_i-y_j|^2 b_j  (test combination)
 *   oracle_softmax_grad O6  softmax-weighted sums / gradients (LSE backward)
 *
 * Every function takes an optional row subset (rows != NULL: evaluate only those rows, outputs
 * indexed by position in `rows`) so large configurations can be checked on a seeded sample.
 * Sum-type functions also return the per-coordinate denominator S_i = sum_j |term_ij| used by the
 * error metric (reading R4).  Parallelism: OpenMP over rows only (rows are independent, Eq. 1).
 *
 * Parity: pinned by tests/test_oracle_pins.py (closed forms, lattice products, invariants,
 * finite differences, brute-force sort); see DESIGN.md Sec. 4 for which pin covers which function.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Neumaier (improved Kahan) compensated summation. */
typedef struct { double sum, comp; } nsum;
static inline void nsum_add(nsum *s, double t) {
    double u = s->sum + t;
    if (fabs(s->sum) >= fabs(t)) s->comp += (s->sum - u) + t;
    else                          s->comp += (t - u) + s->sum;
    s->sum = u;
}
static inline double nsum_get(const nsum *s) { return s->sum + s->comp; }

/* Squared Euclidean distance |x - y|^2, computed directly (never expanded). */
static inline double sqdist(const double *x, const double *y, int D) {
    double acc = 0.0;
    for (int d = 0; d < D; ++d) {
        double diff = x[d] - y[d];
        acc += diff * diff;
    }
    return acc;
}

static inline int64_t row_of(const int64_t *rows, int64_t r) { return rows ? rows[r] : r; }

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* O1: a_i[e] = sum_j exp(-|x_i - y_j|^2 / sigma^2) * b_j[e]   (b == NULL means b == 1, E == 1). */
void oracle_gauss_sum(int64_t M, int64_t N, int D, int E, double sigma,
                      const double *x, const double *y, const double *b,
                      const int64_t *rows, int64_t nrows,
                      double *out, double *denom) {
    int64_t R = rows ? nrows : M;
    double inv_s2 = 1.0 / (sigma * sigma);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < R; ++r) {
        int64_t i = row_of(rows, r);
        nsum *acc = calloc((size_t)E, sizeof(nsum));
        nsum *den = calloc((size_t)E, sizeof(nsum));
        for (int64_t j = 0; j < N; ++j) {
            double k = exp(-sqdist(x + i * D, y + j * D, D) * inv_s2);
            for (int e = 0; e < E; ++e) {
                double t = k * (b ? b[j * E + e] : 1.0);
                nsum_add(&acc[e], t);
                nsum_add(&den[e], fabs(t));
            }
        }
        for (int e = 0; e < E; ++e) {
            out[r * E + e] = nsum_get(&acc[e]);
            if (denom) denom[r * E + e] = nsum_get(&den[e]);
        }
        free(acc);
        free(den);
    }
}

/* O2: G_i[d] = sum_j (-2/sigma^2) (x_i[d] - y_j[d]) exp(-|x_i-y_j|^2/sigma^2) <b_j, g_i>
 * (the vector-Jacobian product of O1 with respect to x_i; b == NULL -> 1, g == NULL -> 1). */
void oracle_gauss_gradx(int64_t M, int64_t N, int D, int E, double sigma,
                        const double *x, const double *y, const double *b, const double *g,
                        const int64_t *rows, int64_t nrows,
                        double *out, double *denom) {
    int64_t R = rows ? nrows : M;
    double inv_s2 = 1.0 / (sigma * sigma);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < R; ++r) {
        int64_t i = row_of(rows, r);
        nsum *acc = calloc((size_t)D, sizeof(nsum));
        nsum *den = calloc((size_t)D, sizeof(nsum));
        for (int64_t j = 0; j < N; ++j) {
            double k = exp(-sqdist(x + i * D, y + j * D, D) * inv_s2);
            double bg = 0.0, bga = 0.0;
            for (int e = 0; e < E; ++e) {
                const double p = (b ? b[j * E + e] : 1.0) * (g ? g[i * E + e] : 1.0);
                bg += p;
                bga += fabs(p);
            }
            for (int d = 0; d < D; ++d) {
                double t = -2.0 * inv_s2 * (x[i * D + d] - y[j * D + d]) * k;
                nsum_add(&acc[d], t * bg);
                /* R4b: the terms are the elementary products t b_je g_ie, so the denominator
                 * sums |t| sum_e |b_je g_ie| (equal to |t bg| when E = 1) */
                nsum_add(&den[d], fabs(t) * bga);
            }
        }
        for (int d = 0; d < D; ++d) {
            out[r * D + d] = nsum_get(&acc[d]);
            if (denom) denom[r * D + d] = nsum_get(&den[d]);
        }
        free(acc);
        free(den);
    }
}

/* Conditioning of O1 (grad = 0) / O2 (grad = 1) for the error metric (reading R4c), per output
 * column c (E columns of O1, D of O2), with term_ij the elementary terms whose |.| sum is the R4
 * denominator and u_ij = |x_i - y_j|^2 / sigma^2 the exponent (k_ij = exp(-u_ij)):
 *   cond[r, c] = sum_j |term_ij| u_ij      -- an fp32 evaluation rounds u_ij by a few ulps, which
 *                                             moves k_ij by that relative amount times u_ij;
 *   tail[r, c] = sum_j |term_ij| [u_ij log2(e) >= 100]  -- terms below 2^-100: a product of k_ij
 *                                             with the other factors leaves fp32's normal range. */
void oracle_gauss_cond(int64_t M, int64_t N, int D, int E, double sigma, int grad,
                       const double *x, const double *y, const double *b, const double *g,
                       const int64_t *rows, int64_t nrows, double *cond, double *tail) {
    int64_t R = rows ? nrows : M;
    double inv_s2 = 1.0 / (sigma * sigma);
    const int C = grad ? D : E;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < R; ++r) {
        int64_t i = row_of(rows, r);
        nsum *cs = calloc((size_t)C, sizeof(nsum));
        nsum *ts = calloc((size_t)C, sizeof(nsum));
        for (int64_t j = 0; j < N; ++j) {
            const double u = sqdist(x + i * D, y + j * D, D) * inv_s2;
            const double k = exp(-u);
            const int deep = u * 1.4426950408889634 >= 100.0;
            double bga = 0.0;
            if (grad)
                for (int e = 0; e < E; ++e)
                    bga += fabs((b ? b[j * E + e] : 1.0) * (g ? g[i * E + e] : 1.0));
            for (int c = 0; c < C; ++c) {
                const double t = grad ? fabs(2.0 * inv_s2 * (x[i * D + c] - y[j * D + c]) * k) * bga
                                      : fabs(k * (b ? b[j * E + c] : 1.0));
                nsum_add(&cs[c], t * u);
                if (deep) nsum_add(&ts[c], t);
            }
        }
        for (int c = 0; c < C; ++c) {
            cond[r * C + c] = nsum_get(&cs[c]);
            tail[r * C + c] = nsum_get(&ts[c]);
        }
        free(cs);
        free(ts);
    }
}

/* O3: F_ij = -|x_i - y_j|^2 / eps + h_j  (h == NULL -> 0);
 *     m_i = max_j F_ij ;  a_i = m_i + log sum_j exp(F_ij - m_i)   (two passes; N == 0 -> -inf). */
void oracle_lse(int64_t M, int64_t N, int D, double eps,
                const double *x, const double *y, const double *h,
                const int64_t *rows, int64_t nrows,
                double *out, double *mmax) {
    int64_t R = rows ? nrows : M;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < R; ++r) {
        int64_t i = row_of(rows, r);
        double m = -INFINITY;
        for (int64_t j = 0; j < N; ++j) {
            double F = -sqdist(x + i * D, y + j * D, D) / eps + (h ? h[j] : 0.0);
            if (F > m) m = F;
        }
        double a;
        if (N == 0 || m == -INFINITY) {
            a = -INFINITY;
        } else {
            nsum s = {0.0, 0.0};
            for (int64_t j = 0; j < N; ++j) {
                double F = -sqdist(x + i * D, y + j * D, D) / eps + (h ? h[j] : 0.0);
                nsum_add(&s, exp(F - m));
            }
            a = m + log(nsum_get(&s));
        }
        out[r] = a;
        if (mmax) mmax[r] = m;
    }
}

/* Conditioning of O3 for the error metric (reading R6b): C_i = sum_j p_ij (|x_i-y_j|^2/eps + |h_j|),
 * p_ij = exp(F_ij - a_i) the softmax weights.  a_i moves by sum_j p_ij dF_ij when each F_ij is
 * perturbed by dF_ij, and an fp32 evaluation perturbs F_ij by a few ulps of its two parts. */
void oracle_lse_cond(int64_t M, int64_t N, int D, double eps,
                     const double *x, const double *y, const double *h,
                     const int64_t *rows, int64_t nrows, const double *a, double *cond) {
    int64_t R = rows ? nrows : M;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < R; ++r) {
        int64_t i = row_of(rows, r);
        nsum c = {0.0, 0.0};
        if (isfinite(a[r])) {
            for (int64_t j = 0; j < N; ++j) {
                const double q = sqdist(x + i * D, y + j * D, D) / eps;
                const double hj = h ? h[j] : 0.0;
                nsum_add(&c, exp(-q + hj - a[r]) * (q + fabs(hj)));
            }
        }
        cond[r] = nsum_get(&c);
    }
}

/* (d, j) lexicographic order: smaller distance first, ties broken by the lower index (R7). */
static inline int lex_less(double d1, int64_t j1, double d2, int64_t j2) {
    return d1 < d2 || (d1 == d2 && j1 < j2);
}

/* O4: the K pairs (d_ij, j) smallest in (d, j) order, ascending; K > N pads (+inf, -1) (R9). */
void oracle_argkmin(int64_t M, int64_t N, int D, int K,
                    const double *x, const double *y,
                    const int64_t *rows, int64_t nrows,
                    double *dist, int64_t *idx) {
    int64_t R = rows ? nrows : M;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < R; ++r) {
        int64_t i = row_of(rows, r);
        double *bd = dist + r * K;
        int64_t *bj = idx + r * K;
        for (int k = 0; k < K; ++k) { bd[k] = INFINITY; bj[k] = -1; }
        int filled = 0;
        for (int64_t j = 0; j < N; ++j) {
            double d = sqdist(x + i * D, y + j * D, D);
            if (filled == K && !lex_less(d, j, bd[K - 1], bj[K - 1])) continue;
            /* insertion into the sorted list */
            int pos = filled < K ? filled : K - 1;
            while (pos > 0 && lex_less(d, j, bd[pos - 1], bj[pos - 1])) {
                bd[pos] = bd[pos - 1];
                bj[pos] = bj[pos - 1];
                --pos;
            }
            bd[pos] = d;
            bj[pos] = j;
            if (filled < K) ++filled;
        }
    }
}

/* O5: a_i[e] = sum_j |x_i - y_j|^2 b_j[e]   (b == NULL -> 1, E == 1). */
void oracle_sqdist_sum(int64_t M, int64_t N, int D, int E,
                       const double *x, const double *y, const double *b,
                       const int64_t *rows, int64_t nrows,
                       double *out, double *denom) {
    int64_t R = rows ? nrows : M;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < R; ++r) {
        int64_t i = row_of(rows, r);
        nsum *acc = calloc((size_t)E, sizeof(nsum));
        nsum *den = calloc((size_t)E, sizeof(nsum));
        for (int64_t j = 0; j < N; ++j) {
            double d2 = sqdist(x + i * D, y + j * D, D);
            for (int e = 0; e < E; ++e) {
                double t = d2 * (b ? b[j * E + e] : 1.0);
                nsum_add(&acc[e], t);
                nsum_add(&den[e], fabs(t));
            }
        }
        for (int e = 0; e < E; ++e) {
            out[r * E + e] = nsum_get(&acc[e]);
            if (denom) denom[r * E + e] = nsum_get(&den[e]);
        }
        free(acc);
        free(den);
    }
}

/* O6 (the backward of O3): softmax-weighted reductions
 *     p_ij   = exp(-|x_i - y_j|^2 / eps + alpha_i + beta_j)
 *     S_i    = sum_j sig_j p_ij                                   (out_sum, M)
 *     G_i[d] = coef_i sum_j sig_j p_ij (-2/eps) (x_i[d] - y_j[d])  (out_grad, M x D)
 * With alpha_i = -a_i (a = O3's LSE), beta = h, sig = coef = 1: S_i = 1 and G_i = da_i/dx_i
 * (the gradient of a reduction is another reduction).  NULL alpha/beta -> 0,
 * NULL sig/coef -> 1.  Denominators: sum_j |sig_j| p_ij and coef-scaled sum of |terms|. */
void oracle_softmax_grad(int64_t M, int64_t N, int D, double eps,
                         const double *x, const double *y, const double *alpha, const double *beta,
                         const double *sig, const double *coef,
                         const int64_t *rows, int64_t nrows,
                         double *out_sum, double *out_grad, double *den_sum, double *den_grad) {
    int64_t R = rows ? nrows : M;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < R; ++r) {
        int64_t i = row_of(rows, r);
        nsum s = {0.0, 0.0}, sd = {0.0, 0.0};
        nsum *g = calloc((size_t)D, sizeof(nsum));
        nsum *gd = calloc((size_t)D, sizeof(nsum));
        double c = coef ? coef[i] : 1.0;
        for (int64_t j = 0; j < N; ++j) {
            double p = exp(-sqdist(x + i * D, y + j * D, D) / eps + (alpha ? alpha[i] : 0.0) +
                           (beta ? beta[j] : 0.0));
            double w = (sig ? sig[j] : 1.0) * p;
            nsum_add(&s, w);
            nsum_add(&sd, fabs(w));
            for (int d = 0; d < D; ++d) {
                double t = c * w * (-2.0 / eps) * (x[i * D + d] - y[j * D + d]);
                nsum_add(&g[d], t);
                nsum_add(&gd[d], fabs(t));
            }
        }
        out_sum[r] = nsum_get(&s);
        if (den_sum) den_sum[r] = nsum_get(&sd);
        for (int d = 0; d < D; ++d) {
            out_grad[r * D + d] = nsum_get(&g[d]);
            if (den_grad) den_grad[r * D + d] = nsum_get(&gd[d]);
        }
        free(g);
        free(gd);
    }
}

/* Conditioning of O6 for the error metric (reading R4c, as oracle_gauss_cond): with the exponent's
 * parts u_ij = |x_i - y_j|^2/eps, alpha_i, beta_j (each rounded in fp32 by a few ulps) and the
 * elementary terms of S_i (w_ij = sig_j p_ij) and G_i[d] (c_i w_ij (-2/eps)(x_i - y_j)_d):
 *   cond = sum_j |term_ij| (u_ij + |alpha_i| + |beta_j|),
 *   tail = sum_j |term_ij| [(-u_ij + alpha_i + beta_j) log2(e) <= -100]. */
void oracle_softmax_cond(int64_t M, int64_t N, int D, double eps,
                         const double *x, const double *y, const double *alpha, const double *beta,
                         const double *sig, const double *coef,
                         const int64_t *rows, int64_t nrows,
                         double *cond_sum, double *cond_grad, double *tail_sum, double *tail_grad) {
    int64_t R = rows ? nrows : M;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < R; ++r) {
        int64_t i = row_of(rows, r);
        nsum cs = {0.0, 0.0}, ts = {0.0, 0.0};
        nsum *cg = calloc((size_t)D, sizeof(nsum));
        nsum *tg = calloc((size_t)D, sizeof(nsum));
        double c = coef ? coef[i] : 1.0;
        double ai = alpha ? alpha[i] : 0.0;
        for (int64_t j = 0; j < N; ++j) {
            const double u = sqdist(x + i * D, y + j * D, D) / eps;
            const double bj = beta ? beta[j] : 0.0;
            const double z = -u + ai + bj;
            const double mag = u + fabs(ai) + fabs(bj);
            const int deep = z * 1.4426950408889634 <= -100.0;
            const double w = fabs((sig ? sig[j] : 1.0) * exp(z));
            nsum_add(&cs, w * mag);
            if (deep) nsum_add(&ts, w);
            for (int d = 0; d < D; ++d) {
                const double t = fabs(c * w * (-2.0 / eps) * (x[i * D + d] - y[j * D + d]));
                nsum_add(&cg[d], t * mag);
                if (deep) nsum_add(&tg[d], t);
            }
        }
        cond_sum[r] = nsum_get(&cs);
        tail_sum[r] = nsum_get(&ts);
        for (int d = 0; d < D; ++d) {
            cond_grad[r * D + d] = nsum_get(&cg[d]);
            tail_grad[r * D + d] = nsum_get(&tg[d]);
        }
        free(cg);
        free(tg);
    }
}
