/*
 * dd_oracle.c -- CPU ORACLE (test infrastructure only; see dd_oracle.h).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fopenmp -shared -fPIC
 * (no -ffast-math). Every floating-point operation is written out in the
 * order DESIGN.md section 4 ("Arithmetic order") fixes.
 */
#include "dd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 0;

void orc_set_threads(int n) {
    g_threads = n;
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#endif
}

int orc_get_threads(void) {
#ifdef _OPENMP
    return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------- Alg. 2 */
/* P:239-261. b_x = n_x / nblk_x, b_y = n_y / nblk_y (b_z unused, R5). */
int orc_labels_geometric(int32_t nx, int32_t ny, int32_t nz, int32_t tx, int32_t ty,
                         int32_t tz, int32_t *part_id) {
    if (tx <= 0 || ty <= 0 || tz <= 0 || nx % tx || ny % ty || nz % tz) return -1;
    int64_t bx = nx / tx, by = ny / ty;
    for (int64_t i = 0; i < nx; i++) {
        int64_t ibx = i / tx;
        for (int64_t j = 0; j < ny; j++) {
            int64_t jby = j / ty;
            for (int64_t k = 0; k < nz; k++) {
                int64_t kbz = k / tz;
                int64_t gidx = i + (int64_t)nx * (j + (int64_t)ny * k);
                int64_t pidx = ibx + bx * (jby + by * kbz);
                part_id[gidx] = (int32_t)pidx;
            }
        }
    }
    return 0;
}

void orc_labels_bfs(int64_t n, const int64_t *rp, const int32_t *ci, int32_t P, int32_t *part_id) {
    int64_t *queue = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) part_id[i] = -1;
    int64_t assigned = 0, seed = 0;
    int32_t part = 0;
    while (assigned < n) {
        int64_t head = 0, tail = 0, filled = 0;
        while (filled < P && assigned < n) {
            if (head == tail) { /* new BFS source: the lowest unassigned row */
                while (part_id[seed] != -1) seed++;
                part_id[seed] = part;
                filled++;
                assigned++;
                queue[tail++] = seed;
                continue;
            }
            int64_t u = queue[head++];
            for (int64_t p = rp[u]; p < rp[u + 1] && filled < P; p++) {
                int64_t v = ci[p];
                if (v != u && part_id[v] == -1) {
                    part_id[v] = part;
                    filled++;
                    assigned++;
                    queue[tail++] = v;
                }
            }
        }
        part++;
    }
    free(queue);
}

void orc_labels_chunks(int64_t n, int32_t P, int32_t *part_id) {
    for (int64_t i = 0; i < n; i++) part_id[i] = (int32_t)(i / P);
}

/* ------------------------------------------------------- P:271-273, R6 */
void orc_permutation(int64_t n, const int32_t *labels, int32_t *new_to_old,
                     int32_t *old_to_new) {
    int32_t maxl = -1;
    for (int64_t i = 0; i < n; i++)
        if (labels[i] > maxl) maxl = labels[i];
    int64_t nl = (int64_t)maxl + 1;
    int64_t *start = (int64_t *)calloc((size_t)(nl + 1), sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) start[labels[i] + 1]++;
    for (int64_t l = 0; l < nl; l++) start[l + 1] += start[l];
    /* stable: scan old rows ascending, append to their label's bucket */
    for (int64_t i = 0; i < n; i++) {
        int64_t pos = start[labels[i]]++;
        new_to_old[pos] = (int32_t)i;
    }
    for (int64_t j = 0; j < n; j++) old_to_new[new_to_old[j]] = (int32_t)j;
    free(start);
}

void orc_subdomain_ptr(int64_t n, const int32_t *labels, int32_t n_sub, int64_t *sub_ptr) {
    for (int32_t s = 0; s <= n_sub; s++) sub_ptr[s] = 0;
    for (int64_t i = 0; i < n; i++) sub_ptr[labels[i] + 1]++;
    for (int32_t s = 0; s < n_sub; s++) sub_ptr[s + 1] += sub_ptr[s];
}

/* ---------------------------------------------------------------- Alg. 3 */
void orc_reorder(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                 const int32_t *new_to_old, const int32_t *old_to_new, int64_t *rp_out,
                 int32_t *ci_out, double *v_out) {
    rp_out[0] = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t k = new_to_old[i];
        rp_out[i + 1] = rp[k + 1] - rp[k];
    }
    for (int64_t i = 0; i < n; i++) rp_out[i + 1] += rp_out[i];
    int64_t nn = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t m = new_to_old[i];
        for (int64_t j = rp[m]; j < rp[m + 1]; j++) {
            ci_out[nn] = old_to_new[ci[j]];
            memcpy(v_out + 9 * nn, v + 9 * j, 9 * sizeof(double));
            nn++;
        }
        /* "Sort colidx[rowptr[i] .. rowptr[i+1]]", blocks move with
         * their columns: plain insertion sort. */
        for (int64_t a = rp_out[i] + 1; a < rp_out[i + 1]; a++) {
            int32_t c = ci_out[a];
            double blk[9];
            memcpy(blk, v_out + 9 * a, sizeof blk);
            int64_t b = a - 1;
            while (b >= rp_out[i] && ci_out[b] > c) {
                ci_out[b + 1] = ci_out[b];
                memcpy(v_out + 9 * (b + 1), v_out + 9 * b, sizeof blk);
                b--;
            }
            ci_out[b + 1] = c;
            memcpy(v_out + 9 * (b + 1), blk, sizeof blk);
        }
    }
}

/* ------------------------------------------------------------ P:319-323 */
int64_t orc_drop(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                 const int32_t *label_new, int64_t *rp_out, int32_t *ci_out, double *v_out) {
    int64_t kept = 0;
    if (rp_out) rp_out[0] = 0;
    for (int64_t r = 0; r < n; r++) {
        for (int64_t p = rp[r]; p < rp[r + 1]; p++) {
            if (label_new[r] == label_new[ci[p]]) {
                if (rp_out) {
                    ci_out[kept] = ci[p];
                    memcpy(v_out + 9 * kept, v + 9 * p, 9 * sizeof(double));
                }
                kept++;
            }
        }
        if (rp_out) rp_out[r + 1] = kept;
    }
    return kept;
}

/* -------------------------------------------------------- 3x3 block algebra
 * DESIGN.md section 4 (arithmetic order). Blocks row-major: B[r][c] = B[3r+c]. */

/* C = A * B:  C_rc = fma(a_r2, b_2c, fma(a_r1, b_1c, a_r0 * b_0c)) */
static void mul3(const double *A, const double *B, double *C) {
    double t[9];
    for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++)
            t[3 * r + c] = fma(A[3 * r + 2], B[6 + c], fma(A[3 * r + 1], B[3 + c], A[3 * r] * B[c]));
    memcpy(C, t, sizeof t);
}

/* W -= L * U:  W_rc = fma(-l_r0, u_0c, W_rc); then l_r1/u_1c; then l_r2/u_2c */
static void elim3(double *W, const double *L, const double *U) {
    for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++) {
            double w = W[3 * r + c];
            w = fma(-L[3 * r + 0], U[0 + c], w);
            w = fma(-L[3 * r + 1], U[3 + c], w);
            w = fma(-L[3 * r + 2], U[6 + c], w);
            W[3 * r + c] = w;
        }
}

/* inverse by adjugate / determinant (R15). Returns 0 or -1 if |det| < floor. */
static int inv3(const double *a, double floor_, double *inv) {
    double a00 = a[0], a01 = a[1], a02 = a[2];
    double a10 = a[3], a11 = a[4], a12 = a[5];
    double a20 = a[6], a21 = a[7], a22 = a[8];
    double C00 = fma(a11, a22, -(a12 * a21));
    double C01 = fma(a12, a20, -(a10 * a22));
    double C02 = fma(a10, a21, -(a11 * a20));
    double C10 = fma(a02, a21, -(a01 * a22));
    double C11 = fma(a00, a22, -(a02 * a20));
    double C12 = fma(a01, a20, -(a00 * a21));
    double C20 = fma(a01, a12, -(a02 * a11));
    double C21 = fma(a02, a10, -(a00 * a12));
    double C22 = fma(a00, a11, -(a01 * a10));
    double det = fma(a00, C00, fma(a01, C01, a02 * C02));
    if (!(fabs(det) >= floor_)) return -1;
    double rdet = 1.0 / det;
    /* inv[r][c] = C_cr * rdet (adjugate = transposed cofactors) */
    inv[0] = C00 * rdet; inv[1] = C10 * rdet; inv[2] = C20 * rdet;
    inv[3] = C01 * rdet; inv[4] = C11 * rdet; inv[5] = C21 * rdet;
    inv[6] = C02 * rdet; inv[7] = C12 * rdet; inv[8] = C22 * rdet;
    return 0;
}

/* ---------------------------------------------------------------- Alg. 7 */
int orc_ilu0(int64_t n, const int64_t *rp, const int32_t *ci, const double *a,
             double pivot_floor, double *lu, double *dinv, int64_t *bad_row) {
    memcpy(lu, a, (size_t)(9 * rp[n]) * sizeof(double));
    for (int64_t i = 0; i < n; i++) {
        int64_t pd = -1;
        for (int64_t p = rp[i]; p < rp[i + 1]; p++)
            if (ci[p] == i) pd = p;
        if (pd < 0) {
            if (bad_row) *bad_row = i;
            return 1;
        }
        /* for k in pattern(i), k < i, ascending */
        for (int64_t p = rp[i]; p < rp[i + 1] && ci[p] < i; p++) {
            int64_t k = ci[p];
            /* L_ik = W_ik * U_kk^-1  (right multiplication, R12) */
            mul3(lu + 9 * p, dinv + 9 * k, lu + 9 * p);
            /* for j in pattern(i), j > k, with (k,j) in pattern(U row k) */
            for (int64_t q = p + 1; q < rp[i + 1]; q++) {
                int64_t j = ci[q];
                for (int64_t r = rp[k]; r < rp[k + 1]; r++) {
                    if (ci[r] == j && j > k) {
                        elim3(lu + 9 * q, lu + 9 * p, lu + 9 * r);
                        break;
                    }
                }
            }
        }
        if (inv3(lu + 9 * pd, pivot_floor, dinv + 9 * i) != 0) {
            if (bad_row) *bad_row = i;
            return 2;
        }
    }
    return 0;
}

void orc_ildu0(int64_t n, const int64_t *rp, const int32_t *ci, const double *lu,
               const double *dinv, double *uunit) {
    for (int64_t i = 0; i < n; i++)
        for (int64_t p = rp[i]; p < rp[i + 1]; p++)
            if (ci[p] > i) mul3(dinv + 9 * i, lu + 9 * p, uunit + 9 * p);
}

/* ---------------------------------------------------------------- Alg. 5 */
void orc_levels_lower(int64_t n, const int64_t *rp, const int32_t *ci, int32_t *hmap) {
    for (int64_t i = 0; i < n; i++) {
        int32_t h = 0;
        for (int64_t p = rp[i]; p < rp[i + 1]; p++)
            if (ci[p] < i && hmap[ci[p]] + 1 > h) h = hmap[ci[p]] + 1;
        hmap[i] = h;
    }
}

void orc_levels_upper(int64_t n, const int64_t *rp, const int32_t *ci, int32_t *hmap) {
    for (int64_t i = n - 1; i >= 0; i--) {
        int32_t h = 0;
        for (int64_t p = rp[i]; p < rp[i + 1]; p++)
            if (ci[p] > i && hmap[ci[p]] + 1 > h) h = hmap[ci[p]] + 1;
        hmap[i] = h;
    }
}

/* ------------------------------------------------ fused ILDU0 apply (4.4) */
void orc_apply(int64_t n, int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp,
               const int32_t *ci, const double *lu, const double *dinv, const double *uunit,
               const double *r, double *z) {
    (void)n;
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t s = 0; s < n_sub; s++) {
        int64_t a = sub_ptr[s], e = sub_ptr[s + 1];
        /* forward unit-lower sweep, rows ascending (Alg. 6 with L_ii = I) */
        for (int64_t i = a; i < e; i++) {
            for (int c = 0; c < 3; c++) {
                double acc = r[3 * i + c];
                for (int64_t p = rp[i]; p < rp[i + 1] && ci[p] < i; p++) {
                    const double *B = lu + 9 * p;
                    const double *zj = z + 3 * (int64_t)ci[p];
                    for (int d = 0; d < 3; d++) acc = fma(-B[3 * c + d], zj[d], acc);
                }
                z[3 * i + c] = acc;
            }
        }
        /* y_i = Dinv_i z_i, then backward unit-upper sweep, rows descending */
        for (int64_t i = e - 1; i >= a; i--) {
            const double *D = dinv + 9 * i;
            double y[3];
            for (int c = 0; c < 3; c++) {
                double t = D[3 * c + 0] * z[3 * i + 0];
                t = fma(D[3 * c + 1], z[3 * i + 1], t);
                t = fma(D[3 * c + 2], z[3 * i + 2], t);
                y[c] = t;
            }
            for (int c = 0; c < 3; c++) {
                double acc = y[c];
                for (int64_t p = rp[i]; p < rp[i + 1]; p++) {
                    if (ci[p] <= i) continue;
                    const double *B = uunit + 9 * p;
                    const double *xj = z + 3 * (int64_t)ci[p];
                    for (int d = 0; d < 3; d++) acc = fma(-B[3 * c + d], xj[d], acc);
                }
                z[3 * i + c] = acc;
            }
        }
    }
}

/* Lower solve alone (Table 3 analogue): z = L^-1 r per subdomain,
 * unit L (sec. 4.3), the forward sweep of orc_apply written out again. */
void orc_lower(int64_t n, int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp, const int32_t *ci,
               const double *lu, const double *r, double *z) {
    (void)n;
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t s = 0; s < n_sub; s++) {
        for (int64_t i = sub_ptr[s]; i < sub_ptr[s + 1]; i++) {
            for (int c = 0; c < 3; c++) {
                double acc = r[3 * i + c];
                for (int64_t p = rp[i]; p < rp[i + 1] && ci[p] < i; p++) {
                    const double *B = lu + 9 * p;
                    const double *zj = z + 3 * (int64_t)ci[p];
                    for (int d = 0; d < 3; d++) acc = fma(-B[3 * c + d], zj[d], acc);
                }
                z[3 * i + c] = acc;
            }
        }
    }
}

/* ILU0 apply with the NON-unit upper factor ("unlike ILU0
 * where scaling follows each row's off-diagonal updates"): forward unit-lower
 * sweep as in orc_apply; backward sweep rows descending with U = the ILU0
 * upper blocks themselves (lu, j > i, not scaled by Dinv_i):
 *   acc_c = z_ic; for U blocks ascending, for d: acc_c = fma(-U[c][d], x_jd, acc_c);
 *   x_ic = D[c][0] acc_0; x_ic = fma(D[c][1], acc_1, x_ic); x_ic = fma(D[c][2], acc_2, x_ic)
 * with D = Dinv_i = U_ii^-1. Mathematically equal to orc_apply (U = D^-1 U_unit). */
void orc_apply_ilu0(int64_t n, int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp, const int32_t *ci,
                    const double *lu, const double *dinv, const double *r, double *z) {
    orc_lower(n, n_sub, sub_ptr, rp, ci, lu, r, z);
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t s = 0; s < n_sub; s++) {
        for (int64_t i = sub_ptr[s + 1] - 1; i >= sub_ptr[s]; i--) {
            double acc[3];
            for (int c = 0; c < 3; c++) {
                acc[c] = z[3 * i + c];
                for (int64_t p = rp[i]; p < rp[i + 1]; p++) {
                    if (ci[p] <= i) continue;
                    const double *B = lu + 9 * p;
                    const double *xj = z + 3 * (int64_t)ci[p];
                    for (int d = 0; d < 3; d++) acc[c] = fma(-B[3 * c + d], xj[d], acc[c]);
                }
            }
            const double *D = dinv + 9 * i;
            for (int c = 0; c < 3; c++) {
                double t = D[3 * c + 0] * acc[0];
                t = fma(D[3 * c + 1], acc[1], t);
                t = fma(D[3 * c + 2], acc[2], t);
                z[3 * i + c] = t;
            }
        }
    }
}

/* ------------------------------------------------------------------ SpMV */
void orc_spmv(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
              const double *x, double *y) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        for (int c = 0; c < 3; c++) {
            double acc = 0.0;
            for (int64_t p = rp[i]; p < rp[i + 1]; p++) {
                const double *B = v + 9 * p;
                const double *xj = x + 3 * (int64_t)ci[p];
                for (int d = 0; d < 3; d++) acc = fma(B[3 * c + d], xj[d], acc);
            }
            y[3 * i + c] = acc;
        }
    }
}

/* ------------------------------------------------------ Dot2 (dd) product */
double orc_dot(int64_t m, const double *x, const double *y) {
    double s = 0.0, cc = 0.0;
    for (int64_t i = 0; i < m; i++) {
        double p = x[i] * y[i];
        double q = fma(x[i], y[i], -p);          /* TwoProd */
        double t = s + p;                         /* TwoSum(s, p) */
        double bb = t - s;
        double r = (s - (t - bb)) + (p - bb);
        s = t;
        cc = cc + (q + r);
    }
    return s + cc;
}

/* ------------------------------------------------------------ BiCGSTAB */
typedef void (*spmv_fn)(int64_t, const int64_t *, const int32_t *, const double *, const double *, double *);
typedef void (*apply_fn)(int64_t, int32_t, const int64_t *, const int64_t *, const int32_t *, const double *,
                         const double *, const double *, const double *, double *);

/* Alg. 1 with K1 = I, K2 = M; bs = unknowns per row (3: BSR3, 1: CSR). */
static int bicgstab_impl(int64_t n, int bs, spmv_fn orc_spmv_, apply_fn orc_apply_, const int64_t *rp_r,
                         const int32_t *ci_r, const double *v_r, int32_t n_sub, const int64_t *sub_ptr,
                         const int64_t *rp_d, const int32_t *ci_d, const double *lu, const double *dinv,
                         const double *uunit, const double *b, double *x, double tol, int32_t max_iter,
                         double *resid_hist, double *out);

int orc_bicgstab(int64_t n, const int64_t *rp_r, const int32_t *ci_r, const double *v_r,
                 int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp_d, const int32_t *ci_d,
                 const double *lu, const double *dinv, const double *uunit, const double *b,
                 double *x, double tol, int32_t max_iter, double *resid_hist, double *out) {
    return bicgstab_impl(n, 3, orc_spmv, orc_apply, rp_r, ci_r, v_r, n_sub, sub_ptr, rp_d, ci_d, lu, dinv, uunit,
                         b, x, tol, max_iter, resid_hist, out);
}

static int bicgstab_impl(int64_t n, int bs, spmv_fn orc_spmv_, apply_fn orc_apply_, const int64_t *rp_r,
                         const int32_t *ci_r, const double *v_r, int32_t n_sub, const int64_t *sub_ptr,
                         const int64_t *rp_d, const int32_t *ci_d, const double *lu, const double *dinv,
                         const double *uunit, const double *b, double *x, double tol, int32_t max_iter,
                         double *resid_hist, double *out) {
    int64_t m = bs * n;
    size_t bytes = (size_t)m * sizeof(double);
    double *r = malloc(bytes), *rh = malloc(bytes), *p = calloc((size_t)m, sizeof(double));
    double *v = calloc((size_t)m, sizeof(double)), *ph = malloc(bytes), *s = malloc(bytes);
    double *sh = malloc(bytes), *t = malloc(bytes);
    int status = 2, nh = 0, n_app = 0;
    double iters = (double)max_iter;

    /* r = b - A x0 */
    orc_spmv_(n, rp_r, ci_r, v_r, x, t);
#pragma omp parallel for
    for (int64_t i = 0; i < m; i++) r[i] = b[i] - t[i];
    memcpy(rh, r, bytes);
    double n0 = sqrt(orc_dot(m, r, r));
    if (resid_hist) resid_hist[nh] = n0;
    nh++;
    double rel = 1.0;
    if (n0 == 0.0) {
        status = 0;
        iters = 0.0;
        rel = 0.0;
        goto done;
    }
    double thr = tol * n0;
    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    for (int32_t k = 1; k <= max_iter; k++) {
        double rho = orc_dot(m, rh, r);
        if (fabs(rho) < 1e-30) { status = 1; iters = k - 1; break; }
        if (k == 1) {
            memcpy(p, r, bytes);
        } else {
            double beta = (rho / rho_prev) * (alpha / omega);
#pragma omp parallel for
            for (int64_t i = 0; i < m; i++) p[i] = fma(beta, fma(-omega, v[i], p[i]), r[i]);
        }
        orc_apply_(n, n_sub, sub_ptr, rp_d, ci_d, lu, dinv, uunit, p, ph);
        n_app++;
        orc_spmv_(n, rp_r, ci_r, v_r, ph, v);
        double sigma = orc_dot(m, rh, v);
        if (fabs(sigma) < 1e-30) { status = 1; iters = k - 1; break; }
        alpha = rho / sigma;
#pragma omp parallel for
        for (int64_t i = 0; i < m; i++) s[i] = fma(-alpha, v[i], r[i]);
        double ns = sqrt(orc_dot(m, s, s));
        if (resid_hist) resid_hist[nh] = ns;
        nh++;
        if (ns < thr) {
#pragma omp parallel for
            for (int64_t i = 0; i < m; i++) x[i] = fma(alpha, ph[i], x[i]);
            status = 0;
            iters = k - 0.5;
            rel = ns / n0;
            break;
        }
        orc_apply_(n, n_sub, sub_ptr, rp_d, ci_d, lu, dinv, uunit, s, sh);
        n_app++;
        orc_spmv_(n, rp_r, ci_r, v_r, sh, t);
        double tau = orc_dot(m, t, t);
        if (tau < 1e-30) { status = 1; iters = k - 0.5; break; }
        omega = orc_dot(m, t, s) / tau;
#pragma omp parallel for
        for (int64_t i = 0; i < m; i++) {
            x[i] = fma(omega, sh[i], fma(alpha, ph[i], x[i]));
            r[i] = fma(-omega, t[i], s[i]);
        }
        double nr = sqrt(orc_dot(m, r, r));
        if (resid_hist) resid_hist[nh] = nr;
        nh++;
        rel = nr / n0;
        if (nr < thr) {
            status = 0;
            iters = k;
            break;
        }
        rho_prev = rho;
    }
done:;
    /* true residual ||b - A x|| / ||b|| */
    orc_spmv_(n, rp_r, ci_r, v_r, x, t);
#pragma omp parallel for
    for (int64_t i = 0; i < m; i++) t[i] = b[i] - t[i];
    double nb = sqrt(orc_dot(m, b, b));
    double tr = nb > 0 ? sqrt(orc_dot(m, t, t)) / nb : 0.0;
    if (out) {
        out[0] = iters;
        out[1] = n_app;
        out[2] = rel;
        out[3] = tr;
        out[4] = status;
        out[5] = nh;
        out[6] = 0;
        out[7] = 0;
    }
    free(r); free(rh); free(p); free(v); free(ph); free(s); free(sh); free(t);
    return status;
}

/* ======================================================================
 * Scalar CSR path (the paper's CSR half: P:110, P:279-305,
 * Alg. 7 P:680-711 in its scalar form). Same steps and arithmetic order as
 * the block functions above with 1x1 blocks: L_ik = w_ik * dinv_k,
 * w_ij = fma(-l_ik, u_kj, w_ij), dinv_i = 1 / u_ii (R15 floor on |u_ii|),
 * uunit_ij = dinv_i * u_ij. The pattern-only steps (labels, permutation,
 * subdomain_ptr, levels) are shared with the block path.
 * ==================================================================== */

void orc_s_reorder(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                   const int32_t *new_to_old, const int32_t *old_to_new, int64_t *rp_out,
                   int32_t *ci_out, double *v_out) {
    rp_out[0] = 0;
    for (int64_t i = 0; i < n; i++) rp_out[i + 1] = rp_out[i] + (rp[new_to_old[i] + 1] - rp[new_to_old[i]]);
    int64_t nn = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t m = new_to_old[i];
        for (int64_t j = rp[m]; j < rp[m + 1]; j++) {
            ci_out[nn] = old_to_new[ci[j]];
            v_out[nn] = v[j];
            nn++;
        }
        /* "Sort colidx[rowptr[i] .. rowptr[i+1]]": insertion sort */
        for (int64_t a = rp_out[i] + 1; a < rp_out[i + 1]; a++) {
            int32_t c = ci_out[a];
            double x = v_out[a];
            int64_t b = a - 1;
            while (b >= rp_out[i] && ci_out[b] > c) {
                ci_out[b + 1] = ci_out[b];
                v_out[b + 1] = v_out[b];
                b--;
            }
            ci_out[b + 1] = c;
            v_out[b + 1] = x;
        }
    }
}

int64_t orc_s_drop(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                   const int32_t *label_new, int64_t *rp_out, int32_t *ci_out, double *v_out) {
    int64_t kept = 0;
    if (rp_out) rp_out[0] = 0;
    for (int64_t r = 0; r < n; r++) {
        for (int64_t p = rp[r]; p < rp[r + 1]; p++) {
            if (label_new[r] == label_new[ci[p]]) {
                if (rp_out) {
                    ci_out[kept] = ci[p];
                    v_out[kept] = v[p];
                }
                kept++;
            }
        }
        if (rp_out) rp_out[r + 1] = kept;
    }
    return kept;
}

int orc_s_ilu0(int64_t n, const int64_t *rp, const int32_t *ci, const double *a,
               double pivot_floor, double *lu, double *dinv, int64_t *bad_row) {
    memcpy(lu, a, (size_t)rp[n] * sizeof(double));
    for (int64_t i = 0; i < n; i++) {
        int64_t pd = -1;
        for (int64_t p = rp[i]; p < rp[i + 1]; p++)
            if (ci[p] == i) pd = p;
        if (pd < 0) {
            if (bad_row) *bad_row = i;
            return 1;
        }
        for (int64_t p = rp[i]; p < rp[i + 1] && ci[p] < i; p++) {
            int64_t k = ci[p];
            lu[p] = lu[p] * dinv[k];                       /* l_ik = w_ik / u_kk */
            for (int64_t q = p + 1; q < rp[i + 1]; q++) {
                int64_t j = ci[q];
                for (int64_t r = rp[k]; r < rp[k + 1]; r++) {
                    if (ci[r] == j && j > k) {
                        lu[q] = fma(-lu[p], lu[r], lu[q]);  /* w_ij -= l_ik u_kj */
                        break;
                    }
                }
            }
        }
        if (!(fabs(lu[pd]) >= pivot_floor)) {
            if (bad_row) *bad_row = i;
            return 2;
        }
        dinv[i] = 1.0 / lu[pd];
    }
    return 0;
}

void orc_s_ildu0(int64_t n, const int64_t *rp, const int32_t *ci, const double *lu,
                 const double *dinv, double *uunit) {
    for (int64_t i = 0; i < n; i++)
        for (int64_t p = rp[i]; p < rp[i + 1]; p++)
            if (ci[p] > i) uunit[p] = dinv[i] * lu[p];
}

void orc_s_apply(int64_t n, int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp,
                 const int32_t *ci, const double *lu, const double *dinv, const double *uunit,
                 const double *r, double *z) {
    (void)n;
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t s = 0; s < n_sub; s++) {
        int64_t a = sub_ptr[s], e = sub_ptr[s + 1];
        for (int64_t i = a; i < e; i++) {
            double acc = r[i];
            for (int64_t p = rp[i]; p < rp[i + 1] && ci[p] < i; p++) acc = fma(-lu[p], z[ci[p]], acc);
            z[i] = acc;
        }
        for (int64_t i = e - 1; i >= a; i--) {
            double acc = dinv[i] * z[i];
            for (int64_t p = rp[i]; p < rp[i + 1]; p++)
                if (ci[p] > i) acc = fma(-uunit[p], z[ci[p]], acc);
            z[i] = acc;
        }
    }
}

void orc_s_spmv(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                const double *x, double *y) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double acc = 0.0;
        for (int64_t p = rp[i]; p < rp[i + 1]; p++) acc = fma(v[p], x[ci[p]], acc);
        y[i] = acc;
    }
}

int orc_s_bicgstab(int64_t n, const int64_t *rp_r, const int32_t *ci_r, const double *v_r,
                   int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp_d, const int32_t *ci_d,
                   const double *lu, const double *dinv, const double *uunit, const double *b,
                   double *x, double tol, int32_t max_iter, double *resid_hist, double *out) {
    return bicgstab_impl(n, 1, orc_s_spmv, orc_s_apply, rp_r, ci_r, v_r, n_sub, sub_ptr, rp_d, ci_d, lu, dinv,
                         uunit, b, x, tol, max_iter, resid_hist, out);
}
