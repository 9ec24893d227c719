/*
 * dd_oracle.h -- CPU ORACLE for arXiv 2508.04917 (fine-grained domain
 * decomposition + per-subdomain ILU0/ILDU0 apply + BiCGSTAB).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the product library
 * (paper_2508_04917_b200/csrc, include/dd.h); neither includes the other.
 *
 * Plain, slow, obviously-correct fp64 C. Every floating-point step follows
 * DESIGN.md "Arithmetic order" (explicit fma(), compiled -ffp-contract=off)
 * so that results are bitwise reproducible and comparable.
 *
 * Citations: P:a-b = /root/reference/PAPER.md lines a-b (section/algorithm
 * named alongside). Readings Rn are listed in DESIGN.md section 3.
 *
 * Conventions: BSR3 = (row_ptr int64[n+1], col_idx int32[nnzb],
 * vals double[9*nnzb]); 3x3 blocks row-major; columns ascending per row.
 * Vectors are double[3n], component c of block row i at index 3i+c.
 *
 * Parity pins: every function below is pinned by tests/test_oracle_*.py
 * (closed forms, paper values, library routines, brute force). None is
 * "parity unpinned".
 */
#ifndef DD_ORACLE_H
#define DD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Number of OpenMP threads used by the parallel-over-subdomain/row loops
 * (apply, spmv, elementwise). 0 = runtime default. Results do not depend on
 * it (each output element is computed by one thread in a fixed order). */
void orc_set_threads(int n);
int orc_get_threads(void);

/* Alg. 2: geometric cuts. Tile dims (tx,ty,tz) = nblk_*.
 * part_id[i + nx*(j + ny*k)] = i/tx + bx*(j/ty + by*(k/tz)).
 * Returns 0, or -1 if a grid dim is not divisible by its tile dim (R26). */
int orc_labels_geometric(int32_t nx, int32_t ny, int32_t nz, int32_t tx, int32_t ty,
                         int32_t tz, int32_t *part_id);
/* Graph-growing partition (METIS stand-in, P:236 / P:1041 "manually
 * balancing"; R35): parts of exactly P rows (last smaller), each
 * grown breadth-first from the lowest-index unassigned row, neighbours visited
 * in ascending column order, part closed as soon as it holds P rows. */
void orc_labels_bfs(int64_t n, const int64_t *rp, const int32_t *ci, int32_t P, int32_t *part_id);
/* Contiguous chunks of P rows (R26: last chunk may be smaller). */
void orc_labels_chunks(int64_t n, int32_t P, int32_t *part_id);

/* P:271-273 + R6/R7: stable grouping of rows by label.
 * new_to_old = Alg. 3's pmap, old_to_new = inv_pmap. */
void orc_permutation(int64_t n, const int32_t *labels, int32_t *new_to_old,
                     int32_t *old_to_new);

/* Subdomain row ranges in reordered space: sub_ptr[s]..sub_ptr[s+1] are the
 * rows with label s. n_sub = max label + 1. sub_ptr has n_sub+1 entries. */
void orc_subdomain_ptr(int64_t n, const int32_t *labels, int32_t n_sub, int64_t *sub_ptr);

/* Alg. 3 at block granularity; columns sorted ascending (R8). */
void orc_reorder(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                 const int32_t *new_to_old, const int32_t *old_to_new, int64_t *rp_out,
                 int32_t *ci_out, double *v_out);

/* P:319-323 (R9): keep block (r,c) iff label(r) == label(c) (labels in the
 * reordered numbering). Returns kept nnzb. If rp_out == NULL only counts. */
int64_t orc_drop(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                 const int32_t *label_new, int64_t *rp_out, int32_t *ci_out, double *v_out);

/* Alg. 7 ILU0, block form (R11-R13, R15): IKJ elimination on
 * pattern(A). Output lu[] in A's pattern: col<row -> L_ij (unit L implied),
 * col>=row -> U_ij. dinv[9i..] = inv(U_ii).
 * Returns 0 ok, 1 missing diagonal block, 2 |det U_ii| < pivot_floor;
 * *bad_row = offending row. */
int orc_ilu0(int64_t n, const int64_t *rp, const int32_t *ci, const double *a,
             double pivot_floor, double *lu, double *dinv, int64_t *bad_row);

/* Alg. 7 ILDU0 post-processing (R14): uunit_ij = dinv_i * U_ij for
 * j > i, written at the same pattern positions of uunit[] (other positions
 * untouched). */
void orc_ildu0(int64_t n, const int64_t *rp, const int32_t *ci, const double *lu,
               const double *dinv, double *uunit);

/* Alg. 5 semantics (R16): longest-path levels. */
void orc_levels_lower(int64_t n, const int64_t *rp, const int32_t *ci, int32_t *hmap);
void orc_levels_upper(int64_t n, const int64_t *rp, const int32_t *ci, int32_t *hmap);

/* Fused ILDU0 apply z = U_unit^-1 D^-1 L^-1 r per subdomain (Alg. 6
 * unit-diagonal form, sec. 4.3, sec. 4.4).
 * L blocks are lu[] at col<row, U_unit blocks are uunit[] at col>row, in the
 * dropped pattern (rp, ci). Rows ascending (lower), then descending (D+U). */
void orc_apply(int64_t n, int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp,
               const int32_t *ci, const double *lu, const double *dinv, const double *uunit,
               const double *r, double *z);
/* Table 3 analogue: the forward unit-lower sweep alone, z = L^-1 r. */
void orc_lower(int64_t n, int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp, const int32_t *ci,
               const double *lu, const double *r, double *z);
/* ILU0 with the non-unit U (scaling after each row's updates). */
void orc_apply_ilu0(int64_t n, int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp, const int32_t *ci,
                    const double *lu, const double *dinv, const double *r, double *z);

/* Block SpMV y = A x (the bsrxmv of P:185; Alg. 1's A-products). */
void orc_spmv(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
              const double *x, double *y);

/* Double-double (Dot2) dot product, ascending index order. */
double orc_dot(int64_t m, const double *x, const double *y);

/* Right-preconditioned BiCGSTAB (Alg. 1 P:135-165 with K1 = I, K2 = LDU; R20,
 * R21, R22, R25). A_r = (rp_r, ci_r, v_r); M from (rp_d, ci_d, lu, dinv,
 * uunit, sub_ptr). x in: x0, out: solution. resid_hist (nullable) gets
 * [||r0||, ||s_1||, ||r_1||, ...] (2*max_iter+1 max). out[8] =
 * {iterations (0.5 steps), n_applies, rel_resid, true_rel_resid, status,
 *  n_hist, 0, 0}. status: 0 converged, 1 breakdown, 2 max_iter. */
int orc_bicgstab(int64_t n, const int64_t *rp_r, const int32_t *ci_r, const double *v_r,
                 int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp_d, const int32_t *ci_d,
                 const double *lu, const double *dinv, const double *uunit, const double *b,
                 double *x, double tol, int32_t max_iter, double *resid_hist, double *out);

/* ---- Scalar CSR path (the paper's CSR half): the
 * same steps with 1x1 blocks -- vals double[nnz], vectors double[n]. The
 * pattern-only functions above (labels, permutation, subdomain_ptr, levels)
 * serve both paths. Arithmetic: DESIGN.md section 4 with 1x1 blocks
 * (l_ik = w_ik * dinv_k; w_ij = fma(-l_ik, u_kj, w_ij); dinv_i = 1/u_ii;
 * uunit_ij = dinv_i * u_ij; sweeps and SpMV as single FMA chains). */
void orc_s_reorder(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                   const int32_t *new_to_old, const int32_t *old_to_new, int64_t *rp_out,
                   int32_t *ci_out, double *v_out);
int64_t orc_s_drop(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                   const int32_t *label_new, int64_t *rp_out, int32_t *ci_out, double *v_out);
int orc_s_ilu0(int64_t n, const int64_t *rp, const int32_t *ci, const double *a,
               double pivot_floor, double *lu, double *dinv, int64_t *bad_row);
void orc_s_ildu0(int64_t n, const int64_t *rp, const int32_t *ci, const double *lu,
                 const double *dinv, double *uunit);
void orc_s_apply(int64_t n, int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp,
                 const int32_t *ci, const double *lu, const double *dinv, const double *uunit,
                 const double *r, double *z);
void orc_s_spmv(int64_t n, const int64_t *rp, const int32_t *ci, const double *v,
                const double *x, double *y);
int orc_s_bicgstab(int64_t n, const int64_t *rp_r, const int32_t *ci_r, const double *v_r,
                   int32_t n_sub, const int64_t *sub_ptr, const int64_t *rp_d, const int32_t *ci_d,
                   const double *lu, const double *dinv, const double *uunit, const double *b,
                   double *x, double tol, int32_t max_iter, double *resid_hist, double *out);

#ifdef __cplusplus
}
#endif
#endif
