// krylov.cuh -- declarations shared by krylov.cu and api.cpp (product-internal).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

struct dd_ctx;

namespace ddk {

// device scalar slots (double sc[S_COUNT])
enum : int {
    S_RHO = 0,
    S_RHO_PREV,
    S_ALPHA,
    S_OMEGA,
    S_SIGMA,
    S_TS,
    S_TT,
    S_SS,
    S_RR,
    S_N0SQ,
    S_RES_TT,
    S_RES_BB,
    S_TOL,   // host-written before a solve
    S_THR,   // tol * ||r0||
    S_COUNT = 16
};

enum : int { FIN_INIT = 1, FIN_ALPHA, FIN_SS, FIN_OMEGA, FIN_RHO, FIN_RESID,
             FIN_SS_OMEGA  // world > 1: (t.s, t.t, s.s) in one collective; FIN_SS first, then FIN_OMEGA
};

// Device-side solver control (int ctl[8]): the finalizing last blocks decide
// convergence / breakdown (R21, R25) and every iteration kernel returns at
// entry unless ctl[C_STATE] == ST_RUN, so the host can enqueue iterations
// ahead without synchronising at each half step.
enum : int { C_STATE = 0, C_K = 1, C_NH = 2, C_CNT = 3, C_ITER = 4, C_MAX = 5 };
enum : int {
    ST_RUN = 0,
    ST_HALF = 1,       // ||s|| < tol ||r0||: x += alpha p_hat pending
    ST_DONE_HALF = 2,  // converged at a half step
    ST_DONE_FULL = 3,  // converged at a full step
    ST_ZERO = 4,       // ||r0|| == 0
    ST_BRK_RHO = 5,
    ST_BRK_SIGMA = 6,
    ST_BRK_TAU = 7,
    ST_COMM = 8        // a peer-transport wait timed out (DD_E_NCCL)
};
enum : int { SPMV_PLAIN = 0, SPMV_SIGMA = 1, SPMV_TS_TT = 2 };

struct DD;

struct RedArgs {
    DD *partials;           // [grid * 2]
    unsigned int *counter;  // zero-initialised, reset by the last block
    double *sc;             // device scalars
    double *loc;            // rank-local results (world > 1)
    int finalize;           // 1: last block finalizes (world == 1)
    int *ctl;               // solver control (nullptr: no control, e.g. plain SpMV)
    double *hist;           // residual history [2*max_iter+1] (device)
    int k;                  // iteration the launch belongs to (< 0: ctl[C_ITER], graph mode)
    int slot;               // world > 1: first (s, c) pair of loc[] this reduction writes
};

// CUDA-graph BiCGSTAB (f4): the iteration body runs under a conditional WHILE
// node; the head kernel advances ctl[C_ITER], the tail kernel sets the loop
// condition from the device-side control state.
void launch_iter_head(int *ctl, cudaStream_t st);
void launch_iter_tail(int *ctl, cudaGraphConditionalHandle h, cudaStream_t st);

void launch_spmv(int mode, const dd_ctx *ctx, const double *x, const double *xg, double *y, const double *aux,
                 const RedArgs &ra, cudaStream_t st);
void launch_init_r(const dd_ctx *ctx, int64_t m, const double *b, const double *t, double *r, double *rh,
                   const RedArgs &ra, cudaStream_t st);
void launch_update_p(const dd_ctx *ctx, int64_t m, int first, const double *r, const double *v, double *p,
                     const double *sc, const int *ctl, cudaStream_t st);
void launch_update_s(const dd_ctx *ctx, int64_t m, const double *r, const double *v, double *s, const RedArgs &ra,
                     cudaStream_t st);
void launch_update_x_half(const dd_ctx *ctx, int64_t m, const double *ph, double *x, const double *sc, int *ctl,
                          cudaStream_t st);
void launch_update_xr(const dd_ctx *ctx, int64_t m, const double *ph, const double *sh, const double *s,
                      const double *t, const double *rh, double *x, double *r, const RedArgs &ra, cudaStream_t st);
void launch_resid(const dd_ctx *ctx, int64_t m, const double *b, double *t, const RedArgs &ra, cudaStream_t st);
void launch_finalize_gathered(int world, int nv, const double *gathered, const RedArgs &ra, int op, cudaStream_t st);
void launch_gather3(const dd_ctx *ctx, int64_t n, const int32_t *idx, const double *in, double *out, cudaStream_t st);
void launch_scatter3(const dd_ctx *ctx, int64_t n, const int32_t *idx, const double *in, double *out,
                     cudaStream_t st);
size_t partials_bytes(const dd_ctx *ctx);
// sliced-ELL SpMV operand from the rank's reordered rows (dd_setup): slot
// (k, lane) of slice s = block k of row 32 s + lane (column -1 and zero
// values past a row's end), values as bs*bs planes of 32 per k
void launch_build_ell(int bs, int64_t n_slices, int64_t n_rows, const int64_t *slot_ptr, const int64_t *rp,
                      const int32_t *ci, const double *av, int32_t *cols, double *vals, cudaStream_t st);

}  // namespace ddk
