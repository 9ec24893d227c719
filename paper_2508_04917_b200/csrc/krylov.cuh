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
    S_COUNT = 16
};

enum : int { FIN_INIT = 1, FIN_ALPHA, FIN_SS, FIN_OMEGA, FIN_RHO, FIN_RESID };
enum : int { SPMV_PLAIN = 0, SPMV_SIGMA = 1, SPMV_TS_TT = 2 };

struct DD;

struct RedArgs {
    DD *partials;           // [grid * 2]
    unsigned int *counter;  // zero-initialised, reset by the last block
    double *sc;             // device scalars
    double *loc;            // rank-local results (world > 1)
    int finalize;           // 1: last block finalizes (world == 1)
};

void launch_spmv(int mode, const dd_ctx *ctx, const double *x, const double *xg, double *y, const double *aux,
                 const RedArgs &ra, cudaStream_t st);
void launch_init_r(const dd_ctx *ctx, int64_t m, const double *b, const double *t, double *r, double *rh,
                   const RedArgs &ra, cudaStream_t st);
void launch_update_p(const dd_ctx *ctx, int64_t m, int first, const double *r, const double *v, double *p,
                     const double *sc, cudaStream_t st);
void launch_update_s(const dd_ctx *ctx, int64_t m, const double *r, const double *v, double *s, const RedArgs &ra,
                     cudaStream_t st);
void launch_update_x_half(const dd_ctx *ctx, int64_t m, const double *ph, double *x, const double *sc,
                          cudaStream_t st);
void launch_update_xr(const dd_ctx *ctx, int64_t m, const double *ph, const double *sh, const double *s,
                      const double *t, const double *rh, double *x, double *r, const RedArgs &ra, cudaStream_t st);
void launch_resid(const dd_ctx *ctx, int64_t m, const double *b, double *t, const RedArgs &ra, cudaStream_t st);
void launch_finalize_gathered(int world, int nv, const double *gathered, double *sc, int op, cudaStream_t st);
void launch_gather3(const dd_ctx *ctx, int64_t n, const int32_t *idx, const double *in, double *out, cudaStream_t st);
void launch_scatter3(const dd_ctx *ctx, int64_t n, const int32_t *idx, const double *in, double *out,
                     cudaStream_t st);
size_t partials_bytes(const dd_ctx *ctx);

}  // namespace ddk
