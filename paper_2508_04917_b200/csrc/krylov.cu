// krylov.cu -- BSR3 SpMV (sliced ELL, fused double-double dot epilogues),
// BLAS-1 updates with fused dots, deterministic last-block reductions and
// permutation gather/scatter for the right-preconditioned BiCGSTAB
// (Alg. 1 P:135-165 with K1 = I, K2 = M; DESIGN.md sec. 4 arithmetic order).
//
// Reductions: every thread accumulates Dot2 pairs (s, c) over its elements in
// a fixed order; blocks combine with a fixed shuffle tree; the last block to
// finish combines the block partials in block order. For a fixed grid the
// result is deterministic; it equals the oracle's sequential Dot2 after the
// final rounding except in rare straddling cases.
#include <cuda_runtime.h>

#include <algorithm>

#include <cstdlib>

#include "dd_internal.h"
#include "krylov.cuh"
#include "peer.cuh"

// Split dot reduction for the fused-dot SpMV modes (default): warps write
// per-slice Dot2 partials and a small second kernel combines them, instead of
// a block barrier + last-block combine inside the SpMV (whose finished warps
// then wait at the barrier and hold their slots: 14 % of the samples). In the
// solve at config 3: 0.424 -> 0.393 ms per SpMV including the second kernel.
// DD_SPMV_SPLITRED=0 builds the one-kernel form (ablation).
#ifndef DD_SPMV_SPLITRED
#define DD_SPMV_SPLITRED 1
#endif

namespace ddk {

struct DD {
    double s, c;
};

__device__ __forceinline__ void dot2_acc(double &s, double &c, double a, double b) {
    const double p = a * b;
    const double q = __fma_rn(a, b, -p);
    const double t = s + p;
    const double bb = t - s;
    const double r = (s - (t - bb)) + (p - bb);
    s = t;
    c = c + (q + r);
}

__device__ __forceinline__ DD dd_plus(DD x, DD y) {
    const double t = x.s + y.s;
    const double bb = t - x.s;
    const double e = (x.s - (t - bb)) + (y.s - bb);
    return DD{t, (x.c + y.c) + e};
}

__device__ __forceinline__ DD shfl_xor_dd(DD v, int m) {
    return DD{__shfl_xor_sync(0xffffffffu, v.s, m), __shfl_xor_sync(0xffffffffu, v.c, m)};
}

__device__ __forceinline__ DD warp_reduce_dd(DD v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v = dd_plus(v, shfl_xor_dd(v, m));
    return v;
}

// ---------------------------------------------------------------- finalize
// Runs in one thread after a reduction completes (last block, or the rank-order
// combine when world > 1). Besides the scalars of Alg. 1 it takes the solver's
// control decisions in the oracle's order (R21, R25):
//   FIN_INIT  ||r0||, rho_1 = r.r, thr = tol ||r0||; ||r0|| = 0 -> done
//   FIN_ALPHA |sigma| < 1e-30 -> breakdown, else alpha = rho / sigma
//   FIN_SS    ||s|| < thr -> half-step convergence (x += alpha p_hat pending)
//   FIN_OMEGA tau < 1e-30 -> breakdown, else omega = (t.s) / tau
//   FIN_RHO   ||r|| < thr -> converged; else |rho_next| < 1e-30 -> breakdown
__device__ __forceinline__ void finalize(double *sc, int op, const double *val, int *ctl, double *hist, int k) {
    if (k < 0 && ctl) k = ctl[C_ITER];  // graph mode: the iteration counter lives on the device
    switch (op) {
        case FIN_INIT: {  // ||r0||^2 and rho_1 = rh.r = r.r
            sc[S_RR] = val[0];
            sc[S_N0SQ] = val[0];
            sc[S_RHO] = val[0];
            const double n0 = sqrt(val[0]);
            sc[S_THR] = sc[S_TOL] * n0;
            if (ctl) {
                hist[0] = n0;
                ctl[C_NH] = 1;
                if (n0 == 0.0) {
                    ctl[C_STATE] = ST_ZERO;
                    ctl[C_K] = 0;
                } else if (fabs(val[0]) < 1e-30) {
                    ctl[C_STATE] = ST_BRK_RHO;
                    ctl[C_K] = 0;
                }
            }
            break;
        }
        case FIN_ALPHA:
            sc[S_SIGMA] = val[0];
            if (ctl && fabs(val[0]) < 1e-30) {
                ctl[C_STATE] = ST_BRK_SIGMA;
                ctl[C_K] = k;
                break;
            }
            sc[S_ALPHA] = sc[S_RHO] / val[0];
            break;
        case FIN_SS: {
            sc[S_SS] = val[0];
            const double ns = sqrt(val[0]);
            if (ctl) {
                hist[2 * k - 1] = ns;
                ctl[C_NH] = 2 * k;
                if (ns < sc[S_THR]) {
                    ctl[C_STATE] = ST_HALF;
                    ctl[C_K] = k;
                }
            }
            break;
        }
        case FIN_OMEGA:
            sc[S_TS] = val[0];
            sc[S_TT] = val[1];
            if (ctl && !(val[1] >= 1e-30)) {
                ctl[C_STATE] = ST_BRK_TAU;
                ctl[C_K] = k;
                break;
            }
            sc[S_OMEGA] = val[0] / val[1];
            break;
        case FIN_RHO: {
            sc[S_RR] = val[0];
            sc[S_RHO_PREV] = sc[S_RHO];
            sc[S_RHO] = val[1];
            const double nr = sqrt(val[0]);
            if (ctl) {
                hist[2 * k] = nr;
                ctl[C_NH] = 2 * k + 1;
                if (nr < sc[S_THR]) {
                    ctl[C_STATE] = ST_DONE_FULL;
                    ctl[C_K] = k;
                } else if (fabs(val[1]) < 1e-30) {
                    ctl[C_STATE] = ST_BRK_RHO;
                    ctl[C_K] = k;
                }
            }
            break;
        }
        case FIN_RESID:
            sc[S_RES_TT] = val[0];
            sc[S_RES_BB] = val[1];
            break;
        default:
            break;
    }
}

__device__ __forceinline__ bool stopped(const int *ctl) {
    return ctl && *reinterpret_cast<const volatile int *>(ctl + C_STATE) != ST_RUN;
}

// Block-reduce NV DD values, write this block's partials, and let the last
// block combine all partials in block order; returns true in thread 0 of the
// last block, which then holds the combined (s, c) pairs in out[].
template <int NV>
__device__ __forceinline__ bool grid_reduce(DD (&v)[NV], DD *partials, unsigned int *counter, DD (&out)[NV]) {
    __shared__ DD sh[NV][32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        DD w = warp_reduce_dd(v[q]);
        if (lane == 0) sh[q][wid] = w;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            DD acc = sh[q][0];
            for (int w = 1; w < nw; ++w) acc = dd_plus(acc, sh[q][w]);
            partials[blockIdx.x * NV + q] = acc;
        }
        __threadfence();
        const unsigned int prev = atomicAdd(counter, 1u);
        last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    // the last block combines the partials: thread t takes blocks t, t + bd,
    // ... in order, then warps and the block combine in a fixed tree (the
    // grid is fixed per context, so the result is deterministic)
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        DD acc{0.0, 0.0};
        for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
            const double2 pv = __ldcg(reinterpret_cast<const double2 *>(&partials[b * NV + q]));
            acc = dd_plus(acc, DD{pv.x, pv.y});
        }
        acc = warp_reduce_dd(acc);
        if (lane == 0) sh[q][wid] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            DD acc = sh[q][0];
            for (int w = 1; w < nw; ++w) acc = dd_plus(acc, sh[q][w]);
            out[q] = acc;
        }
        *counter = 0u;
    }
    return threadIdx.x == 0;
}

// Deliver reduced values: finalize now (world == 1) or publish the rank-local
// (s, c) pairs for the NCCL all-gather (world > 1).
template <int NV>
__device__ __forceinline__ void deliver(const RedArgs &ra, int op, const DD (&out)[NV]) {
    if (ra.finalize) {
        double vals[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) vals[q] = out[q].s + out[q].c;
        finalize(ra.sc, op, vals, ra.ctl, ra.hist, ra.k);
    } else {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            ra.loc[2 * (ra.slot + q)] = out[q].s;
            ra.loc[2 * (ra.slot + q) + 1] = out[q].c;
        }
    }
}

// ------------------------------------------------------------------- SpMV
// One warp per 32-row slice; thread = block row; 3 FMA chains per thread.
template <int BS, int MODE, int MINB>
__global__ void __launch_bounds__(256, MINB) k_spmv(int64_t n_rows, int64_t n_slices, const int64_t *__restrict__ slot_ptr,
                                              const int32_t *__restrict__ cols, const double *__restrict__ vals,
                                              const double *__restrict__ x, const double *__restrict__ xg,
                                              double *__restrict__ y, const double *__restrict__ aux, RedArgs ra) {
    if (MODE != SPMV_PLAIN && stopped(ra.ctl)) return;
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    DD d0{0.0, 0.0}, d1{0.0, 0.0};
    // plain mode: grid-stride over slices; fused-dot modes are launched with
    // one warp per slice, so the dot accumulators are not live across the
    // block loop (register pressure -> occupancy, the SpMV is latency-bound)
    for (int64_t sl = warp0; sl < n_slices; sl += (MODE == SPMV_PLAIN ? nwarps : n_slices)) {
        const int64_t base = slot_ptr[sl];
        const int K = (int)((slot_ptr[sl + 1] - base) >> 5);
        const int64_t row = 32 * sl + lane;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        if constexpr (BS == 1) {
            // scalar CSR rows: one value plane per k, acc = fma(a_ij, x_j, acc)
            for (int k = 0; k < K; ++k) {
                const int64_t slot = base + 32 * k + lane;
                const int32_t j = __ldg(cols + slot);
                if (j < 0) continue;
                const double xj = j < n_rows ? __ldg(x + j) : __ldg(xg + (j - n_rows));
                a0 = __fma_rn(__ldg(vals + slot), xj, a0);
            }
            if (row < n_rows) {
                y[row] = a0;
                if (MODE == SPMV_SIGMA) {
                    dot2_acc(d0.s, d0.c, aux[row], a0);
                } else if (MODE == SPMV_TS_TT) {
                    dot2_acc(d0.s, d0.c, a0, aux[row]);
                    dot2_acc(d1.s, d1.c, a0, a0);
                }
            }
            continue;
        }
        for (int k = 0; k < K; ++k) {
            const int64_t slot = base + 32 * k + lane;
            const int32_t j = __ldg(cols + slot);
            if (j < 0) continue;  // (a branch-free form with zero padding measured 3 % slower)
            const double *vb = vals + 9 * (base + 32 * k) + lane;
            double b[9];
#pragma unroll
            for (int v = 0; v < 9; ++v) b[v] = __ldg(vb + 32 * v);
            // local columns < n_rows, ghost (halo) columns after them (sec. 8e)
            const double *xp = j < n_rows ? x + 3 * (int64_t)j : xg + 3 * ((int64_t)j - n_rows);
            const double x0 = __ldg(xp), x1 = __ldg(xp + 1), x2 = __ldg(xp + 2);
            a0 = __fma_rn(b[0], x0, a0);
            a0 = __fma_rn(b[1], x1, a0);
            a0 = __fma_rn(b[2], x2, a0);
            a1 = __fma_rn(b[3], x0, a1);
            a1 = __fma_rn(b[4], x1, a1);
            a1 = __fma_rn(b[5], x2, a1);
            a2 = __fma_rn(b[6], x0, a2);
            a2 = __fma_rn(b[7], x1, a2);
            a2 = __fma_rn(b[8], x2, a2);
        }
        if (row < n_rows) {
            y[3 * row] = a0;
            y[3 * row + 1] = a1;
            y[3 * row + 2] = a2;
            if (MODE == SPMV_SIGMA) {  // aux = rh : rh . y
                dot2_acc(d0.s, d0.c, aux[3 * row], a0);
                dot2_acc(d0.s, d0.c, aux[3 * row + 1], a1);
                dot2_acc(d0.s, d0.c, aux[3 * row + 2], a2);
            } else if (MODE == SPMV_TS_TT) {  // aux = s : t.s and t.t
                dot2_acc(d0.s, d0.c, a0, aux[3 * row]);
                dot2_acc(d0.s, d0.c, a1, aux[3 * row + 1]);
                dot2_acc(d0.s, d0.c, a2, aux[3 * row + 2]);
                dot2_acc(d1.s, d1.c, a0, a0);
                dot2_acc(d1.s, d1.c, a1, a1);
                dot2_acc(d1.s, d1.c, a2, a2);
            }
        }
    }
#if DD_SPMV_SPLITRED
    // split reduction: each warp (one slice) writes its Dot2 partials; the
    // reduction kernel that follows combines them (no block barrier or
    // atomic here, so finished warps leave at once)
    if (MODE != SPMV_PLAIN) {
        const DD w0 = warp_reduce_dd(d0);
        if (MODE == SPMV_SIGMA) {
            if (lane == 0 && warp0 < n_slices) ra.partials[warp0] = w0;
        } else {
            const DD w1 = warp_reduce_dd(d1);
            if (lane == 0 && warp0 < n_slices) {
                ra.partials[2 * warp0] = w0;
                ra.partials[2 * warp0 + 1] = w1;
            }
        }
    }
#else
    if (MODE == SPMV_SIGMA) {
        DD v[1] = {d0}, out[1];
        if (grid_reduce<1>(v, ra.partials, ra.counter, out)) deliver<1>(ra, FIN_ALPHA, out);
    } else if (MODE == SPMV_TS_TT) {
        DD v[2] = {d0, d1}, out[2];
        if (grid_reduce<2>(v, ra.partials, ra.counter, out)) deliver<2>(ra, FIN_OMEGA, out);
    }
#endif
}

// Second stage of the split SpMV reduction: thread i combines slice partials
// i, i + stride, ... in order, then the usual block tree and last-block
// combine (fixed grid -> deterministic); block partials live after the slice
// partials.
template <int NV>
__global__ void __launch_bounds__(256) k_reduce_slices(int64_t n_slices, RedArgs ra, int op) {
    if (stopped(ra.ctl)) return;
    DD v[NV], out[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = DD{0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_slices; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const double2 pv = __ldcg(reinterpret_cast<const double2 *>(&ra.partials[i * NV + q]));
            v[q] = dd_plus(v[q], DD{pv.x, pv.y});
        }
    }
    if (grid_reduce<NV>(v, ra.partials + NV * n_slices, ra.counter, out)) deliver<NV>(ra, op, out);
}

// ------------------------------------------------------------------ BLAS-1
// r = b - t; rh = r; partial r.r
__global__ void __launch_bounds__(256) k_init_r(int64_t m, const double *__restrict__ b, const double *__restrict__ t,
                                                double *__restrict__ r, double *__restrict__ rh, RedArgs ra) {
    DD d{0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = b[i] - t[i];
        r[i] = v;
        rh[i] = v;
        dot2_acc(d.s, d.c, v, v);
    }
    DD v[1] = {d}, out[1];
    if (grid_reduce<1>(v, ra.partials, ra.counter, out)) deliver<1>(ra, FIN_INIT, out);
}

// Elementwise BLAS-1 kernels: VEC = 16-byte (double2) loads/stores when every
// pointer is 16-byte aligned (the scalar tail element, if 3n is odd, is done
// by thread 0); the grid is fixed per context, so the fused dots are
// deterministic for a given context.
#define GRID_STRIDE(i, n) for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// p = r (first) or p = fma(beta, fma(-omega, v, p), r), beta = (rho/rho_prev)*(alpha/omega)
template <bool VEC>
__global__ void __launch_bounds__(256) k_update_p(int64_t m, int first, const double *__restrict__ r,
                                                  const double *__restrict__ v, double *__restrict__ p,
                                                  const double *__restrict__ sc, const int *ctl) {
    if (stopped(ctl)) return;
    if (first < 0) first = ctl[C_ITER] == 1;  // graph mode
    const double omega = sc[S_OMEGA];
    const double beta = (sc[S_RHO] / sc[S_RHO_PREV]) * (sc[S_ALPHA] / omega);
    auto one = [&](double rv, double vv, double pv) { return first ? rv : __fma_rn(beta, __fma_rn(-omega, vv, pv), rv); };
    if (VEC) {
        const double2 *r2 = reinterpret_cast<const double2 *>(r), *v2 = reinterpret_cast<const double2 *>(v);
        double2 *p2 = reinterpret_cast<double2 *>(p);
        GRID_STRIDE(i, m >> 1) {
            const double2 a = r2[i], b = first ? make_double2(0, 0) : v2[i], c = first ? make_double2(0, 0) : p2[i];
            p2[i] = make_double2(one(a.x, b.x, c.x), one(a.y, b.y, c.y));
        }
        if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[m - 1] = one(r[m - 1], v[m - 1], p[m - 1]);
    } else {
        GRID_STRIDE(i, m) p[i] = one(r[i], v[i], p[i]);
    }
}

// s = fma(-alpha, v, r); partial s.s
template <bool VEC>
__global__ void __launch_bounds__(256) k_update_s(int64_t m, const double *__restrict__ r, const double *__restrict__ v,
                                                  double *__restrict__ s, RedArgs ra) {
    if (stopped(ra.ctl)) return;
    const double alpha = ra.sc[S_ALPHA];
    DD d{0.0, 0.0};
    auto one = [&](double rv, double vv) {
        const double sv = __fma_rn(-alpha, vv, rv);
        dot2_acc(d.s, d.c, sv, sv);
        return sv;
    };
    if (VEC) {
        const double2 *r2 = reinterpret_cast<const double2 *>(r), *v2 = reinterpret_cast<const double2 *>(v);
        double2 *s2 = reinterpret_cast<double2 *>(s);
        GRID_STRIDE(i, m >> 1) {
            const double2 a = r2[i], b = v2[i];
            const double x0 = one(a.x, b.x);
            const double x1 = one(a.y, b.y);
            s2[i] = make_double2(x0, x1);
        }
        if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) s[m - 1] = one(r[m - 1], v[m - 1]);
    } else {
        GRID_STRIDE(i, m) s[i] = one(r[i], v[i]);
    }
    DD vv[1] = {d}, out[1];
    if (grid_reduce<1>(vv, ra.partials, ra.counter, out)) deliver<1>(ra, FIN_SS, out);
}

// x = fma(alpha, ph, x)   (half-step exit; runs only when FIN_SS found
// ||s|| < thr; the last block then marks the solve converged)
__global__ void __launch_bounds__(256) k_update_x_half(int64_t m, const double *__restrict__ ph, double *__restrict__ x,
                                                       const double *__restrict__ sc, int *ctl) {
    if (*reinterpret_cast<const volatile int *>(ctl + C_STATE) != ST_HALF) return;
    const double alpha = sc[S_ALPHA];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __fma_rn(alpha, ph[i], x[i]);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned int *cnt = reinterpret_cast<unsigned int *>(ctl + C_CNT);
        if (atomicAdd(cnt, 1u) == gridDim.x - 1) {
            *cnt = 0u;
            ctl[C_STATE] = ST_DONE_HALF;
        }
    }
}

// x = fma(omega, sh, fma(alpha, ph, x)); r = fma(-omega, t, s); partials r.r, rh.r
template <bool VEC>
__global__ void __launch_bounds__(256) k_update_xr(int64_t m, const double *__restrict__ ph,
                                                   const double *__restrict__ sh, const double *__restrict__ s,
                                                   const double *__restrict__ t, const double *__restrict__ rh,
                                                   double *__restrict__ x, double *__restrict__ r, RedArgs ra) {
    if (stopped(ra.ctl)) return;
    const double alpha = ra.sc[S_ALPHA], omega = ra.sc[S_OMEGA];
    DD d0{0.0, 0.0}, d1{0.0, 0.0};
    auto one = [&](double phv, double shv, double sv, double tv, double rhv, double &xv) {
        xv = __fma_rn(omega, shv, __fma_rn(alpha, phv, xv));
        const double rv = __fma_rn(-omega, tv, sv);
        dot2_acc(d0.s, d0.c, rv, rv);
        dot2_acc(d1.s, d1.c, rhv, rv);
        return rv;
    };
    if (VEC) {
        const double2 *ph2 = reinterpret_cast<const double2 *>(ph), *sh2 = reinterpret_cast<const double2 *>(sh),
                      *s2 = reinterpret_cast<const double2 *>(s), *t2 = reinterpret_cast<const double2 *>(t),
                      *rh2 = reinterpret_cast<const double2 *>(rh);
        double2 *x2 = reinterpret_cast<double2 *>(x), *r2 = reinterpret_cast<double2 *>(r);
        GRID_STRIDE(i, m >> 1) {
            const double2 a = ph2[i], b = sh2[i], c = s2[i], e = t2[i], f = rh2[i];
            double2 xv = x2[i];
            const double r0 = one(a.x, b.x, c.x, e.x, f.x, xv.x);
            const double r1 = one(a.y, b.y, c.y, e.y, f.y, xv.y);
            x2[i] = xv;
            r2[i] = make_double2(r0, r1);
        }
        if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
            double xv = x[m - 1];
            r[m - 1] = one(ph[m - 1], sh[m - 1], s[m - 1], t[m - 1], rh[m - 1], xv);
            x[m - 1] = xv;
        }
    } else {
        GRID_STRIDE(i, m) {
            double xv = x[i];
            r[i] = one(ph[i], sh[i], s[i], t[i], rh[i], xv);
            x[i] = xv;
        }
    }
    DD v[2] = {d0, d1}, out[2];
    if (grid_reduce<2>(v, ra.partials, ra.counter, out)) deliver<2>(ra, FIN_RHO, out);
}

// t = b - t; partials t.t, b.b (true residual)
__global__ void __launch_bounds__(256) k_resid(int64_t m, const double *__restrict__ b, double *__restrict__ t,
                                               RedArgs ra) {
    DD d0{0.0, 0.0}, d1{0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = b[i] - t[i];
        t[i] = v;
        dot2_acc(d0.s, d0.c, v, v);
        dot2_acc(d1.s, d1.c, b[i], b[i]);
    }
    DD v[2] = {d0, d1}, out[2];
    if (grid_reduce<2>(v, ra.partials, ra.counter, out)) deliver<2>(ra, FIN_RESID, out);
}

// multi-rank: combine the gathered per-rank values (in rank order) and
// finalize; rank rr's pairs at gathered[rr * stride ..]
__device__ void combine_finalize(int world, int nv, const volatile double *gathered, int stride, const RedArgs &ra,
                                 int op) {
    double out[3] = {0.0, 0.0, 0.0};
    for (int q = 0; q < nv; ++q) {
        DD acc{0.0, 0.0};
        for (int rr = 0; rr < world; ++rr)
            acc = dd_plus(acc, DD{gathered[rr * stride + 2 * q], gathered[rr * stride + 2 * q + 1]});
        out[q] = acc.s + acc.c;
    }
    if (op == FIN_SS_OMEGA) {
        // the half-step test comes first, as in Alg. 1; omega only if it failed
        finalize(ra.sc, FIN_SS, out + 2, ra.ctl, ra.hist, ra.k);
        if (stopped(ra.ctl)) return;
        op = FIN_OMEGA;
    }
    finalize(ra.sc, op, out, ra.ctl, ra.hist, ra.k);
}

__global__ void k_finalize_gathered(int world, int nv, const double *__restrict__ gathered, RedArgs ra, int op) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (op != FIN_INIT && op != FIN_RESID && stopped(ra.ctl)) return;
    combine_finalize(world, nv, gathered, 2 * nv, ra, op);
}

// peer transport (DD_COMM_LOCAL / DD_COMM_IPC, peer.cuh): publish this rank's
// pairs into every rank's gathered slot (double-buffered by the parity of the
// DOT count: a peer can be at most one all-gather ahead, because the next one
// needs this rank's partial), release the count, wait for every peer, then
// the same rank-order combine. Skipped by the same rule on every rank.
__global__ void k_peer_allgather_finalize(PeerDev d, int nv, const double *__restrict__ loc, RedArgs ra, int op) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (op != FIN_INIT && op != FIN_RESID && stopped(ra.ctl)) return;
    if (*reinterpret_cast<volatile int *>(d.err)) return;
    const unsigned long long s = ++d.seq[PCH_DOT];
    const int par = (int)(s & 1ull);
    double v[6];
    for (int e = 0; e < 2 * nv; ++e) v[e] = loc[e];
    for (int q = 0; q < d.world; ++q) {
        double *g = peer_gath(d, q) + (par * d.world + d.rank) * 6;
        for (int e = 0; e < 2 * nv; ++e) g[e] = v[e];
    }
    __threadfence_system();
    for (int q = 0; q < d.world; ++q)
        if (q != d.rank) peer_st_release(peer_flags(d, q) + PCH_DOT * d.world + d.rank, s);
    const unsigned long long target = ++d.seq[PCH_COUNT + PCH_DOT];
    for (int q = 0; q < d.world; ++q)
        if (q != d.rank && !peer_spin(d, PCH_DOT, q, target)) {
            if (ra.ctl) ra.ctl[C_STATE] = ST_COMM;
            return;
        }
    combine_finalize(d.world, nv, peer_gath(d, d.rank) + par * d.world * 6, 6, ra, op);
}

// permutation helpers: out[3 li + c] = in[3 idx[li] + c] and the reverse
// row gather / scatter of bs-wide rows (bs = 3: BSR3, 1: scalar CSR)
template <int BS>
__global__ void k_gather3(int64_t n, const int32_t *__restrict__ idx, const double *__restrict__ in,
                          double *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < BS * n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[BS * (int64_t)idx[i / BS] + i % BS];
}

template <int BS>
__global__ void k_scatter3(int64_t n, const int32_t *__restrict__ idx, const double *__restrict__ in,
                           double *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < BS * n; i += (int64_t)gridDim.x * blockDim.x)
        out[BS * (int64_t)idx[i / BS] + i % BS] = in[i];
}

}  // namespace ddk

// ---------------------------------------------------------------- launchers
namespace ddk {

// DD_SPMV_MINB_<mode> (experiment knob): min resident blocks per SM for the
// launch bounds of each SpMV mode (1 = compiler's choice).
template <int MODE>
static void spmv_go(int bs, int minb, int grid, cudaStream_t st, int64_t n, const ddi::SpmvDev &S, const double *x,
                    const double *xg, double *y, const double *aux, const RedArgs &ra) {
    if (bs == 1) {
        k_spmv<1, MODE, 1><<<grid, 256, 0, st>>>(n, S.n_slices, S.slot_ptr, S.cols, S.vals, x, xg, y, aux, ra);
        return;
    }
    switch (minb) {
        case 8: k_spmv<3, MODE, 8><<<grid, 256, 0, st>>>(n, S.n_slices, S.slot_ptr, S.cols, S.vals, x, xg, y, aux, ra); break;
        case 6: k_spmv<3, MODE, 6><<<grid, 256, 0, st>>>(n, S.n_slices, S.slot_ptr, S.cols, S.vals, x, xg, y, aux, ra); break;
        case 5: k_spmv<3, MODE, 5><<<grid, 256, 0, st>>>(n, S.n_slices, S.slot_ptr, S.cols, S.vals, x, xg, y, aux, ra); break;
        default: k_spmv<3, MODE, 1><<<grid, 256, 0, st>>>(n, S.n_slices, S.slot_ptr, S.cols, S.vals, x, xg, y, aux, ra); break;
    }
}

static int env_i(const char *n, int d) {
    const char *v = getenv(n);
    return v ? atoi(v) : d;
}

static int reduce_grid(const dd_ctx *ctx) { return ctx->num_sms; }

static int spmv_fused_grid(const dd_ctx *ctx) {
    return (int)std::max<int64_t>(1, (ctx->spmv.n_slices + 7) / 8);
}

void launch_spmv(int mode, const dd_ctx *ctx, const double *x, const double *xg, double *y, const double *aux,
                 const RedArgs &ra, cudaStream_t st) {
    ++ctx->n_launches;
    const auto &S = ctx->spmv;
    const int grid = ctx->num_sms * 8;           // plain: grid-stride
    const int grid1 = spmv_fused_grid(ctx);      // fused dots: one warp per slice (fixed per context)
    static const int mb0 = env_i("DD_SPMV_MINB_0", 1), mb1 = env_i("DD_SPMV_MINB_1", 1),
                     mb2 = env_i("DD_SPMV_MINB_2", 1);
    switch (mode) {
        case SPMV_PLAIN: spmv_go<SPMV_PLAIN>(ctx->bs, mb0, grid, st, ctx->n_local, S, x, xg, y, aux, ra); break;
        case SPMV_SIGMA: spmv_go<SPMV_SIGMA>(ctx->bs, mb1, grid1, st, ctx->n_local, S, x, xg, y, aux, ra); break;
        case SPMV_TS_TT: spmv_go<SPMV_TS_TT>(ctx->bs, mb2, grid1, st, ctx->n_local, S, x, xg, y, aux, ra); break;
    }
#if DD_SPMV_SPLITRED
    if (mode != SPMV_PLAIN) {
        ++ctx->n_launches;
        const int g = reduce_grid(ctx);
        if (mode == SPMV_SIGMA) k_reduce_slices<1><<<g, 256, 0, st>>>(S.n_slices, ra, FIN_ALPHA);
        else k_reduce_slices<2><<<g, 256, 0, st>>>(S.n_slices, ra, FIN_OMEGA);
    }
#endif
}

// BLAS-1 grid: 4 CTAs of 256 threads per SM (config 3: 27.3 ms of BLAS-1 per
// solve; 8 per SM 28.3 ms, 16 28.9, 2 34.1); DD_BLAS_GRID_MULT overrides (1-16)
int blas_grid(const dd_ctx *ctx) {
    static const int mult = std::max(1, std::min(16, env_i("DD_BLAS_GRID_MULT", 4)));
    return ctx->num_sms * mult;
}

__global__ void k_iter_head(int *ctl) {
    if (ctl[C_STATE] == ST_RUN) ctl[C_ITER] += 1;
}
__global__ void k_iter_tail(int *ctl, cudaGraphConditionalHandle h) {
    cudaGraphSetConditional(h, (ctl[C_STATE] == ST_RUN && ctl[C_ITER] < ctl[C_MAX]) ? 1u : 0u);
}
void launch_iter_head(int *ctl, cudaStream_t st) { k_iter_head<<<1, 1, 0, st>>>(ctl); }
void launch_iter_tail(int *ctl, cudaGraphConditionalHandle h, cudaStream_t st) { k_iter_tail<<<1, 1, 0, st>>>(ctl, h); }

static inline bool al16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

void launch_init_r(const dd_ctx *ctx, int64_t m, const double *b, const double *t, double *r, double *rh,
                   const RedArgs &ra, cudaStream_t st) {
    ++ctx->n_launches;
    k_init_r<<<blas_grid(ctx), 256, 0, st>>>(m, b, t, r, rh, ra);
}
void launch_update_p(const dd_ctx *ctx, int64_t m, int first, const double *r, const double *v, double *p,
                     const double *sc, const int *ctl, cudaStream_t st) {
    ++ctx->n_launches;
    if (al16(r) && al16(v) && al16(p)) k_update_p<true><<<blas_grid(ctx), 256, 0, st>>>(m, first, r, v, p, sc, ctl);
    else k_update_p<false><<<blas_grid(ctx), 256, 0, st>>>(m, first, r, v, p, sc, ctl);
}
void launch_update_s(const dd_ctx *ctx, int64_t m, const double *r, const double *v, double *s, const RedArgs &ra,
                     cudaStream_t st) {
    ++ctx->n_launches;
    if (al16(r) && al16(v) && al16(s)) k_update_s<true><<<blas_grid(ctx), 256, 0, st>>>(m, r, v, s, ra);
    else k_update_s<false><<<blas_grid(ctx), 256, 0, st>>>(m, r, v, s, ra);
}
void launch_update_x_half(const dd_ctx *ctx, int64_t m, const double *ph, double *x, const double *sc, int *ctl,
                          cudaStream_t st) {
    ++ctx->n_launches;
    k_update_x_half<<<blas_grid(ctx), 256, 0, st>>>(m, ph, x, sc, ctl);
}
void launch_update_xr(const dd_ctx *ctx, int64_t m, const double *ph, const double *sh, const double *s,
                      const double *t, const double *rh, double *x, double *r, const RedArgs &ra, cudaStream_t st) {
    ++ctx->n_launches;
    if (al16(ph) && al16(sh) && al16(s) && al16(t) && al16(rh) && al16(x) && al16(r))
        k_update_xr<true><<<blas_grid(ctx), 256, 0, st>>>(m, ph, sh, s, t, rh, x, r, ra);
    else
        k_update_xr<false><<<blas_grid(ctx), 256, 0, st>>>(m, ph, sh, s, t, rh, x, r, ra);
}
void launch_resid(const dd_ctx *ctx, int64_t m, const double *b, double *t, const RedArgs &ra, cudaStream_t st) {
    ++ctx->n_launches;
    k_resid<<<blas_grid(ctx), 256, 0, st>>>(m, b, t, ra);
}
void launch_finalize_gathered(int world, int nv, const double *gathered, const RedArgs &ra, int op, cudaStream_t st) {
    k_finalize_gathered<<<1, 32, 0, st>>>(world, nv, gathered, ra, op);
}
template <int BS>
__global__ void k_build_ell(int64_t n_slices, int64_t n_rows, const int64_t *__restrict__ slot_ptr,
                            const int64_t *__restrict__ rp, const int32_t *__restrict__ ci,
                            const double *__restrict__ av, int32_t *__restrict__ cols, double *__restrict__ vals) {
    constexpr int B2 = BS * BS;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t s = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); s < n_slices; s += warps) {
        const int64_t li = 32 * s + lane;
        const int64_t p0 = li < n_rows ? rp[li] : 0, len = li < n_rows ? rp[li + 1] - p0 : 0;
        const int64_t K = (slot_ptr[s + 1] - slot_ptr[s]) / 32;
        for (int64_t k = 0; k < K; ++k) {
            const bool has = k < len;
            const int64_t slot = slot_ptr[s] + 32 * k;
            cols[slot + lane] = has ? ci[p0 + k] : -1;
            if (av || !has)  // av null: the values are gathered later (GPU numeric setup), padding zeroed here
#pragma unroll
                for (int v = 0; v < B2; ++v) vals[B2 * slot + 32 * v + lane] = has ? av[B2 * (p0 + k) + v] : 0.0;
        }
    }
}

void launch_build_ell(int bs, int64_t n_slices, int64_t n_rows, const int64_t *slot_ptr, const int64_t *rp,
                      const int32_t *ci, const double *av, int32_t *cols, double *vals, cudaStream_t st) {
    if (n_slices <= 0) return;
    const int g = (int)std::min<int64_t>(4096, (n_slices + 7) / 8);
    if (bs == 3)
        k_build_ell<3><<<g, 256, 0, st>>>(n_slices, n_rows, slot_ptr, rp, ci, av, cols, vals);
    else
        k_build_ell<1><<<g, 256, 0, st>>>(n_slices, n_rows, slot_ptr, rp, ci, av, cols, vals);
}

void launch_peer_allgather_finalize(const PeerDev &d, int nv, const double *loc, const RedArgs &ra, int op,
                                    cudaStream_t st) {
    k_peer_allgather_finalize<<<1, 32, 0, st>>>(d, nv, loc, ra, op);
}
void launch_gather3(const dd_ctx *ctx, int64_t n, const int32_t *idx, const double *in, double *out, cudaStream_t st) {
    ++ctx->n_launches;
    if (ctx->bs == 1) k_gather3<1><<<ctx->num_sms * 8, 256, 0, st>>>(n, idx, in, out);
    else k_gather3<3><<<ctx->num_sms * 8, 256, 0, st>>>(n, idx, in, out);
}
void launch_scatter3(const dd_ctx *ctx, int64_t n, const int32_t *idx, const double *in, double *out,
                     cudaStream_t st) {
    ++ctx->n_launches;
    if (ctx->bs == 1) k_scatter3<1><<<ctx->num_sms * 8, 256, 0, st>>>(n, idx, in, out);
    else k_scatter3<3><<<ctx->num_sms * 8, 256, 0, st>>>(n, idx, in, out);
}
size_t partials_bytes(const dd_ctx *ctx) {
    // block partials of any grid_reduce; split SpMV reduction: 2 per slice + its block partials
    return sizeof(DD) * 2 * (size_t)std::max<int64_t>(ctx->num_sms * 16, spmv_fused_grid(ctx)) +
           sizeof(DD) * 2 * (size_t)(ctx->spmv.n_slices + reduce_grid(ctx));
}

}  // namespace ddk
