// refactor.cu -- GPU numeric re-factorisation with a fixed pattern (dd_refactor,
// SURVEY 8(f2); nonlinear solvers re-factor one pattern many times).
//
// The symbolic work (partition, reorder, drop pattern, levels, slab layout) is
// done once on the host by dd_setup; here, per call:
//   1. k_gather_blocks: new A values -> the A_dd working layout W (reordered,
//      dropped, subdomain-local order) and -> the sliced-ELL SpMV operand.
//   2. k_refactor: one CTA per subdomain; the rows of each L level are
//      factored in parallel (a row only reads rows of earlier levels), a CTA
//      barrier separates levels. Per row i, in the order of Alg. 7:
//      for each lower block k ascending: L_ik = W_ik Dinv_k, then
//      W_ij -= L_ik U_kj for the U_kj whose column is in row i (ascending j);
//      Dinv_i = inv(U_ii) (adjugate / determinant, R15); U_unit_ij = Dinv_i U_ij.
//      Same fma order as the host setup, so identical bits.
//      L, Dinv and U_unit go straight to their slab positions.
#include <cuda_runtime.h>

#include <cstdint>

#include "dd_internal.h"
#include "refactor.cuh"

namespace ddk {

__device__ __forceinline__ void rf_mul3(const double *A, const double *B, double *C) {
    double t[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            t[3 * r + c] = __fma_rn(A[3 * r + 2], B[6 + c], __fma_rn(A[3 * r + 1], B[3 + c], A[3 * r] * B[c]));
#pragma unroll
    for (int v = 0; v < 9; ++v) C[v] = t[v];
}

__device__ __forceinline__ void rf_sub_mul(double *W, const double *L, const double *U) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double w = W[3 * r + c];
            w = __fma_rn(-L[3 * r + 0], U[c], w);
            w = __fma_rn(-L[3 * r + 1], U[3 + c], w);
            w = __fma_rn(-L[3 * r + 2], U[6 + c], w);
            W[3 * r + c] = w;
        }
}

__device__ __forceinline__ bool rf_inv3(const double *m, double floor_, double *out) {
    const double c00 = __fma_rn(m[4], m[8], -(m[5] * m[7]));
    const double c01 = __fma_rn(m[5], m[6], -(m[3] * m[8]));
    const double c02 = __fma_rn(m[3], m[7], -(m[4] * m[6]));
    const double c10 = __fma_rn(m[2], m[7], -(m[1] * m[8]));
    const double c11 = __fma_rn(m[0], m[8], -(m[2] * m[6]));
    const double c12 = __fma_rn(m[1], m[6], -(m[0] * m[7]));
    const double c20 = __fma_rn(m[1], m[5], -(m[2] * m[4]));
    const double c21 = __fma_rn(m[2], m[3], -(m[0] * m[5]));
    const double c22 = __fma_rn(m[0], m[4], -(m[1] * m[3]));
    const double det = __fma_rn(m[0], c00, __fma_rn(m[1], c01, m[2] * c02));
    if (!(fabs(det) >= floor_)) return false;
    const double rd = 1.0 / det;
    out[0] = c00 * rd; out[1] = c10 * rd; out[2] = c20 * rd;
    out[3] = c01 * rd; out[4] = c11 * rd; out[5] = c21 * rd;
    out[6] = c02 * rd; out[7] = c12 * rd; out[8] = c22 * rd;
    return true;
}

__device__ __forceinline__ void rf_scatter(uint8_t *slab, int64_t off, int32_t st, const double *B) {
#pragma unroll
    for (int v = 0; v < 9; ++v) *reinterpret_cast<double *>(slab + off + (int64_t)st * v) = B[v];
}

// to[q] = from[src[q]] (9 doubles per block); ELL != 0: `to` is the sliced-ELL
// value array (slot q -> planes of 32 per block column), src < 0 = padding.
__global__ void k_gather_blocks(int64_t n, const int64_t *__restrict__ src, const double *__restrict__ from,
                                double *__restrict__ to, int ell) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sidx = src[q];
        if (sidx < 0) continue;
        const double *f = from + 9 * sidx;
        if (ell) {
            const int64_t lane = q & 31, base = 9 * (q - lane);
#pragma unroll
            for (int v = 0; v < 9; ++v) to[base + 32 * v + lane] = f[v];
        } else {
#pragma unroll
            for (int v = 0; v < 9; ++v) to[9 * q + v] = f[v];
        }
    }
}

__global__ void __launch_bounds__(128) k_refactor(RfArgs a) {
    const int q = blockIdx.x;
    for (int lev = a.SubLev[q]; lev < a.SubLev[q + 1]; ++lev) {
        for (int idx = a.LevPtr[lev] + threadIdx.x; idx < a.LevPtr[lev + 1]; idx += blockDim.x) {
            const int64_t li = a.LevRows[idx];
            const int64_t w0 = a.Wrp[li], d = a.Wdiag[li], w1 = a.Wrp[li + 1];
            for (int64_t p = w0; p < d; ++p) {
                const int64_t k = a.Wcol[p];
                double L[9];
                rf_mul3(a.W + 9 * p, a.Dinv + 9 * k, L);  // L_ik = W_ik * U_kk^-1 (R12)
#pragma unroll
                for (int v = 0; v < 9; ++v) a.W[9 * p + v] = L[v];
                const int64_t b = a.Lrp[li] + (p - w0);
                rf_scatter(a.slab, a.Loff[b], a.Lst[b], L);
                for (int64_t u = a.Uptr[p]; u < a.Uptr[p + 1]; ++u)
                    rf_sub_mul(a.W + 9 * (int64_t)a.UpdT[u], L, a.W + 9 * (int64_t)a.UpdQ[u]);
            }
            double inv[9];
            if (!rf_inv3(a.W + 9 * d, a.floor_, inv)) {
                atomicMin(a.bad, (unsigned long long)(a.row_first + li));
                continue;
            }
#pragma unroll
            for (int v = 0; v < 9; ++v) a.Dinv[9 * li + v] = inv[v];
            (void)w1;
        }
        __syncthreads();
    }
    // Dinv and U_unit_ij = Dinv_i U_ij of every row, in the order of the U
    // records (consecutive threads -> consecutive plane elements): no
    // dependencies between rows here, only on this row's final W and Dinv
    for (int idx = a.SubU[q] + threadIdx.x; idx < a.SubU[q + 1]; idx += blockDim.x) {
        const int64_t li = a.URows[idx];
        const int64_t d = a.Wdiag[li], w1 = a.Wrp[li + 1];
        double inv[9];
#pragma unroll
        for (int v = 0; v < 9; ++v) inv[v] = a.Dinv[9 * li + v];
        rf_scatter(a.slab, a.Doff[li], a.Dst[li], inv);
        for (int64_t p = d + 1; p < w1; ++p) {
            double Uu[9];
            rf_mul3(inv, a.W + 9 * p, Uu);  // U_unit_ij = Dinv_i * U_ij
            const int64_t b = a.Urp[li] + (p - d - 1);
            rf_scatter(a.slab, a.Uoff[b], a.Ust[b], Uu);
        }
    }
}

void launch_gather_blocks(int64_t n, const int64_t *src, const double *from, double *to, int ell, int grid,
                          cudaStream_t st) {
    k_gather_blocks<<<grid, 256, 0, st>>>(n, src, from, to, ell);
}

void launch_refactor(int nsl, const RfArgs &a, cudaStream_t st) { k_refactor<<<nsl, 128, 0, st>>>(a); }

}  // namespace ddk
