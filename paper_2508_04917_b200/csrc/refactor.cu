// refactor.cu -- GPU numeric re-factorisation with a fixed pattern (dd_refactor,
// SURVEY 8(f2); nonlinear solvers re-factor one pattern many times).
//
// The symbolic work (partition, reorder, drop pattern, levels, slab layout) is
// done once on the host by dd_setup; here, per call:
//   1. k_gather_w9 / k_gather_blocks: new A values -> the A_dd working layout
//      W (reordered, dropped, subdomain-local order) / -> the sliced-ELL SpMV
//      operand.
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
#include <cstdlib>

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
__global__ void k_gather_blocks(int64_t n, const int32_t *__restrict__ src, const double *__restrict__ from,
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

// Nine lanes per 3x3 block ("a warp per row and 9 lanes per 3x3
// op"): lane v = 3r + c of a 9-lane group owns element (r, c) of every block
// the group touches, so each block load / store is 72 contiguous bytes and
// every element of W is only ever loaded and stored by the same lane (no
// cross-lane memory ordering inside a group); the other elements a product
// needs arrive by warp shuffles. Three groups per warp (lanes 27-31 idle),
// so a 512-thread CTA factors 48 rows of a level at once. Loops run to the
// warp's maximum trip count with predicated memory operations, so every
// shuffle is warp-uniform. Per element the FMA order is rf_mul3 /
// rf_sub_mul / rf_inv3's (= the host setup's): identical bits.
#ifndef RF9_THREADS_DEF
#define RF9_THREADS_DEF 256
#endif
#ifndef RF9_MINB
#define RF9_MINB 4
#endif
constexpr int RF9_THREADS = RF9_THREADS_DEF;

__device__ __forceinline__ double g9(double x, int gbase, int src) {
    return __shfl_sync(0xffffffffu, x, (gbase + src) & 31);
}

__device__ __forceinline__ int warp_max(int x) { return __reduce_max_sync(0xffffffffu, x); }

// Dinv and U_unit_ij = Dinv_i U_ij of subdomain q's rows in the order of the U
// records: no dependencies between rows, only on the L levels' final W and
// Dinv. One thread per row: it loads Dinv_i and each U_ij (72 contiguous bytes
// each) and writes the nine plane elements of each output block; consecutive
// threads take consecutive rows of a U record, so every store instruction
// writes consecutive plane elements (full 32-byte sectors; nine lanes per
// block wrote three rows' elements per warp store: 4.69 -> 4.28 ms per
// dd_refactor at 160^3). rf_mul3's FMA order.
template <bool FROM_A>
__device__ __forceinline__ void rf_upass_rows(const RfArgs &a, int q) {
    const int ulo = a.SubU[q], uhi = a.SubU[q + 1];
    for (int idx = ulo + threadIdx.x; idx < uhi; idx += blockDim.x) {
        const int64_t li = a.URows[idx];
        const int64_t d = a.Wdiag[li], w1 = a.Wrp[li + 1];
        double inv[9];
#pragma unroll
        for (int v = 0; v < 9; ++v) inv[v] = a.Dinv[9 * li + v];
        rf_scatter(a.slab, a.Doff[li], a.Dst[li], inv);
        const int64_t ub = a.Urp[li];
        for (int64_t p = d + 1; p < w1; ++p) {
            double Uu[9];
            // U_unit_ij = Dinv_i * U_ij (FROM_A: U_ij is still the caller's block)
            rf_mul3(inv, FROM_A ? a.A + 9 * (int64_t)a.Wsrc[p] : a.W + 9 * p, Uu);
            const int64_t b = ub + (p - d - 1);
            rf_scatter(a.slab, a.Uoff[b], a.Ust[b], Uu);
        }
    }
}

__global__ void __launch_bounds__(RF9_THREADS, RF9_MINB) k_refactor9(RfArgs a) {
    const int q = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / 9;  // 0..2 active, 3 = idle lanes 27..31
    const int v = lane - 9 * grp, r3 = 3 * (v / 3), c = v % 3;
    const int gbase = 9 * grp;
    const bool live = grp < 3;
    const int per_pass = 3 * (blockDim.x / 32);
    for (int lev = a.SubLev[q]; lev < a.SubLev[q + 1]; ++lev) {
        const int lo = a.LevPtr[lev], hi = a.LevPtr[lev + 1];
        for (int base = lo + 3 * warp; base < hi; base += per_pass) {
            const int idx = base + grp;
            const bool has = live && idx < hi;
            const int64_t li = has ? a.LevRows[idx] : 0;
            const int64_t w0 = has ? a.Wrp[li] : 0, d = has ? a.Wdiag[li] : 0;
            const int nlow = has ? (int)(d - w0) : 0;
            const int maxlow = warp_max(nlow);
            for (int jp = 0; jp < maxlow; ++jp) {
                const bool ok = jp < nlow;
                const int64_t p = w0 + jp;
                const int64_t k = ok ? a.Wcol[p] : 0;
                const double wv = ok ? a.W[9 * p + v] : 0.0;
                const double dv = ok ? a.Dinv[9 * k + v] : 0.0;
                // L_ik = W_ik * U_kk^-1 (R12): rf_mul3(W, Dinv, L)
                const double Lv = __fma_rn(g9(wv, gbase, r3 + 2), g9(dv, gbase, 6 + c),
                                           __fma_rn(g9(wv, gbase, r3 + 1), g9(dv, gbase, 3 + c),
                                                    g9(wv, gbase, r3) * g9(dv, gbase, c)));
                if (ok) {
                    a.W[9 * p + v] = Lv;
                    const int64_t b = a.Lrp[li] + jp;
                    *reinterpret_cast<double *>(a.slab + a.Loff[b] + (int64_t)a.Lst[b] * v) = Lv;
                }
                const int64_t u0 = ok ? a.Uptr[p] : 0;
                const int nup = ok ? (int)(a.Uptr[p + 1] - u0) : 0;
                const int maxup = warp_max(nup);
                for (int ju = 0; ju < maxup; ++ju) {
                    const bool okk = ju < nup;
                    const int64_t t = okk ? a.UpdT[u0 + ju] : 0, qq = okk ? a.UpdQ[u0 + ju] : 0;
                    const double wt = okk ? a.W[9 * t + v] : 0.0;
                    const double uq = okk ? a.W[9 * qq + v] : 0.0;
                    // W_ij -= L_ik U_kj: rf_sub_mul's order
                    double w = __fma_rn(-g9(Lv, gbase, r3), g9(uq, gbase, c), wt);
                    w = __fma_rn(-g9(Lv, gbase, r3 + 1), g9(uq, gbase, 3 + c), w);
                    w = __fma_rn(-g9(Lv, gbase, r3 + 2), g9(uq, gbase, 6 + c), w);
                    if (okk) a.W[9 * t + v] = w;
                }
            }
            // Dinv_i = inv(U_ii): every lane of the group gathers the block
            const double mv = has ? a.W[9 * d + v] : 0.0;
            double m[9], inv[9];
#pragma unroll
            for (int e = 0; e < 9; ++e) m[e] = g9(mv, gbase, e);
            const bool okinv = rf_inv3(m, a.floor_, inv);
            if (has) {
                if (!okinv) {
                    if (v == 0) atomicMin(a.bad, (unsigned long long)(a.row_first + li));
                } else {
                    double mine = inv[0];
#pragma unroll
                    for (int e = 1; e < 9; ++e)
                        if (e == v) mine = inv[e];
                    a.Dinv[9 * li + v] = mine;
                }
            }
        }
        __syncthreads();
    }
    rf_upass_rows<false>(a, q);
}

// Diagonal-update class (every row has <= 3 lower blocks and every ILU0 update
// of its elimination lands on its diagonal block -- the 7-point stencils of the
// paper's matrices: with pattern(i) = {i, i +- 1, i +- nx, i +- nx ny} the only
// j in pattern(i) n pattern(U_k) for a lower neighbour k is j = i). Then the
// lower blocks W_ik and the U_ki the updates use are still the matrix's own
// values when row i is eliminated, and the only operand that crosses rows is
// Dinv_k. Each row's plan (12 words, refactor_api.cpp) names every operand, so
// a 9-lane group issues all of its loads at once and keeps U_ii in registers
// through the updates. Per element the FMA order is rf_mul3 / rf_sub_mul /
// rf_inv3's (the host's): identical bits. The U pass is k_refactor9's.
#ifndef RFD_MINB
#define RFD_MINB 2
#endif
#ifndef RFD_THREADS
#define RFD_THREADS 384
#endif
__global__ void __launch_bounds__(RFD_THREADS, RFD_MINB) k_refactor_diag(RfArgs a, const int32_t *__restrict__ plan) {
    const int q = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / 9;
    const int v = lane - 9 * grp, r3 = 3 * (v / 3), c = v % 3;
    const int gbase = 9 * grp;
    const bool live = grp < 3;
    const int per_pass = 3 * (blockDim.x / 32);
    if (a.ell_vals) {
        // fused sliced-ELL gather: the SpMV operand's slices that start in this
        // subdomain's rows, before the level walk -- a bandwidth-bound copy
        // that overlaps the other resident CTA's latency-bound levels
        // (separate gather kernel: 3.20 ms per dd_refactor, fused: 3.15 ms;
        // spread over the warps idle in each level instead: 3.40 ms)
        const int64_t r0 = a.info[q].row0, r1 = r0 + a.info[q].nrows;
        const int64_t e0 = a.ell_slot_ptr[(r0 + 31) / 32], e1 = a.ell_slot_ptr[(r1 + 31) / 32];
        for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
            const int64_t sidx = __ldg(a.Esrc + e);
            if (sidx < 0) continue;
            const double *f = a.A + 9 * sidx;
            const int64_t ln = e & 31, eb = 9 * (e - ln);
            double x[9];
#pragma unroll
            for (int vv = 0; vv < 9; ++vv) x[vv] = __ldg(f + vv);
#pragma unroll
            for (int vv = 0; vv < 9; ++vv) a.ell_vals[eb + 32 * vv + ln] = x[vv];
        }
    }
    const int lev1 = a.SubLev[q + 1];
    for (int lev = a.SubLev[q]; lev < lev1; ++lev) {
        const int lo = a.LevPtr[lev], hi = a.LevPtr[lev + 1];
        for (int base = lo + 3 * warp; base < hi; base += per_pass) {
            const int idx = base + grp;
            const bool has = live && idx < hi;
            const int4 *P = reinterpret_cast<const int4 *>(plan + (size_t)RFD_PLAN_WORDS * (has ? idx : lo));
            const int4 p0 = __ldg(P), p1 = __ldg(P + 1), p2 = __ldg(P + 2), p3 = __ldg(P + 3);
            // p0: li, w0, dpos | upd-mask << 8, Lb; p1: k0, k1, k2, q0; p2: q1, q2, a0, a1;
            // p3: a2, aii, -, -  (q, a: the caller's blocks of U_ki, W_ik; aii: U_ii)
            const int li = p0.x, Lb = p0.w;
            const int dpos = has ? (p0.z & 255) : 0, upd = p0.z >> 8;
            const int kk[3] = {p1.x, p1.y, p1.z}, qq[3] = {p1.w, p2.x, p2.y}, aa[3] = {p2.z, p2.w, p3.x};
            double wik[3], dk[3], uki[3];
#pragma unroll
            for (int jp = 0; jp < 3; ++jp) {
                const bool ok = jp < dpos;
                wik[jp] = ok ? __ldg(a.A + 9 * (size_t)aa[jp] + v) : 0.0;
                dk[jp] = ok ? a.Dinv[9 * (size_t)kk[jp] + v] : 0.0;
                uki[jp] = ok && ((upd >> jp) & 1) ? __ldg(a.A + 9 * (size_t)qq[jp] + v) : 0.0;
            }
            double wii = has ? __ldg(a.A + 9 * (size_t)p3.y + v) : 0.0;
            int64_t loff[3];
            int32_t lst[3];
#pragma unroll
            for (int jp = 0; jp < 3; ++jp) {
                loff[jp] = jp < dpos ? a.Loff[Lb + jp] : 0;
                lst[jp] = jp < dpos ? a.Lst[Lb + jp] : 0;
            }
            const int dmax = warp_max(dpos);
            double Lk[3];
#pragma unroll
            for (int jp = 0; jp < 3; ++jp) {
                if (jp >= dmax) break;  // warp-uniform
                // L_ik = W_ik * U_kk^-1 (R12): rf_mul3(W, Dinv, L)
                const double wv = wik[jp], dv = dk[jp];
                Lk[jp] = __fma_rn(g9(wv, gbase, r3 + 2), g9(dv, gbase, 6 + c),
                                  __fma_rn(g9(wv, gbase, r3 + 1), g9(dv, gbase, 3 + c),
                                           g9(wv, gbase, r3) * g9(dv, gbase, c)));
                // U_ii -= L_ik U_ki: rf_sub_mul's order
                const double L = Lk[jp], uq = uki[jp];
                double nw = __fma_rn(-g9(L, gbase, r3), g9(uq, gbase, c), wii);
                nw = __fma_rn(-g9(L, gbase, r3 + 1), g9(uq, gbase, 3 + c), nw);
                nw = __fma_rn(-g9(L, gbase, r3 + 2), g9(uq, gbase, 6 + c), nw);
                if (jp < dpos && ((upd >> jp) & 1)) wii = nw;
            }
            // Dinv_i = inv(U_ii)
            double m[9], inv[9];
#pragma unroll
            for (int e = 0; e < 9; ++e) m[e] = g9(wii, gbase, e);
            const bool okinv = rf_inv3(m, a.floor_, inv);
            if (has) {
#pragma unroll
                for (int jp = 0; jp < 3; ++jp)
                    if (jp < dpos) *reinterpret_cast<double *>(a.slab + loff[jp] + (int64_t)lst[jp] * v) = Lk[jp];
                if (!okinv) {
                    if (v == 0) atomicMin(a.bad, (unsigned long long)(a.row_first + li));
                } else {
                    double mine = inv[0];
#pragma unroll
                    for (int e = 1; e < 9; ++e)
                        if (e == v) mine = inv[e];
                    a.Dinv[9 * (size_t)li + v] = mine;
                }
            }
        }
        __syncthreads();
    }
    rf_upass_rows<true>(a, q);
}

void launch_refactor_diag(int nsl, const RfArgs &a, const int32_t *plan, cudaStream_t st) {
    k_refactor_diag<<<nsl, RFD_THREADS, 0, st>>>(a, plan);
}

// to[q] = from[src[q]] for the W layout with nine lanes per block: a
// 288-thread CTA covers 32 consecutive blocks per tile, thread (b, v) moves
// element v of block b, so the stores are one contiguous 2304-byte run and each
// block's 72 bytes are read by one 9-lane group; four tiles per iteration keep
// their map and value loads in flight together. 160^3: 1.6 -> 0.78 ms
// (k_gather_blocks, one thread per block: 36 % of the DRAM peak; one tile per
// iteration: 1.48 ms, latency-bound)
__global__ void __launch_bounds__(288) k_gather_w9(int64_t n, const int32_t *__restrict__ src,
                                                   const double *__restrict__ from, double *__restrict__ to) {
    constexpr int U = 4;
    const int b = threadIdx.x / 9, v = threadIdx.x - 9 * (threadIdx.x / 9);
    for (int64_t q0 = 32 * U * (int64_t)blockIdx.x; q0 < n; q0 += 32 * U * (int64_t)gridDim.x) {
        int64_t sidx[U];
#pragma unroll
        for (int m = 0; m < U; ++m) {
            const int64_t q = q0 + 32 * m + b;
            sidx[m] = q < n ? __ldg(src + q) : -1;
        }
        double x[U];
#pragma unroll
        for (int m = 0; m < U; ++m) x[m] = sidx[m] >= 0 ? __ldg(from + 9 * sidx[m] + v) : 0.0;
#pragma unroll
        for (int m = 0; m < U; ++m)
            if (sidx[m] >= 0) to[9 * (q0 + 32 * m + b) + v] = x[m];
    }
}

void launch_gather_blocks(int64_t n, const int32_t *src, const double *from, double *to, int ell, int grid,
                          cudaStream_t st) {
    if (!ell) {
        k_gather_w9<<<grid, 288, 0, st>>>(n, src, from, to);
        return;
    }
    k_gather_blocks<<<grid, 256, 0, st>>>(n, src, from, to, ell);
}

// DD_REFACTOR_KERNEL=1: the round-1 kernel (one thread per row), for A/B
void launch_refactor(int nsl, const RfArgs &a, cudaStream_t st) {
    static const bool old = getenv("DD_REFACTOR_KERNEL") && atoi(getenv("DD_REFACTOR_KERNEL")) == 1;
    if (old)
        k_refactor<<<nsl, 128, 0, st>>>(a);
    else
        k_refactor9<<<nsl, RF9_THREADS, 0, st>>>(a);
}

}  // namespace ddk
