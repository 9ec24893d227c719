// apply.cu -- fused per-subdomain ILDU0 apply z = U_unit^-1 D^-1 L^-1 r.
//
// One CTA owns one subdomain at a time; the subdomain vector (8*bs*P bytes)
// lives in shared memory for the whole L -> D -> U sequence (sec. 4.4
// P:715-725; Alg. 6 P:582-615 with unit L per sec. 4.3). The
// factor slab is level-ordered and read exactly once.
//
// Kernels
//   k_apply_ring<RING,CH,SPIN>  persistent, warp-specialised: one producer
//       warp streams each subdomain's r slice and factor slab through a
//       shared-memory ring with 1-D bulk async copies (cp.async.bulk, UBLKCP)
//       and full/empty mbarriers; TC consumer threads run the sweeps.
//       SPIN=false: level sets, a CTA barrier between levels (Alg. 6).
//       SPIN=true : sync-free (Alg. 4 P:410-441 with per-row ready flags in
//                   shared memory, R17): each warp walks the same level-ordered
//                   records on its own and waits only on the flags of the rows
//                   it depends on -- no CTA barrier per level.
//   k_apply_direct              ablation: same records read straight from
//       global memory (the paper's "vector in LDS, factors from global"
//       design) with a bulk L2 prefetch running ahead.
//
// Arithmetic: lower row i, component c:
//   acc = r_ic; for blocks (j,B) ascending: for d: acc = fma(-B[c][d], z_jd, acc)
// D+U row i: y_c = D[c][0]*z_i0; y_c = fma(D[c][1], z_i1, y_c); y_c = fma(D[c][2], z_i2, y_c);
//   acc = y_c; for U blocks ascending: acc = fma(-B[c][d], x_jd, acc).
// Compiled with -fmad=false; every fma is explicit (__fma_rn).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "dd_internal.h"
#include "ptx.cuh"

// Branch-free K <= 3 record path for 3x3 rows (default): every lane runs the
// same instruction stream (no BSSY/BSYNC reconvergence per block). Round 1:
// absent blocks loaded from the record start and were replaced by zero values
// and a zero x with selects (404 -> 385 us at config 3). Round 2 (rec7): the
// descriptors name a zero slot of the shared vector for absent blocks and the
// values come from the record's zero count bytes 24..31, so no select is left
// and the negation folds into the DFMA; one straight-line instance per
// triangle (388 -> 354 us). fma(-0, 0, a) == a for every a: bitwise the same.
// DD_PRED=0 builds the branching form (ablation).
#ifndef DD_PRED
#define DD_PRED 1
#endif
// The same for scalar CSR rows (rec1): with selects the branch-free form was
// 5-8 % slower than branching (a row's block is one value); with the zero slot
// it is 3-5 % faster (tools/csr_bench.py). 0 keeps their branching form.
#ifndef DD_PRED1
#define DD_PRED1 1
#endif
// Branch-free inside each group of three of the general-K path (27-point
// rows): 27-point 96^3, P 2048: level set 723 -> 620 us, direct 713 -> 560 us.
#ifndef DD_PRED_GEN
#define DD_PRED_GEN 1
#endif

namespace ddk {

#ifdef DD_TRACE
// development instrumentation (-DDD_TRACE builds only): per-CTA cycle
// counters of the level-set ring kernel, and a subdomain remap (s -> s % submod)
// that makes every CTA stream an L2-resident working set
__device__ unsigned long long g_dd_trace[1024][16];
__device__ int g_dd_submod;
#define DD_SUB(s) (g_dd_submod > 0 ? (s) % g_dd_submod : (s))
#else
#define DD_SUB(s) (s)
#endif

using ddi::RecHdr;
using ddi::SubInfo;
// consumer threads = rows per record (Slab::rows_per_rec): 128 for 3x3 rows;
// 256 for scalar rows, whose per-row work is one short FMA chain, so a level
// needs fewer records (and barriers)
template <int BS>
constexpr int TCB = BS == 1 ? 256 : 128;

__host__ __device__ constexpr uint32_t al8(uint32_t x) { return (x + 7u) & ~7u; }

// shared-vector index of element q = bs*i + c of the subdomain (Swz)
template <int BS>
__device__ __forceinline__ uint32_t vslot(const ddi::Swz &sw, uint32_t q) {
    if constexpr (BS == 1) {
        return sw.slot(q);
    } else {
        const uint32_t i = q / 3u;
        return 3u * sw.slot(i) + (q - 3u * i);
    }
}

// ---- readers: map a byte offset inside the current record to data
struct GlobalRd {  // direct variant: the record in HBM
    const uint8_t *p;
    template <class T>
    __device__ __forceinline__ T ld(uint32_t off) const {
        return __ldg(reinterpret_cast<const T *>(p + off));
    }
};

struct LinRd {  // ring variant, record does not wrap: plain shared pointer
    const uint8_t *p;
    template <class T>
    __device__ __forceinline__ T ld(uint32_t off) const {
        return *reinterpret_cast<const T *>(p + off);
    }
};

template <uint32_t RING>
struct RingRd {  // ring variant, record wraps the ring end
    const uint8_t *ring;
    uint32_t base;  // absolute stream position of the record start
    template <class T>
    __device__ __forceinline__ T ld(uint32_t off) const {
        return *reinterpret_cast<const T *>(ring + ((base + off) & (RING - 1u)));
    }
};

// Sync-free variant: per-row ready bits in shared memory, one bitset for the
// L sweep and one for the U sweep of the current subdomain (cleared while
// the next subdomain's r slice is loaded). 1 bit per row and sweep keeps the
// flags at 512 B for P 2048, so two sync-free CTAs fit on an SM beside their
// 48 KB vectors and 64 KB rings (4-byte epochs needed 8 KB and forced one).
struct SpinFlags {
    uint32_t *L, *U;
};
// Watchdog: a row's dependencies are rows of earlier levels of the same CTA,
// so a wait can only outlast DD_SPIN_TIMEOUT_NS (default 2 s) if the slab is
// corrupt; the kernel then traps (the call fails with a launch error) instead
// of hanging the GPU. The clock is read once per 1024 polls.
#ifndef DD_SPIN_TIMEOUT_NS
#define DD_SPIN_TIMEOUT_NS 2000000000ull
#endif
__device__ __forceinline__ void spin_bit(const uint32_t *bits, uint32_t j) {
    uint32_t n = 0;
    unsigned long long t0 = 0;
    while (!((*reinterpret_cast<const volatile uint32_t *>(bits + (j >> 5)) >> (j & 31u)) & 1u)) {
        if ((++n & 1023u) == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t0 == 0)
                t0 = t;
            else if (t - t0 > DD_SPIN_TIMEOUT_NS)
                __trap();
        }
    }
    __threadfence_block();
}
__device__ __forceinline__ void set_bit(uint32_t *bits, uint32_t i) {
    __threadfence_block();
    atomicOr(bits + (i >> 5), 1u << (i & 31u));
}

// Process one record: thread t owns the t-th row of the record (t < w).
// Every load (descriptor, values, Dinv) is addressed from (t, cnt) alone, so
// all are in flight before the first FMA; the only dependent step is the
// gather of vec[3j..3j+2] through the descriptor's column ids.
// GEN: 0 = rows with at most 3 blocks per triangle only (7-point), 1 = general
// K with blocks in groups of three, 2 = general K one block per step
// NU (ILU0 ablation, DD_ILU0): the U records hold the non-unit upper blocks
// U_ij and the row's D = U_ii^-1 is applied AFTER its off-diagonal updates
// ("unlike ILU0 where scaling follows each row's off-diagonal updates",
// P:823): acc = z_i - sum U_ij x_j, x_i = D acc (orc_apply_ilu0's order).
#ifndef DD_R7_XFIRST
#define DD_R7_XFIRST 1
#endif
// The branch-free 7-point row (K <= 3 blocks per triangle, DD_PRED): one
// straight-line instance per triangle (UP), loads issued in dependency order
// -- the descriptor, then the gathers of x_j it names (the only dependent
// loads), the own row, the block values and (UP) Dinv -- all before the
// first FMA. Absent blocks: the descriptor names the zero slot (x = 0.0) and
// the values come from record bytes 24..31 (cnt[4..7], zero for K <= 3), an
// exact +0.0 with no select, so fma(-b, x, a) == a bitwise.
template <bool SPIN, bool UP, bool NU, class Rd>
__device__ __forceinline__ void rec7(const Rd &rd, const RecHdr &h, const uint4 &c8, int t, double *__restrict__ vec,
                                     SpinFlags F) {
    const uint32_t w = h.w;
    const uint2 d = rd.template ld<uint2>(32u + 8u * t);
    const uint32_t i = d.x & 0xffffu;
    const uint32_t col[3] = {d.x >> 16, d.y & 0xffffu, d.y >> 16};
    const uint32_t cnt[3] = {c8.x & 0xffffu, c8.x >> 16, c8.y & 0xffffu};
    double x[3][3];
    if constexpr (!SPIN && DD_R7_XFIRST) {
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int c = 0; c < 3; ++c) x[k][c] = vec[3 * col[k] + c];
    }
    if (SPIN && UP) spin_bit(F.L, i);  // own L result
    const double z0 = vec[3 * i], z1 = vec[3 * i + 1], z2 = vec[3 * i + 2];
    double b[3][9];
    uint32_t pre = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const bool ok = (uint32_t)t < cnt[k];
        const uint32_t vb = ok ? h.off_val + 72u * pre + 8u * t : 24u, st = ok ? 8u * cnt[k] : 0u;
#pragma unroll
        for (int v = 0; v < 9; ++v) b[k][v] = rd.template ld<double>(vb + st * v);
        pre += cnt[k];
    }
    double D[9];
    if constexpr (UP) {
        const uint32_t off_dinv = (47u + 8u * w) & ~15u;  // rec_off_dinv(K <= 3, w)
#pragma unroll
        for (int v = 0; v < 9; ++v) D[v] = rd.template ld<double>(off_dinv + 8u * (v * w + t));
    }
    if constexpr (SPIN || !DD_R7_XFIRST) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (SPIN && (uint32_t)t < cnt[k]) spin_bit(UP ? F.U : F.L, col[k]);
#pragma unroll
            for (int c = 0; c < 3; ++c) x[k][c] = vec[3 * col[k] + c];
        }
    }
    double a0, a1, a2;
    if (UP && !NU) {
        a0 = D[0] * z0;
        a0 = __fma_rn(D[1], z1, a0);
        a0 = __fma_rn(D[2], z2, a0);
        a1 = D[3] * z0;
        a1 = __fma_rn(D[4], z1, a1);
        a1 = __fma_rn(D[5], z2, a1);
        a2 = D[6] * z0;
        a2 = __fma_rn(D[7], z1, a2);
        a2 = __fma_rn(D[8], z2, a2);
    } else {
        a0 = z0;
        a1 = z1;
        a2 = z2;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a0 = __fma_rn(-b[k][0], x[k][0], a0);
        a0 = __fma_rn(-b[k][1], x[k][1], a0);
        a0 = __fma_rn(-b[k][2], x[k][2], a0);
        a1 = __fma_rn(-b[k][3], x[k][0], a1);
        a1 = __fma_rn(-b[k][4], x[k][1], a1);
        a1 = __fma_rn(-b[k][5], x[k][2], a1);
        a2 = __fma_rn(-b[k][6], x[k][0], a2);
        a2 = __fma_rn(-b[k][7], x[k][1], a2);
        a2 = __fma_rn(-b[k][8], x[k][2], a2);
    }
    if (UP && NU) {
        const double q0 = a0, q1 = a1, q2 = a2;
        a0 = D[0] * q0;
        a0 = __fma_rn(D[1], q1, a0);
        a0 = __fma_rn(D[2], q2, a0);
        a1 = D[3] * q0;
        a1 = __fma_rn(D[4], q1, a1);
        a1 = __fma_rn(D[5], q2, a1);
        a2 = D[6] * q0;
        a2 = __fma_rn(D[7], q1, a2);
        a2 = __fma_rn(D[8], q2, a2);
    }
    vec[3 * i] = a0;
    vec[3 * i + 1] = a1;
    vec[3 * i + 2] = a2;
    if (SPIN) set_bit(UP ? F.U : F.L, i);
}

template <bool SPIN, int GEN, class Rd, bool NU = false>
__device__ __forceinline__ void process_record3(const Rd &rd, const RecHdr &h, const uint4 &c8, int t,
                                                double *__restrict__ vec, SpinFlags F) {
    const uint32_t w = h.w, K = h.K;
    if (t >= (int)w) return;
    const bool upper = (h.flags & ddi::REC_UPPER) != 0;
    const uint32_t off_desc = ddi::rec_off_desc(K);
    const uint32_t off_dinv = ddi::rec_off_dinv(K, w);
    const uint32_t off_val = h.off_val;
#if DD_PRED
    // ring readers: the per-triangle instance; the direct ablation (GlobalRd,
    // values straight from HBM/L2) keeps the one-instance form below, whose
    // schedule issues the value loads first (rec7 there: 461 -> 712 us)
    if (!std::is_same<Rd, GlobalRd>::value && (GEN == 0 || K <= 3)) {
        if (upper)
            rec7<SPIN, true, NU>(rd, h, c8, t, vec, F);
        else
            rec7<SPIN, false, NU>(rd, h, c8, t, vec, F);
        return;
    }
#endif
    constexpr bool SEL = std::is_same<Rd, GlobalRd>::value;
    if (GEN == 0 || K <= 3) {
        // K <= 3: the descriptors start at byte 32, Dinv after them at a
        // 16-byte boundary, and cnt[k] is 0 for k >= K (zeroed count area)
        const uint2 d = rd.template ld<uint2>(32u + 8u * t);
        const uint32_t i = d.x & 0xffffu;
        const uint32_t col[3] = {d.x >> 16, d.y & 0xffffu, d.y >> 16};
        const uint32_t cnt[3] = {c8.x & 0xffffu, c8.x >> 16, c8.y & 0xffffu};
        const uint32_t off_dinv = (47u + 8u * w) & ~15u;
        double b[3][9];
        uint32_t pre = 0;
#if DD_PRED
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            // absent block: nine loads of record bytes 24..31 (cnt[4..7], zero
            // for K <= 3), an exact +0.0 -- no select, and the negation folds
            // into the DFMA. The direct ablation (GlobalRd) keeps the round-1
            // selects: without them ptxas schedules its global loads worse
            // (474 -> 616 us at config 3)
            const bool ok = (uint32_t)t < cnt[k];
            const uint32_t vb = ok ? off_val + 72u * pre + 8u * t : (SEL ? 0u : 24u), st = ok ? 8u * cnt[k] : 0u;
#pragma unroll
            for (int v = 0; v < 9; ++v) {
                const double q = rd.template ld<double>(vb + st * v);
                b[k][v] = SEL ? (ok ? q : 0.0) : q;
            }
            pre += cnt[k];
        }
#else
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if ((uint32_t)t < cnt[k]) {
                const uint32_t vb = off_val + 72u * pre + 8u * t, st = 8u * cnt[k];
#pragma unroll
                for (int v = 0; v < 9; ++v) b[k][v] = rd.template ld<double>(vb + st * v);
            }
            pre += cnt[k];
        }
#endif
        double a0, a1, a2;
        double D[9];
        if (upper) {
#pragma unroll
            for (int v = 0; v < 9; ++v) D[v] = rd.template ld<double>(off_dinv + 8u * (v * w + t));
            if (SPIN) spin_bit(F.L, i);  // own L result
            const double z0 = vec[3 * i], z1 = vec[3 * i + 1], z2 = vec[3 * i + 2];
            if (NU) {
                a0 = z0;
                a1 = z1;
                a2 = z2;
            } else {
                a0 = D[0] * z0;
                a0 = __fma_rn(D[1], z1, a0);
                a0 = __fma_rn(D[2], z2, a0);
                a1 = D[3] * z0;
                a1 = __fma_rn(D[4], z1, a1);
                a1 = __fma_rn(D[5], z2, a1);
                a2 = D[6] * z0;
                a2 = __fma_rn(D[7], z1, a2);
                a2 = __fma_rn(D[8], z2, a2);
            }
        } else {
            a0 = vec[3 * i];
            a1 = vec[3 * i + 1];
            a2 = vec[3 * i + 2];
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
#if DD_PRED
            {
                // absent block: the descriptor names the zero slot (x = 0.0,
                // b = +0.0: fma(-0, 0, a) == a for every a)
                const bool ok = (uint32_t)t < cnt[k];
                const uint32_t j = SEL && !ok ? i : col[k];
                if (SPIN && ok) spin_bit(upper ? F.U : F.L, j);
                const double y0 = vec[3 * j], y1 = vec[3 * j + 1], y2 = vec[3 * j + 2];
                const double x0 = SEL && !ok ? 0.0 : y0, x1 = SEL && !ok ? 0.0 : y1, x2 = SEL && !ok ? 0.0 : y2;
#else
            if ((uint32_t)t < cnt[k]) {
                const uint32_t j = col[k];
                if (SPIN) spin_bit(upper ? F.U : F.L, j);
                const double x0 = vec[3 * j], x1 = vec[3 * j + 1], x2 = vec[3 * j + 2];
#endif
                a0 = __fma_rn(-b[k][0], x0, a0);
                a0 = __fma_rn(-b[k][1], x1, a0);
                a0 = __fma_rn(-b[k][2], x2, a0);
                a1 = __fma_rn(-b[k][3], x0, a1);
                a1 = __fma_rn(-b[k][4], x1, a1);
                a1 = __fma_rn(-b[k][5], x2, a1);
                a2 = __fma_rn(-b[k][6], x0, a2);
                a2 = __fma_rn(-b[k][7], x1, a2);
                a2 = __fma_rn(-b[k][8], x2, a2);
            }
        }
        if (NU && upper) {
            const double q0 = a0, q1 = a1, q2 = a2;
            a0 = D[0] * q0;
            a0 = __fma_rn(D[1], q1, a0);
            a0 = __fma_rn(D[2], q2, a0);
            a1 = D[3] * q0;
            a1 = __fma_rn(D[4], q1, a1);
            a1 = __fma_rn(D[5], q2, a1);
            a2 = D[6] * q0;
            a2 = __fma_rn(D[7], q1, a2);
            a2 = __fma_rn(D[8], q2, a2);
        }
        vec[3 * i] = a0;
        vec[3 * i + 1] = a1;
        vec[3 * i + 2] = a2;
        if (SPIN) set_bit(upper ? F.U : F.L, i);
        return;
    }
    // ---- general K (> 3): descriptor of rec_dw(K) bytes, loop over k. Compiled
    // only into the GEN kernels (slabs with more than 3 blocks per row in a
    // triangle): it needs more registers than the 7-point path.
    if constexpr (GEN) {
    const uint32_t dw = ddi::rec_dw(K);
    const uint32_t i = rd.template ld<uint16_t>(off_desc + dw * t);
    double a0, a1, a2;
    double D[9];
    if (upper && NU) {
#pragma unroll
        for (int v = 0; v < 9; ++v) D[v] = rd.template ld<double>(off_dinv + 8u * (v * w + t));
        a0 = vec[3 * i];
        a1 = vec[3 * i + 1];
        a2 = vec[3 * i + 2];
    } else if (upper) {
#pragma unroll
        for (int v = 0; v < 9; ++v) D[v] = rd.template ld<double>(off_dinv + 8u * (v * w + t));
        if (SPIN) spin_bit(F.L, i);  // own L result
        const double z0 = vec[3 * i], z1 = vec[3 * i + 1], z2 = vec[3 * i + 2];
        a0 = D[0] * z0;
        a0 = __fma_rn(D[1], z1, a0);
        a0 = __fma_rn(D[2], z2, a0);
        a1 = D[3] * z0;
        a1 = __fma_rn(D[4], z1, a1);
        a1 = __fma_rn(D[5], z2, a1);
        a2 = D[6] * z0;
        a2 = __fma_rn(D[7], z1, a2);
        a2 = __fma_rn(D[8], z2, a2);
    } else {
        a0 = vec[3 * i];
        a1 = vec[3 * i + 1];
        a2 = vec[3 * i + 2];
    }
    if constexpr (GEN == 2) {
        // one block per step (fewer registers; the direct variant keeps this form)
    uint32_t pre = 0;
    for (uint32_t k = 0; k < K; ++k) {
        const uint32_t ck = rd.template ld<uint16_t>(16u + 2u * k);
        if ((uint32_t)t >= ck) break;
        const uint32_t j = rd.template ld<uint16_t>(off_desc + dw * t + 2u * (1u + k));
        const uint32_t vb = off_val + 72u * pre + 8u * t;
        double b[9];
#pragma unroll
        for (int v = 0; v < 9; ++v) b[v] = rd.template ld<double>(vb + 8u * ck * v);
        if (SPIN) spin_bit(upper ? F.U : F.L, j);
        const double x0 = vec[3 * j], x1 = vec[3 * j + 1], x2 = vec[3 * j + 2];
        a0 = __fma_rn(-b[0], x0, a0);
        a0 = __fma_rn(-b[1], x1, a0);
        a0 = __fma_rn(-b[2], x2, a0);
        a1 = __fma_rn(-b[3], x0, a1);
        a1 = __fma_rn(-b[4], x1, a1);
        a1 = __fma_rn(-b[5], x2, a1);
        a2 = __fma_rn(-b[6], x0, a2);
        a2 = __fma_rn(-b[7], x1, a2);
        a2 = __fma_rn(-b[8], x2, a2);
        pre += ck;
    }
    } else {
    // blocks in groups of three: a group's counts, columns and values are all
    // loaded before its FMAs (as in the K <= 3 path), so a row with K blocks
    // has ceil(K/3) dependent load rounds instead of K
    uint32_t pre = 0;
    for (uint32_t k0 = 0; k0 < K; k0 += 3) {
        uint32_t ck[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const uint32_t k = k0 + q;
            ck[q] = k < K ? rd.template ld<uint16_t>(16u + 2u * k) : 0u;
        }
        if ((uint32_t)t >= ck[0]) break;  // rows sorted by block count: none further
        uint32_t j[3];
        double b[3][9];
        uint32_t pq = pre;
#if DD_PRED_GEN
        // branch-free inside a group (as in the K <= 3 path): absent blocks
        // are a zero block times a zero x
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const bool ok = (uint32_t)t < ck[q];
            j[q] = ok ? rd.template ld<uint16_t>(off_desc + dw * t + 2u * (1u + k0 + q)) : i;
            const uint32_t vb = ok ? off_val + 72u * pq + 8u * t : 0u, st = ok ? 8u * ck[q] : 0u;
#pragma unroll
            for (int v = 0; v < 9; ++v) {
                const double w = rd.template ld<double>(vb + st * v);
                b[q][v] = ok ? w : 0.0;
            }
            pq += ck[q];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            {
                const bool ok = (uint32_t)t < ck[q];
                if (SPIN && ok) spin_bit(upper ? F.U : F.L, j[q]);
                const double y0 = vec[3 * j[q]], y1 = vec[3 * j[q] + 1], y2 = vec[3 * j[q] + 2];
                const double x0 = ok ? y0 : 0.0, x1 = ok ? y1 : 0.0, x2 = ok ? y2 : 0.0;
#else
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            if ((uint32_t)t < ck[q]) {
                j[q] = rd.template ld<uint16_t>(off_desc + dw * t + 2u * (1u + k0 + q));
                const uint32_t vb = off_val + 72u * pq + 8u * t;
#pragma unroll
                for (int v = 0; v < 9; ++v) b[q][v] = rd.template ld<double>(vb + 8u * ck[q] * v);
            }
            pq += ck[q];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            if ((uint32_t)t < ck[q]) {
                if (SPIN) spin_bit(upper ? F.U : F.L, j[q]);
                const double x0 = vec[3 * j[q]], x1 = vec[3 * j[q] + 1], x2 = vec[3 * j[q] + 2];
#endif
                a0 = __fma_rn(-b[q][0], x0, a0);
                a0 = __fma_rn(-b[q][1], x1, a0);
                a0 = __fma_rn(-b[q][2], x2, a0);
                a1 = __fma_rn(-b[q][3], x0, a1);
                a1 = __fma_rn(-b[q][4], x1, a1);
                a1 = __fma_rn(-b[q][5], x2, a1);
                a2 = __fma_rn(-b[q][6], x0, a2);
                a2 = __fma_rn(-b[q][7], x1, a2);
                a2 = __fma_rn(-b[q][8], x2, a2);
            }
        }
        pre = pq;
    }
    }
    if (NU && upper) {
        const double q0 = a0, q1 = a1, q2 = a2;
        a0 = D[0] * q0;
        a0 = __fma_rn(D[1], q1, a0);
        a0 = __fma_rn(D[2], q2, a0);
        a1 = D[3] * q0;
        a1 = __fma_rn(D[4], q1, a1);
        a1 = __fma_rn(D[5], q2, a1);
        a2 = D[6] * q0;
        a2 = __fma_rn(D[7], q1, a2);
        a2 = __fma_rn(D[8], q2, a2);
    }
    vec[3 * i] = a0;
    vec[3 * i + 1] = a1;
    vec[3 * i + 2] = a2;
    if (SPIN) set_bit(upper ? F.U : F.L, i);
    }
}

// The scalar row with K <= 3 blocks per triangle, branch-free (ring readers):
// absent blocks read the zero slot (x = 0.0) and the zero count bytes 24..31
// (b = +0.0), as in rec7; one straight-line instance per triangle.
template <bool SPIN, bool UP, class Rd>
__device__ __forceinline__ void rec1(const Rd &rd, const RecHdr &h, const uint4 &c8, int t, double *__restrict__ vec,
                                     SpinFlags F) {
    const uint32_t w = h.w;
    const uint2 d = rd.template ld<uint2>(32u + 8u * t);
    const uint32_t i = d.x & 0xffffu;
    const uint32_t col[3] = {d.x >> 16, d.y & 0xffffu, d.y >> 16};
    const uint32_t cnt[3] = {c8.x & 0xffffu, c8.x >> 16, c8.y & 0xffffu};
    double x[3];
    if constexpr (!SPIN) {
#pragma unroll
        for (int k = 0; k < 3; ++k) x[k] = vec[col[k]];
    }
    if (SPIN && UP) spin_bit(F.L, i);
    const double z = vec[i];
    double b[3];
    uint32_t pre = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        b[k] = rd.template ld<double>((uint32_t)t < cnt[k] ? h.off_val + 8u * (pre + t) : 24u);
        pre += cnt[k];
    }
    double a = z;
    if constexpr (UP) a = rd.template ld<double>(((47u + 8u * w) & ~15u) + 8u * t) * z;
    if constexpr (SPIN) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if ((uint32_t)t < cnt[k]) spin_bit(UP ? F.U : F.L, col[k]);
            x[k] = vec[col[k]];
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) a = __fma_rn(-b[k], x[k], a);
    vec[i] = a;
    if (SPIN) set_bit(UP ? F.U : F.L, i);
}

// Scalar CSR rows: the same record walk with 1x1 blocks --
// one value plane per k, one Dinv plane, one FMA chain per row
// (lower: acc = r_i, fma(-l_ij, z_j, acc); upper: acc = dinv_i * z_i,
// fma(-u_ij, x_j, acc); blocks ascending).
template <bool SPIN, int GEN, class Rd>
__device__ __forceinline__ void process_record1(const Rd &rd, const RecHdr &h, const uint4 &c8, int t,
                                                double *__restrict__ vec, SpinFlags F) {
    const uint32_t w = h.w, K = h.K;
    if (t >= (int)w) return;
    const bool upper = (h.flags & ddi::REC_UPPER) != 0;
    const uint32_t off_desc = ddi::rec_off_desc(K);
    const uint32_t off_dinv = ddi::rec_off_dinv(K, w);
    const uint32_t off_val = h.off_val;
#if DD_PRED1
    if (!std::is_same<Rd, GlobalRd>::value && (GEN == 0 || K <= 3)) {
        if (upper)
            rec1<SPIN, true>(rd, h, c8, t, vec, F);
        else
            rec1<SPIN, false>(rd, h, c8, t, vec, F);
        return;
    }
#endif
    if (GEN == 0 || K <= 3) {
        const uint2 d = rd.template ld<uint2>(off_desc + 8u * t);
        const uint32_t i = d.x & 0xffffu;
        const uint32_t col[3] = {d.x >> 16, d.y & 0xffffu, d.y >> 16};
        const uint32_t cnt[3] = {K > 0 ? (c8.x & 0xffffu) : 0u, K > 1 ? (c8.x >> 16) : 0u, K > 2 ? (c8.y & 0xffffu) : 0u};
        double b[3];
        uint32_t pre = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if ((uint32_t)t < cnt[k]) b[k] = rd.template ld<double>(off_val + 8u * (pre + t));
            pre += cnt[k];
        }
        double a;
        if (upper) {
            const double D = rd.template ld<double>(off_dinv + 8u * t);
            if (SPIN) spin_bit(F.L, i);
            a = D * vec[i];
        } else {
            a = vec[i];
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if ((uint32_t)t < cnt[k]) {
                const uint32_t j = col[k];
                if (SPIN) spin_bit(upper ? F.U : F.L, j);
                a = __fma_rn(-b[k], vec[j], a);
            }
        }
        vec[i] = a;
        if (SPIN) set_bit(upper ? F.U : F.L, i);
        return;
    }
    if constexpr (GEN) {
    const uint32_t dw = ddi::rec_dw(K);
    const uint32_t i = rd.template ld<uint16_t>(off_desc + dw * t);
    double a;
    if (upper) {
        const double D = rd.template ld<double>(off_dinv + 8u * t);
        if (SPIN) spin_bit(F.L, i);
        a = D * vec[i];
    } else {
        a = vec[i];
    }
    uint32_t pre = 0;
    for (uint32_t k0 = 0; k0 < K; k0 += 4) {  // groups of four, loads first (see process_record3)
        uint32_t ck[4], j[4];
        double b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) ck[q] = k0 + q < K ? rd.template ld<uint16_t>(16u + 2u * (k0 + q)) : 0u;
        if ((uint32_t)t >= ck[0]) break;
        uint32_t pq = pre;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if ((uint32_t)t < ck[q]) {
                j[q] = rd.template ld<uint16_t>(off_desc + dw * t + 2u * (1u + k0 + q));
                b[q] = rd.template ld<double>(off_val + 8u * (pq + t));
            }
            pq += ck[q];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if ((uint32_t)t < ck[q]) {
                if (SPIN) spin_bit(upper ? F.U : F.L, j[q]);
                a = __fma_rn(-b[q], vec[j[q]], a);
            }
        }
        pre = pq;
    }
    vec[i] = a;
    if (SPIN) set_bit(upper ? F.U : F.L, i);
    }
}

template <int BS, bool SPIN, int GEN, class Rd, bool NU = false>
__device__ __forceinline__ void process_record(const Rd &rd, const RecHdr &h, const uint4 &c8, int t,
                                               double *__restrict__ vec, SpinFlags F) {
    if constexpr (BS == 3)
        process_record3<SPIN, GEN, Rd, NU>(rd, h, c8, t, vec, F);
    else
        process_record1<SPIN, GEN>(rd, h, c8, t, vec, F);
}

// Tree-shuffle record (ablation, R19/R42; the paper's row-parallel design,
// P:409 "threads within a wavefront process the row's nonzero columns in
// parallel"): a group of 4 lanes per row, lane k forms the products of the
// row's blocks k, k+4, ... (p = B x_j, one FMA chain per component), the 4
// partial sums meet in a fixed shuffle tree ((l0+l1)+(l2+l3)), and lane 0
// writes x_i = a_i - S with a_i = z_i (L) or D_i z_i (U). Deterministic but a
// different summation order than the oracle's chain: 1e-10 bar, not bitwise.
// 32 rows per pass, ceil(w / 32) passes per record; all lanes take part in
// every shuffle.
template <int GEN, class Rd>
__device__ __forceinline__ void process_record_tree(const Rd &rd, const RecHdr &h, const uint4 &c8, int t, int TC,
                                                    double *vec) {
    const uint32_t w = h.w, K = h.K;
    const bool upper = (h.flags & ddi::REC_UPPER) != 0;
    const uint32_t off_desc = ddi::rec_off_desc(K), dw = ddi::rec_dw(K);
    const uint32_t off_dinv = ddi::rec_off_dinv(K, w);
    const uint32_t lk = (uint32_t)t & 3u;
    for (uint32_t r0 = 0; r0 < w; r0 += (uint32_t)TC / 4u) {
        const uint32_t r = r0 + (uint32_t)t / 4u;
        const bool row_ok = r < w;
        double p0 = 0.0, p1 = 0.0, p2 = 0.0;
        uint32_t i = 0;
        if (row_ok) {
            i = rd.template ld<uint16_t>(off_desc + dw * r);
            uint32_t pre = 0;
            for (uint32_t k = 0; k < K; ++k) {
                const uint32_t ck = (GEN == 0 || K <= 3) ? (k == 0 ? (c8.x & 0xffffu) : k == 1 ? (c8.x >> 16) : (c8.y & 0xffffu))
                                                          : rd.template ld<uint16_t>(16u + 2u * k);
                if (r >= ck) break;  // rows sorted by block count: no block k or later
                if ((k & 3u) == lk) {
                    const uint32_t j = rd.template ld<uint16_t>(off_desc + dw * r + 2u * (1u + k));
                    const uint32_t vb = h.off_val + 72u * pre + 8u * r, st = 8u * ck;
                    double b[9];
#pragma unroll
                    for (int v = 0; v < 9; ++v) b[v] = rd.template ld<double>(vb + st * v);
                    const double x0 = vec[3 * j], x1 = vec[3 * j + 1], x2 = vec[3 * j + 2];
                    p0 = __fma_rn(b[0], x0, p0);
                    p0 = __fma_rn(b[1], x1, p0);
                    p0 = __fma_rn(b[2], x2, p0);
                    p1 = __fma_rn(b[3], x0, p1);
                    p1 = __fma_rn(b[4], x1, p1);
                    p1 = __fma_rn(b[5], x2, p1);
                    p2 = __fma_rn(b[6], x0, p2);
                    p2 = __fma_rn(b[7], x1, p2);
                    p2 = __fma_rn(b[8], x2, p2);
                }
                pre += ck;
            }
        }
        p0 += __shfl_xor_sync(0xffffffffu, p0, 1);
        p1 += __shfl_xor_sync(0xffffffffu, p1, 1);
        p2 += __shfl_xor_sync(0xffffffffu, p2, 1);
        p0 += __shfl_xor_sync(0xffffffffu, p0, 2);
        p1 += __shfl_xor_sync(0xffffffffu, p1, 2);
        p2 += __shfl_xor_sync(0xffffffffu, p2, 2);
        if (row_ok && lk == 0) {
            double a0 = vec[3 * i], a1 = vec[3 * i + 1], a2 = vec[3 * i + 2];
            if (upper) {
                double D[9];
#pragma unroll
                for (int v = 0; v < 9; ++v) D[v] = rd.template ld<double>(off_dinv + 8u * (v * w + r));
                const double z0 = a0, z1 = a1, z2 = a2;
                a0 = D[0] * z0;
                a0 = __fma_rn(D[1], z1, a0);
                a0 = __fma_rn(D[2], z2, a0);
                a1 = D[3] * z0;
                a1 = __fma_rn(D[4], z1, a1);
                a1 = __fma_rn(D[5], z2, a1);
                a2 = D[6] * z0;
                a2 = __fma_rn(D[7], z1, a2);
                a2 = __fma_rn(D[8], z2, a2);
            }
            vec[3 * i] = a0 - p0;
            vec[3 * i + 1] = a1 - p1;
            vec[3 * i + 2] = a2 - p2;
        }
    }
}

// Edge-centric record (dag_ec_*, Table 3/4 ablation, BSR3): the
// record's nnz blocks are spread over the TC consumer threads (block e of
// the jagged planes: k = the plane it falls in, row slot t = e - prefix_k),
// each thread forms p = B x_j with its own FMA chain and subtracts it from
// vec[i] with a shared-memory (or global) atomicAdd -- the order of the
// atomics is not fixed, so results differ from the oracle in the last bits
// (R19) and BiCGSTAB iteration counts may vary. An L record needs
// no other step (vec[i] holds r_i, lower levels are final); a U record first
// scales its rows, y_i = D_i z_i (one thread per row), then a barrier, then
// the edges. bar() synchronises the consumer threads.
template <int GEN, class Rd, class Bar>
__device__ __forceinline__ void process_record_ec(const Rd &rd, const RecHdr &h, const uint4 &c8, int t, int TC,
                                                  double *vec, Bar &&bar) {
    const uint32_t w = h.w, K = h.K, nnz = h.nnz;
    const bool upper = (h.flags & ddi::REC_UPPER) != 0;
    const uint32_t off_desc = ddi::rec_off_desc(K);
    const uint32_t dw = ddi::rec_dw(K);
    if (upper) {
        const uint32_t off_dinv = ddi::rec_off_dinv(K, w);
        for (uint32_t r = t; r < w; r += TC) {
            const uint32_t i = rd.template ld<uint16_t>(off_desc + dw * r);
            double D[9];
#pragma unroll
            for (int v = 0; v < 9; ++v) D[v] = rd.template ld<double>(off_dinv + 8u * (v * w + r));
            const double z0 = vec[3 * i], z1 = vec[3 * i + 1], z2 = vec[3 * i + 2];
            double a0 = D[0] * z0;
            a0 = __fma_rn(D[1], z1, a0);
            a0 = __fma_rn(D[2], z2, a0);
            double a1 = D[3] * z0;
            a1 = __fma_rn(D[4], z1, a1);
            a1 = __fma_rn(D[5], z2, a1);
            double a2 = D[6] * z0;
            a2 = __fma_rn(D[7], z1, a2);
            a2 = __fma_rn(D[8], z2, a2);
            vec[3 * i] = a0;
            vec[3 * i + 1] = a1;
            vec[3 * i + 2] = a2;
        }
        bar();
    }
    for (uint32_t e = t; e < nnz; e += TC) {
        // plane k of edge e (rows sorted by block count: planes shrink)
        uint32_t k = 0, pre = 0, ck = 0;
        if (GEN == 0 || K <= 3) {
            const uint32_t c0 = c8.x & 0xffffu, c1 = K > 1 ? (c8.x >> 16) : 0u, c2 = K > 2 ? (c8.y & 0xffffu) : 0u;
            if (e >= c0 + c1) {
                k = 2, pre = c0 + c1, ck = c2;
            } else if (e >= c0) {
                k = 1, pre = c0, ck = c1;
            } else {
                k = 0, pre = 0, ck = c0;
            }
        } else {
            for (;; ++k) {
                ck = rd.template ld<uint16_t>(16u + 2u * k);
                if (e < pre + ck) break;
                pre += ck;
            }
        }
        const uint32_t r = e - pre;
        const uint32_t i = rd.template ld<uint16_t>(off_desc + dw * r);
        const uint32_t j = rd.template ld<uint16_t>(off_desc + dw * r + 2u * (1u + k));
        const uint32_t vb = h.off_val + 72u * pre + 8u * r, st = 8u * ck;
        double b[9];
#pragma unroll
        for (int v = 0; v < 9; ++v) b[v] = rd.template ld<double>(vb + st * v);
        const double x0 = vec[3 * j], x1 = vec[3 * j + 1], x2 = vec[3 * j + 2];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double p = b[3 * c] * x0;
            p = __fma_rn(b[3 * c + 1], x1, p);
            p = __fma_rn(b[3 * c + 2], x2, p);
            atomicAdd(vec + 3 * i + c, -p);
        }
    }
}

__device__ __forceinline__ RecHdr hdr_from(uint4 q) {
    RecHdr h;
    h.w = (uint16_t)(q.x & 0xffffu);
    h.K = (uint16_t)(q.x >> 16);
    h.flags = (uint16_t)(q.y & 0xffffu);
    h.nnz = (uint16_t)(q.y >> 16);
    h.bytes = q.z;
    h.off_val = q.w;
    return h;
}

// ------------------------------------------------------------------ direct
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Ablation: level-set sweep reading the records straight from global memory;
// only the vector lives in shared memory (so more CTAs fit per SM). Thread 0
// keeps a bulk L2 prefetch pf_bytes ahead of the record being processed.
// MODE 0: vertex-centric ILDU0 (Alg. 6); 1: edge-centric with atomics
// (process_record_ec); 2: vertex-centric ILU0 with the non-unit U (NU).
// VECG: the vector lives in GLOBAL memory (z itself, initialised from r):
// with MODE 1 the paper's dag_ec_no_lds (Table 3), global atomics.
// phase 1: the lower sweep alone (z = L^-1 r, Table 3's lower solve).
enum : int { AM_VC = 0, AM_EC = 1, AM_NU = 2, AM_TREE = 3 };
template <int BS, int GEN, int MODE = AM_VC, bool VECG = false>
__global__ void __launch_bounds__(TCB<BS>) k_apply_direct(const uint8_t *__restrict__ slab,
                                                     const SubInfo *__restrict__ info, int n_sub,
                                                     const double *__restrict__ r, double *__restrict__ z,
                                                     uint32_t pf_bytes, const int *skip, int phase, ddi::Swz sw,
                                                     double *__restrict__ gvec, int vec_rows) {
    // inside dd_bicgstab: skip (uniformly) once the solver has stopped
    if (skip && *reinterpret_cast<const volatile int *>(skip) != 0) return;
    extern __shared__ __align__(128) uint8_t smem[];
    const int t = threadIdx.x;
    for (int s = blockIdx.x; s < n_sub; s += gridDim.x) {
        const SubInfo si = info[s];
        const uint8_t *base = slab + si.stream_off;
        const uint32_t sz = phase == 1 ? (uint32_t)si.u_off : (uint32_t)si.stream_bytes;
        // VECG: the vector in global memory, in the slot layout of the
        // descriptors (one vec_rows-row region per subdomain of gvec)
        double *vec = VECG ? gvec + BS * (int64_t)s * vec_rows : reinterpret_cast<double *>(smem);
        uint32_t pf = 0;
        if (t == 0 && pf_bytes) {
            pf = min(sz, pf_bytes);
            prefetch_l2(base, pf);
        }
        const int nd = BS * si.nrows;
        const double *rs = r + BS * (int64_t)si.row0;
        for (int q = t; q < nd; q += TCB<BS>) vec[vslot<BS>(sw, q)] = __ldg(rs + q);
        if (t < BS) vec[BS * sw.zslot + t] = 0.0;  // the zero slot
        __syncthreads();
        uint32_t ro = 0;
        while (ro < sz) {
            const uint8_t *p = base + ro;
            const RecHdr h = hdr_from(__ldg(reinterpret_cast<const uint4 *>(p)));
            const uint4 c8 = __ldg(reinterpret_cast<const uint4 *>(p) + 1);
            if (t == 0 && pf_bytes && pf < sz && pf < ro + pf_bytes) {
                const uint32_t e = min(sz, ro + h.bytes + pf_bytes);
                prefetch_l2(base + pf, e - pf);
                pf = e;
            }
            const bool last = (h.flags & ddi::REC_LAST) != 0 || ro + h.bytes >= sz;
            // L level 0 carries no blocks (z_i = r_i in place): no work, no barrier
            const bool skip = !(h.flags & ddi::REC_UPPER) && h.K == 0 && !last;
            if (!skip) {
                if constexpr (MODE == AM_EC) {
                    if constexpr (BS == 3)
                        process_record_ec<GEN>(GlobalRd{p}, h, c8, t, TCB<BS>, vec, [] { __syncthreads(); });
                } else {
                    process_record<BS, false, GEN, GlobalRd, MODE == AM_NU>(GlobalRd{p}, h, c8, t, vec,
                                                                            SpinFlags{nullptr, nullptr});
                }
                __syncthreads();
            }
            ro += h.bytes;
            if (last) break;
        }
        // thread t stores the entries it fills for the next subdomain: no barrier
        double *zs = z + BS * (int64_t)si.row0;
        for (int q = t; q < nd; q += TCB<BS>) zs[q] = vec[vslot<BS>(sw, q)];
    }
}

// -------------------------------------------------------------------- ring
#ifndef DD_CH_DIV
#define DD_CH_DIV 4  // ring chunk = RING / DD_CH_DIV
#endif
#ifndef DD_PF_AHEAD
#define DD_PF_AHEAD -1  // L2 prefetch distance of the ring producer: -1 = half a ring, 0 = off, else bytes
#endif
// SPIN = false (level set, Alg. 6): every consumer thread takes one row of
//   each record; a named barrier separates records (levels).
// SPIN = true  (sync-free, Alg. 4 with per-row ready flags): each warp walks
//   the records on its own (rows 32w..32w+31 of each), waiting only on the
//   ready flags of its dependencies; records are in level (topological) order
//   so the warps pipeline levels. Ring chunks are released per warp (empty
//   barriers count NW arrivals).
// mode 1 (DD_APPLY_MODE=1, measurement only): consumers skip the arithmetic --
//   the streaming ceiling of the ring; mode 2: chunks are handed back as they
//   land (no record walk) -- the raw stream.
template <int BS, uint32_t RING, uint32_t CH, bool SPIN, int GEN, int MODE = AM_VC>
__global__ void __launch_bounds__(TCB<BS> + 32, 1)
    k_apply_ring(const uint8_t *__restrict__ slab, const SubInfo *__restrict__ info, int n_sub,
                 const double *__restrict__ r, double *__restrict__ z, int vec_bytes, int mode, const int *skip,
                 int phase, ddi::HaloOut ho, ddi::Swz sw) {
    // inside dd_bicgstab: skip (uniformly, before any barrier) once the solver has stopped
    if (skip && *reinterpret_cast<const volatile int *>(skip) != 0) return;
    constexpr uint32_t NST = RING / CH;
    constexpr uint32_t PF = DD_PF_AHEAD < 0 ? RING / 2 : (uint32_t)DD_PF_AHEAD;
    constexpr int TC = TCB<BS>;
    constexpr uint32_t NW = TC / 32;
    static_assert((RING & (RING - 1)) == 0 && (CH & (CH - 1)) == 0 && NST >= 4, "ring shape");
    extern __shared__ __align__(128) uint8_t smem[];
    double *vec = reinterpret_cast<double *>(smem);
    uint8_t *ring = smem + vec_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + RING);
    uint64_t *empty = full + NST;
    // sync-free ready bits: L bitset then U bitset, fw words each
    const uint32_t fw = ((uint32_t)vec_bytes / (8u * BS) + 31u) / 32u;
    const SpinFlags F{reinterpret_cast<uint32_t *>(empty + NST), reinterpret_cast<uint32_t *>(empty + NST) + fw};
    const int tid = threadIdx.x;

    if (tid == TC) {
        for (uint32_t q = 0; q < NST; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], SPIN ? NW : 1);
        }
        fence_mbar_init();
    }
    if (SPIN) {
        for (uint32_t q = tid; q < 2 * fw; q += TC + 32) F.L[q] = 0u;
    }
    if (tid < BS) vec[BS * sw.zslot + tid] = 0.0;  // the zero slot (never overwritten)
    __syncthreads();

    if (tid >= TC) {
        // ================= producer: one elected lane streams the CTA's work
        if (tid == TC) {
            const uint64_t pol = policy_evict_first();
            uint32_t g = 0;
#ifdef DD_TRACE
            long long tr_pw = 0;
            const long long tr_p0 = clock64();
#endif
            for (int s = blockIdx.x; s < n_sub; s += gridDim.x) {
                const SubInfo si = info[DD_SUB(s)];
                const int64_t rlo = (8 * BS * (int64_t)si.row0) & ~(int64_t)15;
                const int64_t rhi = (8 * BS * ((int64_t)si.row0 + si.nrows) + 15) & ~(int64_t)15;
                const uint32_t rb = (uint32_t)(rhi - rlo);
                // phase 0: the whole stream; 1: the L section; 2: the D+U section
                const uint32_t sec_lo = phase == 2 ? (uint32_t)si.u_off : 0u;
                const uint32_t sec_hi = phase == 1 ? (uint32_t)si.u_off : (uint32_t)si.stream_bytes;
                const uint32_t total = rb + (sec_hi - sec_lo);
                const uint32_t nch = (total + CH - 1) / CH;
                const uint8_t *rsrc = reinterpret_cast<const uint8_t *>(r) + rlo;
                const uint8_t *fsrc = slab + si.stream_off + sec_lo;
                // L2 prefetch PF bytes ahead of the ring's fill position (into the
                // CTA's next subdomain near the end of this one): when the ring is
                // full because the consumers are in narrow levels, HBM keeps
                // streaming this CTA's next bytes into L2, and the ring refills
                // from L2 once chunks free up (config 3: 425 -> 406 us at PF =
                // half a ring, 32 KB; 410 us at 64 KB, 406 us at 128 KB). Half a
                // ring keeps 296 x 32 KB = 9.5 MB ahead, far below L2; at 256 KB
                // the prefetched lines are evicted before use (457 us; 512 KB:
                // 582 us).
                auto pf_sub = [&](int ss, uint32_t a, uint32_t b) {
                    const SubInfo sj = info[DD_SUB(ss)];
                    const int64_t jlo = (8 * BS * (int64_t)sj.row0) & ~(int64_t)15;
                    const int64_t jhi = (8 * BS * ((int64_t)sj.row0 + sj.nrows) + 15) & ~(int64_t)15;
                    const uint32_t jrb = (uint32_t)(jhi - jlo);
                    const uint32_t jsl = phase == 2 ? (uint32_t)sj.u_off : 0u;
                    const uint32_t jsh = phase == 1 ? (uint32_t)sj.u_off : (uint32_t)sj.stream_bytes;
                    b = min(b, jrb + (jsh - jsl));
                    if (a >= b) return;
                    if (a < jrb) prefetch_l2(reinterpret_cast<const uint8_t *>(r) + jlo + a, min(b, jrb) - a);
                    if (b > jrb) {
                        const uint32_t q = max(a, jrb);
                        prefetch_l2(slab + sj.stream_off + jsl + (q - jrb), b - q);
                    }
                };
                for (uint32_t c = 0; c < nch; ++c, ++g) {
                    const uint32_t st = g % NST;
                    if (PF) {
                        const uint32_t a = c * CH + PF, b = a + CH;
                        if (a < total) pf_sub(s, a, b);
                        if (b > total && s + (int)gridDim.x < n_sub)
                            pf_sub(s + gridDim.x, a > total ? a - total : 0u, b - total);
                    }
#ifdef DD_TRACE
                    const long long tw0 = clock64();
#endif
                    if (g >= NST) mbar_wait(&empty[st], ((g / NST) - 1u) & 1u);
#ifdef DD_TRACE
                    tr_pw += clock64() - tw0;
#endif
                    const uint32_t lo = c * CH, hi = min(total, lo + CH);
                    mbar_arrive_expect_tx(&full[st], hi - lo);
                    uint8_t *dst = ring + st * CH;
                    if (lo < rb) bulk_g2s(dst, rsrc + lo, min(hi, rb) - lo, &full[st], pol);
                    if (hi > rb) {
                        const uint32_t b = max(lo, rb);
                        bulk_g2s(dst + (b - lo), fsrc + (b - rb), hi - b, &full[st], pol);
                    }
                }
            }
#ifdef DD_TRACE
            if (!SPIN && MODE == AM_VC) {
                atomicAdd(&g_dd_trace[blockIdx.x & 1023][8], (unsigned long long)tr_pw);
                atomicAdd(&g_dd_trace[blockIdx.x & 1023][9], (unsigned long long)(clock64() - tr_p0));
            }
#endif
        }
        return;
    }

    // ===================== consumers (TC threads, named barrier 1)
    const int t = tid;
    const uint32_t lane = t & 31u;
    uint32_t gbase = 0;     // chunk index at which the current subdomain starts
    uint32_t ready = 0;     // chunks this thread has seen full
    uint32_t released = 0;  // chunks handed back (SPIN: each warp's lane 0; else t == TC - 32)
#ifdef DD_TRACE
    // [0] r fill, [1] L records, [2] U records, [3] z store + halo, [4] full
    // waits, [5] record barriers, [6] subdomains, [7] records
    long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long trc = clock64();
    auto tmark = [&](int k) {
        const long long c = clock64();
        tr[k] += c - trc;
        trc = c;
    };
#endif
    auto ensure = [&](uint32_t chunk) {
#ifdef DD_TRACE
        const long long w0 = clock64();
#endif
        while (ready <= chunk) {
            mbar_wait(&full[ready % NST], (ready / NST) & 1u);
            ++ready;
        }
#ifdef DD_TRACE
        tr[4] += clock64() - w0;
#endif
    };
    auto release_to = [&](uint32_t upto) {
        // level set: lane 0 of the LAST consumer warp hands chunks back -- its
        // rows are the record's lightest (sorted by block count) or absent, so
        // the releases stay off the slowest warp's path (-1 % at config 3)
        if (SPIN ? lane == 0 : t == TC - 32) {
            while (released < upto) {
                mbar_arrive(&empty[released % NST]);
                ++released;
            }
        }
    };
    for (int s = blockIdx.x; s < n_sub; s += gridDim.x) {
        const SubInfo si = info[DD_SUB(s)];
        const int64_t rlo = (8 * BS * (int64_t)si.row0) & ~(int64_t)15;
        const int64_t rhi = (8 * BS * ((int64_t)si.row0 + si.nrows) + 15) & ~(int64_t)15;
        const uint32_t rb = (uint32_t)(rhi - rlo);
        const uint32_t shift = (uint32_t)(8 * BS * (int64_t)si.row0 - rlo);
        const uint32_t sec_lo = phase == 2 ? (uint32_t)si.u_off : 0u;
        const uint32_t sec_hi = phase == 1 ? (uint32_t)si.u_off : (uint32_t)si.stream_bytes;
        const uint32_t total = rb + (sec_hi - sec_lo);
        const uint32_t nch = (total + CH - 1) / CH;
        const uint32_t nd = (uint32_t)BS * si.nrows;
        const uint32_t abs0 = gbase * CH;
#ifdef DD_TRACE
        trc = clock64();
        tr[6] += 1;
        bool tr_in_u = false;
#endif
        // ---- r slice: ring -> vec, chunk by chunk
        const uint32_t nrc = (rb + CH - 1) / CH;
        for (uint32_t c = 0; c < nrc; ++c) {
            ensure(gbase + c);
            const uint32_t qlo = c == 0 ? 0u : (c * CH - shift) / 8u;
            const uint32_t qhi = min(nd, ((c + 1) * CH - shift) / 8u);
            // thread t fills the entries q = t (mod TC) -- the ones it stored
            // to z for the previous subdomain -- so no barrier is needed
            // between that store and this fill
            for (uint32_t q = qlo + (t + TC - qlo % TC) % TC; q < qhi; q += TC)
                vec[vslot<BS>(sw, q)] = *reinterpret_cast<const double *>(ring + ((abs0 + shift + 8u * q) & (RING - 1u)));
            if ((c + 1) % (NST / 2) == 0 && c + 1 < nrc) {
                named_bar_sync(1, TC);
                release_to(gbase + c + 1);
            }
        }
        // sync-free: clear the ready bits of the previous subdomain (every
        // thread passed its final barrier, nobody reads them until the next)
        if (SPIN)
            for (uint32_t q = t; q < 2 * fw; q += TC) F.L[q] = 0u;
        named_bar_sync(1, TC);
        release_to(gbase + rb / CH);
#ifdef DD_TRACE
        tmark(0);
#endif
        // ---- records
        if (mode == 2) {
            // measurement only: take every chunk as it lands and hand it back
            // at once (no record walk, no barriers) -- the ring's raw stream
            // (every thread tracks the chunks it has seen full)
            for (uint32_t c = rb / CH; c < nch; ++c) {
                ensure(gbase + c);
                release_to(gbase + c + 1);
            }
            named_bar_sync(1, TC);
            gbase += nch;
            continue;
        }
        uint32_t ro = rb;
        while (true) {
            ensure(gbase + ro / CH);
            const uint32_t pos = (abs0 + ro) & (RING - 1u);
            const RecHdr h = hdr_from(*reinterpret_cast<const uint4 *>(ring + pos));
            ensure(gbase + (ro + h.bytes - 1) / CH);
            // the 16 B after the header (cnt[0..7]) never straddle the ring end:
            // records and the ring are 16-byte aligned
            const uint4 c8 = *reinterpret_cast<const uint4 *>(ring + ((pos + 16u) & (RING - 1u)));
            const bool upper = (h.flags & ddi::REC_UPPER) != 0;
            // the section ends with its last record (phase 1 stops before D+U)
            const bool last = (h.flags & ddi::REC_LAST) != 0 || ro + h.bytes >= total;
            // L level 0 carries no blocks (z_i = r_i in place): the level set
            // skips it (no work, no barrier); the sync-free sweep publishes flags
            const bool skip = !SPIN && !upper && h.K == 0 && !last;
#ifdef DD_TRACE
            if (upper && !tr_in_u) {
                tmark(1);
                tr_in_u = true;
            }
            tr[7] += 1;
#endif
            if (mode == 1 || skip) {
            } else if constexpr (MODE == AM_TREE && BS == 3) {
                if (pos + h.bytes <= RING)
                    process_record_tree<GEN>(LinRd{ring + pos}, h, c8, t, TC, vec);
                else
                    process_record_tree<GEN>(RingRd<RING>{ring, abs0 + ro}, h, c8, t, TC, vec);
            } else if constexpr (MODE == AM_EC && BS == 3) {
                auto bar = [] { named_bar_sync(1, TC); };
                if (pos + h.bytes <= RING)
                    process_record_ec<GEN>(LinRd{ring + pos}, h, c8, t, TC, vec, bar);
                else
                    process_record_ec<GEN>(RingRd<RING>{ring, abs0 + ro}, h, c8, t, TC, vec, bar);
            } else if (pos + h.bytes <= RING) {
                process_record<BS, SPIN, GEN, LinRd, MODE == AM_NU>(LinRd{ring + pos}, h, c8, t, vec, F);
            } else {
                process_record<BS, SPIN, GEN, RingRd<RING>, MODE == AM_NU>(RingRd<RING>{ring, abs0 + ro}, h, c8, t,
                                                                          vec, F);
            }
            const uint32_t ro0 = ro;
            ro += h.bytes;
            if (SPIN) {
                // lanes diverge in the flag waits: reconverge before lane 0 hands
                // chunks back (rows of one record never depend on each other, so
                // this cannot deadlock)
                __syncwarp();
            } else if (!skip || ro0 / CH != ro / CH) {
                // a skipped record needs no barrier for the sweep, but when it
                // ends in a later chunk than it started, the chunk handed back
                // below may hold headers a lagging warp has not read yet
#ifdef DD_TRACE
                const long long b0 = clock64();
#endif
                named_bar_sync(1, TC);
#ifdef DD_TRACE
                tr[5] += clock64() - b0;
#endif
            }
            if (last) {
                if (SPIN) named_bar_sync(1, TC);  // every row final before z is stored
                release_to(gbase + nch);
#ifdef DD_TRACE
                tmark(2);
#endif
                break;
            }
            release_to(gbase + ro / CH);
        }
        double *zs = z + BS * (int64_t)si.row0;
        for (uint32_t q = t; q < nd; q += TC) zs[q] = vec[vslot<BS>(sw, q)];
        // fused halo: the subdomain's rows that peers read in
        // the next SpMV go straight from shared memory to their destination
        // (send buffer or the peer's ghost block); the CTA then waits before
        // the next subdomain overwrites the vector
        if (ho.ptr && phase != 1) {
            const int e0 = ho.ptr[s], e1 = ho.ptr[s + 1];
            if (e1 > e0) {
                for (int e = e0 + t; e < e1; e += TC) {
                    const int li = ho.row[e];
                    double *d = ho.dst[e];
#pragma unroll
                    for (int c = 0; c < BS; ++c) d[c] = vec[BS * sw.slot(li) + c];
                }
                // peer transports publish the rows with a flag after this
                // kernel: the NVLink stores must be performed system-wide first
                __threadfence_system();
                named_bar_sync(1, TC);
            }
        }
        gbase += nch;
#ifdef DD_TRACE
        tmark(3);
#endif
    }
#ifdef DD_TRACE
    if (!SPIN && MODE == AM_VC) {
        unsigned long long *o = g_dd_trace[blockIdx.x & 1023];
        if (t == 0)
            for (int k = 0; k < 8; ++k) atomicAdd(o + k, (unsigned long long)tr[k]);
        if (t == TC - 32) {  // the releasing (lightest) warp
            atomicAdd(o + 10, (unsigned long long)tr[5]);
            atomicAdd(o + 11, (unsigned long long)tr[4]);
        }
    }
#endif
}

// ------------------------------------------------------------ host side
using RingFn = void (*)(const uint8_t *, const SubInfo *, int, const double *, double *, int, int, const int *, int,
                        ddi::HaloOut, ddi::Swz);

template <int BS, uint32_t RING, uint32_t CH, bool SPIN, int GEN, int MODE>
static RingFn ring_fn() {
    return k_apply_ring<BS, RING, CH, SPIN, GEN, MODE>;
}

// ring chunk = RING / 4: every chunk costs the consumers one mbarrier
// try_wait round trip (~90 cycles, serial along a record) and the releasing
// thread one arrive, so few large chunks win (measured at config 3: 16 KB
// chunks 434 us, 8 KB 444 us, 4 KB 485 us); a chunk plus the largest record
// must still fit the ring (apply_prepare checks)
template <int BS, int GEN, bool SPIN, int MODE>
static RingFn pick_ring_m(int ring) {
    switch (ring) {
        case 131072: return ring_fn<BS, 131072, 131072 / DD_CH_DIV, SPIN, GEN, MODE>();
        case 65536: return ring_fn<BS, 65536, 65536 / DD_CH_DIV, SPIN, GEN, MODE>();
        case 32768: return ring_fn<BS, 32768, 32768 / DD_CH_DIV, SPIN, GEN, MODE>();
        case 16384: return ring_fn<BS, 16384, 16384 / DD_CH_DIV, SPIN, GEN, MODE>();
    }
    return nullptr;
}

// gen: the slab has rows with more than 3 blocks in a triangle (general-K
// path). mode: AM_VC (the product), AM_EC / AM_NU (ablations: BSR3, level set)
static RingFn pick_ring(int bs, int ring, bool spin, bool gen, int mode = AM_VC) {
    if (mode != AM_VC) {
        if (bs != 3 || spin) return nullptr;
        if (mode == AM_EC) return gen ? pick_ring_m<3, 1, false, AM_EC>(ring) : pick_ring_m<3, 0, false, AM_EC>(ring);
        if (mode == AM_TREE)
            return gen ? pick_ring_m<3, 1, false, AM_TREE>(ring) : pick_ring_m<3, 0, false, AM_TREE>(ring);
        return gen ? pick_ring_m<3, 1, false, AM_NU>(ring) : pick_ring_m<3, 0, false, AM_NU>(ring);
    }
    if (bs == 1)
        return spin ? (gen ? pick_ring_m<1, 1, true, AM_VC>(ring) : pick_ring_m<1, 0, true, AM_VC>(ring))
                    : (gen ? pick_ring_m<1, 1, false, AM_VC>(ring) : pick_ring_m<1, 0, false, AM_VC>(ring));
    return spin ? (gen ? pick_ring_m<3, 1, true, AM_VC>(ring) : pick_ring_m<3, 0, true, AM_VC>(ring))
                : (gen ? pick_ring_m<3, 1, false, AM_VC>(ring) : pick_ring_m<3, 0, false, AM_VC>(ring));
}

using DirectFn = void (*)(const uint8_t *, const SubInfo *, int, const double *, double *, uint32_t, const int *,
                          int, ddi::Swz, double *, int);
// vecg: the vector in global memory (no shared-memory vector)
static DirectFn pick_direct(int bs, bool gen, int mode = AM_VC, bool vecg = false) {
    // the 3x3 direct ablation keeps the one-block-per-step general path compiled
    // in (GEN 2): the compiler schedules its global loads better that way
    // (458 vs 534 us at config 3)
    if (mode == AM_VC && !vecg) {
        if (bs == 1) return gen ? k_apply_direct<1, 1> : k_apply_direct<1, 0>;
        return gen ? k_apply_direct<3, 1> : k_apply_direct<3, 2>;
    }
    if (bs != 3) return nullptr;
    if (mode == AM_EC)
        return vecg ? (gen ? k_apply_direct<3, 1, AM_EC, true> : k_apply_direct<3, 0, AM_EC, true>)
                    : (gen ? k_apply_direct<3, 1, AM_EC, false> : k_apply_direct<3, 0, AM_EC, false>);
    if (mode == AM_VC) return gen ? k_apply_direct<3, 1, AM_VC, true> : k_apply_direct<3, 2, AM_VC, true>;
    return nullptr;
}

static int ring_chunk(int ring) { return ring / DD_CH_DIV; }

// the dynamic shared-memory attribute is per function and shared by every
// context: always raise it to the device maximum minus the static part
template <class F>
static void allow_max_smem(F fn, int smem_max) {
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) return;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max - (int)fa.sharedSizeBytes);
}

}  // namespace ddk

namespace ddi {

static int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v ? atoi(v) : dflt;
}

dd_status apply_prepare(dd_ctx *ctx) {
    using namespace ddk;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, ctx->device) != cudaSuccess) {
        set_error("cudaGetDeviceProperties failed");
        return DD_E_CUDA;
    }
    ctx->num_sms = prop.multiProcessorCount;
    const int smem_max = (int)prop.sharedMemPerBlockOptin;       // 232448 on B200
    const int nsl = ctx->sub_last - ctx->sub_first;
    const int bs = ctx->bs;
    const bool gen = ctx->kmax > 3;
    if (ctx->vec_rows <= 0) ctx->vec_rows = ctx->max_P;
    const int vec_bytes = ((8 * bs * ctx->vec_rows + 127) / 128) * 128;
    // sync-free ready bits: 2 per shared-vector slot
    const int flag_bytes = ((8 * ((ctx->vec_rows + 31) / 32)) + 15) / 16 * 16;
    const int tc = bs == 1 ? TCB<1> : TCB<3>;
    // ---- direct (ablation): one CTA per subdomain, as many per SM as fit
    {
        LaunchCfg &c = ctx->cfg_direct;
        c.smem = vec_bytes;
        c.threads = bs == 1 ? TCB<1> : TCB<3>;
        c.grid = nsl;
        c.consumers = c.threads;
        c.ring = 0;
        if (c.smem > smem_max) {
            set_error("subdomain vector exceeds shared memory");
            return DD_E_SUBDOMAIN_TOO_LARGE;
        }
        // the attribute is per function and shared by every context: set the maximum
        allow_max_smem(pick_direct(bs, gen), smem_max);
    }
    // ---- ring variants: largest ring that fits with the vector; override via DD_RING_KB
    // Ring choice: the consumer sweep is latency-bound, so maximise resident
    // CTAs per SM first (cudaOccupancy: shared memory and registers), then
    // take the largest ring that holds the biggest record plus one chunk.
    auto choose = [&](LaunchCfg &c, bool spin, int64_t max_rec, int mode = AM_VC) -> dd_status {
        const int want = env_int("DD_RING_KB", 0) * 1024;
        const int cands[4] = {131072, 65536, 32768, 16384};
        int occs[4] = {0, 0, 0, 0}, max_occ = 0;
        for (int k = 0; k < 4; ++k) {
            const int rc = cands[k];
            if (want && rc != want) continue;
            const int nst = rc / ring_chunk(rc);
            const int sm = vec_bytes + rc + 16 * nst + (spin ? flag_bytes : 0);
            if (sm > smem_max || max_rec + ring_chunk(rc) > rc) continue;
            allow_max_smem(pick_ring(bs, rc, spin, gen, mode), smem_max);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs[k], pick_ring(bs, rc, spin, gen, mode), tc + 32, sm);
            max_occ = std::max(max_occ, occs[k]);
        }
        // CTAs per SM worth having: no more than the subdomains can fill
        // (128 subdomains on 148 SMs run one CTA per SM whatever the ring), then
        // the largest ring at that occupancy
        const int need = std::max(1, std::min(max_occ, (nsl + ctx->num_sms - 1) / ctx->num_sms));
        int best_ring = 0, best_occ = 0;
        for (int k = 0; k < 4; ++k)
            if (occs[k] >= need && !best_ring) {
                best_ring = cands[k];
                best_occ = occs[k];
            }
        if (!best_ring) {
            set_error("no ring size fits the subdomain vector and the largest record");
            return DD_E_SUBDOMAIN_TOO_LARGE;
        }
        const int nst = best_ring / ring_chunk(best_ring);
        c.ring = best_ring;
        c.smem = vec_bytes + best_ring + 16 * nst + (spin ? flag_bytes : 0);
        c.threads = tc + 32;
        c.consumers = tc;
        c.grid = std::min(nsl, ctx->num_sms * std::max(1, best_occ));
        if (env_int("DD_APPLY_GRID", 0) > 0) c.grid = std::min(nsl, env_int("DD_APPLY_GRID", 0));
        return DD_OK;
    };
    // every variant walks the same level-ordered slab: prepare all of them
    // (DD_ILU0 only if its slab with the non-unit U was built at setup)
    ctx->variants = DD_LEVELSET | DD_SPINLOOP | DD_DIRECT | DD_UNFUSED | (ctx->variants & DD_ILU0);
    {
        dd_status st = choose(ctx->cfg_lvl, false, ctx->slab_lvl.max_rec_bytes);
        if (st != DD_OK) return st;
    }
    // the sync-free variant also needs 2 ready bits per row; when they
    // does not fit it is dropped (dd_apply_variant then reports the error)
    if (choose(ctx->cfg_spin, true, ctx->slab_lvl.max_rec_bytes) != DD_OK) {
        ctx->variants &= ~DD_SPINLOOP;
        ctx->cfg_spin = LaunchCfg{};
    }
    // paper ablations (BSR3): edge-centric atomics with the vector in shared
    // memory (ring) or in global memory, the vertex-centric sweep with the
    // vector in global memory, ILU0 with the non-unit U
    if (bs == 3) {
        if (choose(ctx->cfg_ec, false, ctx->slab_lvl.max_rec_bytes, AM_EC) == DD_OK) ctx->variants |= DD_EDGE;
        if (choose(ctx->cfg_tree, false, ctx->slab_lvl.max_rec_bytes, AM_TREE) == DD_OK) ctx->variants |= DD_TREE;
        ctx->variants |= DD_EDGE_GLOBAL | DD_DIRECT_GLOBAL;
        for (bool vg : {false, true})
            for (int m : {AM_EC, AM_VC})
                if (DirectFn f = pick_direct(bs, gen, m, vg)) allow_max_smem(f, smem_max);
        if ((ctx->variants & DD_ILU0) && choose(ctx->cfg_nu, false, ctx->slab_ilu.max_rec_bytes, AM_NU) != DD_OK)
            ctx->variants &= ~DD_ILU0;
    } else {
        ctx->variants &= ~DD_ILU0;
    }
    cudaGetLastError();
    return DD_OK;
}

// CTA slots (SMs x resident CTAs) the level-set ring kernel gets for
// subdomains of P rows with 7-point records (the largest ring at the best
// occupancy, as apply_prepare picks it); 0 if the vector does not fit. Used
// by dd_choose_tiles to size subdomains in whole waves. Without a device: an
// analytic model (228 KB shared memory and 3 CTAs per SM by registers).
int tile_slots(int device, int bs, int P, int *per_sm) {
    using namespace ddk;
    const int vec_bytes = ((8 * bs * P + 127) / 128) * 128;
    cudaDeviceProp prop;
    const bool dev = device >= 0 && cudaGetDeviceProperties(&prop, device) == cudaSuccess;
    if (!dev) cudaGetLastError();
    const int sms = dev ? prop.multiProcessorCount : 148;
    const int smem_max = dev ? (int)prop.sharedMemPerBlockOptin : 232448;
    const int tc = bs == 1 ? TCB<1> : TCB<3>;
    int best = 0;
    for (int rc : {131072, 65536, 32768}) {
        const int sm = vec_bytes + rc + 16 * (rc / ring_chunk(rc));
        if (sm > smem_max) continue;
        int occ = 0;
        if (dev) {
            allow_max_smem(pick_ring(bs, rc, false, false), smem_max);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pick_ring(bs, rc, false, false), tc + 32, sm);
        } else {
            occ = std::min(3, (233472 - 1024) / (sm + 1024));
        }
        best = std::max(best, occ);
    }
    cudaGetLastError();
    if (per_sm) *per_sm = best;
    return sms * best;
}

#ifdef DD_TRACE
}  // namespace ddi
extern "C" int dd_debug_trace(unsigned long long *host, int reset, int submod) {
    if (host && cudaMemcpyFromSymbol(host, ddk::g_dd_trace, sizeof(ddk::g_dd_trace)) != cudaSuccess) return -1;
    if (reset) {
        static unsigned long long zero[1024][16];
        if (cudaMemcpyToSymbol(ddk::g_dd_trace, zero, sizeof(zero)) != cudaSuccess) return -1;
    }
    if (submod >= 0 && cudaMemcpyToSymbol(ddk::g_dd_submod, &submod, sizeof(int)) != cudaSuccess) return -1;
    return 0;
}
namespace ddi {
#endif

dd_status apply_launch(dd_ctx *ctx, int variant, const double *r, double *z, void *stream, const int *skip,
                       const HaloOut *halo) {
    using namespace ddk;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int nsl = ctx->sub_last - ctx->sub_first;
    if (nsl == 0) return DD_OK;
    const int bs = ctx->bs;
    const bool gen = ctx->kmax > 3;
    const int vec_bytes = ((8 * bs * ctx->vec_rows + 127) / 128) * 128;
    // DD_LOWER: the lower sweep alone, z = L^-1 r (Table 3 analogue)
    const int phase = (variant & DD_LOWER) ? 1 : 0;
    variant &= ~DD_LOWER;
    if (variant == 0) variant = DD_LEVELSET;
    const HaloOut ho = halo ? *halo : HaloOut{};
    if (ho.ptr && variant != DD_LEVELSET) {
        set_error("dd_apply: the fused halo epilogue is a level-set ring-kernel feature");
        return DD_E_INVALID_ARG;
    }
    if (variant != DD_LEVELSET && !(ctx->variants & variant)) {
        set_error("dd_apply: variant not available for this context (sync-free flags or the largest record do not "
                  "fit, DD_ILU0 not requested at dd_setup, or a BSR3-only ablation on a scalar matrix)");
        return variant == DD_SPINLOOP ? DD_E_SUBDOMAIN_TOO_LARGE : DD_E_INVALID_ARG;
    }
    static const int mode = env_int("DD_APPLY_MODE", 0);  // 1: streaming ceiling (measurement only)
    static const uint32_t pf = (uint32_t)env_int("DD_DIRECT_PF_KB", 32) * 1024u;
    const uint8_t *slab = ctx->slab_lvl.d_bytes;
    const SubInfo *info = ctx->slab_lvl.d_info;
    auto ring = [&](const LaunchCfg &c, bool spin, int m, const double *rr, int ph, const uint8_t *sb,
                    const SubInfo *si) {
        pick_ring(bs, c.ring, spin, gen, m)<<<c.grid, c.threads, c.smem, st>>>(sb, si, nsl, rr, z, vec_bytes, mode,
                                                                              skip, ph, ho, ctx->swz);
    };
    auto direct = [&](int m, bool vg, int smem) {
        pick_direct(bs, gen, m, vg)<<<nsl, ctx->cfg_direct.threads, smem, st>>>(
            slab, info, nsl, r, z, pf, skip, phase, ctx->swz, ctx->d_vecg, ctx->vec_rows);
    };
    if ((variant == DD_EDGE_GLOBAL || variant == DD_DIRECT_GLOBAL) && !ctx->d_vecg) {
        // the global-memory vector of the no-LDS ablations (slot layout)
        if (cudaMalloc(&ctx->d_vecg, sizeof(double) * bs * (size_t)ctx->vec_rows * nsl) != cudaSuccess) {
            cudaGetLastError();
            set_error("dd_apply: cannot allocate the global vector of the no-LDS variant");
            return DD_E_OOM;
        }
    }
    switch (variant) {
        case DD_LEVELSET: ring(ctx->cfg_lvl, false, AM_VC, r, phase, slab, info); break;
        case DD_UNFUSED:
            // ablation of the fusion (sec. 4.4): the L sweep and the
            // D+U sweep as two launches of the same kernel; the vector makes a
            // round trip through HBM in between (z holds L^-1 r after the first)
            ring(ctx->cfg_lvl, false, AM_VC, r, 1, slab, info);
            if (!phase) {
                ++ctx->n_launches;
                ring(ctx->cfg_lvl, false, AM_VC, z, 2, slab, info);
            }
            break;
        case DD_SPINLOOP: ring(ctx->cfg_spin, true, AM_VC, r, phase, slab, info); break;
        case DD_DIRECT: direct(AM_VC, false, ctx->cfg_direct.smem); break;
        case DD_EDGE: ring(ctx->cfg_ec, false, AM_EC, r, phase, slab, info); break;
        case DD_TREE: ring(ctx->cfg_tree, false, AM_TREE, r, phase, slab, info); break;
        case DD_EDGE_GLOBAL: direct(AM_EC, true, 0); break;
        case DD_DIRECT_GLOBAL: direct(AM_VC, true, 0); break;
        case DD_ILU0:
            // the L section of the ILU0 slab equals the ILDU0 one
            ring(ctx->cfg_nu, false, AM_NU, r, phase, ctx->slab_ilu.d_bytes, ctx->slab_ilu.d_info);
            break;
        default: set_error("dd_apply: unknown variant"); return DD_E_INVALID_ARG;
    }
    ++ctx->n_launches;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("dd_apply launch: ") + cudaGetErrorString(e));
        return DD_E_CUDA;
    }
    return DD_OK;
}

}  // namespace ddi
