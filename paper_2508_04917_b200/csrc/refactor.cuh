// refactor.cuh -- declarations shared by refactor.cu and api.cpp (product-internal).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ddi {
struct SubInfo;
}

namespace ddk {

struct RfArgs {
    const int32_t *SubLev, *LevPtr, *LevRows;
    const int32_t *SubU, *URows;  // rows in U-record order per subdomain
    const int64_t *Wrp, *Wdiag, *Uptr, *Lrp, *Urp;
    const int32_t *Wcol, *UpdQ, *UpdT;
    double *W, *Dinv;
    uint8_t *slab;
    const int64_t *Loff, *Uoff, *Doff;
    const int32_t *Lst, *Ust, *Dst;
    double floor_;
    unsigned long long *bad;  // min failing (reordered global) row
    int64_t row_first;
    // the caller's blocks and W position -> caller's block (k_refactor_diag
    // reads the matrix's values straight from A: no W buffer)
    const double *A;
    const int32_t *Wsrc;
    // fused sliced-ELL gather (k_refactor_diag): the CTA of a subdomain also
    // refreshes the SpMV operand's slices that start in its rows
    const ddi::SubInfo *info;
    const int64_t *ell_slot_ptr;
    const int32_t *Esrc;
    double *ell_vals;
};

void launch_gather_blocks(int64_t n, const int32_t *src, const double *from, double *to, int ell, int grid,
                          cudaStream_t st);
void launch_refactor(int nsl, const RfArgs &a, cudaStream_t st);
// the diagonal-update class (k_refactor_diag): plan = 16 words per row in
// LevRows order -- li, w0, dpos | (lower block jp has its U_ki update) << (8 + jp),
// Lrp[li], k of the lower blocks (3), caller's block of U_ki (3, -1: none),
// caller's blocks of W_ik (3, -1: none), caller's block of U_ii, 2 unused
constexpr int RFD_PLAN_WORDS = 16;
void launch_refactor_diag(int nsl, const RfArgs &a, const int32_t *plan, cudaStream_t st);

}  // namespace ddk
