// refactor_api.cpp -- dd_refactor: numeric re-factorisation of
// the same pattern on the GPU (k_refactor, refactor.cu), the device copies of
// the symbolic maps built at dd_setup, and the pivot status agreed over ranks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "api_internal.h"
#include "refactor.cuh"

using namespace ddi;

namespace {
dd_status refactor_run(dd_ctx *c, const double *vals, int32_t on_device, cudaStream_t st);

// device copies of the refactor maps (allocated at the first dd_refactor)
struct RfState {
    int32_t *SubU = nullptr, *URows = nullptr;
    int32_t *SubLev = nullptr, *LevPtr = nullptr, *LevRows = nullptr, *Wcol = nullptr, *UpdQ = nullptr,
            *UpdT = nullptr, *Lst = nullptr, *Ust = nullptr, *Dst = nullptr;
    int64_t *Wrp = nullptr, *Wdiag = nullptr, *Uptr = nullptr, *Lrp = nullptr, *Urp = nullptr, *Loff = nullptr,
            *Uoff = nullptr, *Doff = nullptr;
    int32_t *Wsrc = nullptr, *Esrc = nullptr;  // W / sliced-ELL position -> caller's block (-1: padding)
    int32_t *plan = nullptr;  // row plans of k_refactor_diag (null: k_refactor9)
    double *W = nullptr, *Dinv = nullptr, *stage = nullptr;
    unsigned long long *bad = nullptr;
    unsigned long long *h_bad = nullptr;
};

ddk::RfArgs rf_args(const dd_ctx *c, const RfState *rf, const double *A) {
    return ddk::RfArgs{rf->SubLev, rf->LevPtr, rf->LevRows, rf->SubU, rf->URows, rf->Wrp, rf->Wdiag, rf->Uptr,
                       rf->Lrp, rf->Urp, rf->Wcol, rf->UpdQ, rf->UpdT, rf->W, rf->Dinv, c->slab_lvl.d_bytes,
                       rf->Loff, rf->Uoff, rf->Doff, rf->Lst, rf->Ust, rf->Dst, c->pivot_floor, rf->bad,
                       c->row_first, A, rf->Wsrc, c->slab_lvl.d_info, nullptr, nullptr, nullptr};
}

dd_status refactor_init(dd_ctx *c) {
    if (c->rf) return DD_OK;
    auto *rf = new RfState();
    c->rf = rf;
    static const bool trace = getenv("DD_SETUP_TRACE") != nullptr;
    const double t0 = now_ms();
    auto mark = [&](const char *what) {
        if (trace) fprintf(stderr, "[dd refactor_init] %-22s %9.1f ms\n", what, now_ms() - t0);
    };
    // diagonal-update class (refactor.cu, k_refactor_diag): <= 3 lower blocks
    // per row, each with at most one update, on the row's diagonal block
    {
        const int64_t nr = (int64_t)c->LevRows.size();
        ddi::uvector<int32_t> plan((size_t)ddk::RFD_PLAN_WORDS * nr);  // every word written below
        int fits = c->Lrp.empty() || c->Lrp.back() < INT32_MAX;
#pragma omp parallel for schedule(static) reduction(&& : fits)
        for (int64_t idx = 0; idx < nr; ++idx) {
            int32_t *P = plan.data() + (size_t)ddk::RFD_PLAN_WORDS * idx;
            const int64_t li = c->LevRows[idx], w0 = c->Wrp[li], dpos = c->Wdiag[li] - w0;
            bool ok = dpos <= 3;
            int32_t upd = 0;
            for (int w = 4; w < ddk::RFD_PLAN_WORDS; ++w) P[w] = w < 7 ? 0 : -1;
            for (int64_t jp = 0; ok && jp < dpos; ++jp) {
                const int64_t p = w0 + jp, nu = c->Uptr[p + 1] - c->Uptr[p];
                P[4 + jp] = c->Wcol[p];
                P[10 + jp] = c->Wsrc[p];  // W_ik: the caller's block
                if (nu > 1 || (nu == 1 && c->UpdT[c->Uptr[p]] != c->Wdiag[li])) ok = false;
                if (nu == 1) {
                    P[7 + jp] = c->Wsrc[c->UpdQ[c->Uptr[p]]];  // U_ki: the caller's block
                    upd |= 1 << jp;
                }
            }
            P[0] = (int32_t)li;
            P[1] = (int32_t)w0;
            P[2] = (int32_t)(dpos | upd << 8);
            P[3] = (int32_t)c->Lrp[li];
            P[13] = c->Wsrc[c->Wdiag[li]];  // U_ii: the caller's block
            fits = fits && ok;
        }
        static const bool force = getenv("DD_REFACTOR_KERNEL") != nullptr;
        mark("plan built");
        if (fits && !force) TRY(upload_vec(&rf->plan, plan));
    }
    // maps both kernels read (the U pass, the slab stores, the W gather)
    TRY(upload_vec(&rf->SubLev, c->SubLev));
    TRY(upload_vec(&rf->LevPtr, c->LevPtr));
    TRY(upload_vec(&rf->SubU, c->SubU));
    TRY(upload_vec(&rf->URows, c->URows));
    TRY(upload_vec(&rf->Lst, c->SlabLst));
    TRY(upload_vec(&rf->Ust, c->SlabUst));
    TRY(upload_vec(&rf->Dst, c->SlabDst));
    TRY(upload_vec(&rf->Wrp, c->Wrp));
    TRY(upload_vec(&rf->Wdiag, c->Wdiag));
    TRY(upload_vec(&rf->Urp, c->Urp));
    TRY(upload_vec(&rf->Loff, c->SlabLoff));
    TRY(upload_vec(&rf->Uoff, c->SlabUoff));
    TRY(upload_vec(&rf->Doff, c->SlabDoff));
    TRY(upload_vec(&rf->Wsrc, c->Wsrc));
    // the general elimination's index chains: only k_refactor9 walks them (the
    // row plans replace them; ~0.45 GB less to upload at 160^3)
    if (!rf->plan) {
        TRY(upload_vec(&rf->LevRows, c->LevRows));
        TRY(upload_vec(&rf->Wcol, c->Wcol));
        TRY(upload_vec(&rf->UpdQ, c->UpdQ));
        TRY(upload_vec(&rf->UpdT, c->UpdT));
        TRY(upload_vec(&rf->Uptr, c->Uptr));
        TRY(upload_vec(&rf->Lrp, c->Lrp));
    }
    mark("maps uploaded");
    // sliced-ELL slot -> original block index (-1 = padding), same layout as device_setup
    {
        const int64_t nl = c->n_local;
        const auto &S = c->spmv;
        ddi::uvector<int32_t> es(S.n_slots);  // every slot written below (padding: -1)
        std::vector<int64_t> base(S.n_slices + 1, 0);
#pragma omp parallel for schedule(static)
        for (int64_t s = 0; s < S.n_slices; ++s) {
            int64_t K = 0;
            for (int64_t li = 32 * s; li < std::min(nl, 32 * s + 32); ++li) K = std::max(K, c->Arp[li + 1] - c->Arp[li]);
            base[s + 1] = 32 * K;
        }
        for (int64_t s = 0; s < S.n_slices; ++s) base[s + 1] += base[s];
#pragma omp parallel for schedule(static)
        for (int64_t s = 0; s < S.n_slices; ++s)
            for (int lane = 0; lane < 32; ++lane) {
                const int64_t li = 32 * s + lane, K = (base[s + 1] - base[s]) / 32;
                const int64_t len = li < nl ? c->Arp[li + 1] - c->Arp[li] : 0;
                for (int64_t k = 0; k < K; ++k) es[base[s] + 32 * k + lane] = k < len ? c->Asrc[c->Arp[li] + k] : -1;
            }
        mark("ell map built");
        TRY(upload_vec(&rf->Esrc, es));
        mark("ell map uploaded");
    }
    // the working layout W: only the general kernel needs it (the
    // diagonal-update kernel reads the caller's blocks directly)
    if (!rf->plan) TRY(dmalloc(&rf->W, 9 * std::max<size_t>(1, c->Wsrc.size())));
    TRY(dmalloc(&rf->Dinv, 9 * std::max<int64_t>(1, c->n_local)));
    TRY(dmalloc(&rf->stage, 9 * std::max<int64_t>(1, c->nnzb_A)));
    TRY(dmalloc(&rf->bad, 1));
    CK(cudaMallocHost(reinterpret_cast<void **>(&rf->h_bad), sizeof(unsigned long long)));
    return DD_OK;
}

}  // namespace

namespace ddi {
void refactor_free(dd_ctx *c) {
    auto *rf = reinterpret_cast<RfState *>(c->rf);
    if (!rf) return;
    for (void *p : {(void *)rf->SubU, (void *)rf->URows, (void *)rf->SubLev, (void *)rf->LevPtr, (void *)rf->LevRows, (void *)rf->Wcol, (void *)rf->UpdQ,
                    (void *)rf->UpdT, (void *)rf->Lst, (void *)rf->Ust, (void *)rf->Dst, (void *)rf->Wrp,
                    (void *)rf->Wdiag, (void *)rf->Uptr, (void *)rf->Lrp, (void *)rf->Urp, (void *)rf->Loff,
                    (void *)rf->Uoff, (void *)rf->Doff, (void *)rf->Wsrc, (void *)rf->Esrc, (void *)rf->W,
                    (void *)rf->Dinv, (void *)rf->stage, (void *)rf->bad, (void *)rf->plan})
        cudaFree(p);
    cudaFreeHost(rf->h_bad);
    delete rf;
    c->rf = nullptr;
}
dd_status refactor_values(dd_ctx *c, const double *vals, bool on_device, cudaStream_t st) {
    return refactor_run(c, vals, on_device ? 1 : 0, st);
}

bool refactor_has_w(const dd_ctx *c) {
    auto *rf = reinterpret_cast<const RfState *>(c->rf);
    return rf && rf->W;
}

dd_status refactor_fetch(const dd_ctx *c, std::vector<double> &W, std::vector<double> &Dinv) {
    auto *rf = reinterpret_cast<const RfState *>(c->rf);
    if (!rf) {
        set_error("factors are not on the device");
        return DD_E_INVALID_ARG;
    }
    W.clear();
    if (!rf->W) {
        // diagonal-update path: no W; the factors are read from the slab
        Dinv.resize(9 * (size_t)c->n_local);
        if (!Dinv.empty()) CK(cudaMemcpy(Dinv.data(), rf->Dinv, Dinv.size() * sizeof(double), cudaMemcpyDeviceToHost));
        return DD_OK;
    }
    W.resize(9 * c->Wsrc.size());
    Dinv.resize(9 * (size_t)c->n_local);
    if (!W.empty()) CK(cudaMemcpy(W.data(), rf->W, W.size() * sizeof(double), cudaMemcpyDeviceToHost));
    if (!Dinv.empty()) CK(cudaMemcpy(Dinv.data(), rf->Dinv, Dinv.size() * sizeof(double), cudaMemcpyDeviceToHost));
    return DD_OK;
}
}  // namespace ddi

extern "C" {

dd_status dd_refactor(dd_ctx *c, const double *vals, int32_t on_device, void *stream) {
    if (!usable(c)) return DD_E_INVALID_ARG;
    DEVICE_GUARD(c);
    // collective when world > 1: every rank returns the status agreed over
    // the ranks (a singular pivot on one rank fails all of them)
    return comm_agree(c, refactor_run(c, vals, on_device, reinterpret_cast<cudaStream_t>(stream)));
}

}  // extern "C"

namespace {
dd_status refactor_run(dd_ctx *c, const double *vals, int32_t on_device, cudaStream_t st) {
    if (!vals) {
        set_error("dd_refactor: NULL values");
        return DD_E_INVALID_ARG;
    }
    if (!c->refactor) {
        set_error("dd_refactor: context was set up without enable_refactor (and factored on the host)");
        return DD_E_INVALID_ARG;
    }
    TRY(refactor_init(c));
    // the DD_ILU0 ablation slab is not re-factored: the variant goes away
    c->variants &= ~DD_ILU0;
    auto *rf = reinterpret_cast<RfState *>(c->rf);
    const double *src = vals;
    if (!on_device) {
        // pageable host values: through the pinned staging pipeline (h2d_big),
        // ordered before the gathers by a stream synchronisation
        CK(cudaStreamSynchronize(st));
        static const bool trace = getenv("DD_SETUP_TRACE") != nullptr;
        const double tv = now_ms();
        TRY(h2d_big(rf->stage, vals, 9 * c->nnzb_A * sizeof(double)));
        if (trace) fprintf(stderr, "[dd refactor] values H2D         %9.1f ms\n", now_ms() - tv);
        src = rf->stage;
    }
    const int grid = c->num_sms * 8;
    if (!rf->plan) ddk::launch_gather_blocks((int64_t)c->Wsrc.size(), rf->Wsrc, src, rf->W, 0, grid, st);
    // the diagonal-update kernel refreshes the SpMV operand itself (fused gather)
    static const bool sep_ell = getenv("DD_REFACTOR_ELL") && atoi(getenv("DD_REFACTOR_ELL")) == 0;
    const bool fuse_ell = rf->plan && !sep_ell;
    if (!fuse_ell) ddk::launch_gather_blocks(c->spmv.n_slots, rf->Esrc, src, c->spmv.vals, 1, grid, st);
    *rf->h_bad = ~0ull;
    CK(cudaMemcpyAsync(rf->bad, rf->h_bad, sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
    ddk::RfArgs a = rf_args(c, rf, src);
    if (fuse_ell) {
        a.ell_slot_ptr = c->spmv.slot_ptr;
        a.Esrc = rf->Esrc;
        a.ell_vals = c->spmv.vals;
    }
    const int nsl = c->sub_last - c->sub_first;
    if (nsl > 0) {
        if (rf->plan)
            ddk::launch_refactor_diag(nsl, a, rf->plan, st);
        else
            ddk::launch_refactor(nsl, a, st);
    }
    c->n_launches += 3;
    CK(cudaMemcpyAsync(rf->h_bad, rf->bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    if (*rf->h_bad != ~0ull) {
        set_error("singular pivot block (|det| < pivot_floor) at reordered row " +
                  std::to_string(*rf->h_bad));
        return DD_E_SINGULAR_PIVOT;
    }
    return DD_OK;
}
}  // namespace
