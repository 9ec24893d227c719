// solver.cpp -- the BiCGSTAB driver of the C ABI (Alg. 1, right
// preconditioning R20): one iteration as a fixed kernel sequence with
// device-side control, run as one CUDA graph with a
// conditional WHILE node (world 1 and the peer transports) or as a
// host-batched loop (NCCL, profiling, DD_GRAPH=0); per-kernel profiling.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "api_internal.h"

using namespace ddi;

namespace {

// device residual history held from dd_setup: solves of up to this many
// iterations take the captured graph (longer ones the batched loop, with a
// stream-ordered reallocation)
constexpr int kHistIters = 10000;

// Optional per-kernel timing inside dd_bicgstab (dd_profile): CUDA events on
// the solver's stream around every apply / SpMV / BLAS-1 launch, harvested at
// the solver's own synchronisation points (no extra host syncs).
enum { PK_APPLY = 0, PK_SPMV = 1, PK_BLAS = 2 };
struct Prof {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    struct Pend {
        int kind, iter;
        cudaEvent_t a, b;
    };
    std::vector<Pend> pend;
    double ms[3] = {0, 0, 0};
    int64_t n[3] = {0, 0, 0};
};

Prof *prof_of(dd_ctx *c) {
    if (!c->prof) c->prof = new Prof();
    return reinterpret_cast<Prof *>(c->prof);
}

cudaEvent_t prof_ev(Prof *p) {
    if (p->used == p->pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        p->pool.push_back(e);
    }
    return p->pool[p->used++];
}

template <class F>
dd_status timed(dd_ctx *c, int kind, int iter, cudaStream_t st, F &&launch) {
    Prof *p = c->prof ? reinterpret_cast<Prof *>(c->prof) : nullptr;
    if (!p || !p->on) return launch();
    cudaEvent_t a = prof_ev(p), b = prof_ev(p);
    cudaEventRecord(a, st);
    dd_status r = launch();
    cudaEventRecord(b, st);
    p->pend.push_back({kind, iter, a, b});
    return r;
}

// Harvest after the stream is idle. Launches enqueued past the stopping point
// return at entry, so only the first n_real[kind] launches of each kind (and,
// for BLAS-1, those of iterations <= k_last) are counted.
void prof_collect(dd_ctx *c, const int64_t *n_real, int k_last) {
    Prof *p = c->prof ? reinterpret_cast<Prof *>(c->prof) : nullptr;
    if (!p) return;
    int64_t seen[3] = {0, 0, 0};
    for (auto &q : p->pend) {
        const bool real = q.kind == PK_BLAS ? q.iter <= k_last : seen[q.kind] < n_real[q.kind];
        ++seen[q.kind];
        float ms = 0.f;
        if (real && cudaEventElapsedTime(&ms, q.a, q.b) == cudaSuccess) {
            p->ms[q.kind] += ms;
            p->n[q.kind] += 1;
        }
    }
    p->pend.clear();
    p->used = 0;
}

// One Alg. 1 iteration (both half steps). k > 0: the host's iteration index;
// k < 0: graph mode, the kernels read it from ctl[C_ITER]. Every kernel
// (exchange kernels included) returns at entry once ctl[C_STATE] != RUN; the
// decision is identical on every rank, so the ranks skip the same launches.
dd_status enqueue_iteration(dd_ctx *c, ddk::RedArgs ra, int k, double *x, cudaStream_t st) {
    Workspace *ws = ws_of(c);
    const int64_t m = ws->m;
    const int *skip = ws->ctl;
    ra.k = k;
    TRY(timed(c, PK_BLAS, k, st, [&] {
        ddk::launch_update_p(c, m, k < 0 ? -1 : (k == 1), ws->r, ws->v, ws->p, ws->sc, ws->ctl, st);
        return DD_OK;
    }));
    TRY(timed(c, PK_APPLY, k, st, [&] { return apply_halo(c, ws->p, ws->ph, st, skip); }));
    TRY(timed(c, PK_SPMV, k, st,
              [&] { return spmv_mode(c, ddk::SPMV_SIGMA, ws->ph, ws->v, ws->rh, ra, st, true, skip); }));
    TRY(reduce_across(c, 1, ddk::FIN_ALPHA, ra, st));
    // world > 1 (merge_ss): the rank-local s.s waits in loc[4..5] and joins
    // the (t.s, t.t) collective; the half-step test is then taken after the
    // second apply and SpMV, which are wasted only in a solve's last
    // iteration -- the iterates are unchanged (tested bitwise)
    ddk::RedArgs ra_s = ra;
    if (ws->merge_ss) ra_s.slot = 2;
    TRY(timed(c, PK_BLAS, k, st, [&] {
        ddk::launch_update_s(c, m, ws->r, ws->v, ws->s, ra_s, st);
        return DD_OK;
    }));
    if (!ws->merge_ss) {
        TRY(reduce_across(c, 1, ddk::FIN_SS, ra, st));
        ddk::launch_update_x_half(c, m, ws->ph, x, ws->sc, ws->ctl, st);
    }
    TRY(timed(c, PK_APPLY, k, st, [&] { return apply_halo(c, ws->s, ws->sh, st, skip); }));
    TRY(timed(c, PK_SPMV, k, st,
              [&] { return spmv_mode(c, ddk::SPMV_TS_TT, ws->sh, ws->t, ws->s, ra, st, true, skip); }));
    if (ws->merge_ss) {
        TRY(reduce_across(c, 3, ddk::FIN_SS_OMEGA, ra, st));
        ddk::launch_update_x_half(c, m, ws->ph, x, ws->sc, ws->ctl, st);
    } else {
        TRY(reduce_across(c, 2, ddk::FIN_OMEGA, ra, st));
    }
    TRY(timed(c, PK_BLAS, k, st, [&] {
        ddk::launch_update_xr(c, m, ws->ph, ws->sh, ws->s, ws->t, ws->rh, x, ws->r, ra, st);
        return DD_OK;
    }));
    TRY(reduce_across(c, 2, ddk::FIN_RHO, ra, st));
    return DD_OK;
}

// CUDA-graph solve loop: the iteration body captured ONCE at
// dd_setup under a conditional WHILE node, for the workspace solution vector
// ws->xd and the device history ws->d_hist, so a whole solve is one graph
// launch and dd_bicgstab neither captures, instantiates nor allocates (with
// the peer transports a rank may already be spinning on this one's signals;
// a host call that waits for the device -- cudaFree, say -- would then
// deadlock ranks that share a GPU). Used for world == 1 and the peer
// transports when per-kernel profiling is off (DD_GRAPH=0 disables it).
dd_status graph_capture(dd_ctx *c) {
    Workspace *ws = ws_of(c);
    if (!ws->cap) CK(cudaStreamCreateWithFlags(&ws->cap, cudaStreamNonBlocking));
    CK(cudaGraphCreate(&ws->graph, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, ws->graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, ws->graph, nullptr, 0, &p));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    ddk::RedArgs ra = red_args(c);
    ra.ctl = ws->ctl;
    ra.hist = ws->d_hist;
    ra.k = -1;
    const int64_t n0 = c->n_launches;
    CK(cudaStreamBeginCaptureToGraph(ws->cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    ddk::launch_iter_head(ws->ctl, ws->cap);
    dd_status e = enqueue_iteration(c, ra, -1, ws->xd, ws->cap);
    ddk::launch_iter_tail(ws->ctl, h, ws->cap);
    cudaGraph_t out = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(ws->cap, &out);
    if (e != DD_OK) return e;
    if (ce != cudaSuccess) {
        set_error(std::string("dd_setup: graph capture failed: ") + cudaGetErrorString(ce));
        return DD_E_CUDA;
    }
    ws->g_launches = c->n_launches - n0;
    c->n_launches = n0;
    CK(cudaGraphInstantiate(&ws->gexec, ws->graph, 0));
    ws->gx = ws->xd;
    ws->ghist = ws->d_hist;
    return DD_OK;
}

}  // namespace

namespace ddi {
void prof_free(dd_ctx *c) {
    if (!c->prof) return;
    for (auto e : reinterpret_cast<Prof *>(c->prof)->pool) cudaEventDestroy(e);
    delete reinterpret_cast<Prof *>(c->prof);
    c->prof = nullptr;
}

dd_status solver_prepare(dd_ctx *c) {
    Workspace *ws = ws_of(c);
    ws->hist_cap = 2 * (int64_t)kHistIters + 1;
    TRY(dmalloc(&ws->d_hist, (size_t)ws->hist_cap));
    static const bool graphs_env = !getenv("DD_GRAPH") || atoi(getenv("DD_GRAPH")) != 0;
    if (graphs_env && comm_graph_ok(c) && c->n_local > 0) TRY(graph_capture(c));
    return DD_OK;
}
}  // namespace ddi

namespace {

dd_status read_scalars(dd_ctx *c, cudaStream_t st) {
    Workspace *ws = ws_of(c);
    CK(cudaMemcpyAsync(ws->h_sc, ws->sc, ddk::S_COUNT * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(ws->ev[0], st));
    TRY(comm_wait_event(c, ws->ev[0]));
    return DD_OK;
}

}  // namespace

extern "C" {

dd_status dd_bicgstab(dd_ctx *c, const double *b, double *x, double tol, int32_t max_iter, double *hist,
                      dd_report *rep, void *stream) {
    if (!usable(c)) return DD_E_INVALID_ARG;
    if (!(tol > 0) || max_iter < 1) {
        set_error("dd_bicgstab: tol must be > 0 and max_iter >= 1");
        return DD_E_INVALID_ARG;
    }
    if ((!b || !x) && c->n_local) {
        set_error("dd_bicgstab: NULL vector");
        return DD_E_INVALID_ARG;
    }
    DEVICE_GUARD(c);
    const double t0 = now_ms();
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Workspace *ws = ws_of(c);
    const int64_t m = ws->m;
    if (ws->hist_cap < 2 * (int64_t)max_iter + 1) {
        // stream-ordered (no device-wide synchronisation, see graph_capture)
        CK(cudaFreeAsync(ws->d_hist, st));
        ws->d_hist = nullptr;
        ws->hist_cap = 0;
        CK(cudaMallocAsync(reinterpret_cast<void **>(&ws->d_hist), sizeof(double) * (2 * (size_t)max_iter + 1), st));
        ws->hist_cap = 2 * (int64_t)max_iter + 1;
    }
    static const bool graphs_env = !getenv("DD_GRAPH") || atoi(getenv("DD_GRAPH")) != 0;
    const bool use_graph = graphs_env && ws->gexec && ws->ghist == ws->d_hist &&
                           !(c->prof && reinterpret_cast<Prof *>(c->prof)->on);
    // the graph runs on ws->xd: the caller's x goes in and out by D2D copies
    // (2 x 24 n bytes, ~0.03 ms at 160^3)
    double *const x_user = x;
    if (use_graph && x != ws->xd) {
        CK(cudaMemcpyAsync(ws->xd, x, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
        x = ws->xd;
    }
    CK(cudaMemsetAsync(ws->ctl, 0, 8 * sizeof(int), st));
    *ws->h_tol = tol;
    CK(cudaMemcpyAsync(ws->sc + ddk::S_TOL, ws->h_tol, sizeof(double), cudaMemcpyHostToDevice, st));
    ddk::RedArgs ra = red_args(c);
    ra.ctl = ws->ctl;
    ra.hist = ws->d_hist;
    ra.k = 0;
    const ddk::RedArgs ra_plain = red_args(c);

    // r = b - A x0; rh = r; rho_1 = ||r0||^2; thr = tol ||r0|| (FIN_INIT)
    TRY(spmv_mode(c, ddk::SPMV_PLAIN, x, ws->t, nullptr, ra_plain, st));
    ddk::launch_init_r(c, m, b, ws->t, ws->r, ws->rh, ra, st);
    TRY(reduce_across(c, 1, ddk::FIN_INIT, ra, st));

    // Alg. 1 iterations: one graph launch, or enqueued in batches; every
    // kernel returns at entry once the device-side control has stopped. The
    // host looks at the control word one batch behind, so the GPU never idles
    // on a half-step decision; every rank waits on the same batch, so all
    // ranks stop together.
    constexpr int BATCH = 2;
    int k_enq = 0, j = 0;
    const int64_t g_per_iter = ws->g_launches;
    if (use_graph) {
        *ws->h_max = max_iter;
        CK(cudaMemcpyAsync(ws->ctl + ddk::C_MAX, ws->h_max, sizeof(int), cudaMemcpyHostToDevice, st));
        CK(cudaGraphLaunch(ws->gexec, st));
    }
    for (bool stop = use_graph; !stop; ++j) {
        for (int q = 0; q < BATCH && k_enq < max_iter; ++q) {
            const int k = ++k_enq;
            ra.k = k;
            TRY(enqueue_iteration(c, ra, k, x, st));
        }
        int *snap = ws->h_ctl + 8 * (j % 2);
        CK(cudaMemcpyAsync(snap, ws->ctl, 8 * sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(ws->ev[j % 2], st));
        if (j >= 1) {
            TRY(comm_wait_event(c, ws->ev[(j - 1) % 2]));
            if (ws->h_ctl[8 * ((j - 1) % 2) + ddk::C_STATE] != ddk::ST_RUN) stop = true;
        }
        if (k_enq >= max_iter) stop = true;
    }
    CK(cudaMemcpyAsync(ws->h_ctl, ws->ctl, 8 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(ws->ev[0], st));
    TRY(comm_wait_event(c, ws->ev[0]));
    TRY(comm_check(c, st));
    const int state = ws->h_ctl[ddk::C_STATE], kf = ws->h_ctl[ddk::C_K], nh = ws->h_ctl[ddk::C_NH];
    if (use_graph) c->n_launches += g_per_iter * std::max(1, ws->h_ctl[ddk::C_ITER]) + 2 * std::max(1, ws->h_ctl[ddk::C_ITER]);
    std::vector<double> hv(std::max(1, nh));
    CK(cudaMemcpyAsync(hv.data(), ws->d_hist, sizeof(double) * std::max(1, nh), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hist) std::memcpy(hist, hv.data(), sizeof(double) * nh);
    double iters = 0.0;
    int64_t napp = 0;
    int status = DD_OK, brk = 0;
    double rel = 1.0;
    const double n0 = hv[0];
    auto last_full = [&]() { return n0 > 0 ? hv[std::max(0, (nh - 1) & ~1)] / n0 : 0.0; };
    switch (state) {
        case ddk::ST_DONE_HALF: iters = kf - 0.5; napp = 2 * kf - 1; rel = hv[2 * kf - 1] / n0; break;
        case ddk::ST_DONE_FULL: iters = kf; napp = 2 * kf; rel = hv[2 * kf] / n0; break;
        case ddk::ST_ZERO: iters = 0; napp = 0; rel = 0.0; break;
        case ddk::ST_BRK_RHO: status = DD_E_BREAKDOWN; brk = 1; iters = kf; napp = 2 * kf; rel = last_full(); break;
        case ddk::ST_BRK_SIGMA: status = DD_E_BREAKDOWN; brk = 2; iters = kf - 1; napp = 2 * kf - 1; rel = last_full(); break;
        case ddk::ST_BRK_TAU: status = DD_E_BREAKDOWN; brk = 3; iters = kf - 0.5; napp = 2 * kf; rel = last_full(); break;
        case ddk::ST_COMM:
            set_error("peer transport: a device-side wait timed out during the solve");
            return DD_E_NCCL;
        default: status = DD_E_MAXITER; iters = max_iter; napp = 2 * (int64_t)max_iter; rel = last_full(); break;
    }
    {
        const int64_t n_real[3] = {napp, napp, 0};
        prof_collect(c, n_real, (int)std::ceil(iters));
    }
    // true residual ||b - A x|| / ||b||
    TRY(spmv_mode(c, ddk::SPMV_PLAIN, x, ws->t, nullptr, ra_plain, st));
    ddk::launch_resid(c, m, b, ws->t, ra_plain, st);
    TRY(reduce_across(c, 2, ddk::FIN_RESID, ra_plain, st));
    if (x != x_user) CK(cudaMemcpyAsync(x_user, x, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
    TRY(read_scalars(c, st));
    TRY(comm_check(c, st));
    CK(cudaGetLastError());
    const double *sc = ws->h_sc;
    if (rep) {
        rep->iterations = iters;
        rep->n_applies = (int32_t)napp;
        rep->converged = status == DD_OK;
        rep->breakdown = brk;
        rep->status = status;
        rep->rel_resid = rel;
        rep->true_rel_resid = sc[ddk::S_RES_BB] > 0 ? std::sqrt(sc[ddk::S_RES_TT]) / std::sqrt(sc[ddk::S_RES_BB]) : 0.0;
        rep->solve_ms = now_ms() - t0;
    }
    return (dd_status)status;
}

dd_status dd_solve_host(dd_ctx *c, const double *b_host, double *x_host, double tol, int32_t max_iter,
                        dd_report *rep, void *stream) {
    if (!usable(c)) return DD_E_INVALID_ARG;
    DEVICE_GUARD(c);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Workspace *ws = ws_of(c);
    TRY(dd_permute(c, b_host, ws->bd, stream));
    CK(cudaMemsetAsync(ws->xd, 0, ws->m * sizeof(double), st));
    dd_status s = dd_bicgstab(c, ws->bd, ws->xd, tol, max_iter, nullptr, rep, stream);
    if (s != DD_OK && s != DD_E_BREAKDOWN && s != DD_E_MAXITER) return s;
    TRY(dd_unpermute(c, ws->xd, x_host, stream));
    return s;
}

dd_status dd_profile(dd_ctx *c, int32_t mode, double *out) {
    if (!c) return DD_E_INVALID_ARG;
    Prof *p = prof_of(c);
    if (mode == 1) {
        p->on = true;
        for (int q = 0; q < 3; ++q) {
            p->ms[q] = 0;
            p->n[q] = 0;
        }
    } else if (mode == 0) {
        p->on = false;
    }
    if (out) {
        for (int q = 0; q < 3; ++q) {
            out[2 * q] = (double)p->n[q];
            out[2 * q + 1] = p->ms[q];
        }
        out[6] = (double)c->n_launches;
        out[7] = 0;
    }
    return DD_OK;
}

}  // extern "C"
