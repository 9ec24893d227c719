// api.cpp -- the C ABI of include/dd.h: context lifetime, device upload,
// apply / SpMV entry points, the BiCGSTAB driver (Alg. 1, right
// preconditioning R20) and the NCCL plumbing for world > 1 (sec. 8e).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "dd_internal.h"
#include "krylov.cuh"
#include "levels.cuh"
#include "refactor.cuh"

namespace ddi {
const char *last_error_c();
}

using namespace ddi;

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            set_error(std::string(#x) + ": " + cudaGetErrorString(e_));                         \
            return e_ == cudaErrorMemoryAllocation ? DD_E_OOM : DD_E_CUDA;                      \
        }                                                                                       \
    } while (0)

#define NK(x)                                                                                   \
    do {                                                                                        \
        ncclResult_t r_ = (x);                                                                  \
        if (r_ != ncclSuccess) {                                                                \
            set_error(std::string(#x) + ": " + ncclGetErrorString(r_));                         \
            return DD_E_NCCL;                                                                   \
        }                                                                                       \
    } while (0)

namespace {

struct Workspace {
    int64_t m = 0;  // bs * n_local
    double *r = nullptr, *rh = nullptr, *p = nullptr, *v = nullptr, *ph = nullptr, *s = nullptr, *sh = nullptr,
           *t = nullptr, *bd = nullptr, *xd = nullptr;
    double *sc = nullptr;        // device scalars [S_COUNT]
    void *partials = nullptr;    // DD [grid * 2]
    unsigned int *counter = nullptr;
    double *loc = nullptr;       // [4] rank-local (s, c) pairs
    double *gathered = nullptr;  // [world * 4]
    double *h_sc = nullptr;      // pinned [S_COUNT]
    int *ctl = nullptr;          // device solver control [8]
    int *h_ctl = nullptr;        // pinned [16]: two snapshots
    double *d_hist = nullptr;    // device residual history
    int64_t hist_cap = 0;
    double *h_tol = nullptr;     // pinned scalar (tolerance upload)
    cudaEvent_t ev[2] = {nullptr, nullptr};
    double *xg = nullptr;        // ghost rows of the SpMV input [bs * n_ghost]
    double *sendbuf = nullptr;   // [bs * total send rows]
    int32_t *d_send_idx = nullptr;
    std::vector<int64_t> send_off;  // [world + 1]
    // DD_COMM_LOCAL: "my send data is ready" / "I have copied my peers' data"
    cudaEvent_t xev_ready = nullptr, xev_done = nullptr;
    // fused halo (world > 1): the solver's applies write the rows peers need
    // straight from shared memory (send buffer, or DD_COMM_LOCAL the peer's
    // ghost block); xev_app: "my fused apply has written", xev_free: "my SpMV
    // no longer reads my ghost block"
    bool halo_fuse = false;
    bool merge_ss = false;  // world > 1: s.s reduced with (t.s, t.t), see enqueue_iteration
    ddi::HaloOut hout;
    int32_t *d_hptr = nullptr, *d_hrow = nullptr;
    double **d_hdst = nullptr;
    cudaEvent_t xev_app = nullptr, xev_free = nullptr;
    // CUDA-graph solve loop (one executable graph per solution vector)
    cudaStream_t cap = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    double *gx = nullptr, *ghist = nullptr;  // the captured body's x and history buffers
    int64_t g_launches = 0;
    int *h_max = nullptr;  // pinned
};

// ---------------------------------------------------------------- DD_COMM_LOCAL
// Ranks that are contexts of one process. Each exchange: every rank records
// xev_ready after producing its outgoing data; rendezvous; every rank makes
// its stream wait on the producers' events and copies device-to-device;
// records xev_done; rendezvous; every producer's stream waits on its
// consumers' xev_done before it can overwrite the outgoing buffer. All waits
// name events recorded before the rendezvous, so the GPU work of all ranks is
// enqueued before anything waits on it (no cycles).
struct LocalGroup {
    int world = 0;
    std::vector<dd_ctx *> members;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0, refs = 0;
    uint64_t gen = 0;
    bool barrier() {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        return cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g; });
    }
};

std::mutex g_groups_m;
std::map<std::string, LocalGroup *> g_groups;

LocalGroup *group_of(const dd_ctx *c) { return reinterpret_cast<LocalGroup *>(c->group); }

template <class T>
dd_status dmalloc(T **p, size_t count) {
    *p = nullptr;
    if (count == 0) return DD_OK;
    CK(cudaMalloc(reinterpret_cast<void **>(p), count * sizeof(T)));
    return DD_OK;
}

#define TRY(x)                        \
    do {                              \
        dd_status s_ = (x);           \
        if (s_ != DD_OK) return s_;   \
    } while (0)

Workspace *ws_of(dd_ctx *c) { return reinterpret_cast<Workspace *>(c->dev_ws); }

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

// Host -> device copy of a large pageable buffer through two pinned 32 MB
// staging buffers: an OpenMP memcpy fills one while the DMA engine drains the
// other (pageable cudaMemcpy runs at ~3 GB/s; this at ~10-20 GB/s).
dd_status h2d_big(void *dst, const void *src, size_t bytes) {
    constexpr size_t STG = 32u << 20;
    if (bytes < 2 * STG) {
        CK(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
        return DD_OK;
    }
    uint8_t *stg[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaStream_t st = nullptr;
    dd_status rc = DD_OK;
    if (cudaMallocHost(reinterpret_cast<void **>(&stg[0]), STG) != cudaSuccess ||
        cudaMallocHost(reinterpret_cast<void **>(&stg[1]), STG) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        rc = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess ? DD_OK : DD_E_CUDA;
    } else {
        const uint8_t *s8 = reinterpret_cast<const uint8_t *>(src);
        uint8_t *d8 = reinterpret_cast<uint8_t *>(dst);
        for (size_t off = 0, i = 0; off < bytes; off += STG, ++i) {
            const size_t n = std::min(STG, bytes - off);
            uint8_t *b = stg[i % 2];
            if (i >= 2) cudaEventSynchronize(ev[i % 2]);  // its previous DMA is done
            const int nt = 16;
#pragma omp parallel for num_threads(nt) schedule(static)
            for (int q = 0; q < nt; ++q) {
                const size_t a = n * q / nt, e = n * (q + 1) / nt;
                std::memcpy(b + a, s8 + off + a, e - a);
            }
            if (cudaMemcpyAsync(d8 + off, b, n, cudaMemcpyHostToDevice, st) != cudaSuccess) {
                rc = DD_E_CUDA;
                break;
            }
            cudaEventRecord(ev[i % 2], st);
        }
        if (cudaStreamSynchronize(st) != cudaSuccess) rc = DD_E_CUDA;
    }
    for (auto e : ev)
        if (e) cudaEventDestroy(e);
    if (st) cudaStreamDestroy(st);
    for (auto b : stg)
        if (b) cudaFreeHost(b);
    if (rc != DD_OK) set_error("dd_setup: host-to-device upload failed");
    return rc;
}

dd_status upload_slab(Slab &sl) {
    TRY(dmalloc(&sl.d_bytes, sl.bytes.size() + 16));
    TRY(dmalloc(&sl.d_info, sl.info.size() + 1));
    if (!sl.bytes.empty()) TRY(h2d_big(sl.d_bytes, sl.bytes.data(), sl.bytes.size()));
    if (!sl.info.empty())
        CK(cudaMemcpy(sl.d_info, sl.info.data(), sl.info.size() * sizeof(SubInfo), cudaMemcpyHostToDevice));
    std::vector<uint8_t>().swap(sl.bytes);  // device copy is authoritative
    return DD_OK;
}

// DD_COMM_LOCAL: join the group named by the 128-byte key; returns once
// every rank has joined (its workspace is then visible to the peers).
dd_status local_join(dd_ctx *ctx, const void *key) {
    LocalGroup *G;
    {
        std::lock_guard<std::mutex> lk(g_groups_m);
        const std::string k(reinterpret_cast<const char *>(key), 128);
        auto it = g_groups.find(k);
        if (it == g_groups.end()) {
            G = new LocalGroup();
            G->world = ctx->world;
            G->members.assign(ctx->world, nullptr);
            g_groups[k] = G;
        } else {
            G = it->second;
        }
        if (G->world != ctx->world || G->members[ctx->rank]) {
            set_error("dd_setup: DD_COMM_LOCAL group key reused with another world size or rank");
            return DD_E_INVALID_ARG;
        }
        G->members[ctx->rank] = ctx;
        ++G->refs;
        ctx->group = G;
    }
    if (!G->barrier()) {
        set_error("dd_setup: DD_COMM_LOCAL rendezvous timed out (every rank must call dd_setup from its own thread)");
        return DD_E_NCCL;
    }
    // peer access between distinct devices (copies also work without it)
    for (dd_ctx *q : G->members)
        if (q->device != ctx->device) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, ctx->device, q->device);
            if (can && cudaDeviceEnablePeerAccess(q->device, 0) != cudaSuccess) cudaGetLastError();
        }
    return DD_OK;
}

void local_leave(dd_ctx *ctx) {
    LocalGroup *G = group_of(ctx);
    if (!G) return;
    std::lock_guard<std::mutex> lk(g_groups_m);
    // no live peer may still be copying from this rank's buffers: its copies
    // precede its last xev_done record
    for (dd_ctx *q : G->members)
        if (q && q != ctx && q->dev_ws) {
            if (ws_of(q)->xev_done) cudaEventSynchronize(ws_of(q)->xev_done);
            if (ws_of(q)->xev_app) cudaEventSynchronize(ws_of(q)->xev_app);  // fused writes into our ghost block
        }
    G->members[ctx->rank] = nullptr;
    ctx->group = nullptr;
    if (--G->refs == 0) {
        for (auto it = g_groups.begin(); it != g_groups.end(); ++it)
            if (it->second == G) {
                g_groups.erase(it);
                break;
            }
        delete G;
    }
}

#define RENDEZVOUS(G)                                                              \
    do {                                                                           \
        if (!(G)->barrier()) {                                                     \
            set_error("DD_COMM_LOCAL rendezvous timed out (a rank stopped calling)"); \
            return DD_E_NCCL;                                                      \
        }                                                                          \
    } while (0)

// Fused halo lists: for every local subdomain, the rows that
// peers need (send_rows, ascending per peer) and where they go -- this rank's
// NCCL send buffer, or with DD_COMM_LOCAL the consuming peer's ghost block
// directly (peer memory: every member on one device or peer-accessible
// devices; otherwise the unfused gather + copy is kept). DD_HALO_FUSE=0
// disables it (A/B measurements and tests).
dd_status halo_out_build(dd_ctx *ctx) {
    Workspace *ws = ws_of(ctx);
    const char *env = getenv("DD_HALO_FUSE");
    bool fuse = !env || atoi(env) != 0;
    if (fuse && ctx->comm == DD_COMM_LOCAL) {
        for (dd_ctx *a : group_of(ctx)->members)
            for (dd_ctx *b : group_of(ctx)->members) {
                int can = 1;
                if (a->device != b->device) cudaDeviceCanAccessPeer(&can, a->device, b->device);
                if (!can) fuse = false;
            }
    }
    ws->halo_fuse = fuse;
    if (!fuse) return DD_OK;
    const int nsl = ctx->sub_last - ctx->sub_first;
    struct Ent {
        int32_t sub, row;
        double *dst;
    };
    std::vector<Ent> ents;
    for (int q = 0; q < ctx->world; ++q) {
        if (q == ctx->rank || q >= (int)ctx->send_rows.size()) continue;
        const auto &rows = ctx->send_rows[q];
        double *base;
        if (ctx->comm == DD_COMM_LOCAL) {
            dd_ctx *peer = group_of(ctx)->members[q];
            base = ws_of(peer)->xg + ctx->bs * peer->recv_off[ctx->rank];
        } else {
            base = ws->sendbuf + ctx->bs * ws->send_off[q];
        }
        for (size_t p = 0; p < rows.size(); ++p) {
            const int64_t g = ctx->row_first + rows[p];  // reordered global row
            const int32_t s = (int32_t)(std::upper_bound(ctx->sub_ptr.begin() + ctx->sub_first,
                                                         ctx->sub_ptr.begin() + ctx->sub_last + 1, g) -
                                        ctx->sub_ptr.begin()) - 1;
            ents.push_back({s - ctx->sub_first, (int32_t)(g - ctx->sub_ptr[s]), base + ctx->bs * (int64_t)p});
        }
    }
    std::stable_sort(ents.begin(), ents.end(), [](const Ent &a, const Ent &b) { return a.sub < b.sub; });
    std::vector<int32_t> ptr(nsl + 1, 0), row(ents.size());
    std::vector<double *> dst(ents.size());
    for (size_t e = 0; e < ents.size(); ++e) {
        ++ptr[ents[e].sub + 1];
        row[e] = ents[e].row;
        dst[e] = ents[e].dst;
    }
    for (int s = 0; s < nsl; ++s) ptr[s + 1] += ptr[s];
    TRY(dmalloc(&ws->d_hptr, ptr.size()));
    TRY(dmalloc(&ws->d_hrow, std::max<size_t>(1, row.size())));
    TRY(dmalloc(&ws->d_hdst, std::max<size_t>(1, dst.size())));
    CK(cudaMemcpy(ws->d_hptr, ptr.data(), ptr.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (!row.empty()) {
        CK(cudaMemcpy(ws->d_hrow, row.data(), row.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ws->d_hdst, dst.data(), dst.size() * sizeof(double *), cudaMemcpyHostToDevice));
    }
    ws->hout = ddi::HaloOut{ws->d_hptr, ws->d_hrow, ws->d_hdst};
    return DD_OK;
}

// The solver's apply variant: every variant reads the same slab and gives
// bitwise the same z, so dd_setup times each once on this device (3 launches
// after a warm-up, CUDA events, the workspace vectors as scratch) and
// dd_bicgstab uses the fastest -- the level set for 7-point slabs, the
// direct variant for 27-point slabs whose records need the largest ring.
// world > 1 keeps the level set (its kernel carries the fused halo).
dd_status tune_solver_variant(dd_ctx *ctx) {
    ctx->solver_variant = DD_LEVELSET;
    const char *e = getenv("DD_SOLVER_VARIANT");
    const std::string want = e ? e : "auto";
    if (want == "levelset") return DD_OK;
    if (want == "spin" || want == "direct") {
        const int v = want == "spin" ? DD_SPINLOOP : DD_DIRECT;
        if (!(ctx->variants & v)) {
            set_error("DD_SOLVER_VARIANT: variant unavailable for this slab");
            return DD_E_INVALID_ARG;
        }
        ctx->solver_variant = v;
        return DD_OK;
    }
    if (ctx->world > 1 || ctx->n_local == 0) return DD_OK;
    // under Nsight Compute or compute-sanitizer (recognised by the variables
    // their injection sets) kernel times are serialised replays: keep the
    // level set rather than trust them
    for (const char *v : {"NV_COMPUTE_PROFILER_PERFWORKS_DIR", "NVIDIA_PROCESS_INJECTION_CRASH_REPORTING",
                          "NVTX_INJECTION64_PATH", "CUDA_INJECTION64_PATH"})
        if (getenv(v)) return DD_OK;
    Workspace *ws = ws_of(ctx);
    const int64_t launches0 = ctx->n_launches;
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    dd_status rc = DD_OK;
    cudaMemsetAsync(ws->r, 0, sizeof(double) * ws->m, st);
    const int vars[3] = {DD_LEVELSET, DD_SPINLOOP, DD_DIRECT};
    float best = 0.f;
    for (int q = 0; q < 3 && rc == DD_OK; ++q) {
        if (!(ctx->variants & vars[q])) continue;
        rc = apply_launch(ctx, vars[q], ws->r, ws->p, st);  // warm-up
        cudaEventRecord(a, st);
        for (int k = 0; k < 3 && rc == DD_OK; ++k) rc = apply_launch(ctx, vars[q], ws->r, ws->p, st);
        cudaEventRecord(b, st);
        float ms = 0.f;
        if (rc == DD_OK && cudaEventSynchronize(b) == cudaSuccess && cudaEventElapsedTime(&ms, a, b) == cudaSuccess) {
            ctx->variant_ms[q] = ms / 3.0;
            if (best == 0.f || ms < best) {
                best = ms;
                ctx->solver_variant = vars[q];
            }
        }
    }
    ctx->n_launches = launches0;  // setup-time launches are not the caller's
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(st);
    if (rc == DD_OK && cudaGetLastError() != cudaSuccess) {
        set_error("dd_setup: apply variant timing failed");
        rc = DD_E_CUDA;
    }
    return rc;
}

dd_status device_setup(dd_ctx *ctx, const void *nccl_id) {
    const double t0 = now_ms();
    CK(cudaSetDevice(ctx->device));
    if (ctx->world > 1 && ctx->comm == DD_COMM_NCCL) {
        ncclComm_t comm;
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof id);
        NK(ncclCommInitRank(&comm, ctx->world, id, ctx->rank));
        ctx->nccl = comm;
    }
    static const bool trace = getenv("DD_SETUP_TRACE") != nullptr;
    auto tr = [&](const char *what) {
        if (trace) fprintf(stderr, "[dd setup] %-22s %9.1f ms\n", what, now_ms() - t0);
    };
    TRY(apply_prepare(ctx));
    tr("apply_prepare");
    const int64_t nl = ctx->n_local;
    // slabs
    TRY(upload_slab(ctx->slab_lvl));
    tr("slab upload");
    // sliced-ELL SpMV operand
    {
        auto &S = ctx->spmv;
        std::vector<int64_t> sp(S.n_slices + 1, 0);
        for (int64_t s = 0; s < S.n_slices; ++s) {
            int64_t K = 0;
            for (int64_t li = 32 * s; li < std::min(nl, 32 * s + 32); ++li)
                K = std::max(K, ctx->Arp[li + 1] - ctx->Arp[li]);
            sp[s + 1] = sp[s] + 32 * K;
        }
        tr("ell pointers");
        const int b2 = ctx->bs * ctx->bs;
        // uninitialised buffers, every slot written once by the slice that owns
        // it (padding slots: column -1, values 0) -- no serial zero-fill pass
        std::unique_ptr<int32_t[]> cols(new int32_t[std::max<int64_t>(1, S.n_slots)]);
        std::unique_ptr<double[]> vals(new double[std::max<int64_t>(1, b2 * S.n_slots)]);
#pragma omp parallel for schedule(static)
        for (int64_t s = 0; s < S.n_slices; ++s) {
            const int64_t K = (sp[s + 1] - sp[s]) / 32;
            for (int64_t k = 0; k < K; ++k) {
                int32_t *cs = &cols[sp[s] + 32 * k];
                double *vs = &vals[b2 * (sp[s] + 32 * k)];
                for (int lane = 0; lane < 32; ++lane) {
                    const int64_t li = 32 * s + lane;
                    const bool has = li < nl && k < ctx->Arp[li + 1] - ctx->Arp[li];
                    const int64_t p = has ? ctx->Arp[li] + k : 0;
                    cs[lane] = has ? ctx->Aci[p] : -1;
                    for (int v = 0; v < b2; ++v) vs[32 * v + lane] = has ? ctx->Av[b2 * p + v] : 0.0;
                }
            }
        }
        TRY(dmalloc(&S.slot_ptr, sp.size()));
        TRY(dmalloc(&S.cols, std::max<int64_t>(1, S.n_slots)));
        TRY(dmalloc(&S.vals, std::max<int64_t>(1, b2 * S.n_slots)));
        CK(cudaMemcpy(S.slot_ptr, sp.data(), sp.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
        if (S.n_slots) {
            tr("ell fill");
            TRY(h2d_big(S.cols, cols.get(), S.n_slots * sizeof(int32_t)));
            TRY(h2d_big(S.vals, vals.get(), b2 * S.n_slots * sizeof(double)));
            tr("ell upload");
        }
    }
    // permutation index of the local rows (original global row of local row li)
    {
        std::vector<int32_t> idx(nl);
        for (int64_t li = 0; li < nl; ++li) idx[li] = ctx->new_to_old[ctx->row_first + li];
        int32_t *d = nullptr;
        TRY(dmalloc(&d, std::max<int64_t>(1, nl)));
        if (nl) CK(cudaMemcpy(d, idx.data(), nl * sizeof(int32_t), cudaMemcpyHostToDevice));
        ctx->d_new_to_old_local = d;
        TRY(dmalloc(&ctx->d_stage, ctx->bs * ctx->N + 2));
    }
    // BiCGSTAB workspace
    auto *ws = new Workspace();
    ctx->dev_ws = ws;
    ws->m = ctx->bs * nl;
    const size_t mm = (size_t)ws->m + 2;  // +2: 16-byte slack past the end (dd.h)
    for (double **q : {&ws->r, &ws->rh, &ws->p, &ws->v, &ws->ph, &ws->s, &ws->sh, &ws->t, &ws->bd, &ws->xd})
        TRY(dmalloc(q, mm));
    TRY(dmalloc(&ws->sc, ddk::S_COUNT));
    CK(cudaMemset(ws->sc, 0, ddk::S_COUNT * sizeof(double)));
    CK(cudaMalloc(&ws->partials, ddk::partials_bytes(ctx)));
    TRY(dmalloc(&ws->counter, 4));
    CK(cudaMemset(ws->counter, 0, 4 * sizeof(unsigned int)));
    TRY(dmalloc(&ws->loc, 6));
    TRY(dmalloc(&ws->gathered, 6 * (size_t)std::max(1, ctx->world)));
    {
        // world > 1: ||s||^2 joins the (t.s, t.t) collective -- three
        // reduction points per iteration instead of four (DD_MERGE_SS=0: four)
        const char *e = getenv("DD_MERGE_SS");
        ws->merge_ss = ctx->world > 1 && (!e || atoi(e) != 0);
    }
    CK(cudaMallocHost(reinterpret_cast<void **>(&ws->h_sc), ddk::S_COUNT * sizeof(double)));
    TRY(dmalloc(&ws->ctl, 8));
    CK(cudaMemset(ws->ctl, 0, 8 * sizeof(int)));
    CK(cudaMallocHost(reinterpret_cast<void **>(&ws->h_ctl), 16 * sizeof(int)));
    CK(cudaMallocHost(reinterpret_cast<void **>(&ws->h_tol), sizeof(double)));
    CK(cudaMallocHost(reinterpret_cast<void **>(&ws->h_max), sizeof(int)));
    CK(cudaEventCreateWithFlags(&ws->ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ws->ev[1], cudaEventDisableTiming));
    // halo buffers
    const int64_t ng = (int64_t)ctx->ghost_rows.size();
    TRY(dmalloc(&ws->xg, std::max<int64_t>(1, ctx->bs * ng)));
    ws->send_off.assign(ctx->world + 1, 0);
    std::vector<int32_t> sidx;
    for (int q = 0; q < ctx->world; ++q) {
        if (q < (int)ctx->send_rows.size()) sidx.insert(sidx.end(), ctx->send_rows[q].begin(), ctx->send_rows[q].end());
        ws->send_off[q + 1] = (int64_t)sidx.size();
    }
    TRY(dmalloc(&ws->sendbuf, std::max<size_t>(1, ctx->bs * sidx.size())));
    TRY(dmalloc(&ws->d_send_idx, std::max<size_t>(1, sidx.size())));
    if (!sidx.empty())
        CK(cudaMemcpy(ws->d_send_idx, sidx.data(), sidx.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());
    tr("workspace");
    if (ctx->world > 1 && ctx->comm == DD_COMM_LOCAL) {
        CK(cudaEventCreateWithFlags(&ws->xev_ready, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ws->xev_done, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ws->xev_app, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ws->xev_free, cudaEventDisableTiming));
        TRY(local_join(ctx, nccl_id));
    }
    if (ctx->world > 1) TRY(halo_out_build(ctx));
    TRY(tune_solver_variant(ctx));
    ctx->setup_ms[5] = now_ms() - t0;
    return DD_OK;
}

ddk::RedArgs red_args(dd_ctx *c) {
    Workspace *ws = ws_of(c);
    return ddk::RedArgs{reinterpret_cast<ddk::DD *>(ws->partials), ws->counter, ws->sc, ws->loc,
                        c->world <= 1 ? 1 : 0, nullptr, nullptr, 0, 0};
}

// world > 1: all-gather the rank-local (s, c) pairs and finalize in rank order.
// DD_COMM_LOCAL all-gather of the ranks' loc[0 .. 2nv) into gathered[q * 2nv]
dd_status local_allgather(dd_ctx *c, int nv, cudaStream_t st) {
    LocalGroup *G = group_of(c);
    Workspace *ws = ws_of(c);
    const size_t bytes = 2 * (size_t)nv * sizeof(double);
    CK(cudaEventRecord(ws->xev_ready, st));
    RENDEZVOUS(G);
    for (int q = 0; q < c->world; ++q) {
        Workspace *pw = ws_of(G->members[q]);
        if (q != c->rank) CK(cudaStreamWaitEvent(st, pw->xev_ready, 0));
        CK(cudaMemcpyAsync(ws->gathered + 2 * (size_t)nv * q, pw->loc, bytes, cudaMemcpyDefault, st));
    }
    CK(cudaEventRecord(ws->xev_done, st));
    RENDEZVOUS(G);
    for (int q = 0; q < c->world; ++q)
        if (q != c->rank) CK(cudaStreamWaitEvent(st, ws_of(G->members[q])->xev_done, 0));
    return DD_OK;
}

// DD_COMM_LOCAL halo: copy every peer's send segment for this rank into xg
dd_status local_halo(dd_ctx *c, cudaStream_t st) {
    LocalGroup *G = group_of(c);
    Workspace *ws = ws_of(c);
    CK(cudaEventRecord(ws->xev_ready, st));
    RENDEZVOUS(G);
    for (int q = 0; q < c->world; ++q) {
        if (q == c->rank) continue;
        const int64_t ro = c->recv_off[q], rn = c->recv_off[q + 1] - ro;
        if (!rn) continue;
        Workspace *pw = ws_of(G->members[q]);
        CK(cudaStreamWaitEvent(st, pw->xev_ready, 0));
        CK(cudaMemcpyAsync(ws->xg + c->bs * ro, pw->sendbuf + c->bs * pw->send_off[c->rank], c->bs * rn * sizeof(double),
                           cudaMemcpyDefault, st));
    }
    CK(cudaEventRecord(ws->xev_done, st));
    RENDEZVOUS(G);
    for (int q = 0; q < c->world; ++q)
        if (q != c->rank && ws->send_off[q + 1] > ws->send_off[q])
            CK(cudaStreamWaitEvent(st, ws_of(G->members[q])->xev_done, 0));
    return DD_OK;
}

dd_status reduce_across(dd_ctx *c, int nv, int op, const ddk::RedArgs &ra, cudaStream_t st) {
    if (c->world <= 1) return DD_OK;
    Workspace *ws = ws_of(c);
    if (c->comm == DD_COMM_LOCAL)
        TRY(local_allgather(c, nv, st));
    else
        NK(ncclAllGather(ws->loc, ws->gathered, 2 * nv, ncclDouble, reinterpret_cast<ncclComm_t>(c->nccl), st));
    ddk::launch_finalize_gathered(c->world, nv, ws->gathered, ra, op, st);
    ++c->n_launches;
    return DD_OK;
}

// halo exchange of the SpMV input x (local rows) into ws->xg. packed: x was
// produced by a fused-halo apply (apply_halo), which already wrote the rows
// peers need (NCCL: into the send buffer; DD_COMM_LOCAL: into the peers'
// ghost blocks -- only the ordering remains)
dd_status halo(dd_ctx *c, const double *x, cudaStream_t st, bool packed) {
    if (c->world <= 1) return DD_OK;
    Workspace *ws = ws_of(c);
    packed = packed && ws->halo_fuse;
    const int64_t ns = ws->send_off[c->world];
    if (ns && !packed) ddk::launch_gather3(c, ns, ws->d_send_idx, x, ws->sendbuf, st);
    if (c->comm == DD_COMM_LOCAL) {
        if (!packed) return local_halo(c, st);
        // every producer has recorded xev_app after its fused apply
        LocalGroup *G = group_of(c);
        RENDEZVOUS(G);
        for (int q = 0; q < c->world; ++q)
            if (q != c->rank && c->recv_off[q + 1] > c->recv_off[q])
                CK(cudaStreamWaitEvent(st, ws_of(G->members[q])->xev_app, 0));
        return DD_OK;
    }
    auto comm = reinterpret_cast<ncclComm_t>(c->nccl);
    NK(ncclGroupStart());
    for (int q = 0; q < c->world; ++q) {
        if (q == c->rank) continue;
        const int64_t so = ws->send_off[q], sn = ws->send_off[q + 1] - so;
        const int64_t ro = c->recv_off[q], rn = c->recv_off[q + 1] - ro;
        if (sn) NK(ncclSend(ws->sendbuf + c->bs * so, c->bs * sn, ncclDouble, q, comm, st));
        if (rn) NK(ncclRecv(ws->xg + c->bs * ro, c->bs * rn, ncclDouble, q, comm, st));
    }
    NK(ncclGroupEnd());
    return DD_OK;
}

dd_status spmv_mode(dd_ctx *c, int mode, const double *x, double *y, const double *aux, const ddk::RedArgs &ra,
                    cudaStream_t st, bool packed = false) {
    TRY(halo(c, x, st, packed));
    ddk::launch_spmv(mode, c, x, ws_of(c)->xg, y, aux, ra, st);
    // DD_COMM_LOCAL with the fused halo: peers' next fused applies write this
    // rank's ghost block only after this SpMV has read it
    if (c->world > 1 && c->comm == DD_COMM_LOCAL && ws_of(c)->halo_fuse) CK(cudaEventRecord(ws_of(c)->xev_free, st));
    return DD_OK;
}

// The solver's apply r -> z with the fused halo epilogue (world > 1): the rows
// peers read in the following SpMV leave from shared memory. DD_COMM_LOCAL:
// the writes land in the peers' ghost blocks, so they wait until each
// consumer's previous SpMV has read its block (xev_free), and xev_app tells
// the consumers the rows are there.
dd_status apply_halo(dd_ctx *c, const double *r, double *z, cudaStream_t st, const int *skip) {
    Workspace *ws = ws_of(c);
    const bool fuse = c->world > 1 && ws->halo_fuse;
    const bool local = fuse && c->comm == DD_COMM_LOCAL;
    if (local) {
        LocalGroup *G = group_of(c);
        RENDEZVOUS(G);
        for (int q = 0; q < c->world; ++q)
            if (q != c->rank && ws->send_off[q + 1] > ws->send_off[q])
                CK(cudaStreamWaitEvent(st, ws_of(G->members[q])->xev_free, 0));
    }
    TRY(apply_launch(c, fuse ? DD_LEVELSET : c->solver_variant, r, z, reinterpret_cast<void *>(st), skip,
                     fuse ? &ws->hout : nullptr));
    if (local) CK(cudaEventRecord(ws->xev_app, st));
    return DD_OK;
}

dd_status read_scalars(dd_ctx *c, cudaStream_t st) {
    Workspace *ws = ws_of(c);
    CK(cudaMemcpyAsync(ws->h_sc, ws->sc, ddk::S_COUNT * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return DD_OK;
}

// device copies of the refactor maps (allocated at the first dd_refactor)
struct RfState {
    int32_t *SubLev = nullptr, *LevPtr = nullptr, *LevRows = nullptr, *Wcol = nullptr, *UpdQ = nullptr,
            *UpdT = nullptr, *Lst = nullptr, *Ust = nullptr, *Dst = nullptr;
    int64_t *Wrp = nullptr, *Wdiag = nullptr, *Uptr = nullptr, *Lrp = nullptr, *Urp = nullptr, *Loff = nullptr,
            *Uoff = nullptr, *Doff = nullptr, *Wsrc = nullptr, *Esrc = nullptr;
    double *W = nullptr, *Dinv = nullptr, *stage = nullptr;
    unsigned long long *bad = nullptr;
    unsigned long long *h_bad = nullptr;
};

template <class T>
dd_status upload_vec(T **d, const std::vector<T> &h) {
    TRY(dmalloc(d, std::max<size_t>(1, h.size())));
    if (!h.empty()) CK(cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return DD_OK;
}

dd_status refactor_init(dd_ctx *c) {
    if (c->rf) return DD_OK;
    auto *rf = new RfState();
    c->rf = rf;
    TRY(upload_vec(&rf->SubLev, c->SubLev));
    TRY(upload_vec(&rf->LevPtr, c->LevPtr));
    TRY(upload_vec(&rf->LevRows, c->LevRows));
    TRY(upload_vec(&rf->Wcol, c->Wcol));
    TRY(upload_vec(&rf->UpdQ, c->UpdQ));
    TRY(upload_vec(&rf->UpdT, c->UpdT));
    TRY(upload_vec(&rf->Lst, c->SlabLst));
    TRY(upload_vec(&rf->Ust, c->SlabUst));
    TRY(upload_vec(&rf->Dst, c->SlabDst));
    TRY(upload_vec(&rf->Wrp, c->Wrp));
    TRY(upload_vec(&rf->Wdiag, c->Wdiag));
    TRY(upload_vec(&rf->Uptr, c->Uptr));
    TRY(upload_vec(&rf->Lrp, c->Lrp));
    TRY(upload_vec(&rf->Urp, c->Urp));
    TRY(upload_vec(&rf->Loff, c->SlabLoff));
    TRY(upload_vec(&rf->Uoff, c->SlabUoff));
    TRY(upload_vec(&rf->Doff, c->SlabDoff));
    TRY(upload_vec(&rf->Wsrc, c->Wsrc));
    // sliced-ELL slot -> original block index (-1 = padding), same layout as device_setup
    {
        const int64_t nl = c->n_local;
        const auto &S = c->spmv;
        std::vector<int64_t> es(S.n_slots, -1);
        int64_t base = 0;
        for (int64_t s = 0; s < S.n_slices; ++s) {
            int64_t K = 0;
            for (int64_t li = 32 * s; li < std::min(nl, 32 * s + 32); ++li) K = std::max(K, c->Arp[li + 1] - c->Arp[li]);
            for (int lane = 0; lane < 32; ++lane) {
                const int64_t li = 32 * s + lane;
                if (li >= nl) break;
                for (int64_t k = 0; k < c->Arp[li + 1] - c->Arp[li]; ++k) es[base + 32 * k + lane] = c->Asrc[c->Arp[li] + k];
            }
            base += 32 * K;
        }
        TRY(upload_vec(&rf->Esrc, es));
    }
    TRY(dmalloc(&rf->W, 9 * std::max<size_t>(1, c->Wsrc.size())));
    TRY(dmalloc(&rf->Dinv, 9 * std::max<int64_t>(1, c->n_local)));
    TRY(dmalloc(&rf->stage, 9 * std::max<int64_t>(1, c->nnzb_A)));
    TRY(dmalloc(&rf->bad, 1));
    CK(cudaMallocHost(reinterpret_cast<void **>(&rf->h_bad), sizeof(unsigned long long)));
    return DD_OK;
}

void refactor_free(dd_ctx *c) {
    auto *rf = reinterpret_cast<RfState *>(c->rf);
    if (!rf) return;
    for (void *p : {(void *)rf->SubLev, (void *)rf->LevPtr, (void *)rf->LevRows, (void *)rf->Wcol, (void *)rf->UpdQ,
                    (void *)rf->UpdT, (void *)rf->Lst, (void *)rf->Ust, (void *)rf->Dst, (void *)rf->Wrp,
                    (void *)rf->Wdiag, (void *)rf->Uptr, (void *)rf->Lrp, (void *)rf->Urp, (void *)rf->Loff,
                    (void *)rf->Uoff, (void *)rf->Doff, (void *)rf->Wsrc, (void *)rf->Esrc, (void *)rf->W,
                    (void *)rf->Dinv, (void *)rf->stage, (void *)rf->bad})
        cudaFree(p);
    cudaFreeHost(rf->h_bad);
    delete rf;
    c->rf = nullptr;
}

bool usable(dd_ctx *c) {
    if (!c) {
        set_error("NULL context");
        return false;
    }
    if (c->host_only) {
        set_error("context was set up with host_only = 1");
        return false;
    }
    return true;
}

}  // namespace

extern "C" {

const char *dd_last_error(void) { return last_error_c(); }

dd_status dd_nccl_unique_id(void *out128) {
    if (!out128) return DD_E_INVALID_ARG;
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, sizeof id);
    return DD_OK;
}

static dd_status setup_common(const dd_bsr3 *A, const dd_opts *o, dd_ctx **out, int bs);

dd_status dd_setup(const dd_bsr3 *A, const dd_opts *o, dd_ctx **out) { return setup_common(A, o, out, 3); }

dd_status dd_setup_csr(const dd_csr *A, const dd_opts *o, dd_ctx **out) {
    if (!A) {
        if (out) *out = nullptr;
        set_error("dd_setup_csr: NULL argument");
        return DD_E_INVALID_ARG;
    }
    // same layout with 1x1 blocks: n_block_rows = n_rows, nnzb = nnz
    const dd_bsr3 B{A->n_rows, A->nnz, A->row_ptr, A->col_idx, A->vals};
    return setup_common(&B, o, out, 1);
}

static dd_status setup_common(const dd_bsr3 *A, const dd_opts *o, dd_ctx **out, int bs) {
    if (!out) {
        set_error("dd_setup: out is NULL");
        return DD_E_INVALID_ARG;
    }
    *out = nullptr;
    if (!A || !o) {
        set_error("dd_setup: NULL argument");
        return DD_E_INVALID_ARG;
    }
    auto *ctx = new dd_ctx();
    ctx->bs = bs;
    ctx->device = o->device;
    ctx->rank = o->rank;
    ctx->world = std::max(1, o->world);
    ctx->host_only = o->host_only != 0;
    ctx->comm = o->comm;
    if (ctx->comm != DD_COMM_NCCL && ctx->comm != DD_COMM_LOCAL) {
        set_error("dd_setup: unknown comm");
        delete ctx;
        return DD_E_INVALID_ARG;
    }
    if (ctx->rank < 0 || ctx->rank >= ctx->world || (ctx->world > 1 && !o->nccl_unique_id && !ctx->host_only)) {
        set_error("dd_setup: bad rank/world or missing nccl_unique_id");
        delete ctx;
        return DD_E_INVALID_ARG;
    }
    if (!ctx->host_only) {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            set_error("dd_setup: no CUDA device (set host_only for host-side setup only)");
            delete ctx;
            return DD_E_NO_DEVICE;
        }
    }
    dd_status st = host_setup(ctx, A, o);
    if (st == DD_OK && !ctx->host_only) st = device_setup(ctx, o->nccl_unique_id);
    if (st != DD_OK) {
        const std::string msg = last_error_c();
        dd_destroy(ctx);
        set_error(msg);
        return st;
    }
    *out = ctx;
    return DD_OK;
}

void dd_destroy(dd_ctx *c) {
    if (!c) return;
    if (!c->host_only) {
        cudaSetDevice(c->device);
        cudaDeviceSynchronize();
        local_leave(c);
        for (Slab *sl : {&c->slab_lvl, &c->slab_spin}) {
            cudaFree(sl->d_bytes);
            cudaFree(sl->d_info);
        }
        cudaFree(c->spmv.slot_ptr);
        cudaFree(c->spmv.cols);
        cudaFree(c->spmv.vals);
        cudaFree(c->d_new_to_old_local);
        cudaFree(c->d_stage);
        if (Workspace *ws = ws_of(c)) {
            for (double *q : {ws->r, ws->rh, ws->p, ws->v, ws->ph, ws->s, ws->sh, ws->t, ws->bd, ws->xd, ws->sc,
                              ws->loc, ws->gathered, ws->xg, ws->sendbuf})
                cudaFree(q);
            cudaFree(ws->partials);
            cudaFree(ws->counter);
            cudaFree(ws->ctl);
            cudaFree(ws->d_hist);
            cudaFreeHost(ws->h_ctl);
            cudaFreeHost(ws->h_tol);
            cudaFreeHost(ws->h_max);
            if (ws->gexec) cudaGraphExecDestroy(ws->gexec);
            if (ws->graph) cudaGraphDestroy(ws->graph);
            if (ws->cap) cudaStreamDestroy(ws->cap);
            for (auto e : ws->ev)
                if (e) cudaEventDestroy(e);
            for (auto e : {ws->xev_ready, ws->xev_done, ws->xev_app, ws->xev_free})
                if (e) cudaEventDestroy(e);
            cudaFree(ws->d_send_idx);
            cudaFree(ws->d_hptr);
            cudaFree(ws->d_hrow);
            cudaFree(ws->d_hdst);
            cudaFreeHost(ws->h_sc);
            delete ws;
        }
        if (c->nccl) ncclCommDestroy(reinterpret_cast<ncclComm_t>(c->nccl));
        refactor_free(c);
        if (c->prof) {
            for (auto e : reinterpret_cast<Prof *>(c->prof)->pool) cudaEventDestroy(e);
            delete reinterpret_cast<Prof *>(c->prof);
        }
    }
    delete c;
}

dd_status dd_local_range(const dd_ctx *c, int64_t *first, int64_t *n) {
    if (!c) return DD_E_INVALID_ARG;
    if (first) *first = c->row_first;
    if (n) *n = c->n_local;
    return DD_OK;
}

dd_status dd_apply_variant(dd_ctx *c, int32_t variant, const double *r, double *z, void *stream) {
    if (!usable(c)) return DD_E_INVALID_ARG;
    if ((!r || !z) && c->n_local) {
        set_error("dd_apply: NULL vector");
        return DD_E_INVALID_ARG;
    }
    return apply_launch(c, variant, r, z, stream);
}

dd_status dd_apply(dd_ctx *c, const double *r, double *z, void *stream) {
    return dd_apply_variant(c, DD_LEVELSET, r, z, stream);
}

dd_status dd_spmv(dd_ctx *c, const double *x, double *y, void *stream) {
    if (!usable(c)) return DD_E_INVALID_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    TRY(spmv_mode(c, ddk::SPMV_PLAIN, x, y, nullptr, red_args(c), st));
    CK(cudaGetLastError());
    return DD_OK;
}

// One Alg. 1 iteration (both half steps). k > 0: the host's iteration index;
// k < 0: graph mode, the kernels read it from ctl[C_ITER].
dd_status enqueue_iteration(dd_ctx *c, ddk::RedArgs ra, int k, double *x, cudaStream_t st) {
    Workspace *ws = ws_of(c);
    const int64_t m = ws->m;
    ra.k = k;
    TRY(timed(c, PK_BLAS, k, st, [&] {
        ddk::launch_update_p(c, m, k < 0 ? -1 : (k == 1), ws->r, ws->v, ws->p, ws->sc, ws->ctl, st);
        return DD_OK;
    }));
    TRY(timed(c, PK_APPLY, k, st, [&] { return apply_halo(c, ws->p, ws->ph, st, ws->ctl); }));
    TRY(timed(c, PK_SPMV, k, st, [&] { return spmv_mode(c, ddk::SPMV_SIGMA, ws->ph, ws->v, ws->rh, ra, st, true); }));
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
    TRY(timed(c, PK_APPLY, k, st, [&] { return apply_halo(c, ws->s, ws->sh, st, ws->ctl); }));
    TRY(timed(c, PK_SPMV, k, st, [&] { return spmv_mode(c, ddk::SPMV_TS_TT, ws->sh, ws->t, ws->s, ra, st, true); }));
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

// CUDA-graph solve loop: the iteration body captured once per
// solution vector under a conditional WHILE node, so a whole solve is one
// graph launch -- no host round trip per iteration or batch. Used for
// world == 1 when per-kernel profiling is off (DD_GRAPH=0 disables it).
dd_status graph_solve(dd_ctx *c, const ddk::RedArgs &ra, double *x, int32_t max_iter, cudaStream_t st,
                      int64_t *launches_per_iter) {
    Workspace *ws = ws_of(c);
    if (!ws->gexec || ws->gx != x || ws->ghist != ws->d_hist) {
        if (ws->gexec) cudaGraphExecDestroy(ws->gexec);
        if (ws->graph) cudaGraphDestroy(ws->graph);
        ws->gexec = nullptr;
        ws->graph = nullptr;
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
        const int64_t n0 = c->n_launches;
        CK(cudaStreamBeginCaptureToGraph(ws->cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        ddk::launch_iter_head(ws->ctl, ws->cap);
        dd_status e = enqueue_iteration(c, ra, -1, x, ws->cap);
        ddk::launch_iter_tail(ws->ctl, h, ws->cap);
        cudaGraph_t out = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(ws->cap, &out);
        if (e != DD_OK) return e;
        if (ce != cudaSuccess) {
            set_error(std::string("dd_bicgstab: graph capture failed: ") + cudaGetErrorString(ce));
            return DD_E_CUDA;
        }
        ws->g_launches = c->n_launches - n0;
        c->n_launches = n0;
        CK(cudaGraphInstantiate(&ws->gexec, ws->graph, 0));
        ws->gx = x;
        ws->ghist = ws->d_hist;
    }
    *ws->h_max = max_iter;
    CK(cudaMemcpyAsync(ws->ctl + ddk::C_MAX, ws->h_max, sizeof(int), cudaMemcpyHostToDevice, st));
    CK(cudaGraphLaunch(ws->gexec, st));
    *launches_per_iter = ws->g_launches;
    return DD_OK;
}

dd_status dd_bicgstab(dd_ctx *c, const double *b, double *x, double tol, int32_t max_iter, double *hist,
                      dd_report *rep, void *stream) {
    if (!usable(c)) return DD_E_INVALID_ARG;
    if (!(tol > 0) || max_iter < 1) {
        set_error("dd_bicgstab: tol must be > 0 and max_iter >= 1");
        return DD_E_INVALID_ARG;
    }
    const double t0 = now_ms();
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Workspace *ws = ws_of(c);
    const int64_t m = ws->m;
    if (ws->hist_cap < 2 * (int64_t)max_iter + 1) {
        cudaFree(ws->d_hist);
        ws->d_hist = nullptr;
        ws->hist_cap = 0;
        TRY(dmalloc(&ws->d_hist, 2 * (size_t)max_iter + 1));
        ws->hist_cap = 2 * (int64_t)max_iter + 1;
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

    // Alg. 1 iterations, enqueued in batches; every kernel returns at entry
    // once the device-side control has stopped. The host looks at the control
    // word one batch behind, so the GPU never idles on a half-step decision;
    // every rank waits on the same batch, so all ranks stop together.
    constexpr int BATCH = 2;
    int k_enq = 0, j = 0;
    static const bool graphs_env = !getenv("DD_GRAPH") || atoi(getenv("DD_GRAPH")) != 0;
    // world == 1 only: NCCL calls are capturable, but that path is not exercised on this pool
    const bool use_graph = graphs_env && c->world <= 1 && !(c->prof && reinterpret_cast<Prof *>(c->prof)->on);
    int64_t g_per_iter = 0;
    if (use_graph) TRY(graph_solve(c, ra, x, max_iter, st, &g_per_iter));
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
            CK(cudaEventSynchronize(ws->ev[(j - 1) % 2]));
            if (ws->h_ctl[8 * ((j - 1) % 2) + ddk::C_STATE] != ddk::ST_RUN) stop = true;
        }
        if (k_enq >= max_iter) stop = true;
    }
    CK(cudaMemcpyAsync(ws->h_ctl, ws->ctl, 8 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int state = ws->h_ctl[ddk::C_STATE], kf = ws->h_ctl[ddk::C_K], nh = ws->h_ctl[ddk::C_NH];
    if (use_graph) c->n_launches += g_per_iter * std::max(1, ws->h_ctl[ddk::C_ITER]) + 2 * std::max(1, ws->h_ctl[ddk::C_ITER]);
    std::vector<double> hv(std::max(1, nh));
    CK(cudaMemcpy(hv.data(), ws->d_hist, sizeof(double) * std::max(1, nh), cudaMemcpyDeviceToHost));
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
    TRY(read_scalars(c, st));
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

dd_status dd_refactor(dd_ctx *c, const double *vals, int32_t on_device, void *stream) {
    if (!usable(c) || !vals) return DD_E_INVALID_ARG;
    if (!c->refactor) {
        set_error("dd_refactor: context was set up without enable_refactor");
        return DD_E_INVALID_ARG;
    }
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    TRY(refactor_init(c));
    auto *rf = reinterpret_cast<RfState *>(c->rf);
    const double *src = vals;
    if (!on_device) {
        CK(cudaMemcpyAsync(rf->stage, vals, 9 * c->nnzb_A * sizeof(double), cudaMemcpyHostToDevice, st));
        src = rf->stage;
    }
    const int grid = c->num_sms * 8;
    ddk::launch_gather_blocks((int64_t)c->Wsrc.size(), rf->Wsrc, src, rf->W, 0, grid, st);
    ddk::launch_gather_blocks(c->spmv.n_slots, rf->Esrc, src, c->spmv.vals, 1, grid, st);
    *rf->h_bad = ~0ull;
    CK(cudaMemcpyAsync(rf->bad, rf->h_bad, sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
    ddk::RfArgs a{rf->SubLev, rf->LevPtr, rf->LevRows, rf->Wrp, rf->Wdiag, rf->Uptr, rf->Lrp, rf->Urp,
                  rf->Wcol, rf->UpdQ, rf->UpdT, rf->W, rf->Dinv, c->slab_lvl.d_bytes, rf->Loff, rf->Uoff, rf->Doff,
                  rf->Lst, rf->Ust, rf->Dst, c->pivot_floor, rf->bad, c->row_first};
    const int nsl = c->sub_last - c->sub_first;
    if (nsl > 0) ddk::launch_refactor(nsl, a, st);
    c->n_launches += 3;
    CK(cudaMemcpyAsync(rf->h_bad, rf->bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    if (*rf->h_bad != ~0ull) {
        set_error("dd_refactor: singular pivot block (|det| < pivot_floor) at reordered row " +
                  std::to_string(*rf->h_bad));
        return DD_E_SINGULAR_PIVOT;
    }
    return DD_OK;
}

dd_status dd_permute(dd_ctx *c, const double *v_orig_host, double *v_reord_dev, void *stream) {
    if (!usable(c) || !v_orig_host || !v_reord_dev) return DD_E_INVALID_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CK(cudaMemcpyAsync(c->d_stage, v_orig_host, c->bs * c->N * sizeof(double), cudaMemcpyHostToDevice, st));
    ddk::launch_gather3(c, c->n_local, reinterpret_cast<const int32_t *>(c->d_new_to_old_local), c->d_stage,
                        v_reord_dev, st);
    CK(cudaGetLastError());
    return DD_OK;
}

dd_status dd_unpermute(dd_ctx *c, const double *v_reord_dev, double *v_orig_host, void *stream) {
    if (!usable(c) || !v_orig_host || !v_reord_dev) return DD_E_INVALID_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (c->world <= 1) {
        ddk::launch_scatter3(c, c->n_local, reinterpret_cast<const int32_t *>(c->d_new_to_old_local), v_reord_dev,
                             c->d_stage, st);
        CK(cudaMemcpyAsync(v_orig_host, c->d_stage, c->bs * c->N * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    } else {
        const int bs = c->bs;
        std::vector<double> tmp(bs * c->n_local);
        CK(cudaMemcpyAsync(tmp.data(), v_reord_dev, tmp.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int64_t li = 0; li < c->n_local; ++li) {
            const int64_t g = c->new_to_old[c->row_first + li];
            for (int q = 0; q < bs; ++q) v_orig_host[bs * g + q] = tmp[bs * li + q];
        }
    }
    return DD_OK;
}

dd_status dd_solve_host(dd_ctx *c, const double *b_host, double *x_host, double tol, int32_t max_iter,
                        dd_report *rep, void *stream) {
    if (!usable(c)) return DD_E_INVALID_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Workspace *ws = ws_of(c);
    TRY(dd_permute(c, b_host, ws->bd, stream));
    CK(cudaMemsetAsync(ws->xd, 0, ws->m * sizeof(double), st));
    dd_status s = dd_bicgstab(c, ws->bd, ws->xd, tol, max_iter, nullptr, rep, stream);
    if (s != DD_OK && s != DD_E_BREAKDOWN && s != DD_E_MAXITER) return s;
    TRY(dd_unpermute(c, ws->xd, x_host, stream));
    return s;
}

dd_status dd_get_partition(const dd_ctx *c, int32_t *labels, int32_t *new_to_old) {
    if (!c) return DD_E_INVALID_ARG;
    if (labels) std::memcpy(labels, c->labels.data(), c->N * sizeof(int32_t));
    if (new_to_old) std::memcpy(new_to_old, c->new_to_old.data(), c->N * sizeof(int32_t));
    return DD_OK;
}

dd_status dd_get_levels(const dd_ctx *c, int32_t which, int32_t *hmap) {
    if (!c || !hmap || (which != 0 && which != 1)) return DD_E_INVALID_ARG;
    const auto &h = which == 0 ? c->hmapL : c->hmapU;
    std::memcpy(hmap, h.data(), h.size() * sizeof(int32_t));
    return DD_OK;
}

dd_status dd_levels_device(dd_ctx *c, int32_t *hmapL, int32_t *hmapU, double *ms) {
    if (!usable(c)) return DD_E_INVALID_ARG;
    CK(cudaSetDevice(c->device));
    const int nsl = c->sub_last - c->sub_first;
    const int64_t nl = c->n_local;
    std::vector<int64_t> sub(nsl + 1);
    for (int q = 0; q <= nsl; ++q) sub[q] = c->sub_ptr[c->sub_first + q] - c->row_first;
    int64_t *d_sub = nullptr, *d_rp = nullptr;
    int32_t *d_ci = nullptr, *d_h = nullptr;
    const int64_t nci = std::max<int64_t>(1, std::max(c->Lci.size(), c->Uci.size()));
    dd_status st = DD_OK;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    float tot = 0.0f;
    do {
        if ((st = dmalloc(&d_sub, nsl + 1)) != DD_OK || (st = dmalloc(&d_rp, nl + 1)) != DD_OK ||
            (st = dmalloc(&d_ci, nci)) != DD_OK || (st = dmalloc(&d_h, std::max<int64_t>(1, nl))) != DD_OK)
            break;
        if (cudaMemcpy(d_sub, sub.data(), sub.size() * sizeof(int64_t), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
            set_error("dd_levels_device: CUDA setup failed");
            st = DD_E_CUDA;
            break;
        }
        for (int which = 0; which < 2 && st == DD_OK; ++which) {
            const auto &rp = which == 0 ? c->Lrp : c->Urp;
            const auto &ci = which == 0 ? c->Lci : c->Uci;
            int32_t *out = which == 0 ? hmapL : hmapU;
            cudaMemcpy(d_rp, rp.data(), (nl + 1) * sizeof(int64_t), cudaMemcpyHostToDevice);
            if (!ci.empty()) cudaMemcpy(d_ci, ci.data(), ci.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
            cudaEventRecord(e0);
            if (nsl) ddk::launch_levels(nsl, d_sub, d_rp, d_ci, d_h, c->max_P, nullptr);
            cudaEventRecord(e1);
            if (cudaEventSynchronize(e1) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
                set_error("dd_levels_device: kernel failed");
                st = DD_E_CUDA;
                break;
            }
            float t = 0.0f;
            cudaEventElapsedTime(&t, e0, e1);
            tot += t;
            if (out && nl) cudaMemcpy(out, d_h, nl * sizeof(int32_t), cudaMemcpyDeviceToHost);
        }
    } while (0);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    cudaFree(d_sub);
    cudaFree(d_rp);
    cudaFree(d_ci);
    cudaFree(d_h);
    if (ms) *ms = tot;
    return st;
}

dd_status dd_get_factors(const dd_ctx *c, int64_t *nL, int64_t *nU, int64_t *Lrp, int32_t *Lci, double *Lv,
                         int64_t *Urp, int32_t *Uci, double *Uv, double *Dinv) {
    if (!c) return DD_E_INVALID_ARG;
    if (nL) *nL = (int64_t)c->Lci.size();
    if (nU) *nU = (int64_t)c->Uci.size();
    if (Lrp) std::memcpy(Lrp, c->Lrp.data(), c->Lrp.size() * sizeof(int64_t));
    if (Lci) std::memcpy(Lci, c->Lci.data(), c->Lci.size() * sizeof(int32_t));
    if (Lv) std::memcpy(Lv, c->Lv.data(), c->Lv.size() * sizeof(double));
    if (Urp) std::memcpy(Urp, c->Urp.data(), c->Urp.size() * sizeof(int64_t));
    if (Uci) std::memcpy(Uci, c->Uci.data(), c->Uci.size() * sizeof(int32_t));
    if (Uv) std::memcpy(Uv, c->Uv.data(), c->Uv.size() * sizeof(double));
    if (Dinv) std::memcpy(Dinv, c->Dinv.data(), c->Dinv.size() * sizeof(double));
    return DD_OK;
}

dd_status dd_get_halo(const dd_ctx *c, int64_t *n_ghost, int64_t *ghost_rows, int32_t *ghost_owner) {
    if (!c) return DD_E_INVALID_ARG;
    if (n_ghost) *n_ghost = (int64_t)c->ghost_rows.size();
    if (ghost_rows) std::memcpy(ghost_rows, c->ghost_rows.data(), c->ghost_rows.size() * sizeof(int64_t));
    if (ghost_owner) std::memcpy(ghost_owner, c->ghost_owner.data(), c->ghost_owner.size() * sizeof(int32_t));
    return DD_OK;
}

dd_status dd_get_send_rows(const dd_ctx *c, int32_t peer, int64_t *n, int32_t *rows) {
    if (!c || peer < 0 || peer >= c->world) return DD_E_INVALID_ARG;
    static const std::vector<int32_t> none;
    const auto &v = peer < (int)c->send_rows.size() ? c->send_rows[peer] : none;
    if (n) *n = (int64_t)v.size();
    if (rows) std::memcpy(rows, v.data(), v.size() * sizeof(int32_t));
    return DD_OK;
}

dd_status dd_stats(const dd_ctx *c, int64_t *stats, double *setup_ms) {
    if (!c) return DD_E_INVALID_ARG;
    if (stats) {
        const int64_t nL = (int64_t)c->Lci.size(), nU = (int64_t)c->Uci.size(), nl = c->n_local;
        int64_t slab_l = 0, slab_s = 0;
        for (auto &i : c->slab_lvl.info) slab_l += i.stream_bytes;
        for (auto &i : c->slab_spin.info) slab_s += i.stream_bytes;
        stats[0] = c->nnzb_A;
        stats[1] = c->nnzb_dd;
        stats[2] = c->n_sub;
        stats[3] = c->sub_last - c->sub_first;
        stats[4] = c->max_lev_L;
        stats[5] = c->max_lev_U;
        stats[6] = c->max_P;
        stats[7] = slab_l;
        stats[8] = slab_s;
        stats[9] = c->spmv_bytes;
        // canonical bytes: 8 b2 (nL+nU+n) + 4(nL+nU) + 4*2(n+1) + 16 bs n
        // (BSR3: 72(nL+nU+n) + 4(nL+nU) + 8(n+1) + 48n)
        const int64_t b2 = (int64_t)c->bs * c->bs;
        stats[10] = 8 * b2 * (nL + nU + nl) + 4 * (nL + nU) + 8 * (nl + 1) + 16 * c->bs * nl;
        const int64_t nnzA_loc = c->Arp.empty() ? 0 : c->Arp.back();
        stats[11] = (8 * b2 + 4) * nnzA_loc + 4 * (nl + 1) + 16 * c->bs * nl;
        stats[12] = nl;
        stats[13] = (int64_t)c->ghost_rows.size();
        stats[14] = c->n_launches;
        stats[15] = 0;
    }
    if (setup_ms)
        for (int q = 0; q < 6; ++q) setup_ms[q] = c->setup_ms[q];
    return DD_OK;
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

dd_status dd_solver_variant(const dd_ctx *c, int32_t *variant, double *ms) {
    if (!c) return DD_E_INVALID_ARG;
    if (variant) *variant = c->solver_variant;
    if (ms)
        for (int q = 0; q < 3; ++q) ms[q] = c->variant_ms[q];
    return DD_OK;
}

dd_status dd_launch_info(const dd_ctx *c, int32_t variant, int64_t *info) {
    if (!c || !info) return DD_E_INVALID_ARG;
    const LaunchCfg *l = variant == DD_SPINLOOP ? &c->cfg_spin : variant == DD_DIRECT ? &c->cfg_direct : &c->cfg_lvl;
    info[0] = l->grid;
    info[1] = l->threads;
    info[2] = l->smem;
    info[3] = l->ring;
    return DD_OK;
}

}  // extern "C"
