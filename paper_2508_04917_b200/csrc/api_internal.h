// api_internal.h -- declarations shared by the C-ABI translation units
// (api.cpp: context lifetime, setup, apply / SpMV entry points and
// introspection; comm.cpp: transports for world > 1; solver.cpp: the
// BiCGSTAB driver; refactor_api.cpp: GPU re-factorisation). Product-internal.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "dd_internal.h"
#include "krylov.cuh"
#include "peer.cuh"

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            ddi::set_error(std::string(#x) + ": " + cudaGetErrorString(e_));                    \
            return e_ == cudaErrorMemoryAllocation ? DD_E_OOM : DD_E_CUDA;                      \
        }                                                                                       \
    } while (0)

#define TRY(x)                        \
    do {                              \
        dd_status s_ = (x);           \
        if (s_ != DD_OK) return s_;   \
    } while (0)

namespace ddi {

const char *last_error_c();

template <class T>
dd_status dmalloc(T **p, size_t count) {
    *p = nullptr;
    if (count == 0) return DD_OK;
    CK(cudaMalloc(reinterpret_cast<void **>(p), count * sizeof(T)));
    return DD_OK;
}

// host -> device copy of a large pageable buffer through pinned staging (api.cpp)
dd_status h2d_big(void *dst, const void *src, size_t bytes);

template <class T, class A>
dd_status upload_vec(T **d, const std::vector<T, A> &h) {
    TRY(dmalloc(d, std::max<size_t>(1, h.size())));
    if (!h.empty()) TRY(h2d_big(*d, h.data(), h.size() * sizeof(T)));
    return DD_OK;
}

struct Workspace {
    int64_t m = 0;  // bs * n_local
    double *vecs = nullptr;  // one allocation holding the ten vectors below
    double *r = nullptr, *rh = nullptr, *p = nullptr, *v = nullptr, *ph = nullptr, *s = nullptr, *sh = nullptr,
           *t = nullptr, *bd = nullptr, *xd = nullptr;
    double *sc = nullptr;        // device scalars [S_COUNT]
    void *partials = nullptr;    // DD [grid * 2]
    unsigned int *counter = nullptr;
    double *loc = nullptr;       // [6] rank-local (s, c) pairs
    double *gathered = nullptr;  // NCCL: [world * 6]
    double *h_sc = nullptr;      // pinned [S_COUNT]
    int *ctl = nullptr;          // device solver control [8]
    int *h_ctl = nullptr;        // pinned [16]: two snapshots
    double *d_hist = nullptr;    // device residual history
    int64_t hist_cap = 0;
    double *h_tol = nullptr;     // pinned scalar (tolerance upload)
    cudaEvent_t ev[2] = {nullptr, nullptr};
    double *xg = nullptr;        // ghost rows of the SpMV input [bs * n_ghost] (peer transports: inside box)
    // ---- NCCL transport
    double *sendbuf = nullptr;   // [bs * total send rows]
    int32_t *d_send_idx = nullptr;
    std::vector<int64_t> send_off;  // [world + 1]
    // ---- fused halo (world > 1): the solver's applies write the rows peers
    // need straight from shared memory (NCCL: into the send buffer; peer
    // transports: into the consumer's ghost block)
    bool halo_fuse = false;
    bool merge_ss = false;  // world > 1: s.s reduced with (t.s, t.t)
    ddi::HaloOut hout;
    int32_t *d_hptr = nullptr, *d_hrow = nullptr;
    double **d_hdst = nullptr;
    // ---- DD_COMM_LOCAL: the group's contexts and the exchange events
    std::vector<dd_ctx *> local_peers;
    cudaEvent_t xev_ready = nullptr, xev_done = nullptr, xev_app = nullptr, xev_free = nullptr;
    // ---- peer-memory transport (DD_COMM_IPC, peer.cuh)
    uint8_t *box = nullptr;              // own mailbox: flags | gathered | xg
    int64_t box_bytes = 0;
    std::vector<uint8_t *> peer_box;     // [world] mailboxes mapped here (own at [rank])
    std::vector<bool> peer_opened;       // [world] opened with cudaIpcOpenMemHandle
    uint8_t **d_boxes = nullptr;
    uint64_t *seq = nullptr;             // [2 * PCH_COUNT]
    int *perr = nullptr;                 // wait timeout flag
    int32_t *d_send_to = nullptr, *d_recv_from = nullptr;
    int n_send_to = 0, n_recv_from = 0;
    int32_t *d_put_rows = nullptr;       // unfused halo: local row -> peer ghost address
    double **d_put_dst = nullptr;
    int64_t n_put = 0;
    ddk::PeerDev pd;
    // ---- CUDA-graph solve loop (one executable graph per solution vector)
    cudaStream_t cap = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    double *gx = nullptr, *ghist = nullptr;  // the captured body's x and history buffers
    int64_t g_launches = 0;
    int *h_max = nullptr;  // pinned
};

inline Workspace *ws_of(dd_ctx *c) { return reinterpret_cast<Workspace *>(c->dev_ws); }

// Every compute entry point runs on the context's device and restores the
// caller's current device on return.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = cudaSetDevice(dev) == cudaSuccess;
        if (!ok) cudaGetLastError();
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
#define DEVICE_GUARD(c)                                                  \
    ddi::DeviceGuard dg_((c)->device);                                   \
    if (!dg_.ok) {                                                       \
        ddi::set_error("cudaSetDevice failed for the context's device"); \
        return DD_E_CUDA;                                                \
    }

bool peer_comm(const dd_ctx *c);  // world > 1 with DD_COMM_IPC (device-flag transport)

// ---- comm.cpp
// After the host setup: create the NCCL communicator / join the rendezvous
// group, then agree on the status over all ranks (every rank returns the
// same status; a failing rank never leaves its peers waiting).
dd_status comm_begin(dd_ctx *c, const void *key, dd_status host_status);
dd_status comm_agree(dd_ctx *c, dd_status st);
// allocate the ghost block (peer transports: the mailbox) and the send lists
dd_status comm_alloc(dd_ctx *c);
// map every peer's mailbox, build the halo destinations (collective)
dd_status comm_connect(dd_ctx *c);
void comm_end(dd_ctx *c);  // dd_destroy (collective for the peer transports)
// halo exchange of the SpMV input x into xg. packed: x came from a fused-halo
// apply (apply_halo), which already wrote the rows peers need
dd_status halo(dd_ctx *c, const double *x, cudaStream_t st, bool packed, const int *skip);
// after the SpMV that read xg (peer transports: producers may write again)
dd_status halo_consumed(dd_ctx *c, cudaStream_t st, const int *skip);
// the solver's apply r -> z with the fused halo epilogue when world > 1
dd_status apply_halo(dd_ctx *c, const double *r, double *z, cudaStream_t st, const int *skip);
// rank-local (s, c) pairs in loc -> combined over ranks in rank order -> finalize op
dd_status reduce_across(dd_ctx *c, int nv, int op, const ddk::RedArgs &ra, cudaStream_t st);
// host wait for an event recorded on the solver stream; with NCCL polls
// ncclCommGetAsyncError (aborts the communicator and fails on an error)
dd_status comm_wait_event(dd_ctx *c, cudaEvent_t ev);
// after a synchronisation: a peer wait that timed out -> DD_E_NCCL
dd_status comm_check(dd_ctx *c, cudaStream_t st);
// the iteration body can be captured into a CUDA graph (world 1, DD_COMM_IPC)
bool comm_graph_ok(const dd_ctx *c);

// ---- api.cpp
ddk::RedArgs red_args(dd_ctx *c);
dd_status spmv_mode(dd_ctx *c, int mode, const double *x, double *y, const double *aux, const ddk::RedArgs &ra,
                    cudaStream_t st, bool packed = false, const int *skip = nullptr);
bool usable(dd_ctx *c);

// ---- refactor_api.cpp
void refactor_free(dd_ctx *c);
// numeric factorisation of new values on the device (dd_refactor's body; the
// GPU numeric path of dd_setup calls it with the matrix's own values)
dd_status refactor_values(dd_ctx *c, const double *vals, bool on_device, cudaStream_t st);
// the device factor state: W (L blocks, U_ii, U_ij per row in the dropped
// pattern) and Dinv, for dd_get_factors on the GPU numeric path
dd_status refactor_fetch(const dd_ctx *c, std::vector<double> &W, std::vector<double> &Dinv);

// ---- solver.cpp
void prof_free(dd_ctx *c);
// device history + the captured solve graph (dd_setup, after the transport
// is connected and the solver's apply variant is chosen)
dd_status solver_prepare(dd_ctx *c);

}  // namespace ddi
