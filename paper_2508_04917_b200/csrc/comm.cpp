// comm.cpp -- the exchange steps of the multi-rank solver (SURVEY 8(e),
// P:730-734 extended to BiCGSTAB): the SpMV halo and the all-gather of the
// double-double dot partials, over three transports (dd.h):
//   DD_COMM_NCCL  grouped ncclSend/ncclRecv + ncclAllGather, async errors polled
//   DD_COMM_IPC   peer memory between processes (CUDA IPC handles), device flags
//   DD_COMM_LOCAL contexts of one process: device-to-device copies ordered by
//                 CUDA events and a host rendezvous per exchange
// plus the host rendezvous (setup / refactor / destroy only) that agrees on
// a status over the ranks and exchanges the mailbox addresses.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "api_internal.h"

#define NK(x)                                                                                   \
    do {                                                                                        \
        ncclResult_t r_ = (x);                                                                  \
        if (r_ != ncclSuccess) {                                                                \
            set_error(std::string(#x) + ": " + ncclGetErrorString(r_));                         \
            return DD_E_NCCL;                                                                   \
        }                                                                                       \
    } while (0)

namespace ddi {

namespace {

double timeout_s() {
    const char *e = getenv("DD_PEER_TIMEOUT_S");
    const double v = e ? atof(e) : 120.0;
    return v > 0 ? v : 120.0;
}

// ------------------------------------------------------------ rendezvous
// allgather of one fixed-size blob per rank (at most SLOT bytes), rank order;
// false on a timeout (the group is then broken for every rank)
constexpr size_t SLOT = 4096;
constexpr int MAX_WORLD_IPC = 256;

class Rendezvous {
   public:
    virtual ~Rendezvous() = default;
    virtual bool allgather(const void *mine, size_t bytes, std::vector<uint8_t> &all) = 0;
    virtual void setup_done() {}
    bool barrier() {
        std::vector<uint8_t> all;
        const int z = 0;
        return allgather(&z, sizeof z, all);
    }
};

// DD_COMM_LOCAL: ranks are threads of this process. Slots are double-buffered
// by the generation parity: a rank can only be one allgather ahead of the
// slowest, which has already copied the previous generation's slots.
struct LocalGroup {
    int world = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0, refs = 0;
    uint64_t gen = 0;
    bool broken = false;
    std::vector<uint8_t> slots[2];
};
std::mutex g_groups_m;
std::map<std::string, LocalGroup *> g_groups;

class LocalRdv : public Rendezvous {
   public:
    LocalRdv(LocalGroup *g, std::string key, int rank) : G(g), key_(std::move(key)), rank_(rank) {}
    ~LocalRdv() override {
        std::lock_guard<std::mutex> lk(g_groups_m);
        if (--G->refs == 0) {
            g_groups.erase(key_);
            delete G;
        }
    }
    bool allgather(const void *mine, size_t bytes, std::vector<uint8_t> &all) override {
        std::unique_lock<std::mutex> lk(G->m);
        if (G->broken || bytes > SLOT) return false;
        const uint64_t g = G->gen;
        std::vector<uint8_t> &buf = G->slots[g & 1];
        std::memcpy(&buf[SLOT * rank_], mine, bytes);
        if (++G->arrived == G->world) {
            G->arrived = 0;
            ++G->gen;
            G->cv.notify_all();
        } else {
            const bool ok = G->cv.wait_for(lk, std::chrono::duration<double>(timeout_s()),
                                           [&] { return G->gen != g || G->broken; });
            if (!ok || G->broken) {
                G->broken = true;  // a late arrival must not complete a part-counted barrier
                G->cv.notify_all();
                return false;
            }
        }
        all.resize(G->world * bytes);
        for (int q = 0; q < G->world; ++q) std::memcpy(&all[q * bytes], &buf[SLOT * q], bytes);
        return true;
    }

   private:
    LocalGroup *G;
    std::string key_;
    int rank_;
};

Rendezvous *local_join(const void *key, int world, int rank) {
    std::lock_guard<std::mutex> lk(g_groups_m);
    const std::string k(reinterpret_cast<const char *>(key), 128);
    auto it = g_groups.find(k);
    LocalGroup *G;
    if (it == g_groups.end()) {
        G = new LocalGroup();
        G->world = world;
        G->slots[0].assign(SLOT * world, 0);
        G->slots[1].assign(SLOT * world, 0);
        g_groups[k] = G;
    } else {
        G = it->second;
        if (G->world != world) {
            set_error("dd_setup: DD_COMM_LOCAL group key reused with another world size");
            return nullptr;
        }
    }
    ++G->refs;
    return new LocalRdv(G, k, rank);
}

// DD_COMM_IPC: ranks are processes of one node. POSIX shared memory named by
// the key; the kernel zero-fills a new segment, which is the initial state.
struct ShmHdr {
    std::atomic<uint32_t> arrived;
    std::atomic<uint32_t> broken;
    std::atomic<uint64_t> gen;
};
static_assert(std::atomic<uint64_t>::is_always_lock_free, "process-shared atomics");

class ShmRdv : public Rendezvous {
   public:
    static ShmRdv *join(const void *key, int world, int rank) {
        const uint8_t *k = reinterpret_cast<const uint8_t *>(key);
        char name[64];
        int n = snprintf(name, sizeof name, "/dd_rdv_%d_", world);
        for (int q = 0; q < 12; ++q) n += snprintf(name + n, sizeof name - n, "%02x", k[q]);
        const size_t bytes = 64 + 2 * SLOT * (size_t)world;
        const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
        if (fd < 0) {
            set_error(std::string("dd_setup: shm_open failed for the DD_COMM_IPC rendezvous: ") + strerror(errno));
            return nullptr;
        }
        if (ftruncate(fd, (off_t)bytes) != 0) {
            close(fd);
            set_error("dd_setup: ftruncate of the DD_COMM_IPC rendezvous failed");
            return nullptr;
        }
        void *p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (p == MAP_FAILED) {
            set_error("dd_setup: mmap of the DD_COMM_IPC rendezvous failed");
            return nullptr;
        }
        auto *r = new ShmRdv();
        r->name_ = name;
        r->base_ = reinterpret_cast<uint8_t *>(p);
        r->bytes_ = bytes;
        r->world_ = world;
        r->rank_ = rank;
        return r;
    }
    ~ShmRdv() override {
        munmap(base_, bytes_);
        if (!unlinked_ && rank_ == 0) shm_unlink(name_.c_str());
    }
    // every rank has mapped the segment (it passed a barrier): the name can go
    void setup_done() override {
        if (rank_ == 0 && !unlinked_) shm_unlink(name_.c_str());
        unlinked_ = true;
    }
    bool allgather(const void *mine, size_t bytes, std::vector<uint8_t> &all) override {
        ShmHdr *h = reinterpret_cast<ShmHdr *>(base_);
        if (bytes > SLOT || h->broken.load()) return false;
        const uint64_t g = h->gen.load(std::memory_order_acquire);
        uint8_t *buf = base_ + 64 + (g & 1) * SLOT * world_;
        std::memcpy(buf + SLOT * rank_, mine, bytes);
        if ((int)h->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == world_) {
            h->arrived.store(0, std::memory_order_relaxed);
            h->gen.fetch_add(1, std::memory_order_acq_rel);
        } else {
            const auto t0 = std::chrono::steady_clock::now();
            const double lim = timeout_s();
            while (h->gen.load(std::memory_order_acquire) == g) {
                if (h->broken.load()) return false;
                if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > lim) {
                    h->broken.store(1);
                    return false;
                }
                std::this_thread::sleep_for(std::chrono::microseconds(50));
            }
        }
        all.resize(world_ * bytes);
        for (int q = 0; q < world_; ++q) std::memcpy(&all[q * bytes], buf + SLOT * q, bytes);
        return true;
    }

   private:
    std::string name_;
    uint8_t *base_ = nullptr;
    size_t bytes_ = 0;
    int world_ = 0, rank_ = 0;
    bool unlinked_ = false;
};

Rendezvous *rdv_of(const dd_ctx *c) { return reinterpret_cast<Rendezvous *>(c->rdv); }
ncclComm_t nccl_of(const dd_ctx *c) { return reinterpret_cast<ncclComm_t>(c->nccl); }

const char *status_name(int s) {
    static const char *n[] = {"DD_OK", "DD_E_INVALID_ARG", "DD_E_NOT_SQUARE", "DD_E_UNSORTED_OR_DUP",
                              "DD_E_MISSING_DIAG", "DD_E_SINGULAR_PIVOT", "DD_E_SUBDOMAIN_TOO_LARGE",
                              "DD_E_GRID_NOT_DIVISIBLE", "DD_E_CUDA", "DD_E_NCCL", "DD_E_OOM",
                              "DD_E_BREAKDOWN", "DD_E_MAXITER", "DD_E_NO_DEVICE"};
    return s >= 0 && s < (int)(sizeof n / sizeof *n) ? n[s] : "?";
}

// The fused halo lists: for every local subdomain, the rows
// that peers read (send_rows, ascending per peer) and the address each goes
// to; dst_of(q, p) = destination of the p-th row sent to peer q. Also the
// flat (row, address) list of the unfused put (peer transports).
template <class F>
dd_status halo_lists_build(dd_ctx *ctx, F dst_of, bool flat) {
    Workspace *ws = ws_of(ctx);
    const int nsl = ctx->sub_last - ctx->sub_first;
    struct Ent {
        int32_t sub, row, li;
        double *dst;
    };
    std::vector<Ent> ents;
    for (int q = 0; q < ctx->world; ++q) {
        if (q == ctx->rank || q >= (int)ctx->send_rows.size()) continue;
        const auto &rows = ctx->send_rows[q];
        for (size_t p = 0; p < rows.size(); ++p) {
            const int64_t g = ctx->row_first + rows[p];  // reordered global row
            const int32_t s = (int32_t)(std::upper_bound(ctx->sub_ptr.begin() + ctx->sub_first,
                                                         ctx->sub_ptr.begin() + ctx->sub_last + 1, g) -
                                        ctx->sub_ptr.begin()) - 1;
            ents.push_back({s - ctx->sub_first, (int32_t)(g - ctx->sub_ptr[s]), rows[p], dst_of(q, (int64_t)p)});
        }
    }
    if (flat) {
        std::vector<int32_t> li(ents.size());
        std::vector<double *> d(ents.size());
        for (size_t e = 0; e < ents.size(); ++e) {
            li[e] = ents[e].li;
            d[e] = ents[e].dst;
        }
        TRY(upload_vec(&ws->d_put_rows, li));
        TRY(upload_vec(&ws->d_put_dst, d));
        ws->n_put = (int64_t)ents.size();
    }
    if (!ws->halo_fuse) return DD_OK;
    std::stable_sort(ents.begin(), ents.end(), [](const Ent &a, const Ent &b) { return a.sub < b.sub; });
    std::vector<int32_t> ptr(nsl + 1, 0), row(ents.size());
    std::vector<double *> dst(ents.size());
    for (size_t e = 0; e < ents.size(); ++e) {
        ++ptr[ents[e].sub + 1];
        row[e] = ents[e].row;
        dst[e] = ents[e].dst;
    }
    for (int s = 0; s < nsl; ++s) ptr[s + 1] += ptr[s];
    TRY(upload_vec(&ws->d_hptr, ptr));
    TRY(upload_vec(&ws->d_hrow, row));
    TRY(upload_vec(&ws->d_hdst, dst));
    ws->hout = ddi::HaloOut{ws->d_hptr, ws->d_hrow, ws->d_hdst};
    return DD_OK;
}

// one slot of the connect exchange (peer transports)
struct PeerSlot {
    int32_t status, device;
    int64_t pid;
    uint64_t raw;  // DD_COMM_LOCAL: the mailbox pointer
    cudaIpcMemHandle_t handle;
    int64_t recv_off[MAX_WORLD_IPC + 1];
};
static_assert(sizeof(PeerSlot) <= SLOT, "rendezvous slot size");

int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }

}  // namespace

bool peer_comm(const dd_ctx *c) { return c->world > 1 && c->comm == DD_COMM_IPC; }
static bool local_comm(const dd_ctx *c) { return c->world > 1 && c->comm == DD_COMM_LOCAL; }

dd_status comm_agree(dd_ctx *c, dd_status st) {
    if (c->world <= 1 || c->host_only) return st;
    int agreed = (int)st;
    if (c->comm == DD_COMM_NCCL) {
        if (!c->nccl) return st;
        int *d = nullptr;
        cudaStream_t s = nullptr;
        CK(cudaMalloc(&d, sizeof(int)));
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        const int mine = (int)st;
        cudaMemcpyAsync(d, &mine, sizeof(int), cudaMemcpyHostToDevice, s);
        const ncclResult_t r = ncclAllReduce(d, d, 1, ncclInt, ncclMax, nccl_of(c), s);
        cudaMemcpyAsync(&agreed, d, sizeof(int), cudaMemcpyDeviceToHost, s);
        const cudaError_t e = cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
        cudaFree(d);
        if (r != ncclSuccess || e != cudaSuccess) {
            set_error("dd_setup: status all-reduce failed");
            return DD_E_NCCL;
        }
    } else {
        Rendezvous *R = rdv_of(c);
        std::vector<uint8_t> all;
        const int32_t mine = (int32_t)st;
        if (!R || !R->allgather(&mine, sizeof mine, all)) {
            set_error("peer transport: host rendezvous timed out (every rank must make the same collective calls)");
            return DD_E_NCCL;
        }
        for (int q = 0; q < c->world; ++q) {
            int32_t v;
            std::memcpy(&v, &all[4 * q], 4);
            agreed = std::max(agreed, (int)v);
        }
    }
    if (st == DD_OK && agreed != DD_OK)
        set_error(std::string("a peer rank failed with ") + status_name(agreed) + " (status agreed over the ranks)");
    return (dd_status)agreed;
}

dd_status comm_begin(dd_ctx *c, const void *key, dd_status host_status) {
    if (c->world <= 1 || c->host_only) return host_status;
    CK(cudaSetDevice(c->device));
    if (c->comm == DD_COMM_NCCL) {
        ncclComm_t comm;
        ncclUniqueId id;
        std::memcpy(&id, key, sizeof id);
        NK(ncclCommInitRank(&comm, c->world, id, c->rank));
        c->nccl = comm;
    } else {
        if (c->comm == DD_COMM_IPC && c->world > MAX_WORLD_IPC) {
            set_error("dd_setup: DD_COMM_IPC supports at most 256 ranks");
            return DD_E_INVALID_ARG;
        }
        Rendezvous *R = c->comm == DD_COMM_LOCAL ? local_join(key, c->world, c->rank)
                                                  : static_cast<Rendezvous *>(ShmRdv::join(key, c->world, c->rank));
        if (!R) return DD_E_INVALID_ARG;
        c->rdv = R;
    }
    return comm_agree(c, host_status);
}

dd_status comm_alloc(dd_ctx *c) {
    Workspace *ws = ws_of(c);
    const int64_t ng = (int64_t)c->ghost_rows.size();
    ws->send_off.assign(c->world + 1, 0);
    std::vector<int32_t> sidx;
    for (int q = 0; q < c->world; ++q) {
        if (q < (int)c->send_rows.size()) sidx.insert(sidx.end(), c->send_rows[q].begin(), c->send_rows[q].end());
        ws->send_off[q + 1] = (int64_t)sidx.size();
    }
    {
        const char *env = getenv("DD_HALO_FUSE");
        ws->halo_fuse = c->world > 1 && (!env || atoi(env) != 0);
    }
    if (!peer_comm(c)) {
        TRY(dmalloc(&ws->xg, std::max<int64_t>(1, c->bs * ng)));
        TRY(dmalloc(&ws->gathered, 6 * (size_t)std::max(1, c->world)));
        TRY(dmalloc(&ws->sendbuf, std::max<size_t>(1, c->bs * sidx.size())));
        TRY(upload_vec(&ws->d_send_idx, sidx));
        if (local_comm(c))
            for (cudaEvent_t *e : {&ws->xev_ready, &ws->xev_done, &ws->xev_app, &ws->xev_free})
                CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        return DD_OK;
    }
    // mailbox: flags | gathered | xg (+16 B slack)
    ws->pd.world = c->world;
    ws->pd.rank = c->rank;
    ws->pd.off_flags = 0;
    ws->pd.off_gath = align256(ddk::peer_flags_bytes(c->world));
    ws->pd.off_xg = align256(ws->pd.off_gath + ddk::peer_gath_bytes(c->world));
    ws->box_bytes = ws->pd.off_xg + 8 * c->bs * std::max<int64_t>(1, ng) + 16;
    TRY(dmalloc(&ws->box, (size_t)ws->box_bytes));
    CK(cudaMemset(ws->box, 0, ws->box_bytes));
    ws->xg = reinterpret_cast<double *>(ws->box + ws->pd.off_xg);
    TRY(dmalloc(&ws->seq, 2 * ddk::PCH_COUNT));
    CK(cudaMemset(ws->seq, 0, 2 * ddk::PCH_COUNT * sizeof(uint64_t)));
    TRY(dmalloc(&ws->perr, 1));
    CK(cudaMemset(ws->perr, 0, sizeof(int)));
    std::vector<int32_t> to, from;
    for (int q = 0; q < c->world; ++q) {
        if (q == c->rank) continue;
        if (q < (int)c->send_rows.size() && !c->send_rows[q].empty()) to.push_back(q);
        if (c->recv_off[q + 1] > c->recv_off[q]) from.push_back(q);
    }
    TRY(upload_vec(&ws->d_send_to, to));
    TRY(upload_vec(&ws->d_recv_from, from));
    ws->n_send_to = (int)to.size();
    ws->n_recv_from = (int)from.size();
    ws->pd.seq = ws->seq;
    ws->pd.err = ws->perr;
    ws->pd.timeout_ns = (unsigned long long)(timeout_s() * 1e9);
    CK(cudaDeviceSynchronize());  // the zeroed mailbox precedes any peer's first signal
    return DD_OK;
}

dd_status comm_connect(dd_ctx *c) {
    if (c->world <= 1) return DD_OK;
    Workspace *ws = ws_of(c);
    if (local_comm(c)) {
        // the group's contexts (this process): the fused apply stores the rows
        // straight into the consumer's ghost block
        Rendezvous *R = rdv_of(c);
        std::vector<uint8_t> all;
        const dd_ctx *me = c;
        if (!R->allgather(&me, sizeof me, all)) {
            set_error("DD_COMM_LOCAL: host rendezvous timed out during dd_setup");
            return DD_E_NCCL;
        }
        ws->local_peers.assign(c->world, nullptr);
        for (int q = 0; q < c->world; ++q) std::memcpy(&ws->local_peers[q], &all[q * sizeof me], sizeof me);
        dd_status st = DD_OK;
        for (dd_ctx *q : ws->local_peers)
            if (q->device != c->device) {
                int can = 0;
                cudaDeviceCanAccessPeer(&can, c->device, q->device);
                if (can && cudaDeviceEnablePeerAccess(q->device, 0) != cudaSuccess) cudaGetLastError();
                if (!can) ws->halo_fuse = false;  // copies still work without peer access
            }
        st = halo_lists_build(
            c,
            [&](int q, int64_t p) {
                dd_ctx *peer = ws->local_peers[q];
                return ws_of(peer)->xg + c->bs * (peer->recv_off[c->rank] + p);
            },
            false);
        return comm_agree(c, st);
    }
    if (!peer_comm(c)) {
        // NCCL: the fused apply packs the send buffer
        return halo_lists_build(
            c, [&](int q, int64_t p) { return ws->sendbuf + c->bs * (ws->send_off[q] + p); }, false);
    }
    Rendezvous *R = rdv_of(c);
    auto slot = std::make_unique<PeerSlot>();
    std::memset(slot.get(), 0, sizeof(PeerSlot));
    slot->status = DD_OK;
    slot->device = c->device;
    slot->pid = (int64_t)getpid();
    slot->raw = reinterpret_cast<uint64_t>(ws->box);
    for (int q = 0; q <= c->world; ++q) slot->recv_off[q] = c->recv_off[q];
    if (c->comm == DD_COMM_IPC && cudaIpcGetMemHandle(&slot->handle, ws->box) != cudaSuccess) {
        cudaGetLastError();
        slot->status = DD_E_CUDA;
        set_error("dd_setup: cudaIpcGetMemHandle failed for the peer mailbox");
    }
    std::vector<uint8_t> all;
    if (!R->allgather(slot.get(), sizeof(PeerSlot), all)) {
        set_error("peer transport: host rendezvous timed out during dd_setup");
        return DD_E_NCCL;
    }
    std::vector<PeerSlot> slots(c->world);
    for (int q = 0; q < c->world; ++q) std::memcpy(&slots[q], &all[q * sizeof(PeerSlot)], sizeof(PeerSlot));
    dd_status st = DD_OK;
    for (auto &s : slots) st = std::max(st, (dd_status)s.status);
    if (st != DD_OK) {
        if (slot->status == DD_OK) set_error("a peer rank could not export its mailbox");
        return st;
    }
    ws->peer_box.assign(c->world, nullptr);
    ws->peer_opened.assign(c->world, false);
    ws->peer_box[c->rank] = ws->box;
    for (int q = 0; q < c->world && st == DD_OK; ++q) {
        if (q == c->rank) continue;
        if (slots[q].device != c->device) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, c->device, slots[q].device);
            if (!can) {
                set_error("peer transport: device " + std::to_string(c->device) + " cannot access device " +
                          std::to_string(slots[q].device) + " (use DD_COMM_NCCL)");
                st = DD_E_INVALID_ARG;
                break;
            }
            if (c->comm == DD_COMM_LOCAL && cudaDeviceEnablePeerAccess(slots[q].device, 0) != cudaSuccess)
                cudaGetLastError();  // already enabled
        }
        if (c->comm == DD_COMM_LOCAL) {
            ws->peer_box[q] = reinterpret_cast<uint8_t *>(slots[q].raw);
        } else {
            void *p = nullptr;
            const cudaError_t e = cudaIpcOpenMemHandle(&p, slots[q].handle, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                cudaGetLastError();
                set_error(std::string("peer transport: cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
                st = DD_E_CUDA;
                break;
            }
            ws->peer_box[q] = reinterpret_cast<uint8_t *>(p);
            ws->peer_opened[q] = true;
        }
    }
    if (st == DD_OK) {
        std::vector<uint8_t *> boxes(ws->peer_box.begin(), ws->peer_box.end());
        st = upload_vec(&ws->d_boxes, boxes);
    }
    if (st == DD_OK) {
        ws->pd.box = ws->d_boxes;
        st = halo_lists_build(
            c,
            [&](int q, int64_t p) {
                return reinterpret_cast<double *>(ws->peer_box[q] + ws->pd.off_xg) +
                       c->bs * (slots[q].recv_off[c->rank] + p);
            },
            true);
    }
    st = comm_agree(c, st);
    if (st == DD_OK) R->setup_done();
    return st;
}

void comm_end(dd_ctx *c) {
    if (c->world <= 1 || c->host_only) return;
    Workspace *ws = ws_of(c);
    if (peer_comm(c) || local_comm(c)) {
        // no peer may still be storing into this rank's mailbox (a FREE count
        // or the last halo rows): every rank is idle before the memory goes
        if (Rendezvous *R = rdv_of(c)) R->barrier();
        if (ws)
            for (int q = 0; q < (int)ws->peer_opened.size(); ++q)
                if (ws->peer_opened[q]) cudaIpcCloseMemHandle(ws->peer_box[q]);
    }
    if (c->nccl) ncclCommDestroy(nccl_of(c));
    c->nccl = nullptr;
    delete rdv_of(c);
    c->rdv = nullptr;
}

// ---- DD_COMM_LOCAL: every exchange records a "ready" event after the
// outgoing data, meets the group at a host rendezvous, makes its stream wait
// on the producers' events and copies device-to-device, records "done",
// meets again, and waits on its consumers' "done" before the outgoing buffer
// can be overwritten. Every wait names an event recorded before the
// rendezvous, so all GPU work of all ranks is enqueued before anything waits
// on it: no kernel ever waits on another rank (a spinning kernel would
// deadlock ranks that share a GPU with a host call that waits for the device,
// e.g. a cudaMalloc of the test's own tensors).
#define LOCAL_MEET(c)                                                                          \
    do {                                                                                       \
        if (!rdv_of(c)->barrier()) {                                                           \
            set_error("DD_COMM_LOCAL rendezvous timed out (a rank stopped calling)");          \
            return DD_E_NCCL;                                                                  \
        }                                                                                      \
    } while (0)

static dd_status local_allgather(dd_ctx *c, int nv, cudaStream_t st) {
    Workspace *ws = ws_of(c);
    const size_t bytes = 2 * (size_t)nv * sizeof(double);
    CK(cudaEventRecord(ws->xev_ready, st));
    LOCAL_MEET(c);
    for (int q = 0; q < c->world; ++q) {
        Workspace *pw = ws_of(ws->local_peers[q]);
        if (q != c->rank) CK(cudaStreamWaitEvent(st, pw->xev_ready, 0));
        CK(cudaMemcpyAsync(ws->gathered + 2 * (size_t)nv * q, pw->loc, bytes, cudaMemcpyDefault, st));
    }
    CK(cudaEventRecord(ws->xev_done, st));
    LOCAL_MEET(c);
    for (int q = 0; q < c->world; ++q)
        if (q != c->rank) CK(cudaStreamWaitEvent(st, ws_of(ws->local_peers[q])->xev_done, 0));
    return DD_OK;
}

static dd_status local_halo(dd_ctx *c, cudaStream_t st) {
    Workspace *ws = ws_of(c);
    CK(cudaEventRecord(ws->xev_ready, st));
    LOCAL_MEET(c);
    for (int q = 0; q < c->world; ++q) {
        if (q == c->rank) continue;
        const int64_t ro = c->recv_off[q], rn = c->recv_off[q + 1] - ro;
        if (!rn) continue;
        dd_ctx *peer = ws->local_peers[q];
        Workspace *pw = ws_of(peer);
        CK(cudaStreamWaitEvent(st, pw->xev_ready, 0));
        CK(cudaMemcpyAsync(ws->xg + c->bs * ro, pw->sendbuf + c->bs * pw->send_off[c->rank], c->bs * rn * sizeof(double),
                           cudaMemcpyDefault, st));
    }
    CK(cudaEventRecord(ws->xev_done, st));
    LOCAL_MEET(c);
    for (int q = 0; q < c->world; ++q)
        if (q != c->rank && ws->send_off[q + 1] > ws->send_off[q])
            CK(cudaStreamWaitEvent(st, ws_of(ws->local_peers[q])->xev_done, 0));
    return DD_OK;
}

dd_status halo(dd_ctx *c, const double *x, cudaStream_t st, bool packed, const int *skip) {
    if (c->world <= 1) return DD_OK;
    Workspace *ws = ws_of(c);
    packed = packed && ws->halo_fuse;
    if (local_comm(c)) {
        const int64_t ns = ws->send_off[c->world];
        if (!packed) {
            if (ns) ddk::launch_gather3(c, ns, ws->d_send_idx, x, ws->sendbuf, st);
            return local_halo(c, st);
        }
        // every producer has recorded xev_app after its fused apply
        LOCAL_MEET(c);
        for (int q = 0; q < c->world; ++q)
            if (q != c->rank && c->recv_off[q + 1] > c->recv_off[q])
                CK(cudaStreamWaitEvent(st, ws_of(ws->local_peers[q])->xev_app, 0));
        return DD_OK;
    }
    if (peer_comm(c)) {
        if (!packed) {
            ddk::launch_peer_wait(ws->pd, ddk::PCH_FREE, ws->d_send_to, ws->n_send_to, 1, skip, st);
            ddk::launch_put_rows(c->bs, ws->n_put, ws->d_put_rows, ws->d_put_dst, x, st);
            ddk::launch_peer_signal(ws->pd, ddk::PCH_HALO, ws->d_send_to, ws->n_send_to, skip, st);
            c->n_launches += 2 + (ws->n_put > 0);
        }
        ddk::launch_peer_wait(ws->pd, ddk::PCH_HALO, ws->d_recv_from, ws->n_recv_from, 0, skip, st);
        ++c->n_launches;
        return DD_OK;
    }
    const int64_t ns = ws->send_off[c->world];
    if (ns && !packed) ddk::launch_gather3(c, ns, ws->d_send_idx, x, ws->sendbuf, st);
    NK(ncclGroupStart());
    for (int q = 0; q < c->world; ++q) {
        if (q == c->rank) continue;
        const int64_t so = ws->send_off[q], sn = ws->send_off[q + 1] - so;
        const int64_t ro = c->recv_off[q], rn = c->recv_off[q + 1] - ro;
        if (sn) NK(ncclSend(ws->sendbuf + c->bs * so, c->bs * sn, ncclDouble, q, nccl_of(c), st));
        if (rn) NK(ncclRecv(ws->xg + c->bs * ro, c->bs * rn, ncclDouble, q, nccl_of(c), st));
    }
    NK(ncclGroupEnd());
    return DD_OK;
}

dd_status halo_consumed(dd_ctx *c, cudaStream_t st, const int *skip) {
    // DD_COMM_LOCAL with the fused halo: peers' next fused applies write this
    // rank's ghost block only after this SpMV has read it
    if (local_comm(c) && ws_of(c)->halo_fuse) CK(cudaEventRecord(ws_of(c)->xev_free, st));
    if (!peer_comm(c)) return DD_OK;
    Workspace *ws = ws_of(c);
    ddk::launch_peer_signal(ws->pd, ddk::PCH_FREE, ws->d_recv_from, ws->n_recv_from, skip, st);
    ++c->n_launches;
    return DD_OK;
}

dd_status apply_halo(dd_ctx *c, const double *r, double *z, cudaStream_t st, const int *skip) {
    Workspace *ws = ws_of(c);
    const bool fuse = c->world > 1 && ws->halo_fuse;
    const bool peer = fuse && peer_comm(c);
    const bool local = fuse && local_comm(c);
    if (local) {
        LOCAL_MEET(c);
        for (int q = 0; q < c->world; ++q)
            if (q != c->rank && ws->send_off[q + 1] > ws->send_off[q])
                CK(cudaStreamWaitEvent(st, ws_of(ws->local_peers[q])->xev_free, 0));
    }
    // peer transports: the epilogue stores into the consumers' ghost blocks,
    // so every consumer must have read the previous rows first
    if (peer) {
        ddk::launch_peer_wait(ws->pd, ddk::PCH_FREE, ws->d_send_to, ws->n_send_to, 1, skip, st);
        ++c->n_launches;
    }
    TRY(apply_launch(c, fuse ? DD_LEVELSET : c->solver_variant, r, z, reinterpret_cast<void *>(st), skip,
                     fuse ? &ws->hout : nullptr));
    if (peer) {
        ddk::launch_peer_signal(ws->pd, ddk::PCH_HALO, ws->d_send_to, ws->n_send_to, skip, st);
        ++c->n_launches;
    }
    if (local) CK(cudaEventRecord(ws->xev_app, st));
    return DD_OK;
}

dd_status reduce_across(dd_ctx *c, int nv, int op, const ddk::RedArgs &ra, cudaStream_t st) {
    if (c->world <= 1) return DD_OK;
    Workspace *ws = ws_of(c);
    if (peer_comm(c)) {
        ddk::launch_peer_allgather_finalize(ws->pd, nv, ws->loc, ra, op, st);
    } else if (local_comm(c)) {
        TRY(local_allgather(c, nv, st));
        ddk::launch_finalize_gathered(c->world, nv, ws->gathered, ra, op, st);
    } else {
        NK(ncclAllGather(ws->loc, ws->gathered, 2 * nv, ncclDouble, nccl_of(c), st));
        ddk::launch_finalize_gathered(c->world, nv, ws->gathered, ra, op, st);
    }
    ++c->n_launches;
    return DD_OK;
}

dd_status comm_wait_event(dd_ctx *c, cudaEvent_t ev) {
    if (!(c->world > 1 && c->comm == DD_COMM_NCCL && c->nccl)) {
        CK(cudaEventSynchronize(ev));
        return DD_OK;
    }
    while (true) {
        const cudaError_t e = cudaEventQuery(ev);
        if (e == cudaSuccess) return DD_OK;
        if (e != cudaErrorNotReady) CK(e);
        ncclResult_t ar = ncclSuccess;
        ncclCommGetAsyncError(nccl_of(c), &ar);
        if (ar != ncclSuccess && ar != ncclInProgress) {
            ncclCommAbort(nccl_of(c));
            c->nccl = nullptr;
            set_error(std::string("NCCL asynchronous error (communicator aborted): ") + ncclGetErrorString(ar));
            return DD_E_NCCL;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

dd_status comm_check(dd_ctx *c, cudaStream_t st) {
    if (c->world <= 1 || local_comm(c)) return DD_OK;
    if (c->comm == DD_COMM_NCCL) {
        if (!c->nccl) {
            set_error("NCCL communicator was aborted after an asynchronous error");
            return DD_E_NCCL;
        }
        ncclResult_t ar = ncclSuccess;
        ncclCommGetAsyncError(nccl_of(c), &ar);
        if (ar != ncclSuccess && ar != ncclInProgress) {
            set_error(std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar));
            return DD_E_NCCL;
        }
        return DD_OK;
    }
    int err = 0;
    CK(cudaMemcpyAsync(&err, ws_of(c)->perr, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (err) {
        set_error("peer transport: a device-side wait saw no progress for DD_PEER_TIMEOUT_S seconds "
                  "(a rank stopped calling, or its memory is unreachable)");
        return DD_E_NCCL;
    }
    return DD_OK;
}

bool comm_graph_ok(const dd_ctx *c) { return c->world <= 1 || peer_comm(c); }

}  // namespace ddi
