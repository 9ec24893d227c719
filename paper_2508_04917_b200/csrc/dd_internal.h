// dd_internal.h -- product-internal declarations shared by the host setup
// (setup.cpp), the C ABI (api.cpp) and the CUDA kernels (*.cu).
// Never included by the oracle; the oracle never included here.
#pragma once

#include <cstdint>
#include <sys/mman.h>

#include <cstdlib>
#include <memory>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "dd.h"

#if !defined(__CUDACC__) && !defined(__host__)
#define __host__
#endif
#if !defined(__CUDACC__) && !defined(__device__)
#define __device__
#endif

namespace ddi {

// Large host arrays that are fully overwritten after allocation: resize()
// leaves the elements uninitialised (no single-threaded zero fill of GBs).
// Buffers of 32 MB and more come 2 MB-aligned with MADV_HUGEPAGE: the
// first-touch page faults of GBs of 4 KB pages were a visible part of setup.
template <class T>
struct UninitAlloc : std::allocator<T> {
    template <class U>
    struct rebind {
        using other = UninitAlloc<U>;
    };
    UninitAlloc() = default;
    template <class U>
    UninitAlloc(const UninitAlloc<U> &) {}
    static constexpr size_t kBig = 32u << 20, kHuge = 2u << 20;
    T *allocate(size_t n) {
        const size_t bytes = n * sizeof(T);
        if (bytes < kBig) return std::allocator<T>::allocate(n);
        const size_t sz = (bytes + kHuge - 1) / kHuge * kHuge;
        void *p = std::aligned_alloc(kHuge, sz);
        if (!p) throw std::bad_alloc();
        madvise(p, sz, MADV_HUGEPAGE);
        return static_cast<T *>(p);
    }
    void deallocate(T *p, size_t n) {
        if (n * sizeof(T) < kBig)
            std::allocator<T>::deallocate(p, n);
        else
            std::free(p);
    }
    template <class U>
    void construct(U *) noexcept {}
    template <class U, class... A>
    void construct(U *p, A &&...a) {
        ::new ((void *)p) U(std::forward<A>(a)...);
    }
};
template <class T>
using uvector = std::vector<T, UninitAlloc<T>>;

// ---------------------------------------------------------------------------
// Factor-slab record format. One byte stream per
// subdomain, records in consumption order, every record 16-byte aligned:
//   RecHdr (16 B)
//   uint16 cnt[K], padded to 16 B  rows having more than k blocks (jagged
//                                  diagonal; rows sorted by block count desc.)
//   desc[w]: per row DW bytes = {row, col_0 .. col_{K-1}, 0xFFFF pad}
//            DW = 8 for K <= 3, else 2*(1+K) rounded up to 16; padded to 16 B
//   [U records] double dinv[9][w]  (structure of arrays)
//   double val: for k = 0..K-1, 9 planes val_k[v][cnt_k]
//   padded to 16 B.
// One 8-byte descriptor load gives a thread its row and all its columns; the
// value addresses depend only on (t, cnt), so every load of a record can be
// issued before the first FMA.
struct RecHdr {
    uint16_t w;       // rows in this record
    uint16_t K;       // max blocks per row (L: strictly lower, U: strictly upper)
    uint16_t flags;   // REC_BARRIER | REC_UPPER | REC_LAST
    uint16_t nnz;     // blocks in this record (sum of cnt)
    uint32_t bytes;   // total record bytes (multiple of 16)
    uint32_t off_val; // byte offset of val[] from the record start
};
// descriptor width and offsets (shared by the packer and the kernels)
inline __host__ __device__ uint32_t rec_dw(uint32_t K) { return K <= 3 ? 8u : ((2u * (1u + K) + 15u) & ~15u); }
// the count area is at least 16 bytes (also for K = 0): bytes 24..31 of a
// record with K <= 3 are then always zero (cnt[4..7]), the kernels' source
// of an exact 0.0 for the absent blocks of the branch-free 7-point path
inline __host__ __device__ uint32_t rec_off_desc(uint32_t K) { return 32u + (K > 8u ? ((2u * K - 1u) & ~15u) : 0u); }
inline __host__ __device__ uint32_t rec_off_dinv(uint32_t K, uint32_t w) {
    return (rec_off_desc(K) + rec_dw(K) * w + 15u) & ~15u;
}
static_assert(sizeof(RecHdr) == 16, "RecHdr must be 16 bytes");

enum : uint16_t { REC_BARRIER = 1, REC_UPPER = 2, REC_LAST = 4 };

// Per-subdomain descriptor (device array, one per local subdomain).
struct SubInfo {
    int64_t stream_off;   // byte offset of the subdomain's record stream
    int32_t stream_bytes; // multiple of 16
    int32_t row0;         // first local block row
    int32_t nrows;        // P_s
    int32_t n_rec;        // number of records
    int32_t u_off;        // byte offset of the first D+U record (the L section's size)
    int32_t pad_;
};
static_assert(sizeof(SubInfo) == 32, "SubInfo layout");

// Sliced-ELL SpMV operand: slices of 32 consecutive rows, slot (k, lane) of
// slice s at slot_ptr[s] + 32*k + lane; values as 9 planes of 32 per k.
struct SpmvDev {
    int64_t n_slices = 0;
    int64_t n_slots = 0;
    int64_t *slot_ptr = nullptr;  // [n_slices + 1]
    int32_t *cols = nullptr;      // [n_slots], -1 = padding
    double *vals = nullptr;       // [9 * n_slots]
};

struct Slab {
    uvector<uint8_t> bytes;       // host copy (all local subdomains)
    std::vector<SubInfo> info;
    int32_t rows_per_rec = 128;
    int64_t max_rec_bytes = 0;
    uint8_t *d_bytes = nullptr;
    SubInfo *d_info = nullptr;
};

// Halo rows written by the apply's epilogue (world > 1): for
// local subdomain s, entries [ptr[s], ptr[s+1]) name a row of the subdomain
// (row[e], 0-based inside it) and the address its bs values go to -- the
// rank's NCCL send buffer, or (DD_COMM_LOCAL) the consuming peer's ghost block.
struct HaloOut {
    const int32_t *ptr = nullptr;  // [n_local_sub + 1]; nullptr = no halo output
    const int32_t *row = nullptr;  // [E]
    double *const *dst = nullptr;  // [E]
};

// Shared-memory slot of subdomain-local row i (bank-conflict swizzle, chosen
// at setup by a bank model of the slab's access pattern; identity = shifts
// of 31): slot(i) = i + (i >> s1) * p1 + (i >> s2) * p2. The packer writes
// slots (not rows) into the record descriptors, so the sweeps index the
// shared vector directly; only the r fill / z store / halo epilogue map
// element q = bs*i + c to bs*slot(i) + c.
struct Swz {
    uint32_t s1 = 31, p1 = 0, s2 = 31, p2 = 0;
    // the zero slot: one vector slot past the rows that holds 0.0 (the
    // kernels write it once); the descriptors name it for absent blocks, so
    // the branch-free 7-point path gathers an exact zero without a select
    uint32_t zslot = 0xFFFFu;
    __host__ __device__ uint32_t slot(uint32_t i) const { return i + (i >> s1) * p1 + (i >> s2) * p2; }
};

struct LaunchCfg {
    int grid = 0, threads = 0, smem = 0, ring = 0, consumers = 0;
};

}  // namespace ddi

struct dd_ctx {
    // --- topology
    int device = 0, rank = 0, world = 1;
    int bs = 3;  // unknowns per row: 3 (BSR3) or 1 (scalar CSR)
    bool host_only = false;
    // --- global partition
    int64_t N = 0;                 // global block rows
    int64_t nnzb_A = 0;            // nnzb of A (= A_r)
    int64_t nnzb_dd = 0;           // nnzb after the drop (global)
    int32_t n_sub = 0;             // global subdomains
    std::vector<int32_t> labels;   // [N] original order
    std::vector<int32_t> new_to_old, old_to_new;
    std::vector<int64_t> sub_ptr;  // [n_sub + 1] reordered rows
    // --- this rank
    int32_t sub_first = 0, sub_last = 0;  // local subdomains [first, last)
    int64_t row_first = 0, n_local = 0;   // reordered global rows
    int32_t max_P = 0;
    dd_grid grid = {0, 0, 0, 0, 0, 0};  // Alg. 2 grid and tiles used (zeros: chunk / BFS partition)
    ddi::Swz swz;                   // shared-vector slot swizzle (identity for scalar rows)
    int32_t vec_rows = 0;           // slot(max_P - 1) + 1: rows of the shared vector
    int32_t kmax = 0;  // most blocks of a row in one factor triangle (> 3: general-K kernels)
    // factors of the local rows (local numbering)
    std::vector<int64_t> Lrp, Urp;
    ddi::uvector<int32_t> Lci, Uci;
    ddi::uvector<double> Lv, Uv, Dinv;
    std::vector<int32_t> hmapL, hmapU;
    int32_t max_lev_L = 0, max_lev_U = 0;
    // local rows of A_r, columns in local+ghost numbering
    std::vector<int64_t> Arp;
    ddi::uvector<int32_t> Aci;
    ddi::uvector<double> Av;
    std::vector<int64_t> ghost_rows;   // reordered global ids, ascending
    std::vector<int32_t> ghost_owner;
    // halo send lists per peer (local row ids) and recv counts per peer
    std::vector<std::vector<int32_t>> send_rows;  // [world]
    std::vector<int64_t> recv_off;                // [world + 1] into ghost block
    // slabs
    ddi::Slab slab_lvl, slab_spin;
    ddi::Slab slab_ilu;                 // DD_ILU0 ablation: U records with the non-unit U_ij
    ddi::uvector<double> Uraw;          // non-unit U_ij (j > i), only when DD_ILU0 is requested
    int32_t variants = 0;
    int32_t solver_variant = DD_LEVELSET;  // apply variant inside dd_bicgstab (timed at setup)
    double variant_ms[3] = {0, 0, 0};      // level set, sync-free, direct
    ddi::LaunchCfg cfg_lvl, cfg_spin, cfg_direct, cfg_ec, cfg_nu, cfg_tree;
    // spmv
    ddi::SpmvDev spmv;
    int64_t spmv_bytes = 0;
    // timings
    double setup_ms[6] = {0, 0, 0, 0, 0, 0};
    // --- device state
    void *d_new_to_old_local = nullptr;  // int32 [n_local]: global orig row of local row
    void *d_setup_tmp[3] = {nullptr, nullptr, nullptr};  // sliced-ELL build inputs, freed at dd_destroy
    double *d_stage = nullptr;           // staging for permute (3N doubles)
    double *d_vecg = nullptr;            // DD_EDGE_GLOBAL / DD_DIRECT_GLOBAL: global vector (slot layout)
    double *d_xghost = nullptr;          // spmv input with ghost space (world>1)
    double *d_sendbuf = nullptr;
    void *dev_ws = nullptr;              // BiCGSTAB workspace (api.cpp)
    void *nccl = nullptr;                // ncclComm_t
    int comm = 0;                        // DD_COMM_NCCL / DD_COMM_LOCAL / DD_COMM_IPC
    void *rdv = nullptr;                 // host rendezvous of the peer transports (comm.cpp)
    double *h_pinned = nullptr;          // small pinned scalars
    int num_sms = 148;
    // --- refactor (dd_refactor) symbolic maps, built when opts.enable_refactor
    bool refactor = false;               // refactor maps built (enable_refactor, or the GPU numeric path)
    bool gpu_numeric = false;            // dd_setup factors on the device (k_refactor9), host holds no values
    double pivot_floor = 1e-300;
    ddi::uvector<int32_t> Asrc;          // reordered local A_r block -> original block index
    std::vector<int64_t> Wrp;            // A_dd working layout (rank-local rows)
    ddi::uvector<int32_t> Wsrc;
    ddi::uvector<int32_t> Wcol;
    std::vector<int64_t> Wdiag;
    ddi::uvector<int64_t> Uptr;          // per W position: update range
    ddi::uvector<int32_t> UpdQ, UpdT;    // (U_kj position, target position)
    std::vector<int32_t> LevRows, LevPtr, SubLev;
    std::vector<int32_t> URows, SubU;    // rows in U-record order per subdomain (refactor's Dinv / U_unit pass)
    ddi::uvector<int64_t> SlabLoff, SlabUoff, SlabDoff;  // byte offsets into the slab
    ddi::uvector<int32_t> SlabLst, SlabUst, SlabDst;     // plane strides (bytes)
    void *rf = nullptr;                  // device-side refactor state (api.cpp)
    mutable int64_t n_launches = 0;      // kernels launched by this context
    void *prof = nullptr;                // api.cpp profiling state
};

namespace ddi {
// setup.cpp
dd_status host_setup(dd_ctx *ctx, const dd_bsr3 *A, const dd_opts *o);
void set_error(const std::string &msg);
double now_ms();

// kernels (apply.cu / spmv.cu / blas1.cu)
dd_status apply_launch(dd_ctx *ctx, int variant, const double *r, double *z, void *stream,
                       const int *skip = nullptr, const HaloOut *halo = nullptr);
dd_status apply_prepare(dd_ctx *ctx);  // choose launch cfgs, set smem attributes
// CTA slots (SMs x resident CTAs) of the level-set kernel for P-row subdomains
int tile_slots(int device, int bs, int P, int *per_sm = nullptr);
void spmv_launch(const dd_ctx *ctx, const double *x, double *y, void *stream);
}  // namespace ddi
