// peer.cuh -- device side of the peer-memory transport (product-internal).
//
// For world > 1 the solver has two real exchange steps (SURVEY 8(e)
// extended to the solver): the SpMV halo and the dot-product all-gathers. With
// DD_COMM_LOCAL (ranks are contexts of one process) and DD_COMM_IPC (one
// process per rank on one node, memory mapped with CUDA IPC handles) every
// rank owns one device "mailbox" that every peer maps:
//   flags    uint64 [PCH_COUNT][world]  flags[ch][src] = src's signal count on ch
//   gathered double [2][world][6]       dot partials, double-buffered by the
//                                       parity of the DOT signal count
//   xg       double [bs * n_ghost]      ghost rows of the SpMV input
// Producers write straight into the consumer's mailbox (the halo rows leave
// from the apply kernel's epilogue, NVLink stores between GPUs) and publish
// with a release store of a monotone counter; consumers spin (acquire loads,
// bounded by a timeout) in one-thread kernels on their stream. No host
// rendezvous per exchange, so the whole iteration is capturable in a CUDA
// graph at world > 1 too.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "krylov.cuh"

namespace ddk {

enum : int {
    PCH_HALO = 0,  // producer -> consumer: my rows are in your ghost block
    PCH_FREE = 1,  // consumer -> producer: my SpMV has read your rows
    PCH_DOT = 2,   // all -> all: my dot partials are in your gathered slot
    PCH_COUNT = 3
};

struct PeerDev {
    int world = 0, rank = 0;
    uint8_t *const *box = nullptr;  // [world] every rank's mailbox, mapped in this process
    uint64_t *seq = nullptr;        // [2 * PCH_COUNT]: signals sent per channel, then waits done
    int *err = nullptr;             // set to 1 by a wait that timed out; later waits return at once
    int64_t off_flags = 0, off_gath = 0, off_xg = 0;  // byte offsets inside a mailbox
    unsigned long long timeout_ns = 0;
};

// mailbox layout sizes (host side)
inline int64_t peer_flags_bytes(int world) { return 8LL * PCH_COUNT * world; }
inline int64_t peer_gath_bytes(int world) { return 8LL * 2 * world * 6; }

#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long peer_now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned long long peer_ld_acquire(const uint64_t *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void peer_st_release(uint64_t *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t *peer_flags(const PeerDev &d, int q) {
    return reinterpret_cast<uint64_t *>(d.box[q] + d.off_flags);
}
__device__ __forceinline__ double *peer_gath(const PeerDev &d, int q) {
    return reinterpret_cast<double *>(d.box[q] + d.off_gath);
}
// spin until flags[ch][q] >= target in this rank's mailbox; false on timeout
// (then *err = 1, and every later wait returns at once)
__device__ __forceinline__ bool peer_spin(const PeerDev &d, int ch, int q, unsigned long long target) {
    const uint64_t *f = peer_flags(d, d.rank) + ch * d.world + q;
    const unsigned long long t0 = peer_now_ns();
    while (peer_ld_acquire(f) < target) {
        if (*reinterpret_cast<volatile int *>(d.err)) return false;
        if (peer_now_ns() - t0 > d.timeout_ns) {
            atomicExch(d.err, 1);
            return false;
        }
        __nanosleep(64);
    }
    return true;
}
#endif

// signal channel ch to the ranks in peers[0..n): count += 1, then a release
// store of the count into flags[ch][rank] of each peer's mailbox.
// skip: solver control word (nullptr = always); skipped uniformly on every rank.
void launch_peer_signal(const PeerDev &d, int ch, const int32_t *peers, int n, const int *skip, cudaStream_t st);
// wait on channel ch for the ranks in peers[0..n).
//   free_mode 0: target = ++waits[ch] (HALO)
//   free_mode 1: target = sent[HALO] (FREE: every halo this rank sent so far has been read)
void launch_peer_wait(const PeerDev &d, int ch, const int32_t *peers, int n, int free_mode, const int *skip,
                      cudaStream_t st);
// all-gather of loc[0 .. 2nv) into every rank's gathered slot, then (on each
// rank) wait for all peers and combine in rank order + finalize (op as in
// k_finalize_gathered; the same stop rule on every rank).
void launch_peer_allgather_finalize(const PeerDev &d, int nv, const double *loc, const RedArgs &ra, int op,
                                    cudaStream_t st);
// the halo rows of x (local rows rows[e]) straight into the destination
// addresses dst[e] (peers' ghost blocks): the unfused exchange of dd_spmv
void launch_put_rows(int bs, int64_t n, const int32_t *rows, double *const *dst, const double *x, cudaStream_t st);

}  // namespace ddk
