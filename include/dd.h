/*
 * dd.h -- C ABI of the B200-native fine-grained domain-decomposition ILU0
 * library (arXiv 2508.04917, "Mapping Sparse Triangular Solves to GPUs via
 * Fine-grained Domain Decomposition").
 *
 * Citations: P:a-b = PAPER.md lines a-b (section / algorithm named);
 * Rn = reading n in DESIGN.md section 3 (where the paper is silent/garbled).
 *
 * Operation (P:41-46 problem statement; Alg. 1 inputs P:139):
 *   dd_setup    partition (Alg. 2) -> stable row permutation
 *                -> block reorder (Alg. 3) -> drop the
 *               inter-subdomain blocks (sec. 3.2) -> per-subdomain
 *               block ILU0 + ILDU0 (Alg. 7) -> level sets (Alg. 5
 *               semantics P:448-508) -> device-resident factor slabs.
 *   dd_apply    z = M^-1 r with M = L D U_unit: fused forward unit-lower
 *               sweep, 3x3 block-diagonal scaling, backward unit-upper sweep,
 *               one CTA per subdomain with the subdomain vector in shared
 *               memory (Alg. 4 P:410-441 / Alg. 6, sec. 4.3
 *               P:653-678, sec. 4.4).
 *   dd_spmv     y = A_r x with the reordered, UN-dropped matrix (R10).
 *   dd_bicgstab right-preconditioned BiCGSTAB (Alg. 1, K1 = I,
 *               K2 = M; R20-R25).
 *
 * Data layout
 *   BSR3: row_ptr int64[n+1], col_idx int32[nnzb] ascending and unique per
 *   row, vals double[9*nnzb], each 3x3 block row-major. Block dim fixed = 3.
 *   Vectors: double[3*n], component c of block row i at index 3*i + c.
 *   Device vectors passed to dd_apply / dd_spmv / dd_bicgstab live in the
 *   REORDERED, subdomain-contiguous space (the paper solves there),
 *   restricted to this rank's rows (dd_local_range); use dd_permute /
 *   dd_unpermute to map from/to the user's original ordering.
 *
 * Ownership
 *   dd_setup copies A; the caller may free it on return. The context owns
 *   every host and device buffer it allocates; dd_destroy frees them.
 *   Vector pointers are caller-owned, device memory on the context's device,
 *   16-byte aligned, 3*n_local doubles; dd_apply may read r up to the next
 *   16-byte boundary past its end (any cudaMalloc / torch allocation
 *   satisfies this).
 *
 * Streams: dd_apply, dd_spmv, dd_permute, dd_unpermute are ordered on the
 *   given cudaStream_t (passed as void*, NULL = legacy default stream) and do
 *   not synchronise the host unless stated. dd_bicgstab returns when the
 *   solve is done: the convergence test runs on the device,
 *   the host enqueues iterations in batches and reads the solver state one
 *   batch behind.
 *
 * Errors: every call returns a dd_status and never aborts; dd_last_error()
 *   gives a thread-local message for the last failing call. dd_setup failure
 *   leaves *out = NULL. No call falls back to a CPU path.
 *
 * Multi-GPU (sec. 4.5 P:730-734 extended to the solver): one process per GPU;
 *   rank r owns a contiguous, count-balanced range of subdomains (R32).
 *   Every rank passes the same full host matrix. dd_setup, dd_spmv and
 *   dd_bicgstab are collective when world > 1 (halo exchange for SpMV,
 *   all-gather of double-double dot partials; NCCL, or device-to-device
 *   copies between contexts of one process, see DD_COMM_LOCAL).
 *   dd_apply never communicates. Inside dd_bicgstab the apply kernel itself
 *   writes the rows peers read in the next SpMV (NCCL: into the send
 *   buffer; DD_COMM_LOCAL: into the consuming peer's ghost block), and an
 *   iteration has three dot reduction points (s.s joins the (t.s, t.t)
 *   all-gather); neither changes any iterate.
 */
#ifndef DD_H
#define DD_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DD_OK = 0,
    DD_E_INVALID_ARG = 1,       /* NULL pointer, bad size, bad option         */
    DD_E_NOT_SQUARE = 2,        /* reserved (BSR3 input is square by type)    */
    DD_E_UNSORTED_OR_DUP = 3,   /* col_idx not strictly ascending in a row    */
    DD_E_MISSING_DIAG = 4,      /* a block row has no diagonal block          */
    DD_E_SINGULAR_PIVOT = 5,    /* |det U_ii| < pivot_floor during ILU0 (R15) */
    DD_E_SUBDOMAIN_TOO_LARGE = 6, /* 24*P bytes + staging exceed shared mem   */
    DD_E_GRID_NOT_DIVISIBLE = 7,  /* geometric tiles do not tile the grid (R26) */
    DD_E_CUDA = 8,
    DD_E_NCCL = 9,
    DD_E_OOM = 10,
    DD_E_BREAKDOWN = 11,        /* |rho|, |sigma| or tau < 1e-30 (R25)        */
    DD_E_MAXITER = 12,
    DD_E_NO_DEVICE = 13         /* no CUDA device (and host_only not set)     */
} dd_status;

/* Borrowed BSR3 matrix (copied by dd_setup). */
typedef struct {
    int64_t n_block_rows;
    int64_t nnzb;
    const int64_t *row_ptr;  /* [n_block_rows + 1]                         */
    const int32_t *col_idx;  /* [nnzb], ascending, unique per row          */
    const double *vals;      /* [9 * nnzb], 3x3 row-major blocks           */
} dd_bsr3;

/* Alg. 2 geometric cuts: grid (nx,ny,nz), natural order i + nx*(j + ny*k);
 * tile dims (tx,ty,tz) = Alg. 2's nblk_*; P = tx*ty*tz block rows. */
typedef struct {
    int32_t nx, ny, nz, tx, ty, tz;
} dd_grid;

/* Apply-kernel variants (sec. 4.1 vs 4.2). */
#define DD_LEVELSET 1  /* level sets + CTA barriers between levels (Alg. 6)        */
#define DD_SPINLOOP 2  /* per-row ready flags in shared memory, no level barriers (Alg. 4) */
#define DD_DIRECT 4    /* ablation: level-set kernel reading factors straight from HBM  */
#define DD_UNFUSED 8   /* ablation of the L->D->U fusion (sec. 4.4): the L sweep and the
                          D+U sweep as two launches, z makes an HBM round trip between */
/* Paper ablations (BSR3 only; Tables 3-4). Edge-centric variants
 * spread a record's blocks over the threads and accumulate with atomicAdd
 * (P:640-644): their results differ from the oracle in the last bits and the
 * solver's iteration count may vary (R19). */
#define DD_EDGE 16          /* dag_ec_ILDU0_fused: edge-centric atomics, vector in shared
                               memory, factors through the TMA ring (level set)          */
#define DD_EDGE_GLOBAL 32   /* dag_ec_no_lds: edge-centric, vector in GLOBAL memory
                               (global atomics), factors from global             */
#define DD_ILU0 64          /* ILU0 with the non-unit U: each row scaled by U_ii^-1 after its
                               off-diagonal updates; request it in dd_opts.variants
                               (builds a second slab); deterministic, not bitwise ILDU0  */
#define DD_DIRECT_GLOBAL 128 /* vertex-centric level set with the vector in global memory */
#define DD_LOWER 256        /* modifier OR-ed into a variant for dd_apply_variant: the lower
                               sweep alone, z = L^-1 r (Table 3's lower-solve analogue)  */
#define DD_TREE 512         /* row-parallel: 4 lanes per row, one block per lane, partial
                               sums combined by a fixed warp-shuffle tree (R19);
                               deterministic, not bitwise the oracle's chain             */

typedef struct {
    int32_t subdomain_rows;   /* P when grid == NULL: contiguous chunks (R26)   */
    const dd_grid *grid;      /* optional geometric partition                   */
    int32_t variants;         /* OR of DD_LEVELSET | DD_SPINLOOP | DD_DIRECT to
                                 build; 0 = DD_LEVELSET                          */
    int32_t device;           /* CUDA device ordinal                            */
    int32_t rank, world;      /* world <= 1: single GPU                         */
    const void *nccl_unique_id; /* 128-byte ncclUniqueId (rank 0 creates, the
                                   caller broadcasts); NULL if world <= 1       */
    double pivot_floor;       /* 0 -> 1e-300 (R15)                              */
    int32_t host_only;        /* 1: run the host setup only (no device work;
                                 introspection calls work, compute calls
                                 return DD_E_INVALID_ARG)                       */
    int32_t n_threads;        /* host setup threads, 0 = all                   */
    int32_t enable_refactor;  /* 1: keep the symbolic maps dd_refactor needs    */
    int32_t partitioner;      /* without grid: DD_PART_CHUNKS or DD_PART_BFS    */
    int32_t comm;             /* world > 1: DD_COMM_NCCL (default), DD_COMM_IPC or DD_COMM_LOCAL */
} dd_opts;

/* Exchange transports for world > 1 (the SpMV halo and the dot partials):
 *   DD_COMM_NCCL   one process per GPU; nccl_unique_id is an ncclUniqueId.
 *                  Grouped ncclSend/ncclRecv for the halo, ncclAllGather for
 *                  the dot partials; asynchronous NCCL errors are polled
 *                  while the host waits (the communicator is aborted and the
 *                  call fails with DD_E_NCCL).
 *   DD_COMM_IPC    one process per GPU on one node (the 8-GPU NVSwitch box):
 *                  peer-memory transport. Every rank owns a device mailbox
 *                  (ghost block, dot slots, flags) that every peer maps with
 *                  CUDA IPC handles; the apply kernel's epilogue stores the
 *                  halo rows straight into the consumer's ghost block (NVLink
 *                  stores), one-thread kernels publish / wait on monotone
 *                  counters (release / acquire, system scope). No host step
 *                  per exchange, so the whole solve is one CUDA graph at
 *                  world > 1 too. nccl_unique_id is any 128-byte key the ranks
 *                  share (it names the host rendezvous used during dd_setup,
 *                  dd_refactor and dd_destroy: POSIX shared memory).
 *   DD_COMM_LOCAL  the ranks are contexts of ONE process (one per GPU, or
 *                  several sharing a GPU -- the single-GPU test vehicle), each
 *                  created and driven by its own host thread; exchanges are
 *                  device-to-device copies (and the fused apply's stores into
 *                  the peer's ghost block) ordered by CUDA events and a host
 *                  rendezvous per exchange, so no kernel ever waits on another
 *                  rank (ranks sharing a GPU stay deadlock-free whatever the
 *                  host threads do); no graph loop. nccl_unique_id is any
 *                  128-byte key.
 * With DD_COMM_IPC / DD_COMM_LOCAL, dd_setup, dd_spmv, dd_bicgstab,
 * dd_solve_host, dd_refactor and dd_destroy are collective. A device-side
 * wait that sees no progress for DD_PEER_TIMEOUT_S seconds (default 120)
 * stops the solve and the call returns DD_E_NCCL; a host rendezvous that
 * waits longer than that fails the same way. Setup and refactor status is
 * agreed over the ranks (every rank returns the same status). */
#define DD_COMM_NCCL 0
#define DD_COMM_LOCAL 1
#define DD_COMM_IPC 2

/* Borrowed scalar CSR matrix (the paper's CSR half, P:110,
 * P:279-305): the same pipeline with 1x1 blocks. vals[nnz]; vectors passed
 * to the compute calls then hold n_local doubles (one unknown per row). */
typedef struct {
    int64_t n_rows;
    int64_t nnz;
    const int64_t *row_ptr;  /* [n_rows + 1]                               */
    const int32_t *col_idx;  /* [nnz], ascending, unique per row, diagonal present */
    const double *vals;      /* [nnz]                                      */
} dd_csr;

/* Partitioners used when dd_opts.grid == NULL (P = subdomain_rows):
 * contiguous chunks of P rows (R26), or graph growing (METIS stand-in, P:236,
 * S:145-153, R35): parts of exactly P rows (last smaller), each grown
 * breadth-first over the block pattern from the lowest-index unassigned row,
 * neighbours in ascending column order. */
#define DD_PART_CHUNKS 0
#define DD_PART_BFS 1

typedef struct dd_ctx dd_ctx;

typedef struct {
    double iterations;        /* 0.5 granularity (R22)                          */
    int32_t n_applies;        /* preconditioner applies (paper-style count)     */
    int32_t converged;
    int32_t breakdown;
    int32_t status;           /* dd_status of the solve                         */
    double rel_resid;         /* last recursive ||r|| / ||r0||                   */
    double true_rel_resid;    /* ||b - A x|| / ||b|| after the solve    */
    double solve_ms;          /* host wall time of the solve                    */
} dd_report;

/* Setup (collective). Returns DD_OK and *out, or an error and *out = NULL. */
dd_status dd_setup(const dd_bsr3 *A, const dd_opts *opts, dd_ctx **out);
void dd_destroy(dd_ctx *ctx);

/* Numeric re-factorisation with the SAME sparsity pattern (nonlinear solvers
 * re-factor one pattern many times): new block values
 * vals[9*nnzb] in A's ORIGINAL block order (host or device memory per
 * vals_on_device). Runs on the GPU: every subdomain is factored (block ILU0
 * -> ILDU0, Alg. 7, same arithmetic order as dd_setup, so identical
 * bits) level by level -- straight from vals when every ILU0 update lands on
 * a diagonal block (7-point stencils), else from a reordered / dropped copy --
 * and L, Dinv and U_unit are written straight into the apply slab; the SpMV
 * operand is refreshed too. vals is read until the call returns. Requires dd_opts.enable_refactor = 1 (or a
 * context that dd_setup already factored on the GPU, which keeps the maps).
 * Collective when world > 1 (the pivot status is agreed over the ranks).
 * Returns DD_E_SINGULAR_PIVOT (context unusable until a successful refactor)
 * if a pivot block has |det| < pivot_floor. Ordered on `stream`; returns after
 * the pivot check (one synchronisation). */
dd_status dd_refactor(dd_ctx *ctx, const double *vals, int32_t vals_on_device, void *stream);

/* This rank's rows in the reordered global numbering. */
dd_status dd_local_range(const dd_ctx *ctx, int64_t *first_block_row, int64_t *n_block_rows);

/* z = M^-1 r (this rank's subdomains; no communication). variant = one of
 * DD_LEVELSET / DD_SPINLOOP / DD_DIRECT / DD_UNFUSED / DD_EDGE /
 * DD_EDGE_GLOBAL / DD_DIRECT_GLOBAL / DD_ILU0 / DD_TREE, optionally | DD_LOWER;
 * 0 = DD_LEVELSET. r (and z for DD_UNFUSED) must be 16-byte aligned for the
 * ring variants (DD_E_INVALID_ARG otherwise). */
dd_status dd_apply(dd_ctx *ctx, const double *r, double *z, void *stream);
dd_status dd_apply_variant(dd_ctx *ctx, int32_t variant, const double *r, double *z,
                           void *stream);

/* y = A_r x (halo exchange inside when world > 1; collective). */
dd_status dd_spmv(dd_ctx *ctx, const double *x, double *y, void *stream);

/* Solve A_r x = b to ||r|| < tol * ||r0|| (R21). b, x device, reordered,
 * local. x in: x0, out: solution. resid_hist: nullable host array of
 * 2*max_iter+1 doubles receiving [||r0||, ||s_1||, ||r_1||, ...].
 * Returns DD_OK, DD_E_BREAKDOWN or DD_E_MAXITER (rep and x filled in all
 * three cases). */
dd_status dd_bicgstab(dd_ctx *ctx, const double *b, double *x, double tol, int32_t max_iter,
                      double *resid_hist, dd_report *rep, void *stream);

/* End-to-end user call: b_host / x_host are HOST arrays of 3*N doubles in
 * the ORIGINAL ordering (pinned memory recommended). Copies b in, solves,
 * copies this rank's part of x out (other entries of x_host untouched). */
dd_status dd_solve_host(dd_ctx *ctx, const double *b_host, double *x_host, double tol,
                        int32_t max_iter, dd_report *rep, void *stream);

/* Original-ordering host vector (3*N) -> this rank's reordered device slice,
 * and back (scatter of the local rows into the host vector). */
dd_status dd_permute(dd_ctx *ctx, const double *v_orig_host, double *v_reord_dev, void *stream);
dd_status dd_unpermute(dd_ctx *ctx, const double *v_reord_dev, double *v_orig_host,
                       void *stream);

/* Introspection for parity (caller-allocated host arrays). Partition, levels
 * and patterns are what dd_setup computed on the host. Factor VALUES: on a
 * device context with 3x3 blocks (and without DD_ILU0) dd_setup factors on
 * the GPU and dd_get_factors copies the current device
 * factors back (so after dd_refactor it reports the new ones); host_only,
 * scalar CSR, DD_ILU0 or DD_HOST_ILU0=1 contexts factor on the host. */
dd_status dd_get_partition(const dd_ctx *ctx, int32_t *labels /*[N], original order*/,
                           int32_t *new_to_old /*[N]*/);
/* The Alg. 2 grid and tile dims the partition used (the chosen ones when
 * dd_setup picked them; all zeros for a chunk or BFS partition). */
dd_status dd_get_grid(const dd_ctx *ctx, dd_grid *out);
/* which: 0 = L (hmapL), 1 = U (hmapU); local rows, reordered order. */
dd_status dd_get_levels(const dd_ctx *ctx, int32_t which, int32_t *hmap);

/* Scalar CSR variant of dd_setup: identical steps, errors and
 * options (enable_refactor is not supported: DD_E_INVALID_ARG). Every other
 * call works on the returned context; vectors carry one double per row. */
dd_status dd_setup_csr(const dd_csr *A, const dd_opts *o, dd_ctx **out);

/* Alg. 5 on the device: the paper's fixpoint
 * level marking, one CTA per subdomain, over this rank's L and U factor
 * patterns. Writes hmapL and hmapU (host arrays of n_local int32 each, may be
 * NULL) and the kernel time in ms (may be NULL). The result equals
 * dd_get_levels (longest path, R16). Synchronous; DD_E_INVALID_ARG for a
 * host_only context. */
dd_status dd_levels_device(dd_ctx *ctx, int32_t *hmapL, int32_t *hmapU, double *ms);
/* Factors of the local rows in the dropped pattern, reordered local numbering
 * (columns local too). Pass NULL arrays to query sizes only.
 *   L: strictly-lower blocks (unit diagonal implied); U: strictly-upper
 *   blocks of U_unit; Dinv: [9*n_local]. Lrp/Urp: [n_local+1]. */
dd_status dd_get_factors(const dd_ctx *ctx, int64_t *nnzb_L, int64_t *nnzb_U, int64_t *Lrp,
                         int32_t *Lci, double *Lv, int64_t *Urp, int32_t *Uci, double *Uv,
                         double *Dinv);
/* Halo description for world > 1 (sizes only if arrays NULL):
 * ghost_rows: reordered global rows this rank reads from other ranks,
 * ascending; their owner ranks in ghost_owner. */
dd_status dd_get_halo(const dd_ctx *ctx, int64_t *n_ghost, int64_t *ghost_rows,
                      int32_t *ghost_owner);
/* Rows of this rank that peer `peer` reads (its ghosts owned here), local
 * numbering, ascending; sizes only if rows == NULL. */
dd_status dd_get_send_rows(const dd_ctx *ctx, int32_t peer, int64_t *n, int32_t *rows);
/* stats[16]: {nnzb_before, nnzb_after, n_sub_global, n_sub_local, max_levels_L,
 *   max_levels_U, max_P, slab_bytes_levelset, slab_bytes_spin, spmv_bytes,
 *   apply_canonical_bytes, spmv_canonical_bytes, n_local, n_ghost,
 *   kernels launched so far, shared-vector slot swizzle
 *   (s1 | p1 << 8 | s2 << 16 | p2 << 24: slot(i) = i + (i >> s1) p1 + (i >> s2) p2)};
 * setup_ms[6]: {partition+permute, reorder+drop, ilu0+ildu0, levels,
 *   pack, device upload}. Either may be NULL. */
dd_status dd_stats(const dd_ctx *ctx, int64_t *stats, double *setup_ms);
/* Per-kernel timing inside dd_bicgstab (CUDA events on the solver stream,
 * harvested at its own sync points). mode 1: enable + reset, 0: disable,
 * -1: query. out[8] (nullable) = {n_apply, apply_ms, n_spmv, spmv_ms,
 * n_blas1, blas1_ms, kernels launched by this context so far, 0}. */
dd_status dd_profile(dd_ctx *ctx, int32_t mode, double *out);
/* Apply-kernel launch shape chosen at setup: {grid, threads, smem_bytes,
 * ring_bytes} for the given variant. */
dd_status dd_launch_info(const dd_ctx *ctx, int32_t variant, int64_t *info);
/* Apply variant dd_bicgstab uses, picked at dd_setup by timing every
 * available variant once on this device (all variants give bitwise the same
 * z, so the choice never changes a result; world > 1 keeps DD_LEVELSET, whose
 * kernel carries the fused halo epilogue). Environment DD_SOLVER_VARIANT =
 * levelset | spin | direct forces one. *variant (nullable) = DD_LEVELSET |
 * DD_SPINLOOP | DD_DIRECT; ms[3] (nullable) = the measured apply times of
 * {level set, sync-free, direct} in ms (0 = not timed / unavailable). */
dd_status dd_solver_variant(const dd_ctx *ctx, int32_t *variant, double *ms);

/* Subdomain sizing for Alg. 2 tiles (north star: "sizes each subdomain so
 * its vector fits shared memory"): among tile dims (tx,ty,tz) dividing
 * (nx,ny,nz) with P = tx*ty*tz in [P_target/2, 2*P_target] (0 -> 2048, the
 * paper's P:1041) whose vector fits, pick the one whose subdomain count fills
 * whole waves of the apply kernel's CTA slots on `device` (SMs x resident
 * CTAs, from the CUDA occupancy API; device < 0: an analytic model), then P
 * nearest the target, then the most compact tile -- precisely: maximise
 * fill x bw x (1 - 3 x dropped) with fill = the wave fill, bw = 0.82 for one
 * resident CTA per SM (latency-bound), 1 otherwise, dropped = the share of
 * the grid couplings that cross tile faces (uniform weights here). Writes
 * g->tx/ty/tz. dd_setup makes the same choice when opts.grid has
 * tx = ty = tz = 0 (P_target = opts.subdomain_rows), weighting each grid
 * plane by the Frobenius norms of the matrix blocks that cross it.
 * DD_E_GRID_NOT_DIVISIBLE if no tile shape qualifies. */
dd_status dd_choose_tiles(dd_grid *g, int32_t device, int32_t bs, int32_t P_target);

/* 128-byte ncclUniqueId for world > 1 (rank 0 calls it; the caller
 * broadcasts the bytes, e.g. with torch.distributed). */
dd_status dd_nccl_unique_id(void *out128);

const char *dd_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
