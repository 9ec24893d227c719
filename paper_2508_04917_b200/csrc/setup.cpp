// setup.cpp -- host-side setup of the decomposed ILDU0 preconditioner
// (product code; independent of oracle/). Steps, in the paper's order:
//   Alg. 2 geometric cuts or contiguous chunks (R26)
//   stable grouping permutation (R6, R7)
//   Alg. 3 block reorder of this rank's rows (R8)
//   drop of inter-subdomain blocks (R9)
//   block ILU0 + ILDU0 per subdomain (Alg. 7, R11-R15)
//   longest-path level sets per subdomain (Alg. 5 semantics P:448-508, R16)
//   packing of the level-ordered factor slabs (B200 design)
//   sliced-ELL SpMV operand of A_r with halo numbering (sec. 8e)
// Floating point follows DESIGN.md sec. 4 (explicit std::fma, compiled with
// -ffp-contract=off) so the factors equal the oracle's bit for bit.
#include <omp.h>

#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "dd_internal.h"

namespace ddi {

static thread_local std::string g_err;
void set_error(const std::string &m) { g_err = m; }
const char *last_error_c() { return g_err.c_str(); }

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// ------------------------------------------------------------ 3x3 algebra
// C = A*B, C_rc = fma(a_r2, b_2c, fma(a_r1, b_1c, a_r0*b_0c)). C may alias A.
static inline void blk_mul(const double *A, const double *B, double *C) {
    double t[9];
    for (int r = 0; r < 3; ++r) {
        const double a0 = A[3 * r], a1 = A[3 * r + 1], a2 = A[3 * r + 2];
        for (int c = 0; c < 3; ++c) t[3 * r + c] = std::fma(a2, B[6 + c], std::fma(a1, B[3 + c], a0 * B[c]));
    }
    std::memcpy(C, t, sizeof t);
}

// W -= L*U entrywise as three chained fmas in d = 0, 1, 2 order.
static inline void blk_sub_mul(double *W, const double *L, const double *U) {
    for (int r = 0; r < 3; ++r) {
        const double l0 = L[3 * r], l1 = L[3 * r + 1], l2 = L[3 * r + 2];
        for (int c = 0; c < 3; ++c) {
            double w = W[3 * r + c];
            w = std::fma(-l0, U[c], w);
            w = std::fma(-l1, U[3 + c], w);
            w = std::fma(-l2, U[6 + c], w);
            W[3 * r + c] = w;
        }
    }
}

// adjugate / determinant; false if |det| < floor (or NaN).
static inline bool blk_inv(const double *m, double floor_, double *out) {
    const double c00 = std::fma(m[4], m[8], -(m[5] * m[7]));
    const double c01 = std::fma(m[5], m[6], -(m[3] * m[8]));
    const double c02 = std::fma(m[3], m[7], -(m[4] * m[6]));
    const double c10 = std::fma(m[2], m[7], -(m[1] * m[8]));
    const double c11 = std::fma(m[0], m[8], -(m[2] * m[6]));
    const double c12 = std::fma(m[1], m[6], -(m[0] * m[7]));
    const double c20 = std::fma(m[1], m[5], -(m[2] * m[4]));
    const double c21 = std::fma(m[2], m[3], -(m[0] * m[5]));
    const double c22 = std::fma(m[0], m[4], -(m[1] * m[3]));
    const double det = std::fma(m[0], c00, std::fma(m[1], c01, m[2] * c02));
    if (!(std::fabs(det) >= floor_)) return false;
    const double rd = 1.0 / det;
    out[0] = c00 * rd; out[1] = c10 * rd; out[2] = c20 * rd;
    out[3] = c01 * rd; out[4] = c11 * rd; out[5] = c21 * rd;
    out[6] = c02 * rd; out[7] = c12 * rd; out[8] = c22 * rd;
    return true;
}

// block size dispatch: bs = 3 (BSR3, the ops above) or 1 (scalar CSR, the
// same formulas with 1x1 blocks: c = a*b, w = fma(-l, u, w), inv = 1/a)
static inline void bmul(int bs, const double *A, const double *B, double *C) {
    if (bs == 3) blk_mul(A, B, C);
    else C[0] = A[0] * B[0];
}
static inline void bsub_mul(int bs, double *W, const double *L, const double *U) {
    if (bs == 3) blk_sub_mul(W, L, U);
    else W[0] = std::fma(-L[0], U[0], W[0]);
}
static inline bool binv(int bs, const double *m, double floor_, double *out) {
    if (bs == 3) return blk_inv(m, floor_, out);
    if (!(std::fabs(m[0]) >= floor_)) return false;
    out[0] = 1.0 / m[0];
    return true;
}

// ---------------------------------------------------------- slab packing
namespace {

struct RowRef {
    int32_t row;          // subdomain-local row id
    int32_t nblk;         // blocks in this triangle
    const int32_t *cols;  // rank-local column ids (ascending)
    const double *vals;   // 9 per block
    const double *dinv;   // U records only
    int64_t src0;         // Lv / Uv index of the row's first block (refactor maps)
    int64_t li;           // rank-local row (Dinv map)
};

// Slab scatter maps for dd_refactor (null when not requested): byte offset of
// element 0 of every L / U_unit / Dinv block inside its subdomain stream, and
// the plane stride (element v at off + v * stride).
struct SlabMaps {
    int64_t *Loff = nullptr, *Uoff = nullptr, *Doff = nullptr;
    int32_t *Lst = nullptr, *Ust = nullptr, *Dst = nullptr;
    bool on = false;  // (Loff / Uoff are null when a triangle has no blocks, e.g. P = 1)
};

inline size_t al(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Append one record for `rows` (already sorted by nblk descending, stable).
// Output of the packer: p == nullptr sizes the stream only (first pass);
// otherwise records are written at p + pos (p = the subdomain's stream in the
// final slab buffer, second pass).
struct Sink {
    uint8_t *p = nullptr;
    size_t pos = 0;
};

void put_record(Sink &out, const std::vector<RowRef> &rows, bool upper,
                uint16_t flags, int32_t col_base, int64_t &max_rec, const SlabMaps &mp, int b2, const Swz &sw) {
    const int w = (int)rows.size();
    int K = 0;
    int nnz = 0;
    for (auto &r : rows) {
        K = std::max(K, r.nblk);
        nnz += r.nblk;
    }
    const size_t off_desc = rec_off_desc(K), dw = rec_dw(K);
    const size_t off_dinv = rec_off_dinv(K, w);
    const size_t off_val = off_dinv + (upper ? 8 * (size_t)b2 * w : 0);
    const size_t bytes = al(off_val + 8 * (size_t)b2 * nnz, 16);
    const size_t base = out.pos;
    out.pos += bytes;
    max_rec = std::max<int64_t>(max_rec, (int64_t)bytes);
    if (!out.p) return;
    uint8_t *p = out.p + base;
    std::memset(p, 0, bytes);  // padding (the slab buffer is not initialised)
    RecHdr h;
    h.w = (uint16_t)w;
    h.K = (uint16_t)K;
    h.flags = (uint16_t)(flags | (upper ? REC_UPPER : 0));
    h.nnz = (uint16_t)nnz;
    h.bytes = (uint32_t)bytes;
    h.off_val = (uint32_t)off_val;
    std::memcpy(p, &h, sizeof h);
    uint16_t *cnt = reinterpret_cast<uint16_t *>(p + 16);
    for (int k = 0; k < K; ++k) {
        int c = 0;
        for (auto &r : rows) c += (r.nblk > k);
        cnt[k] = (uint16_t)c;
    }
    for (int t = 0; t < w; ++t) {
        uint16_t *d = reinterpret_cast<uint16_t *>(p + off_desc + dw * t);
        // absent blocks name the zero slot (Swz::zslot)
        for (size_t q = 0; q < dw / 2; ++q) d[q] = (uint16_t)sw.zslot;
        // shared-vector slots (Swz), not rows: the kernels index the vector directly
        d[0] = (uint16_t)sw.slot((uint32_t)rows[t].row);
        for (int k = 0; k < rows[t].nblk; ++k) d[1 + k] = (uint16_t)sw.slot((uint32_t)(rows[t].cols[k] - col_base));
    }
    if (upper) {
        double *dv = reinterpret_cast<double *>(p + off_dinv);
        if (rows[0].dinv)  // null: the values come from the device (GPU numeric path)
            for (int v = 0; v < b2; ++v)
                for (int t = 0; t < w; ++t) dv[(size_t)v * w + t] = rows[t].dinv[v];
        if (mp.on)
            for (int t = 0; t < w; ++t) {
                mp.Doff[rows[t].li] = (int64_t)(base + off_dinv + 8 * (size_t)t);
                mp.Dst[rows[t].li] = 8 * w;
            }
    }
    double *vv = reinterpret_cast<double *>(p + off_val);
    size_t pos = 0;
    for (int k = 0; k < K; ++k) {
        const int ck = cnt[k];
        if (rows[0].vals)
            for (int v = 0; v < b2; ++v)
                for (int t = 0; t < ck; ++t) vv[b2 * pos + (size_t)v * ck + t] = rows[t].vals[b2 * (size_t)k + v];
        int64_t *mo = upper ? mp.Uoff : mp.Loff;
        int32_t *ms = upper ? mp.Ust : mp.Lst;
        if (mp.on)
            for (int t = 0; t < ck; ++t) {
                mo[rows[t].src0 + k] = (int64_t)(base + off_val + 8 * (b2 * pos + (size_t)t));
                ms[rows[t].src0 + k] = 8 * ck;
            }
        pos += ck;
    }
}

// groups: sequences of rows; barrier after each group with barrier flag.
void pack_groups(Sink &out, std::vector<std::vector<RowRef>> &groups,
                 const std::vector<bool> &barrier, bool upper, int rmax, int32_t col_base,
                 int32_t &n_rec, int64_t &max_rec, bool last_section, const SlabMaps &mp, int b2, const Swz &sw) {
    for (size_t g = 0; g < groups.size(); ++g) {
        auto &rows = groups[g];
        std::stable_sort(rows.begin(), rows.end(),
                         [](const RowRef &a, const RowRef &b) { return a.nblk > b.nblk; });
        const int w = (int)rows.size();
        for (int s = 0; s < w; s += rmax) {
            const int e = std::min(w, s + rmax);
            std::vector<RowRef> part(rows.begin() + s, rows.begin() + e);
            uint16_t fl = 0;
            if (e == w && barrier[g]) fl |= REC_BARRIER;
            if (last_section && g + 1 == groups.size() && e == w) fl |= REC_LAST;
            put_record(out, part, upper, fl, col_base, max_rec, mp, b2, sw);
            ++n_rec;
        }
    }
}

}  // namespace

// ------------------------------------------------ shared-vector swizzle
// Bank model of the level-set kernel's vector accesses (8-byte accesses, a
// warp served in two 16-lane halves, 32 four-byte banks): per record warp,
// the own row's 3 loads + 3 stores and, for each of up to 3 blocks, the 3
// loads of x_j (absent blocks read the own row, branch-free path). Returns
// the wavefronts of one subdomain under swizzle sw.
namespace {
int64_t bank_cost(const dd_ctx *ctx, int64_t la, int64_t P, int rmax, const Swz &sw) {
    int64_t cost = 0;
    auto wave = [](const uint32_t *word, int n) {
        int64_t tot = 0;
        for (int h0 = 0; h0 < n; h0 += 16) {
            uint32_t seen[32][32];
            int cnt[32] = {0};
            int mx = 0;
            for (int l = h0; l < std::min(n, h0 + 16); ++l)
                for (uint32_t w : {word[l], word[l] + 1}) {
                    const int b = (int)(w & 31u);
                    bool dup = false;
                    for (int q = 0; q < cnt[b]; ++q) dup |= seen[b][q] == w;
                    if (!dup) seen[b][cnt[b]++] = w;
                    mx = std::max(mx, cnt[b]);
                }
            tot += mx;
        }
        return tot;
    };
    for (int up = 0; up < 2; ++up) {
        const auto &hm = up ? ctx->hmapU : ctx->hmapL;
        const auto &rp = up ? ctx->Urp : ctx->Lrp;
        const auto &cl = up ? ctx->Uci : ctx->Lci;
        int32_t hmax = 0;
        for (int64_t i = 0; i < P; ++i) hmax = std::max(hmax, hm[la + i]);
        std::vector<std::vector<int64_t>> lv(hmax + 1);
        for (int64_t i = 0; i < P; ++i) lv[hm[la + i]].push_back(i);
        for (int32_t l = up ? 0 : 1; l <= hmax; ++l) {
            auto &rows = lv[l];
            std::stable_sort(rows.begin(), rows.end(), [&](int64_t a, int64_t b) {
                return rp[la + a + 1] - rp[la + a] > rp[la + b + 1] - rp[la + b];
            });
            for (size_t w0 = 0; w0 < rows.size(); w0 += 32) {
                // warps never straddle records (rmax is a multiple of 32 or smaller)
                const int n = (int)std::min<size_t>(32, std::min(rows.size() - w0, (size_t)rmax - w0 % rmax));
                uint32_t word[32];
                for (int c = 0; c < 3; ++c) {
                    for (int q = 0; q < n; ++q) word[q] = 2u * (3u * sw.slot((uint32_t)rows[w0 + q]) + c);
                    cost += 2 * wave(word, n);
                }
                for (int k = 0; k < 3; ++k)
                    for (int c = 0; c < 3; ++c) {
                        for (int q = 0; q < n; ++q) {
                            const int64_t i = rows[w0 + q], li = la + i;
                            // absent blocks read the zero slot (a broadcast)
                            word[q] = k < rp[li + 1] - rp[li] ? 2u * (3u * sw.slot((uint32_t)(cl[rp[li] + k] - la)) + c)
                                                              : 2u * (3u * (uint32_t)(P + 16) + c);
                        }
                        cost += wave(word, n);
                    }
            }
        }
    }
    return cost;
}
}  // namespace

// Pick the slot swizzle with the fewest modelled wavefronts on (up to 3)
// sample subdomains, among those that add at most 16 slots (384 B: at P 2048
// the level-set and sync-free kernels keep two CTAs per SM; 32 slots cost the
// sync-free variant its second CTA, measured 0.54 -> 0.89 ms). 3x3 rows only; DD_SWZ=0 keeps
// the identity. Sets ctx->swz and ctx->vec_rows.
void choose_swizzle(dd_ctx *ctx, int64_t r0) {
    ctx->swz = Swz{};
    ctx->vec_rows = ctx->max_P;
    // one slot past the rows holds 0.0 (Swz::zslot)
    auto add_zero_slot = [ctx] {
        ctx->swz.zslot = (uint32_t)ctx->vec_rows;
        ctx->vec_rows += 1;
    };
    const char *e = getenv("DD_SWZ");
    if (ctx->bs != 3 || ctx->max_P <= 0 || (e && atoi(e) == 0)) {
        add_zero_slot();
        return;
    }
    const int nsl = ctx->sub_last - ctx->sub_first;
    std::vector<Swz> cands{Swz{}};
    for (uint32_t s1 = 4; s1 <= 9; ++s1)
        for (uint32_t p1 = 1; p1 <= 7; ++p1)
            for (uint32_t s2 : {31u, 8u, 9u, 10u, 11u})
                for (uint32_t p2 : {0u, 1u, 2u, 3u, 5u}) {
                    if ((s2 == 31) != (p2 == 0) || (s2 != 31 && s2 <= s1)) continue;
                    const Swz c{s1, p1, s2, p2};
                    if (c.slot((uint32_t)ctx->max_P - 1) + 1 - (uint32_t)ctx->max_P <= 16) cands.push_back(c);
                }
    std::vector<int64_t> cost(cands.size(), 0);
    const int rmax = ctx->bs == 1 ? 256 : 128;
#pragma omp parallel for schedule(dynamic, 4)
    for (int q = 0; q < (int)cands.size(); ++q)
        for (int s = 0; s < std::min(nsl, 3); ++s) {
            const int32_t g = ctx->sub_first + s * std::max(1, nsl / 3);
            const int64_t a = ctx->sub_ptr[g], P = ctx->sub_ptr[g + 1] - a;
            cost[q] += bank_cost(ctx, a - r0, P, rmax, cands[q]);
        }
    int best = 0;
    for (int q = 1; q < (int)cands.size(); ++q)
        if (cost[q] < cost[best]) best = q;
    // keep the identity unless the gain is worth the extra integer work (> 5 %)
    if (cost[best] * 20 >= cost[0] * 19) best = 0;
    ctx->swz = cands[best];
    ctx->vec_rows = (int32_t)ctx->swz.slot((uint32_t)ctx->max_P - 1) + 1;
    add_zero_slot();
}

// ------------------------------------------------------------ host setup
dd_status host_setup(dd_ctx *ctx, const dd_bsr3 *A, const dd_opts *o) {
    const double t0 = now_ms();
    const int64_t N = A->n_block_rows;
    if (N <= 0 || !A->row_ptr || !A->col_idx || !A->vals || A->nnzb < 0) {
        set_error("dd_setup: empty or NULL matrix");
        return DD_E_INVALID_ARG;
    }
    if (N > INT32_MAX - 1) {
        set_error("dd_setup: more than 2^31-1 block rows");
        return DD_E_INVALID_ARG;
    }
    const int64_t *rp = A->row_ptr;
    const int32_t *ci = A->col_idx;
    const double *av = A->vals;
    if (rp[0] != 0 || rp[N] != A->nnzb) {
        set_error("dd_setup: row_ptr[0] != 0 or row_ptr[n] != nnzb");
        return DD_E_INVALID_ARG;
    }
    if (o->n_threads > 0) omp_set_num_threads(o->n_threads);
    const int bs = ctx->bs, b2 = bs * bs;  // 3: BSR3, 1: scalar CSR
    if (bs == 1 && o->enable_refactor) {
        set_error("dd_setup: enable_refactor is not supported for the scalar CSR path");
        return DD_E_INVALID_ARG;
    }
    ctx->N = N;
    ctx->nnzb_A = A->nnzb;

    // ---- validate: monotone row_ptr, in-range, strictly ascending, diagonal
    int64_t bad_unsorted = INT64_MAX, bad_diag = INT64_MAX, bad_range = INT64_MAX;
#pragma omp parallel for schedule(static) reduction(min : bad_unsorted, bad_diag, bad_range)
    for (int64_t i = 0; i < N; ++i) {
        if (rp[i + 1] < rp[i]) {
            bad_range = std::min(bad_range, i);
            continue;
        }
        bool diag = false;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            if (ci[p] < 0 || ci[p] >= N) bad_range = std::min(bad_range, i);
            if (p > rp[i] && ci[p] <= ci[p - 1]) bad_unsorted = std::min(bad_unsorted, i);
            diag |= (ci[p] == i);
        }
        if (!diag) bad_diag = std::min(bad_diag, i);
    }
    if (bad_range != INT64_MAX) {
        set_error("dd_setup: bad row_ptr or column out of range at row " + std::to_string(bad_range));
        return DD_E_INVALID_ARG;
    }
    if (bad_unsorted != INT64_MAX) {
        set_error("dd_setup: columns not strictly ascending in row " + std::to_string(bad_unsorted));
        return DD_E_UNSORTED_OR_DUP;
    }
    if (bad_diag != INT64_MAX) {
        set_error("dd_setup: missing diagonal block in row " + std::to_string(bad_diag));
        return DD_E_MISSING_DIAG;
    }

    // ---- labels: Alg. 2 or contiguous chunks
    ctx->labels.assign(N, 0);
    if (o->grid) {
        const dd_grid g = *o->grid;
        if (g.nx <= 0 || g.ny <= 0 || g.nz <= 0 || g.tx <= 0 || g.ty <= 0 || g.tz <= 0 ||
            (int64_t)g.nx * g.ny * g.nz != N) {
            set_error("dd_setup: grid does not match the matrix");
            return DD_E_INVALID_ARG;
        }
        if (g.nx % g.tx || g.ny % g.ty || g.nz % g.tz) {
            set_error("dd_setup: grid not divisible by tile dims");
            return DD_E_GRID_NOT_DIVISIBLE;
        }
        const int64_t bx = g.nx / g.tx, by = g.ny / g.ty;
#pragma omp parallel for schedule(static)
        for (int64_t gidx = 0; gidx < N; ++gidx) {
            const int64_t i = gidx % g.nx, j = (gidx / g.nx) % g.ny, k = gidx / ((int64_t)g.nx * g.ny);
            ctx->labels[gidx] = (int32_t)(i / g.tx + bx * (j / g.ty + by * (k / g.tz)));
        }
    } else {
        if (o->subdomain_rows <= 0) {
            set_error("dd_setup: subdomain_rows must be > 0 without a grid");
            return DD_E_INVALID_ARG;
        }
        const int64_t P = o->subdomain_rows;
        if (o->partitioner == DD_PART_BFS) {
            // graph growing: BFS from the lowest unassigned row, exact part size P
            std::fill(ctx->labels.begin(), ctx->labels.end(), -1);
            std::vector<int64_t> q(N);
            int64_t assigned = 0, seed = 0;
            int32_t part = 0;
            while (assigned < N) {
                size_t head = 0, tail = 0;
                int64_t filled = 0;
                while (filled < P && assigned < N) {
                    if (head == tail) {
                        while (ctx->labels[seed] != -1) ++seed;
                        ctx->labels[seed] = part;
                        ++filled;
                        ++assigned;
                        q[tail++] = seed;
                        continue;
                    }
                    const int64_t u = q[head++];
                    for (int64_t e = rp[u]; e < rp[u + 1] && filled < P; ++e) {
                        const int64_t w = ci[e];
                        if (w != u && ctx->labels[w] == -1) {
                            ctx->labels[w] = part;
                            ++filled;
                            ++assigned;
                            q[tail++] = w;
                        }
                    }
                }
                ++part;
            }
        } else {
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < N; ++i) ctx->labels[i] = (int32_t)(i / P);
        }
    }
    int32_t maxl = 0;
    for (int64_t i = 0; i < N; ++i) maxl = std::max(maxl, ctx->labels[i]);
    const int32_t n_sub = maxl + 1;
    ctx->n_sub = n_sub;

    // ---- stable grouping permutation (counting sort)
    ctx->sub_ptr.assign((size_t)n_sub + 1, 0);
    for (int64_t i = 0; i < N; ++i) ctx->sub_ptr[ctx->labels[i] + 1]++;
    for (int32_t s = 0; s < n_sub; ++s) ctx->sub_ptr[s + 1] += ctx->sub_ptr[s];
    ctx->new_to_old.assign(N, 0);
    ctx->old_to_new.assign(N, 0);
    {
        std::vector<int64_t> fill(ctx->sub_ptr.begin(), ctx->sub_ptr.end() - 1);
        for (int64_t i = 0; i < N; ++i) ctx->new_to_old[fill[ctx->labels[i]]++] = (int32_t)i;
    }
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < N; ++j) ctx->old_to_new[ctx->new_to_old[j]] = (int32_t)j;
    int64_t maxP = 0;
    for (int32_t s = 0; s < n_sub; ++s) maxP = std::max(maxP, ctx->sub_ptr[s + 1] - ctx->sub_ptr[s]);
    if (maxP > 65535) {
        set_error("dd_setup: subdomain larger than 65535 block rows");
        return DD_E_SUBDOMAIN_TOO_LARGE;
    }
    ctx->max_P = (int32_t)maxP;

    // ---- this rank's subdomains (count-balanced contiguous range, R32)
    const int world = std::max(1, ctx->world), rank = ctx->rank;
    ctx->sub_first = (int32_t)((int64_t)n_sub * rank / world);
    ctx->sub_last = (int32_t)((int64_t)n_sub * (rank + 1) / world);
    ctx->row_first = ctx->sub_ptr[ctx->sub_first];
    const int64_t nl = ctx->sub_ptr[ctx->sub_last] - ctx->row_first;
    ctx->n_local = nl;
    const int64_t r0 = ctx->row_first;
    const double t1 = now_ms();
    ctx->setup_ms[0] = t1 - t0;

    // ---- Alg. 3 reorder of the local rows (global reordered column ids)
    std::vector<int64_t> &Arp = ctx->Arp;
    Arp.assign(nl + 1, 0);
    for (int64_t li = 0; li < nl; ++li) {
        const int64_t m = ctx->new_to_old[r0 + li];
        Arp[li + 1] = Arp[li] + (rp[m + 1] - rp[m]);
    }
    const int64_t nnz_loc = Arp[nl];
    uvector<int32_t> gcol(nnz_loc);  // every entry written below
    ctx->refactor = o->enable_refactor != 0;
    // GPU numeric path (dd_setup on a device, BSR3, no DD_ILU0 slab): the host
    // does the symbolic work only -- pattern, levels, slab layout, refactor
    // maps -- and k_refactor9 computes L, Dinv and U_unit straight into the
    // slab from the original values; the maps are built
    const bool gpu_num = ctx->gpu_numeric;
    if (gpu_num) ctx->refactor = true;
    if (!gpu_num) ctx->Av.resize(b2 * nnz_loc);  // every block written below (GPU path: values gathered on the device)
    ctx->pivot_floor = o->pivot_floor > 0 ? o->pivot_floor : 1e-300;
    if (ctx->refactor && A->nnzb >= INT32_MAX) {
        // the refactor maps index the caller's blocks with int32 (2^31 blocks
        // would be 155 GB of values alone)
        set_error("dd_setup: enable_refactor / GPU factorisation needs fewer than 2^31 blocks");
        return DD_E_INVALID_ARG;
    }
    if (ctx->refactor) ctx->Asrc.resize(nnz_loc);  // every entry written below
#pragma omp parallel for schedule(static)
    for (int64_t li = 0; li < nl; ++li) {
        const int64_t m = ctx->new_to_old[r0 + li];
        const int64_t nb = rp[m + 1] - rp[m];
        int32_t idx[64];
        int32_t nc[64];
        std::vector<int32_t> big_idx, big_nc;
        int32_t *ix = idx, *cc = nc;
        if (nb > 64) {
            big_idx.resize(nb);
            big_nc.resize(nb);
            ix = big_idx.data();
            cc = big_nc.data();
        }
        for (int64_t t = 0; t < nb; ++t) {
            ix[t] = (int32_t)t;
            cc[t] = ctx->old_to_new[ci[rp[m] + t]];
        }
        std::sort(ix, ix + nb, [&](int32_t a, int32_t b) { return cc[a] < cc[b]; });
        for (int64_t t = 0; t < nb; ++t) {
            gcol[Arp[li] + t] = cc[ix[t]];
            if (!gpu_num) std::memcpy(&ctx->Av[b2 * (Arp[li] + t)], &av[b2 * (rp[m] + ix[t])], b2 * sizeof(double));
            if (ctx->refactor) ctx->Asrc[Arp[li] + t] = (int32_t)(rp[m] + ix[t]);
        }
    }
    // global drop statistics (count of same-label blocks over all rows)
    {
        int64_t kept = 0;
#pragma omp parallel for schedule(static) reduction(+ : kept)
        for (int64_t i = 0; i < N; ++i)
            for (int64_t p = rp[i]; p < rp[i + 1]; ++p) kept += (ctx->labels[i] == ctx->labels[ci[p]]);
        ctx->nnzb_dd = kept;
    }
    // halo numbering: local columns 0..nl-1, ghosts nl.. (ascending global id)
    {
        std::vector<int32_t> gh;
        for (int64_t p = 0; p < nnz_loc; ++p)
            if (gcol[p] < r0 || gcol[p] >= r0 + nl) gh.push_back(gcol[p]);
        std::sort(gh.begin(), gh.end());
        gh.erase(std::unique(gh.begin(), gh.end()), gh.end());
        ctx->ghost_rows.assign(gh.begin(), gh.end());
        ctx->ghost_owner.resize(gh.size());
        for (size_t q = 0; q < gh.size(); ++q) {
            // owner = rank whose subdomain range contains row gh[q]
            const int64_t s = std::upper_bound(ctx->sub_ptr.begin(), ctx->sub_ptr.end(), (int64_t)gh[q]) -
                              ctx->sub_ptr.begin() - 1;
            int own = 0;
            for (int rr = 0; rr < world; ++rr)
                if (s >= (int64_t)n_sub * rr / world && s < (int64_t)n_sub * (rr + 1) / world) own = rr;
            ctx->ghost_owner[q] = own;
        }
        ctx->recv_off.assign(world + 1, 0);
        for (size_t q = 0; q < gh.size(); ++q) ctx->recv_off[ctx->ghost_owner[q] + 1]++;
        for (int rr = 0; rr < world; ++rr) ctx->recv_off[rr + 1] += ctx->recv_off[rr];
        // send lists: my rows that peer q reads (ascending = q's ghost order)
        ctx->send_rows.assign(world, {});
        for (int q = 0; q < world && world > 1; ++q) {
            if (q == rank) continue;
            const int64_t qa = ctx->sub_ptr[(int64_t)n_sub * q / world];
            const int64_t qe = ctx->sub_ptr[(int64_t)n_sub * (q + 1) / world];
            std::vector<int32_t> need;
#pragma omp parallel
            {
                std::vector<int32_t> mine;
#pragma omp for schedule(static) nowait
                for (int64_t g = qa; g < qe; ++g) {
                    const int64_t m = ctx->new_to_old[g];
                    for (int64_t p = rp[m]; p < rp[m + 1]; ++p) {
                        const int64_t c = ctx->old_to_new[ci[p]];
                        if (c >= r0 && c < r0 + nl) mine.push_back((int32_t)(c - r0));
                    }
                }
#pragma omp critical
                need.insert(need.end(), mine.begin(), mine.end());
            }
            std::sort(need.begin(), need.end());
            need.erase(std::unique(need.begin(), need.end()), need.end());
            ctx->send_rows[q] = std::move(need);
        }
        ctx->Aci.resize(nnz_loc);
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < nnz_loc; ++p) {
            const int32_t g = gcol[p];
            if (g >= r0 && g < r0 + nl)
                ctx->Aci[p] = (int32_t)(g - r0);
            else
                ctx->Aci[p] = (int32_t)(nl + (std::lower_bound(gh.begin(), gh.end(), g) - gh.begin()));
        }
    }
    const double t2 = now_ms();
    ctx->setup_ms[1] = t2 - t1;

    // ---- factor pattern sizes (drop: keep same-subdomain blocks)
    const int32_t s0 = ctx->sub_first, s1 = ctx->sub_last, nsl = s1 - s0;
    std::vector<int32_t> row_sub(nl);
    for (int32_t s = s0; s < s1; ++s)
        for (int64_t g = ctx->sub_ptr[s]; g < ctx->sub_ptr[s + 1]; ++g) row_sub[g - r0] = s;
    ctx->Lrp.assign(nl + 1, 0);
    ctx->Urp.assign(nl + 1, 0);
#pragma omp parallel for schedule(static)
    for (int64_t li = 0; li < nl; ++li) {
        const int32_t s = row_sub[li];
        const int64_t a = ctx->sub_ptr[s], e = ctx->sub_ptr[s + 1];
        int64_t nL = 0, nU = 0;
        for (int64_t p = Arp[li]; p < Arp[li + 1]; ++p) {
            const int64_t g = gcol[p];
            if (g >= a && g < e) {
                if (g < r0 + li) ++nL;
                if (g > r0 + li) ++nU;
            }
        }
        ctx->Lrp[li + 1] = nL;
        ctx->Urp[li + 1] = nU;
    }
    for (int64_t li = 0; li < nl; ++li) {
        ctx->Lrp[li + 1] += ctx->Lrp[li];
        ctx->Urp[li + 1] += ctx->Urp[li];
    }
    static const bool trace2 = getenv("DD_SETUP_TRACE") != nullptr;
    if (trace2) fprintf(stderr, "[dd setup] pattern sizes     %9.1f ms\n", now_ms() - t2);
    ctx->Lci.resize(ctx->Lrp[nl]);
    ctx->Uci.resize(ctx->Urp[nl]);
    if (!gpu_num) {
        ctx->Lv.resize(b2 * ctx->Lrp[nl]);  // written by the scatter below
        ctx->Uv.resize(b2 * ctx->Urp[nl]);
    }
    // DD_ILU0 ablation: keep the non-unit U_ij too (a second slab, BSR3 only)
    const bool want_ilu = bs == 3 && (o->variants & DD_ILU0) != 0;
    if (want_ilu) ctx->Uraw.resize(b2 * ctx->Urp[nl]);
    if (!gpu_num) ctx->Dinv.resize(b2 * nl);
    ctx->hmapL.assign(nl, 0);
    ctx->hmapU.assign(nl, 0);
    if (trace2) fprintf(stderr, "[dd setup] factor arrays     %9.1f ms\n", now_ms() - t2);

    // ---- per-subdomain block ILU0 -> ILDU0 -> levels
    const double floor_ = o->pivot_floor > 0 ? o->pivot_floor : 1e-300;
    int64_t bad_pivot = INT64_MAX;
#pragma omp parallel reduction(min : bad_pivot)
    {
        std::vector<int64_t> lrp;
        std::vector<int32_t> lci;
        std::vector<double> W;
        std::vector<int64_t> ldg, pos;
#pragma omp for schedule(dynamic, 1)
        for (int32_t s = s0; s < s1; ++s) {
            const int64_t a = ctx->sub_ptr[s], e = ctx->sub_ptr[s + 1], P = e - a;
            const int64_t la = a - r0;  // local row of the first subdomain row
            // subdomain-local CSR of A_dd
            lrp.assign(P + 1, 0);
            lci.clear();
            W.clear();
            for (int64_t i = 0; i < P; ++i) {
                const int64_t li = la + i;
                for (int64_t p = Arp[li]; p < Arp[li + 1]; ++p) {
                    const int64_t g = gcol[p];
                    if (g >= a && g < e) {
                        lci.push_back((int32_t)(g - a));
                        if (!gpu_num) W.insert(W.end(), &ctx->Av[b2 * p], &ctx->Av[b2 * p] + b2);
                    }
                }
                lrp[i + 1] = (int64_t)lci.size();
            }
            if (gpu_num) {
                // pattern only: the values are factored on the device
                for (int64_t i = 0; i < P; ++i) {
                    const int64_t li = la + i;
                    int64_t qL = ctx->Lrp[li], qU = ctx->Urp[li];
                    for (int64_t p = lrp[i]; p < lrp[i + 1]; ++p) {
                        if (lci[p] < i) ctx->Lci[qL++] = (int32_t)(la + lci[p]);
                        else if (lci[p] > i) ctx->Uci[qU++] = (int32_t)(la + lci[p]);
                    }
                }
            }
            ldg.assign(P, -1);
            for (int64_t i = 0; i < P; ++i)
                for (int64_t p = lrp[i]; p < lrp[i + 1]; ++p)
                    if (lci[p] == i) ldg[i] = p;
            pos.assign(P, -1);
            bool failed = false;
            for (int64_t i = 0; i < P && !failed && !gpu_num; ++i) {
                for (int64_t p = lrp[i]; p < lrp[i + 1]; ++p) pos[lci[p]] = p;
                for (int64_t p = lrp[i]; p < ldg[i]; ++p) {
                    const int64_t k = lci[p];
                    // L_ik = W_ik * U_kk^-1 (right multiplication, R12)
                    bmul(bs, &W[b2 * p], &ctx->Dinv[b2 * (la + k)], &W[b2 * p]);
                    // W_ij -= L_ik U_kj for j in pattern(i) and (k,j) in U
                    for (int64_t q = ldg[k] + 1; q < lrp[k + 1]; ++q) {
                        const int64_t tgt = pos[lci[q]];
                        if (tgt >= 0) bsub_mul(bs, &W[b2 * tgt], &W[b2 * p], &W[b2 * q]);
                    }
                }
                if (!binv(bs, &W[b2 * ldg[i]], floor_, &ctx->Dinv[b2 * (la + i)])) {
                    bad_pivot = std::min(bad_pivot, a + i);
                    failed = true;
                }
                for (int64_t p = lrp[i]; p < lrp[i + 1]; ++p) pos[lci[p]] = -1;
            }
            if (failed) continue;
            // scatter: L (strictly lower) and U_unit = Dinv_i * U_ij (j > i)
            for (int64_t i = 0; i < P && !gpu_num; ++i) {
                const int64_t li = la + i;
                int64_t qL = ctx->Lrp[li], qU = ctx->Urp[li];
                for (int64_t p = lrp[i]; p < lrp[i + 1]; ++p) {
                    if (lci[p] < i) {
                        ctx->Lci[qL] = (int32_t)(la + lci[p]);
                        std::memcpy(&ctx->Lv[b2 * qL], &W[b2 * p], b2 * sizeof(double));
                        ++qL;
                    } else if (lci[p] > i) {
                        ctx->Uci[qU] = (int32_t)(la + lci[p]);
                        bmul(bs, &ctx->Dinv[b2 * li], &W[b2 * p], &ctx->Uv[b2 * qU]);
                        if (want_ilu) std::memcpy(&ctx->Uraw[b2 * qU], &W[b2 * p], b2 * sizeof(double));
                        ++qU;
                    }
                }
            }
            // longest-path levels (Alg. 5 fixpoint == longest path, R16)
            for (int64_t i = 0; i < P; ++i) {
                const int64_t li = la + i;
                int32_t h = 0;
                for (int64_t q = ctx->Lrp[li]; q < ctx->Lrp[li + 1]; ++q) h = std::max(h, ctx->hmapL[ctx->Lci[q]] + 1);
                ctx->hmapL[li] = h;
            }
            for (int64_t i = P - 1; i >= 0; --i) {
                const int64_t li = la + i;
                int32_t h = 0;
                for (int64_t q = ctx->Urp[li]; q < ctx->Urp[li + 1]; ++q) h = std::max(h, ctx->hmapU[ctx->Uci[q]] + 1);
                ctx->hmapU[li] = h;
            }
        }
    }
    const double t3 = now_ms();
    ctx->setup_ms[2] = t3 - t2;
    if (trace2) fprintf(stderr, "[dd setup] subdomain loop    %9.1f ms\n", t3 - t2);
    // global pivot status must agree across ranks; the API layer reduces it.
    if (bad_pivot != INT64_MAX) {
        set_error("dd_setup: singular pivot block (|det| < pivot_floor) at reordered row " +
                  std::to_string(bad_pivot));
        return DD_E_SINGULAR_PIVOT;
    }
    int32_t mL = 0, mU = 0;
    for (int64_t li = 0; li < nl; ++li) {
        mL = std::max(mL, ctx->hmapL[li]);
        mU = std::max(mU, ctx->hmapU[li]);
    }
    ctx->max_lev_L = mL + 1;
    ctx->max_lev_U = mU + 1;
    if (ctx->refactor) {
        // A_dd working layout W (rank-local rows, same order as the host ILU0)
        ctx->Wrp.assign(nl + 1, 0);
        for (int64_t li = 0; li < nl; ++li)
            ctx->Wrp[li + 1] = ctx->Wrp[li] + (ctx->Lrp[li + 1] - ctx->Lrp[li]) + 1 + (ctx->Urp[li + 1] - ctx->Urp[li]);
        const int64_t nW = ctx->Wrp[nl];
        if (nW >= INT32_MAX) {
            set_error("dd_setup: refactor maps need fewer than 2^31 dropped-pattern blocks per rank");
            return DD_E_INVALID_ARG;
        }
        ctx->Wsrc.resize(nW);
        ctx->Wcol.resize(nW);
        ctx->Wdiag.assign(nl, 0);
        ctx->Uptr.resize(nW + 1);
        ctx->Uptr[0] = 0;
        uvector<int32_t> nupd(nW);
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < nW; ++p) nupd[p] = 0;
#pragma omp parallel for schedule(static)
        for (int64_t li = 0; li < nl; ++li) {
            const int32_t s = row_sub[li];
            const int64_t a = ctx->sub_ptr[s], e = ctx->sub_ptr[s + 1];
            int64_t q = ctx->Wrp[li];
            for (int64_t p = Arp[li]; p < Arp[li + 1]; ++p) {
                const int64_t g = gcol[p];
                if (g >= a && g < e) {
                    ctx->Wsrc[q] = ctx->Asrc[p];
                    ctx->Wcol[q] = (int32_t)(g - r0);
                    if (g == r0 + li) ctx->Wdiag[li] = q;
                    ++q;
                }
            }
        }
        static const bool trace = getenv("DD_SETUP_TRACE") != nullptr;
        if (trace) fprintf(stderr, "[dd setup] refactor W layout %9.1f ms\n", now_ms() - t3);
        // update lists: for lower position p = (i, k): every U_kj (j > k) whose
        // column j is in row i's pattern -> (position of U_kj, position of W_ij),
        // in ascending j (the order of the host / oracle elimination)
        auto for_updates = [&](int64_t li, auto &&fn) {
            for (int64_t p = ctx->Wrp[li]; p < ctx->Wdiag[li]; ++p) {
                const int64_t k = ctx->Wcol[p];
                for (int64_t qk = ctx->Wdiag[k] + 1; qk < ctx->Wrp[k + 1]; ++qk) {
                    const int32_t j = ctx->Wcol[qk];
                    // position of column j in row li (rows are short: linear scan)
                    for (int64_t t = p + 1; t < ctx->Wrp[li + 1]; ++t)
                        if (ctx->Wcol[t] == j) {
                            fn(p, qk, t);
                            break;
                        }
                }
            }
        };
#pragma omp parallel for schedule(static)
        for (int64_t li = 0; li < nl; ++li) for_updates(li, [&](int64_t p, int64_t, int64_t) { ++nupd[p]; });
        for (int64_t p = 0; p < nW; ++p) ctx->Uptr[p + 1] = ctx->Uptr[p] + nupd[p];
        ctx->UpdQ.resize(ctx->Uptr[nW]);
        ctx->UpdT.resize(ctx->Uptr[nW]);
#pragma omp parallel for schedule(static)
        for (int64_t li = 0; li < nl; ++li) {
            // for_updates visits the updates of one position p consecutively
            int64_t last = -1, at = 0;
            for_updates(li, [&](int64_t p, int64_t qk, int64_t t) {
                at = p == last ? at + 1 : ctx->Uptr[p];
                last = p;
                ctx->UpdQ[at] = (int32_t)qk;
                ctx->UpdT[at] = (int32_t)t;
            });
        }
        if (trace) fprintf(stderr, "[dd setup] refactor updates  %9.1f ms\n", now_ms() - t3);
        // level lists per local subdomain: L levels ascending, rows in the
        // order of the slab's L records (stable by L block count, descending),
        // so the refactor kernel's L-block stores to the slab planes are
        // coalesced; and all rows in the order of the U records (U levels
        // ascending, stable by U block count) for its Dinv / U_unit pass
        auto nL = [&](int32_t li) { return ctx->Lrp[li + 1] - ctx->Lrp[li]; };
        auto nU = [&](int32_t li) { return ctx->Urp[li + 1] - ctx->Urp[li]; };
        // per subdomain in parallel, then concatenated in subdomain order
        std::vector<std::vector<int32_t>> lrows(nsl), lptr(nsl), urows(nsl);
#pragma omp parallel for schedule(dynamic, 8)
        for (int32_t q = 0; q < nsl; ++q) {
            const int64_t a = ctx->sub_ptr[s0 + q] - r0, e = ctx->sub_ptr[s0 + q + 1] - r0;
            int32_t hl = 0, hu = 0;
            for (int64_t li = a; li < e; ++li) {
                hl = std::max(hl, ctx->hmapL[li]);
                hu = std::max(hu, ctx->hmapU[li]);
            }
            std::vector<std::vector<int32_t>> lv(hl + 1), uv(hu + 1);
            for (int64_t li = a; li < e; ++li) {
                lv[ctx->hmapL[li]].push_back((int32_t)li);
                uv[ctx->hmapU[li]].push_back((int32_t)li);
            }
            for (auto &l : lv) {
                std::stable_sort(l.begin(), l.end(), [&](int32_t x, int32_t y) { return nL(x) > nL(y); });
                lptr[q].push_back((int32_t)lrows[q].size());
                lrows[q].insert(lrows[q].end(), l.begin(), l.end());
            }
            for (auto &u : uv) {
                std::stable_sort(u.begin(), u.end(), [&](int32_t x, int32_t y) { return nU(x) > nU(y); });
                urows[q].insert(urows[q].end(), u.begin(), u.end());
            }
        }
        ctx->SubLev.assign(nsl + 1, 0);
        ctx->SubU.assign(nsl + 1, 0);
        ctx->LevPtr.clear();
        ctx->LevRows.clear();
        ctx->LevRows.reserve(nl);
        ctx->URows.clear();
        ctx->URows.reserve(nl);
        for (int32_t q = 0; q < nsl; ++q) {
            ctx->SubLev[q] = (int32_t)ctx->LevPtr.size();
            const int32_t off = (int32_t)ctx->LevRows.size();
            for (int32_t p : lptr[q]) ctx->LevPtr.push_back(off + p);
            ctx->LevRows.insert(ctx->LevRows.end(), lrows[q].begin(), lrows[q].end());
            ctx->SubU[q] = (int32_t)ctx->URows.size();
            ctx->URows.insert(ctx->URows.end(), urows[q].begin(), urows[q].end());
        }
        ctx->LevPtr.push_back((int32_t)ctx->LevRows.size());
        ctx->SubLev[nsl] = (int32_t)ctx->LevPtr.size() - 1;
        ctx->SubU[nsl] = (int32_t)ctx->URows.size();
    }
    const double t4 = now_ms();
    ctx->setup_ms[3] = t4 - t3;

    // ---- slab packing (level-set and/or spin-loop orders)
    ctx->variants = o->variants ? o->variants : DD_LEVELSET;
    // rows per record: the largest of 128/64/32/16 whose worst-case record
    // (K blocks per row, U records carry Dinv) fits the staging ring that is
    // left next to the subdomain vector (B200: 232448 B opt-in per CTA).
    int32_t Kmax = 0;
    for (int64_t li = 0; li < nl; ++li)
        Kmax = std::max<int32_t>(Kmax, (int32_t)std::max(ctx->Lrp[li + 1] - ctx->Lrp[li], ctx->Urp[li + 1] - ctx->Urp[li]));
    ctx->kmax = Kmax;
    {
        const int64_t vec = (8 * bs * (int64_t)ctx->max_P + 127) / 128 * 128;
        const int64_t avail = 232448 - vec - 2 * (int64_t)ctx->max_P - 1024;
        int64_t ring = 131072;
        while (ring > 16384 && ring > avail) ring /= 2;
        const int64_t ch = ring / 4;  // = the kernels' ring chunk (apply.cu ring_chunk)
        int32_t rmax = bs == 1 ? 256 : 128;  // = the kernels' consumer threads (TCB)
        auto est = [&](int64_t R) {
            return (int64_t)rec_off_dinv(Kmax, (uint32_t)R) + 8 * b2 * R + 8 * b2 * R * Kmax + 16;
        };
        while (rmax > 16 && est(rmax) + ch > ring) rmax /= 2;
        // records may use fewer rows than consumer threads, never more
        if (const char *e = getenv("DD_ROWS_PER_REC")) rmax = std::max(16, std::min(rmax, atoi(e)));
        ctx->slab_lvl.rows_per_rec = rmax;
        ctx->slab_spin.rows_per_rec = rmax;
    }
    choose_swizzle(ctx, r0);
    SlabMaps mp;
    if (ctx->refactor) {
        ctx->SlabLoff.resize(ctx->Lci.size());
        ctx->SlabLst.resize(ctx->Lci.size());
        ctx->SlabUoff.resize(ctx->Uci.size());
        ctx->SlabUst.resize(ctx->Uci.size());
        ctx->SlabDoff.resize(nl);
        ctx->SlabDst.resize(nl);
        mp = SlabMaps{ctx->SlabLoff.data(), ctx->SlabUoff.data(), ctx->SlabDoff.data(),
                      ctx->SlabLst.data(), ctx->SlabUst.data(), ctx->SlabDst.data(), true};
    }
    auto build_slab = [&](ddi::Slab &slab, bool spin, const uvector<double> &Uvals, const SlabMaps &mp) {
        const int rmax = slab.rows_per_rec;
        slab.info.assign(nsl, SubInfo{});
        int64_t max_rec = 0;
        // subdomain q's record stream into `out` (two passes: sizes, then the
        // records written in place in the final buffer -- no per-subdomain
        // staging copies, no zero fill of the whole slab)
        auto pack_sub = [&](int32_t q, Sink &out, const SlabMaps &maps, int32_t &nrec, int64_t &mr, int32_t &u_off) {
            const int32_t s = s0 + q;
            const int64_t a = ctx->sub_ptr[s], e = ctx->sub_ptr[s + 1], P = e - a;
            const int64_t la = a - r0;
            auto rowL = [&](int64_t i) {
                const int64_t li = la + i;
                return RowRef{(int32_t)i, (int32_t)(ctx->Lrp[li + 1] - ctx->Lrp[li]), &ctx->Lci[ctx->Lrp[li]],
                              gpu_num ? nullptr : &ctx->Lv[b2 * ctx->Lrp[li]], nullptr, ctx->Lrp[li], li};
            };
            auto rowU = [&](int64_t i) {
                const int64_t li = la + i;
                return RowRef{(int32_t)i, (int32_t)(ctx->Urp[li + 1] - ctx->Urp[li]), &ctx->Uci[ctx->Urp[li]],
                              gpu_num ? nullptr : &Uvals[b2 * ctx->Urp[li]], gpu_num ? nullptr : &ctx->Dinv[b2 * li],
                              ctx->Urp[li], li};
            };
            std::vector<std::vector<RowRef>> gL, gU;
            std::vector<bool> bL, bU;
            if (!spin) {
                int32_t hl = 0, hu = 0;
                for (int64_t i = 0; i < P; ++i) {
                    hl = std::max(hl, ctx->hmapL[la + i]);
                    hu = std::max(hu, ctx->hmapU[la + i]);
                }
                gL.assign(hl + 1, {});
                gU.assign(hu + 1, {});
                for (int64_t i = 0; i < P; ++i) {
                    gL[ctx->hmapL[la + i]].push_back(rowL(i));
                    gU[ctx->hmapU[la + i]].push_back(rowU(i));
                }
                // L level 0 (no lower blocks: z_i = r_i) stays as a block-free
                // record: the level-set kernels skip it, the sync-free kernel
                // publishes its ready flags from it
                bL.assign(gL.size(), true);
                bU.assign(gU.size(), true);
            } else {
                for (int64_t i = 0; i < P; i += rmax) {
                    gL.emplace_back();
                    for (int64_t t = i; t < std::min(P, i + rmax); ++t) gL.back().push_back(rowL(t));
                }
                for (int64_t i = P - 1; i >= 0; i -= rmax) {
                    gU.emplace_back();
                    for (int64_t t = i; t > std::max<int64_t>(-1, i - rmax); --t) gU.back().push_back(rowU(t));
                }
                bL.assign(gL.size(), true);
                bU.assign(gU.size(), true);
            }
            nrec = 0;
            mr = 0;
            pack_groups(out, gL, bL, false, rmax, (int32_t)la, nrec, mr, false, maps, b2, ctx->swz);
            u_off = (int32_t)out.pos;
            pack_groups(out, gU, bU, true, rmax, (int32_t)la, nrec, mr, true, maps, b2, ctx->swz);
        };
#pragma omp parallel for schedule(dynamic, 4) reduction(max : max_rec)
        for (int32_t q = 0; q < nsl; ++q) {
            Sink sz;
            int32_t nrec = 0, u_off = 0;
            int64_t mr = 0;
            pack_sub(q, sz, SlabMaps{}, nrec, mr, u_off);
            const int32_t s = s0 + q;
            slab.info[q].u_off = u_off;
            slab.info[q].stream_bytes = (int32_t)sz.pos;
            slab.info[q].row0 = (int32_t)(ctx->sub_ptr[s] - r0);
            slab.info[q].nrows = (int32_t)(ctx->sub_ptr[s + 1] - ctx->sub_ptr[s]);
            slab.info[q].n_rec = nrec;
            max_rec = std::max(max_rec, mr);
        }
        int64_t off = 0;
        for (int32_t q = 0; q < nsl; ++q) {
            slab.info[q].stream_off = off;
            off += slab.info[q].stream_bytes;
        }
        slab.bytes.resize(off);
#pragma omp parallel for schedule(dynamic, 4)
        for (int32_t q = 0; q < nsl; ++q) {
            Sink out{slab.bytes.data() + slab.info[q].stream_off, 0};
            int32_t nrec = 0, u_off = 0;
            int64_t mr = 0;
            pack_sub(q, out, mp, nrec, mr, u_off);
            if (mp.on) {  // stream-relative -> slab-absolute offsets
                const int64_t so = slab.info[q].stream_off;
                for (int64_t li = slab.info[q].row0; li < slab.info[q].row0 + slab.info[q].nrows; ++li) {
                    mp.Doff[li] += so;
                    for (int64_t b = ctx->Lrp[li]; b < ctx->Lrp[li + 1]; ++b) mp.Loff[b] += so;
                    for (int64_t b = ctx->Urp[li]; b < ctx->Urp[li + 1]; ++b) mp.Uoff[b] += so;
                }
            }
        }
        slab.max_rec_bytes = max_rec;
    };
    // one level-ordered slab serves every variant (level order is a
    // topological order, which the sync-free variant also walks)
    build_slab(ctx->slab_lvl, false, ctx->Uv, mp);
    if (want_ilu) {
        ctx->slab_ilu.rows_per_rec = ctx->slab_lvl.rows_per_rec;
        build_slab(ctx->slab_ilu, false, ctx->Uraw, SlabMaps{});
        uvector<double>().swap(ctx->Uraw);
    } else {
        ctx->variants &= ~DD_ILU0;
    }

    // ---- sliced-ELL SpMV operand
    {
        auto &S = ctx->spmv;
        S.n_slices = (nl + 31) / 32;
        std::vector<int64_t> sp(S.n_slices + 1, 0);
        for (int64_t s = 0; s < S.n_slices; ++s) {
            int64_t K = 0;
            for (int64_t li = 32 * s; li < std::min(nl, 32 * s + 32); ++li) K = std::max(K, Arp[li + 1] - Arp[li]);
            sp[s + 1] = sp[s] + 32 * K;
        }
        S.n_slots = sp[S.n_slices];
        ctx->spmv_bytes = S.n_slots * (4 + 8 * b2) + 8 * (S.n_slices + 1);
    }
    ctx->setup_ms[4] = now_ms() - t4;
    return DD_OK;
}

}  // namespace ddi
