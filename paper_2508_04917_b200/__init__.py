"""Thin ctypes binding of include/dd.h (libdd.so, built in-tree).

Argument marshalling only: every step of the method runs in the C++ host
setup or the sm_100a kernels of libdd.so. There is no CPU fallback: if the
library is missing this module raises on first use.

Module-level functions carry the C ABI's names (dd_setup, dd_apply, dd_spmv,
dd_bicgstab, dd_solve_host, dd_permute, dd_unpermute, dd_get_*, dd_stats,
dd_launch_info, dd_solver_variant, dd_local_range, dd_destroy, dd_nccl_unique_id); ``Context``
wraps a dd_ctx*. Device vectors are torch CUDA tensors (float64, contiguous);
torch is used only for device memory, streams and process groups.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdd.so")
# development A/B runs may point at another in-tree build of the same library
if os.environ.get("DD_LIB"):
    LIB_PATH = os.path.abspath(os.environ["DD_LIB"])

DD_LEVELSET, DD_SPINLOOP, DD_DIRECT, DD_UNFUSED = 1, 2, 4, 8
# paper ablations (include/dd.h): edge-centric (shared / global vector), ILU0
# with the non-unit U, vertex-centric with the vector in global memory, and the
# DD_LOWER modifier (lower sweep alone)
DD_EDGE, DD_EDGE_GLOBAL, DD_ILU0, DD_DIRECT_GLOBAL, DD_LOWER, DD_TREE = 16, 32, 64, 128, 256, 512
DD_PART_CHUNKS, DD_PART_BFS = 0, 1
DD_COMM_NCCL, DD_COMM_LOCAL, DD_COMM_IPC = 0, 1, 2
STATUS = ["DD_OK", "DD_E_INVALID_ARG", "DD_E_NOT_SQUARE", "DD_E_UNSORTED_OR_DUP", "DD_E_MISSING_DIAG",
          "DD_E_SINGULAR_PIVOT", "DD_E_SUBDOMAIN_TOO_LARGE", "DD_E_GRID_NOT_DIVISIBLE", "DD_E_CUDA",
          "DD_E_NCCL", "DD_E_OOM", "DD_E_BREAKDOWN", "DD_E_MAXITER", "DD_E_NO_DEVICE"]
EXPORTS = ["dd_setup", "dd_setup_csr", "dd_destroy", "dd_local_range", "dd_apply", "dd_apply_variant", "dd_spmv",
           "dd_bicgstab", "dd_solve_host", "dd_permute", "dd_unpermute", "dd_get_partition",
           "dd_get_levels", "dd_levels_device", "dd_get_factors", "dd_get_halo", "dd_get_send_rows", "dd_stats", "dd_launch_info",
           "dd_solver_variant", "dd_profile", "dd_refactor", "dd_nccl_unique_id", "dd_choose_tiles", "dd_get_grid", "dd_last_error"]


class DDError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        self.name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{self.name}: {msg}")


class BSR3(C.Structure):
    _fields_ = [("n_block_rows", C.c_int64), ("nnzb", C.c_int64), ("row_ptr", C.c_void_p),
                ("col_idx", C.c_void_p), ("vals", C.c_void_p)]


class Grid(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("nx", "ny", "nz", "tx", "ty", "tz")]


class Opts(C.Structure):
    _fields_ = [("subdomain_rows", C.c_int32), ("grid", C.c_void_p), ("variants", C.c_int32),
                ("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_unique_id", C.c_void_p), ("pivot_floor", C.c_double), ("host_only", C.c_int32),
                ("n_threads", C.c_int32), ("enable_refactor", C.c_int32), ("partitioner", C.c_int32),
                ("comm", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_double), ("n_applies", C.c_int32), ("converged", C.c_int32),
                ("breakdown", C.c_int32), ("status", C.c_int32), ("rel_resid", C.c_double),
                ("true_rel_resid", C.c_double), ("solve_ms", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    """Load libdd.so (fail loudly if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        P, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        sig = {
            "dd_setup": [P, P, P], "dd_setup_csr": [P, P, P], "dd_destroy": [P], "dd_local_range": [P, P, P],
            "dd_apply": [P, P, P, P], "dd_apply_variant": [P, i32, P, P, P], "dd_spmv": [P, P, P, P],
            "dd_bicgstab": [P, P, P, d, i32, P, P, P], "dd_solve_host": [P, P, P, d, i32, P, P],
            "dd_permute": [P, P, P, P], "dd_unpermute": [P, P, P, P], "dd_get_partition": [P, P, P],
            "dd_get_levels": [P, i32, P], "dd_levels_device": [P, P, P, P], "dd_get_factors": [P] * 10, "dd_get_halo": [P, P, P, P], "dd_get_send_rows": [P, i32, P, P],
            "dd_stats": [P, P, P], "dd_profile": [P, i32, P], "dd_refactor": [P, P, i32, P], "dd_launch_info": [P, i32, P], "dd_solver_variant": [P, P, P], "dd_nccl_unique_id": [P],
            "dd_choose_tiles": [P, i32, i32, i32], "dd_get_grid": [P, P],
            "dd_last_error": [],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_char_p if name == "dd_last_error" else (None if name == "dd_destroy" else C.c_int)
        _lib = L
    return _lib


def _check(st):
    if st != 0:
        raise DDError(st, lib().dd_last_error().decode())
    return st


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _dev_vec(t, n, name, align16=False):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError(f"{name}: expected a contiguous float64 CUDA tensor")
    if t.numel() < n:
        raise ValueError(f"{name}: needs {n} elements, has {t.numel()}")
    if align16 and t.data_ptr() % 16:
        # the ring kernels stream r with 16-byte bulk copies (dd.h); a view at
        # an odd element offset is only 8-byte aligned
        raise ValueError(f"{name}: data pointer must be 16-byte aligned (view at an odd element offset?)")
    return t.data_ptr()


def _host_vec(a, n, name, writable=False):
    """A C-contiguous float64 numpy array of at least n elements (the C side
    reads or writes exactly n)."""
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
        raise TypeError(f"{name}: expected a C-contiguous float64 numpy array")
    if writable and not a.flags.writeable:
        raise ValueError(f"{name}: array is read-only")
    if a.size < n:
        raise ValueError(f"{name}: needs {n} elements, has {a.size}")
    return a.ctypes.data


def dd_choose_tiles(grid, device=0, bs=3, P_target=2048):
    """Tile dims (tx, ty, tz) for Alg. 2 that fill whole waves of the apply
    kernel's CTA slots (include/dd.h); device < 0: analytic occupancy model."""
    g = Grid(*grid, 0, 0, 0)
    _check(lib().dd_choose_tiles(C.byref(g), device, bs, P_target))
    return (g.tx, g.ty, g.tz)


def comm_key() -> bytes:
    """A fresh 128-byte key naming a peer-transport group (comm="ipc" / "local");
    rank 0 draws it and the caller broadcasts it."""
    return os.urandom(128)


def dd_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().dd_nccl_unique_id(buf))
    return buf.raw


class Context:
    """A dd_ctx*. Build with dd_setup(...)."""

    def __init__(self, handle, N, keep, bs=3, nnzb=0):
        self.h = handle
        self.N = N
        self.nnzb = nnzb
        self.bs = bs  # unknowns per row: 3 (BSR3) or 1 (scalar CSR)
        self._keep = keep
        first, nl = C.c_int64(), C.c_int64()
        lib().dd_local_range(self.h, C.byref(first), C.byref(nl))
        self.row_first, self.n_local = first.value, nl.value

    def __del__(self):
        self.destroy()

    def destroy(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.dd_destroy(h)
        self.h = None

    # --- compute
    def apply(self, r, z, variant=DD_LEVELSET, stream=None):
        m = self.bs * self.n_local
        _check(lib().dd_apply_variant(self.h, variant, _dev_vec(r, m, "r", align16=True), _dev_vec(z, m, "z"),
                                      _stream(stream)))

    def spmv(self, x, y, stream=None):
        m = self.bs * self.n_local
        _check(lib().dd_spmv(self.h, _dev_vec(x, m, "x"), _dev_vec(y, m, "y"), _stream(stream)))

    def bicgstab(self, b, x, tol=1e-8, max_iter=1000, hist=False, stream=None):
        m = self.bs * self.n_local
        rep = Report()
        h = np.zeros(2 * max_iter + 1) if hist else None
        st = lib().dd_bicgstab(self.h, _dev_vec(b, m, "b"), _dev_vec(x, m, "x"), tol, max_iter, _ptr(h),
                               C.byref(rep), _stream(stream))
        if st not in (0, 11, 12):
            _check(st)
        out = rep.as_dict()
        out["status_name"] = STATUS[st]
        if hist:
            k = 1 + int(round(2 * out["iterations"])) if st == 0 else None
            out["resid_hist"] = h[:k] if k else h
        return out

    def solve_host(self, b_host: np.ndarray, x_host: np.ndarray, tol=1e-8, max_iter=1000, stream=None):
        n = self.bs * self.N
        rep = Report()
        st = lib().dd_solve_host(self.h, _host_vec(b_host, n, "b_host"), _host_vec(x_host, n, "x_host", True), tol,
                                 max_iter, C.byref(rep), _stream(stream))
        if st not in (0, 11, 12):
            _check(st)
        return rep.as_dict()

    def permute(self, v_orig_host: np.ndarray, v_reord_dev, stream=None):
        v = np.ascontiguousarray(v_orig_host, np.float64)
        _check(lib().dd_permute(self.h, _host_vec(v, self.bs * self.N, "v_orig_host"),
                                _dev_vec(v_reord_dev, self.bs * self.n_local, "v"), _stream(stream)))

    def unpermute(self, v_reord_dev, v_orig_host: np.ndarray, stream=None):
        _check(lib().dd_unpermute(self.h, _dev_vec(v_reord_dev, self.bs * self.n_local, "v"),
                                  _host_vec(v_orig_host, self.bs * self.N, "v_orig_host", True), _stream(stream)))

    def refactor(self, vals, stream=None):
        """New block values (original block order, same pattern): host numpy or
        CUDA float64 tensor."""
        n = 9 * self.nnzb  # dd_refactor reads 9 * nnzb values (BSR3 only)
        if isinstance(vals, np.ndarray):
            vals = np.ascontiguousarray(vals, np.float64)
            _check(lib().dd_refactor(self.h, _host_vec(vals, n, "vals"), 0, _stream(stream)))
        else:
            _check(lib().dd_refactor(self.h, _dev_vec(vals, n, "vals"), 1, _stream(stream)))

    # --- introspection
    def partition(self):
        lab = np.empty(self.N, np.int32)
        n2o = np.empty(self.N, np.int32)
        _check(lib().dd_get_partition(self.h, _ptr(lab), _ptr(n2o)))
        return lab, n2o

    def levels(self, which):
        h = np.empty(self.n_local, np.int32)
        _check(lib().dd_get_levels(self.h, 0 if which in (0, "L") else 1, _ptr(h)))
        return h

    def levels_device(self):
        """Alg. 5 on the device: (hmapL, hmapU, kernel ms)."""
        hl = np.empty(self.n_local, np.int32)
        hu = np.empty(self.n_local, np.int32)
        ms = C.c_double()
        _check(lib().dd_levels_device(self.h, _ptr(hl), _ptr(hu), C.byref(ms)))
        return hl, hu, ms.value

    def factors(self):
        nL, nU = C.c_int64(), C.c_int64()
        _check(lib().dd_get_factors(self.h, C.byref(nL), C.byref(nU), *([None] * 7)))
        n = self.n_local
        b2 = self.bs * self.bs
        Lrp = np.empty(n + 1, np.int64); Lci = np.empty(nL.value, np.int32); Lv = np.empty(b2 * nL.value)
        Urp = np.empty(n + 1, np.int64); Uci = np.empty(nU.value, np.int32); Uv = np.empty(b2 * nU.value)
        D = np.empty(b2 * n)
        _check(lib().dd_get_factors(self.h, None, None, _ptr(Lrp), _ptr(Lci), _ptr(Lv), _ptr(Urp), _ptr(Uci),
                                    _ptr(Uv), _ptr(D)))
        return dict(Lrp=Lrp, Lci=Lci, Lv=Lv, Urp=Urp, Uci=Uci, Uv=Uv, Dinv=D)

    def halo(self):
        ng = C.c_int64()
        _check(lib().dd_get_halo(self.h, C.byref(ng), None, None))
        rows = np.empty(ng.value, np.int64)
        own = np.empty(ng.value, np.int32)
        _check(lib().dd_get_halo(self.h, None, _ptr(rows), _ptr(own)))
        return rows, own

    def send_rows(self, peer):
        n = C.c_int64()
        _check(lib().dd_get_send_rows(self.h, peer, C.byref(n), None))
        rows = np.empty(n.value, np.int32)
        _check(lib().dd_get_send_rows(self.h, peer, None, _ptr(rows)))
        return rows

    STAT_KEYS = ["nnzb_before", "nnzb_after", "n_sub", "n_sub_local", "max_levels_L", "max_levels_U", "max_P",
                 "slab_bytes_levelset", "slab_bytes_spin", "spmv_bytes", "apply_canonical_bytes",
                 "spmv_canonical_bytes", "n_local", "n_ghost", "launches", "swizzle"]
    SETUP_KEYS = ["partition_ms", "reorder_drop_ms", "ilu0_ms", "levels_ms", "pack_ms", "upload_ms"]

    def stats(self):
        s = np.zeros(16, np.int64)
        t = np.zeros(6)
        _check(lib().dd_stats(self.h, _ptr(s), _ptr(t)))
        out = {k: int(s[i]) for i, k in enumerate(self.STAT_KEYS)}
        out.update({k: float(t[i]) for i, k in enumerate(self.SETUP_KEYS)})
        return out

    def profile(self, mode=-1):
        """mode 1: enable+reset, 0: disable, -1: query. Returns the counters."""
        out = np.zeros(8)
        _check(lib().dd_profile(self.h, mode, _ptr(out)))
        return dict(n_apply=int(out[0]), apply_ms=float(out[1]), n_spmv=int(out[2]), spmv_ms=float(out[3]),
                    n_blas=int(out[4]), blas_ms=float(out[5]), launches=int(out[6]))

    def solver_variant(self):
        """(variant dd_bicgstab uses, {variant: apply ms measured at setup})."""
        v = np.zeros(1, np.int32)
        ms = np.zeros(3)
        _check(lib().dd_solver_variant(self.h, _ptr(v), _ptr(ms)))
        return int(v[0]), {DD_LEVELSET: float(ms[0]), DD_SPINLOOP: float(ms[1]), DD_DIRECT: float(ms[2])}

    def launch_info(self, variant=DD_LEVELSET):
        info = np.zeros(4, np.int64)
        _check(lib().dd_launch_info(self.h, variant, _ptr(info)))
        return dict(grid=int(info[0]), threads=int(info[1]), smem=int(info[2]), ring=int(info[3]))


def dd_setup(row_ptr, col_idx, vals, *, grid=None, tiles=None, P=None, variants=DD_LEVELSET, device=0, rank=0,
             world=1, nccl_id: bytes | None = None, pivot_floor=0.0, host_only=False, n_threads=0,
             enable_refactor=False, partitioner="chunks", comm="nccl", csr=False) -> Context:
    """world > 1: comm="nccl" (one process per GPU, nccl_id from dd_nccl_unique_id),
    comm="ipc" (one process per GPU on one node, peer-memory transport through
    CUDA IPC; nccl_id is any 128-byte key the ranks share, e.g. comm_key()) or
    comm="local" (ranks are contexts of this process, each created and driven
    from its own thread; nccl_id is any 128-byte key the ranks share).
    csr=True: a scalar CSR matrix (vals[nnz]) through dd_setup_csr."""
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col_idx = np.ascontiguousarray(col_idx, np.int32)
    vals = np.ascontiguousarray(vals, np.float64)
    n = row_ptr.shape[0] - 1
    b2 = 1 if csr else 9
    if n < 0 or col_idx.shape[0] != row_ptr[-1] or vals.shape[0] != b2 * col_idx.shape[0]:
        raise ValueError(f"dd_setup: inconsistent arrays (row_ptr[-1] = {row_ptr[-1] if n >= 0 else None}, "
                         f"col_idx {col_idx.shape[0]}, vals {vals.shape[0]}, expected {b2} values per block)")
    A = BSR3(n, col_idx.shape[0], _ptr(row_ptr), _ptr(col_idx), _ptr(vals))
    o = Opts()
    g = None
    if isinstance(tiles, str) and tiles == "auto":
        # dd_setup chooses the tiles (wave fill x coupling weight the drop removes, R41)
        tiles = (0, 0, 0)
    if tiles is not None:
        g = Grid(*grid, *tiles)
        o.grid = C.addressof(g)
    o.subdomain_rows = int(P or 0)
    o.variants = variants
    o.device, o.rank, o.world = device, rank, world
    idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
    o.nccl_unique_id = C.addressof(idbuf) if idbuf is not None else None
    o.pivot_floor = pivot_floor
    o.host_only = int(bool(host_only))
    o.n_threads = n_threads
    o.enable_refactor = int(bool(enable_refactor))
    o.partitioner = {"chunks": DD_PART_CHUNKS, "bfs": DD_PART_BFS}[partitioner]
    o.comm = {"nccl": DD_COMM_NCCL, "local": DD_COMM_LOCAL, "ipc": DD_COMM_IPC}[comm]
    h = C.c_void_p()
    _check((lib().dd_setup_csr if csr else lib().dd_setup)(C.byref(A), C.byref(o), C.byref(h)))
    ctx = Context(h, n, keep=(g, idbuf), bs=1 if csr else 3, nnzb=int(col_idx.shape[0]))
    gq = Grid()
    _check(lib().dd_get_grid(h, C.byref(gq)))
    ctx.tiles = (gq.tx, gq.ty, gq.tz) if tiles is not None else None
    return ctx


def dd_setup_csr(row_ptr, col_idx, vals, **kw) -> Context:
    """Scalar CSR path; same options as dd_setup."""
    return dd_setup(row_ptr, col_idx, vals, csr=True, **kw)


# C-ABI-named thin wrappers
def dd_destroy(ctx: Context):
    ctx.destroy()


def dd_apply(ctx, r, z, stream=None):
    ctx.apply(r, z, DD_LEVELSET, stream)


def dd_apply_variant(ctx, variant, r, z, stream=None):
    ctx.apply(r, z, variant, stream)


def dd_spmv(ctx, x, y, stream=None):
    ctx.spmv(x, y, stream)


def dd_bicgstab(ctx, b, x, tol=1e-8, max_iter=1000, hist=False, stream=None):
    return ctx.bicgstab(b, x, tol, max_iter, hist, stream)


def dd_solve_host(ctx, b_host, x_host, tol=1e-8, max_iter=1000, stream=None):
    return ctx.solve_host(b_host, x_host, tol, max_iter, stream)


def dd_permute(ctx, v_orig_host, v_reord_dev, stream=None):
    ctx.permute(v_orig_host, v_reord_dev, stream)


def dd_unpermute(ctx, v_reord_dev, v_orig_host, stream=None):
    ctx.unpermute(v_reord_dev, v_orig_host, stream)


def dd_local_range(ctx):
    return ctx.row_first, ctx.n_local


def dd_get_partition(ctx):
    return ctx.partition()


def dd_levels_device(ctx):
    return ctx.levels_device()


def dd_get_levels(ctx, which):
    return ctx.levels(which)


def dd_get_factors(ctx):
    return ctx.factors()


def dd_get_halo(ctx):
    return ctx.halo()


def dd_get_send_rows(ctx, peer):
    return ctx.send_rows(peer)


def dd_stats(ctx):
    return ctx.stats()


def dd_refactor(ctx, vals, stream=None):
    ctx.refactor(vals, stream)


def dd_profile(ctx, mode=-1):
    return ctx.profile(mode)


def dd_solver_variant(ctx):
    return ctx.solver_variant()


def dd_launch_info(ctx, variant=DD_LEVELSET):
    return ctx.launch_info(variant)
