"""ctypes wrapper around the CPU oracle (liboracle.so, built from dd_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package. The product
(paper_2508_04917_b200) never imports it and shares no code with it.

Every function mirrors one of dd_oracle.h; ``setup`` chains the paper's setup
steps (Alg. 2 -> permutation -> Alg. 3 -> drop -> Alg. 7 ILU0/ILDU0 -> Alg. 5
levels) exactly as the paper orders them.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "dd_oracle.c")

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
          "-fPIC", "-shared", "-Wall", "-Wno-unused-result"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "dd_oracle.h"))):
        cmd = ["gcc", *CFLAGS, "-o", _SO, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        i32, i64, dbl = C.c_int32, C.c_int64, C.c_double
        P = C.c_void_p
        sig = {
            "orc_set_threads": (None, [C.c_int]),
            "orc_get_threads": (C.c_int, []),
            "orc_labels_geometric": (C.c_int, [i32] * 6 + [P]),
            "orc_labels_chunks": (None, [i64, i32, P]),
            "orc_labels_bfs": (None, [i64, P, P, i32, P]),
            "orc_permutation": (None, [i64, P, P, P]),
            "orc_subdomain_ptr": (None, [i64, P, i32, P]),
            "orc_reorder": (None, [i64, P, P, P, P, P, P, P, P]),
            "orc_drop": (i64, [i64, P, P, P, P, P, P, P]),
            "orc_ilu0": (C.c_int, [i64, P, P, P, dbl, P, P, P]),
            "orc_ildu0": (None, [i64, P, P, P, P, P]),
            "orc_levels_lower": (None, [i64, P, P, P]),
            "orc_levels_upper": (None, [i64, P, P, P]),
            "orc_apply": (None, [i64, i32, P, P, P, P, P, P, P, P]),
            "orc_lower": (None, [i64, i32, P, P, P, P, P, P]),
            "orc_apply_ilu0": (None, [i64, i32, P, P, P, P, P, P, P]),
            "orc_spmv": (None, [i64, P, P, P, P, P]),
            "orc_dot": (dbl, [i64, P, P]),
            "orc_bicgstab": (C.c_int, [i64, P, P, P, i32, P, P, P, P, P, P, P, P, dbl, i32,
                                       P, P]),
            "orc_s_reorder": (None, [i64, P, P, P, P, P, P, P, P]),
            "orc_s_drop": (i64, [i64, P, P, P, P, P, P, P]),
            "orc_s_ilu0": (C.c_int, [i64, P, P, P, dbl, P, P, P]),
            "orc_s_ildu0": (None, [i64, P, P, P, P, P]),
            "orc_s_apply": (None, [i64, i32, P, P, P, P, P, P, P, P]),
            "orc_s_spmv": (None, [i64, P, P, P, P, P]),
            "orc_s_bicgstab": (C.c_int, [i64, P, P, P, i32, P, P, P, P, P, P, P, P, dbl, i32,
                                         P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def labels_geometric(grid, tiles):
    nx, ny, nz = grid
    tx, ty, tz = tiles
    out = np.empty(nx * ny * nz, dtype=np.int32)
    rc = lib().orc_labels_geometric(nx, ny, nz, tx, ty, tz, _p(out))
    if rc != 0:
        raise ValueError("grid not divisible by tile dims")
    return out


def labels_chunks(n, P):
    out = np.empty(n, dtype=np.int32)
    lib().orc_labels_chunks(n, P, _p(out))
    return out


def labels_bfs(rp, ci, P):
    rp, ci = _c(rp, np.int64), _c(ci, np.int32)
    out = np.empty(rp.shape[0] - 1, dtype=np.int32)
    lib().orc_labels_bfs(rp.shape[0] - 1, _p(rp), _p(ci), P, _p(out))
    return out


def permutation(labels):
    labels = _c(labels, np.int32)
    n = labels.shape[0]
    n2o = np.empty(n, dtype=np.int32)
    o2n = np.empty(n, dtype=np.int32)
    lib().orc_permutation(n, _p(labels), _p(n2o), _p(o2n))
    return n2o, o2n


def subdomain_ptr(labels_new_or_old, n_sub):
    labels = _c(labels_new_or_old, np.int32)
    sp = np.empty(n_sub + 1, dtype=np.int64)
    lib().orc_subdomain_ptr(labels.shape[0], _p(labels), n_sub, _p(sp))
    return sp


def reorder(rp, ci, v, n2o, o2n):
    rp, ci, v = _c(rp, np.int64), _c(ci, np.int32), _c(v, np.float64)
    n2o, o2n = _c(n2o, np.int32), _c(o2n, np.int32)
    n = rp.shape[0] - 1
    rpo = np.empty_like(rp)
    cio = np.empty_like(ci)
    vo = np.empty_like(v)
    lib().orc_reorder(n, _p(rp), _p(ci), _p(v), _p(n2o), _p(o2n), _p(rpo), _p(cio), _p(vo))
    return rpo, cio, vo


def drop(rp, ci, v, label_new):
    rp, ci, v = _c(rp, np.int64), _c(ci, np.int32), _c(v, np.float64)
    label_new = _c(label_new, np.int32)
    n = rp.shape[0] - 1
    L = lib()
    kept = L.orc_drop(n, _p(rp), _p(ci), _p(v), _p(label_new), None, None, None)
    rpo = np.empty(n + 1, dtype=np.int64)
    cio = np.empty(kept, dtype=np.int32)
    vo = np.empty(9 * kept, dtype=np.float64)
    L.orc_drop(n, _p(rp), _p(ci), _p(v), _p(label_new), _p(rpo), _p(cio), _p(vo))
    return rpo, cio, vo


class OracleError(RuntimeError):
    def __init__(self, code, row):
        self.code, self.row = code, row
        super().__init__({1: "missing diagonal block", 2: "singular pivot block"}.get(code, "?")
                         + f" at row {row}")


def ilu0(rp, ci, a, pivot_floor=1e-300):
    rp, ci, a = _c(rp, np.int64), _c(ci, np.int32), _c(a, np.float64)
    n = rp.shape[0] - 1
    lu = np.empty_like(a)
    dinv = np.empty(9 * n, dtype=np.float64)
    bad = np.zeros(1, dtype=np.int64)
    rc = lib().orc_ilu0(n, _p(rp), _p(ci), _p(a), pivot_floor, _p(lu), _p(dinv), _p(bad))
    if rc != 0:
        raise OracleError(rc, int(bad[0]))
    return lu, dinv


def ildu0(rp, ci, lu, dinv):
    rp, ci = _c(rp, np.int64), _c(ci, np.int32)
    n = rp.shape[0] - 1
    uunit = np.zeros_like(lu)
    lib().orc_ildu0(n, _p(rp), _p(ci), _p(lu), _p(dinv), _p(uunit))
    return uunit


def levels_lower(rp, ci):
    rp, ci = _c(rp, np.int64), _c(ci, np.int32)
    h = np.empty(rp.shape[0] - 1, dtype=np.int32)
    lib().orc_levels_lower(h.shape[0], _p(rp), _p(ci), _p(h))
    return h


def levels_upper(rp, ci):
    rp, ci = _c(rp, np.int64), _c(ci, np.int32)
    h = np.empty(rp.shape[0] - 1, dtype=np.int32)
    lib().orc_levels_upper(h.shape[0], _p(rp), _p(ci), _p(h))
    return h


def apply(S, r):
    r = _c(r, np.float64)
    z = np.empty_like(r)
    f = lib().orc_s_apply if S.get("bs", 3) == 1 else lib().orc_apply
    f(S["n"], S["n_sub"], _p(S["sub_ptr"]), _p(S["rp_d"]), _p(S["ci_d"]),
      _p(S["lu"]), _p(S["dinv"]), _p(S["uunit"]), _p(r), _p(z))
    return z


def lower(S, r):
    """z = L^-1 r per subdomain (unit L): the Table 3 lower solve (BSR3)."""
    r = _c(r, np.float64)
    z = np.empty_like(r)
    lib().orc_lower(S["n"], S["n_sub"], _p(S["sub_ptr"]), _p(S["rp_d"]), _p(S["ci_d"]), _p(S["lu"]), _p(r), _p(z))
    return z


def apply_ilu0(S, r):
    """ILU0 apply with the non-unit upper factor (scaling after each row's
    off-diagonal updates), BSR3."""
    r = _c(r, np.float64)
    z = np.empty_like(r)
    lib().orc_apply_ilu0(S["n"], S["n_sub"], _p(S["sub_ptr"]), _p(S["rp_d"]), _p(S["ci_d"]), _p(S["lu"]),
                         _p(S["dinv"]), _p(r), _p(z))
    return z


def spmv(rp, ci, v, x):
    x = _c(x, np.float64)
    y = np.empty_like(x)
    lib().orc_spmv(rp.shape[0] - 1, _p(rp), _p(ci), _p(v), _p(x), _p(y))
    return y


def dot(x, y):
    x, y = _c(x, np.float64), _c(y, np.float64)
    return float(lib().orc_dot(x.shape[0], _p(x), _p(y)))


def setup(rp, ci, v, *, grid=None, tiles=None, P=None, partitioner="chunks", pivot_floor=1e-300):
    """The paper's setup pipeline, in the paper's order. Returns a dict.
    Labels: geometric cuts (tiles given), else contiguous chunks or BFS graph
    growing ("bfs") of P rows."""
    n = rp.shape[0] - 1
    if tiles is not None:
        labels = labels_geometric(grid, tiles)
    elif partitioner == "bfs":
        labels = labels_bfs(rp, ci, P)
    else:
        labels = labels_chunks(n, P)
    n_sub = int(labels.max()) + 1 if n else 0
    n2o, o2n = permutation(labels)
    rp_r, ci_r, v_r = reorder(rp, ci, v, n2o, o2n)
    label_new = labels[n2o]
    rp_d, ci_d, v_d = drop(rp_r, ci_r, v_r, label_new)
    lu, dinv = ilu0(rp_d, ci_d, v_d, pivot_floor)
    uunit = ildu0(rp_d, ci_d, lu, dinv)
    return dict(n=n, n_sub=n_sub, labels=labels, new_to_old=n2o, old_to_new=o2n,
                sub_ptr=subdomain_ptr(label_new, n_sub), label_new=label_new,
                rp_r=rp_r, ci_r=ci_r, v_r=v_r, rp_d=rp_d, ci_d=ci_d, v_d=v_d,
                lu=lu, dinv=dinv, uunit=uunit,
                hmapL=levels_lower(rp_d, ci_d), hmapU=levels_upper(rp_d, ci_d))


def bicgstab(S, b, x0=None, tol=1e-8, max_iter=1000, hist=True):
    """Returns (x, report dict)."""
    n = S["n"]
    bs = S.get("bs", 3)
    b = _c(b, np.float64)
    x = np.zeros(bs * n) if x0 is None else _c(x0, np.float64).copy()
    rh = np.zeros(2 * max_iter + 1) if hist else None
    out = np.zeros(8)
    f = lib().orc_s_bicgstab if bs == 1 else lib().orc_bicgstab
    f(n, _p(S["rp_r"]), _p(S["ci_r"]), _p(S["v_r"]), S["n_sub"],
                       _p(S["sub_ptr"]), _p(S["rp_d"]), _p(S["ci_d"]), _p(S["lu"]),
                       _p(S["dinv"]), _p(S["uunit"]), _p(b), _p(x), tol, max_iter,
                       _p(rh), _p(out))
    rep = dict(iterations=float(out[0]), n_applies=int(out[1]), rel_resid=float(out[2]),
               true_rel_resid=float(out[3]), status=int(out[4]))
    if hist:
        rep["resid_hist"] = rh[: int(out[5])]
    return x, rep


# ------------------------------------------------- scalar CSR path (8(f3))
def s_reorder(rp, ci, v, n2o, o2n):
    rp, ci, v = _c(rp, np.int64), _c(ci, np.int32), _c(v, np.float64)
    n2o, o2n = _c(n2o, np.int32), _c(o2n, np.int32)
    rpo, cio, vo = np.empty_like(rp), np.empty_like(ci), np.empty_like(v)
    lib().orc_s_reorder(rp.shape[0] - 1, _p(rp), _p(ci), _p(v), _p(n2o), _p(o2n), _p(rpo), _p(cio), _p(vo))
    return rpo, cio, vo


def s_drop(rp, ci, v, label_new):
    rp, ci, v = _c(rp, np.int64), _c(ci, np.int32), _c(v, np.float64)
    label_new = _c(label_new, np.int32)
    n = rp.shape[0] - 1
    L = lib()
    kept = L.orc_s_drop(n, _p(rp), _p(ci), _p(v), _p(label_new), None, None, None)
    rpo, cio, vo = np.empty(n + 1, np.int64), np.empty(kept, np.int32), np.empty(kept, np.float64)
    L.orc_s_drop(n, _p(rp), _p(ci), _p(v), _p(label_new), _p(rpo), _p(cio), _p(vo))
    return rpo, cio, vo


def s_ilu0(rp, ci, a, pivot_floor=1e-300):
    rp, ci, a = _c(rp, np.int64), _c(ci, np.int32), _c(a, np.float64)
    n = rp.shape[0] - 1
    lu, dinv, bad = np.empty_like(a), np.empty(n, np.float64), np.zeros(1, np.int64)
    rc = lib().orc_s_ilu0(n, _p(rp), _p(ci), _p(a), pivot_floor, _p(lu), _p(dinv), _p(bad))
    if rc != 0:
        raise OracleError(rc, int(bad[0]))
    return lu, dinv


def s_ildu0(rp, ci, lu, dinv):
    rp, ci = _c(rp, np.int64), _c(ci, np.int32)
    uunit = np.zeros_like(lu)
    lib().orc_s_ildu0(rp.shape[0] - 1, _p(rp), _p(ci), _p(lu), _p(dinv), _p(uunit))
    return uunit


def s_spmv(rp, ci, v, x):
    x = _c(x, np.float64)
    y = np.empty_like(x)
    lib().orc_s_spmv(rp.shape[0] - 1, _p(rp), _p(ci), _p(v), _p(x), _p(y))
    return y


def setup_csr(rp, ci, v, *, grid=None, tiles=None, P=None, partitioner="chunks", pivot_floor=1e-300):
    """The paper's setup pipeline for a SCALAR CSR matrix (vals[nnz]), in the
    paper's order; the same dict as setup() with bs = 1."""
    n = rp.shape[0] - 1
    if tiles is not None:
        labels = labels_geometric(grid, tiles)
    elif partitioner == "bfs":
        labels = labels_bfs(rp, ci, P)
    else:
        labels = labels_chunks(n, P)
    n_sub = int(labels.max()) + 1 if n else 0
    n2o, o2n = permutation(labels)
    rp_r, ci_r, v_r = s_reorder(rp, ci, v, n2o, o2n)
    label_new = labels[n2o]
    rp_d, ci_d, v_d = s_drop(rp_r, ci_r, v_r, label_new)
    lu, dinv = s_ilu0(rp_d, ci_d, v_d, pivot_floor)
    uunit = s_ildu0(rp_d, ci_d, lu, dinv)
    return dict(bs=1, n=n, n_sub=n_sub, labels=labels, new_to_old=n2o, old_to_new=o2n,
                sub_ptr=subdomain_ptr(label_new, n_sub), label_new=label_new,
                rp_r=rp_r, ci_r=ci_r, v_r=v_r, rp_d=rp_d, ci_d=ci_d, v_d=v_d,
                lu=lu, dinv=dinv, uunit=uunit,
                hmapL=levels_lower(rp_d, ci_d), hmapU=levels_upper(rp_d, ci_d))
