"""Test helpers: assembling oracle outputs into scipy/numpy objects so the pins
can use library routines (sparse matmul, dense solve, dense LU checks)."""
from __future__ import annotations

import json
import os

import numpy as np
import scipy.sparse as sp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def bsr(rp, ci, v, n=None):
    n = rp.shape[0] - 1 if n is None else n
    return sp.bsr_matrix((np.asarray(v).reshape(-1, 3, 3), np.asarray(ci), np.asarray(rp)),
                         shape=(3 * n, 3 * n))


def split_factors(rp, ci, lu, uunit=None):
    """Assemble unit-L, U (incl. diagonal), and (optionally) strictly-upper
    Uunit and block-diag(U_ii) from the oracle's in-pattern arrays."""
    n = rp.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    blocks = lu.reshape(-1, 3, 3)
    lo = ci < rows
    up = ci >= rows
    dg = ci == rows

    def mk(mask, vals):
        m = sp.coo_matrix((np.zeros(0), (np.zeros(0, int), np.zeros(0, int))), shape=(3 * n, 3 * n))
        r = rows[mask]
        c = ci[mask]
        b = vals[mask]
        rr = (3 * r)[:, None, None] + np.arange(3)[None, :, None] + 0 * np.arange(3)[None, None, :]
        cc = (3 * c)[:, None, None] + 0 * np.arange(3)[None, :, None] + np.arange(3)[None, None, :]
        m = sp.csr_matrix((b.ravel(), (rr.ravel(), cc.ravel())), shape=(3 * n, 3 * n))
        return m

    L = mk(lo, blocks) + sp.identity(3 * n, format="csr")
    U = mk(up, blocks)
    D = mk(dg, blocks)
    out = dict(L=L, U=U, D=D)
    if uunit is not None:
        out["Uunit"] = mk(ci > rows, uunit.reshape(-1, 3, 3)) + sp.identity(3 * n, format="csr")
    return out


def dense_pattern_matrix(n, seed, dominance=2.0):
    """Full dense block pattern (every block present), random, dominant."""
    rng = np.random.default_rng(seed)
    rp = np.arange(0, n * n + 1, n, dtype=np.int64)
    ci = np.tile(np.arange(n, dtype=np.int32), n)
    A = rng.uniform(-1, 1, (3 * n, 3 * n))
    A[np.diag_indices(3 * n)] = np.abs(A).sum(axis=1) + dominance
    blocks = A.reshape(n, 3, n, 3).transpose(0, 2, 1, 3).reshape(-1, 9)
    return rp, ci, blocks.ravel(), A


def kron_blocks(S):
    """Scalar dense matrix S (n x n) -> BSR3 arrays with blocks S_ij * I3 for S_ij != 0."""
    S = np.asarray(S, dtype=float)
    n = S.shape[0]
    rp = [0]
    ci = []
    vals = []
    for i in range(n):
        for j in range(n):
            if S[i, j] != 0:
                ci.append(j)
                vals.append((S[i, j] * np.eye(3)).ravel())
        rp.append(len(ci))
    return (np.array(rp, dtype=np.int64), np.array(ci, dtype=np.int32),
            np.concatenate(vals) if vals else np.zeros(0))


def alg5_marking(n, deps_of):
    """Independent sequential rendering of PAPER Alg. 5 on one
    subdomain: hmap initialised to n+1; rows without deps get level 0; then the
    marked/added/level fixpoint loop. deps_of[i] = list of j < i (lower)."""
    hmap = [n + 1] * n
    marked = [0] * n
    for i in range(n):
        if len(deps_of[i]) == 0:
            hmap[i] = 0
    level = 0
    while True:
        added = 0
        for i in range(n):
            if hmap[i] > level:
                valid = True
                for j in deps_of[i]:
                    if hmap[j] > level:
                        valid = False
                        break
                if valid:
                    marked[i] = 1
                    added |= 1
        for i in range(n):
            if marked[i]:
                hmap[i] = level + 1
                marked[i] = 0
        if added == 0:
            break
        level += 1
    return np.array(hmap, dtype=np.int32)
