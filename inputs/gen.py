"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and bench.py.

This module holds NONE of the method's arithmetic (no partitioning, reordering,
factorisation, triangular solve or Krylov step). It only builds the inputs the
paper's workloads are made of:

* ``laplacian_bsr3`` -- the 7-point 3-D Laplacian in 3x3 BSR, natural order
  ``gidx = i + nx*(j + ny*k)`` (Alg. 2 index formula; inputs
  table). Diagonal block 6*I3, neighbour blocks -1*I3 (DESIGN.md
  readings R1/R2).
* ``spe10_style_bsr3`` -- a heterogeneous-permeability reservoir-like BSR3
  matrix on the SPE10 model-2 grid 60x220x85; the
  recipe is DESIGN.md's input recipe (no SPE10 data is available).
* ``random_block_chain`` / ``random_block_grid`` -- small random full-3x3-block
  matrices for the oracle pins.
* ``manufactured_rhs`` / ``apply_input`` -- seeded vectors (reading R23).

All BSR matrices are returned as ``(row_ptr int64[N+1], col_idx int32[nnzb],
vals float64[nnzb*9])`` with each 3x3 block row-major and columns ascending in
every row.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "laplacian_bsr3",
    "spe10_style_bsr3",
    "random_block_grid",
    "random_block_chain",
    "manufactured_rhs",
    "apply_input",
    "bsr_to_scipy",
    "grid_stencil_pattern",
    "laplacian_csr",
    "spe10_style_csr",
    "random_csr_grid",
    "csr_to_scipy",
    "manufactured_rhs_csr",
    "stencil27_pattern",
    "random_block_stencil27",
    "random_csr_stencil27",
]


def grid_stencil_pattern(nx: int, ny: int, nz: int):
    """7-point pattern on an nx*ny*nz grid in natural order.

    Returns (row_ptr, col_idx, slot) where ``slot`` in 0..6 names the stencil
    direction of every stored block in ascending column order:
    0:-z 1:-y 2:-x 3:self 4:+x 5:+y 6:+z.
    """
    n = nx * ny * nz
    g = np.arange(n, dtype=np.int64)
    i = g % nx
    j = (g // nx) % ny
    k = g // (nx * ny)
    offs = (-nx * ny, -nx, -1, 0, 1, nx, nx * ny)
    valid = (k > 0, j > 0, i > 0, np.ones(n, dtype=bool), i < nx - 1, j < ny - 1, k < nz - 1)
    mask = np.stack(valid, axis=1)  # (n, 7), slots already in ascending column order
    counts = mask.sum(axis=1)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    cols = np.empty((n, 7), dtype=np.int64)
    for s, o in enumerate(offs):
        cols[:, s] = g + o
    col_idx = cols[mask].astype(np.int32)
    slot = np.broadcast_to(np.arange(7, dtype=np.int8), (n, 7))[mask]
    return row_ptr, col_idx, slot


def laplacian_bsr3(nx: int, ny: int, nz: int):
    """7-point Laplacian, blocks e*I3 with e = 6 on the diagonal, -1 off it."""
    row_ptr, col_idx, slot = grid_stencil_pattern(nx, ny, nz)
    nnzb = col_idx.shape[0]
    e = np.where(slot == 3, 6.0, -1.0)
    vals = np.zeros((nnzb, 9), dtype=np.float64)
    vals[:, 0] = e
    vals[:, 4] = e
    vals[:, 8] = e
    return row_ptr, col_idx, vals.reshape(-1)


def _box_smooth_xy(f: np.ndarray) -> np.ndarray:
    """3x3 box average in (x, y) of a field shaped (nz, ny, nx), edge-replicated."""
    p = np.pad(f, ((0, 0), (1, 1), (1, 1)), mode="edge")
    out = np.zeros_like(f)
    for dy in range(3):
        for dx in range(3):
            out += p[:, dy:dy + f.shape[1], dx:dx + f.shape[2]]
    return out / 9.0


def _renorm(f: np.ndarray) -> np.ndarray:
    return (f - f.mean()) / f.std()


def spe10_style_bsr3(nx: int = 60, ny: int = 220, nz: int = 85, *, seed: int = 10,
                     dx: float = 20.0, dy: float = 10.0, dz: float = 2.0,
                     upper_ness_from: int = 35):
    """SPE10-style heterogeneous reservoir BSR3 matrix (DESIGN.md input recipe).

    Seeds: ``seed`` (xi fields), ``seed+1`` (channel geometry), ``seed+2``
    (per-face 3-phase mobilities lambda), ``seed+3`` (diagonal perturbation R).
    Returns (row_ptr, col_idx, vals, log10_kx) with log10_kx shaped (nz, ny, nx).
    """
    rng_xi = np.random.default_rng(seed)
    rng_ch = np.random.default_rng(seed + 1)
    rng_lam = np.random.default_rng(seed + 2)
    rng_r = np.random.default_rng(seed + 3)

    xi = rng_xi.standard_normal((nz, ny, nx))
    xi = _renorm(_box_smooth_xy(_box_smooth_xy(xi)))
    logk = np.empty((nz, ny, nx))
    top = slice(0, min(upper_ness_from, nz))
    logk[top] = 1.0 + 1.0 * xi[top]
    if nz > upper_ness_from:
        low = slice(upper_ness_from, nz)
        logk[low] = -1.0 + 0.5 * xi[low]
        xg = np.arange(nx)[None, :]
        yg = np.arange(ny)[:, None]
        for kk in range(upper_ness_from, nz):
            for _ in range(4):
                x0 = rng_ch.uniform(0.1 * nx, 0.9 * nx)
                amp = rng_ch.uniform(0.05 * nx, 0.15 * nx)
                wl = rng_ch.uniform(0.2 * ny, 0.6 * ny)
                ph = rng_ch.uniform(0.0, 2.0 * np.pi)
                xc = x0 + amp * np.sin(2.0 * np.pi * yg / wl + ph)
                chan = np.abs(xg - xc) <= 1.5  # width 3 cells
                logk[kk][chan] = 3.0 + 0.3 * xi[kk][chan]
    np.clip(logk, -3.0, 4.3, out=logk)
    kx = 10.0 ** logk
    kz = 0.1 * kx

    def harm(a, b):
        return 2.0 * a * b / (a + b)

    # transmissibilities of the faces between (cell, +direction neighbour)
    tx = (dy * dz / dx) * harm(kx[:, :, :-1], kx[:, :, 1:])   # (nz, ny, nx-1)
    ty = (dx * dz / dy) * harm(kx[:, :-1, :], kx[:, 1:, :])   # (nz, ny-1, nx)
    tz = (dx * dy / dz) * harm(kz[:-1, :, :], kz[1:, :, :])   # (nz-1, ny, nx)
    lam_x = rng_lam.uniform(0.5, 1.5, tx.shape + (3,))
    lam_y = rng_lam.uniform(0.5, 1.5, ty.shape + (3,))
    lam_z = rng_lam.uniform(0.5, 1.5, tz.shape + (3,))
    c = 1e-3 * np.mean(np.concatenate([tx.ravel(), ty.ravel(), tz.ravel()]))

    n = nx * ny * nz
    # per-cell, per-direction coupling diag(T*lambda) (3 entries), zero if absent
    coup = np.zeros((nz, ny, nx, 7, 3))
    # slot order: 0:-z 1:-y 2:-x 3:self 4:+x 5:+y 6:+z
    coup[:, :, :-1, 4] = (tx[..., None] * lam_x)
    coup[:, :, 1:, 2] = (tx[..., None] * lam_x)
    coup[:, :-1, :, 5] = (ty[..., None] * lam_y)
    coup[:, 1:, :, 1] = (ty[..., None] * lam_y)
    coup[:-1, :, :, 6] = (tz[..., None] * lam_z)
    coup[1:, :, :, 0] = (tz[..., None] * lam_z)
    coup = coup.reshape(n, 7, 3)
    R = rng_r.uniform(-1.0, 1.0, (n, 3, 3))

    row_ptr, col_idx, slot = grid_stencil_pattern(nx, ny, nz)
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    vals = np.zeros((col_idx.shape[0], 3, 3))
    off = slot != 3
    d3 = np.arange(3)
    cv = coup[rows[off], slot[off].astype(np.int64)]  # (nnz_off, 3)
    blk = np.zeros((cv.shape[0], 3, 3))
    blk[:, d3, d3] = -cv
    vals[off] = blk
    diag_pos = np.nonzero(~off)[0]
    dsum = coup.sum(axis=1)  # (n, 3)
    dblk = c * (np.eye(3)[None] + 0.25 * R)
    dblk[:, d3, d3] += dsum
    vals[diag_pos] = dblk
    return row_ptr, col_idx, vals.reshape(-1), logk


# ------------------------------------------------------- scalar CSR inputs
# (the paper's CSR half; rhd is a scalar 128^3 7-point matrix
# and spe10 a scalar 7-point matrix on the 60x220x85 grid, Appendix A)

def laplacian_csr(nx: int, ny: int, nz: int):
    """Scalar 7-point Laplacian: 6 on the diagonal, -1 off it."""
    row_ptr, col_idx, slot = grid_stencil_pattern(nx, ny, nz)
    vals = np.where(slot == 3, 6.0, -1.0).astype(np.float64)
    return row_ptr, col_idx, vals


def spe10_style_csr(nx: int = 60, ny: int = 220, nz: int = 85, *, seed: int = 10,
                    dx: float = 20.0, dy: float = 10.0, dz: float = 2.0, upper_ness_from: int = 35):
    """Scalar SPE10-style two-point-flux pressure matrix on the same
    permeability field as spe10_style_bsr3 (seed, seed+1): off-diagonal
    -T_face, diagonal sum(T_face) + c, c = 1e-3 * mean(T). Returns
    (row_ptr, col_idx, vals, log10_kx)."""
    rng_xi = np.random.default_rng(seed)
    rng_ch = np.random.default_rng(seed + 1)
    xi = rng_xi.standard_normal((nz, ny, nx))
    xi = _renorm(_box_smooth_xy(_box_smooth_xy(xi)))
    logk = np.empty((nz, ny, nx))
    top = slice(0, min(upper_ness_from, nz))
    logk[top] = 1.0 + 1.0 * xi[top]
    if nz > upper_ness_from:
        low = slice(upper_ness_from, nz)
        logk[low] = -1.0 + 0.5 * xi[low]
        xg = np.arange(nx)[None, :]
        yg = np.arange(ny)[:, None]
        for kk in range(upper_ness_from, nz):
            for _ in range(4):
                x0 = rng_ch.uniform(0.1 * nx, 0.9 * nx)
                amp = rng_ch.uniform(0.05 * nx, 0.15 * nx)
                wl = rng_ch.uniform(0.2 * ny, 0.6 * ny)
                ph = rng_ch.uniform(0.0, 2.0 * np.pi)
                xc = x0 + amp * np.sin(2.0 * np.pi * yg / wl + ph)
                logk[kk][np.abs(xg - xc) <= 1.5] = 3.0 + 0.3 * xi[kk][np.abs(xg - xc) <= 1.5]
    np.clip(logk, -3.0, 4.3, out=logk)
    kx = 10.0 ** logk
    kz = 0.1 * kx

    def harm(a, b):
        return 2.0 * a * b / (a + b)

    tx = (dy * dz / dx) * harm(kx[:, :, :-1], kx[:, :, 1:])
    ty = (dx * dz / dy) * harm(kx[:, :-1, :], kx[:, 1:, :])
    tz = (dx * dy / dz) * harm(kz[:-1, :, :], kz[1:, :, :])
    c = 1e-3 * np.mean(np.concatenate([tx.ravel(), ty.ravel(), tz.ravel()]))
    n = nx * ny * nz
    coup = np.zeros((nz, ny, nx, 7))
    coup[:, :, :-1, 4] = tx
    coup[:, :, 1:, 2] = tx
    coup[:, :-1, :, 5] = ty
    coup[:, 1:, :, 1] = ty
    coup[:-1, :, :, 6] = tz
    coup[1:, :, :, 0] = tz
    coup = coup.reshape(n, 7)
    row_ptr, col_idx, slot = grid_stencil_pattern(nx, ny, nz)
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    vals = -coup[rows, slot.astype(np.int64)]
    diag = slot == 3
    vals[diag] = coup.sum(axis=1)[rows[diag]] + c
    return row_ptr, col_idx, vals, logk


def random_csr_grid(nx: int, ny: int, nz: int, seed: int, dominance: float = 1.0):
    """7-point grid pattern, random off-diagonals in [-1, 1), row-diagonally
    dominant diagonal (sum |off| + dominance) with a random sign."""
    rng = np.random.default_rng(seed)
    row_ptr, col_idx, slot = grid_stencil_pattern(nx, ny, nz)
    n = nx * ny * nz
    vals = rng.uniform(-1.0, 1.0, col_idx.shape[0])
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    off = slot != 3
    absrow = np.zeros(n)
    np.add.at(absrow, rows[off], np.abs(vals[off]))
    dpos = np.nonzero(~off)[0]
    sign = np.where(rng.uniform(size=n) < 0.5, -1.0, 1.0)
    vals[dpos] = sign * (absrow + dominance)
    return row_ptr, col_idx, vals


def csr_to_scipy(row_ptr, col_idx, vals):
    import scipy.sparse as sp
    n = row_ptr.shape[0] - 1
    return sp.csr_matrix((vals, col_idx, row_ptr), shape=(n, n))


def manufactured_rhs_csr(row_ptr, col_idx, vals, seed: int = 1):
    """x* ~ U[0,1)^N from default_rng(seed); b = A x* via scipy (library)."""
    n = row_ptr.shape[0] - 1
    xs = np.random.default_rng(seed).random(n)
    return xs, csr_to_scipy(row_ptr, col_idx, vals) @ xs


def random_block_grid(nx: int, ny: int, nz: int, seed: int, dominance: float = 1.0):
    """7-point grid pattern with random full 3x3 blocks, block-row diagonally
    dominant (diagonal block = random + (sum of |off-diag| row sums + dominance) I)."""
    rng = np.random.default_rng(seed)
    row_ptr, col_idx, slot = grid_stencil_pattern(nx, ny, nz)
    nnzb = col_idx.shape[0]
    vals = rng.uniform(-1.0, 1.0, (nnzb, 3, 3))
    n = nx * ny * nz
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    absrow = np.zeros((n, 3))
    off = slot != 3
    np.add.at(absrow, rows[off], np.abs(vals[off]).sum(axis=2))
    dpos = np.nonzero(~off)[0]
    d = vals[dpos]
    d3 = np.arange(3)
    absrow += np.abs(d).sum(axis=2) - np.abs(d[:, d3, d3])
    d[:, d3, d3] = absrow + dominance
    vals[dpos] = d
    return row_ptr, col_idx, vals.reshape(-1)


def half_coupled_bsr3(n_sub: int, P: int, seed: int, dominance: float = 1.0, h: int = 0):
    """n_sub chunks of P block rows; inside each chunk, row i >= h (default P // 2)
    couples to row i - h (both directions) and nothing else, so the first h
    rows of a chunk form one wide level without lower blocks (a long run of
    block-free level-0 records in the factor stream) followed by one level
    with one lower block per row. Random full 3x3 blocks, block-row dominant.
    Used with contiguous chunk partitions of P rows (the ring-release tests)."""
    rng = np.random.default_rng(seed)
    n = n_sub * P
    h = h or P // 2
    rows, cols = [], []
    for c in range(n_sub):
        for i in range(P):
            g = c * P + i
            nb = [g]
            if i >= h:
                nb.append(g - h)
            if i < P - h and i + h < P:
                nb.append(g + h)
            for j in sorted(nb):
                rows.append(g)
                cols.append(j)
    rows = np.array(rows)
    col_idx = np.array(cols, dtype=np.int32)
    row_ptr = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))]).astype(np.int64)
    vals = rng.uniform(-1.0, 1.0, (col_idx.shape[0], 3, 3))
    diag = col_idx == rows
    absrow = np.zeros((n, 3))
    np.add.at(absrow, rows[~diag], np.abs(vals[~diag]).sum(axis=2))
    d3 = np.arange(3)
    dv = vals[diag]
    absrow += np.abs(dv).sum(axis=2) - np.abs(dv[:, d3, d3])
    dv[:, d3, d3] = absrow + dominance
    vals[diag] = dv
    return row_ptr, col_idx, vals.reshape(-1)


def stencil27_pattern(nx: int, ny: int, nz: int):
    """27-point pattern (all neighbours within distance 1 in each coordinate),
    natural order, columns ascending: up to 13 strictly-lower blocks per row."""
    n = nx * ny * nz
    g = np.arange(n, dtype=np.int64)
    i, j, k = g % nx, (g // nx) % ny, g // (nx * ny)
    cols, masks = [], []
    for dk in (-1, 0, 1):
        for dj in (-1, 0, 1):
            for di in (-1, 0, 1):
                ok = (i + di >= 0) & (i + di < nx) & (j + dj >= 0) & (j + dj < ny) & (k + dk >= 0) & (k + dk < nz)
                cols.append(g + di + nx * (dj + ny * dk))
                masks.append(ok)
    cols = np.stack(cols, axis=1)
    mask = np.stack(masks, axis=1)  # offsets ascend with (dk, dj, di) -> columns ascending
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(axis=1), out=row_ptr[1:])
    return row_ptr, cols[mask].astype(np.int32)


def random_block_stencil27(nx: int, ny: int, nz: int, seed: int, dominance: float = 1.0):
    """27-point pattern with random full 3x3 blocks, block-row diagonally dominant
    (rows with up to 13 lower and 13 upper blocks: the general-K record path)."""
    rng = np.random.default_rng(seed)
    row_ptr, col_idx = stencil27_pattern(nx, ny, nz)
    n = nx * ny * nz
    vals = rng.uniform(-1.0, 1.0, (col_idx.shape[0], 3, 3))
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    diag = col_idx == rows
    absrow = np.zeros((n, 3))
    np.add.at(absrow, rows[~diag], np.abs(vals[~diag]).sum(axis=2))
    d3 = np.arange(3)
    dpos = np.nonzero(diag)[0]
    d = vals[dpos]
    absrow += np.abs(d).sum(axis=2) - np.abs(d[:, d3, d3])
    d[:, d3, d3] = absrow + dominance
    vals[dpos] = d
    return row_ptr, col_idx, vals.reshape(-1)


def random_csr_stencil27(nx: int, ny: int, nz: int, seed: int, dominance: float = 1.0):
    """Scalar 27-point analogue of random_block_stencil27."""
    rng = np.random.default_rng(seed)
    row_ptr, col_idx = stencil27_pattern(nx, ny, nz)
    n = nx * ny * nz
    vals = rng.uniform(-1.0, 1.0, col_idx.shape[0])
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    diag = col_idx == rows
    absrow = np.zeros(n)
    np.add.at(absrow, rows[~diag], np.abs(vals[~diag]))
    vals[diag] = absrow + dominance
    return row_ptr, col_idx, vals


def random_block_chain(n: int, seed: int, dominance: float = 1.0):
    """Block-tridiagonal (1-D chain) matrix with random full 3x3 blocks."""
    return random_block_grid(n, 1, 1, seed, dominance)


def manufactured_rhs(row_ptr, col_idx, vals, seed: int = 1):
    """x* ~ U[0,1)^(3N) from default_rng(seed); b = A x* via scipy (library)."""
    n = row_ptr.shape[0] - 1
    xs = np.random.default_rng(seed).random(3 * n)
    b = bsr_to_scipy(row_ptr, col_idx, vals) @ xs
    return xs, b


def apply_input(n_block_rows: int, seed: int = 2):
    """Preconditioner-apply input r ~ U[-1,1)^(3N) from default_rng(seed)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, 3 * n_block_rows)


def bsr_to_scipy(row_ptr, col_idx, vals):
    import scipy.sparse as sp
    n = row_ptr.shape[0] - 1
    return sp.bsr_matrix((np.asarray(vals).reshape(-1, 3, 3), np.asarray(col_idx),
                          np.asarray(row_ptr)), shape=(3 * n, 3 * n))
