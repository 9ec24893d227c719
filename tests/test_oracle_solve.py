"""Pins for the oracle's apply / SpMV / dot / BiCGSTAB (O9-O12)."""
import math
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import oracle
from inputs.gen import (apply_input, laplacian_bsr3, manufactured_rhs, random_block_chain,
                        random_block_grid, spe10_style_bsr3)
from tests.helpers import bsr, golden, kron_blocks, split_factors

G = golden("spec_worked_examples.json")


# ------------------------------------------------------------------ O9 apply
def test_o9_worked_example_2x2():
    """A=[[4,1],[2,3]] one subdomain; b=[2,3] -> x=[0.3,0.8], A x = b."""
    ex = G["apply_2x2"]
    rp, ci, a = kron_blocks(golden("spec_worked_examples.json")["ilu0_2x2"]["A"])
    S = oracle.setup(rp, ci, a, P=2)
    b = np.repeat(np.array(ex["b"], float), 3)
    z = oracle.apply(S, b)
    assert np.allclose(z, np.repeat(ex["x"], 3), rtol=0, atol=1e-15)
    A = bsr(rp, ci, a).toarray()
    assert np.abs(A @ z - b).max() <= 1e-15 * 4


@pytest.mark.parametrize("seed,t", [(0, 4), (1, 5), (2, 16)])
def test_o9_block_jacobi_exact(seed, t):
    """1-D chain subdomains are block-tridiagonal, ILU0 is exact, so the apply
    equals numpy.linalg.solve(A_ss, r_s) per subdomain (block-Jacobi)."""
    n = 4 * t
    rp, ci, a = random_block_chain(n, seed=seed)
    S = oracle.setup(rp, ci, a, grid=(n, 1, 1), tiles=(t, 1, 1))
    r = apply_input(n, seed=2)
    z = oracle.apply(S, r)
    A = bsr(S["rp_r"], S["ci_r"], S["v_r"]).toarray()
    for s in range(S["n_sub"]):
        lo, hi = 3 * S["sub_ptr"][s], 3 * S["sub_ptr"][s + 1]
        ref = np.linalg.solve(A[lo:hi, lo:hi], r[lo:hi])
        assert np.abs(z[lo:hi] - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("grid,tiles,seed", [((4, 4, 4), (2, 2, 2), 0), ((6, 6, 6), (3, 3, 3), 1),
                                             ((6, 4, 4), (6, 2, 4), 2)])
def test_o9_dense_brute_force(grid, tiles, seed):
    """z = (L U)^-1 r with L U assembled from the factors (themselves pinned by
    O6) and solved densely by LAPACK."""
    rp, ci, v = random_block_grid(*grid, seed=seed)
    S = oracle.setup(rp, ci, v, grid=grid, tiles=tiles)
    F = split_factors(S["rp_d"], S["ci_d"], S["lu"])
    M = (F["L"] @ F["U"]).toarray()
    r = apply_input(S["n"], seed=2)
    z = oracle.apply(S, r)
    ref = np.linalg.solve(M, r)
    assert np.abs(z - ref).max() <= 1e-12 * np.abs(ref).max()


def test_o9_scalar_laplacian_triplicated():
    """e*I3 blocks: equal components in -> equal components out (scalar solve x3)."""
    rp, ci, v = laplacian_bsr3(8, 8, 8)
    S = oracle.setup(rp, ci, v, grid=(8, 8, 8), tiles=(4, 4, 4))
    r = np.repeat(np.random.default_rng(3).uniform(-1, 1, S["n"]), 3)
    z = oracle.apply(S, r).reshape(-1, 3)
    assert np.array_equal(z[:, 0], z[:, 1]) and np.array_equal(z[:, 0], z[:, 2])


def test_o9_threads_bitwise():
    rp, ci, v = random_block_grid(8, 8, 8, seed=9)
    S = oracle.setup(rp, ci, v, grid=(8, 8, 8), tiles=(4, 4, 2))
    r = apply_input(S["n"])
    oracle.set_threads(1)
    z1 = oracle.apply(S, r)
    oracle.set_threads(4)
    z4 = oracle.apply(S, r)
    oracle.set_threads(0)
    assert np.array_equal(z1, z4)


# ------------------------------------------------------------------- O10 spmv
@pytest.mark.parametrize("seed", range(3))
def test_o10_spmv_vs_scipy(seed):
    rp, ci, v = random_block_grid(5, 4, 3, seed=seed)
    x = np.random.default_rng(seed).uniform(-1, 1, 3 * 60)
    y = oracle.spmv(rp, ci, v, x)
    ref = bsr(rp, ci, v) @ x
    assert np.abs(y - ref).max() <= 1e-15 * np.abs(ref).max() * 8
    eye = kron_blocks(np.eye(3))
    assert np.array_equal(oracle.spmv(*eye, x[:9]), x[:9])


# -------------------------------------------------------------------- O11 dot
def _exact_dot(x, y):
    return float(sum(Fraction(a) * Fraction(b) for a, b in zip(x, y)))


@pytest.mark.parametrize("seed", range(4))
def test_o11_dot_correctly_rounded(seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, 2000)
    y = rng.uniform(-1, 1, 2000)
    assert oracle.dot(x, y) == _exact_dot(x, y)


def test_o11_dot_cancellation_and_integers():
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, 500)
    y = rng.uniform(-1, 1, 500)
    x = np.concatenate([x, x * 1e8, -x * 1e8])  # heavy cancellation, cond ~ 1e16
    y = np.concatenate([y, y, y])
    ex = _exact_dot(x, y)
    u = 2.0 ** -53
    bound = u * abs(ex) + (len(x) * u) ** 2 * float(np.sum(np.abs(x * y)))
    assert abs(oracle.dot(x, y) - ex) <= bound
    xi = np.arange(-50, 50, dtype=float)
    assert oracle.dot(xi, xi) == float(sum(int(a) ** 2 for a in range(-50, 50)))
    assert math.isclose(oracle.dot(x, y), ex, rel_tol=1e-15, abs_tol=bound)


# --------------------------------------------------------------- O12 BiCGSTAB
def test_o12_identity_converges_half_step():
    rp, ci, a = kron_blocks(np.eye(4))
    S = oracle.setup(rp, ci, a, P=4)
    b = np.arange(1.0, 13.0)
    x, rep = oracle.bicgstab(S, b)
    assert rep["status"] == 0 and rep["iterations"] == 0.5 and rep["n_applies"] == 1
    assert np.array_equal(x, b)


def test_o12_worked_example_2x2():
    """[[4,1],[1,3]] x = [1,2] -> x = [1/11, 7/11] within 2 iterations.
    P=1 makes M the block-Jacobi diagonal (not exact), so the Krylov loop runs."""
    ex = G["bicgstab_2x2"]
    rp, ci, a = kron_blocks(ex["A"])
    S = oracle.setup(rp, ci, a, P=1)
    b = np.repeat(np.array(ex["b"], float), 3)
    x, rep = oracle.bicgstab(S, b, tol=1e-14)
    assert rep["status"] == 0 and rep["iterations"] <= ex["max_iterations"]
    ref = np.repeat(np.array(ex["x_num"]) / ex["x_den"], 3)
    assert np.abs(x - ref).max() <= 1e-14


def _straight_line_bicgstab(A, Minv, b, tol, kmax):
    """Independent textbook right-preconditioned BiCGSTAB (van der Vorst, Alg. 1
    P:139-163 with K1 = I), numpy arithmetic; returns residual history."""
    x = np.zeros_like(b)
    r = b - A @ x
    rh = r.copy()
    n0 = np.linalg.norm(r)
    hist = [n0]
    rho_p = alpha = omega = 1.0
    v = np.zeros_like(b)
    p = np.zeros_like(b)
    for k in range(1, kmax + 1):
        rho = rh @ r
        p = r.copy() if k == 1 else r + (rho / rho_p) * (alpha / omega) * (p - omega * v)
        ph = Minv(p)
        v = A @ ph
        alpha = rho / (rh @ v)
        s = r - alpha * v
        hist.append(np.linalg.norm(s))
        if hist[-1] < tol * n0:
            return hist
        sh = Minv(s)
        t = A @ sh
        omega = (t @ s) / (t @ t)
        x = x + alpha * ph + omega * sh
        r = s - omega * t
        hist.append(np.linalg.norm(r))
        if hist[-1] < tol * n0:
            return hist
        rho_p = rho
    return hist


@pytest.mark.parametrize("seed", range(3))
def test_o12_matches_textbook_and_scipy(seed):
    grid, tiles = (8, 6, 4), (4, 3, 2)
    rp, ci, v = random_block_grid(*grid, seed=seed, dominance=0.2)
    S = oracle.setup(rp, ci, v, grid=grid, tiles=tiles)
    A = bsr(S["rp_r"], S["ci_r"], S["v_r"]).tocsr()
    F = split_factors(S["rp_d"], S["ci_d"], S["lu"])
    Mlu = spla.splu((F["L"] @ F["U"]).tocsc())
    b = np.random.default_rng(seed).uniform(0, 1, A.shape[0])
    x, rep = oracle.bicgstab(S, b, tol=1e-10)
    assert rep["status"] == 0
    hist = _straight_line_bicgstab(A, Mlu.solve, b, 1e-10, 200)
    k = min(8, len(hist), len(rep["resid_hist"]))
    assert np.allclose(rep["resid_hist"][:k], hist[:k], rtol=1e-8, atol=0)
    assert abs(len(hist) - len(rep["resid_hist"])) <= 2
    M = spla.LinearOperator(A.shape, matvec=lambda q: oracle.apply(S, q))
    xs, info = spla.bicgstab(A, b, M=M, rtol=1e-10, atol=0.0, maxiter=500)
    assert info == 0
    assert np.abs(x - xs).max() <= 1e-7 * np.abs(xs).max()


def test_o12_manufactured_and_iteration_ratio():
    """x* recovered with true residual <= 10 tol; decomposed/global iteration
    ratio within [1, 3] (paper's geomean 1.6)."""
    grid = (16, 16, 16)
    rp, ci, v = laplacian_bsr3(*grid)
    xs, b = manufactured_rhs(rp, ci, v, seed=1)
    its = {}
    for name, tiles in (("global", grid), ("dd", (8, 8, 4))):
        S = oracle.setup(rp, ci, v, grid=grid, tiles=tiles)
        br = b.reshape(-1, 3)[S["new_to_old"]].ravel()
        x, rep = oracle.bicgstab(S, br, tol=1e-8)
        assert rep["status"] == 0 and rep["true_rel_resid"] <= 1e-7
        xo = np.empty_like(x).reshape(-1, 3)
        xo[S["new_to_old"]] = x.reshape(-1, 3)
        assert np.abs(xo.ravel() - xs).max() <= 1e-5
        its[name] = rep["iterations"]
    assert 1.0 <= its["dd"] / its["global"] <= 3.0


def test_o12_spe10_style_converges():
    rp, ci, v, _ = spe10_style_bsr3(12, 20, 10, upper_ness_from=5)
    xs, b = manufactured_rhs(rp, ci, v)
    S = oracle.setup(rp, ci, v, grid=(12, 20, 10), tiles=(6, 10, 5))
    br = b.reshape(-1, 3)[S["new_to_old"]].ravel()
    x, rep = oracle.bicgstab(S, br, tol=1e-8, max_iter=2000)
    assert rep["status"] == 0 and rep["true_rel_resid"] <= 1e-7


def test_o12_breakdown_sigma_closed_form():
    """R25 sigma test pinned by exact arithmetic: A = [[1, 2], [0, -1]] (x I3),
    P = 1 -> M = blockdiag(A_ii) = diag(1, -1), b = 1: p_hat = M^-1 r0 =
    (1, -1), v = A p_hat = (-1, 1), sigma = r0.v = 0 exactly -> breakdown at
    k = 1 before any update (iterations 0, one apply), x = x0."""
    rp, ci, a = kron_blocks(np.array([[1.0, 2.0], [0.0, -1.0]]))
    S = oracle.setup(rp, ci, a, P=1)
    b = np.ones(6)
    x, rep = oracle.bicgstab(S, b.reshape(-1, 3)[S["new_to_old"]].ravel(), tol=1e-8)
    assert rep["status"] == 1 and rep["iterations"] == 0.0 and rep["n_applies"] == 1
    assert np.array_equal(x, np.zeros(6))
    assert rep["resid_hist"].tolist() == [math.sqrt(6.0)]


def test_o12_breakdown_rho_initial():
    """R25 rho test: ||r0||^2 = rho_1 < 1e-30 with r0 != 0 (b of 1e-17 on 6
    entries: rho_1 = 6e-34) -> breakdown before the first apply."""
    rp, ci, a = kron_blocks(np.array([[4.0, 1.0], [1.0, 4.0]]))
    S = oracle.setup(rp, ci, a, P=2)
    x, rep = oracle.bicgstab(S, np.full(6, 1e-17), tol=1e-8)
    assert rep["status"] == 1 and rep["iterations"] == 0.0 and rep["n_applies"] == 0
    assert np.array_equal(x, np.zeros(6))


def test_o12_breakdown_tau_exact_preconditioner():
    """R25 tau test: one subdomain with a full block pattern makes ILU0 exact
    (M = A), so s = r0 - alpha A M^-1 r0 is pure rounding; with tol far below
    it the half-step test fails and tau = ||A M^-1 s||^2 < 1e-30 -> breakdown
    at iteration 1/2 (two applies), x unchanged."""
    from tests.breakdown_cases import find_case
    c = find_case("tau_k1", 3)
    assert c is not None and c["P"] == c["S"]["n"]  # one subdomain, exact ILU0
    assert np.array_equal(c["x"], np.zeros_like(c["x"]))
    assert len(c["rep"]["resid_hist"]) == 2 and c["rep"]["resid_hist"][1] < 1e-14 * c["rep"]["resid_hist"][0]


@pytest.mark.parametrize("seed", [1, 2])
def test_o9b_lower_vs_scipy_triangular(seed):
    """Table 3 analogue: orc_lower is the unit-lower solve L z = r of the
    subdomain factors -- pinned against scipy's sparse triangular solve."""
    import scipy.sparse.linalg as sla
    rp, ci, v = random_block_grid(8, 6, 4, seed=seed)
    S = oracle.setup(rp, ci, v, grid=(8, 6, 4), tiles=(4, 3, 2))
    r = apply_input(S["n"], seed=seed)
    F = split_factors(S["rp_d"], S["ci_d"], S["lu"])
    z_ref = sla.spsolve_triangular(F["L"].tocsr(), r, lower=True, unit_diagonal=True)
    z = oracle.lower(S, r)
    assert np.allclose(z, z_ref, rtol=1e-12, atol=1e-12 * np.abs(z_ref).max())


@pytest.mark.parametrize("seed", [3, 4])
def test_o9c_apply_ilu0_nonunit(seed):
    """Non-unit ILU0 apply: the dense brute force
    (L U)^-1 r of the subdomain factors with U = the ILU0 upper triangle
    incl. its diagonal blocks, and equal to the ILDU0 apply to rounding."""
    rp, ci, v = random_block_grid(6, 5, 4, seed=seed)
    S = oracle.setup(rp, ci, v, grid=(6, 5, 4), tiles=(3, 5, 2))
    r = apply_input(S["n"], seed=seed)
    F = split_factors(S["rp_d"], S["ci_d"], S["lu"])
    M = (F["L"] @ F["U"]).toarray()
    z_ref = np.linalg.solve(M, r)
    z = oracle.apply_ilu0(S, r)
    assert np.allclose(z, z_ref, rtol=1e-11, atol=1e-11 * np.abs(z_ref).max())
    z_ildu = oracle.apply(S, r)
    assert np.abs(z - z_ildu).max() <= 1e-12 * np.abs(z_ildu).max()
    # a different rounding path: not bitwise the ILDU0 result in general
    assert not np.array_equal(z, z_ildu)
