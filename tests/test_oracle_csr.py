"""Pins for the oracle's scalar CSR path (the paper's CSR half,
P:110, Alg. 7 P:680-711 with 1x1 blocks). Worked examples of SPEC.md are
scalar, so they apply directly here. CPU only."""
import numpy as np
import pytest
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
from inputs.gen import csr_to_scipy, laplacian_csr, manufactured_rhs_csr, random_csr_grid, spe10_style_csr
from tests.helpers import golden

G = golden("spec_worked_examples.json")


def dense_csr(A):
    A = np.asarray(A, float)
    n = A.shape[0]
    rp, ci, v = [0], [], []
    for i in range(n):
        for j in range(n):
            if A[i, j] != 0.0 or i == j:
                ci.append(j)
                v.append(A[i, j])
        rp.append(len(ci))
    return np.array(rp, np.int64), np.array(ci, np.int32), np.array(v)


def split(rp, ci, lu, dinv, uunit):
    n = rp.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    M = sp.csr_matrix((lu, ci, rp), shape=(n, n)).toarray()
    Lo = np.tril(M, -1) + np.eye(n)
    U = np.triu(M)
    Uu = sp.csr_matrix((np.where(ci > rows, uunit, 0.0), ci, rp), shape=(n, n)).toarray() + np.eye(n)
    return Lo, U, Uu


def test_s1_spmv_worked_example_and_scipy():
    """[[6,-1],[-1,6]] . 1 = 5; random matrix vs scipy csr @ x."""
    rp, ci, v = dense_csr(G["spmv_2x2"]["A"])
    assert np.array_equal(oracle.s_spmv(rp, ci, v, np.ones(2)), np.full(2, 5.0))
    rp, ci, v = random_csr_grid(7, 5, 4, seed=3)
    x = np.random.default_rng(0).standard_normal(rp.shape[0] - 1)
    np.testing.assert_allclose(oracle.s_spmv(rp, ci, v, x), csr_to_scipy(rp, ci, v) @ x, rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("seed", [0, 1])
def test_s2_reorder_and_drop_brute_force(seed):
    """Reordered = dense A[p][:, p]; dropped = mask of same-label pairs."""
    rp, ci, v = random_csr_grid(4, 3, 2, seed=seed)
    n = 24
    lab = np.random.default_rng(seed).integers(0, 5, n).astype(np.int32)
    n2o, o2n = oracle.permutation(lab)
    rpr, cir, vr = oracle.s_reorder(rp, ci, v, n2o, o2n)
    Ad = csr_to_scipy(rp, ci, v).toarray()
    assert np.array_equal(csr_to_scipy(rpr, cir, vr).toarray(), Ad[n2o][:, n2o])
    ln = lab[n2o]
    rpd, cid, vd = oracle.s_drop(rpr, cir, vr, ln)
    assert np.array_equal(csr_to_scipy(rpd, cid, vd).toarray(),
                          np.where(ln[:, None] == ln[None, :], Ad[n2o][:, n2o], 0.0))


def test_s3_ilu0_defining_property_and_exact_cases():
    """(LU)_ij = A_ij on pattern(A); tridiagonal -> exact LU; full pattern ->
    unpivoted LU = scipy.linalg.lu of a diagonally dominant matrix (P = I)."""
    rp, ci, v = random_csr_grid(6, 5, 4, seed=4)
    lu, dinv = oracle.s_ilu0(rp, ci, v)
    n = rp.shape[0] - 1
    Lo, U, _ = split(rp, ci, lu, dinv, np.zeros_like(lu))
    A = csr_to_scipy(rp, ci, v).toarray()
    mask = A != 0
    np.testing.assert_allclose((Lo @ U)[mask], A[mask], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dinv, 1.0 / np.diag(U), rtol=0, atol=0)
    # tridiagonal: ILU0 is the exact LU
    rp, ci, v = random_csr_grid(12, 1, 1, seed=5)
    lu, dinv = oracle.s_ilu0(rp, ci, v)
    Lo, U, _ = split(rp, ci, lu, dinv, np.zeros_like(lu))
    np.testing.assert_allclose(Lo @ U, csr_to_scipy(rp, ci, v).toarray(), rtol=1e-13, atol=1e-13)
    # full pattern: unpivoted LU (diagonally dominant -> scipy's partial pivoting does not pivot)
    rng = np.random.default_rng(6)
    A = rng.uniform(-1, 1, (7, 7)) + 8 * np.eye(7)
    P, L, U = scipy.linalg.lu(A)
    assert np.array_equal(P, np.eye(7))
    rp, ci, v = dense_csr(A)
    lu, dinv = oracle.s_ilu0(rp, ci, v)
    Lo, Uo, _ = split(rp, ci, lu, dinv, np.zeros_like(lu))
    np.testing.assert_allclose(Lo, L, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(Uo, U, rtol=1e-13, atol=1e-13)


def test_s3_worked_examples_and_errors():
    """2x2 worked examples and the error codes."""
    ex = G["ilu0_2x2"]
    rp, ci, v = dense_csr(ex["A"])
    lu, dinv = oracle.s_ilu0(rp, ci, v)
    Lo, U, _ = split(rp, ci, lu, dinv, np.zeros_like(lu))
    np.testing.assert_allclose(Lo, np.array([[1.0, 0.0], [ex["L21"], 1.0]]), rtol=1e-15)
    np.testing.assert_allclose(U, np.array(ex["U"], float), rtol=1e-15)
    with pytest.raises(oracle.OracleError) as e:
        oracle.s_ilu0(*dense_csr([[1.0, 1.0], [1.0, 1.0]]))
    assert e.value.code == 2 and e.value.row == 1
    rp = np.array([0, 1, 2], np.int64)
    with pytest.raises(oracle.OracleError) as e:
        oracle.s_ilu0(rp, np.array([1, 0], np.int32), np.ones(2))
    assert e.value.code == 1


def test_s4_ildu0_reassembly():
    """L . diag(U_ii) . Uunit = L . U."""
    rp, ci, v = random_csr_grid(5, 4, 3, seed=7)
    lu, dinv = oracle.s_ilu0(rp, ci, v)
    uu = oracle.s_ildu0(rp, ci, lu, dinv)
    Lo, U, Uu = split(rp, ci, lu, dinv, uu)
    np.testing.assert_allclose(Lo @ np.diag(np.diag(U)) @ Uu, Lo @ U, rtol=1e-12, atol=1e-12)


def test_s5_apply_vs_library_triangular_solves():
    """Fused apply = scipy spsolve_triangular(L, unit) -> D^-1 -> spsolve_triangular(Uunit, unit),
    per subdomain (library routines, different summation order -> 1e-12)."""
    rp, ci, v = random_csr_grid(8, 6, 4, seed=8)
    S = oracle.setup_csr(rp, ci, v, grid=(8, 6, 4), tiles=(4, 3, 2))
    r = np.random.default_rng(1).uniform(-1, 1, S["n"])
    z = oracle.apply(S, r)
    Lo, U, Uu = split(S["rp_d"], S["ci_d"], S["lu"], S["dinv"], S["uunit"])
    y = spla.spsolve_triangular(sp.csr_matrix(Lo), r, lower=True, unit_diagonal=True)
    y = S["dinv"] * y
    ref = spla.spsolve_triangular(sp.csr_matrix(Uu), y, lower=False, unit_diagonal=True)
    np.testing.assert_allclose(z, ref, rtol=1e-12, atol=1e-12)


def test_s5_apply_worked_example():
    """x = [0.3, 0.8] (S:424 composition example)."""
    ex = G["apply_2x2"]  # factors of ilu0_2x2's A (S:424 composes them by hand)
    rp, ci, v = dense_csr(G["ilu0_2x2"]["A"])
    S = oracle.setup_csr(rp, ci, v, P=2)
    z = oracle.apply(S, np.array(ex["b"], float))
    np.testing.assert_allclose(z, np.array(ex["x"], float), rtol=1e-15)


def test_s6_bicgstab_manufactured_and_2x2():
    """2x2 x = [1/11, 7/11]; manufactured x* recovered on a Laplacian
    and on the scalar SPE10-style matrix (true residual <= 10 tol)."""
    ex = G["bicgstab_2x2"]
    rp, ci, v = dense_csr(ex["A"])
    S = oracle.setup_csr(rp, ci, v, P=1)
    x, rep = oracle.bicgstab(S, np.array(ex["b"], float), tol=1e-12)
    np.testing.assert_allclose(x, np.array(ex["x_num"], float) / ex["x_den"], rtol=1e-10)
    for gen, kw, tol in ((lambda: laplacian_csr(16, 16, 16), dict(grid=(16, 16, 16), tiles=(8, 8, 8)), 1e-8),
                         (lambda: spe10_style_csr(20, 40, 20, upper_ness_from=10)[:3],
                          dict(grid=(20, 40, 20), tiles=(10, 20, 10)), 1e-8)):
        rp, ci, v = gen()
        S = oracle.setup_csr(rp, ci, v, **kw)
        xs, b = manufactured_rhs_csr(rp, ci, v)
        br = b[S["new_to_old"]]
        x, rep = oracle.bicgstab(S, br, tol=tol, max_iter=2000)
        assert rep["status"] == 0 and rep["true_rel_resid"] <= 10 * tol


def test_s6_bicgstab_matches_scipy_with_oracle_preconditioner():
    """scipy.sparse.linalg.bicgstab with M = the oracle's apply converges to the
    same solution (library algorithm; iteration counts may differ by convention)."""
    rp, ci, v = random_csr_grid(10, 8, 6, seed=9)
    S = oracle.setup_csr(rp, ci, v, grid=(10, 8, 6), tiles=(5, 4, 3))
    Ar = csr_to_scipy(S["rp_r"], S["ci_r"], S["v_r"])
    b = np.random.default_rng(2).standard_normal(S["n"])
    M = spla.LinearOperator(Ar.shape, matvec=lambda r: oracle.apply(S, r))
    xs, info = spla.bicgstab(Ar, b, M=M, rtol=1e-12, atol=0, maxiter=500)
    assert info == 0
    x, rep = oracle.bicgstab(S, b, tol=1e-12, max_iter=500)
    np.testing.assert_allclose(x, xs, rtol=1e-8, atol=1e-10)


def test_s7_spe10_scalar_count():
    """The scalar SPE10-style matrix has the paper's spe10 nonzero count."""
    rp, _, v, _ = spe10_style_csr()
    assert rp[-1] == 7_780_000
