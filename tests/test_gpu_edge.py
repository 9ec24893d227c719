"""GPU edge cases of the solver and the apply through the C ABI, against the
oracle: zero right-hand side, one- and two-row systems, A = I (exit at the
half step), a nonzero initial guess, max_iter = 1, P larger than n."""
import numpy as np
import pytest

import oracle
import paper_2508_04917_b200 as dd
from inputs.gen import random_block_grid
from tests.helpers import golden, kron_blocks

pytestmark = pytest.mark.gpu
G = golden("spec_worked_examples.json")


def tvec(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def test_zero_rhs_converges_at_zero_iterations():
    rp, ci, v = random_block_grid(6, 5, 4, seed=1)
    ctx = dd.dd_setup(rp, ci, v, P=40)
    x = tvec(np.zeros(3 * 120))
    rep = ctx.bicgstab(tvec(np.zeros(3 * 120)), x, tol=1e-8)
    assert rep["converged"] == 1 and rep["iterations"] == 0 and rep["n_applies"] == 0
    assert float(x.abs().max()) == 0.0


def test_two_row_worked_example():
    """[[4,1],[1,3]] (x) I3, b = [1,2] (x) 1 -> x = [1/11, 7/11] (x) 1."""
    ex = G["bicgstab_2x2"]
    rp, ci, v = kron_blocks(ex["A"])
    b = np.repeat(np.array(ex["b"], float), 3)
    xs = np.repeat(np.array(ex["x_num"], float) / ex["x_den"], 3)
    for P in (1, 2):
        S = oracle.setup(rp, ci, v, P=P)
        ctx = dd.dd_setup(rp, ci, v, P=P)
        x = tvec(np.zeros(6))
        assert np.array_equal(S["new_to_old"], [0, 1])  # chunks keep the natural order
        rep = ctx.bicgstab(tvec(b), x, tol=1e-12)
        xo, ro = oracle.bicgstab(S, b, tol=1e-12)
        assert rep["converged"] == 1 and rep["iterations"] == ro["iterations"]
        np.testing.assert_allclose(x.cpu().numpy(), xs, rtol=1e-10)


def test_single_row_system():
    rp = np.array([0, 1], np.int64)
    ci = np.array([0], np.int32)
    v = np.array([4.0, 1.0, 0.0, 1.0, 3.0, 1.0, 0.0, 1.0, 5.0])
    S = oracle.setup(rp, ci, v, P=1)
    ctx = dd.dd_setup(rp, ci, v, P=1)
    r = np.array([1.0, -2.0, 3.0])
    z = tvec(np.zeros(3))
    for var in (dd.DD_LEVELSET, dd.DD_SPINLOOP, dd.DD_DIRECT, dd.DD_UNFUSED):
        ctx.apply(tvec(r), z, var)
        assert np.array_equal(z.cpu().numpy(), oracle.apply(S, r))
    x = tvec(np.zeros(3))
    rep = ctx.bicgstab(tvec(r), x, tol=1e-12)
    # M = A exactly (one block): converged at the first half step
    assert rep["converged"] == 1 and rep["iterations"] == 0.5
    np.testing.assert_allclose(x.cpu().numpy(), np.linalg.solve(v.reshape(3, 3), r), rtol=1e-12)


def test_identity_exits_at_half_step():
    """A = I: M = I, s = 0 after the first half step (O12 pin)."""
    n = 50
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int32)
    v = np.tile(np.eye(3).ravel(), n)
    ctx = dd.dd_setup(rp, ci, v, P=7)
    b = np.random.default_rng(0).standard_normal(3 * n)
    x = tvec(np.zeros(3 * n))
    rep = ctx.bicgstab(tvec(b), x, tol=1e-10)
    assert rep["iterations"] == 0.5 and rep["converged"] == 1
    assert np.array_equal(x.cpu().numpy(), b)


def test_nonzero_initial_guess_matches_oracle():
    rp, ci, v = random_block_grid(10, 8, 6, seed=5)
    kw = dict(grid=(10, 8, 6), tiles=(5, 4, 3))
    S = oracle.setup(rp, ci, v, **kw)
    ctx = dd.dd_setup(rp, ci, v, **kw)
    rng = np.random.default_rng(3)
    b, x0 = rng.standard_normal(3 * S["n"]), rng.standard_normal(3 * S["n"])
    xo, ro = oracle.bicgstab(S, b, x0=x0, tol=1e-9, max_iter=500)
    x = tvec(x0)
    rep = ctx.bicgstab(tvec(b), x, tol=1e-9, max_iter=500, hist=True)
    assert rep["converged"] == 1 and abs(rep["iterations"] - ro["iterations"]) <= 2
    k = min(len(rep["resid_hist"]), len(ro["resid_hist"]), 8)
    np.testing.assert_allclose(rep["resid_hist"][:k], ro["resid_hist"][:k], rtol=1e-9)


def test_max_iter_one_and_P_larger_than_n():
    rp, ci, v = random_block_grid(4, 4, 4, seed=9)
    ctx = dd.dd_setup(rp, ci, v, P=1000)  # one subdomain smaller than P
    assert ctx.stats()["n_sub"] == 1
    b = np.random.default_rng(1).standard_normal(3 * 64)
    x = tvec(np.zeros(3 * 64))
    rep = ctx.bicgstab(tvec(b), x, tol=1e-30, max_iter=1)
    assert rep["status_name"] == "DD_E_MAXITER" and rep["iterations"] == 1 and rep["n_applies"] == 2
