"""Multi-rank device path on ONE GPU: world 2 and 3 as contexts of this process
(DD_COMM_LOCAL, one host thread per rank), so the rank ranges, ghost columns
of the SpMV, send-row gathers, halo copies, rank-ordered dot combination and
the collective BiCGSTAB all run on the device and are checked against the
oracle. The NCCL transport differs only in the two exchange calls (halo and
all-gather, api.cpp); its host-side logic is covered by test_multirank_host.py.
"""
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import paper_2508_04917_b200 as dd
from inputs.gen import (apply_input, bsr_to_scipy, laplacian_bsr3, manufactured_rhs, random_block_grid,
                        random_block_stencil27, spe10_style_bsr3)

pytestmark = pytest.mark.gpu

CASES = {
    "random_8sub": (lambda: random_block_grid(16, 12, 10, seed=21), dict(grid=(16, 12, 10), tiles=(8, 6, 5))),
    "laplace_24^3": (lambda: laplacian_bsr3(24, 24, 24), dict(grid=(24, 24, 24), tiles=(8, 8, 8))),
    "chunks_ragged_oddP": (lambda: random_block_grid(10, 10, 10, seed=5), dict(P=77)),
    "spe10_small": (lambda: spe10_style_bsr3(20, 40, 20, upper_ness_from=10)[:3],
                    dict(grid=(20, 40, 20), tiles=(10, 20, 10))),
    # 27-point rows: the general-K apply kernels, edge and corner halo rows
    "stencil27": (lambda: random_block_stencil27(12, 12, 12, seed=33), dict(grid=(12, 12, 12), tiles=(6, 6, 4))),
}


def run_ranks(world, fn):
    """fn(rank, barrier) in `world` threads; returns the per-rank results."""
    bar = threading.Barrier(world)
    with ThreadPoolExecutor(world) as ex:
        futs = [ex.submit(fn, r, bar) for r in range(world)]
        return [f.result(timeout=600) for f in futs]


@pytest.mark.parametrize("name,world", [("random_8sub", 2), ("random_8sub", 3), ("laplace_24^3", 2),
                                        ("laplace_24^3", 4), ("chunks_ragged_oddP", 2), ("chunks_ragged_oddP", 5),
                                        ("spe10_small", 3), ("stencil27", 3)])
def test_local_world_parity(name, world):
    import torch
    gen, kw = CASES[name]
    rp, ci, v = gen()
    S = oracle.setup(rp, ci, v, **kw)
    N = S["n"]
    r_glob = apply_input(N)
    z_ref = oracle.apply(S, r_glob)
    y_ref = oracle.spmv(S["rp_r"], S["ci_r"], S["v_r"], r_glob)
    xs, b = manufactured_rhs(rp, ci, v)
    n2o = S["new_to_old"]
    b_re = b.reshape(-1, 3)[n2o].ravel()
    _, rep_ref = oracle.bicgstab(S, b_re, tol=1e-8, max_iter=2000)
    key = os.urandom(128)

    def rank_fn(rank, bar):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            ctx = dd.dd_setup(rp, ci, v, rank=rank, world=world, nccl_id=key, comm="local", **kw)
            f, n = ctx.row_first, ctx.n_local
            sl = slice(3 * f, 3 * (f + n))
            out = {"first": f, "n": n}
            r = torch.from_numpy(r_glob[sl].copy()).cuda()
            z = torch.empty_like(r)
            ctx.apply(r, z, stream=st)          # never communicates
            y = torch.empty_like(r)
            ctx.spmv(r, y, stream=st)           # collective: halo
            st.synchronize()
            out["z"], out["y"] = z.cpu().numpy(), y.cpu().numpy()
            bl = torch.from_numpy(b_re[sl].copy()).cuda()
            x = torch.zeros_like(bl)
            out["rep"] = ctx.bicgstab(bl, x, tol=1e-8, max_iter=2000, stream=st)
            out["x"] = x.cpu().numpy()
            xh = np.zeros(3 * N)
            out["rep_host"] = ctx.solve_host(b, xh, tol=1e-8, max_iter=2000, stream=st)
            out["xh"] = xh
            bar.wait()
            ctx.destroy()
            return out

    res = run_ranks(world, rank_fn)
    # the ranks own a contiguous cover of the reordered rows, in rank order
    assert res[0]["first"] == 0 and sum(o["n"] for o in res) == N
    assert all(res[q]["first"] + res[q]["n"] == res[q + 1]["first"] for q in range(world - 1))
    assert all(o["n"] > 0 for o in res)
    z = np.concatenate([o["z"] for o in res])
    y = np.concatenate([o["y"] for o in res])
    assert np.array_equal(z, z_ref), "apply not bitwise across ranks"
    assert np.array_equal(y, y_ref), "SpMV with halo not bitwise"
    its = {o["rep"]["iterations"] for o in res}
    assert len(its) == 1, f"ranks disagree on the iteration count: {its}"
    it = its.pop()
    assert all(o["rep"]["converged"] == 1 for o in res)
    assert abs(it - rep_ref["iterations"]) <= 2, (it, rep_ref["iterations"])
    assert max(o["rep"]["true_rel_resid"] for o in res) <= 10 * 1e-8
    # the assembled solution solves the ORIGINAL system (residual computed
    # here with scipy; the SPE10-style case is too ill-conditioned for a
    # forward-error bar at tol 1e-8)
    A = bsr_to_scipy(rp, ci, v)
    x = np.concatenate([o["x"] for o in res])
    x_orig = np.empty_like(x)
    x_orig.reshape(-1, 3)[n2o] = x.reshape(-1, 3)
    assert np.linalg.norm(b - A @ x_orig) <= 10 * 1e-8 * np.linalg.norm(b)
    # dd_solve_host: every rank writes its own rows of the original-order x
    xh = sum(o["xh"] for o in res)
    assert np.linalg.norm(b - A @ xh) <= 10 * 1e-8 * np.linalg.norm(b)
    assert all(o["rep_host"]["iterations"] == it for o in res)


def test_local_world_matches_single_rank_iterations():
    """The same solve at world 1 and world 2 takes the same number of
    iterations (dots combined in rank order in double-double)."""
    import torch
    gen, kw = CASES["laplace_24^3"]
    rp, ci, v = gen()
    xs, b = manufactured_rhs(rp, ci, v)
    ctx1 = dd.dd_setup(rp, ci, v, **kw)
    x1 = np.zeros_like(b)
    it1 = ctx1.solve_host(b, x1, tol=1e-10)["iterations"]
    key = os.urandom(128)

    def rank_fn(rank, bar):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            ctx = dd.dd_setup(rp, ci, v, rank=rank, world=2, nccl_id=key, comm="local", **kw)
            xh = np.zeros_like(b)
            rep = ctx.solve_host(b, xh, tol=1e-10, stream=st)
            bar.wait()
            ctx.destroy()
            return rep["iterations"], xh

    res = run_ranks(2, rank_fn)
    assert res[0][0] == res[1][0]
    assert abs(res[0][0] - it1) <= 0.5
    assert np.abs(res[0][1] + res[1][1] - x1).max() <= 1e-9 * np.abs(x1).max()


def test_local_world_bad_arguments():
    """world > 1 without a group key, or a rank outside the world, fail loudly
    before any rendezvous."""
    rp, ci, v = random_block_grid(8, 8, 8, seed=2)
    with pytest.raises(dd.DDError) as e:
        dd.dd_setup(rp, ci, v, P=64, rank=0, world=2, nccl_id=None, comm="local")
    assert e.value.name == "DD_E_INVALID_ARG"
    with pytest.raises(dd.DDError) as e:
        dd.dd_setup(rp, ci, v, P=64, rank=2, world=2, nccl_id=os.urandom(128), comm="local")
    assert e.value.name == "DD_E_INVALID_ARG"


@pytest.mark.parametrize("name,world", [("laplace_24^3", 3), ("chunks_ragged_oddP", 2), ("spe10_small", 2),
                                        ("random_8sub", 4), ("stencil27", 2)])
def test_fused_halo_and_merged_reduction_equal_plain(name, world, monkeypatch):
    """SURVEY 8(f4), world > 1. (a) Fused halo: the solver's applies write the
    rows peers read in the next SpMV straight from shared memory into the
    peers' ghost blocks (DD_COMM_LOCAL; NCCL: into the send buffer) instead of
    a gather kernel + copy (DD_HALO_FUSE=0). (b) Merged reduction: s.s joins
    the (t.s, t.t) collective, three reduction points per iteration instead
    of four (DD_MERGE_SS=0). Every combination gives the same solve bitwise
    (x, residual history, iterations), with fewer launches."""
    import torch
    gen, kw = CASES[name]
    rp, ci, v = gen()
    xs, b = manufactured_rhs(rp, ci, v)
    S = oracle.setup(rp, ci, v, **kw)
    b_re = b.reshape(-1, 3)[S["new_to_old"]].ravel()
    def solve(knobs, tol):
        monkeypatch.setenv("DD_HALO_FUSE", knobs[0])
        monkeypatch.setenv("DD_MERGE_SS", knobs[1])
        key = os.urandom(128)

        def rank_fn(rank, bar):
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                ctx = dd.dd_setup(rp, ci, v, rank=rank, world=world, nccl_id=key, comm="local", **kw)
                f, n = ctx.row_first, ctx.n_local
                bl = torch.from_numpy(b_re[3 * f:3 * (f + n)].copy()).cuda()
                x = torch.zeros_like(bl)
                l0 = ctx.stats()["launches"]
                rep = ctx.bicgstab(bl, x, tol=tol, max_iter=2000, hist=True, stream=st)
                launches = ctx.stats()["launches"] - l0
                st.synchronize()
                res = (x.cpu().numpy(), rep, launches)
                bar.wait()
                ctx.destroy()
                return res

        return run_ranks(world, rank_fn)

    # a tolerance met first at a half step (so the merged path's deferred
    # half-step test and x += alpha p_hat are exercised)
    h = solve(("0", "0"), 1e-8)[0][1]["resid_hist"]
    j = next(j for j in range(3, len(h), 2) if h[j] < h[:j].min())
    tol_half = h[j] * (1 + 1e-9) / h[0]
    for tol in (1e-8, tol_half):
        out = {knobs: solve(knobs, tol) for knobs in (("0", "0"), ("1", "0"), ("0", "1"), ("1", "1"))}
        base = out[("0", "0")]
        if tol == tol_half:
            assert base[0][1]["iterations"] == (j + 1) / 2 - 0.5, (base[0][1]["iterations"], j)
        for knobs, res in out.items():
            for q in range(world):
                x0, rep0, l0 = base[q]
                x1, rep1, l1 = res[q]
                assert rep1["converged"] == 1 and rep0["iterations"] == rep1["iterations"], (knobs, tol)
                assert np.array_equal(x0, x1), f"rank {q}: {knobs} changed the solve"
                assert np.array_equal(rep0["resid_hist"], rep1["resid_hist"]), (knobs, tol)
                if knobs != ("0", "0"):
                    assert l1 < l0, (knobs, q, l0, l1)


@pytest.mark.parametrize("host", ["0", "1"])
def test_local_world_setup_status_agreed(host, monkeypatch):
    """a singular pivot inside ONE rank's subdomains must
    fail every rank with the same status -- no rank left waiting in a
    collective its peers never reach. Rank 1 owns the second half of the
    chunks; one of its diagonal blocks is made singular. Both the GPU
    factorisation (host "0") and the host ILU0 (host "1") paths."""
    monkeypatch.setenv("DD_HOST_ILU0", host)
    rp, ci, v = random_block_grid(8, 8, 4, seed=13)
    v = v.reshape(-1, 3, 3).copy()
    n = rp.shape[0] - 1
    # the FIRST row of the last chunk (rank 1 of 2, P = 64): its lower
    # neighbours lie in other chunks and are dropped, so U_ii = A_ii = 0
    row = n - 64
    diag = next(p for p in range(rp[row], rp[row + 1]) if ci[p] == row)
    v[diag] = 0.0
    v = v.reshape(-1)
    key = os.urandom(128)

    def rank_fn(rank, bar):
        try:
            ctx = dd.dd_setup(rp, ci, v, rank=rank, world=2, nccl_id=key, comm="local", P=64)
            ctx.destroy()
            return "DD_OK", ""
        except dd.DDError as e:
            return e.name, str(e)

    res = run_ranks(2, rank_fn)
    assert [r[0] for r in res] == ["DD_E_SINGULAR_PIVOT"] * 2, res
    assert "peer rank" in res[0][1] or "singular" in res[0][1]


@pytest.mark.parametrize("name,world", [("random_8sub", 2), ("chunks_ragged_oddP", 3), ("stencil27", 2)])
def test_local_world_refactor(name, world):
    """dd_refactor at world > 1 (collective): every rank re-factors its
    subdomains from new values of the same pattern (7-point: the diagonal-update
    kernel with the fused SpMV-operand copy; 27-point: k_refactor9); the apply
    and the halo SpMV then equal a fresh oracle setup of the new values, bit for
    bit, on every rank."""
    import torch
    gen, kw = CASES[name]
    rp, ci, v1 = gen()
    # new values of the same pattern: a 5 % perturbation keeps every pivot block regular
    v2 = v1 * (1.0 + 0.05 * np.random.default_rng(9).uniform(-1.0, 1.0, v1.shape))
    S2 = oracle.setup(rp, ci, v2, **kw)
    N = S2["n"]
    r_glob = apply_input(N)
    z_ref = oracle.apply(S2, r_glob)
    y_ref = oracle.spmv(S2["rp_r"], S2["ci_r"], S2["v_r"], r_glob)
    key = os.urandom(128)

    def rank_fn(rank, bar):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            ctx = dd.dd_setup(rp, ci, v1, rank=rank, world=world, nccl_id=key, comm="local", enable_refactor=True,
                              **kw)
            ctx.refactor(torch.from_numpy(v2.reshape(-1).copy()).cuda(), stream=st)  # collective
            f, n = ctx.row_first, ctx.n_local
            sl = slice(3 * f, 3 * (f + n))
            r = torch.from_numpy(r_glob[sl].copy()).cuda()
            z = torch.empty_like(r)
            y = torch.empty_like(r)
            ctx.apply(r, z, stream=st)
            ctx.spmv(r, y, stream=st)  # collective: halo
            st.synchronize()
            out = {"first": f, "n": n, "z": z.cpu().numpy(), "y": y.cpu().numpy()}
            bar.wait()
            ctx.destroy()
            return out

    outs = run_ranks(world, rank_fn)
    for o in outs:
        sl = slice(3 * o["first"], 3 * (o["first"] + o["n"]))
        assert np.array_equal(o["z"], z_ref[sl])
        assert np.array_equal(o["y"], y_ref[sl])
