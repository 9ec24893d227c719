"""Multi-PROCESS device path (one process per rank, as under torchrun) on the
single GPU of this pool: world 2 and 3 over the peer-memory transport
DD_COMM_IPC -- mailboxes mapped with CUDA IPC handles, halo rows stored by the
apply epilogue into the peer's ghost block, dot partials published with
release/acquire flags, the solve as one CUDA graph per rank. The processes'
kernels time-slice on the one GPU, so these runs are slow but exercise the
exact code an 8-GPU box runs (only the peer addresses differ).

Parity bars as for world 1: apply and halo SpMV bitwise vs the oracle,
iterations equal on every rank and within +-2 of the oracle (equal to the
world-1 count on the Laplacian), the assembled solution solves A x = b.
The NCCL transport needs one GPU per rank: with two ranks on one GPU NCCL
refuses the communicator, and every rank must fail cleanly with DD_E_NCCL
(no hang) -- that checks the status agreement path of dd_setup.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from inputs.gen import apply_input, manufactured_rhs
from tests.mp_worker import CASES

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "mp_worker.py")


def run_world(case, world, comm, tmp_path, timeout=600, key=None):
    key = key or os.urandom(128).hex()
    outs = [str(tmp_path / f"r{q}.npz") for q in range(world)]
    env = dict(os.environ, DD_PEER_TIMEOUT_S="240")
    procs = [subprocess.Popen([sys.executable, WORKER, case, str(world), str(q), comm, key, outs[q]], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for q in range(world)]
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=timeout)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for q, p in enumerate(procs):
        assert p.returncode == 0, f"rank {q} exited {p.returncode}:\n{logs[q][-3000:]}"
    return [dict(np.load(o, allow_pickle=False)) for o in outs]


@pytest.mark.parametrize("case,world", [("laplace_16^3", 2), ("random_8sub", 3), ("chunks_ragged_oddP", 2),
                                        ("spe10_small", 2)])
def test_ipc_world_parity(case, world, tmp_path):
    gen, kw = CASES[case]
    rp, ci, v = gen()
    S = oracle.setup(rp, ci, v, **kw)
    N = S["n"]
    r = apply_input(N)
    z_ref = oracle.apply(S, r)
    y_ref = oracle.spmv(S["rp_r"], S["ci_r"], S["v_r"], r)
    y2_ref = oracle.spmv(S["rp_r"], S["ci_r"], S["v_r"], z_ref)
    xs, b = manufactured_rhs(rp, ci, v)
    b_re = b.reshape(-1, 3)[S["new_to_old"]].ravel()
    _, rep_ref = oracle.bicgstab(S, b_re, tol=1e-8, max_iter=2000)
    res = run_world(case, world, "ipc", tmp_path)
    assert all(str(q["status"]) == "DD_OK" for q in res), [str(q.get("msg", q["status"])) for q in res]
    z = np.concatenate([q["z"] for q in res])
    y = np.concatenate([q["y"] for q in res])
    y2 = np.concatenate([q["y2"] for q in res])
    assert sum(int(q["n"]) for q in res) == N
    assert np.array_equal(z, z_ref), "apply not bitwise"
    assert np.array_equal(y, y_ref), "halo SpMV not bitwise"
    assert np.array_equal(y2, y2_ref), "second halo SpMV not bitwise"
    its = [float(q["iterations"]) for q in res]
    assert len(set(its)) == 1, its
    assert abs(its[0] - rep_ref["iterations"]) <= 2, (its, rep_ref["iterations"])
    assert all(float(q["iterations_host"]) == its[0] for q in res)
    x = np.concatenate([q["x"] for q in res])
    A = __import__("tests.helpers", fromlist=["bsr"]).bsr(S["rp_r"], S["ci_r"], S["v_r"])
    assert np.linalg.norm(A @ x - b_re) <= 1e-7 * np.linalg.norm(b_re)
    # dd_solve_host: every rank wrote its rows of the original-order solution,
    # the same solve as dd_bicgstab from x0 = 0 -> bitwise the permuted x
    xh = np.zeros(3 * N)
    n2o = S["new_to_old"]
    for q in res:
        f, n = int(q["first"]), int(q["n"])
        rows = n2o[f:f + n]
        xh.reshape(-1, 3)[rows] = q["xh"].reshape(-1, 3)[rows]
    x_orig = np.zeros(3 * N)
    x_orig.reshape(-1, 3)[n2o] = x.reshape(-1, 3)
    assert np.array_equal(xh, x_orig)
    # the manufactured solution, to the accuracy the tolerance allows for this
    # conditioning (SPE10-style: ~7 decades of permeability contrast)
    assert np.linalg.norm(xh - xs) <= (1e-3 if case.startswith("spe10") else 1e-6) * np.linalg.norm(xs)


def test_ipc_iterations_equal_world1_laplacian(tmp_path):
    """Rank-order double-double dots: the world-2 solve takes the world-1
    iteration count and the same residual history to 1e-12."""
    import torch
    import paper_2508_04917_b200 as dd
    gen, kw = CASES["laplace_16^3"]
    rp, ci, v = gen()
    ctx = dd.dd_setup(rp, ci, v, **kw)
    _, b = manufactured_rhs(rp, ci, v)
    lab, n2o = ctx.partition()
    b_re = torch.from_numpy(b.reshape(-1, 3)[n2o].ravel().copy()).cuda()
    x = torch.zeros_like(b_re)
    rep1 = ctx.bicgstab(b_re, x, tol=1e-8, max_iter=2000, hist=True)
    ctx.destroy()
    res = run_world("laplace_16^3", 2, "ipc", tmp_path)
    assert float(res[0]["iterations"]) == rep1["iterations"]
    h = res[0]["hist"][:len(rep1["resid_hist"])]
    assert np.allclose(h, rep1["resid_hist"], rtol=1e-12, atol=0)


def test_nccl_two_ranks_one_gpu_fail_cleanly(tmp_path):
    """NCCL cannot put two ranks on one GPU: both ranks must return the same
    clean error (status agreed, no rank left waiting)."""
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("two GPUs: the NCCL transport itself is tested by test_nccl_world2_parity")
    key = __import__("paper_2508_04917_b200").dd_nccl_unique_id().hex()
    outs = [str(tmp_path / f"n{q}.npz") for q in range(2)]
    procs = [subprocess.Popen([sys.executable, WORKER, "laplace_16^3", "2", str(q), "nccl", key, outs[q]],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for q in range(2)]
    try:
        logs = [p.communicate(timeout=300)[0] for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    res = [dict(np.load(o)) for o in outs]
    st = [str(q["status"]) for q in res]
    assert st[0] == st[1], (st, logs)
    # either NCCL accepted the shared GPU (then the run must be correct) or it failed cleanly
    assert st[0] in ("DD_OK", "DD_E_NCCL"), (st, [str(q.get("msg")) for q in res])


def test_nccl_world2_parity(tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (one NCCL rank per GPU)")
    key = __import__("paper_2508_04917_b200").dd_nccl_unique_id().hex()
    res = run_world("laplace_16^3", 2, "nccl", tmp_path, key=key)
    assert all(str(q["status"]) == "DD_OK" for q in res), [str(q.get("msg")) for q in res]
    gen, kw = CASES["laplace_16^3"]
    rp, ci, v = gen()
    S = oracle.setup(rp, ci, v, **kw)
    r = apply_input(S["n"])
    assert np.array_equal(np.concatenate([q["z"] for q in res]), oracle.apply(S, r))
    assert np.array_equal(np.concatenate([q["y"] for q in res]), oracle.spmv(S["rp_r"], S["ci_r"], S["v_r"], r))
    assert res[0]["iterations"] == res[1]["iterations"]


def test_ipc_setup_status_agreed(tmp_path):
    """The same agreement across PROCESSES (DD_COMM_IPC): one rank's singular
    pivot fails both ranks with DD_E_SINGULAR_PIVOT, neither hangs."""
    key = os.urandom(128).hex()
    outs = [str(tmp_path / f"s{q}.npz") for q in range(2)]
    procs = [subprocess.Popen([sys.executable, WORKER, "singular_rank1", "2", str(q), "ipc", key, outs[q]],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for q in range(2)]
    try:
        logs = [p.communicate(timeout=300)[0] for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    res = [dict(np.load(o)) for o in outs]
    assert [str(q["status"]) for q in res] == ["DD_E_SINGULAR_PIVOT"] * 2, ([str(q.get("msg")) for q in res], logs)


def test_ipc_fused_halo_equals_plain_exchange(tmp_path):
    """The fused halo (rows stored by the apply epilogue into the peer's
    ghost block over the IPC mapping) against the plain exchange (gather
    kernel + put) across processes: identical iterates, bitwise."""
    old = os.environ.get("DD_HALO_FUSE")
    try:
        os.environ["DD_HALO_FUSE"] = "0"
        plain = run_world("random_8sub", 2, "ipc", tmp_path)
    finally:
        if old is None:
            os.environ.pop("DD_HALO_FUSE", None)
        else:
            os.environ["DD_HALO_FUSE"] = old
    fused = run_world("random_8sub", 2, "ipc", tmp_path)
    for a, b in zip(plain, fused):
        assert np.array_equal(a["x"], b["x"]) and float(a["iterations"]) == float(b["iterations"])
        assert np.array_equal(a["hist"], b["hist"])
