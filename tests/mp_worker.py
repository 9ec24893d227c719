"""One rank of the multi-process GPU tests (tests/test_gpu_multiproc.py).

python tests/mp_worker.py CASE WORLD RANK COMM KEYHEX OUT.npz

Every rank builds the same seeded inputs, runs dd_setup (collective), one
apply of its slice of r, one halo SpMV, a BiCGSTAB solve and dd_solve_host,
and saves its results (or the error status) for the parent to compare with
the oracle. No oracle code runs here.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from inputs.gen import (apply_input, laplacian_bsr3, manufactured_rhs, random_block_grid,  # noqa: E402
                        spe10_style_bsr3)

def _singular_rank1():
    """random 8x8x4 grid, one diagonal block of the last chunk (rank 1) zeroed"""
    rp, ci, v = random_block_grid(8, 8, 4, seed=13)
    v = v.reshape(-1, 3, 3).copy()
    row = rp.shape[0] - 1 - 64  # first row of the last chunk: U_ii = A_ii (lower couplings dropped)
    diag = next(p for p in range(rp[row], rp[row + 1]) if ci[p] == row)
    v[diag] = 0.0
    return rp, ci, v.reshape(-1)


CASES = {
    "singular_rank1": (_singular_rank1, dict(P=64)),
    "laplace_16^3": (lambda: laplacian_bsr3(16, 16, 16), dict(grid=(16, 16, 16), tiles=(8, 8, 8))),
    "random_8sub": (lambda: random_block_grid(16, 12, 10, seed=21), dict(grid=(16, 12, 10), tiles=(8, 6, 5))),
    "chunks_ragged_oddP": (lambda: random_block_grid(10, 10, 10, seed=5), dict(P=77)),
    "spe10_small": (lambda: spe10_style_bsr3(20, 40, 20, upper_ness_from=10)[:3],
                    dict(grid=(20, 40, 20), tiles=(10, 20, 10))),
}


def main():
    case, world, rank, comm, keyhex, out = sys.argv[1:7]
    world, rank = int(world), int(rank)
    import torch
    import paper_2508_04917_b200 as dd
    dev = rank % torch.cuda.device_count()  # one GPU per rank when there are enough
    torch.cuda.set_device(dev)
    gen, kw = CASES[case]
    rp, ci, v = gen()
    N = rp.shape[0] - 1
    res = {}
    try:
        ctx = dd.dd_setup(rp, ci, v, rank=rank, world=world, nccl_id=bytes.fromhex(keyhex), comm=comm,
                          device=dev, **kw)
        f, n = ctx.row_first, ctx.n_local
        sl = slice(3 * f, 3 * (f + n))
        res["first"], res["n"] = f, n
        r = torch.from_numpy(apply_input(N)[sl].copy()).cuda()
        z, y = torch.empty_like(r), torch.empty_like(r)
        ctx.apply(r, z)
        ctx.spmv(r, y)
        ctx.spmv(z, r)  # a second exchange on the same ghost block
        torch.cuda.synchronize()
        res["z"], res["y"], res["y2"] = z.cpu().numpy(), y.cpu().numpy(), r.cpu().numpy()
        _, b = manufactured_rhs(rp, ci, v)
        lab, n2o = ctx.partition()
        b_re = b.reshape(-1, 3)[n2o].ravel()
        bl = torch.from_numpy(b_re[sl].copy()).cuda()
        x = torch.zeros_like(bl)
        rep = ctx.bicgstab(bl, x, tol=1e-8, max_iter=2000, hist=True)
        res["x"] = x.cpu().numpy()
        res["hist"] = rep["resid_hist"]
        res["iterations"] = rep["iterations"]
        res["n_applies"] = rep["n_applies"]
        res["true_rel_resid"] = rep["true_rel_resid"]
        xh = np.zeros(3 * N)
        rep2 = ctx.solve_host(b, xh, tol=1e-8, max_iter=2000)
        res["xh"] = xh
        res["iterations_host"] = rep2["iterations"]
        res["status"] = "DD_OK"
        ctx.destroy()
    except dd.DDError as e:
        res["status"] = e.name
        res["msg"] = str(e)
    np.savez(out, **{k: np.asarray(val) for k, val in res.items()})


if __name__ == "__main__":
    main()
