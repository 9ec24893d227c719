"""Small end-to-end run for compute-sanitizer (memcheck / synccheck): every
apply variant, SpMV, BiCGSTAB (CUDA graph), the scalar CSR path, and a
world-2 DD_COMM_LOCAL solve with the fused halo and merged reduction."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import random_block_grid, laplacian_csr, apply_input, manufactured_rhs, random_block_stencil27

_held = []


def one(rp, ci, v, kw, csr=False):
    ctx = (dd.dd_setup_csr if csr else dd.dd_setup)(rp, ci, v, variants=7 | (0 if csr else dd.DD_ILU0),
                                                     enable_refactor=not csr and os.environ.get("SAN_REFACTOR") == "1",
                                                     **kw)
    bs = 1 if csr else 3
    r = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, bs * ctx.n_local)).cuda()
    z = torch.empty_like(r)
    for var in [int(q) for q in os.environ.get("SAN_VARS", "1,2,4,8").split(",") if q]:
        try:
            ctx.apply(r, z, var)
        except dd.DDError:
            pass
    if os.environ.get("SAN_SPMV", "1") == "1":
        ctx.spmv(r, z)
    if not csr and os.environ.get("SAN_REFACTOR", "0") == "1":
        ctx.refactor(torch.from_numpy(v).cuda())  # k_refactor9 (dd_setup already ran it once)
    x = torch.zeros_like(r)
    rep = ctx.bicgstab(r, x, tol=1e-8, max_iter=200)
    torch.cuda.synchronize()
    if os.environ.get("SAN_KEEP", "0") == "1":
        _held.append((ctx, r, z, x))
    else:
        ctx.destroy()
    return rep["iterations"]

CASES = {
    "1": lambda: one(*random_block_grid(12, 10, 8, seed=3), dict(grid=(12, 10, 8), tiles=(6, 5, 4))),
    "2": lambda: one(*random_block_grid(10, 10, 10, seed=5), dict(P=77)),
    "3": lambda: one(*random_block_stencil27(8, 8, 8, seed=31), dict(grid=(8, 8, 8), tiles=(4, 4, 4))),
    "4": lambda: one(*laplacian_csr(16, 16, 16), dict(P=512, partitioner="bfs"), csr=True),
}
for c in os.environ.get("SAN_CASES", "1,2,3,4").split(","):
    print(c, CASES[c](), flush=True)
if os.environ.get("SAN_WORLD2", "1") != "1":
    sys.exit(0)
rp, ci, v = random_block_grid(16, 12, 10, seed=21)
key = os.urandom(128)
out = [None, None]
def rank(q):
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ctx = dd.dd_setup(rp, ci, v, grid=(16, 12, 10), tiles=(8, 6, 5), rank=q, world=2, nccl_id=key, comm="local")
        b = torch.ones(3 * ctx.n_local, dtype=torch.float64, device="cuda")
        x = torch.zeros_like(b)
        out[q] = ctx.bicgstab(b, x, tol=1e-8, max_iter=200, stream=st)["iterations"]
        st.synchronize()
        ctx.destroy()
ts = [threading.Thread(target=rank, args=(q,)) for q in range(2)]
[t.start() for t in ts]; [t.join() for t in ts]
print("world2", out)
