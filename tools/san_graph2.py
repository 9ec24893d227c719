"""compute-sanitizer probe: two contexts in sequence, each with a CUDA-graph
solve; KEEP=1 keeps the first alive while the second solves."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import random_block_grid
keep = os.environ.get("KEEP", "0") == "1"
same = os.environ.get("SAME", "0") == "1"
held = []
for k, (gen, kw) in enumerate([(lambda: random_block_grid(12, 10, 8, seed=3), dict(grid=(12, 10, 8), tiles=(6, 5, 4))),
                               ((lambda: random_block_grid(12, 10, 8, seed=3), dict(grid=(12, 10, 8), tiles=(6, 5, 4))) if same else
                                (lambda: random_block_grid(10, 10, 10, seed=5), dict(P=77)))]):
    rp, ci, v = gen()
    ctx = dd.dd_setup(rp, ci, v, variants=int(os.environ.get("VARS", "1")), **kw)
    r = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, 3 * ctx.n_local)).cuda()
    if os.environ.get("ZALLOC", "0") == "1":
        z = torch.empty_like(r)
    x = torch.zeros_like(r)
    rep = ctx.bicgstab(r, x, tol=1e-8, max_iter=200)
    torch.cuda.synchronize()
    print(k, rep["iterations"], flush=True)
    if keep:
        held.append(ctx)
    else:
        ctx.destroy()
