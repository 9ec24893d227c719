import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import random_block_grid
rp, ci, v = random_block_grid(10, 10, 10, seed=5)
ctx = dd.dd_setup(rp, ci, v, variants=7, P=77)
print("solver variant", ctx.solver_variant(), flush=True)
r = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, 3 * ctx.n_local)).cuda()
x = torch.zeros_like(r)
rep = ctx.bicgstab(r, x, tol=1e-8, max_iter=200)
torch.cuda.synchronize()
print(rep["iterations"], flush=True)
