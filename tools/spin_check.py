import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd, oracle
from inputs.gen import laplacian_bsr3, apply_input
g = int(sys.argv[1]) if len(sys.argv) > 1 else 32
grid, tiles = (g, g, g), (16, 16, 8)
rp, ci, v = laplacian_bsr3(*grid)
ctx = dd.dd_setup(rp, ci, v, grid=grid, tiles=tiles)
print(ctx.launch_info(dd.DD_SPINLOOP), flush=True)
S = oracle.setup(rp, ci, v, grid=grid, tiles=tiles)
r = apply_input(ctx.n_local); zr = oracle.apply(S, r)
rd = torch.from_numpy(r).cuda(); z = torch.zeros_like(rd)
ctx.apply(rd, z, dd.DD_SPINLOOP); torch.cuda.synchronize()
print("spin equal:", np.array_equal(z.cpu().numpy(), zr), flush=True)
