"""Launch sequence for ncu captures of dd_refactor at config 3 (160^3, P 2048):
dd_setup with enable_refactor (device values), then N dd_refactor calls.
Development aid; prints the wall time per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
grid, tiles = (160, 160, 160), (16, 16, 8)
rp, ci, v = laplacian_bsr3(*grid)
ctx = dd.dd_setup(rp, ci, v, grid=grid, tiles=tiles, enable_refactor=True)
vd = torch.from_numpy(v.reshape(-1)).cuda()
for i in range(n):
    torch.cuda.synchronize()
    t = time.perf_counter()
    ctx.refactor(vd)
    print("refactor ms", 1e3 * (time.perf_counter() - t), flush=True)
