"""One config-3 BiCGSTAB solve for ncu captures of the in-solve kernels
(fused-dot SpMV modes, BLAS-1). Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3, manufactured_rhs
rp, ci, v = laplacian_bsr3(160, 160, 160)
ctx = dd.dd_setup(rp, ci, v, grid=(160, 160, 160), tiles=(16, 16, 8))
_, b = manufactured_rhs(rp, ci, v)
lab, n2o = ctx.partition()
bd = torch.from_numpy(b.reshape(-1, 3)[n2o].ravel().copy()).cuda()
x = torch.zeros_like(bd)
ctx.profile(1)  # batched loop (plain stream launches)
print(ctx.bicgstab(bd, x, tol=1e-8, max_iter=3))
