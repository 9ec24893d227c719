"""One config-3 solve setup, then timed solves with and without dd_profile (dev aid)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3, manufactured_rhs
grid, tiles = (160, 160, 160), (16, 16, 8)
rp, ci, v = laplacian_bsr3(*grid)
_, b = manufactured_rhs(rp, ci, v)
ctx = dd.dd_setup(rp, ci, v, grid=grid, tiles=tiles)
bd = torch.empty(3 * ctx.n_local + 2, dtype=torch.float64, device="cuda"); ctx.permute(b, bd)
x = torch.zeros_like(bd)
for _ in range(2): x.zero_(); ctx.bicgstab(bd, x)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): x.zero_(); rep = ctx.bicgstab(bd, x)
e1.record(); torch.cuda.synchronize()
ctx.profile(1)
for _ in range(2): x.zero_(); ctx.bicgstab(bd, x)
p = ctx.profile(0)
tag = " ".join(f"{k}={os.environ[k]}" for k in sorted(os.environ) if k.startswith("DD_"))
print(f"{tag:40s} solve {e0.elapsed_time(e1)/5:.2f} ms  its {rep['iterations']}  apply {p['apply_ms']/p['n_apply']*1e3:.1f} us  spmv {p['spmv_ms']/p['n_spmv']*1e3:.1f} us  blas/solve {p['blas_ms']/2:.2f} ms", flush=True)
