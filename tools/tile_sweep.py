"""Design space: subdomain shape at 160^3 -> apply time, launch
shape, BiCGSTAB iterations and time-to-solution (dev/measurement aid)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3, manufactured_rhs, apply_input
grid = (160, 160, 160)
rp, ci, v = laplacian_bsr3(*grid)
_, b = manufactured_rhs(rp, ci, v)
for tiles in [tuple(map(int, t.split("x"))) for t in sys.argv[1:]]:
    ctx = dd.dd_setup(rp, ci, v, grid=grid, tiles=tiles)
    bd = torch.empty(3 * ctx.n_local + 2, dtype=torch.float64, device="cuda"); ctx.permute(b, bd)
    x = torch.zeros_like(bd)
    x.zero_(); rep = ctx.bicgstab(bd, x)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): x.zero_(); rep = ctx.bicgstab(bd, x)
    e1.record(); torch.cuda.synchronize()
    ctx.profile(1); x.zero_(); ctx.bicgstab(bd, x); p = ctx.profile(0)
    st = ctx.stats()
    print(json.dumps(dict(tiles=tiles, P=int(np.prod(tiles)), n_sub=st["n_sub"], levels=st["max_levels_L"],
                          nnzb_after=st["nnzb_after"], iterations=rep["iterations"], solve_ms=round(e0.elapsed_time(e1) / 3, 2),
                          apply_us=round(p["apply_ms"] / p["n_apply"] * 1e3, 1), spmv_us=round(p["spmv_ms"] / p["n_spmv"] * 1e3, 1),
                          apply_gbs=round(st["apply_canonical_bytes"] / (p["apply_ms"] / p["n_apply"]) / 1e6, 1),
                          launch=ctx.launch_info())), flush=True)
    ctx.destroy()
