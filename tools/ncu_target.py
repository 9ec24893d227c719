"""Small, fixed launch sequence for ncu captures at a bench config:
N level-set applies, N SpMVs, N spin and direct applies (no timing here).
Optional third argument: only that apply variant (levelset | spin | direct),
N launches of it (config 2 spin vs level-set captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3, apply_input, spe10_style_bsr3

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if cfg == "cfg3":
    grid, tiles = (160, 160, 160), (16, 16, 8)
    rp, ci, v = laplacian_bsr3(*grid)
elif cfg in ("cfg2a", "cfg2b"):
    grid, tiles = (64, 64, 64), ((16, 16, 8) if cfg == "cfg2a" else (32, 16, 16))
    rp, ci, v = laplacian_bsr3(*grid)
elif cfg == "cfg4":
    grid, tiles = (60, 220, 85), (10, 20, 17)
    rp, ci, v, _ = spe10_style_bsr3(*grid)
ctx = dd.dd_setup(rp, ci, v, grid=grid, tiles=tiles, variants=7)
r = torch.from_numpy(apply_input(ctx.n_local)).cuda()
z = torch.empty_like(r)
only = sys.argv[3] if len(sys.argv) > 3 else None
if only:
    var = {"levelset": dd.DD_LEVELSET, "spin": dd.DD_SPINLOOP, "direct": dd.DD_DIRECT}[only]
    for _ in range(n):
        ctx.apply(r, z, var)
    torch.cuda.synchronize()
    print("done", only, ctx.launch_info(var))
    sys.exit(0)
for _ in range(n):
    ctx.apply(r, z, dd.DD_LEVELSET)
for _ in range(n):
    ctx.spmv(r, z)
for _ in range(2):
    ctx.apply(r, z, dd.DD_DIRECT)
for _ in range(2):
    ctx.apply(r, z, dd.DD_SPINLOOP)
torch.cuda.synchronize()
print("done", ctx.launch_info(dd.DD_LEVELSET))
