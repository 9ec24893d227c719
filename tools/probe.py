"""Quick GPU probe: per-variant apply / SpMV timing at a config (CUDA events,
L2 flushed between reps), plus one BiCGSTAB solve. Development aid."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3, apply_input, manufactured_rhs, spe10_style_bsr3

ap = argparse.ArgumentParser()
ap.add_argument("--grid", default="160,160,160")
ap.add_argument("--tiles", default="16,16,8")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--solve", type=int, default=1)
ap.add_argument("--spe10", type=int, default=0)
ap.add_argument("--stencil27", type=int, default=0, help="1: random 27-point BSR3 (general-K record path)")
ap.add_argument("--warm", type=int, default=0, help="1: no L2 flush between reps (L2-warm)")
a = ap.parse_args()
grid = tuple(map(int, a.grid.split(","))); tiles = tuple(map(int, a.tiles.split(","))) if a.tiles != "auto" else "auto"
t = time.time()
if a.spe10:
    rp, ci, v, _ = spe10_style_bsr3(*grid)
elif a.stencil27:
    from inputs.gen import random_block_stencil27
    rp, ci, v = random_block_stencil27(*grid, seed=41)
else:
    rp, ci, v = laplacian_bsr3(*grid)
print("gen", time.time() - t, flush=True)
t = time.time()
ctx = dd.dd_setup(rp, ci, v, grid=grid, tiles=tiles if a.tiles != "auto" else "auto", variants=7 | dd.DD_ILU0)
print("tiles", ctx.tiles, "swizzle", [(ctx.stats()["swizzle"] >> s) & 255 for s in (0, 8, 16, 24)], flush=True)
print("setup", time.time() - t, json.dumps(ctx.stats()), flush=True)
n = ctx.n_local
r = torch.from_numpy(apply_input(n)).cuda(); z = torch.empty_like(r)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
st = ctx.stats()
def timeit(fn, reps):
    ts = []
    for i in range(reps + 3):
        if not a.warm:
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(np.min(ts))
VARS = [(1, "levelset"), (2, "spin"), (4, "direct"), (8, "unfused"), (16, "edge"), (32, "edge_global"),
        (128, "direct_glob"), (64, "ilu0"), (512, "tree")]
if os.environ.get("PROBE_LOWER", "1") == "1":  # Table 3 analogue: the lower sweep alone
    VARS += [(v | dd.DD_LOWER, n + "+L") for v, n in VARS]
for var, name in VARS:
    try:
        med, mn = timeit(lambda: ctx.apply(r, z, var), a.reps)
    except dd.DDError as e:
        print(f"apply {name:9s} unavailable: {e}", flush=True)
        continue
    print(f"apply {name:13s} median {med*1e3:8.1f} us  min {mn*1e3:8.1f} us  canonical {st['apply_canonical_bytes']/med/1e6:7.1f} GB/s  slab {st['slab_bytes_levelset']/med/1e6:7.1f} GB/s  launch {ctx.launch_info(var)}", flush=True)
y = torch.empty_like(r)
med, mn = timeit(lambda: ctx.spmv(r, y), a.reps)
print(f"spmv median {med*1e3:.1f} us  canonical {st['spmv_canonical_bytes']/med/1e6:.1f} GB/s", flush=True)
if a.solve:
    _, b = manufactured_rhs(rp, ci, v)
    lab, n2o = ctx.partition()
    br = torch.from_numpy(b.reshape(-1, 3)[n2o].ravel().copy()).cuda()
    for i in range(2):
        x = torch.zeros_like(br)
        torch.cuda.synchronize(); t = time.time()
        rep = ctx.bicgstab(br, x, tol=1e-8, max_iter=3000)
        print("bicgstab", json.dumps(rep), "wall ms", (time.time() - t) * 1e3, flush=True)
