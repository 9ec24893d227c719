"""Where the level-set apply's time goes (development aid; needs a -DDD_TRACE
build, e.g. tools/ab_build.sh trace -DDD_TRACE, then DD_LIB=exp/trace.so).

Per-CTA cycle counters of k_apply_ring (consumer warp 0 and the releasing
warp, producer lane), averaged per subdomain; with --submod K every CTA
streams only the first K subdomains' data (an L2-resident working set), which
times the consumers without the HBM stream."""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3, apply_input, spe10_style_bsr3

ap = argparse.ArgumentParser()
ap.add_argument("--grid", default="160,160,160")
ap.add_argument("--tiles", default="16,16,8")
ap.add_argument("--spe10", type=int, default=0)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--submods", default="0,16,32,64")
a = ap.parse_args()
grid = tuple(map(int, a.grid.split(",")))
tiles = tuple(map(int, a.tiles.split(","))) if a.tiles != "auto" else "auto"
if a.spe10:
    rp, ci, v, _ = spe10_style_bsr3(*grid)
else:
    rp, ci, v = laplacian_bsr3(*grid)
ctx = dd.dd_setup(rp, ci, v, grid=grid, tiles=tiles)
lib = dd.lib()
f = lib.dd_debug_trace
f.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
n = ctx.n_local
r = torch.from_numpy(apply_input(n)).cuda()
z = torch.empty_like(r)
buf = np.zeros((1024, 16), dtype=np.uint64)
li = ctx.launch_info(dd.DD_LEVELSET)
print("launch", li, flush=True)
grid_n = li["grid"] if isinstance(li, dict) else 296
for sm in map(int, a.submods.split(",")):
    f(None, 1, sm)
    for _ in range(3):
        ctx.apply(r, z, dd.DD_LEVELSET)
    torch.cuda.synchronize()
    f(None, 1, -1)
    ts = []
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); ctx.apply(r, z, dd.DD_LEVELSET); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    f(buf.ctypes.data, 1, 0)
    b = buf[:grid_n].astype(np.float64)
    nsub = b[:, 6].sum()
    per = lambda k: b[:, k].sum() / nsub
    tot = per(0) + per(1) + per(2) + per(3)
    print(f"submod {sm:3d}: apply median {np.median(ts)*1e3:7.1f} us | cycles per subdomain (warp 0): "
          f"total {tot:8.0f} rfill {per(0):7.0f} L {per(1):7.0f} U {per(2):7.0f} zstore {per(3):6.0f} | "
          f"full-wait {per(4):7.0f} bar-wait {per(5):7.0f} | last warp: bar-wait {per(10):7.0f} full-wait {per(11):7.0f} | "
          f"producer: empty-wait {per(8):7.0f} of {per(9):8.0f} | records/sub {b[:, 7].sum() / nsub:.1f}", flush=True)
