"""dd_setup phase trace at config 3 (DD_SETUP_TRACE=1 prints the host and device
phases on stderr). Development aid. Argument: "auto" for dd_setup's tile choice."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3
tiles = "auto" if len(sys.argv) > 1 and sys.argv[1] == "auto" else (16, 16, 8)
rp, ci, v = laplacian_bsr3(160, 160, 160)
for i in range(2):
    t = time.perf_counter()
    ctx = dd.dd_setup(rp, ci, v, grid=(160, 160, 160), tiles=tiles, enable_refactor=True)
    st = ctx.stats()
    print("setup s", time.perf_counter() - t, ctx.tiles, {k: round(st[k], 1) for k in dd.Context.SETUP_KEYS if k in st},
          flush=True)
    ctx.destroy()
