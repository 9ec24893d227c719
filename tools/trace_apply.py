"""Per-record clock64 trace of CTA 0 of the ring apply kernel (debug)."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3, apply_input
grid, tiles = (160, 160, 160), (16, 16, 8)
rp, ci, v = laplacian_bsr3(*grid)
ctx = dd.dd_setup(rp, ci, v, grid=grid, tiles=tiles, variants=1)
VAR = int(os.environ.get("VAR", "1"))
r = torch.from_numpy(apply_input(ctx.n_local)).cuda(); z = torch.empty_like(r)
for _ in range(3): ctx.apply(r, z, VAR)
buf = torch.zeros(4 * 4 * 4096, dtype=torch.int64, device="cuda")
L = dd.lib(); L.dd_debug_trace.argtypes = [ctypes.c_void_p]
L.dd_debug_trace(buf.data_ptr()); ctx.apply(r, z, VAR); torch.cuda.synchronize(); L.dd_debug_trace(None)
t = buf.cpu().numpy().reshape(4096, 4, 4)
n = int((t[:, 0, 0] != 0).sum())
t = t[:n]
w = (t[:, 0, 3] >> 48) & 0xFFF
up = (t[:, 0, 3] >> 60) & 1
t3 = t[:, :, 3] & ((1 << 48) - 1)
act = t[:, :, 0] != 0
t0 = np.where(act, t[:, :, 0], np.nan); t1 = np.where(act, t[:, :, 1], np.nan); t2 = np.where(act, t[:, :, 2], np.nan)
t3 = np.where(act, t3, np.nan)
start = np.nanmin(t0, axis=1)
rec_total = np.diff(np.concatenate([start, [np.nanmax(t3[-1])]]))
wait = np.nanmax(t1 - t0, axis=1)       # ensure + header
proc = np.nanmax(t2 - t1, axis=1)       # slowest warp's process_record
procmin = np.nanmin(t2 - t1, axis=1)
bar = np.nanmax(t3, axis=1) - np.nanmax(t2, axis=1)
print("records", n, "total cycles", int(np.nanmax(t3) - start[0]))
print("per record (median cycles): total %.0f  ensure+hdr(max over warps) %.0f  process(max) %.0f process(min) %.0f  barrier-tail %.0f" % (
    np.median(rec_total), np.median(wait), np.median(proc), np.median(procmin), np.median(bar)))
for q in (0, 1):
    m = up == q
    print("U" if q else "L", "records", m.sum(), "median total", np.median(rec_total[m]), "mean", rec_total[m].mean(), "median proc", np.median(proc[m]), "median wait", np.median(wait[m]))
print("first 80 records: w, up, total, wait, proc")
for k in range(min(80, n)):
    print(k, w[k], up[k], int(rec_total[k]), int(wait[k]), int(proc[k]), int(procmin[k]), int(bar[k]))
