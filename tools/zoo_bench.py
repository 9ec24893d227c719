"""Apply / SpMV / solve timing for non-7-point workloads (development aid):
27-point random-block BSR3 (general-K record path) and scalar 27-point CSR.
CUDA events, 256 MB L2 flush between reps."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import random_block_stencil27, random_csr_stencil27

flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=10):
    ts = []
    for i in range(reps + 2):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for name, gen, csr, kw in (("bsr3_27pt_96^3_P2048", lambda: random_block_stencil27(96, 96, 96, seed=1), False,
                            dict(grid=(96, 96, 96), tiles=(16, 16, 8))),
                           ("csr_27pt_192^3_P8192", lambda: random_csr_stencil27(192, 192, 192, seed=2), True,
                            dict(grid=(192, 192, 192), tiles=(32, 16, 16)))):
    rp, ci, v = gen()
    ctx = (dd.dd_setup_csr if csr else dd.dd_setup)(rp, ci, v, variants=7, **kw)
    st = ctx.stats()
    m = ctx.bs * ctx.n_local
    r = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, m)).cuda()
    z = torch.empty_like(r)
    res = dict(case=name, n=ctx.n_local, nnzb=st["nnzb_before"], levels_L=st["max_levels_L"], launch=ctx.launch_info())
    for nm, var in (("levelset", 1), ("direct", 4)):
        res["apply_us_" + nm] = round(1e3 * timeit(lambda: ctx.apply(r, z, var)), 1)
    res["apply_gbs"] = round(st["apply_canonical_bytes"] / (res["apply_us_levelset"] * 1e-6) / 1e9, 1)
    y = torch.empty_like(r)
    res["spmv_us"] = round(1e3 * timeit(lambda: ctx.spmv(r, y)), 1)
    res["spmv_gbs"] = round(st["spmv_canonical_bytes"] / (res["spmv_us"] * 1e-6) / 1e9, 1)
    print(json.dumps(res), flush=True)
    ctx.destroy()
