"""Scalar CSR path measurements on the paper's CSR-sized
workloads: the SPE10-style scalar pressure matrix (60x220x85, 7.78M nnz =
the paper's spe10 count) and a scalar 128^3 Laplacian (rhd-sized, 14.58M
nnz), both with 8192-row subdomains from the BFS partitioner (the paper used
METIS with 8192 rows, Table 5), plus a 256^3 scalar Laplacian large
enough that the factors exceed L2. CUDA events, 256 MB L2 flush between reps.
Context numbers: paper Table 4 (MI210) spe10 / rhd."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2508_04917_b200 as dd
from inputs.gen import laplacian_csr, manufactured_rhs_csr, spe10_style_csr

flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=20):
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


cases = [
    ("spe10_csr_bfs_P8192", lambda: spe10_style_csr()[:3], dict(P=8192, partitioner="bfs"), 1e-6,
     dict(table5_dropped_pct_metis=4.84, n_sub=137, mi210_ms=dict(rocsparse_ILU0=3.22, dag_ec_ILD_U0=0.36,
                                                                  dag_vc_ILDU0_fused=0.68, dag_ec_ILDU0_fused=0.34))),
    ("laplace128_csr_bfs_P8192", lambda: laplacian_csr(128, 128, 128), dict(P=8192, partitioner="bfs"), 1e-8,
     dict(note="rhd-sized (scalar 128^3, 14.58M nnz); paper rhd (real matrix): METIS 256 subdomains, "
               "5.15 % dropped", mi210_ms=dict(rocsparse_ILU0=6.38, dag_ec_ILD_U0=0.55,
                                              dag_vc_ILDU0_fused=1.03, dag_ec_ILDU0_fused=0.51))),
    ("laplace256_csr_geo_P8192", lambda: laplacian_csr(256, 256, 256), dict(grid=(256, 256, 256), tiles=(32, 16, 16)),
     1e-8, dict(note="factors > L2")),
]
only = sys.argv[1:]
for name, gen, kw, tol, paper in cases:
    if only and name not in only:
        continue
    rp, ci, v = gen()
    t0 = time.perf_counter()
    ctx = dd.dd_setup_csr(rp, ci, v, variants=7, **kw)
    setup_s = time.perf_counter() - t0
    st = ctx.stats()
    n = ctx.n_local
    r = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, n)).cuda()
    z = torch.empty_like(r)
    res = dict(case=name, n=n, nnz=st["nnzb_before"], nnz_after=st["nnzb_after"],
               dropped_pct=round(100 * (st["nnzb_before"] - st["nnzb_after"]) / st["nnzb_before"], 2),
               n_sub=st["n_sub"], max_levels_L=st["max_levels_L"], setup_s=round(setup_s, 2),
               launch=ctx.launch_info(), canonical_bytes=st["apply_canonical_bytes"])
    for nm, var in (("levelset", 1), ("spin", 2), ("direct", 4), ("unfused", 8)):
        try:
            res[f"apply_us_{nm}"] = round(1e3 * timeit(lambda: ctx.apply(r, z, var)), 1)
        except dd.DDError as e:
            res[f"apply_us_{nm}"] = e.name
    res["apply_gbs_levelset"] = round(st["apply_canonical_bytes"] / (res["apply_us_levelset"] * 1e-6) / 1e9, 1)
    y = torch.empty_like(r)
    res["spmv_us"] = round(1e3 * timeit(lambda: ctx.spmv(r, y)), 1)
    res["spmv_gbs"] = round(st["spmv_canonical_bytes"] / (res["spmv_us"] * 1e-6) / 1e9, 1)
    xs, b = manufactured_rhs_csr(rp, ci, v)
    lab, n2o = ctx.partition()
    bd = torch.from_numpy(b[n2o].copy()).cuda()
    best = None
    for _ in range(3):
        x = torch.zeros_like(bd)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        rep = ctx.bicgstab(bd, x, tol=tol, max_iter=5000)
        e1.record(); torch.cuda.synchronize()
        best = min(best or 1e30, e0.elapsed_time(e1))
    res.update(tol=tol, solve_ms=round(best, 2), iterations=rep["iterations"], true_rel_resid=rep["true_rel_resid"])
    res["paper"] = paper
    print(json.dumps(res), flush=True)
    ctx.destroy()
