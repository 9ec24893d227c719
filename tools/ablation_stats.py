"""Accuracy and convergence of the non-deterministic / reordered ablations
(DD_EDGE, DD_EDGE_GLOBAL, DD_TREE) against the oracle on the same seeded
inputs: max relative error and max ulp distance of one apply, and the
BiCGSTAB iteration count with the variant as the solver's apply (DESIGN.md
7.2c; the paper reports +-10 % iterations for its atomics).
Writes one JSON line per (case, variant)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2508_04917_b200 as dd  # noqa: E402
from inputs.gen import apply_input, laplacian_bsr3, manufactured_rhs, spe10_style_bsr3  # noqa: E402

CASES = {
    "laplacian_64^3_P2048": (lambda: laplacian_bsr3(64, 64, 64), dict(grid=(64, 64, 64), tiles=(16, 16, 8))),
    "spe10style_60x220x85_P2040": (lambda: spe10_style_bsr3()[:3], dict(grid=(60, 220, 85), tiles=(6, 20, 17))),
}
VARS = {"edge": dd.DD_EDGE, "edge_global": dd.DD_EDGE_GLOBAL, "tree": dd.DD_TREE, "levelset": dd.DD_LEVELSET}


def ulps(a, b):
    ia = a.view(np.int64)
    ib = b.view(np.int64)
    ia = np.where(ia < 0, np.int64(-0x8000000000000000) - ia, ia)
    ib = np.where(ib < 0, np.int64(-0x8000000000000000) - ib, ib)
    return np.abs(ia - ib)


for name, (gen, kw) in CASES.items():
    rp, ci, v = gen()
    S = oracle.setup(rp, ci, v, **kw)
    r = apply_input(S["n"])
    z_ref = oracle.apply(S, r)
    _, b = manufactured_rhs(rp, ci, v)
    br = b.reshape(-1, 3)[S["new_to_old"]].ravel()
    _, rep_o = oracle.bicgstab(S, br, tol=1e-8, max_iter=3000, hist=False)
    for vn, var in VARS.items():
        os.environ["DD_SOLVER_VARIANT"] = vn if vn != "levelset" else "levelset"
        ctx = dd.dd_setup(rp, ci, v, **kw)
        z = torch.empty(3 * S["n"], dtype=torch.float64, device="cuda")
        ctx.apply(torch.from_numpy(r).cuda(), z, var)
        torch.cuda.synchronize()
        zz = z.cpu().numpy()
        its = []
        for rep_i in range(3):  # repeat: the atomics' order varies from run to run
            x = torch.zeros_like(z)
            its.append(ctx.bicgstab(torch.from_numpy(br).cuda(), x, tol=1e-8, max_iter=3000)["iterations"])
        print(json.dumps({"case": name, "variant": vn,
                          "max_rel_err": float(np.abs(zz - z_ref).max() / np.abs(z_ref).max()),
                          "max_ulps": int(ulps(zz, z_ref).max()),
                          "frac_entries_differing": float(np.mean(zz != z_ref)),
                          "iterations": its, "oracle_iterations": rep_o["iterations"]}), flush=True)
        ctx.destroy()
