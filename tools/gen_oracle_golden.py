"""Writes tests/golden/oracle_bicgstab.json: the ORACLE's own BiCGSTAB
iteration counts on the benchmark configurations (calls only oracle/ and
inputs/; no CUDA path). Used by bench.py --impl reference to scale its bounded
per-iteration sample to a full solve, and by GPU tests as a stored pin."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from inputs.gen import laplacian_bsr3, manufactured_rhs, spe10_style_bsr3

CONFIGS = {
    "cfg3_laplacian160_P2048": dict(kind="laplacian", grid=(160, 160, 160), tiles=(16, 16, 8), tol=1e-8),
    "cfg4_spe10style_P3400": dict(kind="spe10", grid=(60, 220, 85), tiles=(10, 20, 17), tol=1e-8),
    "cfg4_spe10style_P3400_tol1e-6": dict(kind="spe10", grid=(60, 220, 85), tiles=(10, 20, 17), tol=1e-6),
    "cfg2a_laplacian64_P2048": dict(kind="laplacian", grid=(64, 64, 64), tiles=(16, 16, 8), tol=1e-8),
}

def main(names):
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "oracle_bicgstab.json")
    res = json.load(open(out_path)) if os.path.exists(out_path) else {
        "source": "written by tools/gen_oracle_golden.py (oracle only); manufactured rhs b = A x*, x* ~ U[0,1) seed 1, x0 = 0"}
    for name in names:
        c = CONFIGS[name]
        if c["kind"] == "laplacian":
            rp, ci, v = laplacian_bsr3(*c["grid"])
        else:
            rp, ci, v, _ = spe10_style_bsr3(*c["grid"])
        S = oracle.setup(rp, ci, v, grid=c["grid"], tiles=c["tiles"])
        _, b = manufactured_rhs(rp, ci, v, seed=1)
        br = b.reshape(-1, 3)[S["new_to_old"]].ravel()
        t = time.time()
        _, rep = oracle.bicgstab(S, br, tol=c["tol"], max_iter=5000, hist=False)
        rep["oracle_seconds"] = time.time() - t
        rep["threads"] = oracle.get_threads()
        rep.update({k: list(v) if isinstance(v, tuple) else v for k, v in c.items()})
        res[name] = rep
        print(name, rep, flush=True)
        json.dump(res, open(out_path, "w"), indent=1)

if __name__ == "__main__":
    main(sys.argv[1:] or list(CONFIGS))
