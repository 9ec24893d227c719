"""Seeded BiCGSTAB breakdown cases (R25, Alg. 1): small dense-pattern
systems (BSR3 blocks or scalar CSR) scaled so that one of the three
breakdown tests of the oracle (|rho| < 1e-30, |sigma| < 1e-30, tau < 1e-30)
fires at the first or a later iteration. The case for each category is the
first (seed, P, scale) in a fixed search order whose ORACLE solve ends in that
category -- the search calls only the oracle and the seeded generators."""
from __future__ import annotations

import numpy as np

import oracle

# (iterations, n_applies) of each category, as the oracle reports them
CATEGORIES = {
    "rho_init": (0.0, 0), "sigma_k1": (0.0, 1), "tau_k1": (0.5, 2),
    "rho_mid": (1.0, 2), "sigma_mid": (1.0, 3), "tau_mid": (1.5, 4),
}
SCALES = [1e-15, 1e-14, 1e-12, 1e0, 1e4, 1e8, 1e12]


def _system(seed, bs):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 4 if bs == 3 else 5))
    m = bs * n
    A = rng.uniform(-1, 1, (m, m))
    A[np.diag_indices(m)] += rng.uniform(0.5, 3, m) * rng.choice([-1, 1], m)
    rp = np.arange(0, n * n + 1, n, dtype=np.int64)
    ci = np.tile(np.arange(n, dtype=np.int32), n)
    v = A.reshape(n, bs, n, bs).transpose(0, 2, 1, 3).reshape(-1).copy()
    return rng, n, rp, ci, v


def find_case(category, bs, max_iter=12, seeds=range(400)):
    want = CATEGORIES[category]
    for seed in seeds:
        rng, n, rp, ci, v = _system(seed, bs)
        for P in (1, n):
            try:
                S = oracle.setup(rp, ci, v, P=P) if bs == 3 else oracle.setup_csr(rp, ci, v, P=P)
            except oracle.OracleError:
                continue
            for sc in SCALES:
                b = rng.uniform(-1, 1, bs * n) * sc
                br = b.reshape(-1, bs)[S["new_to_old"]].ravel()
                x, rep = oracle.bicgstab(S, br, tol=1e-300, max_iter=max_iter)
                if rep["status"] == 1 and (rep["iterations"], rep["n_applies"]) == want:
                    return dict(rp=rp, ci=ci, v=v, P=P, b=br, S=S, x=x, rep=rep, seed=seed, scale=sc)
    return None
