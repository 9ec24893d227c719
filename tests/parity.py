"""Shared parity checks: the product's setup (read back through the C ABI
introspection calls) against the oracle's setup, bit for bit."""
from __future__ import annotations

import numpy as np


def oracle_local_factors(S, row_first, n_local):
    """The oracle's L / U_unit / Dinv restricted to reordered rows
    [row_first, row_first + n_local), columns shifted to local numbering."""
    rp, ci = S["rp_d"], S["ci_d"]
    n = S["n"]
    b2 = S.get("bs", 3) ** 2
    rows = np.repeat(np.arange(n), np.diff(rp))
    sel = (rows >= row_first) & (rows < row_first + n_local)
    lo = (ci < rows) & sel
    up = (ci > rows) & sel
    out = {}
    for key, mask, vals in (("L", lo, S["lu"]), ("U", up, S["uunit"])):
        r = rows[mask] - row_first
        out[key + "rp"] = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=n_local))]).astype(np.int64)
        out[key + "ci"] = (ci[mask] - row_first).astype(np.int32)
        out[key + "v"] = vals.reshape(-1, b2)[mask].ravel()
    out["Dinv"] = S["dinv"][b2 * row_first:b2 * (row_first + n_local)]
    return out


def assert_setup_bitwise(ctx, S):
    """Partition, permutation, level sets and factor pattern bit-exact; factor
    values equal to the last bit (0 ulps)."""
    lab, n2o = ctx.partition()
    assert np.array_equal(lab, S["labels"]), "labels differ"
    assert np.array_equal(n2o, S["new_to_old"]), "permutation differs"
    a, n = ctx.row_first, ctx.n_local
    assert np.array_equal(ctx.levels("L"), S["hmapL"][a:a + n]), "hmapL differs"
    assert np.array_equal(ctx.levels("U"), S["hmapU"][a:a + n]), "hmapU differs"
    f = ctx.factors()
    ref = oracle_local_factors(S, a, n)
    for k in ("Lrp", "Lci", "Urp", "Uci"):
        assert np.array_equal(f[k], ref[k]), f"{k} (pattern) differs"
    for k in ("Lv", "Uv", "Dinv"):
        assert np.array_equal(f[k], ref[k]), f"{k} (values) differ; max |d| = {np.abs(f[k] - ref[k]).max()}"
    st = ctx.stats()
    assert st["nnzb_before"] == S["rp_r"][-1] and st["nnzb_after"] == S["rp_d"][-1]
    assert st["n_sub"] == S["n_sub"]
