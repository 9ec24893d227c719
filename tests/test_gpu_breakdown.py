"""GPU vs oracle on BiCGSTAB breakdowns (R25; Alg. 1): every
breakdown branch of the device-side control (rho at the start and in a later
iteration, sigma, tau) must report the oracle's status, iteration count,
apply count and residual history, and leave the oracle's last iterate in x,
bitwise -- for BSR3 and scalar CSR, with the CUDA-graph loop and the
host-batched loop."""
import numpy as np
import pytest

import paper_2508_04917_b200 as dd
from tests.breakdown_cases import CATEGORIES, find_case

pytestmark = pytest.mark.gpu
BREAK_CODE = {"rho": 1, "sigma": 2, "tau": 3}


@pytest.mark.parametrize("graph", ["1", "0"])
@pytest.mark.parametrize("bs", [3, 1])
@pytest.mark.parametrize("category", list(CATEGORIES))
def test_breakdown_matches_oracle(category, bs, graph, monkeypatch):
    import torch
    monkeypatch.setenv("DD_GRAPH", graph)
    c = find_case(category, bs)
    assert c is not None, f"no seeded case for {category} (bs {bs})"
    ctx = dd.dd_setup(c["rp"], c["ci"], c["v"], P=c["P"], csr=bs == 1)
    if graph == "0":
        ctx.profile(1)  # per-kernel timing forces the host-batched loop
    b = torch.from_numpy(c["b"].copy()).cuda()
    x = torch.zeros_like(b)
    rep = ctx.bicgstab(b, x, tol=1e-300, max_iter=12, hist=True)
    ro = c["rep"]
    assert rep["status_name"] == "DD_E_BREAKDOWN", rep
    assert rep["breakdown"] == BREAK_CODE[category.split("_")[0]], rep
    assert rep["iterations"] == ro["iterations"] and rep["n_applies"] == ro["n_applies"], (rep, ro)
    assert np.array_equal(x.cpu().numpy(), c["x"]), "last iterate differs"
    nh = len(ro["resid_hist"])
    assert np.array_equal(rep["resid_hist"][:nh], ro["resid_hist"]), (rep["resid_hist"][:nh], ro["resid_hist"])
    assert rep["true_rel_resid"] == pytest.approx(ro["true_rel_resid"], rel=1e-12)
    ctx.destroy()
