"""CPU tests of the product library: it loads, exports every symbol include/dd.h
declares, and its host-side setup (run with host_only = 1, no device work)
equals the oracle's setup bit for bit. No compute calls are made here."""
import re
import os

import numpy as np
import pytest

import oracle
import paper_2508_04917_b200 as dd
from inputs.gen import laplacian_bsr3, random_block_grid, spe10_style_bsr3
from tests.helpers import kron_blocks
from tests.parity import assert_setup_bitwise

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="session", autouse=True)
def _built():
    from paper_2508_04917_b200 import build
    build.build()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "dd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dd_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    L = dd.lib()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), f"libdd.so does not export {s}"
    assert sorted(dd.EXPORTS) == syms


def test_no_device_is_an_error_not_a_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    rp, ci, v = laplacian_bsr3(4, 4, 4)
    with pytest.raises(dd.DDError) as e:
        dd.dd_setup(rp, ci, v, P=8)
    assert e.value.name == "DD_E_NO_DEVICE"


CASES = {
    "cfg1_16^3": (lambda: laplacian_bsr3(16, 16, 16), dict(grid=(16, 16, 16), tiles=(8, 8, 8))),
    "cfg2a_64^3": (lambda: laplacian_bsr3(64, 64, 64), dict(grid=(64, 64, 64), tiles=(16, 16, 8))),
    "random_blocks": (lambda: random_block_grid(12, 10, 8, seed=3), dict(grid=(12, 10, 8), tiles=(6, 5, 4))),
    "chunks_ragged_oddP": (lambda: random_block_grid(10, 10, 10, seed=5), dict(P=77)),
    "P1": (lambda: random_block_grid(6, 5, 4, seed=6), dict(P=1)),
    "one_subdomain": (lambda: random_block_grid(9, 8, 7, seed=7), dict(grid=(9, 8, 7), tiles=(9, 8, 7))),
    "spe10_small": (lambda: spe10_style_bsr3(20, 40, 20, upper_ness_from=10)[:3],
                    dict(grid=(20, 40, 20), tiles=(10, 20, 10))),
    "bfs_random": (lambda: random_block_grid(12, 10, 8, seed=13), dict(P=100, partitioner="bfs")),
    "bfs_spe10_small": (lambda: spe10_style_bsr3(20, 40, 20, upper_ness_from=10)[:3], dict(P=1000, partitioner="bfs")),
}


@pytest.mark.parametrize("name", list(CASES))
def test_host_setup_bitwise_vs_oracle(name):
    gen, kw = CASES[name]
    rp, ci, v = gen()
    S = oracle.setup(rp, ci, v, **kw)
    ctx = dd.dd_setup(rp, ci, v, host_only=True, variants=7, **kw)
    assert_setup_bitwise(ctx, S)
    st = ctx.stats()
    # canonical apply bytes: 72(nL+nU+n) + 4(nL+nU) + 8(n+1) + 48n
    n = S["n"]
    rows = np.repeat(np.arange(n), np.diff(S["rp_d"]))
    nLU = int(np.sum(S["ci_d"] != rows))
    assert st["apply_canonical_bytes"] == 72 * (nLU + n) + 4 * nLU + 8 * (n + 1) + 48 * n


def test_config_table_D1_counts():
    """SURVEY Table D1 rows 2a and 4: nnzb, drop and level counts."""
    rp, ci, v = laplacian_bsr3(64, 64, 64)
    ctx = dd.dd_setup(rp, ci, v, grid=(64, 64, 64), tiles=(16, 16, 8), host_only=True)
    st = ctx.stats()
    assert (st["nnzb_before"], st["nnzb_after"], st["n_sub"], st["max_levels_L"]) == (1810432, 1703936, 128, 38)
    rp, ci, v, _ = spe10_style_bsr3()
    ctx = dd.dd_setup(rp, ci, v, grid=(60, 220, 85), tiles=(10, 20, 17), host_only=True)
    st = ctx.stats()
    assert (st["nnzb_before"], st["nnzb_after"], st["n_sub"], st["max_levels_L"]) == (7780000, 7385400, 330, 45)


def test_errors_match_oracle():
    # missing diagonal
    rp = np.array([0, 1, 2], np.int64)
    ci = np.array([1, 0], np.int32)
    with pytest.raises(dd.DDError) as e:
        dd.dd_setup(rp, ci, np.ones(18), P=2, host_only=True)
    assert e.value.name == "DD_E_MISSING_DIAG"
    # unsorted columns
    rp = np.array([0, 2, 4], np.int64)
    ci = np.array([1, 0, 0, 1], np.int32)
    with pytest.raises(dd.DDError) as e:
        dd.dd_setup(rp, ci, np.ones(36), P=2, host_only=True)
    assert e.value.name == "DD_E_UNSORTED_OR_DUP"
    # grid not divisible
    rp, ci, v = laplacian_bsr3(5, 4, 4)
    with pytest.raises(dd.DDError) as e:
        dd.dd_setup(rp, ci, v, grid=(5, 4, 4), tiles=(2, 2, 2), host_only=True)
    assert e.value.name == "DD_E_GRID_NOT_DIVISIBLE"
    # singular pivot at the same row as the oracle
    rp, ci, a = kron_blocks([[1.0, 1.0], [1.0, 1.0]])
    with pytest.raises(oracle.OracleError) as eo:
        oracle.ilu0(rp, ci, a)
    with pytest.raises(dd.DDError) as e:
        dd.dd_setup(rp, ci, a, P=2, host_only=True)
    assert e.value.name == "DD_E_SINGULAR_PIVOT" and f"row {eo.value.row}" in str(e.value)


# ------------------------------------------- scalar CSR path
from inputs.gen import laplacian_csr, random_csr_grid, spe10_style_csr  # noqa: E402

CSR_CASES = {
    "csr_laplace_16^3": (lambda: laplacian_csr(16, 16, 16), dict(grid=(16, 16, 16), tiles=(8, 8, 8))),
    "csr_random_ragged": (lambda: random_csr_grid(12, 10, 8, seed=11), dict(P=77)),
    "csr_random_bfs": (lambda: random_csr_grid(12, 10, 8, seed=12), dict(P=100, partitioner="bfs")),
    "csr_spe10_small": (lambda: spe10_style_csr(20, 40, 20, upper_ness_from=10)[:3],
                        dict(grid=(20, 40, 20), tiles=(10, 20, 10))),
    "csr_P1": (lambda: random_csr_grid(5, 4, 3, seed=13), dict(P=1)),
}


@pytest.mark.parametrize("name", list(CSR_CASES))
def test_host_setup_csr_bitwise_vs_oracle(name):
    gen, kw = CSR_CASES[name]
    rp, ci, v = gen()
    S = oracle.setup_csr(rp, ci, v, **kw)
    ctx = dd.dd_setup_csr(rp, ci, v, host_only=True, variants=7, **kw)
    assert ctx.bs == 1
    assert_setup_bitwise(ctx, S)
    st = ctx.stats()
    n = S["n"]
    rows = np.repeat(np.arange(n), np.diff(S["rp_d"]))
    nLU = int(np.sum(S["ci_d"] != rows))
    # canonical scalar apply bytes: 8(nL+nU+n) + 4(nL+nU) + 8(n+1) + 16n
    assert st["apply_canonical_bytes"] == 8 * (nLU + n) + 4 * nLU + 8 * (n + 1) + 16 * n


def test_csr_errors_and_refactor_rejected():
    rp = np.array([0, 1, 2], np.int64)
    with pytest.raises(dd.DDError) as e:
        dd.dd_setup_csr(rp, np.array([1, 0], np.int32), np.ones(2), P=2, host_only=True)
    assert e.value.name == "DD_E_MISSING_DIAG"
    rp, ci, v = random_csr_grid(4, 4, 4, seed=1)
    with pytest.raises(dd.DDError) as e:
        dd.dd_setup_csr(rp, ci, v, P=8, host_only=True, enable_refactor=True)
    assert e.value.name == "DD_E_INVALID_ARG"
    # singular pivot at the oracle's row
    rp, ci, a = np.array([0, 2, 4], np.int64), np.array([0, 1, 0, 1], np.int32), np.ones(4)
    with pytest.raises(oracle.OracleError) as eo:
        oracle.s_ilu0(rp, ci, a)
    with pytest.raises(dd.DDError) as e:
        dd.dd_setup_csr(rp, ci, a, P=2, host_only=True)
    assert e.value.name == "DD_E_SINGULAR_PIVOT" and f"row {eo.value.row}" in str(e.value)


def _slots_model(P, bs=3):
    """the analytic occupancy model of tile_slots (no device): 228 KB shared
    memory per SM, at most 3 CTAs per SM, the ring kernel's smem per CTA;
    returns (CTAs per SM, slots)"""
    vec = (8 * bs * P + 127) // 128 * 128
    best = 0
    for rc in (131072, 65536, 32768):
        sm = vec + rc + 16 * 4
        if sm <= 232448:
            best = max(best, min(3, (233472 - 1024) // (sm + 1024)))
    return best, 148 * best


@pytest.mark.parametrize("grid,P", [((160, 160, 160), 2048), ((60, 220, 85), 2048), ((64, 64, 64), 2048),
                                    ((96, 96, 48), 1024)])
def test_choose_tiles_score(grid, P):
    """dd_choose_tiles (host model, R41): the tiles divide the grid, P is
    inside [P/2, 2P], and no admissible tile shape scores higher on
    fill x bw x (1 - 3 dropped) (fill = wave fill of the CTA slots, bw = 0.82
    for one CTA per SM, dropped = share of the grid's couplings crossing tile
    faces; 0.5 % buckets)."""
    import math
    tx, ty, tz = dd.dd_choose_tiles(grid, device=-1, P_target=P)
    nx, ny, nz = grid
    assert nx % tx == 0 and ny % ty == 0 and nz % tz == 0
    assert P / 2 <= tx * ty * tz <= 2 * P
    N = nx * ny * nz
    tot = (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)

    def score(a, b, c):
        p = a * b * c
        per_sm, s = _slots_model(p)
        n = N // p
        fill = n / (-(-n // s) * s)
        drop = ((nx // a - 1) * ny * nz + (ny // b - 1) * nx * nz + (nz // c - 1) * nx * ny) / tot
        return math.floor(fill * (0.82 if per_sm <= 1 else 1.0) * (1 - 3 * drop) * 200) / 200
    best = max(score(a, b, c) for a in range(1, nx + 1) if nx % a == 0 for b in range(1, ny + 1) if ny % b == 0
               for c in range(1, nz + 1) if nz % c == 0 if P / 2 <= a * b * c <= 2 * P)
    assert score(tx, ty, tz) == best


def test_setup_auto_tiles_equals_choose_tiles():
    rp, ci, v = laplacian_bsr3(24, 24, 24)
    t = dd.dd_choose_tiles((24, 24, 24), device=-1, P_target=512)
    # the Laplacian's couplings weigh the same on every plane: the matrix-weighted
    # choice inside dd_setup equals the geometric one
    ctx = dd.dd_setup(rp, ci, v, grid=(24, 24, 24), tiles="auto", P=512, host_only=True)
    S = oracle.setup(rp, ci, v, grid=(24, 24, 24), tiles=t)
    lab, _ = ctx.partition()
    assert ctx.tiles == t and np.array_equal(lab, S["labels"])
    # the C entry point with tile dims 0 makes the same choice
    ctx0 = dd.dd_setup(rp, ci, v, grid=(24, 24, 24), tiles=(0, 0, 0), P=512, host_only=True)
    assert np.array_equal(ctx0.partition()[0], S["labels"])
