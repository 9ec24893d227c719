"""Pins for the oracle's setup steps (O1-O8).

Each test names what pins it: a paper value, a worked example, a closed form,
an invariant, a library routine or brute force. CPU only."""
import numpy as np
import pytest

import oracle
from inputs.gen import (laplacian_bsr3, random_block_chain, random_block_grid,
                        spe10_style_bsr3, grid_stencil_pattern)
from tests.helpers import (alg5_marking, bsr, dense_pattern_matrix, golden, kron_blocks,
                           split_factors)

G = golden("spec_worked_examples.json")
T5 = golden("table5_partitions.json")


# ----------------------------------------------------------------- O1 inputs
@pytest.mark.parametrize("grid", [(1, 1, 1), (2, 1, 1), (4, 3, 2), (16, 16, 16), (60, 220, 85)])
def test_o1_block_count_closed_form(grid):
    """Closed form nnzb = 7 nx ny nz - 2(ny nz + nx nz + nx ny)."""
    nx, ny, nz = grid
    rp, ci, _ = grid_stencil_pattern(nx, ny, nz)
    assert rp[-1] == 7 * nx * ny * nz - 2 * (ny * nz + nx * nz + nx * ny)
    # columns strictly ascending per row
    rows = np.repeat(np.arange(nx * ny * nz), np.diff(rp))
    same = rows[1:] == rows[:-1]
    assert np.all(ci[1:][same] > ci[:-1][same])


def test_o1_paper_counts():
    """Table 5 P:965-966 nnz (scalar = 9 x blocks) and spe10's 7,780,000."""
    for row in T5["rows"]:
        nx, ny, nz = row["grid"]
        nnzb = 7 * nx * ny * nz - 2 * (ny * nz + nx * nz + nx * ny)
        assert 9 * nnzb == row["nnz"]
    rp, _, _ = grid_stencil_pattern(*T5["spe10_nnz"]["grid"])
    assert rp[-1] == T5["spe10_nnz"]["nnz"]


def test_o1_laplacian_values_spmv_example():
    """[[6,-1],[-1,6]] (x) I3 times ones = 5 (S:71-73 worked example)."""
    rp, ci, v = laplacian_bsr3(2, 1, 1)
    A = bsr(rp, ci, v).toarray()
    S = np.array(G["spmv_2x2"]["A"], dtype=float)
    assert np.array_equal(A, np.kron(S, np.eye(3)))
    y = oracle.spmv(rp, ci, v, np.ones(6))
    assert np.array_equal(y, np.full(6, 5.0))


def test_o1_spe10_style_dominant():
    rp, ci, v, logk = spe10_style_bsr3(12, 20, 10, upper_ness_from=5)
    A = bsr(rp, ci, v).tocsr()
    d = np.abs(A.diagonal())
    off = np.asarray(abs(A).sum(axis=1)).ravel() - d
    assert np.all(d > off)
    assert logk.min() >= -3.0 and logk.max() <= 4.3


# ----------------------------------------------------------------- O2 labels
def test_o2_worked_example():
    ex = G["labels_geometric"]
    lab = oracle.labels_geometric(ex["grid"], ex["tiles"])
    assert lab[ex["gidx"]] == ex["label"]


def test_o2_paper_subdomain_counts():
    """Table 5: 128^3 with (16,16,8) tiles -> 1024 subdomains of 2048 rows."""
    row = T5["rows"][0]
    lab = oracle.labels_geometric(row["grid"], row["tiles"])
    cnt = np.bincount(lab)
    assert cnt.shape[0] == row["n_subdomains"]
    assert np.all(cnt == row["rows_per_subdomain"])


@pytest.mark.parametrize("grid,tiles", [((8, 6, 4), (4, 3, 2)), ((6, 6, 6), (3, 2, 6))])
def test_o2_labels_are_boxes(grid, tiles):
    """Invariant: each label's vertices form one tx*ty*tz box."""
    nx, ny, nz = grid
    lab = oracle.labels_geometric(grid, tiles)
    g = np.arange(nx * ny * nz)
    i, j, k = g % nx, (g // nx) % ny, g // (nx * ny)
    for l in np.unique(lab):
        m = lab == l
        assert m.sum() == np.prod(tiles)
        for coord, t in ((i, tiles[0]), (j, tiles[1]), (k, tiles[2])):
            c = coord[m]
            assert c.max() - c.min() + 1 == t and c.min() % t == 0


def test_o2_not_divisible():
    with pytest.raises(ValueError):
        oracle.labels_geometric((5, 4, 4), (2, 2, 2))


# ----------------------------------------------------------- O3 permutation
def test_o3_worked_examples():
    for case in G["permutation"]["cases"]:
        n2o, o2n = oracle.permutation(np.array(case["labels"], dtype=np.int32))
        assert n2o.tolist() == case["new_to_old"]
        assert np.array_equal(n2o[o2n], np.arange(len(n2o)))


def test_o3_equals_stable_argsort():
    """Library routine: numpy's stable argsort by label is the stable grouping."""
    lab = np.random.default_rng(5).integers(0, 17, 1000).astype(np.int32)
    n2o, o2n = oracle.permutation(lab)
    assert np.array_equal(n2o, np.argsort(lab, kind="stable"))
    assert np.array_equal(o2n[n2o], np.arange(1000))


# ---------------------------------------------------------------- O4 reorder
def test_o4_identity_and_swap():
    rp, ci, v = random_block_grid(3, 2, 2, seed=3)
    idp = np.arange(12, dtype=np.int32)
    r2 = oracle.reorder(rp, ci, v, idp, idp)
    assert all(np.array_equal(a, b) for a, b in zip(r2, (rp, ci, v)))
    ex = G["reorder_swap"]
    rp, ci, v = kron_blocks(ex["A"])
    n2o = np.array(ex["new_to_old"], dtype=np.int32)
    rpo, cio, vo = oracle.reorder(rp, ci, v, n2o, np.argsort(n2o).astype(np.int32))
    assert np.array_equal(bsr(rpo, cio, vo).toarray(), np.kron(np.array(ex["result"], float), np.eye(3)))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_o4_dense_PAPt(seed):
    """Brute force: reordered matrix == dense A[p][:, p] (block-expanded)."""
    rng = np.random.default_rng(seed)
    rp, ci, v = random_block_grid(4, 3, 2, seed=seed)
    n = 24
    lab = rng.integers(0, 5, n).astype(np.int32)
    n2o, o2n = oracle.permutation(lab)
    rpo, cio, vo = oracle.reorder(rp, ci, v, n2o, o2n)
    rows = np.repeat(np.arange(n), np.diff(rpo))
    same = rows[1:] == rows[:-1]
    assert np.all(cio[1:][same] > cio[:-1][same])
    p3 = (3 * n2o[:, None] + np.arange(3)).ravel()
    Ad = bsr(rp, ci, v).toarray()
    assert np.array_equal(bsr(rpo, cio, vo).toarray(), Ad[p3][:, p3])


# ------------------------------------------------------------------- O5 drop
def test_o5_tridiagonal_worked_example():
    ex = G["drop_tridiagonal"]
    rp, ci, v = random_block_chain(ex["n"], seed=1)
    assert rp[-1] == ex["nnz"]
    lab = oracle.labels_chunks(ex["n"], ex["P"])
    rpd, cid, vd = oracle.drop(rp, ci, v, lab)
    assert rp[-1] - rpd[-1] == ex["dropped"]


def test_o5_brute_force_and_closed_form():
    grid, tiles = (8, 6, 4), (4, 3, 2)
    rp, ci, v = random_block_grid(*grid, seed=7)
    lab = oracle.labels_geometric(grid, tiles)
    n2o, o2n = oracle.permutation(lab)
    rpr, cir, vr = oracle.reorder(rp, ci, v, n2o, o2n)
    ln = lab[n2o]
    rpd, cid, vd = oracle.drop(rpr, cir, vr, ln)
    Ar = bsr(rpr, cir, vr).toarray()
    same = (ln[:, None] == ln[None, :])
    mask = np.kron(same, np.ones((3, 3), bool))
    assert np.array_equal(bsr(rpd, cid, vd).toarray(), np.where(mask, Ar, 0.0))
    nx, ny, nz = grid
    tx, ty, tz = tiles
    dropped = 2 * ((nx // tx - 1) * ny * nz + (ny // ty - 1) * nx * nz + (nz // tz - 1) * nx * ny)
    assert rpr[-1] - rpd[-1] == dropped


@pytest.mark.parametrize("row", T5["rows"], ids=[r["name"] for r in T5["rows"]])
def test_o5_table5_exact(row):
    """PAPER Table 5: exact nonzeros after decomposition."""
    rp, ci, v = laplacian_bsr3(*row["grid"])
    lab = oracle.labels_geometric(row["grid"], row["tiles"])
    n2o, o2n = oracle.permutation(lab)
    rpr, cir, vr = oracle.reorder(rp, ci, v, n2o, o2n)
    assert 9 * rpr[-1] == row["nnz"]
    rpd, _, _ = oracle.drop(rpr, cir, vr, lab[n2o])
    assert 9 * rpd[-1] == row["nnz_post"]
    assert round(100 * (row["nnz"] - row["nnz_post"]) / row["nnz"], 2) == row["dropped_pct"]


# ------------------------------------------------------------------ O6 ILU0
def _ilu_on_pattern_ok(rp, ci, a, lu, tol=1e-12):
    F = split_factors(rp, ci, lu)
    LU = (F["L"] @ F["U"]).toarray()
    A = bsr(rp, ci, a).toarray()
    pat = bsr(rp, ci, np.ones_like(a)).toarray() != 0
    err = np.abs(LU - A)[pat].max()
    return err <= tol * np.abs(A).max(), LU, A


@pytest.mark.parametrize("seed", range(4))
def test_o6_ilu0_defining_property(seed):
    """(L U)_ij = A_ij for every (i,j) in pattern(A) -- the ILU0 definition."""
    rp, ci, a = random_block_grid(4, 3, 3, seed=seed)
    lu, dinv = oracle.ilu0(rp, ci, a)
    ok, LU, A = _ilu_on_pattern_ok(rp, ci, a, lu)
    assert ok


@pytest.mark.parametrize("seed", range(3))
def test_o6_block_tridiagonal_is_exact_lu(seed):
    """Block-tridiagonal chain: ILU0 has no fill to drop -> L U == A everywhere."""
    rp, ci, a = random_block_chain(12, seed=seed)
    lu, _ = oracle.ilu0(rp, ci, a)
    F = split_factors(rp, ci, lu)
    A = bsr(rp, ci, a).toarray()
    assert np.abs((F["L"] @ F["U"]).toarray() - A).max() <= 1e-12 * np.abs(A).max()


@pytest.mark.parametrize("n", [2, 5])
def test_o6_full_pattern_is_dense_lu(n):
    """Full dense block pattern: ILU0 == unpivoted block LU; unique, so L U == A."""
    rp, ci, a, A = dense_pattern_matrix(n, seed=n)
    lu, _ = oracle.ilu0(rp, ci, a)
    F = split_factors(rp, ci, lu)
    assert np.abs((F["L"] @ F["U"]).toarray() - A).max() <= 1e-10 * np.abs(A).max()
    # unit block-lower L and block-upper U (block structure pinned)
    Ld, Ud = F["L"].toarray(), F["U"].toarray()
    for i in range(n):
        assert np.array_equal(Ld[3 * i:3 * i + 3, 3 * i:3 * i + 3], np.eye(3))
        assert not np.any(Ld[3 * i:3 * i + 3, 3 * (i + 1):])
        assert not np.any(Ud[3 * i:3 * i + 3, :3 * i])


def test_o6_worked_example_2x2():
    ex = G["ilu0_2x2"]
    rp, ci, a = kron_blocks(ex["A"])
    lu, dinv = oracle.ilu0(rp, ci, a)
    blocks = lu.reshape(-1, 3, 3)  # positions: (0,0) (0,1) (1,0) (1,1)
    assert np.array_equal(blocks[2], ex["L21"] * np.eye(3))
    U = np.array(ex["U"], float)
    assert np.array_equal(blocks[0], U[0, 0] * np.eye(3))
    assert np.array_equal(blocks[1], U[0, 1] * np.eye(3))
    assert np.array_equal(blocks[3], U[1, 1] * np.eye(3))
    ex2 = G["ildu0_2x2"]
    uu = oracle.ildu0(rp, ci, lu, dinv).reshape(-1, 3, 3)
    d = dinv.reshape(-1, 3, 3)
    assert np.array_equal(d[0], ex2["inv_D"][0] * np.eye(3))
    assert np.array_equal(d[1], ex2["inv_D"][1] * np.eye(3))
    assert np.array_equal(uu[1], ex2["Uunit01"] * np.eye(3))


def test_o6_whole_equals_per_subdomain_bitwise():
    """Factoring A_dd whole == factoring every subdomain alone, bitwise."""
    grid, tiles = (6, 4, 4), (3, 2, 2)
    rp, ci, v = random_block_grid(*grid, seed=11)
    S = oracle.setup(rp, ci, v, grid=grid, tiles=tiles)
    for s in range(S["n_sub"]):
        a, e = S["sub_ptr"][s], S["sub_ptr"][s + 1]
        p0, p1 = S["rp_d"][a], S["rp_d"][e]
        rps = S["rp_d"][a:e + 1] - p0
        cis = S["ci_d"][p0:p1] - a
        lu_s, dinv_s = oracle.ilu0(rps, cis, S["v_d"][9 * p0:9 * p1])
        assert np.array_equal(lu_s, S["lu"][9 * p0:9 * p1])
        assert np.array_equal(dinv_s, S["dinv"][9 * a:9 * e])


def test_o6_scalar_laplacian_structure():
    """e*I3 Laplacian: every factor block is a scalar multiple of I3."""
    rp, ci, v = laplacian_bsr3(6, 5, 4)
    lu, dinv = oracle.ilu0(rp, ci, v)
    for arr in (lu, dinv):
        b = arr.reshape(-1, 3, 3)
        assert np.array_equal(b, b[:, 0, 0][:, None, None] * np.eye(3)[None])
    assert _ilu_on_pattern_ok(rp, ci, v, lu)[0]


def test_o6_one_subdomain_is_global_ilu0():
    grid = (4, 4, 3)
    rp, ci, v = random_block_grid(*grid, seed=4)
    S = oracle.setup(rp, ci, v, grid=grid, tiles=grid)
    lu, dinv = oracle.ilu0(rp, ci, v)
    assert S["rp_d"][-1] == rp[-1]
    assert np.array_equal(S["lu"], lu) and np.array_equal(S["dinv"], dinv)


def test_o6_errors():
    rp = np.array([0, 1, 2], dtype=np.int64)
    ci = np.array([1, 0], dtype=np.int32)  # no diagonal blocks
    with pytest.raises(oracle.OracleError) as e:
        oracle.ilu0(rp, ci, np.ones(18))
    assert e.value.code == 1 and e.value.row == 0
    rp, ci, a = kron_blocks([[1.0, 1.0], [1.0, 1.0]])  # U_11 = 0 after elimination
    with pytest.raises(oracle.OracleError) as e:
        oracle.ilu0(rp, ci, a)
    assert e.value.code == 2 and e.value.row == 1


# ----------------------------------------------------------------- O7 ILDU0
@pytest.mark.parametrize("seed", range(3))
def test_o7_reassembly(seed):
    """L blkdiag(U_ii) Uunit == L U and Dinv_i == numpy.linalg.inv(U_ii)."""
    rp, ci, a = random_block_grid(3, 3, 3, seed=seed)
    lu, dinv = oracle.ilu0(rp, ci, a)
    uu = oracle.ildu0(rp, ci, lu, dinv)
    F = split_factors(rp, ci, lu, uu)
    lhs = (F["L"] @ F["D"] @ F["Uunit"]).toarray()
    rhs = (F["L"] @ F["U"]).toarray()
    assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()
    n = rp.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    Uii = lu.reshape(-1, 3, 3)[ci == rows]
    ref = np.linalg.inv(Uii)
    assert np.abs(dinv.reshape(-1, 3, 3) - ref).max() <= 1e-13 * np.abs(ref).max()


# ---------------------------------------------------------------- O8 levels
def test_o8_worked_examples():
    ex = G["levels_lower"]
    S = np.eye(ex["n"])
    for i, j in ex["deps"]:
        S[i, j] = 1.0
    rp, ci, _ = kron_blocks(S)
    assert oracle.levels_lower(rp, ci).tolist() == ex["hmap"]
    rp, ci, _ = kron_blocks(np.triu(np.ones((4, 4))))
    assert oracle.levels_upper(rp, ci).tolist() == golden("spec_worked_examples.json")[
        "levels_upper_dense4"]["hmap"]


@pytest.mark.parametrize("grid,tiles", [((8, 8, 8), (4, 4, 4)), ((16, 16, 8), (16, 16, 8)),
                                        ((12, 8, 6), (6, 4, 3))])
def test_o8_tile_closed_form(grid, tiles):
    """7-point tiles: hmapL = i'+j'+k', hmapU = (tx-1-i')+(ty-1-j')+(tz-1-k')."""
    rp, ci, v = laplacian_bsr3(*grid)
    S = oracle.setup(rp, ci, v, grid=grid, tiles=tiles)
    nx, ny, nz = grid
    tx, ty, tz = tiles
    g = S["new_to_old"].astype(np.int64)
    i, j, k = g % nx % tx, (g // nx) % ny % ty, g // (nx * ny) % tz
    assert np.array_equal(S["hmapL"], i + j + k)
    assert np.array_equal(S["hmapU"], (tx - 1 - i) + (ty - 1 - j) + (tz - 1 - k))
    assert S["hmapL"].max() + 1 == tx + ty + tz - 2


@pytest.mark.parametrize("seed", range(6))
def test_o8_alg5_marking_loop_and_brute_force(seed):
    """Independent sequential Alg. 5 marking loop == oracle's longest path;
    every dependency sits at a strictly earlier level and each level-h>0 row
    has a dependency at level h-1 (tightness)."""
    rng = np.random.default_rng(seed)
    n = 60
    S = np.eye(n)
    for i in range(n):
        for j in range(i):
            if rng.random() < 0.08:
                S[i, j] = 1.0
    rp, ci, _ = kron_blocks(S)
    h = oracle.levels_lower(rp, ci)
    deps = [list(np.nonzero(S[i, :i])[0]) for i in range(n)]
    assert np.array_equal(h, alg5_marking(n, deps))
    for i in range(n):
        if deps[i]:
            assert all(h[j] < h[i] for j in deps[i])
            assert any(h[j] == h[i] - 1 for j in deps[i])
        else:
            assert h[i] == 0
    # mirror for upper
    rpu, ciu, _ = kron_blocks(S.T)
    hu = oracle.levels_upper(rpu, ciu)
    rev = alg5_marking(n, [list(n - 1 - np.nonzero(S.T[n - 1 - i, n - i:])[0] - (n - i)) for i in range(n)])
    assert np.array_equal(hu, rev[::-1])


# ------------------------------------------------ O2b graph-growing partition
def test_o2b_bfs_worked_example_and_trivial_cases():
    """path graph n=8, P=2 -> [0,0,1,1,2,2,3,3]; P = n -> one part; P = 1
    -> singleton parts in seed order (ascending)."""
    rp, ci, _ = random_block_chain(8, seed=1)
    assert oracle.labels_bfs(rp, ci, 2).tolist() == [0, 0, 1, 1, 2, 2, 3, 3]
    rp, ci, _ = random_block_grid(5, 4, 3, seed=2)
    assert np.all(oracle.labels_bfs(rp, ci, 60) == 0)
    assert np.array_equal(oracle.labels_bfs(rp, ci, 1), np.arange(60))


@pytest.mark.parametrize("grid,P", [((8, 8, 8), 37), ((12, 10, 6), 64), ((20, 3, 2), 7)])
def test_o2b_bfs_sizes_and_first_part_is_scipy_bfs(grid, P):
    """Exact part sizes (last smaller); part 0 = the first P vertices of
    scipy.sparse.csgraph.breadth_first_order from vertex 0 (library routine,
    same ascending neighbour order)."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import breadth_first_order
    rp, ci, _ = grid_stencil_pattern(*grid)
    n = rp.shape[0] - 1
    lab = oracle.labels_bfs(rp, ci, P)
    cnt = np.bincount(lab)
    assert np.all(cnt[:-1] == P) and 0 < cnt[-1] <= P and cnt.sum() == n
    A = sp.csr_matrix((np.ones(ci.shape[0]), ci, rp), shape=(n, n))
    order = breadth_first_order(A, 0, directed=True, return_predecessors=False)
    assert set(np.nonzero(lab == 0)[0].tolist()) == set(order[:P].tolist())
