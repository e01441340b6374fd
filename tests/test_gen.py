"""Generators: determinism, canonical CSR, and the shapes DESIGN.md §4 states."""
import numpy as np
import pytest

import gen


def canonical(g):
    rp, ci = g.rowptr, g.colidx
    assert rp.dtype == np.int32 and ci.dtype == np.int32 and g.val.dtype == np.float32
    assert rp[0] == 0 and rp[-1] == len(ci) == len(g.val)
    assert np.all(np.diff(rp) >= 0)
    assert ci.min(initial=0) >= 0 and ci.max(initial=0) < g.n
    deg = np.diff(rp.astype(np.int64))
    rows = np.repeat(np.arange(g.n), deg)
    # strictly increasing within each row
    same = rows[1:] == rows[:-1]
    assert np.all(np.diff(ci.astype(np.int64))[same] > 0)


@pytest.mark.parametrize("make", [
    lambda: gen.uniform(1000, 8, 7), lambda: gen.powerlaw(2000, 6, 2.1, 3),
    lambda: gen.banded(8, 1, 0), lambda: gen.community(500, 20, 7, 0.8, 2),
    lambda: gen.giant_row(300, 290, 3, 1),
    lambda: gen.config_graph("cora"), lambda: gen.config_graph("reddit", 0.002),
    lambda: gen.config_graph("products", 0.0005), lambda: gen.config_graph("proteins", 0.002),
    lambda: gen.config_graph("roadnet", 0.001),
    lambda: gen.config_graph("proteins_clustered", 0.02)])
def test_deterministic_and_canonical(make):
    a, b = make(), make()
    canonical(a)
    assert np.array_equal(a.rowptr, b.rowptr) and np.array_equal(a.colidx, b.colidx)
    assert np.array_equal(a.val, b.val)


def test_banded_bmax():
    g = gen.banded(8, 1, 0)
    deg = np.diff(g.rowptr)
    for i in range(g.n):
        if deg[i]:
            assert g.colidx[g.rowptr[i + 1] - 1] - g.colidx[g.rowptr[i]] <= 2


def test_powerlaw_cv_above_one():
    g = gen.powerlaw(2000, 6, 2.1, 3)
    deg = np.diff(g.rowptr.astype(np.int64))
    assert deg.std() / deg.mean() > 1.0


def test_config_shapes_small():
    c = gen.config_graph("cora")
    assert c.n == 2708 and c.nnz == 10556 and c.K == 16
    # symmetric, no self loops
    deg = np.diff(c.rowptr.astype(np.int64))
    rows = np.repeat(np.arange(c.n), deg)
    keys = set(zip(rows.tolist(), c.colidx.tolist()))
    assert all((j, i) in keys for i, j in keys)
    assert all(i != j for i, j in keys)
    r = gen.config_graph("roadnet", 0.01)
    assert r.nnz % 2 == 0
    # locality order: every edge within one lattice row / adjacent rows
    deg = np.diff(r.rowptr.astype(np.int64))
    rows = np.repeat(np.arange(r.n), deg)
    W = int(np.ceil(np.sqrt(r.n)))
    assert np.abs(rows - r.colidx).max() <= W + 1


def test_proteins_clustered_shape():
    """SURVEY §8(d) variant (ii): about half of each row's draws stay in its
    1024-node community, so the diagonal 1024-blocks hold ~half the nonzeros
    (a little less after duplicates), plus the uniform draws that land in
    the row's own community by chance (1024 / n of them)."""
    g = gen.config_graph("proteins_clustered", 0.05)
    rows = np.repeat(np.arange(g.n), np.diff(g.rowptr))
    inside = (rows // 1024) == (g.colidx // 1024)
    frac = inside.mean()
    expect = 0.5 + 0.5 * 1024 / g.n
    assert expect - 0.06 < frac < expect + 0.01, (frac, expect)
    # community-ordered IDs: the in-community share per 1024-row block is flat
    blocks = rows // 1024
    per = np.bincount(blocks, weights=inside) / np.bincount(blocks)
    assert per[:-1].min() > 0.35
