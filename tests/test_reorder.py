"""(f1) Locality reordering (host, CPU) — SPEC S:381-401 properties: a
bijection, identity strategy, BFS restores a scrambled path's bandwidth
(S:388), BFS reduces mean bandwidth b on scrambled banded graphs in >= 95 %
of seeds, degree order, determinism, permutation-invariant features
unchanged."""
import numpy as np
import pytest

import gen
import oracle


def _api():
    from paper_2605_15695_b200 import api
    return api


def bandwidths(rp, ci):
    return np.array([(ci[rp[i + 1] - 1] - ci[rp[i]]) if rp[i + 1] > rp[i] else 0
                     for i in range(len(rp) - 1)])


def scrambled(g, seed):
    perm = np.random.default_rng(seed).permutation(g.n)
    return gen.permute(g.n, g.rowptr, g.colidx, perm)


@pytest.mark.parametrize("strategy", ["identity", "bfs", "degree"])
def test_bijection_and_determinism(strategy):
    api = _api()
    for g in (gen.powerlaw(500, 6, 2.1, 1), gen.with_empty_rows(gen.uniform(300, 3, 2), 0.3, 3),
              gen.community(400, 20, 6, 0.9, 4, ordered=False)):
        p = api.pspmm_reorder(g.rowptr, g.colidx, strategy)
        assert sorted(p.tolist()) == list(range(g.n))
        assert np.array_equal(p, api.pspmm_reorder(g.rowptr, g.colidx, strategy))
        if strategy == "identity":
            assert np.array_equal(p, np.arange(g.n))


def test_bfs_restores_scrambled_path():
    api = _api()
    n = 300
    rows = np.concatenate([np.arange(n - 1), np.arange(1, n)])
    cols = np.concatenate([np.arange(1, n), np.arange(n - 1)])
    rp, ci = gen.csr_from_pairs(n, rows, cols)
    g = gen.Graph("path", n, rp, ci, np.ones(len(ci), np.float32))
    srp, sci = scrambled(g, 7)
    assert bandwidths(srp, sci).max() > 10
    p = api.pspmm_reorder(srp, sci, "bfs")
    rrp, rci = gen.permute(n, srp, sci, p.astype(np.int64))
    assert bandwidths(rrp, rci).max() <= 2


def test_bfs_reduces_bandwidth_on_scrambled_banded():
    api = _api()
    wins = 0
    for seed in range(100):
        g = gen.banded(150, 3, seed)
        srp, sci = scrambled(g, 1000 + seed)
        p = api.pspmm_reorder(srp, sci, "bfs")
        rrp, rci = gen.permute(g.n, srp, sci, p.astype(np.int64))
        wins += bandwidths(rrp, rci).mean() < bandwidths(srp, sci).mean()
    assert wins >= 95


def test_degree_strategy_orders_hubs_first():
    api = _api()
    g = gen.powerlaw(800, 8, 2.0, 5)
    p = api.pspmm_reorder(g.rowptr, g.colidx, "degree")
    # symmetrised degree (the strategy's key), non-increasing in the new order
    deg = np.zeros(g.n, np.int64)
    dr = np.diff(g.rowptr.astype(np.int64))
    rows = np.repeat(np.arange(g.n), dr)
    pairs = {(min(a, b), max(a, b)) for a, b in zip(rows.tolist(), g.colidx.tolist()) if a != b}
    for a, b in pairs:
        deg[a] += 1
        deg[b] += 1
    inv = np.empty(g.n, np.int64)
    inv[p] = np.arange(g.n)
    assert np.all(np.diff(deg[inv]) <= 0)


def test_reordering_preserves_invariant_features():
    api = _api()
    g = gen.community(600, 30, 8, 0.8, 6, ordered=False)
    p = api.pspmm_reorder(g.rowptr, g.colidx, "bfs")
    rrp, rci = gen.permute(g.n, g.rowptr, g.colidx, p.astype(np.int64))
    f0 = oracle.features(g.rowptr, g.colidx, g.val, 32)
    f1 = oracle.features(rrp, rci, np.ones(len(rci)), 32)
    for k in ("n", "n_hat", "nnz", "d", "d_max", "cv", "cv_hat", "rho"):
        assert f1[k] == pytest.approx(f0[k], rel=1e-12), k
