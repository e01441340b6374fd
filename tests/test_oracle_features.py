"""Pins for the Table 3 features oracle (c-3): SPEC's worked cases (S:281,
S:282), the hand-derived pin X, and an independent numpy brute force."""
import math

import numpy as np
import pytest

import gen
import oracle
from conftest import golden


def test_identity_s281():
    f = oracle.features(np.arange(5), np.arange(4), np.ones(4), 32)
    want = dict(n=4, n_hat=4, nnz=4, delta=1, d=1, d_hat=1, d_max=1, cv=0, cv_hat=0,
                rho=0.25, b=0, b_max=0, pr1=0, pr2=0.5, sr1=1, sr2=1)
    assert f == {k: float(v) for k, v in want.items()}


def test_one_empty_row_s282():
    # rows 0,1,3 non-empty, row 2 empty
    f = oracle.features([0, 2, 3, 3, 5], [0, 3, 1, 0, 2], np.ones(5), 32)
    assert f["delta"] == 0.75
    assert f["d_hat"] == 5 / 3
    assert f["d_hat"] >= f["d"]


def test_pin_x_features():
    g = golden("pin_x.json")
    w = g["features_omega4"]
    f = oracle.features(g["rowPtr"], g["colIdx"], g["val"], g["omega"])

    def val(x):
        return x[0] / x[1] if isinstance(x, list) else float(x)

    for k in ("n", "n_hat", "nnz", "delta", "d", "d_hat", "d_max", "rho", "b", "b_max",
              "pr1", "pr2", "sr1", "sr2"):
        assert f[k] == pytest.approx(val(w[k]), rel=1e-15, abs=1e-15), k
    assert f["cv"] == pytest.approx(math.sqrt(w["cv_sqrt_num"]) / w["cv_den"], rel=1e-14)
    assert f["cv_hat"] == pytest.approx(math.sqrt(w["cv_hat_sqrt_num"]) / w["cv_hat_den"],
                                        rel=1e-14)
    f32 = oracle.features(g["rowPtr"], g["colIdx"], g["val"], 32)
    assert f32["sr1"] == g["features_omega32"]["sr1"]
    assert f32["sr2"] == g["features_omega32"]["sr2"]


def brute_features(rowptr, colidx, n, omega):
    deg = np.diff(rowptr.astype(np.int64))
    nz = deg > 0
    nnz = int(deg.sum())
    bw = np.zeros(n)
    for i in range(n):
        if deg[i]:
            bw[i] = colidx[rowptr[i + 1] - 1] - colidx[rowptr[i]]
    out = dict(n=n, n_hat=int(nz.sum()), nnz=nnz, delta=nz.sum() / n, d=nnz / n,
               d_hat=nnz / nz.sum(), d_max=int(deg.max()), cv=deg.std() / deg.mean(),
               cv_hat=deg[nz].std() / deg[nz].mean(), rho=nnz / n / n, b=bw.mean(),
               b_max=bw.max())
    for V in (1, 2):
        pairs = set()
        for i in range(n):
            for c in colidx[rowptr[i]:rowptr[i + 1]]:
                pairs.add((i // V, int(c)))
        nnzv = len(pairs)
        P = -(-n // V)
        L = np.zeros(P, np.int64)
        for pnl, _ in pairs:
            L[pnl] += 1
        nonempty = int((L > 0).sum())
        SG = -(-nnzv // (nonempty * omega)) * omega
        chunks = sum(max(1, -(-int(x) // SG)) for x in L)
        out[f"pr{V}"] = 1 - nnz / (nnzv * V)
        out[f"sr{V}"] = (chunks + 1) / (P + 1)
    return out


@pytest.mark.parametrize("make", [
    lambda: gen.uniform(150, 5, 1),
    lambda: gen.powerlaw(257, 7, 2.0, 2),
    lambda: gen.banded(99, 4, 3),
    lambda: gen.with_empty_rows(gen.community(200, 10, 6, 0.8, 4), 0.25, 5),
    lambda: gen.giant_row(120, 110, 2, 6),
    lambda: gen.config_graph("cora"),
])
@pytest.mark.parametrize("omega", [4, 32])
def test_brute_force(make, omega):
    g = make()
    f = oracle.features(g.rowptr, g.colidx, g.val, omega)
    b = brute_features(g.rowptr, g.colidx, g.n, omega)
    for k, v in b.items():
        assert f[k] == pytest.approx(v, rel=1e-12, abs=1e-14), k


def test_permutation_invariance_s285():
    g = gen.powerlaw(300, 9, 2.1, 7)
    perm = np.random.default_rng(1).permutation(g.n)
    rp, ci = gen.permute(g.n, g.rowptr, g.colidx, perm)
    f0 = oracle.features(g.rowptr, g.colidx, g.val, 32)
    f1 = oracle.features(rp, ci, np.ones(len(ci)), 32)
    for k in ("n", "nnz", "d", "d_max", "cv", "rho", "n_hat", "cv_hat"):
        assert f1[k] == pytest.approx(f0[k], rel=1e-12), k
    assert f1["b"] != f0["b"]


def test_empty_matrix_rejected():
    with pytest.raises(oracle.OracleError) as e:
        oracle.features(np.zeros(4, np.int32), [], [], 32)
    assert e.value.code == 5
