"""Pins of oracle.gnn_layer (f3: H' = A H W)
against facts independent of its own code path: a hand-worked 3x3 case, W =
identity reducing to the c-1 SpMM oracle (oracle.c), associativity against a
dense fp64 brute force, and the magnitude bound."""
import numpy as np

import gen
import oracle


def test_hand_case():
    # A = [[0, 2, 0], [1, 0, 3], [0, 0, 0]], H = [[1, 2], [3, 4], [5, 6]],
    # W = [[1, -1], [2, 0]]: H W = [[5, -1], [11, -3], [17, -5]]
    # A H W = [[22, -6], [56, -16], [0, 0]]
    rp = np.array([0, 1, 3, 3])
    ci = np.array([1, 0, 2])
    vl = np.array([2.0, 1.0, 3.0], np.float32)
    H = np.array([[1, 2], [3, 4], [5, 6]], np.float32)
    W = np.array([[1, -1], [2, 0]], np.float32)
    Y, mag = oracle.gnn_layer(rp, ci, vl, H, W)
    assert np.array_equal(Y, np.array([[22, -6], [56, -16], [0, 0]], np.float64))
    assert np.array_equal(mag, np.array([[22, 6], [56, 16], [0, 0]], np.float64))


def test_identity_weight_is_the_spmm_oracle():
    g = gen.powerlaw(500, 9, 2.2, 3)
    X = gen.dense(g.n, 24, 4)
    Y, mag = oracle.gnn_layer(g.rowptr, g.colidx, g.val, X, np.eye(24, dtype=np.float32))
    ref, refmag = oracle.spmm(g.rowptr, g.colidx, g.val, X)
    assert np.allclose(Y, ref, rtol=1e-13, atol=1e-13)
    assert np.allclose(mag, refmag, rtol=1e-13, atol=1e-13)


def test_matches_dense_brute_force_both_orders():
    g = gen.uniform(300, 7, 5)
    A = np.zeros((g.n, g.n))
    for i in range(g.n):
        A[i, g.colidx[g.rowptr[i]:g.rowptr[i + 1]]] = g.val[g.rowptr[i]:g.rowptr[i + 1]]
    X = gen.dense(g.n, 16, 6).astype(np.float64)
    W = gen.dense(16, 40, 7).astype(np.float64)
    Y, mag = oracle.gnn_layer(g.rowptr, g.colidx, g.val, X, W)
    assert np.allclose(Y, (A @ X) @ W, rtol=1e-11, atol=1e-11)
    assert np.allclose(Y, A @ (X @ W), rtol=1e-11, atol=1e-11)
    assert np.all(np.abs(Y) <= mag + 1e-12)
