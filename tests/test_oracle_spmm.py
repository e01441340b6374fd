"""Pins for the SpMM oracle (c-1): each test checks oracle.spmm against
something other than itself — a hand-worked case, a closed form, a library
routine on the densified matrix, or exact integer arithmetic."""
import numpy as np
import pytest

import gen
import oracle
from conftest import golden


def dense_of(rowptr, colidx, val, n):
    A = np.zeros((n, n), dtype=np.float64)
    for i in range(n):
        for p in range(rowptr[i], rowptr[i + 1]):
            A[i, colidx[p]] = val[p]
    return A


def test_hand_case_s68():
    # [[1,2],[0,3]] . [[1,0],[1,1]] = [[3,2],[3,3]]
    C, mag = oracle.spmm([0, 2, 3], [0, 1, 1], [1, 2, 3], np.array([[1, 0], [1, 1]], np.float32))
    assert C.tolist() == [[3, 2], [3, 3]]
    assert mag.tolist() == [[3, 2], [3, 3]]


def test_pin_x_integer_exact():
    g = golden("pin_x.json")
    K = g["spmm"]["K"]
    B = np.array([[4 * i + k for k in range(K)] for i in range(g["n"])], np.float32)
    C, _ = oracle.spmm(g["rowPtr"], g["colIdx"], g["val"], B)
    assert C.tolist() == g["spmm"]["C"]


@pytest.mark.parametrize("n,K", [(1, 1), (5, 3), (64, 16), (300, 17)])
def test_identity_gives_B(n, K):
    B = gen.dense(n, K, 7)
    C, _ = oracle.spmm(np.arange(n + 1), np.arange(n), np.ones(n), B)
    assert np.array_equal(C, B.astype(np.float64))


def test_permutation_and_diagonal_closed_forms():
    n, K = 97, 12
    rng = np.random.default_rng(3)
    perm = rng.permutation(n)
    B = gen.dense(n, K, 8)
    # permutation matrix P[i, perm[i]] = 1 -> C[i] = B[perm[i]]
    C, _ = oracle.spmm(np.arange(n + 1), perm, np.ones(n), B)
    assert np.array_equal(C, B[perm].astype(np.float64))
    # diagonal -> scaled rows, each a single exact fp64 product of fp32 values
    d = gen.values(n, 9)
    C, _ = oracle.spmm(np.arange(n + 1), np.arange(n), d, B)
    assert np.array_equal(C, d.astype(np.float64)[:, None] * B.astype(np.float64))


def test_zero_matrix_and_empty_rows():
    n, K = 10, 4
    B = gen.dense(n, K, 1)
    C, mag = oracle.spmm(np.zeros(n + 1, np.int32), np.zeros(0), np.zeros(0), B)
    assert not C.any() and not mag.any()


GRAPHS = [
    lambda: gen.uniform(200, 6, 11),
    lambda: gen.powerlaw(300, 8, 2.1, 12),
    lambda: gen.banded(256, 3, 13),
    lambda: gen.community(320, 32, 10, 0.8, 14),
    lambda: gen.giant_row(150, 140, 3, 15),
    lambda: gen.with_empty_rows(gen.uniform(128, 5, 16), 0.3, 17),
    lambda: gen.config_graph("cora"),
]


@pytest.mark.parametrize("make", GRAPHS)
@pytest.mark.parametrize("K", [1, 7, 32])
def test_brute_force_dense_fp64(make, K):
    g = make()
    if g.n > 3000:
        pytest.skip("dense brute force only for small n")
    B = gen.dense(g.n, K, 21)
    C, mag = oracle.spmm(g.rowptr, g.colidx, g.val, B)
    A = dense_of(g.rowptr, g.colidx, g.val, g.n)
    ref = A @ B.astype(np.float64)
    refmag = np.abs(A) @ np.abs(B.astype(np.float64))
    assert np.allclose(C, ref, rtol=0, atol=1e-12 * (1 + refmag.max()))
    assert np.allclose(mag, refmag, rtol=1e-13, atol=1e-300)
    assert np.all(np.abs(C) <= mag * (1 + 1e-12))


def test_integer_inputs_exact():
    g = gen.powerlaw(400, 12, 2.2, 31, kind="int")
    B = gen.dense(g.n, 9, 32, kind="int")
    C, _ = oracle.spmm(g.rowptr, g.colidx, g.val, B)
    A = dense_of(g.rowptr, g.colidx, g.val, g.n).astype(np.int64)
    assert np.array_equal(C, (A @ B.astype(np.int64)).astype(np.float64))


def test_permuted_graph_identity():
    # (P A P^T)(P B) = P (A B)
    g = gen.community(256, 16, 9, 0.7, 41)
    n = g.n
    perm = np.random.default_rng(5).permutation(n)
    B = gen.dense(n, 8, 42, kind="int")
    g_int = gen.community(256, 16, 9, 0.7, 41, kind="int")
    C, _ = oracle.spmm(g_int.rowptr, g_int.colidx, g_int.val, B)
    # relabel node i -> perm[i]; values follow their (row, col) entry
    deg = np.diff(g_int.rowptr.astype(np.int64))
    rows = np.repeat(np.arange(n), deg)
    keys = perm[rows].astype(np.int64) * n + perm[g_int.colidx]
    order = np.argsort(keys)
    keys = keys[order]
    vals = g_int.val[order]
    prow = keys // n
    pcol = (keys % n).astype(np.int32)
    prowptr = np.concatenate([[0], np.cumsum(np.bincount(prow, minlength=n))])
    PB = np.empty_like(B)
    PB[perm] = B
    C2, _ = oracle.spmm(prowptr, pcol, vals, PB)
    assert np.array_equal(C2[perm], C)


def test_row_subset_matches_full():
    g = gen.powerlaw(500, 10, 2.0, 51)
    B = gen.dense(g.n, 24, 52)
    C, mag = oracle.spmm(g.rowptr, g.colidx, g.val, B)
    rows = np.array([0, 499, 250, 3, 3, 17])
    Cs, ms = oracle.spmm(g.rowptr, g.colidx, g.val, B, rows=rows, threads=2)
    assert np.array_equal(Cs, C[rows]) and np.array_equal(ms, mag[rows])


def test_threads_do_not_change_results():
    g = gen.uniform(2000, 7, 61)
    B = gen.dense(g.n, 16, 62)
    C1, _ = oracle.spmm(g.rowptr, g.colidx, g.val, B, threads=1)
    C4, _ = oracle.spmm(g.rowptr, g.colidx, g.val, B, threads=4)
    assert np.array_equal(C1, C4)
