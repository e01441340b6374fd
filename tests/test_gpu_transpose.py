"""(f3) GPU CSR transpose: bit-exact against the definition (A^T[j, i] =
A[i, j], canonical row order), and the backward SpMM A^T . dC through the
engine matches the fp64 oracle run on the brute-force transpose."""
import numpy as np
import pytest

import gen
import oracle
from gpu_util import assert_parity, dev

pytestmark = pytest.mark.gpu


def brute_transpose(g, n_cols):
    deg = np.diff(g.rowptr.astype(np.int64))
    rows = np.repeat(np.arange(g.n), deg)
    order = np.lexsort((rows, g.colidx))  # by column, then row
    cols = g.colidx[order]
    t_rp = np.zeros(n_cols + 1, np.int64)
    np.add.at(t_rp, cols + 1, 1)
    return np.cumsum(t_rp).astype(np.int32), rows[order].astype(np.int32), g.val[order]


@pytest.mark.parametrize("make", [
    lambda: gen.powerlaw(3001, 12, 2.0, 2), lambda: gen.with_empty_rows(gen.uniform(2000, 7, 3), 0.3, 4),
    lambda: gen.giant_row(4001, 3990, 3, 5), lambda: gen.config_graph("reddit", 0.01),
    lambda: gen.config_graph("cora")])
def test_transpose_bit_exact(make):
    import torch
    from paper_2605_15695_b200 import api
    g = make()
    rp, ci, vl = dev(g)
    t_rp, t_ci, t_vl = api.pspmm_csr_transpose(g.n, g.n, rp, ci, vl)
    torch.cuda.synchronize()
    w_rp, w_ci, w_vl = brute_transpose(g, g.n)
    assert np.array_equal(t_rp.cpu().numpy(), w_rp)
    assert np.array_equal(t_ci.cpu().numpy(), w_ci)
    assert np.array_equal(t_vl.cpu().numpy().view(np.uint32), w_vl.view(np.uint32))


def test_transpose_rectangular_and_empty():
    import torch
    from paper_2605_15695_b200 import api
    g = gen.uniform(500, 6, 9)
    rp, ci, vl = dev(g)
    t_rp, t_ci, t_vl = api.pspmm_csr_transpose(g.n, 800, rp, ci, vl)  # n_cols > max column
    w_rp, w_ci, _ = brute_transpose(g, 800)
    assert np.array_equal(t_rp.cpu().numpy(), w_rp) and np.array_equal(t_ci.cpu().numpy(), w_ci)
    e = gen.Graph("e", 10, np.zeros(11, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float32))
    rp, ci, vl = dev(e)
    t_rp, _, _ = api.pspmm_csr_transpose(10, 10, rp, ci, vl)
    assert not t_rp.cpu().numpy().any()


@pytest.mark.parametrize("V,S", [(1, 0), (1, 1), (2, 1)])
def test_backward_spmm(V, S):
    """dB = A^T dC: transpose on the GPU, PCSR + engine, vs the oracle."""
    import torch
    from paper_2605_15695_b200 import api
    g = gen.powerlaw(3001, 12, 2.0, 2)
    K = 64
    dC = gen.dense(g.n, K, 11)
    rp, ci, vl = dev(g)
    t_rp, t_ci, t_vl = api.pspmm_csr_transpose(g.n, g.n, rp, ci, vl)
    A_T = api.pspmm_pcsr_build(g.n, g.nnz, t_rp, t_ci, t_vl, V, S)
    out = torch.empty((g.n, K), device="cuda")
    A_T.run(torch.from_numpy(dC).cuda(), out, api.Config(V=V, S=S))
    torch.cuda.synchronize()
    w_rp, w_ci, w_vl = brute_transpose(g, g.n)
    ref, mag = oracle.spmm(w_rp, w_ci, w_vl, dC)
    assert_parity(out.cpu().numpy(), ref, mag, f"backward V{V} S{S}")
