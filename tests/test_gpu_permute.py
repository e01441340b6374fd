"""(f1) Device side of reordering: P A P^T bit-exact against the host
definition, dense row permutations, and SpMM(P A P^T, P B) = P SpMM(A, B)
 through the engine, checked against the oracle."""
import numpy as np
import pytest

import gen
import oracle
from gpu_util import assert_parity, dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("strategy", ["bfs", "degree"])
def test_csr_permute_bit_exact(strategy):
    import torch
    from paper_2605_15695_b200 import api
    g = gen.community(5000, 64, 12, 0.85, 3, ordered=False)
    perm = api.pspmm_reorder(g.rowptr, g.colidx, strategy)
    rp, ci, vl = dev(g)
    o_rp, o_ci, o_vl = api.pspmm_csr_permute(rp, ci, vl, torch.from_numpy(perm).cuda())
    # host definition: entry (i, j, v) -> (perm[i], perm[j], v), rows sorted by column
    deg = np.diff(g.rowptr.astype(np.int64))
    rows = np.repeat(np.arange(g.n), deg)
    keys = perm[rows].astype(np.int64) * g.n + perm[g.colidx]
    order = np.argsort(keys, kind="stable")
    w_rows = (keys[order] // g.n)
    w_rp = np.concatenate([[0], np.cumsum(np.bincount(w_rows, minlength=g.n))]).astype(np.int32)
    assert np.array_equal(o_rp.cpu().numpy(), w_rp)
    assert np.array_equal(o_ci.cpu().numpy(), (keys[order] % g.n).astype(np.int32))
    assert np.array_equal(o_vl.cpu().numpy().view(np.uint32), g.val[order].view(np.uint32))


@pytest.mark.parametrize("V,S", [(1, 0), (2, 1)])
def test_spmm_on_reordered_graph(V, S):
    import torch
    from paper_2605_15695_b200 import api
    g = gen.community(6000, 128, 16, 0.9, 4, ordered=False)
    K = 64
    B = gen.dense(g.n, K, 5)
    ref, mag = oracle.spmm(g.rowptr, g.colidx, g.val, B)
    perm = torch.from_numpy(api.pspmm_reorder(g.rowptr, g.colidx, "bfs")).cuda()
    rp, ci, vl = dev(g)
    p_rp, p_ci, p_vl = api.pspmm_csr_permute(rp, ci, vl, perm)
    Bp = api.pspmm_permute_rows(torch.from_numpy(B).cuda(), perm)            # B' = P B
    A = api.pspmm_pcsr_build(g.n, g.nnz, p_rp, p_ci, p_vl, V, S)
    Cp = torch.empty((g.n, K), device="cuda")
    A.run(Bp, Cp, api.Config(V=V, S=S))
    C = api.pspmm_permute_rows(Cp, perm, inverse=True)                        # C = P^T C'
    torch.cuda.synchronize()
    assert_parity(C.cpu().numpy(), ref, mag, f"reordered V{V} S{S}")


def test_reordering_lowers_padding_on_shuffled_communities():
    """reordering creates consecutive nonzeros in the same columns ->
    less zero padding at V = 2 (PR_2 drops)."""
    from paper_2605_15695_b200 import api
    import torch
    g = gen.community(20000, 64, 24, 0.95, 8, ordered=False)
    rp, ci, vl = dev(g)
    pr_before = api.pspmm_features_compute(g.n, g.nnz, rp, ci)["pr2"]
    perm = torch.from_numpy(api.pspmm_reorder(g.rowptr, g.colidx, "bfs")).cuda()
    p_rp, p_ci, _ = api.pspmm_csr_permute(rp, ci, vl, perm)
    pr_after = api.pspmm_features_compute(g.n, g.nnz, p_rp, p_ci)["pr2"]
    assert pr_after < pr_before
