"""(e) Multi-GPU path in single-GPU simulated-shard mode: all P shards run
sequentially on one device, the all-gather replaced by the same padded
layout built with local copies.  The gathered C must match the full-graph
oracle (c-5).  (Real NCCL runs need P GPUs; the CPU gloo test covers the
collective plumbing.)"""
import numpy as np
import pytest

import gen
from gpu_util import assert_parity, oracle_ref

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 2, 3])
@pytest.mark.parametrize("V,S", [(1, 0), (1, 1), (2, 0), (2, 1)])
def test_spmm_accumulate(mode, V, S):
    """pspmm_spmm_accumulate: C0 + A.B for every engine / PCSR corner."""
    import torch
    from paper_2605_15695_b200 import api
    from gpu_util import dev
    if mode == 3 and (V, S) != (1, 0):
        pytest.skip("mode 3 is V = 1, S = 0 only")
    g = gen.config_graph("reddit", 0.01)
    K = 64
    B = gen.dense(g.n, K, 6006)
    C0 = gen.dense(g.n, K, 6007)
    ref, mag = oracle_ref(g, B, key=("reddit_s_acc", K))
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, S, 32, 64 if S else 0)
    C = torch.from_numpy(C0).cuda()
    api.pspmm_spmm_accumulate(A, torch.from_numpy(B).cuda(), C, api.Config(V=V, S=S, mode=mode))
    torch.cuda.synchronize()
    assert_parity(C.cpu().numpy(), ref + C0.astype(np.float64), mag + np.abs(C0), "accumulate")


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("V,S", [(1, 0), (1, 1), (2, 1)])
def test_simulated_overlap_split(P, V, S):
    """The overlapped step's math: own-column block on the local B rows, then
    the remote block accumulated with the gathered B, equals the full SpMM."""
    import torch
    from paper_2605_15695_b200 import api, dist
    g = gen.config_graph("reddit", 0.01)
    K = 64
    B = gen.dense(g.n, K, 5005)
    ref, mag = oracle_ref(g, B, key=("reddit_s_dist", K))
    shards = [dist.make_shard(g.rowptr, g.colidx, g.val, P, r, align=2) for r in range(P)]
    n_max = shards[0].n_max
    Bd = torch.from_numpy(B).cuda()
    B_full = torch.cat([dist.pad_rows(Bd[s.lo:s.hi], n_max) for s in shards], 0)
    outs = []
    for s in shards:
        cfg = api.Config(V=V, S=S, W=4)
        run = dist.ShardedSpmm(s, K, cfg)
        assert run.A_own is not None
        B_loc = dist.pad_rows(Bd[s.lo:s.hi], n_max)
        run.A_own.run(B_loc, run.C, cfg)
        if run.A_rem is not None:
            api.pspmm_spmm_accumulate(run.A_rem, B_full, run.C, cfg)
        outs.append(run.C.clone())
    C_full = dist.unpad_gathered(torch.cat(outs, 0), shards[0].bounds, n_max)
    torch.cuda.synchronize()
    assert_parity(C_full.cpu().numpy(), ref, mag, f"overlap split P{P} V{V} S{S}")


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("V,S", [(1, 0), (1, 1), (2, 0), (2, 1)])
def test_simulated_shards(P, V, S):
    import torch
    from paper_2605_15695_b200 import api, dist
    g = gen.config_graph("reddit", 0.01)
    K = 64
    B = gen.dense(g.n, K, 5005)
    ref, mag = oracle_ref(g, B, key=("reddit_s_dist", K))
    shards = [dist.make_shard(g.rowptr, g.colidx, g.val, P, r, align=2) for r in range(P)]
    n_max = shards[0].n_max
    Bd = torch.from_numpy(B).cuda()
    B_full = torch.cat([dist.pad_rows(Bd[s.lo:s.hi], n_max) for s in shards], 0)
    outs = []
    for s in shards:
        cfg = api.Config(V=V, S=S, W=4)
        run = dist.ShardedSpmm(s, K, cfg)
        run.B_full.copy_(B_full)              # what the all-gather produces
        run.A.run(run.B_full, run.C, cfg)
        outs.append(run.C.clone())
    C_full = dist.unpad_gathered(torch.cat(outs, 0), shards[0].bounds, n_max)
    torch.cuda.synchronize()
    assert_parity(C_full.cpu().numpy(), ref, mag, f"P{P} V{V} S{S}")
    # nnz balance: no shard holds more than its share plus one row
    deg = np.diff(g.rowptr.astype(np.int64))
    for s in shards:
        assert g.rowptr[s.hi] - g.rowptr[s.lo] <= -(-g.nnz // P) + 2 * deg.max()
