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
