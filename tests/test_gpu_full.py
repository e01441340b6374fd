"""Full-size BASELINE.json configs on the GPU, in the launch configuration
bench.py times: PCSR bit-exact against the oracle's arrays, and SpMM checked
element by element against the oracle on sampled rows (all rows for Cora):
random rows, the heaviest rows, split-panel rows, first and last rows."""
import numpy as np
import pytest

import gen
import oracle
from gpu_util import assert_parity, dev

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def sample_rows(g, count, seed):
    rng = np.random.default_rng(seed)
    deg = np.diff(g.rowptr.astype(np.int64))
    heavy = np.argsort(deg)[-32:]
    rows = np.concatenate([rng.choice(g.n, size=min(count, g.n), replace=False), heavy,
                           [0, 1, g.n - 2, g.n - 1]])
    return np.unique(rows).astype(np.int64)


@pytest.mark.parametrize("name", ["cora", "roadnet", "reddit", "proteins", "products",
                                  "proteins_clustered"])
def test_full_config(name):
    import torch
    from paper_2605_15695_b200 import api
    g = gen.config_graph(name)
    K = g.K
    rp, ci, vl = dev(g)
    cfg = api.auto_config(g.n, g.nnz, rp, ci, K)  # what bench.py runs
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega, cfg.sg_override)
    # PCSR bit-exact at full size
    ref = oracle.pcsr_build(g.rowptr, g.colidx, g.val, cfg.V, cfg.S, cfg.omega, cfg.sg_override)
    e = A.export()
    assert np.array_equal(e["rowPtr"], ref["rowPtr"])
    assert np.array_equal(e["colIdx"], ref["colIdx"])
    assert np.array_equal(e["val"].view(np.uint32), ref["val"].view(np.uint32))
    assert np.array_equal(e["TRow"], ref["TRow"])
    del e, ref
    cfg, dense = api.auto_dense(A, rp, ci, vl, K, cfg)  # engine mode 1 rule, as bench.py
    if name == "proteins_clustered":
        assert cfg.mode == 1 and dense["nnz_dense"] > 0.3 * g.nnz
    cfg, A, blocks = api.auto_blocks(A, rp, ci, vl, K, cfg)  # engine mode 5 rule, as bench.py
    if name == "proteins":
        assert cfg.mode == 5 and blocks["taken"], blocks
    cfg, A, band = api.auto_band(A, rp, ci, vl, K, cfg)  # engine mode 6 rule, as bench.py
    if name == "roadnet":
        assert cfg.mode == 6 and band["taken"], band
    # SpMM, sampled rows (every row for Cora)
    B = gen.config_B(name, g.n)
    Bd = torch.from_numpy(B).cuda()
    C = torch.full((g.n, K), float("nan"), device="cuda")
    A.run(Bd, C, cfg)
    torch.cuda.synchronize()
    Ch = C.cpu().numpy()
    assert np.isfinite(Ch).all()
    rows = None if g.n < 10000 else sample_rows(g, 3000, 7)
    refC, mag = oracle.spmm(g.rowptr, g.colidx, g.val, B, rows=rows, threads=16)
    got = Ch if rows is None else Ch[rows]
    assert_parity(got, refC, mag, f"{name} full size {cfg}")
