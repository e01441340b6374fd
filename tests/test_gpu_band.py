"""(a6 on locality-ordered graphs) Engine mode 6 — 128-row blocks
whose touched B-row ranges are staged in shared memory by bulk copies —
against the fp64 oracle (c-1 bound, every element): staged and over-budget
(global-gather) blocks, K tails, padded leading dimensions, accumulate,
rectangular A, the host entry and the error surface
(include/pspmm.h, pspmm_pcsr_attach_band)."""
import numpy as np
import pytest

import gen
from gpu_util import assert_parity, dev, oracle_ref

pytestmark = pytest.mark.gpu


def _graph_rect(n, nc, density, seed, band=None):
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for i in range(n):
        if band is None:
            c = np.nonzero(rng.random(nc) < density)[0]
        else:
            lo, hi = max(0, i - band), min(nc, i + band + 1)
            c = lo + np.nonzero(rng.random(hi - lo) < density)[0]
        rows.append(np.full(len(c), i))
        cols.append(c)
    r, c = np.concatenate(rows), np.concatenate(cols)
    rp = np.zeros(n + 1, np.int32)
    rp[1:] = np.cumsum(np.bincount(r, minlength=n))
    return gen.Graph(f"rect{n}_{seed}", n, rp, c.astype(np.int32),
                     gen.values(len(c), seed + 1), 0)


GRAPHS = {
    "roadnet_small": lambda: gen.config_graph("roadnet", 0.01),
    "banded": lambda: gen.banded(5000, 6, 3, fill=0.7),
    "community": lambda: gen.community(3000, 128, 20, 0.9, 5),
    "shuffled": lambda: gen.uniform(4000, 12, 6),              # bands over budget
    "hubs": lambda: gen.powerlaw(3000, 20, 1.8, 7),            # rows longer than G
    "empty_rows": lambda: gen.with_empty_rows(gen.banded(2000, 4, 9, fill=0.8), 0.4, 10),
    "wide_band": lambda: _graph_rect(700, 700, 0.3, 11, band=200),
}


def _run(g, K, k_max=None, pad=0, accumulate=False, n_cols=None, seed=3):
    import torch
    from paper_2605_15695_b200 import api
    rp, ci, vl = dev(g)
    nc = n_cols or g.n
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0, n_cols=nc)
    frac = api.pspmm_pcsr_attach_band(A, k_max or max(4, K + pad))
    B = gen.dense(nc, K, seed)
    Bb = torch.zeros((nc, K + pad), device="cuda")
    Bb[:, :K] = torch.from_numpy(B).cuda()
    Cb = torch.full((g.n, K + pad), float("nan"), device="cuda")
    C0 = None
    if accumulate:
        C0 = gen.dense(g.n, K, seed + 5)
        Cb[:, :K] = torch.from_numpy(C0).cuda()
        api.pspmm_spmm_accumulate(A, Bb[:, :K], Cb[:, :K], api.Config(mode=6))
    else:
        A.run(Bb[:, :K], Cb[:, :K], api.Config(mode=6))
    torch.cuda.synchronize()
    return A, frac, B, Cb.cpu().numpy(), C0


@pytest.mark.parametrize("name", list(GRAPHS))
@pytest.mark.parametrize("K", [4, 16, 32, 48, 64, 128])
def test_band_engine_parity(name, K):
    g = GRAPHS[name]()
    _, frac, B, C, _ = _run(g, K)
    ref, mag = oracle_ref(g, B)
    assert_parity(C[:, :K], ref, mag, f"mode 6 {name} K={K}")
    assert 0.0 <= frac <= 1.0
    if name in ("roadnet_small", "banded"):
        assert frac == 1.0
    if name == "shuffled" and K >= 8:
        assert frac < 0.5  # the global-gather path is exercised (4000 rows x K x 4 B > 64 KB)


@pytest.mark.parametrize("name", ["roadnet_small", "shuffled", "hubs"])
def test_band_engine_accumulate_and_padded_ld(name):
    """C += A.B with ldb = ldc = K + 4 <= k_max; columns past K untouched."""
    g = GRAPHS[name]()
    _, _, B, C, C0 = _run(g, 28, k_max=32, pad=4, accumulate=True)
    ref, mag = oracle_ref(g, B)
    assert_parity(C[:, :28], ref + C0, mag + np.abs(C0), f"mode 6 accumulate {name}")
    assert np.isnan(C[:, 28:]).all()


def test_band_engine_rectangular():
    """n_cols != n (a shard's gathered B)."""
    g = _graph_rect(500, 1700, 0.01, 12, band=None)
    g2 = _graph_rect(600, 900, 0.2, 13, band=20)
    for gg, nc in ((g, 1700), (g2, 900)):
        _, _, B, C, _ = _run(gg, 32, n_cols=nc)
        ref, mag = oracle_ref(gg, B)
        assert_parity(C, ref, mag, f"mode 6 rect {gg.name}")


def test_band_engine_all_positive_long_rows():
    """c-24 stress: all-positive values, rows of ~2000 nonzeros in one band."""
    g = _graph_rect(400, 2400, 0.85, 14, band=1200)
    g.val = gen.values(g.nnz, 15, "positive")
    B2 = np.abs(gen.dense(2400, 64, 16))
    import torch
    from paper_2605_15695_b200 import api
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0, n_cols=2400)
    api.pspmm_pcsr_attach_band(A, 64)
    Cd = torch.empty((g.n, 64), device="cuda")
    A.run(torch.from_numpy(B2).cuda(), Cd, api.Config(mode=6))
    torch.cuda.synchronize()
    ref, mag = oracle_ref(g, B2)
    assert_parity(Cd.cpu().numpy(), ref, mag, "mode 6 all-positive")


def test_band_errors_and_host_entry():
    import torch
    from paper_2605_15695_b200 import api
    g = GRAPHS["banded"]()
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
    B = torch.from_numpy(gen.dense(g.n, 32, 1)).cuda()
    C = torch.empty((g.n, 32), device="cuda")
    with pytest.raises(api.PspmmError) as e:  # no pack attached
        A.run(B, C, api.Config(mode=6))
    assert e.value.status == api.PSPMM_ERR_UNSUPPORTED
    for bad in (0, 3, 132, 256):
        with pytest.raises(api.PspmmError) as e:
            api.pspmm_pcsr_attach_band(A, bad)
        assert e.value.status == api.PSPMM_ERR_INVALID_ARG
    api.pspmm_pcsr_attach_band(A, 16)
    with pytest.raises(api.PspmmError) as e:  # K > k_max
        A.run(B, C, api.Config(mode=6))
    assert e.value.status == api.PSPMM_ERR_UNSUPPORTED
    A2 = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 2, 0)
    with pytest.raises(api.PspmmError) as e:
        api.pspmm_pcsr_attach_band(A2, 32)
    assert e.value.status == api.PSPMM_ERR_UNSUPPORTED
    # host end-to-end entry runs mode 6 whole
    api.pspmm_pcsr_attach_band(A, 32)
    Bh = gen.dense(g.n, 32, 21)
    hB = torch.from_numpy(Bh).pin_memory()
    hC = torch.empty((g.n, 32)).pin_memory()
    api.pspmm_spmm_run_host(A, hB, hC, api.Config(mode=6), B, C)
    ref, mag = oracle_ref(g, Bh)
    assert_parity(hC.numpy(), ref, mag, "mode 6 host entry")
