"""(a6, "B's data reuse through ... shared memory") Engine mode 5 — row
blocks of 15 x rw rows with every touched 128-row window of B staged in
shared memory by TMA — against the fp64 oracle (c-1 bound, every element), the
device-computed reuse against its definition written out in numpy, the rule,
and the error surface (include/pspmm.h, pspmm_pcsr_attach_blocks)."""
import numpy as np
import pytest

import gen
from gpu_util import assert_parity, dev, oracle_ref

pytestmark = pytest.mark.gpu


def _reuse_def(g, block_rows=128):
    """nnz / (sum over row blocks of touched 128-column windows x 128)."""
    rows = np.repeat(np.arange(g.n), np.diff(g.rowptr))
    key = (rows // block_rows).astype(np.int64) * (1 << 32) + g.colidx // 128
    touched = len(np.unique(key))
    return g.nnz / (touched * 128.0) if touched else 0.0, touched


def _run(g, K, seed=3, accumulate=False, ld_pad=0, n_cols=None, runs=1):
    import torch
    from paper_2605_15695_b200 import api
    rp, ci, vl = dev(g)
    nc = n_cols or g.n
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0, n_cols=nc)
    windows = api.pspmm_pcsr_attach_blocks(A)
    B = gen.dense(nc, K, seed)
    Bp = np.zeros((nc, K + ld_pad), np.float32)
    Bp[:, :K] = B
    Bd = torch.from_numpy(Bp).cuda()[:, :K]
    C0 = gen.dense(g.n, K, seed + 7) if accumulate else None
    Cbuf = torch.full((g.n, K + ld_pad), float("nan"), device="cuda")
    C = Cbuf[:, :K]
    if accumulate:
        C.copy_(torch.from_numpy(C0))
        api.pspmm_spmm_accumulate(A, Bd, C, api.Config(mode=5))
    outs = []
    for _ in range(runs if not accumulate else 0):
        A.run(Bd, C, api.Config(mode=5))
        torch.cuda.synchronize()
        outs.append(C.cpu().numpy().copy())
    torch.cuda.synchronize()
    return A, windows, B, (C.cpu().numpy() if accumulate else outs[-1]), C0, outs


def _graph(n, rows, cols, seed, kind="uniform"):
    rp, ci = gen.csr_from_pairs(n, np.asarray(rows, np.int64), np.asarray(cols, np.int64))
    return gen.Graph(f"g{n}_{seed}", n, rp, ci, gen.values(int(rp[-1]), seed, kind), 0)


GRAPHS = {
    "proteins_small": lambda: gen.config_graph("proteins", 0.03),
    "clustered_small": lambda: gen.config_graph("proteins_clustered", 0.02),
    "community": lambda: gen.community(1000, 256, 40, 0.8, 5),
    "uniform": lambda: gen.uniform(700, 12, 6),
    "powerlaw_hubs": lambda: gen.powerlaw(900, 20, 1.8, 7),
    "giant_row": lambda: gen.giant_row(600, 590, 3, 8),
    "empty_rows": lambda: gen.with_empty_rows(gen.community(520, 128, 30, 0.9, 9), 0.4, 10),
    "full_window": lambda: _graph(300, *np.nonzero(np.ones((300, 300), bool)), seed=11),
}


@pytest.mark.parametrize("name", list(GRAPHS))
@pytest.mark.parametrize("K", [128, 256])
def test_block_engine_parity(name, K):
    g = GRAPHS[name]()
    A, windows, B, C, _, _ = _run(g, K)
    ref, mag = oracle_ref(g, B)
    assert_parity(C, ref, mag, f"mode 5 {name} K={K}")
    from paper_2605_15695_b200 import api
    rows, w = api.pspmm_block_info(A)
    assert rows in (120, 152, 184, 240) and w == windows
    r, touched = _reuse_def(g, rows)
    assert windows == touched


@pytest.mark.parametrize("rw,nw", [("16", "15"), ("8", "19"), ("8", "15")])
@pytest.mark.parametrize("name", ["clustered_small", "giant_row", "empty_rows", "full_window"])
def test_block_engine_instances(name, rw, nw, monkeypatch):
    """The other kernel instances (rows per warp x consumer warps), chosen by
    the tools' A/B knobs."""
    monkeypatch.setenv("PSPMM_BLOCK_RW", rw)
    monkeypatch.setenv("PSPMM_BLOCK_NW", nw)
    g = GRAPHS[name]()
    A, windows, B, C, _, _ = _run(g, 128)
    from paper_2605_15695_b200 import api
    assert api.pspmm_block_info(A)[0] == int(rw) * int(nw)
    ref, mag = oracle_ref(g, B)
    assert_parity(C, ref, mag, f"mode 5 rw={rw} nw={nw} {name}")


@pytest.mark.parametrize("name", ["proteins_small", "uniform", "empty_rows"])
def test_block_reuse_matches_definition(name):
    from paper_2605_15695_b200 import api
    g = GRAPHS[name]()
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
    r, _ = _reuse_def(g)
    assert api.pspmm_block_reuse(A) == pytest.approx(r, rel=1e-12)


def test_block_engine_accumulate_ld_and_wide_K():
    """C += A.B, padded leading dimensions, K = 384 (three column slices)."""
    g = GRAPHS["community"]()
    A, _, B, C, C0, _ = _run(g, 384, accumulate=True, ld_pad=4)
    ref, mag = oracle_ref(g, B)
    assert_parity(C, ref + C0, mag + np.abs(C0), "mode 5 accumulate K=384 ld=K+4")


def test_block_engine_rectangular_and_deterministic():
    """n_cols != n (a shard's gathered B), ragged last window; two runs are
    bit-identical (one writer per element, fixed summation order)."""
    rng = np.random.default_rng(12)
    n, nc = 333, 1000
    m = rng.random((n, nc)) < 0.05
    r, c = np.nonzero(m)  # row-major: rows ascending, columns ascending within a row
    rp = np.zeros(n + 1, np.int32)
    rp[1:] = np.cumsum(np.bincount(r, minlength=n))
    ci = c.astype(np.int32)
    g = gen.Graph("rect", n, rp, ci, gen.values(int(rp[-1]), 13), 0)
    A, _, B, C, _, outs = _run(g, 128, n_cols=nc, runs=2)
    ref = oracle_ref(g, B)
    assert_parity(C, *ref, "mode 5 rectangular")
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))


def test_block_engine_all_positive_long_rows():
    """c-24 stress: all-positive values, rows of ~3000 nonzeros inside one
    3000-column block (24 windows per row)."""
    rng = np.random.default_rng(14)
    n = 3000
    m = rng.random((n, n)) < 0.9
    r, c = np.nonzero(m)
    rp, ci = gen.csr_from_pairs(n, r.astype(np.int64), c.astype(np.int64))
    g = gen.Graph("pos", n, rp, ci, gen.values(int(rp[-1]), 15, "positive"), 0)
    import torch
    from paper_2605_15695_b200 import api
    d = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, *d, 1, 0)
    api.pspmm_pcsr_attach_blocks(A)
    B = np.abs(gen.dense(n, 128, 16))
    C = torch.empty((n, 128), device="cuda")
    A.run(torch.from_numpy(B).cuda(), C, api.Config(mode=5))
    torch.cuda.synchronize()
    ref, mag = oracle_ref(g, B)
    assert_parity(C.cpu().numpy(), ref, mag, "mode 5 all-positive")


def test_block_rule_and_errors():
    import torch
    from paper_2605_15695_b200 import api
    g = GRAPHS["proteins_small"]()
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
    B = torch.from_numpy(gen.dense(g.n, 128, 1)).cuda()
    C = torch.empty((g.n, 128), device="cuda")
    with pytest.raises(api.PspmmError) as e:  # no pack attached
        A.run(B, C, api.Config(mode=5))
    assert e.value.status == api.PSPMM_ERR_UNSUPPORTED
    assert api.pspmm_decide_blocks(A, 128, 2.0, api.Config(mode=5)).mode == 0
    api.pspmm_pcsr_attach_blocks(A)
    assert api.pspmm_decide_blocks(A, 128, 2.0, api.Config()).mode == 5
    assert api.pspmm_decide_blocks(A, 64, 2.0, api.Config()).mode == 0      # K % 128
    assert api.pspmm_decide_blocks(A, 128, 1e9, api.Config(mode=5)).mode == 0
    B64 = torch.from_numpy(gen.dense(g.n, 64, 1)).cuda()
    with pytest.raises(api.PspmmError) as e:
        A.run(B64, torch.empty((g.n, 64), device="cuda"), api.Config(mode=5))
    assert e.value.status == api.PSPMM_ERR_UNSUPPORTED
    A2 = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 2, 0)
    with pytest.raises(api.PspmmError) as e:
        api.pspmm_pcsr_attach_blocks(A2)
    assert e.value.status == api.PSPMM_ERR_UNSUPPORTED
    # the auto path picks mode 5 on the species-block shape
    cfg, H, info = api.auto_blocks(A2, rp, ci, vl, 256, api.Config(V=2, S=0))
    assert info["taken"] and cfg.mode == 5 and H.V == 1, info


def test_block_host_entry():
    """The host end-to-end entry runs mode 5 whole (no slices)."""
    import torch
    from paper_2605_15695_b200 import api
    g = GRAPHS["community"]()
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
    api.pspmm_pcsr_attach_blocks(A)
    B = gen.dense(g.n, 128, 21)
    hB = torch.from_numpy(B).pin_memory()
    hC = torch.empty((g.n, 128)).pin_memory()
    dB = torch.empty((g.n, 128), device="cuda")
    dC = torch.empty((g.n, 128), device="cuda")
    api.pspmm_spmm_run_host(A, hB, hC, api.Config(mode=5), dB, dC)
    ref, mag = oracle_ref(g, B)
    assert_parity(hC.numpy(), ref, mag, "mode 5 host entry")
