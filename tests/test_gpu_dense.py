"""(a6, conditional) Engine mode 1 — dense 128 x 32 tiles on tcgen05
(kind::tf32, 3xTF32) plus the rest on the mode-0 engine — against the fp64
oracle (c-1 bound), the split's tile counts against a numpy count of the
same definition (include/pspmm.h, pspmm_pcsr_attach_dense), and the error
surface."""
import numpy as np
import pytest

import gen
from gpu_util import assert_parity, dev, oracle_ref

pytestmark = pytest.mark.gpu


def _graph(n, rows, cols, seed, kind="uniform"):
    rp, ci = gen.csr_from_pairs(n, np.asarray(rows, np.int64), np.asarray(cols, np.int64))
    return gen.Graph(f"g{n}_{seed}", n, rp, ci, gen.values(int(rp[-1]), seed, kind), 0)


def _dense_block(n, density, seed):
    rng = np.random.default_rng(seed)
    m = rng.random((n, n)) < density
    r, c = np.nonzero(m)
    return _graph(n, r, c, seed)


def _community(n, csize, d, p_in, seed, kind="uniform"):
    g = gen.community(n, csize, d, p_in, seed, kind=kind)
    return g


def _tile_counts(g, thr):
    """(panels with dense tiles, dense tiles, nnz inside them) — the split's
    definition written out: 128 x 32 tiles with >= thr nonzeros."""
    rows = np.repeat(np.arange(g.n), np.diff(g.rowptr))
    key = (rows // 128).astype(np.int64) * ((g.n + 31) // 32 + 1) + g.colidx // 32
    u, cnt = np.unique(key, return_counts=True)
    dense = cnt >= thr
    stride = (g.n + 31) // 32 + 1
    return len(np.unique(u[dense] // stride)), int(dense.sum()), int(cnt[dense].sum())


def _run(g, K, cfg_kw, min_density, seed=2, accumulate=False, B=None):
    import torch
    from paper_2605_15695_b200 import api
    rp, ci, vl = dev(g)
    cfg = api.Config(mode=1, **cfg_kw)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S)
    info = api.pspmm_pcsr_attach_dense(A, rp, ci, vl, min_density, k_max=max(16, -(-K // 16) * 16))
    if B is None:
        B = gen.dense(g.n, K, seed)
    Bd = torch.from_numpy(B).cuda()
    C0 = gen.dense(g.n, K, seed + 7) if accumulate else None
    C = torch.from_numpy(C0).cuda() if accumulate else torch.full((g.n, K), float("nan"),
                                                                   device="cuda")
    if accumulate:
        api.pspmm_spmm_accumulate(A, Bd, C, cfg)
    else:
        A.run(Bd, C, cfg)
    torch.cuda.synchronize()
    return A, info, B, C.cpu().numpy(), C0


@pytest.mark.parametrize("n", [128, 200, 300])
@pytest.mark.parametrize("K", [16, 32, 48, 256, 272])
def test_dense_block_all_tiles(n, K):
    """A dense random block: every tile goes to the tensor cores (ragged
    last panel / tile, N passes of 256 + 16 at K = 272)."""
    g = _dense_block(n, 0.6, seed=n + K)
    A, info, B, C, _ = _run(g, K, dict(W=2, F=1), min_density=1 / 4096)
    ref, mag = oracle_ref(g, B)
    assert info["nnz_dense"] == g.nnz
    assert_parity(C, ref, mag, f"dense block n={n} K={K}")


@pytest.mark.parametrize("thr_frac", [1 / 4096, 0.05, 0.2, 0.5, 1.0])
@pytest.mark.parametrize("VS", [(1, 0), (1, 1), (2, 0), (2, 1)])
def test_community_split(thr_frac, VS):
    """Community graph (dense diagonal blocks + uniform rest): tile counts
    equal the definition; C matches the oracle for every split."""
    V, S = VS
    g = _community(3000, 256, 60, 0.6, seed=41)
    K = 64
    A, info, B, C, _ = _run(g, K, dict(W=4, F=1, V=V, S=S), min_density=thr_frac)
    thr = max(1, int(np.ceil(thr_frac * 4096 - 1e-9)))
    panels, tiles, nnz_dense = _tile_counts(g, thr)
    assert (info["num_panels"], info["num_tiles"], info["nnz_dense"]) == (panels, tiles, nnz_dense)
    ref, mag = oracle_ref(g, B, key=("comm3000", K))
    assert_parity(C, ref, mag, f"community thr={thr_frac} V={V} S={S}")


def test_integer_exact():
    """Small-integer A and B: every TF32 hi part is exact and every lo part
    zero, so the 3xTF32 products and fp32 sums are exact — bit-equal to the
    fp64 oracle."""
    g = _community(1024, 128, 40, 0.8, seed=5, kind="int")
    B = gen.dense(g.n, 128, 6, kind="int")
    A, info, B, C, _ = _run(g, 128, dict(W=2, F=2), min_density=0.02, B=B)
    assert info["num_tiles"] > 0
    ref, _ = oracle_ref(g, B)
    assert np.array_equal(C.astype(np.float64), ref)


def test_all_positive_long_rows():
    """c-24 stress: all-positive values, rows of ~1000 nonzeros, mostly dense."""
    g = _community(2048, 1024, 900, 0.9, seed=9, kind="ones")
    B = np.abs(gen.dense(g.n, 64, 10))
    A, info, B, C, _ = _run(g, 64, dict(W=2, F=1), min_density=0.1, B=B)
    assert info["num_tiles"] > 0
    ref, mag = oracle_ref(g, B)
    assert_parity(C, ref, mag, "all-positive long rows")


def test_accumulate_mode1():
    g = _community(1500, 256, 50, 0.7, seed=13)
    A, info, B, C, C0 = _run(g, 32, dict(W=2, F=1), min_density=0.03, accumulate=True)
    ref, mag = oracle_ref(g, B)
    assert_parity(C, ref + C0.astype(np.float64), mag + np.abs(C0), "accumulate mode 1")


def test_mode1_errors():
    import torch
    from paper_2605_15695_b200 import api
    g = _community(600, 128, 30, 0.7, seed=3)
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
    B = torch.from_numpy(gen.dense(g.n, 32, 1)).cuda()
    C = torch.empty((g.n, 32), device="cuda")
    cfg = api.Config(W=2, F=1, mode=1)
    with pytest.raises(api.PspmmError) as e:  # nothing attached
        A.run(B, C, cfg)
    assert e.value.status == 7
    for bad in (0.0, -1.0, 1.5):
        with pytest.raises(api.PspmmError) as e:
            api.pspmm_pcsr_attach_dense(A, rp, ci, vl, bad)
        assert e.value.status == 1
    for bad_k in (0, 8, 24):
        with pytest.raises(api.PspmmError) as e:
            api.pspmm_pcsr_attach_dense(A, rp, ci, vl, 0.05, k_max=bad_k)
        assert e.value.status == 1
    api.pspmm_pcsr_attach_dense(A, rp, ci, vl, 0.05, k_max=32)
    B48 = torch.from_numpy(gen.dense(g.n, 48, 1)).cuda()
    C48 = torch.empty((g.n, 48), device="cuda")
    with pytest.raises(api.PspmmError) as e:  # K > k_max
        A.run(B48, C48, cfg)
    assert e.value.status == 7
    B24 = torch.from_numpy(gen.dense(g.n, 24, 1)).cuda()
    C24 = torch.empty((g.n, 24), device="cuda")
    with pytest.raises(api.PspmmError) as e:  # K % 16 != 0
        A.run(B24, C24, cfg)
    assert e.value.status == 7
    # re-attaching replaces the split; destroy frees both
    info = api.pspmm_pcsr_attach_dense(A, rp, ci, vl, 1.0)
    assert info["num_tiles"] == 0
    A.run(B, C, cfg)
    torch.cuda.synchronize()
    ref, mag = oracle_ref(g, B.cpu().numpy())
    assert_parity(C.cpu().numpy(), ref, mag, "no dense tiles")
    A.close()


def test_empty_matrix_mode1():
    import torch
    from paper_2605_15695_b200 import api
    g = _graph(300, [], [], 1)
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, 0, rp, ci, vl, 1, 0)
    info = api.pspmm_pcsr_attach_dense(A, rp, ci, vl, 0.1)
    assert info == {"num_panels": 0, "num_tiles": 0, "nnz_dense": 0}
    B = torch.ones((300, 16), device="cuda")
    C = torch.full((300, 16), 5.0, device="cuda")
    A.run(B, C, api.Config(W=2, F=1, mode=1))
    torch.cuda.synchronize()
    assert float(C.abs().max()) == 0.0


@pytest.mark.parametrize("kind", ["community", "uniform"])
def test_decide_dense_rule(kind):
    """pspmm_decide_dense: mode 1 iff the >= 10 %-dense tiles hold >= 5 % of
    the nonzeros; the decided config (rest knobs from the rest's features)
    matches the oracle."""
    import torch
    from paper_2605_15695_b200 import api
    g = _community(4096, 512, 120, 0.8, seed=21) if kind == "community" else \
        gen.uniform(4096, 40, 22)
    K = 64
    rp, ci, vl = dev(g)
    cfg = api.auto_config(g.n, g.nnz, rp, ci, K)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S)
    cfg2, info = api.auto_dense(A, rp, ci, vl, K, cfg)
    thr = int(np.ceil(0.1 * 4096))
    _, tiles, nnz_dense = _tile_counts(g, thr)
    assert info["num_tiles"] == tiles and info["nnz_dense"] == nnz_dense
    assert (cfg2.mode == 1) == (tiles > 0 and nnz_dense >= 0.05 * g.nnz)
    assert cfg2.mode == (1 if kind == "community" else cfg.mode)
    assert (cfg2.V, cfg2.S) == (cfg.V, cfg.S)
    B = gen.dense(g.n, K, 3)
    C = torch.full((g.n, K), float("nan"), device="cuda")
    A.run(torch.from_numpy(B).cuda(), C, cfg2)
    torch.cuda.synchronize()
    ref, mag = oracle_ref(g, B)
    assert_parity(C.cpu().numpy(), ref, mag, f"decided {cfg2}")
    # K % 16 != 0 never takes mode 1
    assert api.pspmm_decide_dense(A, 40, 0.05, cfg).mode != 1


def test_host_entries_mode1():
    """The host entries run mode 1 whole: pspmm_spmm_run_host and the batch
    entry (3 products through two rotating buffer sets)."""
    import torch
    from paper_2605_15695_b200 import api
    g = _community(2000, 256, 60, 0.7, seed=31)
    K = 32
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
    info = api.pspmm_pcsr_attach_dense(A, rp, ci, vl, 0.05, k_max=K)
    assert info["num_tiles"] > 0
    cfg = api.Config(W=2, F=1, mode=1)
    Bs = [gen.dense(g.n, K, 40 + i) for i in range(3)]
    hB = [torch.from_numpy(b).pin_memory() for b in Bs]
    hC = [torch.full((g.n, K), float("nan")).pin_memory() for _ in Bs]
    dB = [torch.empty((g.n, K), device="cuda") for _ in range(2)]
    dC = [torch.empty((g.n, K), device="cuda") for _ in range(2)]
    api.pspmm_spmm_run_host_batch(A, hB, hC, cfg, dB, dC)
    for b, c in zip(Bs, hC):
        ref, mag = oracle_ref(g, b)
        assert_parity(c.numpy(), ref, mag, "host batch mode 1")
    h1 = torch.full((g.n, K), float("nan")).pin_memory()
    api.pspmm_spmm_run_host(A, hB[0], h1, cfg, dB[0], dC[0])
    ref, mag = oracle_ref(g, Bs[0])
    assert_parity(h1.numpy(), ref, mag, "host mode 1")
