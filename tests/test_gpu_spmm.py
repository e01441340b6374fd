"""(a6, a7) GPU SpMM engine parity against the fp64 oracle (c-1): every
element within |C - C_ref| <= 1e-5 sum|a||b| + 1e-6 (BASELINE.json), over
the kernel family lattice, K values with ragged tails, layouts, and the
degenerate cases."""
import itertools

import numpy as np
import pytest

import gen
import oracle
from gpu_util import assert_parity, dev, oracle_ref

pytestmark = pytest.mark.gpu


def _api():
    from paper_2605_15695_b200 import api
    return api


def _torch():
    import torch
    return torch


def run(g, B, cfg, A=None, C=None, stream=None):
    api, torch = _api(), _torch()
    rp, ci, vl = dev(g)
    if A is None:
        A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega, cfg.sg_override)
    Bd = B if isinstance(B, torch.Tensor) else torch.from_numpy(B).cuda()
    if C is None:
        C = torch.full((g.n, Bd.shape[1]), float("nan"), device="cuda")  # every element must be written
    api.pspmm_spmm_run(A, Bd, C, cfg, stream)
    torch.cuda.synchronize()
    return C.cpu().numpy(), A


G_MAIN = {}


def main_graph():
    if "g" not in G_MAIN:
        # several tiles per warp, hub rows that split under S=1, empty rows, odd n
        G_MAIN["g"] = gen.with_empty_rows(gen.powerlaw(3001, 14, 1.9, 21, d_max=1500), 0.05, 22)
    return G_MAIN["g"]


@pytest.mark.parametrize("V,S", [(1, 0), (1, 1), (2, 0), (2, 1)])
@pytest.mark.parametrize("F", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("G", [1, 2, 4, 8, 16, 32])
def test_every_vector_instance(V, S, F, G):
    """All 192 128-bit kernel instances, K = 64 (several passes for small G F)."""
    api = _api()
    g = main_graph()
    K = 64
    B = gen.dense(g.n, K, 31)
    ref, mag = oracle_ref(g, B, key="main64")
    C, _ = run(g, B, api.Config(W=4, F=F, V=V, S=S, G=G))
    assert_parity(C, ref, mag, f"V{V} S{S} F{F} G{G}")


@pytest.mark.parametrize("V,S", [(1, 0), (1, 1), (2, 0), (2, 1)])
@pytest.mark.parametrize("K", [1, 3, 5, 17, 33, 50])
def test_scalar_variant_odd_K(V, S, K):
    api = _api()
    g = main_graph()
    B = gen.dense(g.n, K, 32)
    ref, mag = oracle_ref(g, B, key=f"main{K}")
    C, _ = run(g, B, api.Config(W=4, V=V, S=S))
    assert_parity(C, ref, mag, f"scalar K{K}")


GRAPHS = {
    "cora": lambda: gen.config_graph("cora"),
    "reddit_s": lambda: gen.config_graph("reddit", 0.01),
    "products_s": lambda: gen.config_graph("products", 0.005),
    "proteins_s": lambda: gen.config_graph("proteins", 0.02),
    "roadnet_s": lambda: gen.config_graph("roadnet", 0.01),
    "giant": lambda: gen.giant_row(4001, 3990, 4, 5),
    "banded": lambda: gen.banded(3001, 6, 6),
    "empty_rows": lambda: gen.with_empty_rows(gen.config_graph("roadnet", 0.004), 0.3, 8),
}
_gcache = {}


def graph(name):
    if name not in _gcache:
        _gcache[name] = GRAPHS[name]()
    return _gcache[name]


@pytest.mark.parametrize("name", sorted(GRAPHS))
@pytest.mark.parametrize("K", [4, 16, 32, 48, 64, 96, 128, 160, 256])
def test_decided_and_alternative_configs(name, K):
    """The decider's config plus the other V/S corners, per K (Table 4 dims)."""
    api = _api()
    g = graph(name)
    B = gen.dense(g.n, K, 40 + K)
    ref, mag = oracle_ref(g, B, key=(name, K, "decided"))
    rp, ci, _ = dev(g)
    f = api.pspmm_features_compute(g.n, g.nnz, rp, ci)
    cfg = api.pspmm_decide_config(f, K)
    cfgs = [cfg] + [api.Config(W=W, F=cfg.F, V=V, S=S, G=cfg.G)
                    for (V, S), W in zip(itertools.product((1, 2), (0, 1)), (1, 2, 4, 8))]
    for c in cfgs:
        C, _ = run(g, B, c)
        assert_parity(C, ref, mag, f"{name} K{K} {c}")


AUTO_GRAPHS = {
    "cora": lambda: gen.config_graph("cora"),
    "roadnet_s": lambda: gen.config_graph("roadnet", 0.02),
    "proteins_s": lambda: gen.config_graph("proteins", 0.05),
    "clustered_s": lambda: gen.config_graph("proteins_clustered", 0.05),
    "reddit_s": lambda: gen.config_graph("reddit", 0.01),
}


@pytest.mark.parametrize("name", sorted(AUTO_GRAPHS))
@pytest.mark.parametrize("K", [32, 128])
def test_api_spmm_full_selection(name, K):
    """api.spmm with no cfg runs the library's full selection (auto_select:
    decider, then the mode-1 / 5 / 6 rules); whatever engine it picks, the
    product matches the oracle, and the handle is reusable."""
    api, torch = _api(), _torch()
    g = AUTO_GRAPHS[name]()
    B = gen.dense(g.n, K, 90 + K)
    ref, mag = oracle.spmm(g.rowptr, g.colidx, g.val, B)
    rp, ci, vl = dev(g)
    Bd = torch.from_numpy(B).cuda()
    C, cfg, A = api.spmm(rp, ci, vl, Bd)
    torch.cuda.synchronize()
    assert_parity(C.cpu().numpy(), ref, mag, f"api.spmm {name} K{K} {cfg}")
    C2 = torch.full_like(C, float("nan"))
    A.run(Bd, C2, cfg)
    torch.cuda.synchronize()
    assert_parity(C2.cpu().numpy(), ref, mag, f"reuse {name} K{K} {cfg}")
    assert cfg.mode in (0, 1, 2, 3, 5, 6)


@pytest.mark.parametrize("V,S", [(1, 0), (1, 1), (2, 0), (2, 1)])
@pytest.mark.parametrize("K", [32, 64, 96, 128, 256, 512])
@pytest.mark.parametrize("W", [1, 4, 8])
def test_tma_gather_engine(V, S, K, W):
    """Engine mode 2 (TMA tile::gather4 into shared memory)."""
    api = _api()
    g = main_graph()
    B = gen.dense(g.n, K, 300 + K)
    ref, mag = oracle_ref(g, B, key=("main_tma", K))
    if W * 8 * (4 * min(K, 256) * 4) > 227 * 1024:  # W warps x 8 slots x 4 rows
        pytest.skip("ring does not fit shared memory at this W")
    C, _ = run(g, B, api.Config(W=W, V=V, S=S, mode=2))
    assert_parity(C, ref, mag, f"tma V{V} S{S} K{K} W{W}")


@pytest.mark.parametrize("mode", [3])
@pytest.mark.parametrize("name", ["roadnet_s", "cora", "giant", "banded", "reddit_s",
                                  "empty_rows"])
@pytest.mark.parametrize("K", [16, 32, 64, 128, 160])
@pytest.mark.parametrize("F", [1, 2, 4])
def test_short_row_engines(mode, name, K, F):
    """Engine mode 3 (V = 1, S = 0): rows of any length (the inner window
    loop), every (F, G) the dispatcher can pick, several column passes
    (K = 160)."""
    api = _api()
    g = graph(name)
    B = gen.dense(g.n, K, 500 + K)
    ref, mag = oracle_ref(g, B, key=(name, K, "short"))
    for W in (2, 8):
        C, _ = run(g, B, api.Config(W=W, F=F, V=1, S=0, mode=mode))
        assert_parity(C, ref, mag, f"mode {mode} {name} K{K} F{F} W{W}")


@pytest.mark.parametrize("mode", [3])
def test_short_row_engine_rejects_other_corners(mode):
    api = _api()
    g = graph("cora")
    B = gen.dense(g.n, 16, 1)
    for V, S in ((2, 0), (1, 1)):
        with pytest.raises(api.PspmmError) as e:
            run(g, B, api.Config(V=V, S=S, mode=mode))
        assert e.value.status == api.PSPMM_ERR_UNSUPPORTED


def test_retired_mode_4_rejected():
    """Mode 4 (a cp.async short-row stream, never selected) was retired in
    round 2: the engine reports it as an unsupported mode."""
    api = _api()
    g = graph("cora")
    B = gen.dense(g.n, 16, 1)
    with pytest.raises(api.PspmmError) as e:
        run(g, B, api.Config(W=4, F=1, V=1, S=0, mode=4))
    assert e.value.status == api.PSPMM_ERR_UNSUPPORTED


@pytest.mark.parametrize("rows", [1, 2, 31, 32, 33, 64, 65, 1000])
def test_short_row_engine_tiny_edges(rows):
    """Mode 3 with fewer rows than groups and row counts around warp
    multiples, including all-empty matrices."""
    api = _api()
    for density in (0.0, 3.0):
        g = gen.uniform(rows, density, 7) if density else gen.Graph(
            "empty", rows, np.zeros(rows + 1, np.int32), np.zeros(0, np.int32),
            np.zeros(0, np.float32))
        B = gen.dense(g.n, 32, 9)
        ref, mag = oracle_ref(g, B)
        C, _ = run(g, B, api.Config(W=4, F=1, V=1, S=0, mode=3))
        assert_parity(C, ref, mag, f"short rows {rows} d {density}")


def test_tma_engine_rejects_unsupported_K():
    api = _api()
    g = graph("cora")
    B = gen.dense(g.n, 20, 1)
    with pytest.raises(api.PspmmError) as e:
        run(g, B, api.Config(V=1, S=0, mode=2))
    assert e.value.status == api.PSPMM_ERR_UNSUPPORTED


def test_identity_exact_all_corners():
    api = _api()
    n = 1537
    g = gen.Graph("I", n, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32),
                  np.ones(n, np.float32))
    for K in (4, 64, 7):
        B = gen.dense(n, K, 5)
        for V, S in itertools.product((1, 2), (0, 1)):
            C, _ = run(g, B, api.Config(V=V, S=S))
            assert np.array_equal(C, B)


def test_integer_inputs_bitwise():
    api = _api()
    g = gen.powerlaw(2500, 20, 2.0, 51, kind="int")
    B = gen.dense(g.n, 32, 52, kind="int")
    ref, _ = oracle.spmm(g.rowptr, g.colidx, g.val, B)
    for V, S in itertools.product((1, 2), (0, 1)):
        C, _ = run(g, B, api.Config(V=V, S=S, F=2))
        assert np.array_equal(C.astype(np.float64), ref), (V, S)


def test_balanced_repeat_runs_tolerance_equal():
    api = _api()
    g = main_graph()
    B = gen.dense(g.n, 64, 31)
    ref, mag = oracle_ref(g, B, key="main64")
    cfg = api.Config(V=2, S=1, F=1, sg_override=32)
    C1, A = run(g, B, cfg)
    for _ in range(3):
        C2, _ = run(g, B, cfg, A=A)
        assert_parity(C2, ref, mag, "repeat")
        assert np.allclose(C1, C2, rtol=0, atol=2e-5 * (1 + np.abs(ref).max()))


def test_all_positive_long_rows_stress():
    """c-24: all-positive values on 40k-nnz rows stay within the tolerance."""
    api = _api()
    g = gen.giant_row(40001, 40000, 3, 61, kind="positive")
    B = gen.dense(g.n, 64, 62, kind="positive")
    ref, mag = oracle.spmm(g.rowptr, g.colidx, g.val, B, threads=8)
    for V, S in itertools.product((1, 2), (0, 1)):
        C, _ = run(g, B, api.Config(V=V, S=S))
        assert_parity(C, ref, mag, f"positive V{V} S{S}")


def test_leading_dimensions_and_misalignment():
    api, torch = _api(), _torch()
    g = graph("reddit_s")
    K = 32
    B = gen.dense(g.n, K, 71)
    ref, mag = oracle_ref(g, B, key=("reddit_s", K, "ld"))
    Bbig = torch.zeros((g.n, 40), device="cuda")
    Bbig[:, :K] = torch.from_numpy(B).cuda()
    Cbig = torch.full((g.n, 44), 7.0, device="cuda")
    for V, S in itertools.product((1, 2), (0, 1)):
        run(g, Bbig[:, :K], api.Config(V=V, S=S), C=Cbig[:, :K])
        out = Cbig.cpu().numpy()
        assert_parity(out[:, :K], ref, mag, "ld")
        assert np.all(out[:, K:] == 7.0)  # columns beyond K untouched
    # misaligned base pointers -> masked scalar variant
    flat = torch.zeros(g.n * K + 1, device="cuda")
    Bm = flat[1:].view(g.n, K)
    Bm.copy_(torch.from_numpy(B))
    C, _ = run(g, Bm, api.Config(V=2, S=1))
    assert_parity(C, ref, mag, "misaligned")


def test_empty_matrix_writes_zeros():
    api = _api()
    g = gen.Graph("empty", 100, np.zeros(101, np.int32), np.zeros(0, np.int32),
                  np.zeros(0, np.float32))
    B = gen.dense(100, 16, 1)
    C, _ = run(g, B, api.Config(V=1, S=0))
    assert not C.any()
    C, _ = run(g, B, api.Config(V=2, S=1, sg_override=32))
    assert not C.any()


def test_config_errors():
    api, torch = _api(), _torch()
    g = graph("cora")
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 2, 1)
    B = torch.zeros((g.n, 16), device="cuda")
    C = torch.zeros((g.n, 16), device="cuda")
    cases = [(api.Config(V=1, S=1), api.PSPMM_ERR_CONFIG_MISMATCH),
             (api.Config(V=2, S=0), api.PSPMM_ERR_CONFIG_MISMATCH),
             (api.Config(V=2, S=1, omega=16), api.PSPMM_ERR_CONFIG_MISMATCH),
             (api.Config(V=2, S=1, W=3), api.PSPMM_ERR_CONFIG),
             (api.Config(V=2, S=1, F=9), api.PSPMM_ERR_CONFIG),
             (api.Config(V=2, S=1, G=3), api.PSPMM_ERR_CONFIG),
             (api.Config(V=2, S=1, mode=1), api.PSPMM_ERR_UNSUPPORTED)]
    for cfg, want in cases:
        with pytest.raises(api.PspmmError) as e:
            api.pspmm_spmm_run(A, B, C, cfg)
        assert e.value.status == want, cfg
    import ctypes
    st = api._lib.pspmm_spmm_run(A.handle, ctypes.c_void_p(B.data_ptr()), 8, 16,
                                 ctypes.c_void_p(C.data_ptr()), 16, api.Config(V=2, S=1), None)
    assert st == api.PSPMM_ERR_DIM_MISMATCH  # ldb < K
    st = api._lib.pspmm_spmm_run(A.handle, ctypes.c_void_p(B.data_ptr()), 16, 0,
                                 ctypes.c_void_p(C.data_ptr()), 16, api.Config(V=2, S=1), None)
    assert st == api.PSPMM_ERR_DIM_MISMATCH  # K < 1


@pytest.mark.parametrize("V,S", [(1, 0), (1, 1), (2, 0), (2, 1)])
@pytest.mark.parametrize("mode", [0, 2])
def test_host_e2e_entry(V, S, mode):
    """Host entry: H2D, engine in 8 panel-aligned slices, overlapped D2H."""
    api, torch = _api(), _torch()
    g = graph("products_s")
    K = 128
    B = gen.dense(g.n, K, 81)
    ref, mag = oracle_ref(g, B, key=("products_s", K, "e2e"))
    rp, ci, vl = dev(g)
    cfg = api.Config(V=V, S=S, F=1, mode=mode, sg_override=0)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, S, 32, 16 if S else 0)  # many splits
    hB = torch.from_numpy(B).pin_memory()
    hC = torch.full((g.n, K), float("nan")).pin_memory()
    dB = torch.empty((g.n, K), device="cuda")
    dC = torch.empty((g.n, K), device="cuda")
    for _ in range(2):  # second call reuses the handle's copy stream
        api.pspmm_spmm_run_host(A, hB, hC, cfg, dB, dC)
        assert_parity(hC.numpy(), ref, mag, f"host e2e V{V} S{S} mode{mode}")


@pytest.mark.parametrize("name,V,S,mode,order", [
    ("products_s", 1, 1, 0, 0), ("products_s", 2, 0, 0, 1), ("giant", 1, 0, 0, 1),
    ("roadnet_s", 1, 0, 3, 0), ("roadnet_s", 1, 0, 0, 0), ("reddit_s", 1, 1, 2, 0)])
def test_host_entries_whole_and_batch(name, V, S, mode, order):
    """pspmm_spmm_run_host on skewed S = 0 handles (hub rows: the whole-matrix
    path) and pspmm_spmm_run_host_batch (two rotating buffer sets, copies on
    internal streams): every product of the batch matches the oracle."""
    api, torch = _api(), _torch()
    g = graph(name)
    K = 64
    rp, ci, vl = dev(g)
    cfg = api.Config(V=V, S=S, F=1, W=4, mode=mode, order=order)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, S)
    Bs = [gen.dense(g.n, K, 700 + i) for i in range(5)]
    refs = [oracle_ref(g, B) for B in Bs]
    hB = [torch.from_numpy(B).pin_memory() for B in Bs]
    hC = [torch.full((g.n, K), float("nan")).pin_memory() for _ in Bs]
    dB = [torch.empty((g.n, K), device="cuda") for _ in range(2)]
    dC = [torch.empty((g.n, K), device="cuda") for _ in range(2)]
    api.pspmm_spmm_run_host(A, hB[0], hC[0], cfg, dB[0], dC[0])
    assert_parity(hC[0].numpy(), *refs[0], f"host {name} V{V} S{S} m{mode}")
    for count in (5, 1, 0, 5):  # reuse of the handle's streams / events
        for c in hC:
            c.fill_(float("nan"))
        api.pspmm_spmm_run_host_batch(A, hB[:count], hC[:count], cfg, dB, dC)
        for i in range(count):
            assert_parity(hC[i].numpy(), *refs[i], f"batch {i}/{count} {name} m{mode}")


def test_graph_capture_and_streams():
    """spmm_run allocates nothing, so it can be captured in a CUDA graph and
    replayed on a side stream."""
    api, torch = _api(), _torch()
    g = graph("reddit_s")
    K = 64
    B = gen.dense(g.n, K, 91)
    ref, mag = oracle_ref(g, B, key=("reddit_s", K, "graph"))
    rp, ci, vl = dev(g)
    cfg = api.Config(V=1, S=1)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 1)
    Bd = torch.from_numpy(B).cuda()
    C = torch.zeros((g.n, K), device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg, stream=s):
            api.pspmm_spmm_run(A, Bd, C, cfg, stream=s)
        C.fill_(float("nan"))
        cg.replay()
    torch.cuda.synchronize()
    assert_parity(C.cpu().numpy(), ref, mag, "graph replay")


def test_cusparse_baseline_agrees():
    """The vendor baseline bench.py compares against computes the same C."""
    import ctypes
    import os
    torch = _torch()
    from paper_2605_15695_b200 import build_ext
    lib = ctypes.CDLL(build_ext.LIB_CUSPARSE)
    g = graph("reddit_s")
    K = 64
    B = gen.dense(g.n, K, 91)
    ref, mag = oracle_ref(g, B, key=("reddit_s", K, "graph"))
    rp, ci, vl = dev(g)
    Bd = torch.from_numpy(B).cuda()
    C = torch.zeros((g.n, K), device="cuda")
    plan = ctypes.c_void_p()
    P = ctypes.c_void_p
    lib.pspmm_cusparse_create.argtypes = [ctypes.c_int64] * 3 + [P] * 4 + [ctypes.c_int64,
                                          ctypes.c_int32, P, ctypes.c_int64, ctypes.c_int32, P,
                                          ctypes.POINTER(P)]
    lib.pspmm_cusparse_run.argtypes = [P, P]
    lib.pspmm_cusparse_destroy.argtypes = [P]
    st = lib.pspmm_cusparse_create(g.n, g.n, g.nnz, rp.data_ptr(), ci.data_ptr(), vl.data_ptr(),
                                   Bd.data_ptr(), K, K, C.data_ptr(), K, 0, None,
                                   ctypes.byref(plan))
    assert st == 0
    assert lib.pspmm_cusparse_run(plan, None) == 0
    torch.cuda.synchronize()
    lib.pspmm_cusparse_destroy(plan)
    assert_parity(C.cpu().numpy(), ref, mag, "cusparse")
    assert os.path.exists(build_ext.LIB_CUSPARSE)
