"""(f3) pspmm_dense_gemm and pspmm_gnn_layer (H' = A H W) against the fp64
oracle (oracle.gnn_layer): both orders (SpMM on the narrower side), ragged
widths, several engine configs, and the decided config."""
import numpy as np
import pytest

import gen
import oracle
from gpu_util import RTOL_MAG, ATOL, dev

pytestmark = pytest.mark.gpu


def _check(Y, ref, mag, what):
    # c-1 style bound; the fp32 dense product adds at most Ki 2^-24 of the
    # same magnitude, far inside 1e-5
    err = np.abs(np.asarray(Y, np.float64) - ref)
    bad = err > RTOL_MAG * mag + ATOL
    assert not bad.any(), f"{what}: {int(bad.sum())} elements out of tolerance"


@pytest.mark.parametrize("n,Ki,Ko", [(1, 4, 4), (777, 64, 64), (1000, 16, 200), (513, 130, 7),
                                     (4097, 256, 64)])
def test_dense_gemm(n, Ki, Ko):
    import torch
    from paper_2605_15695_b200 import api
    X = gen.dense(n, Ki, 11)
    W = gen.dense(Ki, Ko, 12)
    T = torch.full((n, Ko), float("nan"), device="cuda")
    api.pspmm_dense_gemm(torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda(), T)
    torch.cuda.synchronize()
    ref = X.astype(np.float64) @ W.astype(np.float64)
    mag = np.abs(X.astype(np.float64)) @ np.abs(W.astype(np.float64))
    _check(T.cpu().numpy(), ref, mag, f"gemm {n}x{Ki}x{Ko}")


@pytest.mark.parametrize("force_cc", [False, True])
@pytest.mark.parametrize("n,Ki,Ko,pad", [(1, 32, 16, 0), (127, 64, 64, 0), (128, 64, 64, 0),
                                         (129, 64, 64, 4), (1000, 128, 128, 0),
                                         (4097, 256, 64, 0), (3000, 64, 256, 8),
                                         (20000, 32, 48, 0), (300, 96, 112, 0),
                                         (1000, 256, 256, 0), (777, 64, 512, 4)])
def test_dense_gemm_tensor_core_shapes(n, Ki, Ko, pad, force_cc, monkeypatch):
    """Shapes the tcgen05 3xTF32 product takes (gemm_tc.cu: Ki % 32, Ko % 16;
    W's image in column blocks when it is too large: 256 x 256, 64 x 512),
    ragged tiles (n % 128 != 0), padded leading dimensions; the
    same shapes forced onto the CUDA-core kernel (PSPMM_GEMM_CC=1).  Both
    against the fp64 product with the c-1 bound on |X| |W|."""
    import torch
    from paper_2605_15695_b200 import api
    if force_cc:
        monkeypatch.setenv("PSPMM_GEMM_CC", "1")
    X = gen.dense(n, Ki, 31)
    W = gen.dense(Ki, Ko, 32)
    Xb = torch.zeros((n, Ki + pad), device="cuda")
    Xb[:, :Ki] = torch.from_numpy(X).cuda()
    Tb = torch.full((n, Ko + pad), float("nan"), device="cuda")
    api.pspmm_dense_gemm(Xb[:, :Ki], torch.from_numpy(W).cuda(), Tb[:, :Ko])
    torch.cuda.synchronize()
    ref = X.astype(np.float64) @ W.astype(np.float64)
    mag = np.abs(X.astype(np.float64)) @ np.abs(W.astype(np.float64))
    T = Tb.cpu().numpy()
    _check(T[:, :Ko], ref, mag, f"gemm {n}x{Ki}x{Ko} pad {pad} cc={force_cc}")
    if pad:
        assert np.isnan(T[:, Ko:]).all(), "padding columns of T were written"


@pytest.mark.parametrize("env", [{}, {"PSPMM_GEMM_OB": "2"}, {"PSPMM_GEMM_OB": "0"},
                                 {"PSPMM_GEMM_WT": "0"}, {"PSPMM_GEMM_WT128": "0"},
                                 {"PSPMM_GEMM_FUSE": "0"}, {"PSPMM_GEMM_FUSE": "0", "PSPMM_GEMM_OB": "0"}])
@pytest.mark.parametrize("n,Ki,Ko,pad", [(1, 32, 128, 0), (127, 96, 128, 4), (5000, 64, 128, 0),
                                         (300, 128, 128, 8), (2049, 64, 256, 0),
                                         (1000, 128, 256, 4), (1, 32, 64, 0), (2049, 64, 64, 0),
                                         (300, 128, 64, 8), (129, 96, 64, 4)])
def test_dense_gemm_w_in_tmem(n, Ki, Ko, pad, env, monkeypatch):
    """The W-in-TMEM form (Ko == 128, Ki <= 128: T^T = W^T X^T with W^T as
    the tensor-memory A operand), with one (default) / two / no staged
    output tiles, against the shared-memory form (PSPMM_GEMM_WT=0), and
    Ko = 256 as 128-column blocks (default) or one shared-memory launch
    (PSPMM_GEMM_WT128=0); ragged tiles and padded ld.  The Ko = 64 shapes
    take the shared-memory form, with the fused N = 2 Ko MMA or without it
    (PSPMM_GEMM_FUSE=0)."""
    import torch
    from paper_2605_15695_b200 import api
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    X = gen.dense(n, Ki, 41)
    W = gen.dense(Ki, Ko, 42)
    Xb = torch.zeros((n, Ki + pad), device="cuda")
    Xb[:, :Ki] = torch.from_numpy(X).cuda()
    Tb = torch.full((n, Ko + pad), float("nan"), device="cuda")
    api.pspmm_dense_gemm(Xb[:, :Ki], torch.from_numpy(W).cuda(), Tb[:, :Ko])
    torch.cuda.synchronize()
    ref = X.astype(np.float64) @ W.astype(np.float64)
    mag = np.abs(X.astype(np.float64)) @ np.abs(W.astype(np.float64))
    T = Tb.cpu().numpy()
    _check(T[:, :Ko], ref, mag, f"gemm {n}x{Ki}x{Ko} pad {pad} {env}")
    if pad:
        assert np.isnan(T[:, Ko:]).all(), "padding columns of T were written"


@pytest.mark.parametrize("name", ["reddit_s", "roadnet_s", "empty_rows"])
@pytest.mark.parametrize("Ki,Ko", [(64, 32), (32, 64), (48, 48), (128, 16), (64, 64),
                                   (128, 128)])
def test_gnn_layer(name, Ki, Ko):
    import torch
    from paper_2605_15695_b200 import api
    g = {"reddit_s": lambda: gen.config_graph("reddit", 0.005),
         "roadnet_s": lambda: gen.config_graph("roadnet", 0.005),
         "empty_rows": lambda: gen.with_empty_rows(gen.powerlaw(2000, 12, 2.1, 3), 0.2, 4)}[name]()
    X = gen.dense(g.n, Ki, 21)
    W = gen.dense(Ki, Ko, 22)
    ref, mag = oracle.gnn_layer(g.rowptr, g.colidx, g.val, X, W)
    rp, ci, vl = dev(g)
    K = min(Ki, Ko)
    feats = api.pspmm_features_compute(g.n, g.nnz, rp, ci)
    cfgs = [api.pspmm_decide_config(feats, K), api.Config(V=1, S=1, W=4),
            api.Config(V=2, S=0, W=2, F=2)]
    Xd, Wd = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
    for cfg in cfgs:
        A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S)
        T = torch.empty((g.n, K), device="cuda")
        Y = torch.full((g.n, Ko), float("nan"), device="cuda")
        api.pspmm_gnn_layer(A, Xd, Wd, T, Y, cfg)
        torch.cuda.synchronize()
        _check(Y.cpu().numpy(), ref, mag, f"layer {name} {Ki}->{Ko} {cfg}")
