"""Tiny end-to-end run of every native kernel for compute-sanitizer
(tests/test_gpu_sanitizer.py): CSR validation, features, the PCSR builder
(V x S corners), engine modes 0 / 2 / 3, mode 1 (dense-tile split,
split_b_kernel, dense_tc_kernel), mode 5 (row blocks: touched-window metric,
TMA-staged windows), mode 6 (staged bands, staged and global blocks), the
fan-out epilogue (peer stores), the transpose, the permutation kernels and
both dense products (tcgen05 and CUDA cores) with the GNN layer."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import gen
    from paper_2605_15695_b200 import api
    g = gen.giant_row(301, 280, 3, 7)  # a split row (S = 1 atomics), odd n (V = 2 tail)
    rp = torch.from_numpy(g.rowptr).cuda()
    ci = torch.from_numpy(g.colidx).cuda()
    vl = torch.from_numpy(g.val).cuda()
    f = api.pspmm_features_compute(g.n, g.nnz, rp, ci)
    for K in (7, 32, 64):
        B = torch.rand((g.n, K), device="cuda")
        C = torch.empty((g.n, K), device="cuda")
        for V in (1, 2):
            for S in (0, 1):
                A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, S, 32, 16 if S else 0)
                cfg = api.pspmm_decide_config(f, K)
                for mode in (0, 2, 3):
                    if mode == 2 and K % 32:
                        continue
                    if mode == 3 and (V, S) != (1, 0) or mode == 3 and K % 4:
                        continue
                    c = api.Config(W=cfg.W, F=max(1, min(cfg.F, 2)), V=V, S=S, G=cfg.G,
                                   mode=mode, sg_override=0)
                    if mode == 3:
                        c.F, c.G = 2, 4 if K == 32 else 8
                    A.run(B, C, c)
                # fan-out: two peer copies of C
                peers = [torch.empty_like(C) for _ in range(2)]
                api.pspmm_spmm_run_fanout(A, B, C, peers, api.Config(W=4, V=V, S=S, F=1))
    # mode 1: dense tiles on the tensor cores (a community graph with dense panels)
    gd = gen.community(600, 128, 60, 0.95, 11)
    rpd, cid, vld = (torch.from_numpy(x).cuda() for x in (gd.rowptr, gd.colidx, gd.val))
    Ad = api.pspmm_pcsr_build(gd.n, gd.nnz, rpd, cid, vld, 1, 0)
    api.pspmm_pcsr_attach_dense(Ad, rpd, cid, vld, 0.2, k_max=64)
    Bd = torch.rand((gd.n, 64), device="cuda")
    Cd = torch.empty((gd.n, 64), device="cuda")
    Ad.run(Bd, Cd, api.Config(mode=1))
    # mode 5: row blocks (reuse metric, virtual windows of a dense block)
    api.pspmm_block_reuse(Ad)
    api.pspmm_pcsr_attach_blocks(Ad)
    B5 = torch.rand((gd.n, 128), device="cuda")
    C5 = torch.empty((gd.n, 128), device="cuda")
    Ad.run(B5, C5, api.Config(mode=5))
    # mode 6: staged bands (a banded graph) and over-budget blocks (giant row)
    gb = gen.banded(700, 5, 13, fill=0.8)
    rpb, cib, vlb = (torch.from_numpy(x).cuda() for x in (gb.rowptr, gb.colidx, gb.val))
    for gg, (r_, c_, v_) in ((gb, (rpb, cib, vlb)), (g, (rp, ci, vl))):
        A6 = api.pspmm_pcsr_build(gg.n, gg.nnz, r_, c_, v_, 1, 0)
        api.pspmm_pcsr_attach_band(A6, 128)
        for K in (16, 48, 128):
            B6 = torch.rand((gg.n, K), device="cuda")
            C6 = torch.empty((gg.n, K), device="cuda")
            A6.run(B6, C6, api.Config(mode=6))
    # transpose, permutation
    n = g.n
    api.pspmm_csr_transpose(n, n, rp, ci, vl)
    perm = torch.from_numpy(np.random.default_rng(3).permutation(n).astype(np.int32)).cuda()
    api.pspmm_csr_permute(rp, ci, vl, perm)
    X = torch.rand((n, 32), device="cuda")
    api.pspmm_permute_rows(X, perm)
    api.pspmm_permute_rows(X, perm, inverse=True)
    # dense products (tcgen05 and CUDA cores) and the GNN layer
    for Ki, Ko in ((64, 64), (32, 48), (20, 12)):
        Xg = torch.rand((300, Ki), device="cuda")
        Wg = torch.rand((Ki, Ko), device="cuda")
        Tg = torch.empty((300, Ko), device="cuda")
        api.pspmm_dense_gemm(Xg, Wg, Tg)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
    Xl = torch.rand((g.n, 64), device="cuda")
    Wl = torch.rand((64, 32), device="cuda")
    Tl = torch.empty((g.n, 32), device="cuda")
    Yl = torch.empty((g.n, 32), device="cuda")
    api.pspmm_gnn_layer(A, Xl, Wl, Tl, Yl, api.Config(W=4))
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
