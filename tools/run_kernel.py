"""Launch the engine on one workload a few times (for ncu captures).

python tools/run_kernel.py --workload reddit [--V 1 --S 1 --F 1 --G 16 --W 4] [--iters 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import gen
    from paper_2605_15695_b200 import api
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="reddit")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--dense", type=float, default=0.0,
                    help="> 0: attach the dense-tile split (min density) and run mode 1")
    for k in ("V", "S", "F", "G", "W", "sg", "mode", "order"):
        ap.add_argument(f"--{k}", type=int, default=None)
    a = ap.parse_args()
    g = bench.load_graph(a.workload)
    rp = torch.from_numpy(g.rowptr).cuda()
    ci = torch.from_numpy(g.colidx).cuda()
    vl = torch.from_numpy(g.val).cuda()
    cfg = api.auto_config(g.n, g.nnz, rp, ci, g.K)
    overridden = any(getattr(a, k) is not None for k in ("V", "S", "F", "G", "W", "mode", "order"))
    if not overridden and a.dense <= 0:  # the library's full selection, as bench.py times it
        feats = api.pspmm_features_compute(g.n, g.nnz, rp, ci)
        A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega, cfg.sg_override)
        cfg, _ = api.auto_dense(A, rp, ci, vl, g.K, cfg)
        cfg, A, _ = api.auto_blocks(A, rp, ci, vl, g.K, cfg)
        cfg, A, _ = api.auto_band(A, rp, ci, vl, g.K, cfg, feats)
        B = torch.from_numpy(gen.config_B(g.name, g.n)).cuda()
        C = torch.empty((g.n, g.K), device="cuda")
        for _ in range(a.iters):
            A.run(B, C, cfg)
        torch.cuda.synchronize()
        print(a.workload, cfg, A.info)
        return
    for k in ("V", "S", "F", "G", "W", "mode", "order"):
        if getattr(a, k) is not None:
            setattr(cfg, k, getattr(a, k))
    if a.sg is not None:
        cfg.sg_override = a.sg
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega, cfg.sg_override)
    if cfg.mode == 5:
        print("blocks: windows", api.pspmm_pcsr_attach_blocks(A))
    if cfg.mode == 6:
        print("band: staged fraction", api.pspmm_pcsr_attach_band(A, g.K))
    if a.dense > 0:
        print(api.pspmm_pcsr_attach_dense(A, rp, ci, vl, a.dense, k_max=g.K))
        cfg.mode = 1
    B = torch.from_numpy(gen.config_B(g.name, g.n)).cuda()
    C = torch.empty((g.n, g.K), device="cuda")
    for _ in range(a.iters):
        A.run(B, C, cfg)
    torch.cuda.synchronize()
    print(a.workload, cfg, A.info)


if __name__ == "__main__":
    main()
