"""Tiny end-to-end run of every native kernel (validation, PCSR build, both
engines, features) for compute-sanitizer (tests/test_gpu_sanitizer.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
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
                for mode in (0, 2):
                    if mode == 2 and K % 32:
                        continue
                    c = api.Config(W=cfg.W, F=cfg.F, V=V, S=S, G=cfg.G, mode=mode, sg_override=0)
                    A.run(B, C, c)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
