"""Launch the dense product a few times on Reddit-sized X (for ncu captures).

python tools/gemm_run.py [--Ki 64 --Ko 64 --iters 3]   (PSPMM_GEMM_* knobs apply)
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2605_15695_b200 import api
    ap = argparse.ArgumentParser()
    ap.add_argument("--Ki", type=int, default=64)
    ap.add_argument("--Ko", type=int, default=64)
    ap.add_argument("--n", type=int, default=232965)
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    X = torch.rand((a.n, a.Ki), device="cuda") * 2 - 1
    W = torch.rand((a.Ki, a.Ko), device="cuda") * 2 - 1
    T = torch.empty((a.n, a.Ko), device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(a.iters):
        api.pspmm_dense_gemm(X, W, T, s)
    torch.cuda.synchronize()
    print("ok", a.Ki, a.Ko, float((T - X @ W).abs().max()))


if __name__ == "__main__":
    main()
