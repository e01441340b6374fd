"""A/B of pspmm_dense_gemm: the tcgen05 3xTF32 product (gemm_tc.cu) against
the CUDA-core kernel (PSPMM_GEMM_CC=1) on Reddit-sized X (n = 232,965), with
achieved GB/s (4 n (Ki + Ko) bytes) and the layer's fused timing
(pspmm_gnn_layer vs its SpMM alone).

python tools/gemm_ab.py [--out gpurun_out/gemm_ab.jsonl]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2605_15695_b200 import api
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/gemm_ab.jsonl")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    flush_buf = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")

    def flush():
        with torch.cuda.stream(stream):
            flush_buf.fill_(1.0)
    n = 232965
    out = open(a.out, "a")
    for Ki, Ko in ((64, 64), (128, 128), (256, 64), (64, 256), (128, 64), (256, 256)):
        X = torch.rand((n, Ki), device="cuda") * 2 - 1
        W = torch.rand((Ki, Ko), device="cuda") * 2 - 1
        T = torch.empty((n, Ko), device="cuda")
        rec = {"n": n, "Ki": Ki, "Ko": Ko, "bytes": 4 * n * (Ki + Ko)}
        ref = None
        for tag, cc in (("tc", "0"), ("cc", "1")):
            os.environ["PSPMM_GEMM_CC"] = cc
            with torch.cuda.stream(stream):
                step = lambda: api.pspmm_dense_gemm(X, W, T, stream)
                cold = bench.time_steps(step, a.iters, 3, flush, stream)
                warm = bench.time_steps(step, a.iters, 3, lambda: None, stream)
            torch.cuda.synchronize()
            if ref is None:
                ref = T.clone()
            rec[tag] = {"cold_ms": float(np.median(cold)), "warm_ms": float(np.median(warm)),
                        "cold_gbs": rec["bytes"] / (np.median(cold) * 1e-3) / 1e9,
                        "warm_gbs": rec["bytes"] / (np.median(warm) * 1e-3) / 1e9}
        os.environ["PSPMM_GEMM_CC"] = "0"
        rec["tc_vs_cc_maxdiff"] = float((T - ref).abs().max())
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")
        del X, W, T
    # pipeline-depth / epilogue variants of the tensor-core product at 64 x 64
    X = torch.rand((n, 64), device="cuda") * 2 - 1
    W = torch.rand((64, 64), device="cuda") * 2 - 1
    T = torch.empty((n, 64), device="cuda")
    for ops in ("2", "4", "8"):
        for so in ("2", "0"):
            os.environ["PSPMM_GEMM_XS"], os.environ["PSPMM_GEMM_OB"] = ops, so
            with torch.cuda.stream(stream):
                step = lambda: api.pspmm_dense_gemm(X, W, T, stream)
                cold = bench.time_steps(step, a.iters, 3, flush, stream)
            torch.cuda.synchronize()
            rec = {"variant": f"xs{ops}_ob{so}", "cold_ms": float(np.median(cold)),
                   "cold_gbs": 4 * n * 128 / (np.median(cold) * 1e-3) / 1e9}
            print(json.dumps(rec), flush=True)
            out.write(json.dumps(rec) + "\n")
    os.environ.pop("PSPMM_GEMM_XS")
    os.environ.pop("PSPMM_GEMM_OB")
    # the layer on Reddit: Y = A (X W) with Ki = Ko = 64 vs the SpMM alone
    g = bench.load_graph("reddit")
    rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
    cfg = api.auto_config(g.n, g.nnz, rp, ci, 64)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega, cfg.sg_override)
    X = torch.rand((g.n, 64), device="cuda") * 2 - 1
    W = torch.rand((64, 64), device="cuda") * 2 - 1
    T = torch.empty((g.n, 64), device="cuda")
    Y = torch.empty((g.n, 64), device="cuda")
    with torch.cuda.stream(stream):
        tl = bench.time_steps(lambda: api.pspmm_gnn_layer(A, X, W, T, Y, cfg, stream), a.iters, 3,
                              flush, stream)
        ts = bench.time_steps(lambda: A.run(X, Y, cfg, stream), a.iters, 3, flush, stream)
    torch.cuda.synchronize()
    rec = {"layer": "reddit Ki=Ko=64", "layer_ms": float(np.median(tl)),
           "spmm_ms": float(np.median(ts)), "ratio": float(np.median(tl) / np.median(ts))}
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main()
