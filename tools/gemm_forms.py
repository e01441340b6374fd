"""A/B of the tensor-core dense product (gemm_tc.cu) at several ring depths /
output-buffer counts, next to a plain device copy of the same bytes, cold (L2
flushed) and warm medians, each checked against the fp64 product.

python tools/gemm_forms.py [--out gpurun_out/gemm_forms.jsonl] [--iters 30]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (the round-2 A/B of the earlier "direct" form, one 32-KB stage per X chunk
# holding X and its lo, against these: profiles/r02/gemm_r3/gemm_forms.jsonl)
VARIANTS = [
    ("default", {}),
    ("ring", {"PSPMM_GEMM_WT": "0"}),
    ("nofuse", {"PSPMM_GEMM_FUSE": "0"}),
    ("no_wt128", {"PSPMM_GEMM_WT128": "0"}),
    ("ob2", {"PSPMM_GEMM_OB": "2"}),
    ("ring_lo3", {"PSPMM_GEMM_LO": "3"}),
    ("ring_xs4", {"PSPMM_GEMM_XS": "4"}),
    ("ring_ob1", {"PSPMM_GEMM_OB": "1"}),
    ("ring_ob0", {"PSPMM_GEMM_OB": "0"}),
]
KNOBS = ("PSPMM_GEMM_LO", "PSPMM_GEMM_XS", "PSPMM_GEMM_OB", "PSPMM_GEMM_WT", "PSPMM_GEMM_WT128",
         "PSPMM_GEMM_FUSE")


def main():
    import torch

    import bench
    from paper_2605_15695_b200 import api
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/gemm_forms.jsonl")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--shapes", default="64x64,128x64,64x128,128x128,256x64,64x256")
    ap.add_argument("--variants", default=",".join(v for v, _ in VARIANTS))
    a = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    flush_buf = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")

    def flush():
        with torch.cuda.stream(stream):
            flush_buf.fill_(1.0)
    n = 232965
    out = open(a.out, "a")
    want = a.variants.split(",")
    for shp in a.shapes.split(","):
        Ki, Ko = (int(x) for x in shp.split("x"))
        g = torch.Generator(device="cpu").manual_seed(Ki * 1000 + Ko)
        X = (torch.rand((n, Ki), generator=g) * 2 - 1).cuda()
        W = (torch.rand((Ki, Ko), generator=g) * 2 - 1).cuda()
        T = torch.empty((n, Ko), device="cuda")
        ref = (X.double() @ W.double())
        bound = (X.abs().double() @ W.abs().double()) * 1e-5 + 1e-6
        nbytes = 4 * n * (Ki + Ko)
        if Ki == Ko:  # the same bytes moved by a plain device copy (torch), cold / warm
            with torch.cuda.stream(stream):
                step = lambda: T.copy_(X)
                cold = bench.time_steps(step, a.iters, 3, flush, stream)
                warm = bench.time_steps(step, a.iters, 3, lambda: None, stream)
            torch.cuda.synchronize()
            rec = {"Ki": Ki, "Ko": Ko, "variant": "torch_copy", "cold_ms": float(np.median(cold)),
                   "warm_ms": float(np.median(warm)),
                   "cold_gbs": nbytes / (np.median(cold) * 1e-3) / 1e9,
                   "warm_gbs": nbytes / (np.median(warm) * 1e-3) / 1e9}
            print(json.dumps(rec), flush=True)
            out.write(json.dumps(rec) + "\n")
        for name, env in VARIANTS:
            if name not in want:
                continue
            for k in KNOBS:
                os.environ.pop(k, None)
            os.environ.update(env)
            T.fill_(float("nan"))
            with torch.cuda.stream(stream):
                step = lambda: api.pspmm_dense_gemm(X, W, T, stream)
                cold = bench.time_steps(step, a.iters, 3, flush, stream)
                warm = bench.time_steps(step, a.iters, 3, lambda: None, stream)
            torch.cuda.synchronize()
            err = (T.double() - ref).abs()
            ok = bool((err <= bound).all())
            rec = {"Ki": Ki, "Ko": Ko, "variant": name, "cold_ms": float(np.median(cold)),
                   "warm_ms": float(np.median(warm)),
                   "cold_gbs": nbytes / (np.median(cold) * 1e-3) / 1e9,
                   "warm_gbs": nbytes / (np.median(warm) * 1e-3) / 1e9,
                   "parity": ok, "max_err_over_bound": float((err / bound).max())}
            print(json.dumps(rec), flush=True)
            out.write(json.dumps(rec) + "\n")
        del X, W, T, ref, bound
        torch.cuda.empty_cache()
    for k in KNOBS:
        os.environ.pop(k, None)


if __name__ == "__main__":
    main()
