"""Streaming ceilings of the dense product's data movement (tools/mb_stream.cu):
a TMA ring per SM reading X (2-D boxes per 32-column chunk or one 3-D box per
tile), optionally storing every tile to T by TMA, next to LDG.128 streaming
reads and torch's device copy; n = 232,965 rows, cold (L2 flushed) and warm.

python tools/stream_ceiling.py [--out gpurun_out/stream_ceiling.jsonl]
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "tools", "libmb_stream.so")


def main():
    import torch

    import bench
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/stream_ceiling.jsonl")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    if not os.path.exists(LIB):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", LIB,
                               os.path.join(ROOT, "tools", "mb_stream.cu"), "-lcuda"])
    lib = ctypes.CDLL(LIB)
    lib.mb_tma_stream.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    lib.mb_ldg_stream.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                  ctypes.c_void_p]
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    flush_buf = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")

    def flush():
        with torch.cuda.stream(stream):
            flush_buf.fill_(1.0)
    n = 232965
    out = open(a.out, "a")

    def rec(name, Ki, nbytes, step):
        with torch.cuda.stream(stream):
            cold = bench.time_steps(step, a.iters, 3, flush, stream)
            warm = bench.time_steps(step, a.iters, 3, lambda: None, stream)
        torch.cuda.synchronize()
        r = {"Ki": Ki, "variant": name, "bytes": nbytes, "cold_us": 1e3 * float(np.median(cold)),
             "warm_us": 1e3 * float(np.median(warm)),
             "cold_gbs": nbytes / (np.median(cold) * 1e-3) / 1e9,
             "warm_gbs": nbytes / (np.median(warm) * 1e-3) / 1e9}
        print(json.dumps(r), flush=True)
        out.write(json.dumps(r) + "\n")

    for Ki in (64, 128):
        X = torch.rand((n, Ki), device="cuda")
        T = torch.empty((n, Ki), device="cuda")
        o = torch.zeros(4, device="cuda")
        rb = X.numel() * 4
        rec("torch_copy", Ki, 2 * rb, lambda: T.copy_(X))
        for blocks in (148 * 4, 148 * 8, 148 * 16):
            rec(f"ldg_read_b{blocks}", Ki, rb,
                lambda: lib.mb_ldg_stream(X.data_ptr(), X.numel(), o.data_ptr(), blocks, sp))
        chunks = Ki // 32
        for box3d in (0, 1):
            for stages in (2, 4, 6, 8, 12):
                if stages * chunks * 16384 + 2048 > 227 * 1024:
                    continue
                for store in (0, 1):
                    def step(box3d=box3d, stages=stages, store=store):
                        st = lib.mb_tma_stream(X.data_ptr(), T.data_ptr(), n, Ki, stages, box3d,
                                               store, sp)
                        assert st == 0, st
                    rec(f"tma_{'3d' if box3d else '2d'}_s{stages}_{'copy' if store else 'read'}",
                        Ki, rb * (2 if store else 1), step)
        if not torch.equal(T, X):
            print(json.dumps({"Ki": Ki, "error": "TMA copy mismatch"}), flush=True)
        del X, T


if __name__ == "__main__":
    main()
