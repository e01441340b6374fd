"""Bare B-row gather ceilings on this B200 (tools/mb_gather.cu), measured with
each workload's OWN column stream (its CSR colIdx in order) next to uniform
random rows of the same count, plus the narrow-row
gathers of a K-sliced products engine: a contiguous n x k_s slice of B
(16 B .. 128 B rows, 39 MB .. 313 MB) gathered by the products column stream
(SURVEY §8(d) "K-slicing").  Warm: B stays resident in L2
where it fits (the steady state of back-to-back launches).

python tools/gather_ceiling.py [--out gpurun_out/gather_ceiling_r02.json] [--workloads ...]
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (graph cache: PSPMM_GEN_CACHE)

LIB = os.path.join(ROOT, "tools", "libmb_gather.so")


def lib():
    src = os.path.join(ROOT, "tools", "mb_gather.cu")
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-shared", "-Xcompiler", "-fPIC", "-o", LIB, src])
    so = ctypes.CDLL(LIB)
    so.mb_gather.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                             ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                             ctypes.c_void_p]
    return so


def shapes(row_bytes):
    f4 = row_bytes // 16
    out = []
    for G in (1, 2, 4, 8, 16, 32):
        for F in (1, 2):
            if G * F == f4:
                out.append((G, F))
    return out


def time_case(so, B, stride, idx, row_bytes, stream, reps=5):
    out = torch.zeros(4, device="cuda")
    best = None
    for G, F in shapes(row_bytes):
        for U in (4, 8, 16):
            def run():
                st = so.mb_gather(B.data_ptr(), stride, idx.data_ptr(), idx.numel(), G, F, U,
                                  out.data_ptr(), ctypes.c_void_p(stream.cuda_stream))
                assert st == 0, st
            for _ in range(2):
                run()
            ts = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                run()
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            ms = float(np.median(ts))
            tbps = idx.numel() * row_bytes / (ms * 1e-3) / 1e12
            if best is None or ms < best["ms"]:
                best = {"ms": ms, "tbps": tbps, "G": G, "F": F, "U": U}
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/gather_ceiling_r02.json")
    ap.add_argument("--workloads", default="reddit,proteins,products,roadnet")
    args = ap.parse_args()
    so = lib()
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    res = {"what": __doc__.split("\n\n")[0], "gpu": torch.cuda.get_device_name(0)}
    with torch.cuda.stream(stream):
        for name in args.workloads.split(","):
            g = bench.load_graph(name)
            K = g.K
            gen_rng = np.random.default_rng(7)
            idx_w = torch.from_numpy(g.colidx).cuda()
            idx_u = torch.from_numpy(gen_rng.integers(0, g.n, g.nnz, dtype=np.int32)).cuda()
            r = {"n": g.n, "nnz": g.nnz, "K": K}
            B = torch.rand((g.n, K), device="cuda")
            rb = K * 4
            r["full_rows"] = {"row_bytes": rb, "B_MB": g.n * rb / 1e6,
                              "workload_stream": time_case(so, B, rb, idx_w, rb, stream),
                              "uniform": time_case(so, B, rb, idx_u, rb, stream)}
            del B
            if name == "products":
                sl = []
                for ks in (4, 8, 16, 32):
                    Bs = torch.rand((g.n, ks), device="cuda")
                    e = {"k_s": ks, "row_bytes": ks * 4, "slice_MB": g.n * ks * 4 / 1e6,
                         "workload_stream": time_case(so, Bs, ks * 4, idx_w, ks * 4, stream),
                         "uniform": time_case(so, Bs, ks * 4, idx_u, ks * 4, stream)}
                    # the same slice left in place inside the full row-major B
                    # (stride K*4): L2 caches whole lines, so this shows what
                    # slicing without a re-layout would get
                    Bf = torch.rand((g.n, K), device="cuda")
                    e["strided_in_full_B"] = time_case(so, Bf, K * 4, idx_w, ks * 4, stream)
                    del Bf
                    ms_total = e["workload_stream"]["ms"] * (K // ks)
                    e["all_slices_ms"] = ms_total
                    sl.append(e)
                    del Bs
                    print(json.dumps(e), flush=True)
                r["slices"] = sl
            print(name, json.dumps(r["full_rows"]), flush=True)
            res[name] = r
            del idx_w, idx_u
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
