"""Time engine mode 1 (dense 128 x 32 tiles on tcgen05 + the rest on mode 0)
against mode 0 on the proteins-shaped workloads; one JSON line per point.

python tools/dense_ab.py --workloads proteins_clustered,proteins --dens 0.03,0.06,0.1,0.2
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import gen
    from paper_2605_15695_b200 import api
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="proteins_clustered,proteins")
    ap.add_argument("--dens", default="0.03,0.06,0.1,0.2")
    ap.add_argument("--iters", type=int, default=9)
    a = ap.parse_args()
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, device="cuda")

    def flush():
        flush_buf.fill_(1.0)

    for w in a.workloads.split(","):
        g = bench.load_graph(w)
        rp = torch.from_numpy(g.rowptr).cuda()
        ci = torch.from_numpy(g.colidx).cuda()
        vl = torch.from_numpy(g.val).cuda()
        B = torch.from_numpy(gen.config_B(w, g.n)).cuda()
        C = torch.empty((g.n, g.K), device="cuda")
        flops = 2.0 * g.nnz * g.K
        A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
        for (F, G, order) in ((4, 8, 1), (2, 32, 1), (2, 32, 0)):
            cfg = api.Config(W=2, F=F, V=1, S=0, G=G, order=order)
            ts = bench.time_steps(lambda: A.run(B, C, cfg), a.iters, 3, flush, stream)
            ms = float(np.median(ts))
            print(json.dumps({"workload": w, "n": g.n, "nnz": g.nnz, "K": g.K, "mode": 0,
                              "F": F, "G": G, "order": order, "ms": ms,
                              "gflops": flops / ms / 1e6}), flush=True)
        ref = C.clone()
        for dens in [float(x) for x in a.dens.split(",")]:
            t0 = time.perf_counter()
            info = api.pspmm_pcsr_attach_dense(A, rp, ci, vl, dens, k_max=g.K)
            t_split = time.perf_counter() - t0
            for (F, G, order) in ((4, 8, 1), (2, 32, 1)):
                cfg = api.Config(W=2, F=F, V=1, S=0, G=G, order=order, mode=1)
                ts = bench.time_steps(lambda: A.run(B, C, cfg), a.iters, 3, flush, stream)
                ms = float(np.median(ts))
                diff = float((C - ref).abs().max())
                print(json.dumps({"workload": w, "mode": 1, "min_density": dens, **info,
                                  "dense_frac": info["nnz_dense"] / g.nnz, "split_s": t_split,
                                  "F": F, "G": G, "order": order, "ms": ms,
                                  "gflops": flops / ms / 1e6, "max_diff_vs_mode0": diff}),
                      flush=True)
        del A, C


if __name__ == "__main__":
    main()
