"""Measurement A/B: the L2 flush between timed launches as a plain 256 MiB
write (dirty lines left in L2, written back while the next launch runs)
versus the same write followed by a 256 MiB read (L2 left clean and cold).
Decided config per workload; median of 15 launches each.

python tools/flush_ab.py --workloads roadnet,reddit
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
    import gen
    from paper_2605_15695_b200 import api
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="roadnet,reddit,products")
    ap.add_argument("--iters", type=int, default=15)
    a = ap.parse_args()
    stream = torch.cuda.current_stream()
    wbuf = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    rbuf = torch.ones(256 * 1024 * 1024 // 4, device="cuda")
    sink = torch.empty(1, device="cuda")

    def flush_write():
        wbuf.fill_(1.0)

    def flush_write_read():
        wbuf.fill_(1.0)
        torch.sum(rbuf, dim=0, out=sink[0])

    for w in a.workloads.split(","):
        g = bench.load_graph(w)
        rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
        cfg = api.auto_config(g.n, g.nnz, rp, ci, g.K)
        A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S)
        B = torch.from_numpy(gen.config_B(w, g.n)).cuda()
        C = torch.empty((g.n, g.K), device="cuda")
        for rnd in range(2):
            for name, fl in (("write", flush_write), ("write+read", flush_write_read)):
                ts = bench.time_steps(lambda: A.run(B, C, cfg), a.iters, 3, fl, stream)
                print(json.dumps({"workload": w, "round": rnd, "flush": name,
                                  "ms_median": float(np.median(ts)), "ms_mean": float(np.mean(ts)),
                                  "ms_min": float(min(ts))}), flush=True)
        del A, B, C


if __name__ == "__main__":
    main()
