"""A/B on one box: the same (W, F, G, order) with V = 1 and V = 2 (S = 0),
alternating, on one workload; median ms per round.

python tools/vs_ab.py --workload products --cfg 2,2,16,1 --rounds 3
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
    ap.add_argument("--workload", default="products")
    ap.add_argument("--cfg", default="2,2,16,1", help="W,F,G,order")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--iters", type=int, default=15)
    a = ap.parse_args()
    W, F, G, order = (int(x) for x in a.cfg.split(","))
    g = bench.load_graph(a.workload)
    rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
    B = torch.from_numpy(gen.config_B(a.workload, g.n)).cuda()
    C = torch.empty((g.n, g.K), device="cuda")
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    hs = {V: api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, 0) for V in (1, 2)}
    for r in range(a.rounds):
        for V in (1, 2):
            cfg = api.Config(W=W, F=F, V=V, S=0, G=G, order=order)
            ts = bench.time_steps(lambda: hs[V].run(B, C, cfg), a.iters, 3,
                                  lambda: flush_buf.fill_(1.0), stream)
            print(json.dumps({"workload": a.workload, "round": r, "V": V, "cfg": a.cfg,
                              "ms_median": float(np.median(ts)), "ms_min": float(min(ts))}),
                  flush=True)


if __name__ == "__main__":
    main()
