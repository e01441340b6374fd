"""A/B: K-slicing (column passes of 64 = 256-B B segments whose slice fits
L2) against the decided config, on one workload at large K.

python tools/slice_ab.py --workload reddit --Ks 128,256
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
    ap.add_argument("--workload", default="reddit")
    ap.add_argument("--Ks", default="128,256")
    ap.add_argument("--iters", type=int, default=9)
    a = ap.parse_args()
    g = bench.load_graph(a.workload)
    rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
    feats = api.pspmm_features_compute(g.n, g.nnz, rp, ci)
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    hs = {}
    for K in [int(k) for k in a.Ks.split(",")]:
        B = torch.from_numpy(gen.dense(g.n, K, 7000 + K)).cuda()
        C = torch.empty((g.n, K), device="cuda")
        dec = api.pspmm_decide_config(feats, K)
        cands = [("decided", dec)]
        for V in (1, 2):
            for (F, G) in ((1, 16), (2, 8), (1, 32)):
                cands.append((f"V{V} F{F} G{G} o1", api.Config(W=2, F=F, V=V, S=0, G=G, order=1)))
        for name, cfg in cands:
            key = (cfg.V, cfg.S)
            if key not in hs:
                hs[key] = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S)
            ts = bench.time_steps(lambda: hs[key].run(B, C, cfg), a.iters, 3,
                                  lambda: flush_buf.fill_(1.0), stream)
            print(json.dumps({"workload": a.workload, "K": K, "variant": name, "cfg": cfg.as_dict(),
                              "passes": -(-K // (4 * cfg.F * cfg.G)),
                              "ms": float(np.median(ts))}), flush=True)
        del B, C


if __name__ == "__main__":
    main()
