"""speedup over cuSPARSE (best CSR algorithm) across the K
sweep, per workload, with the config the library selects at each K (forest
+ guards, then the mode-1 / mode-5 / mode-6 rules, as bench.py), L2 flushed
between launches.  One JSON line per (workload, K), then a
summary line with the geomeans.

python tools/k_sweep.py --workloads cora,roadnet,products,proteins,reddit --Ks 16,32,64,128,256
"""
import argparse
import json
import math
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
    ap.add_argument("--workloads", default="cora,roadnet,products,proteins,reddit")
    ap.add_argument("--Ks", default="16,32,64,128,256")
    ap.add_argument("--steps", type=int, default=7)
    a = ap.parse_args()
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, device="cuda")

    def flush():
        flush_buf.fill_(1.0)

    speedups = {}
    for w in a.workloads.split(","):
        g = bench.load_graph(w)
        rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
        feats = api.pspmm_features_compute(g.n, g.nnz, rp, ci)
        for K in [int(k) for k in a.Ks.split(",")]:
            cfg = api.pspmm_decide_config(feats, K)
            A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega,
                                     cfg.sg_override)
            cfg, dense = api.auto_dense(A, rp, ci, vl, K, cfg)
            cfg, A, _ = api.auto_blocks(A, rp, ci, vl, K, cfg)   # mode 5 rule
            cfg, A, _ = api.auto_band(A, rp, ci, vl, K, cfg, feats)  # mode 6 rule
            B = torch.from_numpy(gen.dense(g.n, K, 7000 + K)).cuda()
            C = torch.empty((g.n, K), device="cuda")
            ts = bench.time_steps(lambda: A.run(B, C, cfg), a.steps, 3, flush, stream)
            ours = float(np.median(ts))
            gk = gen.Graph(g.name, g.n, g.rowptr, g.colidx, g.val, K)
            cs = bench.cusparse_best(gk, rp, ci, vl, B, K, a.steps, flush, stream)
            rec = {"workload": w, "K": K, "cfg": cfg.as_dict(), "ms": ours,
                   "gflops": 2.0 * g.nnz * K / ours / 1e6,
                   "cusparse_best": cs.get("best"), "cusparse_best_ms": cs.get("best_ms"),
                   "cusparse_default_ms": cs.get("default_ms")}
            if cs.get("best_ms"):
                rec["speedup_vs_cusparse_best"] = cs["best_ms"] / ours
                speedups.setdefault(w, []).append(rec["speedup_vs_cusparse_best"])
            print(json.dumps(rec), flush=True)
            del A, B, C
            torch.cuda.empty_cache()
    geo = {w: math.exp(np.mean(np.log(v))) for w, v in speedups.items()}
    allv = [x for v in speedups.values() for x in v]
    print(json.dumps({"summary": True, "geomean_per_workload": geo,
                      "geomean_all": math.exp(np.mean(np.log(allv))) if allv else None,
                      "points": len(allv), "min": min(allv) if allv else None}), flush=True)


if __name__ == "__main__":
    main()
