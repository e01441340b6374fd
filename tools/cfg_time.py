"""Median time of the decided config (auto_config) per workload, for A/B of
library variants (PSPMM_LIB=...): one JSON line per workload.

PSPMM_LIB=paper_2605_15695_b200/variants/libpspmm_X.so python tools/cfg_time.py --workloads reddit
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
    ap.add_argument("--workloads", default="reddit,proteins,products")
    ap.add_argument("--iters", type=int, default=15)
    ap.add_argument("--tag", default=os.path.basename(os.environ.get("PSPMM_LIB", "main")))
    a = ap.parse_args()
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    for w in a.workloads.split(","):
        g = bench.load_graph(w)
        rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
        cfg = api.auto_config(g.n, g.nnz, rp, ci, g.K)
        A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S)
        B = torch.from_numpy(gen.config_B(w, g.n)).cuda()
        C = torch.empty((g.n, g.K), device="cuda")
        ts = bench.time_steps(lambda: A.run(B, C, cfg), a.iters, 3,
                              lambda: flush_buf.fill_(1.0), stream)
        print(json.dumps({"tag": a.tag, "workload": w, "cfg": cfg.as_dict(),
                          "ms_median": float(np.median(ts)), "ms_min": float(min(ts))}),
              flush=True)
        del A, B, C


if __name__ == "__main__":
    main()
