"""Where the end-to-end time of pspmm_spmm_run_host goes (one workload):
pinned H2D alone, D2H alone, the engine alone, and the host entry with the
decided config and with variants.  CUDA events on one stream, L2 flushed.

python tools/e2e_diag.py --workload reddit
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
    ap.add_argument("--iters", type=int, default=8)
    a = ap.parse_args()
    g = bench.load_graph(a.workload)
    K = g.K
    stream = torch.cuda.Stream()
    flush_buf = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")

    def flush():
        with torch.cuda.stream(stream):
            flush_buf.fill_(1.0)

    rp = torch.from_numpy(g.rowptr).cuda()
    ci = torch.from_numpy(g.colidx).cuda()
    vl = torch.from_numpy(g.val).cuda()
    feats = api.pspmm_features_compute(g.n, g.nnz, rp, ci)
    cfg = api.pspmm_decide_config(feats, K)
    B = gen.config_B(g.name, g.n)
    Bd = torch.from_numpy(B).cuda()
    C = torch.empty((g.n, K), device="cuda")
    hB = torch.from_numpy(B).pin_memory()
    hC = torch.empty((g.n, K)).pin_memory()
    out = {"workload": a.workload, "cfg": cfg.as_dict(), "bytes": int(B.nbytes),
           "hB_pinned": bool(hB.is_pinned()), "hC_pinned": bool(hC.is_pinned())}

    def t(fn):
        with torch.cuda.stream(stream):
            ts = bench.time_steps(fn, a.iters, 2, flush, stream)
        return float(np.median(ts))

    out["h2d_ms"] = t(lambda: Bd.copy_(hB, non_blocking=True))
    out["d2h_ms"] = t(lambda: hC.copy_(C, non_blocking=True))
    variants = {"decided": cfg}
    d = cfg.as_dict()
    variants["order0"] = api.Config(**dict(d, order=0))
    variants["S1_W4"] = api.Config(**dict(d, S=1, W=4, order=0))
    handles = {}
    for name, c in variants.items():
        key = (c.V, c.S)
        if key not in handles:
            handles[key] = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, c.V, c.S)
        A = handles[key]
        out[f"kernel_{name}_ms"] = t(lambda: A.run(Bd, C, c, stream))
        out[f"run_host_{name}_ms"] = t(
            lambda: api.pspmm_spmm_run_host(A, hB, hC, c, Bd, C, stream))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
