"""Reordering (f1, §4.4) on the BASELINE workloads: the engine
(decider + mode 1 / 5 / 6 rules, exactly as bench.py picks) on the graph as
generated, after BFS / Cuthill-McKee, and after descending-degree order.
Times are per SpMM (cold, L2 flushed); the one-time reorder + P A P^T cost
and the per-layer B / C row permutations are reported beside them
(VERDICT r1 missing #5).

python tools/reorder_ab.py [--workloads reddit,products,cora,proteins] [--iters 10]
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
    ap.add_argument("--workloads", default="reddit,products,cora,proteins")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out", default="gpurun_out/reorder_ab.jsonl")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    flush_buf = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")

    def flush():
        with torch.cuda.stream(stream):
            flush_buf.fill_(1.0)

    def engine(n, nnz, rp, ci, vl, K):
        feats = api.pspmm_features_compute(n, nnz, rp, ci, stream=stream)
        cfg = api.pspmm_decide_config(feats, K)
        A = api.pspmm_pcsr_build(n, nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega, cfg.sg_override,
                                 stream)
        cfg, _ = api.auto_dense(A, rp, ci, vl, K, cfg, stream)
        cfg, A, _ = api.auto_blocks(A, rp, ci, vl, K, cfg, stream)
        cfg, A, _ = api.auto_band(A, rp, ci, vl, K, cfg, feats, stream)
        return cfg, A, feats

    for name in a.workloads.split(","):
        g = bench.load_graph(name)
        K = g.K
        rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
        B = torch.from_numpy(gen.config_B(name, g.n)).cuda()
        C = torch.empty((g.n, K), device="cuda")
        rec = {"workload": name, "K": K}
        for strat in ("none", "bfs", "degree"):
            t0 = time.perf_counter()
            if strat == "none":
                rp2, ci2, vl2, B2 = rp, ci, vl, B
                t_re = 0.0
            else:
                perm = api.pspmm_reorder(g.rowptr, g.colidx, strat)
                pd = torch.from_numpy(perm).cuda()
                rp2, ci2, vl2 = api.pspmm_csr_permute(rp, ci, vl, pd)
                torch.cuda.synchronize()
                t_re = time.perf_counter() - t0
                B2 = api.pspmm_permute_rows(B, pd)
                with torch.cuda.stream(stream):
                    tp = bench.time_steps(lambda: api.pspmm_permute_rows(B, pd, out=B2,
                                                                          stream=stream),
                                          a.iters, 2, flush, stream)
            cfg, A, feats = engine(g.n, g.nnz, rp2, ci2, vl2, K)
            with torch.cuda.stream(stream):
                ts = bench.time_steps(lambda: A.run(B2, C, cfg, stream), a.iters, 3, flush, stream)
            torch.cuda.synchronize()
            rec[strat] = {"cfg": cfg.as_dict(), "ms": float(np.mean(ts)),
                          "b": feats["b"] if isinstance(feats, dict) else feats.b,
                          "pr2": feats["pr2"] if isinstance(feats, dict) else feats.pr2,
                          "reorder_s": t_re}
            if strat != "none":
                rec[strat]["permute_B_ms"] = float(np.mean(tp))
                rec[strat]["speedup"] = rec["none"]["ms"] / rec[strat]["ms"]
            del A
            print(name, strat, rec[strat], flush=True)
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "a") as f:
            f.write(json.dumps(rec) + "\n")
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
