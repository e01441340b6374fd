"""Launch floor and CUDA-graph replay (VERDICT r1 missing #6):
the event-timed duration of the smallest possible engine launch (a one-row,
one-nonzero graph), of the Cora step as issued (S = 1: zeroing kernel +
engine, a programmatic dependent launch pair), and of the same step captured
once into a CUDA graph and replayed (pspmm_spmm_run allocates nothing, so it
is capturable).  Warm, back to back, median of --iters.

python tools/launch_floor.py [--out gpurun_out/launch_floor.json]
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
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--out", default="gpurun_out/launch_floor.json")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    out = {}

    def timed(fn, n):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(n)]
        with torch.cuda.stream(stream):
            for _ in range(10):
                fn()
            for e0, e1 in evs:
                e0.record(stream)
                fn()
                e1.record(stream)
        torch.cuda.synchronize()
        t = [x.elapsed_time(y) * 1000.0 for x, y in evs]
        return {"median_us": float(np.median(t)), "min_us": float(np.min(t))}

    # the smallest launch: one row, one nonzero, K = 16
    rp = torch.tensor([0, 1], dtype=torch.int32, device="cuda")
    ci = torch.tensor([0], dtype=torch.int32, device="cuda")
    vl = torch.tensor([1.0], dtype=torch.float32, device="cuda")
    A1 = api.pspmm_pcsr_build(1, 1, rp, ci, vl, 1, 0)
    B1 = torch.ones((1, 16), device="cuda")
    C1 = torch.empty((1, 16), device="cuda")
    c1 = api.Config(W=1, F=1, G=4)
    out["one_nonzero_launch"] = timed(lambda: A1.run(B1, C1, c1, stream), a.iters)
    # Cora at K = 16 .. 256, as issued and as a replayed CUDA graph
    g = bench.load_graph("cora")
    rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
    for K in (16, 64, 256):
        cfg = api.auto_config(g.n, g.nnz, rp, ci, K)
        A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega, cfg.sg_override)
        B = torch.from_numpy(gen.dense(g.n, K, 5)).cuda()
        C = torch.empty((g.n, K), device="cuda")
        rec = {"cfg": cfg.as_dict(), "issued": timed(lambda: A.run(B, C, cfg, stream), a.iters)}
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            A.run(B, C, cfg, stream)  # warm
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=stream):
                A.run(B, C, cfg, stream)
        rec["graph_replay"] = timed(lambda: graph.replay(), a.iters)
        ref = C.clone()
        A.run(B, C, cfg, stream)
        torch.cuda.synchronize()
        rec["graph_matches_issued"] = bool(torch.equal(ref, C)) or bool(
            torch.allclose(ref, C, rtol=1e-5, atol=1e-6))
        out[f"cora_K{K}"] = rec
        print(K, rec, flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
