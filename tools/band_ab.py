"""A/B of engine mode 6 (staged bands) against the decided config on
locality-ordered workloads (cold: L2 flushed between launches; warm: back
to back), at several K, with a sampled-row parity check against the oracle,
plus the same graphs after RCM reordering of shuffled workloads (f1).

python tools/band_ab.py [--workloads roadnet] [--Ks 16,32,64,128] [--iters 20]
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
    import oracle
    from paper_2605_15695_b200 import api
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="roadnet")
    ap.add_argument("--Ks", default="")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default="gpurun_out/band_ab.jsonl")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    flush_buf = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")

    def flush():
        with torch.cuda.stream(stream):
            flush_buf.fill_(1.0)
    for name in a.workloads.split(","):
        g = bench.load_graph(name)
        Ks = [int(k) for k in a.Ks.split(",")] if a.Ks else [g.K]
        rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
        H = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 1, 0)
        for K in Ks:
            t0 = time.perf_counter()
            frac = api.pspmm_pcsr_attach_band(H, K)  # the band budget scales with k_max
            t_attach = time.perf_counter() - t0
            cfg = api.auto_config(g.n, g.nnz, rp, ci, K)
            A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega,
                                     cfg.sg_override)
            Bn = gen.dense(g.n, K, 2002)
            B = torch.from_numpy(Bn).cuda()
            C = torch.empty((g.n, K), device="cuda")
            R = 4.0 * (g.n + 1) + 8.0 * g.nnz + 8.0 * g.n * K
            rec = {"workload": name, "K": K, "staged_frac": frac, "attach_s": t_attach}
            with torch.cuda.stream(stream):
                F3 = 1 if K <= 16 else 2
                G3 = max(2, min(32, K // (4 * F3)))
                runs = [("decided", A, cfg, None), ("mode3", H, api.Config(W=2, F=F3, G=G3, mode=3),
                                                    None)]
                runs += [(f"mode6_s{st}" if st != "2" else "mode6", H, api.Config(mode=6), st)
                         for st in ("2", "3", "4")]
                for tag, h, c, st in runs:
                    if st is not None:
                        os.environ["PSPMM_BAND_STAGES"] = st
                    cold = bench.time_steps(lambda: h.run(B, C, c, stream), a.iters, 3, flush,
                                            stream)
                    warm = bench.time_steps(lambda: h.run(B, C, c, stream), a.iters, 3,
                                            lambda: None, stream)
                    rec[tag] = {"cfg": c.as_dict(), "cold_mean": float(np.mean(cold)),
                                "cold_median": float(np.median(cold)),
                                "warm_median": float(np.median(warm)),
                                "frac_cold": R / (np.mean(cold) * 1e-3) / 6552.3e9}
                    torch.cuda.synchronize()
                    rows = np.unique(np.concatenate([
                        np.random.default_rng(1).choice(g.n, 1500, replace=False),
                        [0, g.n - 1]])).astype(np.int64)
                    ref, mag = oracle.spmm(g.rowptr, g.colidx, g.val, Bn, rows=rows, threads=16)
                    got = C.cpu().numpy()[rows].astype(np.float64)
                    rec[tag]["parity_ok"] = bool((np.abs(got - ref) <= 1e-5 * mag + 1e-6).all())
            rec["speedup_cold"] = rec["decided"]["cold_mean"] / rec["mode6"]["cold_mean"]
            print(json.dumps(rec), flush=True)
            os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
            with open(a.out, "a") as f:
                f.write(json.dumps(rec) + "\n")
            del A, B, C
        del H
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
