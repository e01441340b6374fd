"""A/B of engine mode 5 (row blocks, B windows staged in shared memory)
against the decided mode-0 config on the full-size workloads (cold: L2
flushed between launches; warm: back to back), with a sampled-row parity
check against the oracle.

python tools/block_ab.py [--workloads proteins,proteins_clustered] [--iters 20]
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
    ap.add_argument("--workloads", default="proteins,proteins_clustered")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default="gpurun_out/block_ab.jsonl")
    ap.add_argument("--variants", default="8x15,8x19,8x23,16x15",
                    help="rows-per-warp x consumer-warp instances of mode 5 "
                         "(PSPMM_BLOCK_RW / PSPMM_BLOCK_NW)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    flush_buf = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")

    def flush():
        with torch.cuda.stream(stream):
            flush_buf.fill_(1.0)
    for name in a.workloads.split(","):
        g = bench.load_graph(name)
        K = g.K
        rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
        cfg = api.auto_config(g.n, g.nnz, rp, ci, K)
        A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, cfg.V, cfg.S, cfg.omega, cfg.sg_override)
        H = A if (cfg.V == 1 and cfg.S == 0) else api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl,
                                                                        1, 0)
        reuse = api.pspmm_block_reuse(H)
        B = torch.from_numpy(gen.config_B(name, g.n)).cuda()
        C = torch.empty((g.n, K), device="cuda")
        rec = {"workload": name, "K": K, "reuse": reuse}
        runs = [("mode0", None)] + [("mode5_" + v, v) for v in a.variants.split(",")]
        with torch.cuda.stream(stream):
            for tag, var in runs:
                h, c = A, cfg
                if var is not None:
                    os.environ["PSPMM_BLOCK_RW"], os.environ["PSPMM_BLOCK_NW"] = var.split("x")
                    t0 = time.perf_counter()
                    try:
                        win = api.pspmm_pcsr_attach_blocks(H)
                    except api.PspmmError as e:
                        rec[tag] = {"unsupported": str(e)}
                        print(tag, rec[tag], flush=True)
                        continue
                    rec[tag + "_attach_s"] = time.perf_counter() - t0
                    rec[tag + "_windows"] = win
                    h, c = H, api.Config(mode=5)
                cold = bench.time_steps(lambda: h.run(B, C, c, stream), a.iters, 3, flush, stream)
                warm = bench.time_steps(lambda: h.run(B, C, c, stream), a.iters, 3, lambda: None,
                                        stream)
                rec[tag] = {"cfg": c.as_dict(), "cold_mean": float(np.mean(cold)),
                            "cold_median": float(np.median(cold)),
                            "warm_median": float(np.median(warm))}
                torch.cuda.synchronize()
                if var is not None:
                    rows = np.unique(np.concatenate([
                        np.random.default_rng(1).choice(g.n, 1500, replace=False),
                        np.argsort(np.diff(g.rowptr))[-16:], [0, g.n - 1]])).astype(np.int64)
                    ref, mag = oracle.spmm(g.rowptr, g.colidx, g.val, gen.config_B(name, g.n),
                                           rows=rows, threads=16)
                    got = C.cpu().numpy()[rows].astype(np.float64)
                    ok = np.abs(got - ref) <= 1e-5 * mag + 1e-6
                    rec[tag]["parity_rows"] = int(len(rows))
                    rec[tag]["parity_ok"] = bool(ok.all())
                print(tag, rec[tag], flush=True)
        for tag, var in runs[1:]:
            if "cold_mean" in rec[tag]:
                rec[tag]["speedup_cold"] = rec["mode0"]["cold_mean"] / rec[tag]["cold_mean"]
        print(json.dumps(rec), flush=True)
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "a") as f:
            f.write(json.dumps(rec) + "\n")
        del A, H, rp, ci, vl, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
