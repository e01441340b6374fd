"""Column blocking for B far beyond L2 (products): C = sum_p A_p . B_p with A
split into P column blocks (B row ranges of n / P rows), run as one
pspmm_spmm_run on block 0 and pspmm_spmm_accumulate (C += A_p . B) on the
others, so each launch gathers from a B slice that can stay in L2; the price
is a read-modify-write of C per block.  Times P in a list against P = 1 (the
plain engine), cold (L2 flushed), and checks sampled rows against the oracle.

python tools/colblock_ab.py [--workload products] [--Ps 1,4,8,12,16,24]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def split_columns(rp, ci, vl, n, P):
    """(rowptr, colidx, val) of each column block [p n / P, (p + 1) n / P),
    canonical (columns stay sorted inside a row), on the device."""
    import torch
    deg = rp[1:] - rp[:-1]
    rows = torch.repeat_interleave(torch.arange(n, device=rp.device, dtype=torch.int64),
                                   deg.to(torch.int64))
    blk = (ci.to(torch.int64) * P) // n
    key = blk * n + rows
    order = torch.sort(key, stable=True).indices
    ci_s, vl_s = ci[order], vl[order]
    counts = torch.bincount(key, minlength=P * n).view(P, n)
    out, off = [], 0
    for p in range(P):
        c = counts[p]
        rpp = torch.zeros(n + 1, dtype=torch.int32, device=rp.device)
        rpp[1:] = torch.cumsum(c, 0).to(torch.int32)
        m = int(rpp[-1])
        out.append((rpp, ci_s[off:off + m].contiguous(), vl_s[off:off + m].contiguous(), m))
        off += m
    return out


def main():
    import torch

    import bench
    import gen
    import oracle
    from paper_2605_15695_b200 import api
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="products")
    ap.add_argument("--Ps", default="1,4,8,12,16,24")
    ap.add_argument("--iters", type=int, default=7)
    ap.add_argument("--K", type=int, default=0)
    ap.add_argument("--out", default="gpurun_out/colblock_ab.jsonl")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    flush_buf = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")

    def flush():
        with torch.cuda.stream(stream):
            flush_buf.fill_(1.0)
    g = bench.load_graph(a.workload)
    K = a.K or g.K
    rp, ci, vl = (torch.from_numpy(x).cuda() for x in (g.rowptr, g.colidx, g.val))
    cfg = api.auto_config(g.n, g.nnz, rp, ci, K)
    B = torch.from_numpy(gen.config_B(g.name, g.n, K)).cuda()
    C = torch.empty((g.n, K), device="cuda")
    rows = np.sort(np.random.default_rng(5).choice(g.n, 2000, replace=False)).astype(np.int64)
    ref, mag = oracle.spmm(g.rowptr, g.colidx, g.val, B.cpu().numpy(), rows=rows, threads=16)
    out = open(a.out, "a")
    for P in (int(x) for x in a.Ps.split(",")):
        c = api.Config(**cfg.as_dict())
        c.V, c.S = 1, 0  # every block a plain row-per-unit handle
        parts = split_columns(rp, ci, vl, g.n, P)
        hs = [api.pspmm_pcsr_build(g.n, m, rpp, cip, vlp, 1, 0, n_cols=g.n)
              for rpp, cip, vlp, m in parts]
        del parts

        def step():
            api.pspmm_spmm_run(hs[0], B, C, c, stream)
            for h in hs[1:]:
                api.pspmm_spmm_accumulate(h, B, C, c, stream)
        with torch.cuda.stream(stream):
            ts = bench.time_steps(step, a.iters, 2, flush, stream)
        torch.cuda.synchronize()
        got = C.cpu().numpy()[rows].astype(np.float64)
        ok = bool((np.abs(got - ref) <= 1e-5 * mag + 1e-6).all())
        rec = {"workload": a.workload, "K": K, "P": P, "cfg": c.as_dict(),
               "ms_median": float(np.median(ts)), "ms_mean": float(np.mean(ts)), "parity": ok,
               "B_slice_MB": g.n * K * 4 / P / 1e6}
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")
        del hs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
