"""Autotune sweep of the engine's config lattice (decider training data and
kernel-design evidence).

For each graph and K: build the PCSR once per (V, S), then time every
lattice point (W, F, G) with CUDA events (median of --iters launches, L2
flushed between launches, like bench.py).  Writes one JSON record per
(graph, K) with the Table-3 features and the full timing table.

python tools/sweep.py --workloads reddit,products --out gpurun_out/sweep.json
python tools/sweep.py --corpus 40 --Ks 16,32,64,128,256 --out gpurun_out/corpus.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def lattice(K, Ws=(2, 4, 8), max_passes=16):
    out = []
    q = (K + 3) // 4
    for F in range(1, 9):
        for G in (1, 2, 4, 8, 16, 32):
            cover = G * F
            passes = -(-q // cover)
            if passes > max_passes:
                continue
            # skip configs that waste more than half a pass of lanes
            if passes * cover - q >= max(cover, 4) and passes > 1:
                continue
            if passes == 1 and cover >= 2 * q and G > 1:
                continue
            for W in Ws:
                out.append((W, F, G))
    return out


def corpus_graphs(count, seed=12345):
    """Moderate synthetic graphs across generators, exponents and ID orders
    (decider training corpus; n ~ 2e4 .. 4e5)."""
    import gen
    rng = np.random.default_rng(seed)
    gs = []
    for i in range(count):
        kind = ["powerlaw", "uniform", "banded", "community", "chung_lu", "community_shuffled"][i % 6]
        n = int(rng.integers(20000, 400000))
        s = int(rng.integers(1, 1 << 30))
        if kind == "powerlaw":
            g = gen.powerlaw(n, float(rng.uniform(4, 64)), float(rng.uniform(1.8, 3.0)), s)
        elif kind == "uniform":
            g = gen.uniform(n, float(rng.uniform(2, 48)), s)
        elif kind == "banded":
            g = gen.banded(n, int(rng.integers(1, 24)), s, fill=float(rng.uniform(0.3, 0.9)))
        elif kind in ("community", "community_shuffled"):
            g = gen.community(n, int(rng.choice([32, 128, 512, 2048])), float(rng.uniform(4, 64)),
                              float(rng.uniform(0.5, 0.95)), s, ordered=(kind == "community"))
        else:
            d = float(min(rng.uniform(4, 200), 2e7 / n))  # keep nnz <= 2e7 (sweep time)
            nnz = int(n * d) // 2 * 2
            rp, ci = gen.chung_lu(n, nnz, int(min(n - 1, d * rng.uniform(10, 60))), s,
                                  shuffle_seed=s + 1)
            g = gen.Graph(f"chunglu_n{n}_d{d:.0f}", n, rp, ci, gen.values(len(ci), s + 2))
        g.name = f"{i:03d}_{g.name}"
        gs.append(g)
    return gs


def sweep_graph(g, Ks, iters, flush, stream, Ws, VS=((1, 0), (1, 1), (2, 0), (2, 1)), modes=(0,),
                orders=(0,)):
    import torch
    from paper_2605_15695_b200 import api
    rp = torch.from_numpy(g.rowptr).cuda()
    ci = torch.from_numpy(g.colidx).cuda()
    vl = torch.from_numpy(g.val).cuda()
    feats = api.pspmm_features_compute(g.n, g.nnz, rp, ci)
    handles = {}
    for V, S in VS:
        handles[(V, S)] = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, S)
    recs = []
    for K in Ks:
        B = torch.rand((g.n, K), device="cuda") * 2 - 1
        C = torch.empty((g.n, K), device="cuda")
        table = []
        for (V, S), A in handles.items():
            points = [(0, W, F, G, o) for (W, F, G) in lattice(K, Ws) for o in orders] \
                if 0 in modes else []
            if 2 in modes and K % 32 == 0:  # TMA gather engine: only W matters
                points += [(2, W, 0, 0, 0) for W in (1, 2, 4, 8)
                           if W * 8 * 16 * min(K, 256) <= 227 * 1024]
            for m in (3, 4):  # short-row engines
                if m in modes and V == 1 and S == 0 and K % 4 == 0:
                    for F in (1, 2, 4):
                        G = 1
                        while G < -(-(K // 4) // F) and G < 32:
                            G <<= 1
                        points += [(m, W, F, max(G, 2), 0) for W in (2, 4, 8)]
            for (mode, W, F, G, order) in points:
                cfg = api.Config(W=W, F=max(F, 1), V=V, S=S, G=G, mode=mode, order=order)
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(iters)]
                try:
                    A.run(B, C, cfg, stream)
                except api.PspmmError as e:  # outside this engine's domain (e.g. smem)
                    if e.status != api.PSPMM_ERR_CONFIG:
                        raise
                    continue
                for e0, e1 in evs:
                    flush()
                    e0.record(stream)
                    A.run(B, C, cfg, stream)
                    e1.record(stream)
                torch.cuda.synchronize()
                ts = [a.elapsed_time(b) for a, b in evs]
                table.append({"V": V, "S": S, "W": W, "F": F, "G": G, "mode": mode, "order": order,
                              "ms": float(np.median(ts))})
        best = min(table, key=lambda r: r["ms"])
        recs.append({"graph": g.name, "n": g.n, "nnz": g.nnz, "K": K, "features": feats,
                     "table": table, "best": best,
                     "best_gflops": 2.0 * g.nnz * K / (best["ms"] * 1e-3) / 1e9,
                     "decided": api.pspmm_decide_config(feats, K).as_dict()})
        del B, C
    del handles
    torch.cuda.empty_cache()
    return recs


def main():
    import torch

    import bench
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="")
    ap.add_argument("--corpus", type=int, default=0)
    ap.add_argument("--corpus-seed", type=int, default=12345)
    ap.add_argument("--Ks", default="")
    ap.add_argument("--iters", type=int, default=7)
    ap.add_argument("--Ws", default="2,4,8")
    ap.add_argument("--VS", default="10,11,20,21", help="PCSR corners to sweep, e.g. 11,21")
    ap.add_argument("--modes", default="0", help="engine modes to sweep: 0 (LDG), 2 (TMA), 3")
    ap.add_argument("--orders", default="0", help="mode-0 unit orders to sweep: 0, 1")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    Ws = tuple(int(x) for x in a.Ws.split(","))
    VS = tuple((int(x[0]), int(x[1])) for x in a.VS.split(","))
    modes = tuple(int(x) for x in a.modes.split(","))
    orders = tuple(int(x) for x in a.orders.split(","))
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")

    def flush():
        flush_buf.fill_(1.0)

    recs = []
    t0 = time.time()
    for name in [w for w in a.workloads.split(",") if w]:
        g = bench.load_graph(name)
        Ks = [int(k) for k in a.Ks.split(",")] if a.Ks else [g.K]
        recs += sweep_graph(g, Ks, a.iters, flush, stream, Ws, VS, modes, orders)
        print(f"[{time.time() - t0:.0f}s] {name}: best {recs[-1]['best']} "
              f"{recs[-1]['best_gflops']:.0f} GFLOP/s", flush=True)
        json.dump(recs, open(a.out, "w"))
    if a.corpus:
        Ks = [int(k) for k in a.Ks.split(",")] if a.Ks else [16, 32, 64, 128, 256]
        for g in corpus_graphs(a.corpus, a.corpus_seed):
            recs += sweep_graph(g, Ks, a.iters, flush, stream, Ws, VS, modes, orders)
            print(f"[{time.time() - t0:.0f}s] {g.name} n={g.n} nnz={g.nnz}", flush=True)
            json.dump(recs, open(a.out, "w"))
    json.dump(recs, open(a.out, "w"))


if __name__ == "__main__":
    main()
