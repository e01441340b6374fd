"""Autotune sweep of the engine's config lattice (decider training data and
kernel-design evidence).

For each graph and K: build the PCSR once per (V, S), then time every
lattice point (W, F, G) with CUDA events (median of --iters launches, L2
flushed between launches, like bench.py).  Writes one JSON record per
(graph, K) with the Table-3 features and the full timing table.

python tools/sweep.py --workloads reddit,products --out gpurun_out/sweep.json
python tools/sweep.py --corpus 40 --Ks 16,32,64,128,256 --out gpurun_out/corpus.json
python tools/sweep.py --recheck profiles/r01/sweeps/sweep_*.json --corpus 60 --top 8 \
    --iters 21 --out gpurun_out/recheck.json
    (re-time the top-8 labels of every (graph, K) record, plus the decided
    config, with 21 launches each, round-robin across the candidates so clock
    drift hits them alike: the labels' noise check)
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


def corpus_graphs(count, seed=12345, n_lo=20000, n_hi=400000, prefix="",
                  kinds=("powerlaw", "uniform", "banded", "community", "chung_lu",
                         "community_shuffled"), d_range=None):
    """Synthetic graphs across generators, exponents and ID orders (decider
    training corpus; n ~ 2e4 .. 4e5 by default; the round-2 supplements use
    n ~ 1e3 .. 2e4 and 8e5 .. 3e6 so the bench graphs' sizes are inside the
    training range)."""
    import gen
    rng = np.random.default_rng(seed)
    gs = []
    for i in range(count):
        kind = kinds[i % len(kinds)]
        n = int(np.exp(rng.uniform(np.log(n_lo), np.log(n_hi)))) if n_lo < 20000 or \
            n_hi > 400000 else int(rng.integers(n_lo, n_hi))
        s = int(rng.integers(1, 1 << 30))
        if kind == "powerlaw":
            g = gen.powerlaw(n, float(rng.uniform(*(d_range or (4, 64)))),
                             float(rng.uniform(1.8, 3.0)), s)
        elif kind == "uniform":
            g = gen.uniform(n, float(rng.uniform(2, 48)), s)
        elif kind == "banded":
            g = gen.banded(n, int(rng.integers(1, 24)), s, fill=float(rng.uniform(0.3, 0.9)))
        elif kind in ("community", "community_shuffled"):
            g = gen.community(n, int(rng.choice([32, 128, 512, 2048])), float(rng.uniform(4, 64)),
                              float(rng.uniform(0.5, 0.95)), s, ordered=(kind == "community"))
        else:
            d = float(min(rng.uniform(*(d_range or (4, 200))), 2e7 / n,
                          max(4.0, n / 8.0)))  # nnz <= 2e7
            nnz = int(n * d) // 2 * 2
            rp, ci = gen.chung_lu(n, nnz, int(min(n - 1, d * rng.uniform(10, 60))), s,
                                  shuffle_seed=s + 1)
            g = gen.Graph(f"chunglu_n{n}_d{d:.0f}", n, rp, ci, gen.values(len(ci), s + 2))
        g.name = f"{prefix}{i:03d}_{g.name}"
        gs.append(g)
    return gs


def sweep_graph(g, Ks, iters, flush, stream, Ws, VS=((1, 0), (1, 1), (2, 0), (2, 1)), modes=(0,),
                orders=(0,), cands=None):
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
            for m in (3,):  # short-row engine
                if m in modes and V == 1 and S == 0 and K % 4 == 0:
                    for F in (1, 2, 4):
                        G = 1
                        while G < -(-(K // 4) // F) and G < 32:
                            G <<= 1
                        points += [(m, W, F, max(G, 2), 0) for W in (2, 4, 8)]
            if cands is not None:  # restricted sweep: the per-K candidate labels only
                points = [(m, W, F, G, o) for (v, s_, W, F, G, m, o) in cands.get(K, ())
                          if (v, s_) == (V, S)]
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


def recheck_graph(g, recs, top, iters, flush, stream):
    """Re-time the `top` fastest table entries of each of g's records (and the
    currently decided config) with `iters` launches, round-robin."""
    import torch
    from paper_2605_15695_b200 import api
    rp = torch.from_numpy(g.rowptr).cuda()
    ci = torch.from_numpy(g.colidx).cuda()
    vl = torch.from_numpy(g.val).cuda()
    handles = {}
    out = []
    for r in recs:
        K = r["K"]
        cands = sorted(r["table"], key=lambda t: t["ms"])[:top]
        d = api.pspmm_decide_config(api.pspmm_features_compute(g.n, g.nnz, rp, ci), K).as_dict()
        key = lambda t: (t["V"], t["S"], t["W"], t["F"], t["G"], t.get("mode", 0),
                         t.get("order", 0))
        if d["mode"] in (0, 2, 3) and key(d) not in {key(t) for t in cands}:
            cands.append({k: d[k] for k in ("V", "S", "W", "F", "G", "mode", "order")})
        B = torch.rand((g.n, K), device="cuda") * 2 - 1
        C = torch.empty((g.n, K), device="cuda")
        cfgs = []
        for t in cands:
            vs = (t["V"], t["S"])
            if vs not in handles:
                handles[vs] = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, *vs)
            cfg = api.Config(W=t["W"], F=max(t["F"], 1), V=t["V"], S=t["S"], G=t["G"],
                             mode=t.get("mode", 0), order=t.get("order", 0))
            handles[vs].run(B, C, cfg, stream)  # warm-up / domain check
            cfgs.append((t, handles[vs], cfg))
        ts = [[] for _ in cfgs]
        for _ in range(iters):
            for j, (t, A, cfg) in enumerate(cfgs):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                flush()
                e0.record(stream)
                A.run(B, C, cfg, stream)
                e1.record(stream)
                ts[j].append((e0, e1))
        torch.cuda.synchronize()
        table = []
        for (t, _, _), ev in zip(cfgs, ts):
            ms = [a.elapsed_time(b) for a, b in ev]
            e = {k: t.get(k, 0) for k in ("V", "S", "W", "F", "G", "mode", "order")}
            e.update({"ms": float(np.median(ms)), "ms_min": float(np.min(ms)),
                      "ms_iqr": float(np.percentile(ms, 75) - np.percentile(ms, 25)),
                      "ms_sweep7": t.get("ms")})
            table.append(e)
        best = min(table, key=lambda x: x["ms"])
        out.append({"graph": r["graph"], "n": r["n"], "nnz": r["nnz"], "K": K,
                    "features": r["features"], "table": table, "best": best, "recheck": iters,
                    "decided": d})
        del B, C
    del handles
    torch.cuda.empty_cache()
    return out


def main():
    import torch

    import bench
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="")
    ap.add_argument("--corpus", type=int, default=0)
    ap.add_argument("--corpus-seed", type=int, default=12345)
    ap.add_argument("--corpus-n", default="20000,400000", help="node-count range lo,hi")
    ap.add_argument("--corpus-prefix", default="")
    ap.add_argument("--corpus-d", default="", help="mean-degree range lo,hi (power law, Chung-Lu)")
    ap.add_argument("--corpus-kinds", default="",
                    help="comma list of generators to cycle (default: all six)")
    ap.add_argument("--Ks", default="")
    ap.add_argument("--iters", type=int, default=7)
    ap.add_argument("--Ws", default="2,4,8")
    ap.add_argument("--VS", default="10,11,20,21", help="PCSR corners to sweep, e.g. 11,21")
    ap.add_argument("--modes", default="0", help="engine modes to sweep: 0 (LDG), 2 (TMA), 3")
    ap.add_argument("--orders", default="0", help="mode-0 unit orders to sweep: 0, 1")
    ap.add_argument("--out", required=True)
    ap.add_argument("--recheck", nargs="*", default=None,
                    help="sweep files whose top labels to re-time (graphs: --workloads names "
                         "and --corpus N regenerated)")
    ap.add_argument("--top", type=int, default=8)
    ap.add_argument("--candidates", nargs="*", default=None,
                    help="sweep files: restrict the lattice to the labels within 2 %% of the "
                         "best of some record at the same K (large graphs)")
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
    if a.recheck:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from train_decider import load
        old = load(a.recheck)
        by_graph = {}
        for r in old:
            by_graph.setdefault(r["graph"], []).append(r)
        graphs = []
        for name in by_graph:
            if name in bench.WORKLOADS:
                graphs.append(bench.load_graph(name))
        for g in corpus_graphs(a.corpus, a.corpus_seed) if a.corpus else []:
            if g.name in by_graph:
                graphs.append(g)
        for g in graphs:
            recs += recheck_graph(g, sorted(by_graph[g.name], key=lambda r: r["K"]), a.top,
                                  a.iters, flush, stream)
            print(f"[{time.time() - t0:.0f}s] recheck {g.name}: {len(recs)} records", flush=True)
            json.dump(recs, open(a.out, "w"))
        json.dump(recs, open(a.out, "w"))
        return
    for name in [w for w in a.workloads.split(",") if w]:
        g = bench.load_graph(name)
        Ks = [int(k) for k in a.Ks.split(",")] if a.Ks else [g.K]
        recs += sweep_graph(g, Ks, a.iters, flush, stream, Ws, VS, modes, orders)
        print(f"[{time.time() - t0:.0f}s] {name}: best {recs[-1]['best']} "
              f"{recs[-1]['best_gflops']:.0f} GFLOP/s", flush=True)
        json.dump(recs, open(a.out, "w"))
    cands = None
    if a.candidates:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from train_decider import load
        cands = {}
        for r in load(a.candidates):
            b = min(t["ms"] for t in r["table"])
            for t in r["table"]:
                if t["ms"] <= 1.02 * b:
                    cands.setdefault(r["K"], set()).add(
                        (t["V"], t["S"], t["W"], t["F"], t["G"], t.get("mode", 0),
                         t.get("order", 0)))
        print({K: len(v) for K, v in cands.items()}, flush=True)
    if a.corpus:
        Ks = [int(k) for k in a.Ks.split(",")] if a.Ks else [16, 32, 64, 128, 256]
        lo, hi = (int(x) for x in a.corpus_n.split(","))
        kinds = tuple(a.corpus_kinds.split(",")) if a.corpus_kinds else (
            "powerlaw", "uniform", "banded", "community", "chung_lu", "community_shuffled")
        d_range = tuple(float(x) for x in a.corpus_d.split(",")) if a.corpus_d else None
        for g in corpus_graphs(a.corpus, a.corpus_seed, lo, hi, a.corpus_prefix, kinds, d_range):
            recs += sweep_graph(g, Ks, a.iters, flush, stream, Ws, VS, modes, orders, cands)
            print(f"[{time.time() - t0:.0f}s] {g.name} n={g.n} nnz={g.nnz}", flush=True)
            json.dump(recs, open(a.out, "w"))
    json.dump(recs, open(a.out, "w"))


if __name__ == "__main__":
    main()
