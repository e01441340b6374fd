"""Train the SpMM-decider stand-in (§5.2 P:337-341,
protocol P:399) from tools/sweep.py records and emit csrc/decider_model.h.

Label space: (mode, V, S, W, F, P) with P = column passes; the library derives
G = min(32, pow2ceil(ceil(K/4 / (F P)))).  The tree is cost-sensitive: each
leaf takes the label with the highest mean normalized performance
(t_best / t_label) over its records, and splits are chosen greedily to
maximise the sum of those leaf scores.  Features: the 16 Table-3 features +
log2(K).

python tools/train_decider.py gpurun_out/sweep_*.json --out-header ... --eval-json ...
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FEATS = ("n", "n_hat", "nnz", "delta", "d", "d_hat", "d_max", "cv", "cv_hat", "sr1", "sr2", "rho",
         "b", "b_max", "pr1", "pr2")
WORKLOADS = ("cora", "roadnet", "products", "proteins", "reddit", "proteins_clustered")
L2_BYTES = 132644864.0  # B200 L2 (decide.cpp kL2Bytes)
NFEAT = len(FEATS) + 2   # + log2(K), log2(B bytes / L2)


def ceil_pow2(x):
    p = 1
    while p < x and p < 32:
        p <<= 1
    return p


def passes_of(K, F, G):
    q = (K + 3) // 4
    return -(-q // (G * F))


def derived_G(K, F, P):
    q = (K + 3) // 4
    return ceil_pow2(-(-q // (F * P)))


def load(paths):
    """Sweep records; records of the same (graph, K) from several files
    (e.g. a later sweep of another engine mode) are merged into one table."""
    by_key = {}
    for p in paths:
        for r in json.load(open(p)):
            k = (r["graph"], r["K"])
            if k in by_key:
                by_key[k]["table"] = by_key[k]["table"] + r["table"]
            else:
                by_key[k] = dict(r)
    return list(by_key.values())


def label_of(K, t):
    """(mode, V, S, W, F, P) of a sweep entry, or None if the library could
    not re-derive its G from (K, F, P)."""
    mode = t.get("mode", 0)
    if mode == 2:
        return (2, t["V"], t["S"], t["W"], 1, 1, 0)
    P = passes_of(K, t["F"], t["G"])
    if derived_G(K, t["F"], P) != t["G"]:
        return None
    return (mode, t["V"], t["S"], t["W"], t["F"], P, t.get("order", 0) if mode == 0 else 0)


def apply_recheck(recs, paths):
    """Override sweep timings with the re-timed (21-launch, round-robin)
    medians of tools/sweep.py --recheck.  The recheck ran on another day /
    box, so each record's other entries are scaled by the median ratio of
    its re-timed entries (no bias between re-timed and 7-launch entries)."""
    key = lambda t: (t["V"], t["S"], t["W"], t["F"], t["G"], t.get("mode", 0), t.get("order", 0))
    rc = {}
    for p in paths:
        for r in json.load(open(p)):
            rc[(r["graph"], r["K"])] = {key(t): t["ms"] for t in r["table"]}
    n = 0
    for r in recs:
        m = rc.get((r["graph"], r["K"]))
        if not m:
            continue
        ratios = [m[key(t)] / t["ms"] for t in r["table"] if key(t) in m and t["ms"] > 0]
        scale = float(np.median(ratios)) if ratios else 1.0
        table = []
        for t in r["table"]:
            t = dict(t)
            t["ms"] = m[key(t)] if key(t) in m else t["ms"] * scale
            table.append(t)
        r["table"] = table
        n += 1
    return n


def guard_label(r, lab):
    """decide.cpp's guards applied to a forest label (mirror)."""
    mode, V, S, W, F, P, order = lab
    f = r["features"]
    K = r["K"]
    if mode == 3 and (K % 4 != 0 or f["d_max"] > 64.0):
        mode = 0
    if V == 2 and f["pr2"] >= 0.45:
        V = 1
    if mode == 0 and P > 1 and f["n"] * K * 4.0 > 2.0 * L2_BYTES and (((K + 3) // 4) + 31) // 32 <= 8:
        F, P = ((K + 3) // 4 + 31) // 32, 1
    if mode == 0 and V == 1 and S == 0:  # the sub-wave hub guard
        q = (K + 3) // 4
        G = 1
        while G < -(-q // (F * P)) and G < 32:
            G <<= 1
        if f["n"] <= 148 * 24 * (32 / G) and f["d_max"] >= 4 * (-(-f["d_hat"] // 32) * 32):
            S = 1
    return (mode, V, S, W, F, P, order if mode == 0 else 0)


def build_matrix(recs):
    keys = set()
    for r in recs:
        for t in r["table"]:
            k = label_of(r["K"], t)
            if k is not None:
                keys.add(k)
    keys = sorted(keys)
    kidx = {k: i for i, k in enumerate(keys)}
    perf = np.zeros((len(recs), len(keys)))
    X = np.zeros((len(recs), NFEAT))
    for i, r in enumerate(recs):
        best = min(t["ms"] for t in r["table"])
        for t in r["table"]:
            k = label_of(r["K"], t)
            if k is not None:
                perf[i, kidx[k]] = best / t["ms"]
        X[i, :16] = [r["features"][f] for f in FEATS]
        X[i, 16] = math.log2(r["K"])
        X[i, 17] = math.log2(max(r["features"]["n"], 1.0) * r["K"] * 4.0 / L2_BYTES)
    return keys, X, perf


class Node:
    def __init__(self, label=None, feat=-1, thr=0.0, left=None, right=None):
        self.label, self.feat, self.thr, self.left, self.right = label, feat, thr, left, right


def fit(X, perf, depth, min_leaf, rng=None, mtry=None):
    """Cost-sensitive CART.  With rng, each split draws `mtry` candidate
    features (random-forest trees)."""
    score = perf.sum(0)
    label = int(np.argmax(score))
    node = Node(label=label)
    if depth == 0 or len(X) < 2 * min_leaf:
        return node
    base = score[label]
    best = (base + 1e-9, None, None)
    feats = range(X.shape[1])
    if rng is not None:
        feats = rng.choice(X.shape[1], size=mtry or int(math.sqrt(X.shape[1])) + 1, replace=False)
    for f in feats:
        order = np.argsort(X[:, f], kind="stable")
        xs = X[order, f]
        cum = np.cumsum(perf[order], 0)
        tot = cum[-1]
        for i in range(min_leaf - 1, len(xs) - min_leaf):
            if xs[i] == xs[i + 1]:
                continue
            s = cum[i].max() + (tot - cum[i]).max()
            if s > best[0]:
                best = (s, f, 0.5 * (xs[i] + xs[i + 1]))
    if best[1] is None:
        return node
    f, thr = best[1], best[2]
    m = X[:, f] <= thr
    node.feat, node.thr = f, thr
    node.left = fit(X[m], perf[m], depth - 1, min_leaf, rng, mtry)
    node.right = fit(X[~m], perf[~m], depth - 1, min_leaf, rng, mtry)
    return node


def fit_forest(X, perf, trees, depth, min_leaf, seed=2605, mtry=None):
    """Random forest of cost-sensitive trees: bootstrap records,
    random feature subsets per split; prediction = majority vote."""
    if trees <= 1:
        return [fit(X, perf, depth, min_leaf)]
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(trees):
        idx = rng.integers(0, len(X), len(X))
        out.append(fit(X[idx], perf[idx], depth, min_leaf, rng, mtry))
    return out


def predict(model, x):
    roots = model if isinstance(model, list) else [model]
    votes = {}
    for node in roots:
        while node.feat >= 0:
            node = node.left if x[node.feat] <= node.thr else node.right
        votes[node.label] = votes.get(node.label, 0) + 1
    best = max(votes.values())
    return min(k for k, v in votes.items() if v == best)  # ties -> lowest label id


def flatten(root):
    nodes = []

    def walk(n):
        i = len(nodes)
        nodes.append(n)
        if n.feat >= 0:
            n._l = walk(n.left)
            n._r = walk(n.right)
        return i
    walk(root)
    return nodes


def rule_label(r, keys):
    """The pre-training rule of decide.cpp, for comparison."""
    f = r["features"]
    V = 2 if f["pr2"] < 0.30 else 1
    S = 1 if f["d_max"] > 8.0 * f["d_hat"] else 0
    d = r["decided"]
    return (0, V, S, 4, d["F"], passes_of(r["K"], d["F"], d["G"]), 0)


def evaluate(recs, keys, X, perf, test_idx, root, seed=0, guards=False):
    rng = np.random.default_rng(seed)
    pre, rnd, rule = [], [], []
    kidx = {k: i for i, k in enumerate(keys)}
    for i in test_idx:
        li = predict(root, X[i])
        if guards:
            g = guard_label(recs[i], keys[li])
            li = kidx.get(g, li)
        pre.append(perf[i, li])
        valid = np.nonzero(perf[i] > 0)[0]
        rnd.append(perf[i, rng.choice(valid)])
        rk = rule_label(recs[i], keys)
        rule.append(perf[i, kidx[rk]] if rk in kidx else float("nan"))
    return {"pre": float(np.mean(pre)), "rnd": float(np.mean(rnd)),
            "rule": float(np.nanmean(rule)) if rule else None, "n_test": len(test_idx)}


def emit_header(path, keys, model, source):
    """Forest -> csrc/decider_model.h: concatenated node arrays, per-tree roots,
    per-node label ids into a table of distinct labels."""
    roots = model if isinstance(model, list) else [model]
    nodes, root_idx = [], []
    for r in roots:
        base = len(nodes)
        ns = flatten(r)
        root_idx.append(base)
        for n in ns:
            n._gl = base + getattr(n, "_l", -1 - base) if n.feat >= 0 else -1
            n._gr = base + getattr(n, "_r", -1 - base) if n.feat >= 0 else -1
        nodes += ns
    used = sorted({n.label for n in nodes if n.feat < 0})
    lid = {k: i for i, k in enumerate(used)}
    lines = ["// Random-forest model of the SpMM-decider (DESIGN.md section 6).",
             f"// GENERATED by tools/train_decider.py from {source}; do not edit.",
             "#pragma once", "#define PSPMM_DECIDER_TRAINED 1",
             f'#define PSPMM_DECIDER_SOURCE "{source}"',
             "namespace pspmm_model {", f"constexpr int kTrees = {len(roots)};",
             f"constexpr int kNodes = {len(nodes)};", f"constexpr int kNumLabels = {len(used)};",
             "// feature index: 0..15 = pspmm_features fields in header order, 16 = log2(K),",
             "// 17 = log2(n K 4 / L2 bytes)"]
    lines.append("constexpr int kRoot[kTrees] = {" + ", ".join(map(str, root_idx)) + "};")
    lines.append("constexpr int kFeature[kNodes] = {" + ", ".join(str(n.feat) for n in nodes) + "};")
    lines.append("constexpr double kThreshold[kNodes] = {" +
                 ", ".join(repr(float(n.thr)) for n in nodes) + "};")
    lines.append("constexpr int kLeft[kNodes] = {" + ", ".join(str(n._gl) for n in nodes) + "};")
    lines.append("constexpr int kRight[kNodes] = {" + ", ".join(str(n._gr) for n in nodes) + "};")
    lines.append("// leaf -> label id (-1 for inner nodes)")
    lines.append("constexpr int kLeafLabel[kNodes] = {" +
                 ", ".join(str(lid[n.label]) if n.feat < 0 else "-1" for n in nodes) + "};")
    lines.append("// label: {mode, V, S, W, F, P (column passes), order}")
    lines.append("constexpr int kLabel[kNumLabels][7] = {" +
                 ", ".join("{" + ", ".join(map(str, keys[k])) + "}" for k in used) + "};")
    lines.append("}  // namespace pspmm_model")
    open(path, "w").write("\n".join(lines) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("inputs", nargs="+")
    ap.add_argument("--depth", type=int, default=10)
    ap.add_argument("--min-leaf", type=int, default=2)
    ap.add_argument("--trees", type=int, default=96, help="forest size (1 = a single CART tree)")
    ap.add_argument("--mtry", type=int, default=12, help="candidate features per split")
    ap.add_argument("--out-header", default=os.path.join(ROOT, "paper_2605_15695_b200", "csrc",
                                                         "decider_model.h"))
    ap.add_argument("--eval-json", default=None)
    ap.add_argument("--split-seed", type=int, default=2605,
                    help="seed of the 80/20 graph split (hyper-parameters are chosen on the "
                         "mean over several split seeds, DESIGN.md §6)")
    ap.add_argument("--recheck", nargs="*", default=[],
                    help="tools/sweep.py --recheck outputs overriding the sweep timings")
    ap.add_argument("--ship", choices=["split", "all"], default="split",
                    help="ship the forest evaluated on the 80/20 split (default) or refit on all")
    ap.add_argument("--train-workloads", action="store_true",
                    help="also train on the five bench workloads (default: held out, so the "
                         "bench's decided configs are out of sample; VERDICT r1 #8)")
    a = ap.parse_args()
    recs = load(a.inputs)
    n_re = apply_recheck(recs, a.recheck) if a.recheck else 0
    keys, X, perf = build_matrix(recs)
    is_wl = [r["graph"] in WORKLOADS for r in recs]
    graphs = sorted({r["graph"] for r, w in zip(recs, is_wl) if not w})
    rng = np.random.default_rng(a.split_seed)
    test_graphs = set(rng.choice(graphs, size=max(1, len(graphs) // 5), replace=False).tolist())
    tr = [i for i, r in enumerate(recs) if r["graph"] not in test_graphs and
          (a.train_workloads or not is_wl[i])]
    te = [i for i, r in enumerate(recs) if r["graph"] in test_graphs]
    wl = [i for i in range(len(recs)) if is_wl[i]]
    report = {"records": len(recs), "graphs": len(graphs), "labels": len(keys),
              "rechecked_records": n_re, "split_seed": a.split_seed,
              "test_graphs": sorted(test_graphs),
              "workloads_in_training": bool(a.train_workloads),
              "protocol": "80/20 split by corpus graph (P:399); the five bench workloads are "
                          "never trained on (unless --train-workloads) and reported apart; "
                          "normalized performance = t_best / t; rnd = a uniformly random valid "
                          "lattice config; rule = the untrained decide.cpp rule; "
                          "+guards = decide.cpp's three guards applied to the forest's label"}
    for name, trees in (("tree", 1), ("forest", a.trees)):
        model = fit_forest(X[tr], perf[tr], trees, a.depth, a.min_leaf, mtry=a.mtry)
        per_k = {}
        for K in sorted({r["K"] for r in recs}):
            idx = [i for i in te if recs[i]["K"] == K]
            if idx:
                per_k[K] = evaluate(recs, keys, X, perf, idx, model)
        report[name] = {"held_out": evaluate(recs, keys, X, perf, te, model),
                        "held_out_guards": evaluate(recs, keys, X, perf, te, model, guards=True),
                        "train": evaluate(recs, keys, X, perf, tr, model),
                        "held_out_per_K": per_k}
        if wl:
            report[name]["workloads"] = {
                recs[i]["graph"]: {"K": recs[i]["K"],
                                   "pre": float(perf[i, predict(model, X[i])]),
                                   "pre_guards": evaluate(recs, keys, X, perf, [i], model,
                                                          guards=True)["pre"],
                                   "label": list(keys[predict(model, X[i])])}
                for i in wl}
    # the shipped model is the evaluated one: the forest fit on the training
    # split, so the held-out and per-workload numbers above describe exactly
    # what the library does (--ship all: refit on every corpus record)
    if a.ship == "all":
        fit_idx = [i for i in range(len(recs)) if a.train_workloads or not is_wl[i]]
        model = fit_forest(X[fit_idx], perf[fit_idx], a.trees, a.depth, a.min_leaf, mtry=a.mtry)
    report["shipped"] = a.ship
    emit_header(a.out_header, keys, model, ",".join(os.path.basename(x) for x in a.inputs))
    print(json.dumps(report, indent=1))
    if a.eval_json:
        json.dump(report, open(a.eval_json, "w"), indent=1)


if __name__ == "__main__":
    sys.exit(main())
