"""(a3) The compiled decider: the C function evaluates exactly the tree that
tools/train_decider.py emitted into csrc/decider_model.h (re-walked here in
Python from the header's arrays), and the trainer's cost-sensitive CART
recovers a planted rule.  Parity of C is independent of the config (c-4:
"parity unpinned" for the decider itself); these tests pin the plumbing."""
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "paper_2605_15695_b200", "csrc", "decider_model.h")
FEATS = ("n", "n_hat", "nnz", "delta", "d", "d_hat", "d_max", "cv", "cv_hat", "sr1", "sr2", "rho",
         "b", "b_max", "pr1", "pr2")


def parse_header():
    text = open(HEADER).read()
    trained = "#define PSPMM_DECIDER_TRAINED 1" in text

    def arr(name):
        m = re.search(r"\b" + name + r"\[\w+\](?:\[\d\])? = \{(.*)\};", text)
        return m.group(1)

    roots = [int(x) for x in arr("kRoot").split(",")]
    feat = [int(x) for x in arr("kFeature").split(",")]
    thr = [float(x) for x in arr("kThreshold").split(",")]
    left = [int(x) for x in arr("kLeft").split(",")]
    right = [int(x) for x in arr("kRight").split(",")]
    leaf = [int(x) for x in arr("kLeafLabel").split(",")]
    labs = [tuple(int(y) for y in g.split(",")) for g in re.findall(r"\{([-\d, ]+)\}",
                                                                     arr("kLabel"))]
    return trained, roots, feat, thr, left, right, leaf, labs


def walk(model, f, K):
    """Majority vote of the forest, ties to the lowest label id."""
    _, roots, feat, thr, left, right, leaf, labs = model
    x = [f[k] for k in FEATS] + [math.log2(K), math.log2(max(f["n"], 1.0) * K * 4.0 / L2_B200)]
    votes = [0] * len(labs)
    for node in roots:
        while feat[node] >= 0:
            node = left[node] if x[feat[node]] <= thr[node] else right[node]
        votes[leaf[node]] += 1
    return labs[votes.index(max(votes))]


def ceil_pow2(x):
    p = 1
    while p < x and p < 32:
        p <<= 1
    return p


L2_B200 = 132644864.0  # decide.cpp kL2Bytes


def test_c_decider_evaluates_the_header_tree():
    from paper_2605_15695_b200 import api
    model = parse_header()
    if not model[0]:
        pytest.skip("decider not trained yet (rule mode)")
    rng = np.random.default_rng(0)
    for _ in range(400):
        n = float(rng.integers(1000, 3_000_000))
        d = float(rng.uniform(1, 600))
        f = dict(n=n, n_hat=n * rng.uniform(0.5, 1), nnz=n * d, delta=rng.uniform(0.5, 1), d=d,
                 d_hat=d * rng.uniform(1, 2), d_max=d * rng.uniform(1, 100),
                 cv=rng.uniform(0, 5), cv_hat=rng.uniform(0, 5), sr1=rng.uniform(1, 2),
                 sr2=rng.uniform(1, 2), rho=d / n, b=rng.uniform(0, n), b_max=n - 1, pr1=0.0,
                 pr2=rng.uniform(0, 0.5))
        K = int(rng.choice([8, 16, 32, 48, 64, 96, 128, 160, 256]))
        mode, V, S, W, F, P, order = walk(model, f, K)
        if mode == 3 and f["d_max"] > 64:  # hub-row guard (decide.cpp)
            mode = 0
        if V == 2 and f["pr2"] >= 0.45:  # padding guard (decide.cpp)
            V = 1
        c = api.pspmm_decide_config(f, K)
        q = (K + 3) // 4
        G = ceil_pow2(-(-q // (F * P))) if mode != 2 else 0
        if mode == 0 and -(-K // (4 * G * F)) > 1 and n * K * 4 > 2 * L2_B200 and -(-q // 32) <= 8:
            # the single-pass guard for B far beyond L2 (decide.cpp)
            F = -(-q // 32)
            G = ceil_pow2(-(-q // F))
        if (mode == 0 and V == 1 and S == 0 and
                n <= 148 * 24 * (32 / G) and f["d_max"] >= 4 * (-(-f["d_hat"] // 32) * 32)):
            S = 1  # the sub-wave hub guard (decide.cpp)
        if mode == 2 and K % 32 == 0:
            assert (c.mode, c.V, c.S, c.W) == (2, V, S, W)
        elif mode == 3 and K % 4 == 0:
            assert (c.mode, c.V, c.S, c.W, c.F) == (mode, V, S, W, F)
        else:
            assert (c.mode, c.V, c.S, c.W) == (0, V, S, W)
            if mode == 0:
                assert c.F == F and c.G == G
                assert c.order == order


def test_single_pass_guard():
    """B far beyond L2 (n K 4 > 2 x L2): whatever the forest says, one column
    pass of up to 32 lanes; below that size the forest's passes stand."""
    from paper_2605_15695_b200 import api
    f = dict(n=2449029.0, n_hat=2449029.0, nnz=123718280.0, delta=1.0, d=50.5, d_hat=50.5,
             d_max=17425.0, cv=1.08, cv_hat=1.08, sr1=1.23, sr2=1.2, rho=2.06e-5, b=2.3e6,
             b_max=2449010.0, pr1=0.0, pr2=0.5)
    for K in (128, 256, 512):
        c = api.pspmm_decide_config(f, K)
        if c.mode == 0:
            assert -(-K // (4 * c.G * c.F)) == 1, (K, c)


def test_trainer_recovers_planted_rule():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import train_decider as td
    rng = np.random.default_rng(1)
    recs = []
    for i in range(120):
        f = {k: float(rng.uniform(0, 1)) for k in FEATS}
        f["d_max"] = float(rng.uniform(0, 100))
        K = 64
        # planted: S = 1 is 2x faster iff d_max > 50, V = 2 iff pr2 < 0.3
        table = []
        for V in (1, 2):
            for S in (0, 1):
                ms = 1.0
                ms *= 0.5 if (S == 1) == (f["d_max"] > 50) else 1.0
                ms *= 0.7 if (V == 2) == (f["pr2"] < 0.3) else 1.0
                table.append({"V": V, "S": S, "W": 2, "F": 1, "G": 16, "mode": 0, "ms": ms})
        recs.append({"graph": f"g{i}", "K": K, "features": f, "table": table,
                     "decided": {"F": 1, "G": 16}})
    keys, X, perf = td.build_matrix(recs)
    root = td.fit(X, perf, 4, 3)
    ev = td.evaluate(recs, keys, X, perf, list(range(len(recs))), root)
    assert ev["pre"] > 0.99 and ev["rnd"] < 0.8


def test_sub_wave_hub_guard():
    """Every S = 0 unit in one wave and rows of >= 4 SG nonzeros: split them
    (S = 1), at every K; Cora-shaped features (n = 2708, d_max = 168, SG =
    32).  (Graphs outside the regime: test_c_decider_evaluates_the_header_tree
    mirrors the guard over 400 random feature vectors.)"""
    from paper_2605_15695_b200 import api
    cora = dict(n=2708.0, n_hat=2485.0, nnz=10556.0, delta=0.918, d=3.9, d_hat=4.25,
                d_max=168.0, cv=1.56, cv_hat=1.47, sr1=1.01, sr2=1.02, rho=0.00144, b=1078.0,
                b_max=2706.0, pr1=0.0, pr2=0.5)
    for K in (16, 32, 64, 128, 256):
        c = api.pspmm_decide_config(cora, K)
        assert c.mode != 0 or c.V != 1 or c.S == 1, (K, c)
