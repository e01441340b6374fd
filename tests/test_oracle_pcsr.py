"""Pins for the PCSR / metric oracle (c-2): the paper's Table 2 values,
SPEC's worked example S:125, the hand-derived pin X, and properties that
hold for every input (losslessness, conservation, bound, metric ranges)
checked by brute force that does not call the oracle's procedure."""
from fractions import Fraction

import numpy as np
import pytest

import gen
import oracle
from conftest import golden


# ---------------------------------------------------------------- Eq. 1 / T2
def test_gap_table2_every_cell():
    t = golden("table2_gap.json")
    for F, row in t["gap"].items():
        for dim, want in zip(t["dims"], row):
            if want is None:  # N/A: F > CEIL(dim/omega)
                assert int(F) > -(-dim // t["omega"])
                continue
            assert oracle.gap(dim, int(F), t["omega"]) == want, (dim, F)


def test_gap_spec_examples():
    # S:134-137
    assert oracle.gap(96, 2, 32) == 32
    assert oracle.gap(128, 3, 32) == 64
    assert oracle.gap(64, 2, 32) == 0
    assert oracle.gap(160, 4, 32) == 96
    # dim smaller than one segment: tn = dim, tr = dim -> no gap
    assert oracle.gap(16, 1, 32) == 16 - 16


# ------------------------------------------------------------ worked examples
def test_spec_s125_example():
    t = golden("spec_s125_pcsr.json")
    sym = t["symbols"]
    ent = sorted((r, c, sym[s]) for r, c, s in t["entries"])
    n = t["n"]
    rowptr = np.zeros(n + 1, np.int32)
    for r, _, _ in ent:
        rowptr[r + 1] += 1
    rowptr = np.cumsum(rowptr)
    p = oracle.pcsr_build(rowptr, [c for _, c, _ in ent], [v for _, _, v in ent], t["V"], t["S"])
    assert p["rowPtr"].tolist() == t["rowPtr"]
    assert p["colIdx"].tolist() == t["colIdx"]
    assert p["val"].tolist() == [sym[x] if isinstance(x, str) else x for x in t["val"]]
    assert p["TRow"].tolist() == t["TRow"]


@pytest.mark.parametrize("key", ["V1S0", "V1S1", "V2S0", "V2S1"])
def test_pin_x(key):
    g = golden("pin_x.json")
    want = g["pcsr"][key]
    V, S = int(key[1]), int(key[3])
    p = oracle.pcsr_build(g["rowPtr"], g["colIdx"], g["val"], V, S, g["omega"])
    assert p["rowPtr"].tolist() == want["rowPtr"]
    assert p["colIdx"].tolist() == want["colIdx"]
    assert p["val"].tolist() == want["val"]
    assert p["TRow"].tolist() == want["TRow"]
    if "sg" in want:
        assert p["sg"] == want["sg"]
    pr = Fraction(want["pr_num"], want["pr_den"]) if "pr_num" in want else Fraction(want["pr"])
    sr = Fraction(want["sr_num"], want["sr_den"]) if "sr_num" in want else Fraction(want["sr"])
    assert p["pr"] == pytest.approx(float(pr), abs=1e-15)
    assert p["sr"] == pytest.approx(float(sr), abs=1e-15)


def _panels_9_2(n=9):
    # row 0 has 9 nonzeros, row 1 has 2, the rest are empty (V=1)
    rowptr = [0, 9, 11] + [11] * (n - 2)
    colidx = list(range(9)) + [0, 5]
    return rowptr, colidx, list(range(1, 12))


def test_c18_chunking_eq3_reading():
    # c-18: Eq. 3 with omega=4 gives SG = ceil(11/(2*4))*4 = 8
    r, c, v = _panels_9_2()
    p = oracle.pcsr_build(r, c, v, 1, 1, omega=4)
    assert p["sg"] == 8
    assert p["rowPtr"].tolist() == [0, 8, 9, 11] + [11] * 7
    assert p["TRow"].tolist() == [0, 0, 1, 2, 3, 4, 5, 6, 7, 8]
    assert p["sr"] == pytest.approx(11 / 10)


def test_c18_chunking_spec_sg4():
    # S:127 with the SG=4 override: 9 -> 4+4+1, then 2
    r, c, v = _panels_9_2()
    p = oracle.pcsr_build(r, c, v, 1, 1, omega=4, sg_override=4)
    assert p["rowPtr"].tolist()[:5] == [0, 4, 8, 9, 11]
    assert p["TRow"].tolist()[:4] == [0, 0, 0, 1]
    assert p["sr"] == pytest.approx(12 / 10)


# ---------------------------------------------------------- brute-force props
def brute_vectors(rowptr, colidx, val, n, V):
    """{(panel, col): [V values]} straight from the definition."""
    vec = {}
    for i in range(n):
        for p in range(rowptr[i], rowptr[i + 1]):
            key = (i // V, int(colidx[p]))
            vec.setdefault(key, [0.0] * V)[i % V] = float(val[p])
    return vec


GRAPHS = [
    lambda: gen.uniform(61, 4, 1),
    lambda: gen.powerlaw(200, 9, 2.1, 2),
    lambda: gen.banded(101, 2, 3),
    lambda: gen.community(130, 8, 7, 0.9, 4),
    lambda: gen.giant_row(90, 85, 2, 5),
    lambda: gen.with_empty_rows(gen.uniform(77, 6, 6), 0.4, 7),
    lambda: gen.config_graph("cora"),
]


@pytest.mark.parametrize("make", GRAPHS)
@pytest.mark.parametrize("V", [1, 2, 3])
@pytest.mark.parametrize("omega", [4, 32])
def test_pcsr_properties(make, V, omega):
    g = make()
    n = g.n
    ref = brute_vectors(g.rowptr, g.colidx, g.val, n, V)
    p0 = oracle.pcsr_build(g.rowptr, g.colidx, g.val, V, 0, omega)
    P = -(-n // V)
    assert p0["num_panels"] == P and len(p0["rowPtr"]) == P + 1
    assert p0["nnz_v"] == len(ref)
    # lossless: the (panel, col) -> values map equals the definition, ordered
    got = {}
    for pnl in range(P):
        cols = p0["colIdx"][p0["rowPtr"][pnl]:p0["rowPtr"][pnl + 1]]
        assert np.all(np.diff(cols) > 0)  # ascending within a panel (c-8)
        for j, c in enumerate(cols):
            i = p0["rowPtr"][pnl] + j
            got[(pnl, int(c))] = p0["val"][i * V:(i + 1) * V].tolist()
    assert got == {k: [np.float32(x).item() for x in v] for k, v in ref.items()}
    # metrics: PR = 1 - nnz/(nnz_V V) in [0, 1-1/V]
    if g.nnz:
        assert p0["pr"] == pytest.approx(1 - g.nnz / (len(ref) * V), abs=1e-15)
        assert -1e-15 <= p0["pr"] <= 1 - 1 / V + 1e-15
        if V == 1:
            assert p0["pr"] == 0.0
    # S = 1: conservation, bound, TRow, SG, SR
    p1 = oracle.pcsr_build(g.rowptr, g.colidx, g.val, V, 1, omega)
    assert np.array_equal(p1["colIdx"], p0["colIdx"]) and np.array_equal(p1["val"], p0["val"])
    SG = p1["sg"]
    L = np.diff(p0["rowPtr"])
    nonempty = int((L > 0).sum())
    assert SG % omega == 0 and SG >= omega
    assert SG == -(-len(ref) // (nonempty * omega)) * omega  # Eq. 3 brute
    chunks = np.diff(p1["rowPtr"])
    assert chunks.max() <= SG
    assert len(p1["TRow"]) == len(chunks)
    assert np.all(np.diff(p1["TRow"]) >= 0)
    for pnl in range(P):
        mine = chunks[p1["TRow"] == pnl]
        assert mine.sum() == L[pnl]
        assert len(mine) == max(1, -(-int(L[pnl]) // SG))
    assert p1["sr"] == pytest.approx((len(chunks) + 1) / (P + 1), abs=1e-15)
    assert p1["sr"] >= 1.0
    assert (p1["sr"] == 1.0) == bool(L.max() <= SG)
    # S = 0 bound = max panel workload
    assert chunks.max() <= L.max()


def test_v1_is_csr():
    g = gen.powerlaw(500, 11, 2.3, 9)
    p = oracle.pcsr_build(g.rowptr, g.colidx, g.val, 1, 0)
    assert np.array_equal(p["rowPtr"], g.rowptr)
    assert np.array_equal(p["colIdx"], g.colidx)
    assert np.array_equal(p["val"], g.val)
    assert p["pr"] == 0.0


def test_pr_examples():
    # S:145 identity V=2 -> 0.5; S:146 dense 2x2 -> 0
    I = oracle.pcsr_build(np.arange(5), np.arange(4), np.ones(4), 2, 0)
    assert I["pr"] == 0.5
    D = oracle.pcsr_build([0, 2, 4], [0, 1, 0, 1], [1, 2, 3, 4], 2, 0)
    assert D["pr"] == 0.0
    # monotonicity S:170: duplicate each row into its panel partner -> PR2 = 0
    g = gen.uniform(40, 5, 3)
    rows, cols = [], []
    for i in range(0, g.n, 2):
        cs = g.colidx[g.rowptr[i]:g.rowptr[i + 1]]
        for r in (i, i + 1):
            rows += [r] * len(cs)
            cols += list(cs)
    rp, ci = gen.csr_from_pairs(g.n, np.array(rows), np.array(cols))
    dup = oracle.pcsr_build(rp, ci, np.ones(len(ci)), 2, 0)
    assert dup["pr"] == 0.0


@pytest.mark.parametrize("dhat,omega,want", [(5, 32, 32), (33, 32, 64), (64, 32, 64)])
def test_sg_examples(dhat, omega, want):
    # one non-empty panel holding d^_V vectors
    n = max(dhat, 2)
    p = oracle.pcsr_build([0, dhat] + [dhat] * (n - 1), list(range(dhat)), [1.0] * dhat, 1, 1, omega)
    assert p["sg"] == want


def test_all_empty_matrix():
    with pytest.raises(oracle.OracleError) as e:
        oracle.pcsr_build(np.zeros(6, np.int32), [], [], 1, 1)
    assert e.value.code == 5  # EMPTY: SG undefined
    p = oracle.pcsr_build(np.zeros(6, np.int32), [], [], 2, 0)
    assert p["nnz_v"] == 0 and p["rowPtr"].tolist() == [0, 0, 0, 0]
