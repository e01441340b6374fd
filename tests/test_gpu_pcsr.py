"""(a1, a4, a5) GPU PCSR builder: bit-exact against the oracle's arrays
(oracle/oracle.c, c-2), including the derived metrics, edge cases and the
CSR intake errors."""
import numpy as np
import pytest

import gen
import oracle
from conftest import golden
from gpu_util import dev

pytestmark = pytest.mark.gpu


def _api():
    from paper_2605_15695_b200 import api
    return api


def pin_x():
    g = golden("pin_x.json")
    return gen.Graph("pin_x", g["n"], np.array(g["rowPtr"], np.int32),
                     np.array(g["colIdx"], np.int32), np.array(g["val"], np.float32))


GRAPHS = {
    "pin_x": pin_x,
    "uniform": lambda: gen.uniform(1001, 7, 1),
    "powerlaw": lambda: gen.powerlaw(3000, 12, 2.0, 2),
    "banded": lambda: gen.banded(2049, 5, 3),
    "community": lambda: gen.community(4000, 64, 20, 0.85, 4),
    "giant": lambda: gen.giant_row(5001, 4990, 3, 5),
    "empty_rows": lambda: gen.with_empty_rows(gen.uniform(777, 9, 6), 0.35, 7),
    "cora": lambda: gen.config_graph("cora"),
    "reddit_s": lambda: gen.config_graph("reddit", 0.01),
    "roadnet_s": lambda: gen.config_graph("roadnet", 0.005),
    "proteins_s": lambda: gen.config_graph("proteins", 0.02),
    "one_row": lambda: gen.Graph("one", 1, np.array([0, 1], np.int32), np.array([0], np.int32),
                                 np.array([2.5], np.float32)),
}


def compare(g, V, S, omega, sg_override=0):
    api = _api()
    ref = oracle.pcsr_build(g.rowptr, g.colidx, g.val, V, S, omega, sg_override)
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, S, omega, sg_override)
    e = A.export()
    assert np.array_equal(e["rowPtr"], ref["rowPtr"])
    assert np.array_equal(e["colIdx"], ref["colIdx"])
    assert np.array_equal(e["val"].view(np.uint32), ref["val"].view(np.uint32))  # bit-exact
    assert np.array_equal(e["TRow"], ref["TRow"])
    assert e["nnz_v"] == ref["nnz_v"] and e["num_panels"] == ref["num_panels"]
    assert e["num_chunks"] == ref["num_chunks"] and e["sg"] == ref["sg"]
    assert e["sr"] == ref["sr"]
    assert (np.isnan(e["pr"]) and np.isnan(ref["pr"])) or e["pr"] == ref["pr"]
    return e


@pytest.mark.parametrize("name", sorted(GRAPHS))
@pytest.mark.parametrize("V", [1, 2])
@pytest.mark.parametrize("S", [0, 1])
@pytest.mark.parametrize("omega", [4, 32])
def test_bit_exact(name, V, S, omega):
    compare(GRAPHS[name](), V, S, omega)


@pytest.mark.parametrize("sg", [1, 3, 4, 64])
def test_sg_override(sg):
    compare(GRAPHS["powerlaw"](), 2, 1, 32, sg)


def test_pin_x_golden_on_gpu():
    g = golden("pin_x.json")
    for key, want in g["pcsr"].items():
        e = compare(pin_x(), int(key[1]), int(key[3]), g["omega"])
        assert e["rowPtr"].tolist() == want["rowPtr"]
        assert e["TRow"].tolist() == want["TRow"]


def test_empty_matrix():
    api = _api()
    g = gen.Graph("empty", 9, np.zeros(10, np.int32), np.zeros(0, np.int32),
                  np.zeros(0, np.float32))
    for V in (1, 2):
        compare(g, V, 0, 32)
    rp, ci, vl = dev(g)
    with pytest.raises(api.PspmmError) as e:
        api.pspmm_pcsr_build(g.n, 0, rp, ci, vl, 1, 1)
    assert e.value.status == api.PSPMM_ERR_EMPTY
    compare(g, 2, 1, 32, sg_override=8)  # defined with an explicit SG


def test_rect_build_matches_oracle_arrays():
    api = _api()
    import torch
    g = gen.uniform(300, 6, 11)
    # widen the column space: columns stay valid, n_cols > n_rows
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, 2, 1, n_cols=5000)
    ref = oracle.pcsr_build(g.rowptr, g.colidx, g.val, 2, 1)
    e = A.export()
    assert np.array_equal(e["colIdx"], ref["colIdx"]) and np.array_equal(e["rowPtr"], ref["rowPtr"])
    bad = torch.tensor([0, 1, 2], dtype=torch.int32, device="cuda")
    with pytest.raises(api.PspmmError):
        api.pspmm_pcsr_build(2, 2, bad, torch.tensor([0, 7], dtype=torch.int32, device="cuda"),
                             torch.ones(2, device="cuda"), 1, 0, n_cols=5)


@pytest.mark.parametrize("case", ["unsorted", "duplicate", "col_range", "negative_col",
                                  "rowptr_decreasing", "rowptr_end", "rowptr_start"])
def test_not_canonical(case):
    api = _api()
    import torch
    rp = [0, 2, 4, 5]
    ci = [0, 2, 1, 2, 0]
    if case == "unsorted":
        ci = [2, 0, 1, 2, 0]
    elif case == "duplicate":
        ci = [1, 1, 1, 2, 0]
    elif case == "col_range":
        ci = [0, 3, 1, 2, 0]
    elif case == "negative_col":
        ci = [0, 2, -1, 2, 0]
    elif case == "rowptr_decreasing":
        rp = [0, 3, 2, 5]
    elif case == "rowptr_end":
        rp = [0, 2, 4, 4]
    elif case == "rowptr_start":
        rp = [1, 2, 4, 5]
    t = lambda x, d: torch.tensor(x, dtype=d, device="cuda")  # noqa: E731
    with pytest.raises(api.PspmmError) as e:
        api.pspmm_pcsr_build(3, 5, t(rp, torch.int32), t(ci, torch.int32),
                             t([1.0] * 5, torch.float32), 1, 0)
    assert e.value.status == api.PSPMM_ERR_NOT_CANONICAL
    with pytest.raises(api.PspmmError):
        api.pspmm_csr_validate(3, 5, t(rp, torch.int32), t(ci, torch.int32))


def test_bad_config():
    api = _api()
    g = GRAPHS["uniform"]()
    rp, ci, vl = dev(g)
    for V, S, omega in [(3, 0, 32), (0, 0, 32), (1, 2, 32), (1, 0, 0)]:
        with pytest.raises(api.PspmmError) as e:
            api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, S, omega)
        assert e.value.status == api.PSPMM_ERR_CONFIG
