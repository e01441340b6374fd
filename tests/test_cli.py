"""(f4) CLI host logic (no GPU): Matrix Market intake into canonical CSR and
the argument surface (SPEC cli module)."""
import numpy as np
import pytest

from paper_2605_15695_b200 import cli


def _write(tmp_path, text, name="a.mtx"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_mtx_general_real_sorted_and_duplicates_summed(tmp_path):
    p = _write(tmp_path, "%%MatrixMarket matrix coordinate real general\n% comment\n"
               "3 4 5\n3 1 2.5\n1 4 1.0\n1 2 -1.0\n3 1 0.5\n2 3 7\n")
    rp, ci, val, n, nc = cli.read_mtx(p)
    assert (n, nc) == (3, 4)
    assert rp.tolist() == [0, 2, 3, 4]
    assert ci.tolist() == [1, 3, 2, 0]
    assert val.tolist() == [-1.0, 1.0, 7.0, 3.0]  # (3,1) = 2.5 + 0.5
    assert rp.dtype == np.int32 and ci.dtype == np.int32 and val.dtype == np.float32


def test_mtx_symmetric_pattern_mirrors_off_diagonal(tmp_path):
    p = _write(tmp_path, "%%MatrixMarket matrix coordinate pattern symmetric\n"
               "3 3 3\n2 1\n3 3\n3 1\n")
    rp, ci, val, n, nc = cli.read_mtx(p)
    dense = np.zeros((3, 3))
    for i in range(3):
        dense[i, ci[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    assert np.array_equal(dense, np.array([[0, 1, 1], [1, 0, 0], [1, 0, 1]]))


def test_mtx_empty_matrix(tmp_path):
    p = _write(tmp_path, "%%MatrixMarket matrix coordinate real general\n5 5 0\n")
    rp, ci, val, n, nc = cli.read_mtx(p)
    assert rp.tolist() == [0] * 6 and len(ci) == 0 and n == 5


@pytest.mark.parametrize("text", [
    "not a header\n1 1 0\n",
    "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
])
def test_mtx_rejects_bad_input(tmp_path, text):
    with pytest.raises(cli.InputError):
        cli.read_mtx(_write(tmp_path, text))


def test_npz_input(tmp_path):
    p = str(tmp_path / "g.npz")
    np.savez(p, rowptr=np.array([0, 1, 2]), colidx=np.array([1, 0]))
    rp, ci, val, n, nc = cli.read_matrix(p)
    assert n == nc == 2 and val.tolist() == [1.0, 1.0]


def test_parser_rejects_v3_and_requires_dim():
    ap = cli.build_parser()
    with pytest.raises(SystemExit) as e:
        ap.parse_args(["convert", "x.mtx", "--v", "3", "--out", "y"])
    assert e.value.code == 2
    with pytest.raises(SystemExit):
        ap.parse_args(["predict", "x.mtx"])
    a = ap.parse_args(["spmm", "x.mtx", "--dim", "48", "--v", "2", "--balance", "--auto"])
    assert (a.dim, a.v, a.balance, a.auto) == (48, 2, True, True)


def test_missing_input_is_an_input_error(tmp_path):
    assert cli.main(["features", str(tmp_path / "nope.mtx")]) == cli.EXIT_INPUT


@pytest.mark.parametrize("dim", [16, 32, 48, 64, 128, 200, 256])
def test_bench_lattice_covers_dim(dim):
    q = (dim + 3) // 4
    lat = cli.lattice(dim)
    assert len(lat) == len(set(lat)) > 0
    for V, S, W, F, G in lat:
        assert V in (1, 2) and S in (0, 1) and W in (2, 4, 8)
        assert G & (G - 1) == 0 and G <= 32
        assert G * F >= q or G == 32


def test_mtx_explicit_zeros_dropped(tmp_path):
    """SPEC load_matrix_market: explicit zeros (and duplicates summing to 0)
    are not stored, so nnz and the Table-3 features see only true nonzeros."""
    p = _write(tmp_path, "%%MatrixMarket matrix coordinate real general\n"
               "3 3 5\n1 1 0.0\n1 2 2.0\n2 3 1.5\n2 3 -1.5\n3 1 4\n")
    rp, ci, val, n, nc = cli.read_mtx(p)
    assert rp.tolist() == [0, 1, 1, 2]
    assert ci.tolist() == [1, 0] and val.tolist() == [2.0, 4.0]
