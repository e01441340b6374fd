"""(f4) PCSR binary file (pspmm_pcsr_save / pspmm_pcsr_load) and
the CLI end to end.  A loaded file must reproduce the oracle's PCSR arrays
bit-exactly (pin X golden included), drive the engine like a freshly built
handle, and corrupt files must be rejected with the documented status."""
import os
import struct

import numpy as np
import pytest

import gen
import oracle
from conftest import golden
from gpu_util import assert_parity, dev, oracle_ref
from test_gpu_pcsr import GRAPHS

pytestmark = pytest.mark.gpu


def _api():
    from paper_2605_15695_b200 import api
    return api


@pytest.mark.parametrize("name", ["pin_x", "powerlaw", "giant", "empty_rows", "one_row",
                                  "reddit_s"])
@pytest.mark.parametrize("V,S", [(1, 0), (1, 1), (2, 0), (2, 1)])
def test_file_round_trip_matches_oracle(tmp_path, name, V, S):
    api = _api()
    g = GRAPHS[name]()
    omega = 4 if name == "pin_x" else 32
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, S, omega)
    path = str(tmp_path / "a.pcsr")
    api.pspmm_pcsr_save(A, path)
    L = api.pspmm_pcsr_load(path)
    ref = oracle.pcsr_build(g.rowptr, g.colidx, g.val, V, S, omega, 0)
    e = L.export()
    assert np.array_equal(e["rowPtr"], ref["rowPtr"])
    assert np.array_equal(e["colIdx"], ref["colIdx"])
    assert np.array_equal(e["val"].view(np.uint32), ref["val"].view(np.uint32))
    assert np.array_equal(e["TRow"], ref["TRow"])
    assert e["sg"] == ref["sg"] and e["sr"] == ref["sr"] and e["num_chunks"] == ref["num_chunks"]
    assert (np.isnan(e["pr"]) and np.isnan(ref["pr"])) or e["pr"] == ref["pr"]
    assert L.n_rows == g.n and L.n_cols == g.n
    # header: the SPEC's fields at the SPEC's offsets
    head = open(path, "rb").read(36)
    assert head[:4] == b"PCSR"
    ver, n, P, nv = struct.unpack_from("<IQQQ", head, 4)
    assert (ver, n, P, nv) == (1, g.n, ref["num_panels"], ref["nnz_v"])
    assert struct.unpack_from("<BBH", head, 32) == (V, S, omega)
    # the loaded handle drives the engine like the built one
    import torch
    K = 16
    B = gen.dense(g.n, K, 31)
    Bd = torch.from_numpy(B).cuda()
    C = torch.empty((g.n, K), device="cuda")
    api.pspmm_spmm_run(L, Bd, C, api.Config(V=V, S=S, omega=omega, W=4))
    torch.cuda.synchronize()
    r, mag = oracle_ref(g, B)
    assert_parity(C.cpu().numpy(), r, mag, f"loaded {name} V{V} S{S}")
    if name == "pin_x":
        gold = golden("pin_x.json")["pcsr"][f"V{V}S{S}"]
        assert e["rowPtr"].tolist() == gold["rowPtr"]
        assert e["TRow"].tolist() == gold.get("TRow", [])


def _saved(tmp_path, V=2, S=1):
    api = _api()
    g = GRAPHS["powerlaw"]()
    rp, ci, vl = dev(g)
    A = api.pspmm_pcsr_build(g.n, g.nnz, rp, ci, vl, V, S, 32)
    path = str(tmp_path / "ok.pcsr")
    api.pspmm_pcsr_save(A, path)
    return path, A.info


def _load_status(path):
    api = _api()
    try:
        api.pspmm_pcsr_load(path)
    except api.PspmmError as e:
        return e.status
    return 0


def test_corrupt_files_rejected(tmp_path):
    path, info = _saved(tmp_path)
    raw = bytearray(open(path, "rb").read())

    def variant(name, mutate):
        b = bytearray(raw)
        mutate(b)
        p = str(tmp_path / name)
        open(p, "wb").write(bytes(b))
        return _load_status(p)

    assert _load_status(path) == 0
    assert _load_status(str(tmp_path / "missing.pcsr")) == 1
    assert variant("magic", lambda b: b.__setitem__(0, ord("X"))) == 1
    assert variant("version", lambda b: struct.pack_into("<I", b, 4, 2)) == 7
    assert variant("v3", lambda b: struct.pack_into("<B", b, 32, 3)) == 1
    assert variant("trunc", lambda b: b.__delitem__(slice(len(b) - 4, len(b)))) == 1
    assert variant("extra", lambda b: b.extend(b"\0")) == 1
    rl = info["num_chunks"] + 1
    col0 = 72 + 8 * rl  # colIdx[0], colIdx[1] of panel 0: swap -> not ascending

    def swap_cols(b):
        a0, a1 = struct.unpack_from("<II", b, col0)
        struct.pack_into("<II", b, col0, a1, a0)
    assert variant("cols", swap_cols) == 2
    # rowPtr[1] beyond rowPtr[2] -> not monotone
    assert variant("rowptr", lambda b: struct.pack_into("<Q", b, 72 + 8, 10**9)) == 2
    trow0 = 72 + 8 * rl + 4 * info["nnz_v"] + 4 * info["nnz_v"] * info["V"]
    assert variant("trow", lambda b: struct.pack_into("<I", b, trow0, 5)) == 2


def _mtx(path, g):
    r = np.repeat(np.arange(g.n), np.diff(g.rowptr.astype(np.int64)))
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{g.n} {g.n} {g.nnz}\n")
        for i, j, v in zip(r, g.colidx, g.val):
            f.write(f"{i + 1} {j + 1} {float(v)!r}\n")


def test_cli_convert_inspect_spmm(tmp_path, capsys):
    import json
    from paper_2605_15695_b200 import api, cli
    g = gen.config_graph("reddit", 0.003)
    mtx = str(tmp_path / "g.mtx")
    _mtx(mtx, g)
    pc = str(tmp_path / "g.pcsr")
    assert cli.main(["convert", mtx, "--v", "2", "--balance", "--out", pc]) == 0
    conv = json.loads(capsys.readouterr().out)
    assert conv["V"] == 2 and conv["S"] == 1 and conv["nnz"] == g.nnz
    assert cli.main(["inspect", pc]) == 0
    ins = json.loads(capsys.readouterr().out)
    assert ins["nnz_v"] == conv["nnz_v"] and ins["n_cols"] == g.n
    K = 32
    B = gen.dense(g.n, K, 77)
    bp = str(tmp_path / "B.npy")
    np.save(bp, B)
    ref, mag = oracle_ref(g, B)
    for args in (["spmm", pc, "--dim", str(K), "--v", "2", "--balance"],
                 ["spmm", mtx, "--dim", str(K), "--auto"],
                 ["spmm", mtx, "--dim", str(K), "--f", "2", "--w", "8"]):
        out = str(tmp_path / "C.npy")
        assert cli.main(args + ["--b", bp, "--out", out]) == 0, args
        capsys.readouterr()
        assert_parity(np.load(out), ref, mag, " ".join(args[:2]))
    assert cli.main(["predict", mtx, "--dim", "64"]) == 0
    cfg = json.loads(capsys.readouterr().out)
    assert cfg["V"] in (1, 2) and cfg["S"] in (0, 1) and cfg["mode"] in (0, 2, 3)
    assert cli.main(["features", mtx]) == 0
    f = json.loads(capsys.readouterr().out)
    assert f["nnz"] == g.nnz and f["n"] == g.n
    # mismatched config for a PCSR file is an input error; a library error is 4
    assert cli.main(["spmm", pc, "--dim", "8", "--v", "1"]) == cli.EXIT_INPUT
    assert cli.main(["spmm", pc, "--dim", "8", "--v", "2", "--balance", "--w", "3"]) == \
        cli.EXIT_LIB
    csv_out = str(tmp_path / "bench.csv")
    assert cli.main(["bench", mtx, "--dims", "16", "--repeats", "2", "--out", csv_out]) == 0
    lines = open(csv_out).read().strip().splitlines()
    assert len(lines) == 1 + len(cli.lattice(16))
    assert os.path.getsize(csv_out) > 0
    _ = api
