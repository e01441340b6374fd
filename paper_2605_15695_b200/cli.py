"""Command-line surface (SPEC's cli module):
convert, inspect, features, predict, spmm, bench.

    python -m paper_2605_15695_b200.cli convert G.mtx --v 2 --balance --out G.pcsr
    python -m paper_2605_15695_b200.cli inspect G.pcsr
    python -m paper_2605_15695_b200.cli features G.mtx
    python -m paper_2605_15695_b200.cli predict G.mtx --dim 64
    python -m paper_2605_15695_b200.cli spmm G.mtx --dim 64 --auto --out C.npy
    python -m paper_2605_15695_b200.cli bench G.mtx --dims 32,64 --out sweep.csv

Inputs: Matrix Market coordinate files (real / integer / pattern; general or
symmetric; duplicates summed, pattern entries = 1.0), `.npz` archives with
rowptr / colidx / val, or (spmm, inspect) a PCSR file.  Every compute step
runs in libpspmm.so on the GPU; there is no CPU path.  Decider training is
tools/train_decider.py (the model is compiled into the library).
Exit codes: 0 ok, 2 usage error (argparse), 3 input error, 4 library error.
"""
from __future__ import annotations

import argparse
import csv
import json
import sys

import numpy as np

EXIT_INPUT = 3
EXIT_LIB = 4


class InputError(Exception):
    pass


# ---------------------------------------------------------------- input
def read_mtx(path):
    """Matrix Market coordinate file -> canonical CSR (rowptr, colidx, val,
    n_rows, n_cols)."""
    with open(path, "r") as f:
        header = f.readline().split()
        if len(header) < 5 or header[0] != "%%MatrixMarket" or header[1] != "matrix":
            raise InputError(f"{path}: not a Matrix Market matrix file")
        fmt, field, sym = header[2].lower(), header[3].lower(), header[4].lower()
        if fmt != "coordinate":
            raise InputError(f"{path}: only coordinate format is supported")
        if field not in ("real", "integer", "pattern"):
            raise InputError(f"{path}: field '{field}' not supported")
        if sym not in ("general", "symmetric"):
            raise InputError(f"{path}: symmetry '{sym}' not supported")
        line = f.readline()
        while line.startswith("%") or not line.strip():
            line = f.readline()
            if not line:
                raise InputError(f"{path}: missing size line")
        try:
            nr, nc, nz = (int(x) for x in line.split()[:3])
        except ValueError as e:
            raise InputError(f"{path}: bad size line") from e
        cols = 2 if field == "pattern" else 3
        data = np.loadtxt(f, ndmin=2, usecols=range(cols), comments="%") if nz else \
            np.zeros((0, cols))
    if data.shape[0] != nz:
        raise InputError(f"{path}: expected {nz} entries, found {data.shape[0]}")
    r = data[:, 0].astype(np.int64) - 1
    c = data[:, 1].astype(np.int64) - 1
    v = np.ones(nz, np.float64) if field == "pattern" else data[:, 2].astype(np.float64)
    if nz and (r.min() < 0 or c.min() < 0 or r.max() >= nr or c.max() >= nc):
        raise InputError(f"{path}: entry index out of range")
    if sym == "symmetric":
        off = r != c
        r, c, v = np.concatenate([r, c[off]]), np.concatenate([c, r[off]]), \
            np.concatenate([v, v[off]])
    return coo_to_csr(r, c, v, nr, nc)


def coo_to_csr(r, c, v, nr, nc):
    """Sort by (row, col), sum duplicates, drop zeros -> canonical CSR (int32 / fp32)."""
    if nr >= 2**31 or nc >= 2**31 or len(r) >= 2**31:
        raise InputError("matrix exceeds int32 indexing")
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    if len(r):
        new = np.ones(len(r), bool)
        new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        idx = np.cumsum(new) - 1
        v = np.bincount(idx, weights=v, minlength=int(idx[-1]) + 1)
        r, c = r[new], c[new]
        # explicit zeros (and duplicates summing to zero) are not stored
        # (SPEC load_matrix_market): they would inflate nnz and the features
        keep = v != 0
        r, c, v = r[keep], c[keep], v[keep]
    rowptr = np.zeros(nr + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=nr), out=rowptr[1:])
    return (rowptr.astype(np.int32), c.astype(np.int32), v.astype(np.float32), nr, nc)


def read_matrix(path):
    if path.endswith(".npz"):
        z = np.load(path)
        rp, ci = z["rowptr"].astype(np.int32), z["colidx"].astype(np.int32)
        val = z["val"].astype(np.float32) if "val" in z else np.ones(len(ci), np.float32)
        n = len(rp) - 1
        nc = int(z["n_cols"]) if "n_cols" in z else n
        return rp, ci, val, n, nc
    return read_mtx(path)


def is_pcsr(path):
    with open(path, "rb") as f:
        return f.read(4) == b"PCSR"


# ---------------------------------------------------------------- helpers
def _device_csr(rp, ci, val):
    import torch
    return (torch.from_numpy(rp).cuda(),
            torch.from_numpy(ci if len(ci) else np.zeros(1, np.int32)).cuda(),
            torch.from_numpy(val if len(val) else np.zeros(1, np.float32)).cuda())


def _features(api, rp, ci, n, omega):
    d_rp, d_ci, _ = _device_csr(rp, ci, np.zeros(0, np.float32))
    return api.pspmm_features_compute(n, int(rp[-1]), d_rp, d_ci, omega)


def _config(api, a, feats=None):
    if a.auto:
        if feats is None:
            raise InputError("--auto needs a CSR input (features), not a PCSR file")
        return api.pspmm_decide_config(feats, a.dim)
    return api.Config(W=a.w, F=a.f, V=a.v, S=int(a.balance), omega=a.omega, sg_override=a.sg,
                      G=a.g, mode=a.mode, order=a.order)


def _B(a, n_cols):
    if a.b:
        B = np.load(a.b).astype(np.float32)
        if B.ndim != 2 or B.shape[0] != n_cols:
            raise InputError(f"--b must be a {n_cols} x dim matrix")
        return np.ascontiguousarray(B)
    rng = np.random.default_rng(a.seed)
    return (rng.random((n_cols, a.dim), dtype=np.float32) * 2 - 1).astype(np.float32)


# ---------------------------------------------------------------- commands
def cmd_convert(a, api):
    rp, ci, val, n, nc = read_matrix(a.input)
    d_rp, d_ci, d_val = _device_csr(rp, ci, val)
    A = api.pspmm_pcsr_build(n, int(rp[-1]), d_rp, d_ci, d_val, a.v, int(a.balance), a.omega,
                             a.sg, n_cols=nc)
    api.pspmm_pcsr_save(A, a.out)
    print(json.dumps({"out": a.out, **A.info}))


def cmd_inspect(a, api):
    A = api.pspmm_pcsr_load(a.input)
    info = dict(A.info, n_cols=A.n_cols)
    if a.arrays:
        ex = A.export()
        info.update({k: ex[k].tolist() for k in ("rowPtr", "colIdx", "val", "TRow")})
    print(json.dumps(info))


def cmd_features(a, api):
    rp, ci, _, n, nc = read_matrix(a.input)
    if n != nc:
        raise InputError("Table-3 features are defined for square adjacency matrices")
    print(json.dumps(_features(api, rp, ci, n, a.omega)))


def cmd_predict(a, api):
    rp, ci, _, n, nc = read_matrix(a.input)
    if n != nc:
        raise InputError("the decider needs a square adjacency matrix")
    cfg = api.pspmm_decide_config(_features(api, rp, ci, n, a.omega), a.dim)
    print(json.dumps(cfg.as_dict()))


def cmd_spmm(a, api):
    import torch
    if is_pcsr(a.input):
        A = api.pspmm_pcsr_load(a.input)
        cfg = _config(api, a)
        if (cfg.V, cfg.S) != (A.V, A.S):
            raise InputError(f"the PCSR file has V={A.V}, S={A.S}; pass matching --v/--balance")
        n, nc = A.n_rows, A.n_cols
    else:
        rp, ci, val, n, nc = read_matrix(a.input)
        feats = _features(api, rp, ci, n, a.omega) if (a.auto and n == nc) else None
        cfg = _config(api, a, feats)
        d_rp, d_ci, d_val = _device_csr(rp, ci, val)
        A = api.pspmm_pcsr_build(n, int(rp[-1]), d_rp, d_ci, d_val, cfg.V, cfg.S, cfg.omega,
                                 cfg.sg_override, n_cols=nc)
        if feats is not None:  # the library's engine rules, in bench.py's order
            K = int(_B(a, nc).shape[1])
            cfg, _ = api.auto_dense(A, d_rp, d_ci, d_val, K, cfg)
            cfg, A, _ = api.auto_blocks(A, d_rp, d_ci, d_val, K, cfg)
            cfg, A, _ = api.auto_band(A, d_rp, d_ci, d_val, K, cfg, feats)
    B = torch.from_numpy(_B(a, nc)).cuda()
    C = torch.empty((n, B.shape[1]), device="cuda")
    api.pspmm_spmm_run(A, B, C, cfg)
    torch.cuda.synchronize()
    if a.out:
        np.save(a.out, C.cpu().numpy())
    print(json.dumps({"n": n, "dim": int(B.shape[1]), "config": cfg.as_dict(),
                      "out": a.out}))


def lattice(dim):
    """The bench lattice: V, S corners x W x the zero-waste (F, G) covers."""
    q = (dim + 3) // 4
    out = []
    for V in (1, 2):
        for S in (0, 1):
            for W in (2, 4, 8):
                for F in (1, 2, 4, 8):
                    G = 1
                    while G * F < q and G < 32:
                        G *= 2
                    if F > 1 and G * F > 2 * q:
                        continue
                    out.append((V, S, W, F, G))
    return out


def cmd_bench(a, api):
    import torch
    rp, ci, val, n, nc = read_matrix(a.input)
    nnz = int(rp[-1])
    d_rp, d_ci, d_val = _device_csr(rp, ci, val)
    dims = [int(x) for x in a.dims.split(",")]
    handles = {}
    rows = []
    for dim in dims:
        rng = np.random.default_rng(a.seed)
        B = torch.from_numpy((rng.random((nc, dim), dtype=np.float32) * 2 - 1)).cuda()
        C = torch.empty((n, dim), device="cuda")
        for V, S, W, F, G in lattice(dim):
            if (V, S) not in handles:
                handles[(V, S)] = api.pspmm_pcsr_build(n, nnz, d_rp, d_ci, d_val, V, S, a.omega,
                                                       0, n_cols=nc)
            cfg = api.Config(W=W, F=F, V=V, S=S, omega=a.omega, G=G)
            A = handles[(V, S)]
            A.run(B, C, cfg)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(a.repeats)]
            for e0, e1 in ev:
                e0.record()
                A.run(B, C, cfg)
                e1.record()
            torch.cuda.synchronize()
            ms = float(np.median([x.elapsed_time(y) for x, y in ev]))
            rows.append({"matrix": a.input, "dim": dim, "V": V, "S": S, "W": W, "F": F, "G": G,
                         "ms": ms, "gflops": 2.0 * nnz * dim / (ms * 1e-3) / 1e9})
    with (open(a.out, "w", newline="") if a.out else sys.stdout) as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0].keys()) if rows else ["matrix"])
        w.writeheader()
        w.writerows(rows)


# ---------------------------------------------------------------- parser
def build_parser():
    ap = argparse.ArgumentParser(prog="pspmm", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)

    def config_flags(p, dim=True):
        if dim:
            p.add_argument("--dim", type=int, required=True, help="K, columns of B")
        p.add_argument("--omega", type=int, default=32)
        p.add_argument("--v", type=int, default=1, choices=[1, 2],
                       help="panel height V (P:91: V in {1, 2})")
        p.add_argument("--balance", action="store_true", help="S = 1 (nnz chunks of SG)")
        p.add_argument("--sg", type=int, default=0, help="SG override (0 = Eq. 3)")

    p = sub.add_parser("convert", help="CSR (.mtx / .npz) -> PCSR file")
    p.add_argument("input")
    config_flags(p, dim=False)
    p.add_argument("--out", required=True)
    p = sub.add_parser("inspect", help="print a PCSR file's header / metrics")
    p.add_argument("input")
    p.add_argument("--arrays", action="store_true", help="also print the four arrays")
    p = sub.add_parser("features", help="Table-3 features of a matrix")
    p.add_argument("input")
    p.add_argument("--omega", type=int, default=32)
    p = sub.add_parser("predict", help="decider config for a matrix and dim")
    p.add_argument("input")
    p.add_argument("--dim", type=int, required=True)
    p.add_argument("--omega", type=int, default=32)
    p = sub.add_parser("spmm", help="C = A . B (decide -> build -> run), C saved as .npy")
    p.add_argument("input", help=".mtx / .npz CSR or a PCSR file")
    config_flags(p)
    p.add_argument("--auto", action="store_true", help="use the decider (P:337-341)")
    p.add_argument("--w", type=int, default=4)
    p.add_argument("--f", type=int, default=1)
    p.add_argument("--g", type=int, default=0)
    p.add_argument("--mode", type=int, default=0, choices=[0, 2, 3])
    p.add_argument("--order", type=int, default=0, choices=[0, 1])
    p.add_argument("--b", default="", help="B as .npy (n_cols x dim); default seeded U[-1,1)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", default="")
    p = sub.add_parser("bench", help="time the config lattice -> CSV (GFLOPS = 2 nnz dim / t)")
    p.add_argument("input")
    p.add_argument("--dims", default="16,32,64,128,256")
    p.add_argument("--omega", type=int, default=32)
    p.add_argument("--repeats", type=int, default=10)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", default="")
    return ap


COMMANDS = {"convert": cmd_convert, "inspect": cmd_inspect, "features": cmd_features,
            "predict": cmd_predict, "spmm": cmd_spmm, "bench": cmd_bench}


def main(argv=None) -> int:
    a = build_parser().parse_args(argv)
    if getattr(a, "dim", 1) is not None and getattr(a, "dim", 1) < 1:
        print("error: --dim must be >= 1", file=sys.stderr)
        return 2
    try:
        from . import api
        COMMANDS[a.cmd](a, api)
    except InputError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    except Exception as e:  # library errors (api.PspmmError) and CUDA failures
        if type(e).__name__ == "PspmmError":
            print(f"error: {e}", file=sys.stderr)
            return EXIT_LIB
        raise
    return 0


if __name__ == "__main__":
    sys.exit(main())
