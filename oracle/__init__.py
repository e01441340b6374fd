"""ORACLE — test infrastructure only (see oracle/oracle.c header).

Thin ctypes wrapper around ``oracle/liboracle.so`` (plain C, gcc-built).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with ``paper_2605_15695_b200`` and never imports it.

Functions (each cites the paper passage it follows, see oracle.c):
  spmm(rowptr, colidx, val, B, rows=None, threads=1) -> (C fp64, mag fp64)
  gap(dim, F, omega)                     Eq. 1, P:138-146 (+ c-1a)
  pcsr_build(rowptr, colidx, val, V, S, omega, sg_override=0) -> dict
  features(rowptr, colidx, val, omega)   Table 3, P:307-334 -> dict
  gnn_layer(rowptr, colidx, val, X, W)  H' = A H W -> (Y, mag)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

FEATURE_NAMES = ("n", "n_hat", "nnz", "delta", "d", "d_hat", "d_max", "cv",
                 "cv_hat", "sr1", "sr2", "rho", "b", "b_max", "pr1", "pr2")


def build(force: bool = False) -> str:
    """Compile oracle.c with plain gcc -O2 (no hand vectorisation)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class _Pcsr(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "n", "V", "S", "omega", "num_panels", "nnz", "nnz_v", "nonempty_panels",
        "sg", "num_chunks", "rowptr_len")] + [
        ("pr", ctypes.c_double), ("sr", ctypes.c_double),
        ("rowPtr", ctypes.POINTER(ctypes.c_int32)),
        ("colIdx", ctypes.POINTER(ctypes.c_int32)),
        ("TRow", ctypes.POINTER(ctypes.c_int32)),
        ("val", ctypes.POINTER(ctypes.c_float))]


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        _lib.oracle_spmm_rows.argtypes = [i64, P, P, P, P, i64, ctypes.c_int32, i64, P, P, P,
                                          ctypes.c_int32]
        _lib.oracle_spmm_rows.restype = ctypes.c_int
        _lib.oracle_gap.argtypes = [i64, i64, i64]
        _lib.oracle_gap.restype = i64
        _lib.oracle_pcsr_build.argtypes = [i64, P, P, P, i64, i64, i64, i64,
                                           ctypes.POINTER(_Pcsr)]
        _lib.oracle_pcsr_build.restype = ctypes.c_int
        _lib.oracle_pcsr_free.argtypes = [ctypes.POINTER(_Pcsr)]
        _lib.oracle_pcsr_free.restype = None
        _lib.oracle_features.argtypes = [i64, P, P, P, i64, P]
        _lib.oracle_features.restype = ctypes.c_int
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _csr(rowptr, colidx, val):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int32)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float32)
    return rowptr, colidx, val


def spmm(rowptr, colidx, val, B, rows=None, threads: int = 1, with_mag: bool = True):
    """c-1: fp64 C = A.B (Alg. 1) and mag = sum |a||b|.

    ``rows``: optional int64 array of matrix rows to compute (sampled checks
    at full size); output row r is matrix row rows[r].  ``with_mag=False``
    skips the tolerance bound (mag is returned as None): the plain product,
    as bench.py's cpu_baseline times it.
    """
    rowptr, colidx, val = _csr(rowptr, colidx, val)
    B = np.ascontiguousarray(B, dtype=np.float32)
    n = rowptr.shape[0] - 1
    K = B.shape[1]
    if rows is not None:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        cnt = rows.shape[0]
    else:
        cnt = n
    out = np.empty((cnt, K), dtype=np.float64)
    mag = np.empty((cnt, K), dtype=np.float64) if with_mag else None
    st = _L().oracle_spmm_rows(n, _ptr(rowptr), _ptr(colidx), _ptr(val), _ptr(B), K, K,
                               cnt, _ptr(rows), _ptr(out), _ptr(mag), int(threads))
    if st:
        raise OracleError(st, "spmm")
    return out, mag


def gap(dim: int, F: int, omega: int = 32) -> int:
    """Eq. 1 with c-1a."""
    return int(_L().oracle_gap(dim, F, omega))


def pcsr_build(rowptr, colidx, val, V: int, S: int, omega: int = 32, sg_override: int = 0):
    """c-2: PCSR generation (Eq. 2-4).  Returns a dict of numpy
    arrays (rowPtr, colIdx, val, TRow) and metrics."""
    rowptr, colidx, val = _csr(rowptr, colidx, val)
    n = rowptr.shape[0] - 1
    p = _Pcsr()
    st = _L().oracle_pcsr_build(n, _ptr(rowptr), _ptr(colidx), _ptr(val), V, S, omega,
                                sg_override, ctypes.byref(p))
    if st:
        raise OracleError(st, "pcsr_build")
    try:
        nv = p.nnz_v
        out = {
            "n": p.n, "V": p.V, "S": p.S, "omega": p.omega,
            "num_panels": p.num_panels, "nnz": p.nnz, "nnz_v": nv,
            "nonempty_panels": p.nonempty_panels, "sg": p.sg,
            "num_chunks": p.num_chunks, "pr": p.pr, "sr": p.sr,
            "rowPtr": np.ctypeslib.as_array(p.rowPtr, shape=(p.rowptr_len,)).copy(),
            "colIdx": (np.ctypeslib.as_array(p.colIdx, shape=(nv,)).copy() if nv
                       else np.zeros(0, np.int32)),
            "val": (np.ctypeslib.as_array(p.val, shape=(nv * p.V,)).copy() if nv
                    else np.zeros(0, np.float32)),
            "TRow": (np.ctypeslib.as_array(p.TRow, shape=(p.num_chunks,)).copy()
                     if p.S else np.zeros(0, np.int32)),
        }
    finally:
        _L().oracle_pcsr_free(ctypes.byref(p))
    return out


def features(rowptr, colidx, val, omega: int = 32):
    """c-3: Table 3 features."""
    rowptr, colidx, val = _csr(rowptr, colidx, val)
    n = rowptr.shape[0] - 1
    f = np.empty(16, dtype=np.float64)
    st = _L().oracle_features(n, _ptr(rowptr), _ptr(colidx), _ptr(val), omega, _ptr(f))
    if st:
        raise OracleError(st, "features")
    return dict(zip(FEATURE_NAMES, f.tolist()))


def gnn_layer(rowptr, colidx, val, X, W):
    """f3: one GCN/GIN-style layer H' = A . H . W (where
    SpMM is the aggregation of a GNN layer; P:449-460 trains GCN and GIN).
    Plain fp64: T = H . W (numpy matmul), then Y = A . T over the CSR (the
    definition of P:48 with fp64 values, scipy's CSR product as the library
    primitive).  mag = |A| . (|H| . |W|) bounds every product term for the
    c-1 style tolerance.  Test infrastructure only."""
    import scipy.sparse as sp
    rowptr, colidx, val = _csr(rowptr, colidx, val)
    n = rowptr.shape[0] - 1
    X = np.asarray(X, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    A = sp.csr_matrix((val.astype(np.float64), colidx, rowptr), shape=(n, X.shape[0]))
    Y = A @ (X @ W)
    mag = abs(A) @ (np.abs(X) @ np.abs(W))
    return np.asarray(Y), np.asarray(mag)
