"""Thin Python binding of libpspmm.so (include/pspmm.h) — argument
marshalling only: every step of the hot path runs in the library's CUDA
kernels.  Device arrays are torch CUDA tensors (PyTorch is used for device
memory and streams only); host arrays are numpy.  If the native library is
missing this module raises at import time — there is no fallback.

The functions carry the C names (pspmm_pcsr_build, pspmm_spmm_run, ...);
`Pcsr` and `spmm` are small conveniences on top of them.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpspmm.so")
# tools/variants.py experiments may point at another build of the same sources
LIB_PATH = os.environ.get("PSPMM_LIB", LIB_PATH)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -m paper_2605_15695_b200.build_ext` "
        "(the CUDA library is the only implementation — there is no fallback)")

_lib = ctypes.CDLL(LIB_PATH)

STATUS = ("PSPMM_OK", "PSPMM_ERR_INVALID_ARG", "PSPMM_ERR_NOT_CANONICAL",
          "PSPMM_ERR_DIM_MISMATCH", "PSPMM_ERR_CONFIG", "PSPMM_ERR_CONFIG_MISMATCH",
          "PSPMM_ERR_EMPTY", "PSPMM_ERR_UNSUPPORTED", "PSPMM_ERR_OOM", "PSPMM_ERR_CUDA")
for _i, _name in enumerate(STATUS):
    globals()[_name] = _i


class PspmmError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.pspmm_last_error().decode()
        name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{where}: {name}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    """pspmm_config: <W, F, V, S> + omega, sg_override, G, mode."""
    _fields_ = [(n, ctypes.c_int32) for n in ("W", "F", "V", "S", "omega", "sg_override", "G",
                                              "mode", "order")]

    def __init__(self, W=4, F=1, V=1, S=0, omega=32, sg_override=0, G=0, mode=0, order=0):
        super().__init__(W, F, V, S, omega, sg_override, G, mode, order)

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}

    def __repr__(self):
        return "Config(" + ", ".join(f"{k}={v}" for k, v in self.as_dict().items()) + ")"


FEATURE_NAMES = ("n", "n_hat", "nnz", "delta", "d", "d_hat", "d_max", "cv", "cv_hat", "sr1",
                 "sr2", "rho", "b", "b_max", "pr1", "pr2")


class Features(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in FEATURE_NAMES]

    def as_dict(self):
        return {n: getattr(self, n) for n in FEATURE_NAMES}


class PcsrInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("n", "num_panels", "nnz", "nnz_v", "num_chunks",
                                              "sg")] + \
        [(n, ctypes.c_int32) for n in ("V", "S", "omega", "reserved")] + \
        [("pr", ctypes.c_double), ("sr", ctypes.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "reserved"}


_P = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_st = ctypes.c_int


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("pspmm_status_string", ctypes.c_char_p, _st)
_sig("pspmm_last_error", ctypes.c_char_p)
_sig("pspmm_version", ctypes.c_char_p)
_sig("pspmm_csr_validate", _st, _i64, _i64, _P, _P, _P)
_sig("pspmm_csr_validate_rect", _st, _i64, _i64, _i64, _P, _P, _P)
_sig("pspmm_pcsr_build", _st, _i64, _i64, _P, _P, _P, _i32, _i32, _i32, _i32, _P,
     ctypes.POINTER(_P))
_sig("pspmm_pcsr_build_rect", _st, _i64, _i64, _i64, _P, _P, _P, _i32, _i32, _i32, _i32, _P,
     ctypes.POINTER(_P))
_sig("pspmm_pcsr_get_info", _st, _P, ctypes.POINTER(PcsrInfo))
_sig("pspmm_pcsr_export", _st, _P, _P, _P, _P, _P)
_sig("pspmm_pcsr_destroy", None, _P)
_sig("pspmm_pcsr_save", _st, _P, ctypes.c_char_p)
_sig("pspmm_pcsr_load", _st, ctypes.c_char_p, _P, ctypes.POINTER(_P))
_sig("pspmm_spmm_run", _st, _P, _P, _i64, _i32, _P, _i64, Config, _P)
_sig("pspmm_spmm_run_host", _st, _P, _P, _i64, _i32, _P, _i64, Config, _P, _P, _P)
_sig("pspmm_spmm_accumulate", _st, _P, _P, _i64, _i32, _P, _i64, Config, _P)
_sig("pspmm_pcsr_attach_dense", _st, _P, _P, _P, _P, ctypes.c_double, _i32, _P,
     ctypes.POINTER(_i64))
_sig("pspmm_decide_dense", _st, _P, _i32, ctypes.c_double, ctypes.POINTER(Config))
_sig("pspmm_block_reuse", _st, _P, _P, ctypes.POINTER(ctypes.c_double))
_sig("pspmm_pcsr_attach_blocks", _st, _P, _P, ctypes.POINTER(_i64))
_sig("pspmm_decide_blocks", _st, _P, _i32, ctypes.c_double, ctypes.POINTER(Config))
_sig("pspmm_block_info", _st, _P, ctypes.POINTER(_i32), ctypes.POINTER(_i64))
_sig("pspmm_pcsr_attach_band", _st, _P, _i32, _P, ctypes.POINTER(ctypes.c_double))
_sig("pspmm_pcsr_dense_info", _st, _P, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
     ctypes.POINTER(_i64))
_sig("pspmm_spmm_run_host_batch", _st, _P, _P, _i64, _i32, _P, _i64, _i32, Config, _P, _P, _P)
_sig("pspmm_dense_gemm", _st, _i64, _i32, _i32, _P, _i64, _P, _i64, _P, _i64, _P)
_sig("pspmm_gnn_layer", _st, _P, _P, _i64, _i32, _P, _i64, _i32, _P, _i64, _P, _i64, Config, _P)
_sig("pspmm_spmm_run_fanout", _st, _P, _P, _i64, _i32, _P, _i64, _P, _i32, Config, _P)
_sig("pspmm_spmm_run_multicast", _st, _P, _P, _i64, _i32, _P, _i64, _P, Config, _P)
_sig("pspmm_ipc_get_handle", _st, _P, _P, ctypes.POINTER(_i64))
_sig("pspmm_ipc_open", _st, _P, ctypes.POINTER(_P))
_sig("pspmm_ipc_close", _st, _P)
_sig("pspmm_features_compute", _st, _i64, _i64, _P, _P, _i32, _P, ctypes.POINTER(Features))
_sig("pspmm_csr_transpose", _st, _i64, _i64, _i64, _P, _P, _P, _P, _P, _P, _P)
_sig("pspmm_reorder", _st, _i64, _P, _P, _i32, _P)
_sig("pspmm_csr_permute", _st, _i64, _i64, _P, _P, _P, _P, _P, _P, _P, _P)
_sig("pspmm_permute_rows", _st, _i64, _i32, _P, _i64, _P, _P, _i64, _i32, _P)
_sig("pspmm_decide_config", _st, ctypes.POINTER(Features), _i32, ctypes.POINTER(Config))
_sig("pspmm_shard_plan", _st, _i64, _P, _i32, _i32, _P)
_sig("pspmm_shard_extract", _st, _i64, _P, _P, _P, _i32, _P, _i32, _P, _P, _P,
     ctypes.POINTER(_i64))


def _check(status, where):
    if status != 0:
        raise PspmmError(status, where)


def version() -> str:
    return _lib.pspmm_version().decode()


# ---------------------------------------------------------------- marshalling
def _torch():
    import torch
    return torch


def _dev(t, dtype, what):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{what} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _dense(t, what):
    """Row-major fp32 CUDA matrix with unit column stride -> (ptr, ld)."""
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise TypeError(f"{what} must be a float32 CUDA tensor")
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{what} must be 2-D row-major (stride(1) == 1)")
    return ctypes.c_void_p(t.data_ptr()), max(t.stride(0), t.shape[1])


def _stream(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _host(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- ABI calls
def pspmm_csr_validate(n, nnz, rowptr, colidx, stream=None, n_cols=None):
    st = _lib.pspmm_csr_validate_rect(n, n if n_cols is None else n_cols, nnz,
                                      _dev(rowptr, _torch().int32, "rowptr"),
                                      _dev(colidx, _torch().int32, "colidx"), _stream(stream))
    _check(st, "pspmm_csr_validate")


class Pcsr:
    """Owner of a pspmm_pcsr handle (destroyed with the object)."""

    def __init__(self, handle, n_rows, n_cols):
        self.handle = handle
        self.n_rows = n_rows
        self.n_cols = n_cols
        self.info = pspmm_pcsr_get_info(self)

    @property
    def V(self):
        return self.info["V"]

    @property
    def S(self):
        return self.info["S"]

    def run(self, B, C, cfg: Config, stream=None):
        pspmm_spmm_run(self, B, C, cfg, stream)
        return C

    def export(self):
        return pspmm_pcsr_export(self)

    def close(self):
        if self.handle is not None:
            _lib.pspmm_pcsr_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pspmm_pcsr_build(n, nnz, rowptr, colidx, val, V, S, omega=32, sg_override=0, stream=None,
                     n_cols=None) -> Pcsr:
    torch = _torch()
    h = ctypes.c_void_p()
    nc = n if n_cols is None else n_cols
    st = _lib.pspmm_pcsr_build_rect(n, nc, nnz, _dev(rowptr, torch.int32, "rowptr"),
                                    _dev(colidx, torch.int32, "colidx"),
                                    _dev(val, torch.float32, "val"), V, S, omega, sg_override,
                                    _stream(stream), ctypes.byref(h))
    _check(st, "pspmm_pcsr_build")
    return Pcsr(h, n, nc)


def pspmm_pcsr_get_info(A: Pcsr) -> dict:
    info = PcsrInfo()
    _check(_lib.pspmm_pcsr_get_info(A.handle, ctypes.byref(info)), "pspmm_pcsr_get_info")
    return info.as_dict()


def pspmm_pcsr_export(A: Pcsr) -> dict:
    i = A.info
    rl = (i["num_chunks"] if i["S"] else i["num_panels"]) + 1
    rowptr = np.empty(rl, np.int32)
    colidx = np.empty(i["nnz_v"], np.int32)
    val = np.empty(i["nnz_v"] * i["V"], np.float32)
    trow = np.empty(i["num_chunks"] if i["S"] else 0, np.int32)
    st = _lib.pspmm_pcsr_export(A.handle, rowptr.ctypes.data_as(_P), colidx.ctypes.data_as(_P),
                                val.ctypes.data_as(_P), trow.ctypes.data_as(_P) if i["S"] else None)
    _check(st, "pspmm_pcsr_export")
    return {"rowPtr": rowptr, "colIdx": colidx, "val": val, "TRow": trow, **i}


def pspmm_pcsr_save(A: Pcsr, path):
    """Write the PCSR binary file (include/pspmm.h)."""
    _check(_lib.pspmm_pcsr_save(A.handle, os.fsencode(path)), "pspmm_pcsr_save")


def pspmm_pcsr_load(path, stream=None) -> Pcsr:
    """Read and validate a PCSR file into a device handle."""
    h = ctypes.c_void_p()
    _check(_lib.pspmm_pcsr_load(os.fsencode(path), _stream(stream), ctypes.byref(h)),
           "pspmm_pcsr_load")
    info = PcsrInfo()
    _check(_lib.pspmm_pcsr_get_info(h, ctypes.byref(info)), "pspmm_pcsr_get_info")
    # rows / columns: the handle knows both; n_cols is not in pcsr_info
    return Pcsr(h, int(info.n), _load_ncols(path))


def _load_ncols(path) -> int:
    with open(path, "rb") as f:
        head = f.read(72)
    return int(np.frombuffer(head[64:72], "<u8")[0])


def pspmm_pcsr_destroy(A: Pcsr):
    A.close()


def pspmm_spmm_run(A: Pcsr, B, C, cfg: Config, stream=None, K=None):
    b, ldb = _dense(B, "B")
    c, ldc = _dense(C, "C")
    K = B.shape[1] if K is None else K
    if C.shape[1] < K or B.shape[0] < A.n_cols or C.shape[0] < A.n_rows:
        raise ValueError("B / C shapes do not match the PCSR handle and K")
    _check(_lib.pspmm_spmm_run(A.handle, b, ldb, K, c, ldc, cfg, _stream(stream)),
           "pspmm_spmm_run")


def pspmm_spmm_accumulate(A: Pcsr, B, C, cfg: Config, stream=None, K=None):
    """C += A . B."""
    b, ldb = _dense(B, "B")
    c, ldc = _dense(C, "C")
    K = B.shape[1] if K is None else K
    if C.shape[1] < K or B.shape[0] < A.n_cols or C.shape[0] < A.n_rows:
        raise ValueError("B / C shapes do not match the PCSR handle and K")
    _check(_lib.pspmm_spmm_accumulate(A.handle, b, ldb, K, c, ldc, cfg, _stream(stream)),
           "pspmm_spmm_accumulate")


def pspmm_pcsr_attach_dense(A: Pcsr, rowptr, colidx, val, min_density, k_max=256,
                            stream=None) -> dict:
    """Split A for engine mode 1: dense 128 x 32 tiles (>= min_density full)
    on the tensor cores, the rest on the mode-0 engine.  (rowptr, colidx,
    val) = the device CSR A was built from.  Returns pspmm_pcsr_dense_info."""
    torch = _torch()
    nt = _i64()
    st = _lib.pspmm_pcsr_attach_dense(A.handle, _dev(rowptr, torch.int32, "rowptr"),
                                      _dev(colidx, torch.int32, "colidx"),
                                      _dev(val, torch.float32, "val"), float(min_density),
                                      int(k_max), _stream(stream), ctypes.byref(nt))
    _check(st, "pspmm_pcsr_attach_dense")
    return pspmm_pcsr_dense_info(A)


def pspmm_decide_dense(A: Pcsr, K: int, min_frac: float, cfg: Config) -> Config:
    """Mode-1 rule of the C library (include/pspmm.h); returns a new Config."""
    out = Config(**cfg.as_dict())
    _check(_lib.pspmm_decide_dense(A.handle, K, float(min_frac), ctypes.byref(out)),
           "pspmm_decide_dense")
    return out


def pspmm_block_reuse(A: Pcsr, stream=None) -> float:
    """Engine mode 5: nonzeros per staged B row (device-computed, V1 S0 handle)."""
    r = ctypes.c_double()
    _check(_lib.pspmm_block_reuse(A.handle, _stream(stream), ctypes.byref(r)), "pspmm_block_reuse")
    return r.value


def pspmm_pcsr_attach_blocks(A: Pcsr, stream=None) -> int:
    """Build the mode-5 pack (row blocks of 15 x rw rows, windows of 128 B
    rows); returns the number of touched (block, window) pairs."""
    w = _i64()
    _check(_lib.pspmm_pcsr_attach_blocks(A.handle, _stream(stream), ctypes.byref(w)),
           "pspmm_pcsr_attach_blocks")
    return w.value


def pspmm_block_info(A: Pcsr) -> tuple:
    """(rows per block, touched windows) of the attached mode-5 pack."""
    r, w = _i32(), _i64()
    _check(_lib.pspmm_block_info(A.handle, ctypes.byref(r), ctypes.byref(w)), "pspmm_block_info")
    return r.value, w.value


def pspmm_pcsr_attach_band(A: Pcsr, k_max: int, stream=None) -> float:
    """Build the mode-6 pack (staged bands of 128-row blocks; K, ldb <= k_max);
    returns the fraction of non-empty blocks whose band is staged."""
    f = ctypes.c_double()
    _check(_lib.pspmm_pcsr_attach_band(A.handle, int(k_max), _stream(stream), ctypes.byref(f)),
           "pspmm_pcsr_attach_band")
    return f.value


def pspmm_decide_blocks(A: Pcsr, K: int, min_reuse: float, cfg: Config) -> Config:
    """Mode-5 rule of the C library (include/pspmm.h); returns a new Config."""
    out = Config(**cfg.as_dict())
    _check(_lib.pspmm_decide_blocks(A.handle, K, float(min_reuse), ctypes.byref(out)),
           "pspmm_decide_blocks")
    return out


def pspmm_pcsr_dense_info(A: Pcsr) -> dict:
    p, t, z = _i64(), _i64(), _i64()
    _check(_lib.pspmm_pcsr_dense_info(A.handle, ctypes.byref(p), ctypes.byref(t), ctypes.byref(z)),
           "pspmm_pcsr_dense_info")
    return {"num_panels": p.value, "num_tiles": t.value, "nnz_dense": z.value}


def pspmm_spmm_run_host_batch(A: Pcsr, hBs, hCs, cfg: Config, dBs, dCs, stream=None):
    """C_i = A . B_i for pinned host tensors hBs[i] -> hCs[i] (same shapes),
    two device buffer sets dBs[0..1] / dCs[0..1] rotating so copies overlap
    the engine.  Synchronous."""
    torch = _torch()
    if len(hBs) != len(hCs) or len(dBs) != 2 or len(dCs) != 2:
        raise ValueError("need as many outputs as inputs and two device buffer sets")
    K = None
    hb, hc = [], []
    for b, c in zip(hBs, hCs):
        for t in (b, c):
            if not (isinstance(t, torch.Tensor) and t.device.type == "cpu" and
                    t.dtype == torch.float32 and t.is_contiguous()):
                raise TypeError("host matrices must be contiguous float32 CPU tensors")
        if K is None:
            K = b.shape[1]
        if b.shape[1] != K or c.shape[1] != K:
            raise ValueError("every B_i / C_i must have K columns")
        hb.append(b.data_ptr())
        hc.append(c.data_ptr())
    db = [_dense(t, "dB") for t in dBs]
    dc = [_dense(t, "dC") for t in dCs]
    if K is None:
        return
    if db[0][1] != db[1][1] or dc[0][1] != dc[1][1] or db[0][1] != K or dc[0][1] != K:
        raise ValueError("device buffers must be contiguous n x K like the host matrices")
    n = len(hb)
    HB = (ctypes.c_void_p * n)(*hb)
    HC = (ctypes.c_void_p * n)(*hc)
    DB = (ctypes.c_void_p * 2)(db[0][0].value, db[1][0].value)
    DC = (ctypes.c_void_p * 2)(dc[0][0].value, dc[1][0].value)
    _check(_lib.pspmm_spmm_run_host_batch(A.handle, HB, K, K, HC, K, n, cfg, DB, DC,
                                          _stream(stream)), "pspmm_spmm_run_host_batch")


def pspmm_dense_gemm(X, W, T, stream=None):
    """T = X . W (fp32, device)."""
    x, ldx = _dense(X, "X")
    w, ldw = _dense(W, "W")
    t, ldt = _dense(T, "T")
    n, Ki = X.shape
    Ko = W.shape[1]
    if W.shape[0] != Ki or T.shape[0] < n or T.shape[1] < Ko:
        raise ValueError("X (n x Ki), W (Ki x Ko), T (n x Ko) shapes do not match")
    _check(_lib.pspmm_dense_gemm(n, Ki, Ko, x, ldx, w, ldw, t, ldt, _stream(stream)),
           "pspmm_dense_gemm")


def pspmm_gnn_layer(A: Pcsr, X, W, T, Y, cfg: Config, stream=None):
    """Y = A . X . W (the SpMM on min(Ki, Ko) columns; T: n x min(Ki, Ko))."""
    x, ldx = _dense(X, "X")
    w, ldw = _dense(W, "W")
    t, ldt = _dense(T, "T")
    y, ldy = _dense(Y, "Y")
    Ki, Ko = W.shape
    if X.shape[1] != Ki or X.shape[0] < A.n_cols or Y.shape[0] < A.n_rows or Y.shape[1] < Ko:
        raise ValueError("X (n x Ki), W (Ki x Ko), Y (n x Ko) shapes do not match A")
    if T.shape[1] < min(Ki, Ko) or T.shape[0] < max(A.n_rows, A.n_cols):
        raise ValueError("T must be n x min(Ki, Ko)")
    _check(_lib.pspmm_gnn_layer(A.handle, x, ldx, Ki, w, ldw, Ko, t, ldt, y, ldy, cfg,
                                _stream(stream)), "pspmm_gnn_layer")


MAX_PEERS = 7  # PSPMM_MAX_PEERS


def pspmm_spmm_run_multicast(A: Pcsr, B, C, c_mc: int, cfg: Config, stream=None):
    """C = A . B with every C write issued once as a multimem store to c_mc,
    the multicast address (int) of C's first element (f2 i over NVLS)."""
    b, ldb = _dense(B, "B")
    c, ldc = _dense(C, "C")
    K = B.shape[1]
    if B.shape[0] < A.n_cols or C.shape[0] < A.n_rows or C.shape[1] < K:
        raise ValueError("B (n_cols x K) / C (n_rows x K) shapes do not match A")
    _check(_lib.pspmm_spmm_run_multicast(A.handle, b, ldb, K, c, ldc, ctypes.c_void_p(int(c_mc)),
                                         cfg, _stream(stream)), "pspmm_spmm_run_multicast")


def pspmm_spmm_run_fanout(A: Pcsr, B, C, peers, cfg: Config, stream=None, K=None):
    """C = A . B with every written C element also stored at the same offset
    of each peer buffer (f2).  peers: device addresses (int, e.g. from
    pspmm_ipc_open plus an offset) or CUDA tensors laid out like C."""
    b, ldb = _dense(B, "B")
    c, ldc = _dense(C, "C")
    K = B.shape[1] if K is None else K
    if C.shape[1] < K or B.shape[0] < A.n_cols or C.shape[0] < A.n_rows:
        raise ValueError("B / C shapes do not match the PCSR handle and K")
    torch = _torch()
    addrs = []
    for p in peers:
        if isinstance(p, torch.Tensor):
            q, ld = _dense(p, "peer")
            if ld != ldc or p.shape[0] < A.n_rows:
                raise ValueError("a peer tensor must be laid out like C")
            addrs.append(q.value)
        else:
            addrs.append(int(p))
    if len(addrs) > MAX_PEERS:
        raise ValueError(f"at most {MAX_PEERS} peers")
    arr = (ctypes.c_void_p * max(1, len(addrs)))(*addrs)
    _check(_lib.pspmm_spmm_run_fanout(A.handle, b, ldb, K, c, ldc, arr, len(addrs), cfg,
                                      _stream(stream)), "pspmm_spmm_run_fanout")


def pspmm_ipc_get_handle(t) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding tensor t, byte
    offset of t inside it)."""
    buf = ctypes.create_string_buffer(64)
    off = _i64()
    _check(_lib.pspmm_ipc_get_handle(ctypes.c_void_p(t.data_ptr()), buf, ctypes.byref(off)),
           "pspmm_ipc_get_handle")
    return buf.raw, off.value


def pspmm_ipc_open(handle: bytes) -> int:
    """Map a peer process's allocation; returns its base device address."""
    if len(handle) != 64:
        raise ValueError("an IPC handle is 64 bytes")
    p = _P()
    _check(_lib.pspmm_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(p)),
           "pspmm_ipc_open")
    return p.value


def pspmm_ipc_close(base: int):
    _check(_lib.pspmm_ipc_close(ctypes.c_void_p(base)), "pspmm_ipc_close")


def pspmm_spmm_run_host(A: Pcsr, hB, hC, cfg: Config, dB, dC, stream=None):
    """hB / hC: pinned host torch tensors (or numpy) n x K fp32; dB / dC: device staging."""
    torch = _torch()

    def hptr(t):
        if isinstance(t, torch.Tensor):
            assert t.device.type == "cpu" and t.dtype == torch.float32 and t.is_contiguous()
            return ctypes.c_void_p(t.data_ptr()), t.shape[1]
        assert t.dtype == np.float32 and t.flags.c_contiguous
        return t.ctypes.data_as(_P), t.shape[1]

    hb, K = hptr(hB)
    hc, Kc = hptr(hC)
    # the C side copies n_cols x ldb floats from hB and n_rows x ldc into hC:
    # host and device shapes must agree exactly (no padded staging buffers)
    if tuple(hB.shape) != (A.n_cols, K) or hC.shape[0] < A.n_rows or Kc != K:
        raise ValueError(f"run_host: need hB ({A.n_cols}, K) and hC (>= {A.n_rows}, K); got "
                         f"{tuple(hB.shape)} / {tuple(hC.shape)}")
    for t, name, rows in ((dB, "dB", A.n_cols), (dC, "dC", A.n_rows)):
        if not (t.is_contiguous() and t.dim() == 2 and t.shape[1] == K and t.shape[0] >= rows):
            raise ValueError(f"run_host: {name} must be contiguous (>= {rows}, {K})")
    db, ldb = _dense(dB, "dB")
    dc, ldc = _dense(dC, "dC")
    _check(_lib.pspmm_spmm_run_host(A.handle, hb, ldb, K, hc, ldc, cfg, db, dc, _stream(stream)),
           "pspmm_spmm_run_host")


def pspmm_features_compute(n, nnz, rowptr, colidx, omega=32, stream=None) -> dict:
    torch = _torch()
    f = Features()
    st = _lib.pspmm_features_compute(n, nnz, _dev(rowptr, torch.int32, "rowptr"),
                                     _dev(colidx, torch.int32, "colidx"), omega, _stream(stream),
                                     ctypes.byref(f))
    _check(st, "pspmm_features_compute")
    return f.as_dict()


def pspmm_csr_transpose(n_rows, n_cols, rowptr, colidx, val, stream=None):
    """CSR of A^T (device tensors in, new device tensors out)."""
    torch = _torch()
    nnz = int(rowptr[-1].item())
    t_rp = torch.empty(n_cols + 1, dtype=torch.int32, device=rowptr.device)
    t_ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=rowptr.device)
    t_vl = torch.empty(max(nnz, 1), dtype=torch.float32, device=rowptr.device)
    st = _lib.pspmm_csr_transpose(n_rows, n_cols, nnz, _dev(rowptr, torch.int32, "rowptr"),
                                  _dev(colidx, torch.int32, "colidx"),
                                  _dev(val, torch.float32, "val"), _dev(t_rp, torch.int32, "t"),
                                  _dev(t_ci, torch.int32, "t"), _dev(t_vl, torch.float32, "t"),
                                  _stream(stream))
    _check(st, "pspmm_csr_transpose")
    return t_rp, t_ci[:nnz], t_vl[:nnz]


REORDER = {"identity": 0, "bfs": 1, "degree": 2}


def pspmm_reorder(rowptr, colidx, strategy="bfs") -> np.ndarray:
    """perm[old] = new (host numpy int32) — P:271-272 reordering stand-in."""
    rp, prp = _host(rowptr, np.int32)
    ci, pci = _host(colidx, np.int32)
    n = rp.shape[0] - 1
    perm = np.empty(n, np.int32)
    st = _lib.pspmm_reorder(n, prp, pci, REORDER.get(strategy, strategy),
                            perm.ctypes.data_as(_P))
    _check(st, "pspmm_reorder")
    return perm


def pspmm_csr_permute(rowptr, colidx, val, perm, stream=None):
    """A' = P A P^T on the device (torch tensors in and out)."""
    torch = _torch()
    n = rowptr.shape[0] - 1
    nnz = int(rowptr[-1].item())
    o_rp = torch.empty(n + 1, dtype=torch.int32, device=rowptr.device)
    o_ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=rowptr.device)
    o_vl = torch.empty(max(nnz, 1), dtype=torch.float32, device=rowptr.device)
    st = _lib.pspmm_csr_permute(n, nnz, _dev(rowptr, torch.int32, "rowptr"),
                                _dev(colidx, torch.int32, "colidx"),
                                _dev(val, torch.float32, "val"), _dev(perm, torch.int32, "perm"),
                                _dev(o_rp, torch.int32, "o"), _dev(o_ci, torch.int32, "o"),
                                _dev(o_vl, torch.float32, "o"), _stream(stream))
    _check(st, "pspmm_csr_permute")
    return o_rp, o_ci[:nnz], o_vl[:nnz]


def pspmm_permute_rows(X, perm, inverse=False, out=None, stream=None):
    """inverse=False: out[perm[i]] = X[i]; inverse=True: out[i] = X[perm[i]]
    (a row gather; len(perm) may be smaller than X's row count), i < len(perm)."""
    torch = _torch()
    x, ldi = _dense(X, "X")
    m = perm.shape[0]
    if out is None:
        out = torch.empty((m if inverse else X.shape[0], X.shape[1]), dtype=X.dtype,
                          device=X.device)
    o, ldo = _dense(out, "out")
    if (not inverse and m > X.shape[0]) or (inverse and m > out.shape[0]):
        raise ValueError("perm longer than the matrix it indexes")
    st = _lib.pspmm_permute_rows(m, X.shape[1], x, ldi, _dev(perm, torch.int32, "perm"),
                                 o, ldo, 1 if inverse else 0, _stream(stream))
    _check(st, "pspmm_permute_rows")
    return out


def pspmm_decide_config(features: dict, K: int) -> Config:
    f = Features(*[float(features[k]) for k in FEATURE_NAMES])
    c = Config()
    _check(_lib.pspmm_decide_config(ctypes.byref(f), K, ctypes.byref(c)), "pspmm_decide_config")
    return c


def pspmm_shard_plan(rowptr, P: int, align: int = 1) -> np.ndarray:
    rp, p = _host(rowptr, np.int32)
    bounds = np.zeros(P + 1, np.int64)
    _check(_lib.pspmm_shard_plan(rp.shape[0] - 1, p, P, align, bounds.ctypes.data_as(_P)),
           "pspmm_shard_plan")
    return bounds


def pspmm_shard_extract(rowptr, colidx, val, P: int, bounds, r: int):
    rp, prp = _host(rowptr, np.int32)
    ci, pci = _host(colidx, np.int32)
    vl, pvl = _host(val, np.float32)
    bd, pbd = _host(bounds, np.int64)
    n = rp.shape[0] - 1
    lo, hi = int(bd[r]), int(bd[r + 1])
    cnt = int(rp[hi]) - int(rp[lo])
    lrp = np.empty(hi - lo + 1, np.int32)
    lci = np.empty(max(cnt, 1), np.int32)
    lvl = np.empty(max(cnt, 1), np.float32)
    nmax = ctypes.c_int64()
    st = _lib.pspmm_shard_extract(n, prp, pci, pvl, P, pbd, r, lrp.ctypes.data_as(_P),
                                  lci.ctypes.data_as(_P), lvl.ctypes.data_as(_P),
                                  ctypes.byref(nmax))
    _check(st, "pspmm_shard_extract")
    return lrp, lci[:cnt], lvl[:cnt], int(nmax.value)


# ---------------------------------------------------------------- convenience
def auto_config(n, nnz, rowptr, colidx, K, stream=None) -> Config:
    """Phase 1 of P:192: Table-3 features on the device, then the decider."""
    f = pspmm_features_compute(n, nnz, rowptr, colidx, stream=stream)
    return pspmm_decide_config(f, K)


# engine mode 1 rule: 128 x 32 tiles with >= 10 % nonzeros go
# to the tensor cores when they hold >= 5 % of A's nonzeros
DENSE_MIN_DENSITY = 0.1
DENSE_MIN_FRAC = 0.05


def auto_dense(A: Pcsr, rowptr, colidx, val, K, cfg: Config, stream=None):
    """Attach the dense-tile split (K % 16 == 0) and apply the library's
    mode-1 rule; returns (cfg, split info or None)."""
    if K % 16 != 0:
        return cfg, None
    info = pspmm_pcsr_attach_dense(A, rowptr, colidx, val, DENSE_MIN_DENSITY, k_max=K,
                                   stream=stream)
    cfg = pspmm_decide_dense(A, K, DENSE_MIN_FRAC, cfg)
    info.update(min_density=DENSE_MIN_DENSITY, min_frac=DENSE_MIN_FRAC, taken=cfg.mode == 1)
    return cfg, info


BLOCK_MIN_REUSE = 2.0


def auto_blocks(A: Pcsr, rowptr, colidx, val, K, cfg: Config, stream=None):
    """Engine mode 5 when the row blocks' staged B rows would be reused
    enough (K % 128 == 0): returns (cfg, handle to run, info or None).  The
    reuse is measured on a V = 1, S = 0 handle (A itself when it is one)."""
    if K % 128 != 0 or cfg.mode == 1:
        return cfg, A, None
    H = A
    if not (A.V == 1 and A.info["S"] == 0):
        H = pspmm_pcsr_build(A.n_rows, int(colidx.shape[0]), rowptr, colidx, val, 1, 0,
                             stream=stream, n_cols=A.n_cols)
    reuse = pspmm_block_reuse(H, stream)
    info = {"reuse": reuse, "min_reuse": BLOCK_MIN_REUSE, "taken": False}
    if reuse < BLOCK_MIN_REUSE:
        return cfg, A, info
    info["windows"] = pspmm_pcsr_attach_blocks(H, stream)
    c = Config(**cfg.as_dict())
    c.V, c.S = 1, 0
    c = pspmm_decide_blocks(H, K, BLOCK_MIN_REUSE, c)
    info["taken"] = c.mode == 5
    return (c, H, info) if c.mode == 5 else (cfg, A, info)


# engine mode 6 rule: locality-ordered graphs (mean row
# bandwidth below n / BAND_MAX_B_FRAC) whose 128-row blocks' bands fit the
# shared-memory budget for >= BAND_MIN_STAGED of the blocks
BAND_MAX_B_FRAC = 64.0
BAND_MIN_STAGED = 0.9


def auto_band(A: Pcsr, rowptr, colidx, val, K, cfg: Config, features=None, stream=None):
    """Engine mode 6 (staged bands) for locality-ordered graphs, K % 4 == 0,
    K <= 128, when the decider's pick is a CUDA-core gather engine: returns
    (cfg, handle to run, info or None)."""
    if K % 4 != 0 or K > 128 or cfg.mode in (1, 5):
        return cfg, A, None
    f = features if features is not None else pspmm_features_compute(
        A.n_rows, int(colidx.shape[0]), rowptr, colidx, stream=stream)
    b = f["b"] if isinstance(f, dict) else f.b
    info = {"b": b, "max_b": A.n_rows / BAND_MAX_B_FRAC, "taken": False}
    if not b < A.n_rows / BAND_MAX_B_FRAC:
        return cfg, A, info
    H = A
    if not (A.V == 1 and A.info["S"] == 0):
        H = pspmm_pcsr_build(A.n_rows, int(colidx.shape[0]), rowptr, colidx, val, 1, 0,
                             stream=stream, n_cols=A.n_cols)
    info["staged_frac"] = pspmm_pcsr_attach_band(H, K, stream)
    if info["staged_frac"] < BAND_MIN_STAGED:
        return cfg, A, info
    info["taken"] = True
    return Config(V=1, S=0, mode=6), H, info


def auto_select(rowptr, colidx, val, K, stream=None):
    """The library's full selection for a square CSR A and K columns (what
    bench.py, tools/k_sweep.py and the CLI run): Table-3 features -> decider
     -> PCSR -> the engine rules of DESIGN.md §5 in order:
    dense tiles (mode 1), row blocks (mode 5), staged bands (mode 6).
    One-time preprocessing; returns (cfg, handle to run, info) and the
    handle serves every later product with this K (or a smaller one)."""
    n = rowptr.shape[0] - 1
    nnz = colidx.shape[0]
    f = pspmm_features_compute(n, nnz, rowptr, colidx, stream=stream)
    cfg = pspmm_decide_config(f, K)
    A = pspmm_pcsr_build(n, nnz, rowptr, colidx, val, cfg.V, cfg.S, cfg.omega, cfg.sg_override,
                         stream)
    info = {}
    cfg, info["dense"] = auto_dense(A, rowptr, colidx, val, K, cfg, stream)
    cfg, A, info["blocks"] = auto_blocks(A, rowptr, colidx, val, K, cfg, stream)
    cfg, A, info["band"] = auto_band(A, rowptr, colidx, val, K, cfg, f, stream)
    return cfg, A, info


def spmm(rowptr, colidx, val, B, cfg: Config | None = None, stream=None, C=None):
    """The three-phase workflow in one call: features -> decider ->
    PCSR -> engine, with the engine rules of auto_select when no cfg is
    given.  Returns (C, cfg, Pcsr) so the handle can be reused."""
    torch = _torch()
    n = rowptr.shape[0] - 1
    nnz = colidx.shape[0]
    K = B.shape[1]
    if cfg is None:
        cfg, A, _ = auto_select(rowptr, colidx, val, K, stream)
    else:
        A = pspmm_pcsr_build(n, nnz, rowptr, colidx, val, cfg.V, cfg.S, cfg.omega,
                             cfg.sg_override, stream)
    if C is None:
        C = torch.empty((n, K), dtype=torch.float32, device=B.device)
    A.run(B, C, cfg, stream)
    return C, cfg, A
