"""Helpers shared by the -m gpu parity tests (test infrastructure)."""
import numpy as np

import oracle

# BASELINE.json north_star tolerance, per element
RTOL_MAG = 1e-5
ATOL = 1e-6


def dev(g, device="cuda"):
    import torch
    rp = torch.from_numpy(np.ascontiguousarray(g.rowptr)).to(device)
    ci = torch.from_numpy(np.ascontiguousarray(g.colidx) if len(g.colidx) else
                          np.zeros(1, np.int32)).to(device)
    vl = torch.from_numpy(np.ascontiguousarray(g.val) if len(g.val) else
                          np.zeros(1, np.float32)).to(device)
    return rp, ci, vl


def within_tol(C_gpu, ref, mag):
    """Boolean mask of elements meeting |C - ref| <= 1e-5 mag + 1e-6."""
    C = np.asarray(C_gpu, dtype=np.float64)
    return np.abs(C - ref) <= RTOL_MAG * mag + ATOL


def assert_parity(C_gpu, ref, mag, what=""):
    ok = within_tol(C_gpu, ref, mag)
    if not ok.all():
        bad = np.argwhere(~ok)[:5]
        C = np.asarray(C_gpu, dtype=np.float64)
        detail = [(tuple(i), C[tuple(i)], ref[tuple(i)], mag[tuple(i)]) for i in bad]
        raise AssertionError(f"{what}: {int((~ok).sum())} elements out of tolerance, e.g. {detail}")


_cache = {}


def oracle_ref(g, B, key=None):
    # the fingerprint of B guards against two tests sharing a key with different B
    k = (key, B.shape, B.ravel()[:64].tobytes(), float(B.sum())) if key is not None else None
    if k is not None and k in _cache:
        return _cache[k]
    ref = oracle.spmm(g.rowptr, g.colidx, g.val, B, threads=8)
    if k is not None:
        _cache[k] = ref
    return ref
