"""Seeded synthetic graph generators (see gen/__init__.py and DESIGN.md §4).

Every generator returns canonical CSR: int32 rowptr (n+1), int32 colidx with
strictly increasing columns per row, float32 values.  Determinism: fixed
seed -> bit-identical arrays (numpy PCG64 Generator).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Graph:
    name: str
    n: int
    rowptr: np.ndarray
    colidx: np.ndarray
    val: np.ndarray
    K: int = 0
    seeds: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])


# --------------------------------------------------------------------------
# helpers
# --------------------------------------------------------------------------

def values(nnz: int, seed: int, kind: str = "uniform") -> np.ndarray:
    """A values: U[-1,1) (c-16), all-ones ("pattern") or small integers."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return (rng.random(nnz, dtype=np.float32) * 2.0 - 1.0).astype(np.float32)
    if kind == "ones":
        return np.ones(nnz, dtype=np.float32)
    if kind == "int":
        return rng.integers(-4, 5, size=nnz).astype(np.float32)
    if kind == "positive":
        return rng.random(nnz, dtype=np.float32) + np.float32(1e-3)
    raise ValueError(kind)


def dense(n: int, K: int, seed: int, kind: str = "uniform") -> np.ndarray:
    """Dense B (n x K, row-major float32): U[-1,1) (c-17) or small integers."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return (rng.random((n, K), dtype=np.float32) * 2.0 - 1.0).astype(np.float32)
    if kind == "int":
        return rng.integers(-4, 5, size=(n, K)).astype(np.float32)
    if kind == "positive":
        return rng.random((n, K), dtype=np.float32) + np.float32(1e-3)
    raise ValueError(kind)


def _uniq(a: np.ndarray) -> np.ndarray:
    """Sorted distinct values (np.unique is hash-based and slow here)."""
    s = np.sort(a)
    if s.shape[0] == 0:
        return s
    keep = np.empty(s.shape[0], dtype=bool)
    keep[0] = True
    np.not_equal(s[1:], s[:-1], out=keep[1:])
    return s[keep]


def csr_from_pairs(n: int, rows: np.ndarray, cols: np.ndarray):
    """Canonical CSR pattern from (row, col) pairs: sorted, duplicates dropped."""
    keys = rows.astype(np.int64) * n + cols.astype(np.int64)
    keys = _uniq(keys)
    r = (keys // n).astype(np.int64)
    c = (keys % n).astype(np.int32)
    counts = np.bincount(r, minlength=n)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    if rowptr[-1] >= 2**31:
        raise ValueError("nnz exceeds int32")
    return rowptr.astype(np.int32), c


def _finish(name, n, rowptr, colidx, val_seed, K=0, seeds=None, kind="uniform"):
    return Graph(name=name, n=n, rowptr=rowptr, colidx=colidx,
                 val=values(int(rowptr[-1]), val_seed, kind), K=K, seeds=seeds or {})


def permute(n: int, rowptr, colidx, perm):
    """Relabel node i -> perm[i] on both sides (pattern only)."""
    deg = np.diff(rowptr.astype(np.int64))
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    return csr_from_pairs(n, perm[rows], perm[colidx.astype(np.int64)])


# --------------------------------------------------------------------------
# undirected edge samplers
# --------------------------------------------------------------------------

def _sample_undirected(n, m, draw, rng, extra=1.08):
    """Draw undirected edges {u,v}, u != v, distinct, until exactly m exist.

    draw(count) -> (u, v) int64 arrays.  Top up while short, trim a random
    excess if over (SURVEY §8(d) generator mechanics).
    """
    keys = np.zeros(0, dtype=np.int64)
    want = int(m * extra) + 16
    for _ in range(200):
        u, v = draw(want)
        ok = u != v
        u, v = u[ok], v[ok]
        new = _uniq(np.minimum(u, v) * n + np.maximum(u, v))
        if keys.shape[0]:
            pos = np.searchsorted(keys, new)
            pos[pos == keys.shape[0]] = 0
            new = new[keys[pos] != new]
            # both runs sorted: the stable (tim/radix) sort merges them cheaply
            keys = np.sort(np.concatenate([keys, new]))
        else:
            keys = new
        if keys.shape[0] >= m:
            break
        deficit = m - keys.shape[0]
        yield_rate = max(new.shape[0] / max(want, 1), 0.02)
        want = int(deficit / yield_rate * 1.25) + 1024
    if keys.shape[0] < m:
        raise RuntimeError("generator could not reach the target edge count")
    if keys.shape[0] > m:
        keep = rng.choice(keys.shape[0], size=m, replace=False)
        keys = np.sort(keys[keep])
    return keys // n, keys % n


def _undirected_csr(n, u, v):
    return csr_from_pairs(n, np.concatenate([u, v]), np.concatenate([v, u]))


def _zipf_alpha(n, d_mean, d_max, iters=60):
    """alpha such that mean(d_max (i+1)^-alpha) = d_mean (bisection)."""
    i = np.arange(1, n + 1, dtype=np.float64)
    li = np.log(i)
    lo, hi = 0.0, 8.0
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        m = d_max * np.exp(-mid * li).mean()
        if m > d_mean:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def _weighted_drawer(w, rng, offset=0):
    cdf = np.cumsum(w / w.sum())
    cdf[-1] = 1.0

    def draw(count):
        # sorted queries make searchsorted cache-friendly; v is re-shuffled so
        # the (u, v) pairing stays independent
        u = np.searchsorted(cdf, np.sort(rng.random(count)), side="right").astype(np.int64)
        v = np.searchsorted(cdf, np.sort(rng.random(count)), side="right").astype(np.int64)
        v = v[rng.permutation(count)]
        return u + offset, v + offset
    return draw


def chung_lu(n, nnz, d_max, seed, shuffle_seed=None):
    """Chung-Lu power law: Zipf-rank weights w_i = d_max (i+1)^-alpha with
    alpha solved so mean(w) = nnz/n; symmetric, no self-loops, exact nnz
    (nnz must be even).  IDs shuffled with shuffle_seed (else rank order)."""
    assert nnz % 2 == 0
    rng = np.random.default_rng(seed)
    alpha = _zipf_alpha(n, nnz / n, d_max)
    w = d_max * np.arange(1, n + 1, dtype=np.float64) ** (-alpha)
    u, v = _sample_undirected(n, nnz // 2, _weighted_drawer(w, rng), rng)
    if shuffle_seed is not None:
        perm = np.random.default_rng(shuffle_seed).permutation(n).astype(np.int64)
        u, v = perm[u], perm[v]
    return _undirected_csr(n, u, v)


def roadnet_like(n, nnz, seed, diag_frac=0.02):
    """Poisson-like planar graph: a ceil(sqrt n)-wide lattice in row-major
    IDs (locality order); exactly nnz/2 undirected lattice edges kept,
    a diag_frac share of them diagonals."""
    assert nnz % 2 == 0
    rng = np.random.default_rng(seed)
    Wd = int(np.ceil(np.sqrt(n)))
    ids = np.arange(n, dtype=np.int64)
    right = ids[((ids % Wd) != Wd - 1) & (ids + 1 < n)]
    down = ids[ids + Wd < n]
    diag = ids[((ids % Wd) != Wd - 1) & (ids + Wd + 1 < n)]
    m = nnz // 2
    m_diag = int(round(diag_frac * m))
    m_lat = m - m_diag
    lat_u = np.concatenate([right, down])
    lat_v = np.concatenate([right + 1, down + Wd])
    pick = rng.choice(lat_u.shape[0], size=m_lat, replace=False)
    dpick = rng.choice(diag.shape[0], size=m_diag, replace=False)
    u = np.concatenate([lat_u[pick], diag[dpick]])
    v = np.concatenate([lat_v[pick], diag[dpick] + Wd + 1])
    return _undirected_csr(n, u, v)


def block_lognormal(n, nnz, blocks, d_max, sigma, seed, community_order=True):
    """proteins-shaped: `blocks` diagonal blocks, edges only inside a block,
    Chung-Lu with lognormal(sigma) weights clipped at d_max; block-ordered IDs."""
    assert nnz % 2 == 0
    rng = np.random.default_rng(seed)
    bounds = np.linspace(0, n, blocks + 1).astype(np.int64)
    m_total = nnz // 2
    sizes = np.diff(bounds)
    m_b = (m_total * sizes // n).astype(np.int64)
    m_b[-1] += m_total - m_b.sum()
    us, vs = [], []
    for b in range(blocks):
        nb = int(sizes[b])
        w = rng.lognormal(0.0, sigma, nb)
        w = np.minimum(w / w.mean() * (2.0 * m_b[b] / nb), d_max)
        u, v = _sample_undirected(nb, int(m_b[b]), _weighted_drawer(w, rng), rng)
        us.append(u + bounds[b])
        vs.append(v + bounds[b])
    u = np.concatenate(us)
    v = np.concatenate(vs)
    if not community_order:
        perm = rng.permutation(n).astype(np.int64)
        u, v = perm[u], perm[v]
    return _undirected_csr(n, u, v)


# --------------------------------------------------------------------------
# small generic generators (tests, decider corpus)
# --------------------------------------------------------------------------

def uniform(n, d, seed, kind="uniform"):
    """Directed Erdos-Renyi-like: each row draws ~Poisson(d) random columns."""
    rng = np.random.default_rng(seed)
    deg = rng.poisson(d, n)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    cols = rng.integers(0, n, rows.shape[0])
    rowptr, colidx = csr_from_pairs(n, rows, cols)
    return _finish(f"uniform_n{n}_d{d}", n, rowptr, colidx, seed + 1000, kind=kind)


def powerlaw(n, d, exponent, seed, kind="uniform", d_max=None):
    """Directed power law: row degrees ~ Zipf-rank (exponent), random cols,
    rows shuffled."""
    rng = np.random.default_rng(seed)
    d_max = d_max or max(2, n // 2)
    w = np.arange(1, n + 1, dtype=np.float64) ** (-1.0 / (exponent - 1.0))
    w = w / w.mean() * d
    deg = np.minimum(rng.poisson(w), n).astype(np.int64)
    deg = np.minimum(deg, d_max)
    rng.shuffle(deg)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    cols = rng.integers(0, n, rows.shape[0])
    rowptr, colidx = csr_from_pairs(n, rows, cols)
    return _finish(f"powerlaw_n{n}_d{d}_e{exponent}", n, rowptr, colidx, seed + 1000, kind=kind)


def banded(n, half_width, seed, fill=0.7, kind="uniform"):
    """Banded pattern |i-j| <= half_width, each band entry kept w.p. fill."""
    rng = np.random.default_rng(seed)
    offs = np.arange(-half_width, half_width + 1, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), offs.shape[0])
    cols = rows + np.tile(offs, n)
    ok = (cols >= 0) & (cols < n) & (rng.random(rows.shape[0]) < fill)
    rowptr, colidx = csr_from_pairs(n, rows[ok], cols[ok])
    return _finish(f"banded_n{n}_h{half_width}", n, rowptr, colidx, seed + 1000, kind=kind)


def _community_pattern(n, csize, d, p_in, seed, ordered=True):
    """(rowptr, colidx) of community(); see there."""
    rng = np.random.default_rng(seed)
    deg = rng.poisson(d, n)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    inside = rng.random(rows.shape[0]) < p_in
    base = (rows // csize) * csize
    span = np.minimum(csize, n - base)
    cols = np.where(inside, base + (rng.random(rows.shape[0]) * span).astype(np.int64),
                    rng.integers(0, n, rows.shape[0]))
    if not ordered:
        perm = rng.permutation(n).astype(np.int64)
        rows, cols = perm[rows], perm[cols]
    return csr_from_pairs(n, rows, cols)


def community(n, csize, d, p_in, seed, ordered=True, kind="uniform"):
    """Communities of csize nodes; a p_in share of each row's edges stays in
    its community.  ordered=True keeps community-contiguous IDs."""
    rowptr, colidx = _community_pattern(n, csize, d, p_in, seed, ordered)
    return _finish(f"community_n{n}_c{csize}", n, rowptr, colidx, seed + 1000, kind=kind)


def with_empty_rows(g: Graph, frac, seed):
    """Copy of g with a random `frac` of rows emptied (edge cases)."""
    rng = np.random.default_rng(seed)
    keep_row = rng.random(g.n) >= frac
    deg = np.diff(g.rowptr.astype(np.int64))
    rows = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    mask = keep_row[rows]
    colidx = g.colidx[mask]
    val = g.val[mask]
    counts = np.bincount(rows[mask], minlength=g.n)
    rowptr = np.zeros(g.n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    return Graph(g.name + "_empty", g.n, rowptr.astype(np.int32), colidx, val)


def giant_row(n, giant, d, seed, kind="uniform"):
    """One row (n//3) with `giant` nonzeros, the others ~Poisson(d)."""
    rng = np.random.default_rng(seed)
    deg = rng.poisson(d, n)
    deg[n // 3] = min(giant, n)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    cols = rng.integers(0, n, rows.shape[0])
    big = n // 3
    cols[rows == big] = rng.permutation(n)[: int(deg[big])]
    rowptr, colidx = csr_from_pairs(n, rows, cols)
    return _finish(f"giant_n{n}", n, rowptr, colidx, seed + 1000, kind=kind)


# --------------------------------------------------------------------------
# the five BASELINE.json configs
# --------------------------------------------------------------------------

CONFIGS = {
    #  name       n          nnz          K    seeds (graph, vals, B, shuffle)
    "cora":     dict(n=2708, nnz=10556, K=16, seeds=(1, 1001, 2001, 3001), d_max=168),
    "roadnet":  dict(n=1965206, nnz=5533214, K=32, seeds=(2, 1002, 2002, None)),
    "products": dict(n=2449029, nnz=123718280, K=128, seeds=(3, 1003, 2003, 3003),
                     d_max=17481),
    "proteins": dict(n=132534, nnz=79122504, K=256, seeds=(4, 1004, 2004, None),
                     d_max=7750),
    "reddit":   dict(n=232965, nnz=114615892, K=64, seeds=(5, 1005, 2005, 3005),
                     d_max=21657),
    # SURVEY §8(d) proteins variant (ii), for the dense-panel path (a6):
    # communities of 1024 community-ordered nodes, half of each row's
    # Poisson(597) draws inside its community (~25 % dense diagonal blocks
    # after duplicates are dropped, ~74M nnz realized), half uniform
    "proteins_clustered": dict(n=132534, nnz=79122504, K=256, seeds=(6, 1006, 2006, None),
                               csize=1024, p_in=0.5),
}


def config_graph(name: str, scale: float = 1.0) -> Graph:
    """The named BASELINE.json workload.  scale < 1 gives a same-shaped graph
    with n and nnz scaled by `scale` (parity tests that the oracle finishes in
    seconds); scale == 1 is the full bench size."""
    c = CONFIGS[name]
    # scaled-down shape: n * scale nodes, the same mean degree capped at n/8
    # (so small graphs stay sparse), d_max scaled like the mean
    n = max(64, int(round(c["n"] * scale)))
    d = c["nnz"] / c["n"]
    cap = n / 32.0 if name.startswith("proteins") else n / 8.0  # proteins: 8 dense blocks
    shrink = 1.0 if scale >= 1.0 else min(1.0, cap / d)
    nnz = int(round(n * d * shrink)) if scale < 1.0 else c["nnz"]
    nnz -= nnz % 2
    gs, vs, _bs, ss = c["seeds"]
    if name in ("cora", "products", "reddit"):
        d_max = max(8, min(n - 1, int(round(c["d_max"] * shrink))))
        rowptr, colidx = chung_lu(n, nnz, d_max, gs, shuffle_seed=ss)
    elif name == "roadnet":
        rowptr, colidx = roadnet_like(n, nnz, gs)
    elif name == "proteins_clustered":
        dd = d * shrink if scale < 1.0 else d
        rowptr, colidx = _community_pattern(n, c["csize"], dd, c["p_in"], gs)
    elif name == "proteins":
        blocks = 8
        d_max = max(8, min(n // blocks - 1, int(round(c["d_max"] * shrink))))
        rowptr, colidx = block_lognormal(n, nnz, blocks, d_max, 0.75, gs)
    else:
        raise KeyError(name)
    return Graph(name=name, n=n, rowptr=rowptr, colidx=colidx,
                 val=values(int(rowptr[-1]), vs), K=c["K"],
                 seeds=dict(graph=gs, val=vs, B=_bs, shuffle=ss, scale=scale))


def config_B(name: str, n: int, K: int | None = None) -> np.ndarray:
    c = CONFIGS[name]
    return dense(n, K or c["K"], c["seeds"][2])
