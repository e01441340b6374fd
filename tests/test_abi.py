"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
headers declare, and its host-only logic (decider, shard plan / remap) is
right.  No device compute is called here."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2605_15695_b200", "libpspmm.so")
LIB_CS = os.path.join(ROOT, "paper_2605_15695_b200", "libpspmm_cusparse.so")


@pytest.fixture(scope="module", autouse=True)
def built():
    if not (os.path.exists(LIB) and os.path.exists(LIB_CS)):
        from paper_2605_15695_b200 import build_ext
        build_ext.build()


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pspmm_\w+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", [("pspmm.h", LIB), ("pspmm_baseline.h", LIB_CS)])
def test_exports_every_declared_symbol(header, lib):
    names = declared(header)
    assert len(names) >= 3
    so = ctypes.CDLL(lib)
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_header_signatures_have_no_torch_types():
    for h in ("pspmm.h", "pspmm_baseline.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        assert "torch" not in text.lower().replace("torch.distributed", "")
        assert "#include <cuda" not in text


def test_status_strings_and_version():
    from paper_2605_15695_b200 import api
    for i, name in enumerate(api.STATUS):
        assert api._lib.pspmm_status_string(i).decode() == name
    assert "sm_100a" in api.version()


FEATS = dict(n=1000, n_hat=900, nnz=20000, delta=0.9, d=20, d_hat=22.2, d_max=900, cv=1.5,
             cv_hat=1.4, sr1=1.2, sr2=1.3, rho=0.02, b=400, b_max=999, pr1=0, pr2=0.4)


@pytest.mark.parametrize("K", [1, 3, 4, 7, 16, 17, 32, 48, 64, 80, 96, 112, 128, 160, 200, 256, 512])
def test_decider_returns_valid_config(K):
    from paper_2605_15695_b200 import api
    for pr2, dmax in [(0.1, 10.0), (0.45, 5000.0)]:
        c = api.pspmm_decide_config(dict(FEATS, pr2=pr2, d_max=dmax), K)
        assert c.V in (1, 2) and c.S in (0, 1) and c.W in (1, 2, 4, 8)
        assert 1 <= c.F <= 8 and c.G in (1, 2, 4, 8, 16, 32) and c.omega == 32
        assert c.mode == 0 or (c.mode == 2 and K % 32 == 0) or (
            c.mode == 3 and K % 4 == 0 and c.V == 1 and c.S == 0)
        # pure: same input, same output
        assert api.pspmm_decide_config(dict(FEATS, pr2=pr2, d_max=dmax), K).as_dict() == c.as_dict()


def test_decider_rejects_empty():
    from paper_2605_15695_b200 import api
    with pytest.raises(api.PspmmError) as e:
        api.pspmm_decide_config(dict(FEATS, nnz=0), 16)
    assert e.value.status == api.PSPMM_ERR_EMPTY


def brute_plan(rowptr, P, align):
    n = len(rowptr) - 1
    nnz = rowptr[-1]
    b = [0]
    for g in range(1, P):
        t = -(-g * nnz // P)
        r = next(i for i in range(n + 1) if rowptr[i] >= t)
        r = min(n, -(-r // align) * align)
        b.append(max(r, b[-1]))
    return b + [n]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("align", [1, 2, 128])
def test_shard_plan_matches_definition(P, align):
    import gen
    from paper_2605_15695_b200 import api
    for g in (gen.powerlaw(700, 9, 2.1, 3), gen.giant_row(300, 290, 2, 4), gen.uniform(50, 3, 5)):
        b = api.pspmm_shard_plan(g.rowptr, P, align)
        assert b.tolist() == brute_plan(g.rowptr.tolist(), P, align)
        assert np.all(np.diff(b) >= 0) and b[0] == 0 and b[-1] == g.n


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_shard_extract_remap(P):
    import gen
    from paper_2605_15695_b200 import api
    g = gen.community(400, 20, 8, 0.7, 9)
    b = api.pspmm_shard_plan(g.rowptr, P, 2)
    B = gen.dense(g.n, 5, 1)
    n_max = int(np.diff(b).max())
    Bfull = np.zeros((P * n_max, 5), np.float32)
    for r in range(P):
        Bfull[r * n_max: r * n_max + b[r + 1] - b[r]] = B[b[r]:b[r + 1]]
    for r in range(P):
        lrp, lci, lvl, nm = api.pspmm_shard_extract(g.rowptr, g.colidx, g.val, P, b, r)
        assert nm == n_max
        lo, hi = b[r], b[r + 1]
        assert np.array_equal(lrp, g.rowptr[lo:hi + 1] - g.rowptr[lo])
        orig = g.colidx[g.rowptr[lo]:g.rowptr[hi]]
        assert np.array_equal(Bfull[lci], B[orig])          # same B rows after the remap
        assert np.array_equal(lvl, g.val[g.rowptr[lo]:g.rowptr[hi]])
        for i in range(hi - lo):                            # still canonical per row
            assert np.all(np.diff(lci[lrp[i]:lrp[i + 1]]) > 0)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_own_remote_column_split(P):
    """dist.split_own_columns: the two blocks partition every row's nonzeros,
    the own block is remapped to local B rows, both stay canonical."""
    import gen
    from paper_2605_15695_b200 import dist
    g = gen.community(500, 25, 9, 0.7, 12)
    for r in range(P):
        sh = dist.make_shard(g.rowptr, g.colidx, g.val, P, r, align=2)
        (orp, oci, ovl), (rrp, rci, rvl) = dist.split_own_columns(sh)
        assert np.array_equal(np.diff(orp) + np.diff(rrp), np.diff(sh.rowptr))
        lo = r * sh.n_max
        for i in range(sh.rows):
            full = sh.colidx[sh.rowptr[i]:sh.rowptr[i + 1]]
            own = oci[orp[i]:orp[i + 1]]
            rem = rci[rrp[i]:rrp[i + 1]]
            assert np.all(np.diff(own) > 0) and np.all(np.diff(rem) > 0)
            assert np.all((own >= 0) & (own < sh.rows))
            assert sorted(np.concatenate([own + lo, rem]).tolist()) == full.tolist()


def test_product_path_never_touches_oracle():
    """The product (package + native sources) never imports, links or loads
    the oracle, and the oracle never includes the product's headers."""
    pkg = os.path.join(ROOT, "paper_2605_15695_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text and "oracle/" not in text, f
    src = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    assert "pspmm.h" not in src and "common.cuh" not in src
    py = open(os.path.join(ROOT, "oracle", "__init__.py")).read()
    assert "paper_2605_15695_b200" not in py.split('"""')[2]
