"""(a2) GPU Table-3 features against the oracle (c-3, c-23): integer-valued
features and the formula-identical ratios bit-exact; CV / CV^ (exact-integer
variance on the GPU vs two-pass fp64 in the oracle) to 1e-12 relative."""
import numpy as np
import pytest

import gen
import oracle
from gpu_util import dev

pytestmark = pytest.mark.gpu

EXACT = ("n", "n_hat", "nnz", "delta", "d", "d_hat", "d_max", "sr1", "sr2", "rho", "b",
         "b_max", "pr1", "pr2")


@pytest.mark.parametrize("make", [
    lambda: gen.uniform(1001, 7, 1), lambda: gen.powerlaw(3000, 12, 2.0, 2),
    lambda: gen.banded(2049, 5, 3), lambda: gen.with_empty_rows(gen.community(4000, 64, 20, 0.85, 4), 0.2, 9),
    lambda: gen.giant_row(5001, 4990, 3, 5), lambda: gen.config_graph("cora"),
    lambda: gen.config_graph("reddit", 0.01), lambda: gen.config_graph("roadnet", 0.01)])
@pytest.mark.parametrize("omega", [4, 32])
def test_features_match_oracle(make, omega):
    from paper_2605_15695_b200 import api
    g = make()
    ref = oracle.features(g.rowptr, g.colidx, g.val, omega)
    rp, ci, _ = dev(g)
    f = api.pspmm_features_compute(g.n, g.nnz, rp, ci, omega)
    for k in EXACT:
        assert f[k] == ref[k], (k, f[k], ref[k])
    for k in ("cv", "cv_hat"):
        assert f[k] == pytest.approx(ref[k], rel=1e-12, abs=1e-15), k


def test_features_empty_rejected():
    from paper_2605_15695_b200 import api
    g = gen.Graph("empty", 10, np.zeros(11, np.int32), np.zeros(0, np.int32),
                  np.zeros(0, np.float32))
    rp, ci, _ = dev(g)
    with pytest.raises(api.PspmmError) as e:
        api.pspmm_features_compute(g.n, 0, rp, ci)
    assert e.value.status == api.PSPMM_ERR_EMPTY
