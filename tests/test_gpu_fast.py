"""GPU: the specialised order-3 pass (K = 10, 16, 8) against the oracle and
against the generic kernels on the same inputs (HQ_FORCE_GENERIC=1)."""
import os

import numpy as np
import pytest

import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import uniform_coo

pytestmark = pytest.mark.gpu


@pytest.fixture()
def generic_env():
    os.environ["HQ_FORCE_GENERIC"] = "1"
    yield
    os.environ.pop("HQ_FORCE_GENERIC", None)


def _case(dims, draws, k, seed, skew=False):
    coords, vals = uniform_coo(dims, draws, seed)
    if skew:  # a few heavy rows in every mode -> segmented long-row path
        coords[: draws // 4, 0] = 3
        coords[draws // 4: draws // 2, 1] = 5
    x = hq.SparseTensor(dims, coords, vals)
    u = hq.random_factors(dims, [k] * 3, seed + 1)
    return x, u


@pytest.mark.parametrize("k", [10, 16, 8])
@pytest.mark.parametrize("skew", [False, True])
def test_fast_pass_matches_oracle(k, skew):
    from oracle_bind import Oracle
    o = Oracle()
    dims = [3000, 2500, 2000]
    x, u = _case(dims, 60000, k, 17 + k, skew)
    core = hq.ttmc_core(x, u)
    oc = o.ttmc_core(dims, [k] * 3, x.coords(), x.values(), u.factors).reshape(-1)
    assert np.abs(core.data - oc).max() <= 1e-11 * max(1.0, np.abs(oc).max())
    for m in range(3):
        a = hq.ttmctc_elementwise(x, u, m, core)
        ao = o.ttmctc(dims, [k] * 3, x.coords(), x.values(), u.factors, m, core.data)
        assert np.abs(a - ao).max() <= 1e-11 * max(1.0, np.abs(ao).max()), (k, m)
        assert (a == hq.ttmctc_elementwise(x, u, m, core)).all()  # bitwise repeatable


@pytest.mark.parametrize("k", [10, 16])
def test_fast_and_generic_agree(k, request):
    dims = [1500, 1200, 1000]
    x, u = _case(dims, 30000, k, 5 + k, skew=True)
    core = hq.ttmc_core(x, u)
    fast = [hq.ttmctc_elementwise(x, u, m, core) for m in range(3)]
    cfg = hq.SolverConfig(ranks=[k] * 3, max_sweeps=4, tol_fit_change=0.0)
    rf = hq.hoqri(x, cfg, init_factors=u.factors)
    os.environ["HQ_FORCE_GENERIC"] = "1"
    try:
        core_g = hq.ttmc_core(x, u)
        gen = [hq.ttmctc_elementwise(x, u, m, core_g) for m in range(3)]
        rg = hq.hoqri(x, cfg, init_factors=u.factors)
    finally:
        os.environ.pop("HQ_FORCE_GENERIC", None)
    assert np.abs(core.data - core_g.data).max() <= 1e-12 * np.abs(core_g.data).max()
    for a, b in zip(fast, gen):
        assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()
    rel = np.linalg.norm(rf.model.core.data - rg.model.core.data) / np.linalg.norm(rg.model.core.data)
    assert rel <= 1e-10
    np.testing.assert_allclose([s.objective for s in rf.trace.sweeps], [s.objective for s in rg.trace.sweeps],
                               rtol=1e-10)
