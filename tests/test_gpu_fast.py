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


def _long_case(order, k, seed):
    """Every row of mode 0 long, lengths straddling kShortMax (256), the
    128-nonzero staging chunk and kSegLen (4096) boundaries; at order 4 all
    modes are long (config 5's regime)."""
    rng = np.random.default_rng(seed)
    if order == 3:
        dims = [24, 1800, 1500]
        lens = [257, 300, 383, 384, 385, 511, 4095, 4096, 4097, 4224, 8192, 8193, 9000, 1000, 600, 700,
                257, 2000, 3000, 129, 128, 5, 0, 12000]
    else:
        dims = [20, 160, 140, 120]
        lens = [4097, 3000, 5000, 4096, 257, 9000, 2500, 2600, 2700, 2800, 3100, 3200, 3300, 3400, 3500,
                3600, 3700, 3800, 3900, 4000]
    rows = np.repeat(np.arange(len(lens), dtype=np.uint32), lens)
    coords = np.empty((rows.size, order), np.uint32)
    coords[:, 0] = rows
    for m in range(1, order):
        coords[:, m] = rng.integers(0, dims[m], rows.size, dtype=np.uint32)
    vals = rng.standard_normal(rows.size)
    x = hq.SparseTensor(dims, coords, vals)
    u = hq.random_factors(dims, [k] * order, seed + 1)
    return dims, x, u


@pytest.mark.parametrize("order,k", [(3, 10), (3, 16), (3, 8), (4, 8)])
def test_long_rows_fast_matches_oracle_and_generic(order, k):
    from oracle_bind import Oracle
    o = Oracle()
    dims, x, u = _long_case(order, k, 71 + k + order)
    ranks = [k] * order
    core = hq.ttmc_core(x, u)
    oc = o.ttmc_core(dims, ranks, x.coords(), x.values(), u.factors).reshape(-1)
    assert np.abs(core.data - oc).max() <= 1e-11 * max(1.0, np.abs(oc).max())
    fast = []
    for m in range(order):
        a = hq.ttmctc_elementwise(x, u, m, core)
        ao = o.ttmctc(dims, ranks, x.coords(), x.values(), u.factors, m, core.data)
        assert np.abs(a - ao).max() <= 1e-11 * max(1.0, np.abs(ao).max()), (order, k, m)
        assert (a == hq.ttmctc_elementwise(x, u, m, core)).all()  # bitwise repeatable
        fast.append(a)
    cfg = hq.SolverConfig(ranks=ranks, max_sweeps=3, tol_fit_change=0.0)
    rf = hq.hoqri(x, cfg, init_factors=u.factors)
    ref = o.hoqri(dims, ranks, x.coords(), x.values(), u.factors, 3)
    np.testing.assert_allclose([s.objective for s in rf.trace.sweeps], ref["objective"], rtol=1e-9)
    os.environ["HQ_FORCE_GENERIC"] = "1"
    try:
        gen = [hq.ttmctc_elementwise(x, u, m, core) for m in range(order)]
    finally:
        os.environ.pop("HQ_FORCE_GENERIC", None)
    for a, b in zip(fast, gen):
        assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()


@pytest.mark.parametrize("variant", ["0", "1"])
def test_long_row_segment_variants_in_subprocess(variant):
    """HQ_LONG_SYNC=0/1 (read once per process): the pipelined (k_longseg_mma) and the synchronous
    (k_longseg_sync) long-row segment kernels, each on every long-row shape, against the oracle."""
    import subprocess, sys, textwrap
    code = textwrap.dedent("""
        import sys, numpy as np
        sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
        import paper_2510_16930_b200 as hq
        from oracle_bind import Oracle
        from test_gpu_fast import _long_case
        o = Oracle()
        for order, k in [(3, 10), (3, 16), (3, 8), (4, 8)]:
            dims, x, u = _long_case(order, k, 171 + k + order)
            ranks = [k] * order
            core = hq.ttmc_core(x, u)
            for m in range(order):
                a = hq.ttmctc_elementwise(x, u, m, core)
                ao = o.ttmctc(dims, ranks, x.coords(), x.values(), u.factors, m, core.data)
                assert np.abs(a - ao).max() <= 1e-11 * max(1.0, np.abs(ao).max()), (order, k, m)
        print("ok")
    """)
    env = dict(os.environ, HQ_LONG_SYNC=variant)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
