"""GPU: skewed (Zipf) tensors -- the shape of BASELINE config 3 at test scale.

Every mode of a Zipf tensor is "hot" (rows longer than 32x the mean hold >= 5 %
of the nonzeros), so the passes gather those factors L1-allocating
(cp.async.ca) and the heavy rows run through the segmented long-row kernels.
Results must match the oracle (restatement of the reference's kernels.cpp /
solvers.cpp) exactly as for uniform tensors, and be bitwise repeatable."""
import numpy as np
import pytest

import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import uniform_coo, zipf_coo

pytestmark = pytest.mark.gpu

DIMS = [20000, 4000, 400]
K = 10


@pytest.fixture(scope="module")
def zipf_tensor():
    coords, vals = zipf_coo(DIMS, 300000, 3)
    return hq.SparseTensor(DIMS, coords, vals)


def test_mode_plan_marks_skewed_modes_hot(zipf_tensor):
    for m in range(3):
        p = zipf_tensor.mode_plan(m)
        assert p["rows"] == DIMS[m]
        assert p["hot"], (m, p)
        assert p["long_rows"] > 0 and p["long_segments"] >= p["long_rows"]
    coords, vals = uniform_coo([3000, 2500, 2000], 60000, 5)
    u = hq.SparseTensor([3000, 2500, 2000], coords, vals)
    assert not any(u.mode_plan(m)["hot"] for m in range(3))
    with pytest.raises(hq.RangeError):
        u.mode_plan(3)


def test_zipf_kernels_match_oracle(oracle, zipf_tensor):
    x = zipf_tensor
    u = hq.random_factors(DIMS, [K] * 3, 21)
    core = hq.ttmc_core(x, u)
    oc = oracle.ttmc_core(DIMS, [K] * 3, x.coords(), x.values(), u.factors).reshape(-1)
    scale = max(1.0, np.abs(oc).max())
    assert np.abs(core.data - oc).max() <= 1e-11 * scale
    for m in range(3):
        a = hq.ttmctc_elementwise(x, u, m, core)
        ao = oracle.ttmctc(DIMS, [K] * 3, x.coords(), x.values(), u.factors, m, core.data)
        assert np.abs(a - ao).max() <= 1e-11 * max(1.0, np.abs(ao).max()), m
        assert (a == hq.ttmctc_elementwise(x, u, m, core)).all()  # bitwise repeatable


def test_zipf_hoqri_matches_oracle(oracle, zipf_tensor):
    x = zipf_tensor
    sweeps = 4
    u0 = oracle.random_factors(DIMS, [K] * 3, 13)
    r = hq.hoqri(x, hq.SolverConfig(ranks=[K] * 3, max_sweeps=sweeps, tol_fit_change=0.0), init_factors=u0)
    ro = oracle.hoqri(DIMS, [K] * 3, x.coords(), x.values(), u0, sweeps)
    rel = np.linalg.norm(r.model.core.data - ro["core"].reshape(-1)) / np.linalg.norm(ro["core"])
    assert rel <= 1e-9, rel
    obj = np.array([s.objective for s in r.trace.sweeps])
    np.testing.assert_allclose(obj, ro["objective"], rtol=1e-9, atol=0)


@pytest.mark.parametrize("k", [8, 10])
def test_all_long_rows_with_empty_rows(oracle, k):
    """A mode whose non-empty rows are ALL long (no tile kernel runs) and that also has empty rows: the empty
    rows' A must read as 0 (the A buffer is shared by the modes, so stale rows of another mode's update would
    leak into the QR).  Mode 1 has 6 distinct indices, so its A has rank <= 6 < K and every mode-1 update
    takes the reference's seeded fill."""
    rng = np.random.default_rng(5)
    dims, n = [300, 240, 200], 6000
    coords = np.empty((n, 3), np.uint32)
    coords[:, 0] = rng.integers(0, dims[0], n)
    coords[:, 1] = rng.choice(np.array([3, 50, 77, 120, 199, 230], np.uint32), n)
    coords[:, 2] = rng.integers(0, dims[2], n)
    vals = rng.random(n)
    x = hq.SparseTensor(dims, coords, vals)
    p = x.mode_plan(1)
    assert p["nonempty_rows"] == 6 and p["long_rows"] == 6, p
    sweeps = 4
    u0 = oracle.random_factors(dims, [k] * 3, 13)
    r = hq.hoqri(x, hq.SolverConfig(ranks=[k] * 3, max_sweeps=sweeps, tol_fit_change=0.0), init_factors=u0)
    ro = oracle.hoqri(dims, [k] * 3, x.coords(), x.values(), u0, sweeps)
    obj = np.array([s.objective for s in r.trace.sweeps])
    np.testing.assert_allclose(obj, ro["objective"], rtol=1e-9)
    rel = np.linalg.norm(r.model.core.data - ro["core"].reshape(-1)) / np.linalg.norm(ro["core"])
    assert rel <= 1e-9, rel


# ---- fiber units (hq_pass.cu plan_fibers): the long rows' Kronecker products taken once per fiber


def _with_fibers(flag, fn):
    import os
    old = os.environ.get("HQ_FIBERS")
    os.environ["HQ_FIBERS"] = flag
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["HQ_FIBERS"]
        else:
            os.environ["HQ_FIBERS"] = old


def test_fiber_units_cover_the_long_rows():
    coords, vals = zipf_coo(DIMS, 300000, 3)
    x = _with_fibers("1", lambda: hq.SparseTensor(DIMS, coords, vals))
    off = _with_fibers("0", lambda: hq.SparseTensor(DIMS, coords, vals))
    c = x.coords()
    for m in range(3):
        p, f = x.mode_plan(m), x.fiber_plan(m)
        cnt = np.bincount(c[:, m], minlength=DIMS[m])
        sm = f["short_max"]
        assert sm == (64 if p["hot"] else 256) and off.fiber_plan(m)["short_max"] == 256
        long_nnz = int(cnt[cnt > sm].sum())
        assert f["long_nnz"] == long_nnz and p["long_rows"] == int((cnt > sm).sum())
        # units = sum over fibers (row, first other index) of the long rows of ceil(len / 16)
        o = [v for v in range(3) if v != m][0]
        sel = cnt[c[:, m]] > sm
        key = c[sel, m].astype(np.int64) * DIMS[o] + c[sel, o]
        _, lens = np.unique(key, return_counts=True)
        lo = int(np.ceil(lens / 16).sum())
        # a fiber that straddles a 4096-nonzero segment boundary is cut there: at most one more unit per segment
        assert lo <= f["units"] <= lo + p["long_segments"], (m, f, lo)
        assert 1 <= f["segments"] <= p["long_segments"]
        assert off.fiber_plan(m)["units"] == 0


@pytest.mark.parametrize("k", [10, 16, 8])
def test_fiber_units_match_oracle_and_plain_long_rows(oracle, k):
    coords, vals = zipf_coo(DIMS, 300000, 3)
    u = hq.random_factors(DIMS, [k] * 3, 21)
    res = {}
    for flag in ("1", "0"):
        x = _with_fibers(flag, lambda: hq.SparseTensor(DIMS, coords, vals))
        assert (x.fiber_plan(1)["units"] > 0) == (flag == "1")
        core = hq.ttmc_core(x, u)
        res[flag] = [core.data] + [hq.ttmctc_elementwise(x, u, m, core) for m in range(3)]
        if flag == "1":
            oc = oracle.ttmc_core(DIMS, [k] * 3, x.coords(), x.values(), u.factors).reshape(-1)
            assert np.abs(core.data - oc).max() <= 1e-11 * max(1.0, np.abs(oc).max())
            for m in range(3):
                ao = oracle.ttmctc(DIMS, [k] * 3, x.coords(), x.values(), u.factors, m, core.data)
                assert np.abs(res[flag][1 + m] - ao).max() <= 1e-11 * max(1.0, np.abs(ao).max()), m
                assert (res[flag][1 + m] == hq.ttmctc_elementwise(x, u, m, core)).all()  # bitwise repeatable
    for a, b in zip(res["1"], res["0"]):
        assert np.abs(a - b).max() <= 1e-11 * max(1.0, np.abs(b).max())


def test_fiber_units_hoqri_matches_oracle(oracle):
    coords, vals = zipf_coo(DIMS, 300000, 3)
    x = _with_fibers("1", lambda: hq.SparseTensor(DIMS, coords, vals))
    sweeps = 4
    u0 = oracle.random_factors(DIMS, [K] * 3, 13)
    r = hq.hoqri(x, hq.SolverConfig(ranks=[K] * 3, max_sweeps=sweeps, tol_fit_change=0.0), init_factors=u0)
    ro = oracle.hoqri(DIMS, [K] * 3, x.coords(), x.values(), u0, sweeps)
    rel = np.linalg.norm(r.model.core.data - ro["core"].reshape(-1)) / np.linalg.norm(ro["core"])
    assert rel <= 1e-9, rel
    obj = np.array([s.objective for s in r.trace.sweeps])
    np.testing.assert_allclose(obj, ro["objective"], rtol=1e-9, atol=0)
