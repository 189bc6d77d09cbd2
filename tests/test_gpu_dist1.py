"""GPU: the distributed code path (hq_solver_create_dist: row-partitioned pass,
all-reduce points, owner row gather, the host-driven Householder continuation
for every update that is not plain CholeskyQR2) on a one-rank communicator --
identity collectives, or a real one-rank NCCL communicator inside the
captured sweep.  Checked against the oracle and the single-GPU path.  The
two-rank path runs in test_gpu_dist2.py."""
import numpy as np
import pytest

import paper_2510_16930_b200 as hq
from conftest import golden
from paper_2510_16930_b200.workloads import config_coo, uniform_coo

pytestmark = pytest.mark.gpu


def _solve(x, ranks, sweeps, u, comm):
    cfg = hq.SolverConfig(ranks=ranks, max_sweeps=sweeps, tol_fit_change=0.0)
    sol = hq.Solver(x, cfg, init_factors=u, comm=comm)
    sol.run(sweeps)
    sol.sync()
    return sol.download(), sol.status()


@pytest.fixture(params=["identity", "nccl"])
def one_rank(request, monkeypatch):
    """a one-rank communicator: identity collectives, or a real one-rank NCCL
    communicator (HQ_NCCL_ONE_RANK=1) so the NCCL calls run inside the captured sweep"""
    if request.param == "nccl":
        monkeypatch.setenv("HQ_NCCL_ONE_RANK", "1")
    return lambda: hq.Comm(1, 0, hq.nccl_unique_id())


@pytest.mark.parametrize("name", ["h3", "h4"])
def test_dist_path_matches_oracle(oracle, name, one_rank):
    g = golden("hoqri.npz")
    dims = [int(d) for d in g[f"{name}_dims"]]
    ranks = [int(r) for r in g[f"{name}_ranks"]]
    coords, vals = g[f"{name}_coords"], g[f"{name}_vals"]
    u0 = [g[f"{name}_U0_{m}"] for m in range(len(dims))]
    x = hq.SparseTensor(dims, coords, vals)
    r, st = _solve(x, ranks, 6, u0, one_rank())
    ref = oracle.hoqri(dims, ranks, coords, vals, u0, 6)
    np.testing.assert_allclose([s.objective for s in r.trace.sweeps], ref["objective"], rtol=1e-9)
    for m in range(len(dims)):
        ug, ur = r.model.factors.factors[m], ref["factors"][m]
        assert np.sqrt(2) * np.linalg.norm(ug - ur @ (ur.T @ ug)) <= 1e-8


def test_dist_path_ill_conditioned_matches_single_gpu(one_rank):
    """Updates the single-GPU path runs as shifted CholeskyQR3 go to the Householder continuation on the
    distributed path: the same decisions, results within rounding."""
    dims, k = [5000, 5000, 5000], 10
    coords, vals = uniform_coo(dims, 50000, 3)
    x = hq.SparseTensor(dims, coords, vals)
    u = hq.random_factors(dims, [k] * 3, 4).factors
    r1, s1 = _solve(x, [k] * 3, 20, u, None)
    r2, s2 = _solve(x, [k] * 3, 20, u, one_rank())
    assert s1["shifted"] > 0 and s2["shifted"] == 0 and s2["dist_householder"] > 0
    np.testing.assert_allclose([s.objective for s in r2.trace.sweeps], [s.objective for s in r1.trace.sweeps],
                               rtol=1e-9)
    for m in range(3):
        a, b = r1.model.factors.factors[m], r2.model.factors.factors[m]
        assert np.linalg.norm(a - b @ (b.T @ a)) <= 1e-8


def test_dist_path_rank_deficient_seeded_fill(one_rank):
    """BASELINE config 2 (seed 1): its later sweeps need the seeded fill (dense_core.cpp:145-157); the
    distributed path reproduces it through the Householder continuation and tracks the single-GPU solve."""
    coords, vals = config_coo(2)
    dims, k = [1000000] * 3, 10
    x = hq.SparseTensor(dims, coords, vals)
    u = hq.random_factors(dims, [k] * 3, 1).factors
    r1, s1 = _solve(x, [k] * 3, 20, u, None)
    r2, s2 = _solve(x, [k] * 3, 20, u, one_rank())
    assert s2["dist_householder"] > 0 and s2["abort"] in (0, 2)
    assert len(r2.trace.sweeps) == 20
    o1 = np.array([s.objective for s in r1.trace.sweeps])
    o2 = np.array([s.objective for s in r2.trace.sweeps])
    np.testing.assert_allclose(o2, o1, rtol=1e-9)
    assert np.all(np.isfinite(o2)) and r2.model.factors.orthonormality_defect() <= 1e-10
