"""GPU: the desk-scale dense paths against the reference
(tests/golden/dense.npz): densify_unfold, ttmc_unfold_dense, svd_leading,
HOSVD init, HOQRI from HOSVD, HOOI (random / HOSVD, traced).  The eigen-solve
is cuSOLVER's, so factors are compared as subspaces and every other quantity
(objective, fit, drift, gradient) is rotation-invariant."""
import numpy as np
import pytest

import paper_2510_16930_b200 as hq
from conftest import golden

pytestmark = pytest.mark.gpu
G = golden("dense.npz")
NAMES = [str(n) for n in G["names"]]


def _x(name):
    return hq.SparseTensor([int(d) for d in G[f"{name}_dims"]], G[f"{name}_coords"], G[f"{name}_vals"])


def _subspace(u, v):
    return float(np.sqrt(2.0) * np.linalg.norm(u - v @ (v.T @ u)))


@pytest.mark.parametrize("name", NAMES)
def test_dense_unfoldings(name):
    x = _x(name)
    ranks = [int(r) for r in G[f"{name}_ranks"]]
    u0 = [G[f"{name}_U0_{m}"] for m in range(x.order())]
    for m in range(x.order()):
        np.testing.assert_array_equal(hq.densify_unfold(x, m), G[f"{name}_dense{m}"])
        y = hq.ttmc_unfold_dense(x, u0, m)
        ref = G[f"{name}_Y{m}"]
        assert np.abs(y - ref).max() <= 1e-11 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("sv", [str(n) for n in G["svd_names"]])
def test_svd_leading(sv):
    a, k, ref = G[f"{sv}_A"], int(G[f"{sv}_k"]), G[f"{sv}_U"]
    u = hq.svd_leading(a, k)
    assert np.abs(u.T @ u - np.eye(k)).max() <= 1e-12
    r = int(np.linalg.matrix_rank(a))
    if 0 < r < k:
        # beyond the numerical rank the reference back-transforms round-off directions
        # (sigma ~ 1e-8 sigma_max passes its 1e-12 test): only the range part is defined
        assert _subspace(u[:, :r], ref[:, :r]) <= 1e-9
    else:
        assert _subspace(u, ref) <= 1e-9


@pytest.mark.parametrize("name", NAMES)
def test_hosvd_init_and_solves(name):
    x = _x(name)
    ranks = [int(r) for r in G[f"{name}_ranks"]]
    sweeps, seed = int(G[f"{name}_sweeps"]), int(G[f"{name}_seed"])
    fs = hq.init_factors(x, hq.SolverConfig(ranks=ranks, seed=seed, init=hq.INIT_HOSVD))
    for m in range(x.order()):
        assert _subspace(fs.factors[m], G[f"{name}_hosvd{m}"]) <= 1e-8
    for tag, solve, init, traced in (("hoqri_hosvd", hq.hoqri, hq.INIT_HOSVD, False),
                                     ("hooi_rand", hq.hooi, hq.INIT_RANDOM, True),
                                     ("hooi_hosvd", hq.hooi, hq.INIT_HOSVD, False)):
        cfg = hq.SolverConfig(ranks=ranks, max_sweeps=sweeps, tol_fit_change=0.0, seed=seed, init=init,
                              trace_gradients=traced)
        r = solve(x, cfg)
        assert len(r.trace.sweeps) == int(G[f"{name}_{tag}_sweeps"]), tag
        obj = np.array([s.objective for s in r.trace.sweeps])
        np.testing.assert_allclose(obj, G[f"{name}_{tag}_objective"], rtol=1e-9, err_msg=tag)
        np.testing.assert_allclose(r.trace.initial_objective, float(G[f"{name}_{tag}_initial_objective"]),
                                   rtol=1e-9)
        dr = np.array([s.drift for s in r.trace.sweeps]).reshape(-1)
        np.testing.assert_allclose(dr, G[f"{name}_{tag}_drift"], atol=1e-8, err_msg=tag)
        if traced:
            gr = np.array([s.grad_norm_sq for s in r.trace.sweeps]).reshape(-1)
            scale = max(1.0, 4 * float(np.max(obj)))
            assert np.abs(gr - G[f"{name}_{tag}_grad"]).max() <= 1e-9 * scale, tag
            assert len(r.trace.updates) == len(gr)
        for m in range(x.order()):
            assert _subspace(r.model.factors.factors[m], G[f"{name}_{tag}_U{m}"]) <= 1e-7, (tag, m)
        assert r.model.factors.orthonormality_defect() <= 1e-10


def test_planted_recovery_and_capacity():
    x = _x("pl")
    fs = hq.init_factors(x, hq.SolverConfig(ranks=[2, 2, 2], init=hq.INIT_HOSVD))
    g = hq.ttmc_core(x, fs)
    assert hq.norm_sq(x) - float(np.sum(g.data ** 2)) <= 1e-10 * hq.norm_sq(x)  # solvers_test.cpp:71-79
    xc = hq.SparseTensor([40, 40, 40], G["cap_coords"], G["cap_vals"])
    with pytest.raises(hq.CapacityError) as e:
        hq.init_factors(xc, hq.SolverConfig(ranks=[2, 2, 2], init=hq.INIT_HOSVD, capacity_cap=1000))
    assert str(e.value) == str(G["cap_message"])
    with pytest.raises(hq.CapacityError):
        hq.hooi(xc, hq.SolverConfig(ranks=[2, 2, 2], capacity_cap=3))


def test_hooi_degenerate():
    x = hq.SparseTensor([3, 3, 3], np.array([[1, 1, 1]], np.uint32), np.array([0.0]))
    with pytest.raises(hq.DegenerateStateError) as e:
        hq.hooi(x, hq.SolverConfig(ranks=[1, 1, 1], max_sweeps=5))
    assert e.value.mode == 1


@pytest.mark.parametrize("n", [1, 3, 10, 40])
def test_sym_eig(n):
    """jacobi_eig_sym contract (dense_core.cpp:200-262): the symmetrised input's eigenpairs, descending."""
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, n))
    m = b @ b.T + 1e-13 * rng.standard_normal((n, n))  # slightly asymmetric: the call symmetrises
    vals, vecs = hq.jacobi_eig_sym(m)
    ms = 0.5 * (m + m.T)
    ref = np.linalg.eigvalsh(ms)[::-1]
    scale = max(1.0, float(np.abs(ref).max()))
    assert np.all(np.diff(vals) <= 0)
    assert np.abs(vals - ref).max() <= 1e-12 * scale
    assert np.abs(ms @ vecs - vecs * vals).max() <= 1e-11 * scale
    assert np.abs(vecs.T @ vecs - np.eye(n)).max() <= 1e-12
