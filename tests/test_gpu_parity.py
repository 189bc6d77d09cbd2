"""GPU parity: the CUDA engine (through its C-ABI) against the reference's own
outputs (tests/golden, produced by the unmodified reference library) and the
C restatement oracle.  Bars:
  layout                      bit-exact coords / offsets / entries
  merged values               <= m * eps relative
  TTMcTC / core per call      1e-11 abs (kernels_test.cpp:82-90, acceptance.cpp:157-189)
  core / objective / fit      1e-9 relative per iteration (north_star)
  factor subspace             sqrt(2) ||U_g - U_r (U_r^T U_g)||_F <= 1e-8 (north_star)
  drift                       1e-10 abs
  run-to-run                  bitwise
"""
import hashlib

import numpy as np
import pytest

import paper_2510_16930_b200 as hq
from conftest import golden
from paper_2510_16930_b200.workloads import uniform_coo

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def subspace_gap(ug, ur):
    """sqrt(2) ||U_g - U_r (U_r^T U_g)||_F == ||U_g U_g^T - U_r U_r^T||_F for
    orthonormal bases, without the cancellation of 2K - 2||U_r^T U_g||_F^2."""
    d = ug - ur @ (ur.T @ ug)
    return float(np.sqrt(2.0) * np.linalg.norm(d))


# ------------------------------------------------------------------ layout --
def test_long_duplicate_runs():
    """Hot cells (runs far above the one-thread merge length) merge to the per-cell sum, deterministically,
    next to ordinary short runs; coordinates / order are the reference's (sorted, unique)."""
    rng = np.random.default_rng(5)
    dims = [50, 40, 30]
    hot = np.array([[3, 4, 5]] * 20000 + [[7, 1, 2]] * 300 + [[0, 0, 0]] * 129, np.uint32)
    rest = np.stack([rng.integers(0, d, 10000) for d in dims], 1).astype(np.uint32)
    coords = np.concatenate([hot, rest])
    perm = rng.permutation(len(coords))
    coords = coords[perm]
    vals = rng.standard_normal(len(coords))
    x = hq.SparseTensor(dims, coords, vals)
    uc, inv = np.unique(coords, axis=0, return_inverse=True)
    sums = np.zeros(len(uc))
    np.add.at(sums, inv.reshape(-1), vals)
    assert (x.coords() == uc).all()
    np.testing.assert_allclose(x.values(), sums, rtol=1e-12, atol=1e-12)
    y = hq.SparseTensor(dims, coords, vals)
    assert sha(y.values()) == sha(x.values())


@pytest.mark.parametrize("name", ["hand", "gs4", "gs2", "gs3", "dups"])
def test_layout_bit_exact(name):
    g = golden("tensors.npz")
    dims = [int(d) for d in g[f"{name}_dims"]]
    x = hq.SparseTensor(dims, g[f"{name}_in_coords"], g[f"{name}_in_vals"])
    assert x.nnz() == g[f"{name}_coords"].shape[0]
    assert (x.coords() == g[f"{name}_coords"]).all()
    np.testing.assert_allclose(x.values(), g[f"{name}_vals"], rtol=1e-14, atol=1e-15)
    for m in range(len(dims)):
        off, ent = x.mode_bucket(m)
        assert (off == g[f"{name}_off{m}"]).all()
        assert (ent == g[f"{name}_ent{m}"]).all()
    assert abs(hq.norm_sq(x) - float(g[f"{name}_norm_sq"])) <= 1e-13 * max(1.0, float(g[f"{name}_norm_sq"]))


def test_layout_config1_hashes():
    g = golden("config1.npz")
    dims = [int(d) for d in g["dims"]]
    coords, vals = uniform_coo(dims, int(g["draws"]), int(g["gen_seed"]))
    x = hq.SparseTensor(dims, coords, vals)
    assert x.nnz() == int(g["nnz"])
    assert sha(x.coords()) == str(g["coords_sha"])
    assert sha(x.values()) == str(g["vals_sha"])
    for m in range(3):
        off, ent = x.mode_bucket(m)
        assert sha(off) == str(g[f"off{m}_sha"]) and sha(ent) == str(g[f"ent{m}_sha"])


def test_layout_errors_and_edges():
    with pytest.raises(hq.RangeError, match="out of range for mode 2"):
        hq.SparseTensor([3, 3, 3], np.array([[0, 0, 0], [1, 3, 0]], np.uint32), np.array([1.0, 2.0]))
    with pytest.raises(hq.ValueError_, match="entry 1"):
        hq.SparseTensor([3, 3, 3], np.array([[0, 0, 0], [1, 1, 0]], np.uint32), np.array([1.0, np.inf]))
    with pytest.raises(hq.ShapeError):
        hq.SparseTensor([3, 0, 3], np.zeros((0, 3), np.uint32), np.zeros(0))
    e = hq.SparseTensor([2, 2, 2], np.zeros((0, 3), np.uint32), np.zeros(0))  # empty tensor
    assert e.nnz() == 0 and hq.norm_sq(e) == 0.0
    off, ent = e.mode_bucket(1)
    assert off.tolist() == [0, 0, 0] and ent.size == 0
    one = hq.load_tns("1 1 1 3.0\n")
    assert hq.norm_sq(one) == 9.0
    # 72-bit keys (4 modes x 18 bits): two-word radix sort path
    rng = np.random.default_rng(3)
    dims = [200000] * 4
    c = rng.integers(0, 200000, size=(5000, 4)).astype(np.uint32)
    c[100] = c[7]
    v = rng.random(5000)
    x = hq.SparseTensor(dims, c, v)
    order = np.lexsort(c.T[::-1])
    cs = c[order]
    keep = np.ones(len(cs), bool)
    keep[1:] = (cs[1:] != cs[:-1]).any(axis=1)
    assert (x.coords() == cs[keep]).all()


# ----------------------------------------------------------------- kernels --
def _kcase(g, name):
    dims = [int(d) for d in g[f"{name}_dims"]]
    ranks = [int(r) for r in g[f"{name}_ranks"]]
    x = hq.SparseTensor(dims, g[f"{name}_coords"], g[f"{name}_vals"])
    u = [g[f"{name}_U{m}"] for m in range(len(dims))]
    return dims, ranks, x, u


def test_kernels_against_reference():
    g = golden("kernels.npz")
    worst = 0.0
    for name in g["names"]:
        dims, ranks, x, u = _kcase(g, name)
        core = hq.ttmc_core(x, u)
        assert np.abs(core.data - g[f"{name}_core"].reshape(-1)).max() <= 1e-12
        ref_core = hq.CoreTensor(ranks, g[f"{name}_core"].reshape(-1).copy())
        for m in range(len(dims)):
            a = hq.ttmctc_elementwise(x, u, m, ref_core)
            worst = max(worst, np.abs(a - g[f"{name}_A{m}"]).max())
            am = hq.ttmctc_matrix(x, u, m)
            worst = max(worst, np.abs(am - g[f"{name}_Am{m}"]).max())
    assert worst <= 1e-11, worst


def test_precomputed_core_reproduces_internal_exactly():
    # kernels_test.cpp:192-203
    g = golden("kernels.npz")
    dims, ranks, x, u = _kcase(g, "k6x5x4")
    core = hq.ttmc_core(x, u)
    for m in range(3):
        a1 = hq.ttmctc_elementwise(x, u, m)
        a2 = hq.ttmctc_elementwise(x, u, m, core)
        assert np.abs(a1 - a2).max() == 0.0
    with pytest.raises(hq.ShapeError):
        hq.ttmctc_elementwise(x, u, 0, hq.CoreTensor([2, 2, 2], np.zeros(8)))
    with pytest.raises(hq.RangeError):
        hq.ttmctc_elementwise(x, u, 3)
    bad = [np.zeros((dims[0] + 1, 2))] + u[1:]
    with pytest.raises(hq.ShapeError):
        hq.ttmc_core(x, bad)


def test_kernel_kats():
    # kernels_test.cpp:34-45, 64-80, 100-116
    x = hq.SparseTensor([2, 2, 2], np.array([[0, 0, 0]], np.uint32), np.array([2.0]))
    e0 = np.array([[1.0], [0.0]])
    assert hq.ttmc_core(x, [e0, e0, e0]).data[0] == pytest.approx(2.0)
    eye = [np.eye(2)] * 3
    a = hq.ttmctc_elementwise(x, eye, 0)
    assert a[0, 0] == pytest.approx(4.0)
    assert np.abs(a).sum() - abs(a[0, 0]) == 0.0
    z = hq.SparseTensor([3, 3, 3], np.array([[1, 1, 1]], np.uint32), np.array([0.0]))
    u = hq.random_factors([3, 3, 3], [2, 2, 2], 9)
    assert np.abs(hq.ttmctc_elementwise(z, u, 1)).max() == 0.0
    assert np.abs(hq.ttmctc_matrix(z, u, 1)).max() == 0.0
    x = hq.SparseTensor([2, 2, 2], np.array([[1, 0, 1]], np.uint32), np.array([3.0]))
    c = np.array([[0.6], [0.8]])
    a = hq.ttmctc_matrix(x, [c, c, c], 0)
    y1 = 3.0 * 0.6 * 0.8
    assert a[0, 0] == pytest.approx(0.0)
    assert a[1, 0] == pytest.approx(y1 * (y1 * 0.8), rel=1e-13)


def test_kernel_determinism_and_long_rows():
    """Bitwise repeatability, and rows long enough for the segmented path."""
    rng = np.random.default_rng(11)
    dims = [3, 4000, 50]
    c = np.stack([rng.integers(0, d, 30000) for d in dims], axis=1).astype(np.uint32)
    v = rng.random(30000)
    x = hq.SparseTensor(dims, c, v)
    u = hq.random_factors(dims, [3, 4, 5], 7)
    from oracle_bind import Oracle
    o = Oracle()
    core = hq.ttmc_core(x, u)
    oc = o.ttmc_core(dims, [3, 4, 5], x.coords(), x.values(), u.factors)
    assert np.abs(core.data - oc.reshape(-1)).max() <= 1e-10 * np.abs(oc).max()
    for m in range(3):
        a1 = hq.ttmctc_elementwise(x, u, m, core)
        a2 = hq.ttmctc_elementwise(x, u, m, core)
        assert (a1 == a2).all()
        ao = o.ttmctc(dims, [3, 4, 5], x.coords(), x.values(), u.factors, m, core.data)
        assert np.abs(a1 - ao).max() <= 1e-10 * np.abs(ao).max()


# --------------------------------------------------------------------- QR --
def test_qr_against_reference():
    g = golden("qr.npz")
    for name in g["names"]:
        q = hq.qr_orthonormal(g[f"{name}_A"])
        assert np.abs(q - g[f"{name}_Q"]).max() <= 1e-12, name
        q2 = hq.qr_orthonormal(g[f"{name}_A"])
        assert (q == q2).all(), (name, float(np.abs(q - q2).max()), np.argwhere(q != q2)[:5].tolist())
    np.testing.assert_allclose(hq.qr_orthonormal(np.array([[3.0], [4.0]]))[:, 0], [0.6, 0.8], rtol=1e-14)
    with pytest.raises(hq.ShapeError):
        hq.qr_orthonormal(np.zeros((2, 3)))


def test_qr_large_cholqr2():
    from oracle_bind import Oracle
    o = Oracle()
    rng = np.random.default_rng(5)
    a = rng.standard_normal((200000, 10)) @ np.diag(np.logspace(0, 4, 10))
    q = hq.qr_orthonormal(a)
    r = o.qr(a)
    assert np.abs(q - r).max() <= 1e-10
    assert np.abs(q.T @ q - np.eye(10)).max() <= 1e-13


def test_random_factors_match_reference_init():
    g = golden("hoqri.npz")
    for name in g["names"]:
        if int(g[f"{name}_status"]):
            continue
        dims = [int(d) for d in g[f"{name}_dims"]]
        ranks = [int(r) for r in g[f"{name}_ranks"]]
        u = hq.random_factors(dims, ranks, int(g[f"{name}_seed"]))
        for m in range(len(dims)):
            assert np.abs(u.factors[m] - g[f"{name}_U0_{m}"]).max() <= 1e-12


def test_subspace_distance():
    rng = np.random.default_rng(1)
    u = hq.qr_orthonormal(rng.standard_normal((30, 4)))
    assert hq.subspace_distance(u, u) <= 1e-12
    from oracle_bind import Oracle
    v = hq.qr_orthonormal(rng.standard_normal((30, 4)))
    assert abs(hq.subspace_distance(u, v) - Oracle().subspace_distance(u, v)) <= 1e-12


# ------------------------------------------------------------------ HOQRI --
def _hcase(g, name):
    dims = [int(d) for d in g[f"{name}_dims"]]
    ranks = [int(r) for r in g[f"{name}_ranks"]]
    x = hq.SparseTensor(dims, g[f"{name}_coords"], g[f"{name}_vals"])
    return dims, ranks, x


@pytest.mark.parametrize("name", ["h3", "h4", "h2", "h50"])
def test_hoqri_per_iteration_parity(name):
    g = golden("hoqri.npz")
    dims, ranks, x = _hcase(g, name)
    sweeps = int(g[f"{name}_sweeps"])
    u0 = [g[f"{name}_U0_{m}"] for m in range(len(dims))]
    csnap = g[f"{name}_core_snap"]
    # per-iteration: the core and factors after sweep s, from the same start
    for s in sorted({1, 2, 3, sweeps // 2, sweeps}):
        cfg = hq.SolverConfig(ranks=ranks, max_sweeps=s, tol_fit_change=0.0)
        r = hq.hoqri(x, cfg, init_factors=u0)
        assert len(r.trace.sweeps) == s
        ref_core = csnap[s - 1].reshape(-1)
        rel = np.linalg.norm(r.model.core.data - ref_core) / np.linalg.norm(ref_core)
        assert rel <= 1e-9, (s, rel)
        for m in range(len(dims)):
            assert subspace_gap(r.model.factors.factors[m], g[f"{name}_Usnap{m}"][s - 1]) <= 1e-8
    # full trace from the seeded init (random_factors on the device path)
    cfg = hq.SolverConfig(ranks=ranks, max_sweeps=sweeps, tol_fit_change=0.0, seed=int(g[f"{name}_seed"]))
    r = hq.hoqri(x, cfg)
    obj = np.array([s.objective for s in r.trace.sweeps])
    fit = np.array([s.fit for s in r.trace.sweeps])
    drift = np.array([s.drift for s in r.trace.sweeps])
    np.testing.assert_allclose(obj, g[f"{name}_objective"], rtol=1e-9)
    np.testing.assert_allclose(fit, g[f"{name}_fit"], rtol=1e-9, atol=1e-9 * float(g[f"{name}_norm_sq"]))
    assert np.abs(drift - g[f"{name}_drift"]).max() <= 1e-10
    assert r.trace.initial_objective == pytest.approx(float(g[f"{name}_initial_objective"]), rel=1e-9)
    assert r.model.factors.orthonormality_defect() <= 1e-10
    # bitwise run-to-run determinism (solvers_test.cpp:295-310)
    r2 = hq.hoqri(x, cfg)
    assert [s.objective for s in r2.trace.sweeps] == list(obj)
    assert [s.drift for s in r2.trace.sweeps] == [list(d) for d in drift]
    assert (r2.model.core.data == r.model.core.data).all()


def test_hoqri_degenerate_mode():
    x = hq.SparseTensor([3, 3, 3], np.array([[1, 1, 1]], np.uint32), np.array([0.0]))
    with pytest.raises(hq.DegenerateStateError) as ei:
        hq.hoqri(x, hq.SolverConfig(ranks=[1, 1, 1], seed=1))
    assert ei.value.mode == 1


def test_hoqri_stop_rule_and_fit():
    g = golden("hoqri.npz")
    dims, ranks, x = _hcase(g, "h3")
    cfg = hq.SolverConfig(ranks=ranks, max_sweeps=200, tol_fit_change=1e-9, seed=5)
    r = hq.hoqri(x, cfg)
    fits = [s.fit for s in r.trace.sweeps]
    assert len(fits) < 200
    assert abs(fits[-1] - fits[-2]) < 1e-9
    assert all(abs(a - b) >= 1e-9 for a, b in zip([r.trace.data_norm_sq - r.trace.initial_objective] + fits[:-2],
                                                 fits[:-1]))
    fe = hq.fit_error(x, r.model)
    assert fe == pytest.approx(max(hq.norm_sq(x) - hq.norm_sq(r.model.core), 0.0), rel=1e-12)
    fresh = hq.ttmc_core(x, r.model.factors)
    assert np.abs(fresh.data - r.model.core.data).max() <= 1e-10


def test_hoqri_config1_full():
    """BASELINE config 1 at full size, 20 sweeps: trace and final state vs the
    reference (tests/golden/config1.npz)."""
    g = golden("config1.npz")
    dims = [int(d) for d in g["dims"]]
    ranks = [int(r) for r in g["ranks"]]
    coords, vals = uniform_coo(dims, int(g["draws"]), int(g["gen_seed"]))
    x = hq.SparseTensor(dims, coords, vals)
    cfg = hq.SolverConfig(ranks=ranks, max_sweeps=int(g["sweeps"]), tol_fit_change=0.0, seed=int(g["seed"]))
    r = hq.hoqri(x, cfg)
    obj = np.array([s.objective for s in r.trace.sweeps])
    np.testing.assert_allclose(obj, g["objective"], rtol=1e-9)
    np.testing.assert_allclose([s.fit for s in r.trace.sweeps], g["fit"], rtol=1e-9)
    assert np.abs(np.array([s.drift for s in r.trace.sweeps]) - g["drift"]).max() <= 1e-10
    rel = np.linalg.norm(r.model.core.data - g["core"].reshape(-1)) / np.linalg.norm(g["core"])
    assert rel <= 1e-9, rel
    for m in range(3):
        assert subspace_gap(r.model.factors.factors[m], g[f"U{m}"]) <= 1e-8


@pytest.mark.parametrize("name", ["g3", "g4", "gk", "gstop"])
def test_hoqri_gradient_trace_matches_reference(name):
    """trace_gradients / tol_grad on the device (solvers.cpp:126-150, 165-167):
    every ModeUpdateRecord and the gradient stop against tucker::hoqri."""
    g = golden("grad.npz")
    dims = [int(d) for d in g[f"{name}_dims"]]
    ranks = [int(r) for r in g[f"{name}_ranks"]]
    x = hq.SparseTensor(dims, g[f"{name}_coords"], g[f"{name}_vals"])
    tol_grad = float(g[f"{name}_tol_grad"])
    cfg = hq.SolverConfig(ranks=ranks, max_sweeps=int(g[f"{name}_max_sweeps"]), tol_fit_change=0.0,
                          seed=int(g[f"{name}_seed"]), trace_gradients=True, tol_grad=tol_grad)
    r = hq.hoqri(x, cfg)
    assert len(r.trace.sweeps) == int(g[f"{name}_sweeps"])
    ups = r.trace.updates
    assert len(ups) == int(g[f"{name}_updates"])
    gr = np.array([u.grad_norm_sq for u in ups])
    scale = max(1.0, float(np.max(g[f"{name}_f_before"])) * 4)
    assert np.abs(gr - g[f"{name}_grad"]).max() <= 1e-9 * scale
    np.testing.assert_allclose([u.f_before for u in ups], g[f"{name}_f_before"], rtol=1e-9)
    np.testing.assert_allclose([u.f_after for u in ups], g[f"{name}_f_after"], rtol=1e-9)
    for i, u in enumerate(ups):
        k = ranks[u.mode]
        assert u.sweep == i // len(dims) + 1 and u.mode == i % len(dims)
        np.testing.assert_allclose(u.sigma, g[f"{name}_sigma"][i][:k], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(u.lambda_, g[f"{name}_lambda_"][i][:k], rtol=1e-9, atol=1e-12)
        assert u.elapsed_s >= 0.0
    sw = np.array([s.grad_norm_sq for s in r.trace.sweeps]).reshape(-1)
    np.testing.assert_allclose(sw, gr, rtol=0, atol=0)
    np.testing.assert_allclose([s.objective for s in r.trace.sweeps], g[f"{name}_objective"], rtol=1e-9)


def test_cached_device_memory_is_reused_and_released():
    """Device buffers of a destroyed tensor stay on the engine's free lists (no driver allocation for the next
    tensor of the same shape) until hq_release_cached_memory hands them back."""
    import torch
    from paper_2510_16930_b200.workloads import uniform_coo
    dims = [3000, 2500, 2000]
    coords, vals = uniform_coo(dims, 200000, 3)
    hq.release_cached_memory()
    x = hq.SparseTensor(dims, coords, vals)
    n1 = hq.norm_sq(x)
    del x
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    x = hq.SparseTensor(dims, coords, vals)  # same sizes: served from the free lists
    assert hq.norm_sq(x) == n1
    assert torch.cuda.mem_get_info()[0] == free0, "the second build allocated from the driver"
    del x
    freed = hq.release_cached_memory()
    assert freed >= coords.nbytes + vals.nbytes
    assert torch.cuda.mem_get_info()[0] >= free0 + freed // 2
    assert hq.release_cached_memory() == 0
