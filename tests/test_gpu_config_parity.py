"""GPU parity on the BENCHMARKED configurations (north_star: "results must
match the reference on the same seeded inputs and the same seeded initial
factors").

Fixtures: tests/golden/cfg{C}_s{SEED}.npz, written by oracle/gen_config_traces.py
from the UNMODIFIED reference (oracle/_ref) on the exact COO arrays
paper_2510_16930_b200/workloads.py generates (hashes checked here first) and
the reference's seeded initial factors (tucker::random_factors).  Per sweep
they hold the core, f = ||G||^2, the fit, the per-mode drift and a
fingerprint of every factor (tests/sketch.py).

Bars (north_star; SURVEY 8(c) parity contract):
  core        ||G_gpu - G_ref||_F / ||G_ref||_F   <= 1e-9
  f           relative                             <= 1e-9
  fit         |dfit| / max(|fit|, f)               <= 1e-9   (fit = ||X||^2 - f)
  drift       absolute                             <= 1e-10
  subspaces   ||U_g U_g^T - U_r U_r^T||_F <= 2 ||U_g - U_r||_F, estimated
              from the 256-column sketch (within ~10 %)  -> bound <= 1e-8
  sampled rows of U (128 per factor)               <= 1e-8 abs
Ill-conditioned sweeps.  Where a sweep's TTMcTC outputs are ill-conditioned
(kappa(A) ~ 1e9 and beyond: config 2 from seed 1 reaches the shifted and
rank-deficient regimes), every QR -- the reference's included -- determines
the factor subspace only to ~u kappa(A), and no implementation can hold the
1e-8 bar there.  The yardstick is then the reference's OWN rounding spread:
tests/golden/cfg{C}_s{SEED}_matrix.npz is the same trajectory run with the
reference's other kernel (ttmctc_matrix: same math, different summation
order).  A sweep passes when the engine's deviation from the element-wise
reference is within the north_star bar OR within 10x the reference's
element-wise-vs-matrix spread on that sweep; the test prints both.
config 5 (N = 4, 2e8 nonzeros; ~2-3 h per reference sweep) is checked as
single calls: ttmc_core at the seeded factors and one TTMcTC per mode with
that core, ||dA||_F / ||A||_F <= 1e-11.
"""
import hashlib
import os

import numpy as np
import pytest

import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import CONFIGS, config_coo
from sketch import sample_rows, sketch_torch

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BAR_CORE, BAR_F, BAR_DRIFT, BAR_SUB, BAR_ROWS = 1e-9, 1e-9, 1e-10, 1e-8, 1e-8


def _fixtures(kind):
    out = []
    for name in sorted(os.listdir(GOLDEN)):
        if not (name.startswith("cfg") and name.endswith(".npz")) or "_matrix" in name:
            continue
        z = np.load(os.path.join(GOLDEN, name))
        if int(z["config"]) == 1:
            continue  # config 1 is covered at full size by test_gpu_parity.py
        sweeps = int(z["done_sweeps"]) if "done_sweeps" in z else 0
        if kind == "trajectory" and sweeps > 0:
            out.append(name)
        if kind == "calls" and "done_modes" in z:
            out.append(name)
    return out


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _inputs(z):
    cfg = int(z["config"])
    coords, vals = config_coo(cfg)
    assert _sha(coords) == str(z["input_coords_sha"]), "generator drift: coordinates differ from the fixture's"
    assert _sha(vals) == str(z["input_vals_sha"]), "generator drift: values differ from the fixture's"
    dims = [int(d) for d in z["dims"]]
    ranks = [int(r) for r in z["ranks"]]
    x = hq.SparseTensor(dims, coords, vals)
    assert x.nnz() == int(z["nnz_merged"])
    # ||X||^2: the reference sums nnz squares sequentially (sparse_tensor.cpp:91-95) after merging duplicates in
    # std::sort's order; the device sums them in a fixed tree.  Both carry ~sqrt(nnz) u relative rounding.
    nnz = int(z["nnz_merged"])
    assert abs(hq.norm_sq(x) - float(z["norm_sq"])) <= 2.2e-16 * np.sqrt(nnz) * float(z["norm_sq"])
    return cfg, dims, ranks, x


def _factor_dev(u, z, n, key_sketch, key_rows, s, cache):
    """(sketch-estimated ||U_g - U_r||_F, max |row diff|) of factor n."""
    import torch
    ut = torch.from_numpy(np.ascontiguousarray(u)).cuda()
    sk = sketch_torch(ut, cache=cache)
    ref_sk = z[key_sketch] if s is None else z[key_sketch][s]
    ref_rows = z[key_rows] if s is None else z[key_rows][s]
    idx = z[f"rows_idx{n}"]
    assert (idx == sample_rows(u.shape[0])).all()
    return float(np.linalg.norm(sk - ref_sk)), float(np.abs(u[idx] - ref_rows).max())


@pytest.mark.parametrize("name", _fixtures("trajectory"))
def test_config_trajectory_matches_reference(name):
    z = np.load(os.path.join(GOLDEN, name))
    cfg, dims, ranks, x = _inputs(z)
    N = len(dims)
    seed = int(z["factor_seed"])
    S = int(z["done_sweeps"])
    u0 = hq.random_factors(dims, ranks, seed)
    cache = {}
    for n in range(N):  # the seeded initial factors: reference stream + device QR vs the reference's Householder
        d, r = _factor_dev(u0.factors[n], z, n, f"init_sketch{n}", f"init_rows{n}", None, cache)
        assert 2 * d <= BAR_SUB and r <= BAR_ROWS, (n, d, r)
    solver = hq.Solver(x, hq.SolverConfig(ranks=ranks, max_sweeps=S, tol_fit_change=0.0), init_factors=u0.factors)
    worst = dict(core=0.0, f=0.0, fit=0.0, drift=0.0, sub=0.0, rows=0.0)
    report = []
    for s in range(S):
        solver.run(1)
        solver.sync()
        res = solver.download()
        g = res.model.core.data.reshape(-1)
        gr = z["cores"][s].reshape(-1)
        e_core = float(np.linalg.norm(g - gr) / np.linalg.norm(gr))
        sw = res.trace.sweeps[s]
        e_f = abs(sw.objective - float(z["objective"][s])) / abs(float(z["objective"][s]))
        # fit = ||X||^2 - f (solvers.cpp:154-155): a 1e-9 relative error of f is 1e-9 f absolute in the fit,
        # which where f ~ ||X||^2 (configs 3-4) is many times the fit itself -- the fit is held to the bar on
        # the larger of |fit| and f
        e_fit = abs(sw.fit - float(z["fit"][s])) / max(abs(float(z["fit"][s])), abs(float(z["objective"][s])))
        e_drift = float(np.abs(np.asarray(sw.drift) - z["drift"][s]).max())
        e_sub, e_rows = 0.0, 0.0
        for n in range(N):
            d, r = _factor_dev(res.model.factors.factors[n], z, n, f"sketch{n}", f"rows{n}", s, cache)
            e_sub, e_rows = max(e_sub, 2 * d), max(e_rows, r)
        report.append((s + 1, e_core, e_f, e_fit, e_drift, e_sub, e_rows))
        for k, v in zip(("core", "f", "fit", "drift", "sub", "rows"), report[-1][1:]):
            worst[k] = max(worst[k], v)
    st = solver.status()
    spread = _reference_spread(name, z, S, N)
    print(f"\n{name}: status {st}")
    print("  per sweep: engine vs reference (element-wise)  |  reference element-wise vs matrix variant")
    bars = (BAR_CORE, BAR_F, BAR_F, BAR_DRIFT, BAR_SUB, BAR_ROWS)
    failures = []
    for i, r in enumerate(report):
        sp = spread[i] if i < len(spread) else None
        line = "  sweep %2d core %.2e f %.2e fit %.2e drift %.2e subspace<= %.2e rows %.2e" % r
        if sp is not None:
            line += "  | core %.2e f %.2e drift %.2e subspace<= %.2e" % (sp[0], sp[1], sp[3], sp[4])
        print(line)
        for j, (v, bar) in enumerate(zip(r[1:], bars)):
            limit = bar if sp is None or j == 5 else max(bar, 10.0 * sp[j])
            if v > limit:
                failures.append((r[0], ("core", "f", "fit", "drift", "subspace", "rows")[j], v, limit))
    assert not failures, failures


def _reference_spread(name, z, S, N):
    """Per sweep (core, f, fit, drift, subspace) distance between the element-wise reference trajectory and
    the reference's ttmctc_matrix trajectory from the same start (tests/golden/*_matrix.npz)."""
    path = os.path.join(GOLDEN, name.replace(".npz", "_matrix.npz"))
    if not os.path.exists(path):
        return []
    zm = np.load(path)
    out = []
    for s in range(min(S, int(zm["done_sweeps"]))):
        g, gm = z["cores"][s].reshape(-1), zm["cores"][s].reshape(-1)
        e_core = float(np.linalg.norm(g - gm) / np.linalg.norm(g))
        e_f = abs(float(z["objective"][s]) - float(zm["objective"][s])) / abs(float(z["objective"][s]))
        e_fit = abs(float(z["fit"][s]) - float(zm["fit"][s])) / max(abs(float(z["fit"][s])), abs(float(z["objective"][s])))
        e_drift = float(np.abs(z["drift"][s] - zm["drift"][s]).max())
        e_sub = max(2 * float(np.linalg.norm(z[f"sketch{n}"][s] - zm[f"sketch{n}"][s])) for n in range(N))
        out.append((e_core, e_f, e_fit, e_drift, e_sub))
    return out


@pytest.mark.parametrize("name", _fixtures("calls"))
def test_config_single_calls_match_reference(name):
    z = np.load(os.path.join(GOLDEN, name))
    cfg, dims, ranks, x = _inputs(z)
    u0 = hq.random_factors(dims, ranks, int(z["factor_seed"]))
    core = hq.ttmc_core(x, u0)
    gr = z["core0"].reshape(-1)
    e_core = float(np.linalg.norm(core.data.reshape(-1) - gr) / np.linalg.norm(gr))
    assert e_core <= 1e-11, e_core
    import torch
    cache = {}
    for n in range(int(z["done_modes"])):
        a = hq.ttmctc_elementwise(x, u0, n, hq.CoreTensor(ranks, gr.copy()))
        sk = sketch_torch(torch.from_numpy(np.ascontiguousarray(a)).cuda(), cache=cache)
        fro = float(z[f"A{n}_fro"])
        e_a = float(np.linalg.norm(sk - z[f"A{n}_sketch"])) / fro
        idx = z[f"A{n}_rows_idx"]
        e_rows = float(np.abs(a[idx] - z[f"A{n}_rows"]).max()) / float(np.abs(z[f"A{n}_rows"]).max())
        print(f"\n{name} mode {n}: ||dA||/||A|| ~ {e_a:.2e}, sampled rows {e_rows:.2e}")
        assert e_a <= 1e-11 and e_rows <= 1e-11, (n, e_a, e_rows)
