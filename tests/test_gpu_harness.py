"""GPU: the harness surface on the device engine -- run_experiment writes the
reference's trace/summary schema with the same numbers the reference's run
records (tests/golden/trace.npz), bench_kernel times device TTMcTC calls."""
import io
import json
import os

import numpy as np
import pytest

import paper_2510_16930_b200 as hq
from paper_2510_16930_b200 import harness
from conftest import golden

pytestmark = pytest.mark.gpu


def test_run_experiment_trace_matches_reference(tmp_path):
    g = golden("trace.npz")
    ref = harness.read_trace_csv(io.StringIO(str(g["csv"])))
    spec = harness.ExperimentSpec(
        config=hq.SolverConfig(ranks=[int(k) for k in g["ranks"]], max_sweeps=int(g["sweeps"]), tol_fit_change=0.0,
                               seed=int(g["seed"])),
        out_dir=str(tmp_path), synthetic=harness.SyntheticSpec([int(d) for d in g["dims"]], int(g["nnz"]),
                                                               int(g["tensor_seed"])), repetitions=2)
    res = harness.run_experiment(spec)
    assert len(res.trace_paths) == 2 and os.path.exists(res.summary_path)
    t = harness.read_trace_csv(open(res.trace_paths[0]))
    tj = harness.read_trace_json(open(res.trace_paths[0][:-4] + ".json"))
    assert t.columns == ref.columns and list(t.header) == list(ref.header)
    assert tj.columns == t.columns and tj.header == t.header
    for k in ref.header:
        if k in ("data_norm_sq", "initial_objective"):  # device reductions: same value to rounding
            assert abs(float(t.header[k]) - float(ref.header[k])) <= 1e-12 * abs(float(ref.header[k])), k
        elif k != "timestamp":
            assert t.header[k] == ref.header[k], k
    a, r = np.array(t.rows), np.array(ref.rows)
    assert a.shape == r.shape
    np.testing.assert_array_equal(a[:, 0], r[:, 0])
    np.testing.assert_allclose(a[:, 2:4], r[:, 2:4], rtol=1e-9)       # objective, fit
    np.testing.assert_allclose(a[:, 5:], r[:, 5:], rtol=1e-7, atol=1e-10)  # drifts
    assert (np.diff(a[:, 1]) >= 0).all() and a[0, 1] > 0               # device elapsed_s
    s = json.load(open(res.summary_path))
    assert s["repetitions"] == 2 and len(s["hoqri"]["runs"]) == 2 and s["nnz"] == int(g["nnz"])
    t1 = harness.read_trace_csv(open(res.trace_paths[1]))
    assert t1.header["seed"] == str(int(g["seed"]) + 1)  # repetition r uses seed + r


def test_bench_kernel_device_timing():
    x = hq.gen_synthetic([2000, 1500, 1000], 50000, 3)
    u = hq.random_factors(x.dims(), [10, 10, 10], 4)
    for mode in range(3):
        st = harness.bench_kernel(x, u, mode, 0, 7)
        assert st.repetitions == 7 and 0 < st.min_s <= st.median_s <= st.max_s < 1.0
        assert st.peak_slots >= x.dims()[mode] * 10 and st.largest_alloc_slots <= st.peak_slots


def test_harness_errors(tmp_path):
    cfg = hq.SolverConfig(ranks=[2, 2])
    res = harness.run_experiment(harness.ExperimentSpec(hq.SolverConfig(ranks=[2, 2], max_sweeps=3), str(tmp_path),
                                                        synthetic=harness.SyntheticSpec([5, 5], 12, 1),
                                                        solver=harness.SOLVER_BOTH))
    assert [p.rsplit("/", 1)[-1] for p in res.trace_paths] == ["hoqri_rep0.trace.csv", "hooi_rep0.trace.csv"]
    s = json.load(open(res.summary_path))
    assert "hoqri" in s and "hooi" in s
    with pytest.raises(hq.ShapeError):
        harness.run_experiment(harness.ExperimentSpec(cfg, str(tmp_path), synthetic=harness.SyntheticSpec([5, 5], 5, 1),
                                                      solver="svd"))
    with pytest.raises(hq.ShapeError):
        harness.run_experiment(harness.ExperimentSpec(cfg, str(tmp_path)))
    with pytest.raises(hq.InfeasibleError):
        harness.run_experiment(harness.ExperimentSpec(cfg, str(tmp_path), synthetic=harness.SyntheticSpec([2, 2], 9, 1)))
