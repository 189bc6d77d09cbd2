"""CPU: the harness surface (harness.hpp) -- gen_synthetic's stream and the
trace file schema -- against the reference (tests/golden/trace.npz,
hoqri.npz; oracle/gen_golden.py)."""
import io
import json

import numpy as np
import pytest

import paper_2510_16930_b200 as hq
from paper_2510_16930_b200 import harness
from conftest import golden


@pytest.mark.parametrize("name", ["h3", "h4", "h2", "h50"])
def test_gen_synthetic_matches_reference_stream(name):
    """hq_gen_synthetic (host) reproduces tucker::gen_synthetic bit for bit
    (the golden tensors were drawn by the reference's gen_synthetic)."""
    g = golden("hoqri.npz")
    spec = {"h3": ([20, 18, 16], 200, 41), "h4": ([10, 9, 8, 7], 120, 44), "h2": ([12, 9], 40, 45),
            "h50": ([50, 50, 50], 500, 31)}[name]
    coords, vals = hq.gen_synthetic_coo(*spec)
    order = np.lexsort(coords.T[::-1])
    np.testing.assert_array_equal(coords[order], g[f"{name}_coords"])
    np.testing.assert_array_equal(vals[order], g[f"{name}_vals"])


def test_gen_synthetic_errors():
    with pytest.raises(hq.InfeasibleError):
        hq.gen_synthetic_coo([2, 2], 5, 1)
    with pytest.raises(hq.ShapeError):
        hq.gen_synthetic_coo([3, 0], 1, 1)


def test_trace_csv_json_round_trip_reference_text():
    g = golden("trace.npz")
    ref_csv, ref_json = str(g["csv"]), str(g["json"])
    t = harness.read_trace_csv(io.StringIO(ref_csv))
    out = io.StringIO()
    harness.write_trace_csv(out, t)
    assert out.getvalue() == ref_csv  # byte-identical rendering (%.17g, sorted header)
    tj = harness.read_trace_json(io.StringIO(ref_json))
    assert tj.header == t.header and tj.columns == t.columns
    np.testing.assert_array_equal(np.array(tj.rows), np.array(t.rows))
    out = io.StringIO()
    harness.write_trace_json(out, t)
    assert json.loads(out.getvalue()) == json.loads(ref_json)


class _FakeTensor:
    def __init__(self, dims, nnz):
        self._d, self._n = dims, nnz

    def dims(self):
        return self._d

    def nnz(self):
        return self._n

    def order(self):
        return len(self._d)


def test_make_trace_file_schema_matches_reference():
    g = golden("trace.npz")
    ref = harness.read_trace_csv(io.StringIO(str(g["csv"])))
    cfg = hq.SolverConfig(ranks=[3, 3, 3], max_sweeps=6, tol_fit_change=0.0, seed=5)
    sweeps = [hq.SweepRecord(int(r[0]), r[1], r[2], r[3], r[4], [0.0, 0.0, 0.0], list(r[5:])) for r in ref.rows]
    tr = hq.IterationTrace(float(ref.header["data_norm_sq"]), float(ref.header["initial_objective"]), sweeps, [])
    t = harness.make_trace_file("hoqri", cfg, _FakeTensor([20, 18, 16], 200), tr)
    assert list(t.header) == list(ref.header) and t.columns == ref.columns
    for k in ref.header:
        if k != "timestamp":
            assert t.header[k] == ref.header[k], k
    np.testing.assert_array_equal(np.array(t.rows), np.array(ref.rows))


def test_read_trace_csv_errors():
    with pytest.raises(hq.ParseError) as e:
        harness.read_trace_csv("# a=1\nx,y\n1,2\n3,zz\n")
    assert e.value.line_number == 4
    with pytest.raises(hq.ParseError):
        harness.read_trace_csv("x,y\n1\n")
    with pytest.raises(hq.ParseError):
        harness.read_trace_csv("# only=header\n")
    with pytest.raises(hq.ParseError):
        harness.read_trace_json("{\"columns\": []}")
