"""The reference's experiment / trace surface (proj/include/tucker/harness.hpp,
proj/src/harness.cpp) over the B200 engine.

Same trace schema (header keys, columns ``sweep, elapsed_s, objective, fit,
grad_norm_sq, drift_1..drift_N``, ``%.17g`` cells), same file layout
(``<out>/hoqri_rep<r>.trace.csv`` + ``.trace.json`` + ``summary.json``) and
the same exceptions, so plots and tests written for the reference consume GPU
runs unchanged.  What differs is the clock: ``elapsed_s`` is device time of
the solve, and :func:`bench_kernel` times each TTMcTC call with CUDA events on
a resident state (harness.cpp:350-381 times host calls).
"""
from __future__ import annotations

import dataclasses
import io
import json
import os
import time
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import (CapacityError, InfeasibleError, IterationTrace, ParseError, SolverConfig, ShapeError, SparseTensor,
               _check, _factors_of, _check_factors, _ptr_array, gen_synthetic, hooi, hoqri, load_library, load_tns)

K_TOOL_VERSION = "0.1.0"  # harness.hpp:15-16
K_TRACE_VERSION = 1
SOLVER_HOQRI, SOLVER_HOOI, SOLVER_BOTH = "hoqri", "hooi", "both"


def _fmt(v: float) -> str:  # harness.cpp:27-31 ("%.17g")
    return "%.17g" % v


@dataclasses.dataclass
class TraceFile:
    """harness.hpp:33-38"""
    header: Dict[str, str]
    columns: List[str]
    rows: List[List[float]]


def make_trace_file(solver_name: str, config: SolverConfig, x: SparseTensor, trace: IterationTrace) -> TraceFile:
    """harness.cpp:101-140: same keys and columns."""
    h = {
        "trace_version": str(K_TRACE_VERSION),
        "tool_version": K_TOOL_VERSION,
        "timestamp": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
        "solver": solver_name,
        "dims": ",".join(str(int(d)) for d in x.dims()),
        "nnz": str(int(x.nnz())),
        "ranks": ",".join(str(int(k)) for k in config.ranks),
        "seed": str(int(config.seed)),
        "init": "random" if int(config.init) != 1 else "hosvd",
        "kernel": "elementwise" if int(config.kernel) == 0 else "matrix",
        "max_sweeps": str(int(config.max_sweeps)),
        "tol": _fmt(float(config.tol_fit_change)),
        "data_norm_sq": _fmt(trace.data_norm_sq),
        "initial_objective": _fmt(trace.initial_objective),
    }
    cols = ["sweep", "elapsed_s", "objective", "fit", "grad_norm_sq"] + [f"drift_{n + 1}" for n in range(x.order())]
    rows = [[float(r.sweep), r.elapsed_s, r.objective, r.fit, r.total_grad_norm_sq] + [float(d) for d in r.drift]
            for r in trace.sweeps]
    return TraceFile(dict(sorted(h.items())), cols, rows)


def write_trace_csv(out, t: TraceFile) -> None:
    """harness.cpp:142-153"""
    lines = [f"# {k}={v}" for k, v in sorted(t.header.items())]
    lines.append(",".join(t.columns))
    lines += [",".join(_fmt(v) for v in row) for row in t.rows]
    out.write("\n".join(lines) + "\n")


def write_trace_json(out, t: TraceFile) -> None:
    """harness.cpp:155-161 (keys sorted, two-space indent)"""
    doc = {"columns": t.columns, "header": dict(sorted(t.header.items())),
           "rows": [[None if not np.isfinite(v) else float(v) for v in row] for row in t.rows]}
    out.write(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def read_trace_csv(src) -> TraceFile:
    """harness.cpp:163-199: same parse rules; ParseError carries the line."""
    text = src.read() if hasattr(src, "read") else src
    header, columns, rows = {}, None, []
    for line_no, line in enumerate(text.split("\n"), start=1):
        if not line:
            continue
        if line[0] == "#":
            body = line[1:].lstrip(" \t")
            if not body or "=" not in body:
                continue
            k, v = body.split("=", 1)
            header[k] = v
            continue
        cells = line.split(",")
        if columns is None:
            columns = cells
            continue
        row = []
        for cell in cells:
            try:
                if cell != cell.strip() or cell == "" or cell.lower() in ("infinity", "+inf", "+nan"):
                    raise ValueError
                row.append(float(cell))
            except ValueError:
                raise ParseError(f"bad numeric cell '{cell}'", line_no) from None
        if len(row) != len(columns):
            raise ParseError("row width does not match the column header", line_no)
        rows.append(row)
    if columns is None:
        raise ParseError("trace has no column header")
    return TraceFile(header, columns, rows)


def read_trace_json(src) -> TraceFile:
    """harness.cpp:201-209"""
    text = src.read() if hasattr(src, "read") else src
    try:
        j = json.loads(text)
        return TraceFile({str(k): str(v) for k, v in j["header"].items()}, [str(c) for c in j["columns"]],
                         [[float("nan") if v is None else float(v) for v in row] for row in j["rows"]])
    except (KeyError, TypeError, ValueError) as e:
        raise ParseError(f"trace json: {e}") from None


@dataclasses.dataclass
class SyntheticSpec:
    dims: Sequence[int]
    nnz: int = 0
    seed: int = 0


@dataclasses.dataclass
class ExperimentSpec:
    """harness.hpp:50-60"""
    config: SolverConfig
    out_dir: str
    input_path: Optional[str] = None
    synthetic: Optional[SyntheticSpec] = None
    dims_override: Optional[Sequence[int]] = None
    solver: str = SOLVER_HOQRI
    repetitions: int = 1
    parallel_reps: bool = False  # accepted; repetitions share one GPU and run in order


@dataclasses.dataclass
class ExperimentResult:
    trace_paths: List[str]
    summary_path: str


def run_experiment(spec: ExperimentSpec) -> ExperimentResult:
    """harness.cpp:241-345, HOQRI on the device."""
    if spec.repetitions < 1:
        raise ShapeError("repetitions must be at least 1")
    if (spec.input_path is None) == (spec.synthetic is None):
        raise ShapeError("specify exactly one input source (file or synthetic)")
    if not spec.out_dir:
        raise ShapeError("output directory required")
    if spec.solver not in (SOLVER_HOQRI, SOLVER_HOOI, SOLVER_BOTH):
        raise ShapeError(f"unknown solver choice {spec.solver!r}")
    if spec.input_path is not None:
        x = load_tns(spec.input_path, spec.dims_override)
    else:
        s = spec.synthetic
        total = 1
        for d in s.dims:
            total *= int(d)
        if s.nnz > 0 and s.nnz > total:
            raise InfeasibleError("synthetic nnz exceeds the number of cells")
        x = gen_synthetic(s.dims, s.nnz, s.seed)
    os.makedirs(spec.out_dir, exist_ok=True)
    chosen = [("hoqri", hoqri)] if spec.solver == SOLVER_HOQRI else [("hooi", hooi)] if spec.solver == SOLVER_HOOI \
        else [("hoqri", hoqri), ("hooi", hooi)]
    paths = []
    summary = {"tool_version": K_TOOL_VERSION, "dims": [int(d) for d in x.dims()], "nnz": int(x.nnz()),
               "ranks": [int(k) for k in spec.config.ranks], "repetitions": spec.repetitions}
    for name, solve in chosen:
        runs = []
        for rep in range(spec.repetitions):  # repetitions share the GPU: in order
            cfg = dataclasses.replace(spec.config, seed=int(spec.config.seed) + rep)
            res = solve(x, cfg)
            t = make_trace_file(name, cfg, x, res.trace)
            base = os.path.join(spec.out_dir, f"{name}_rep{rep}")
            with open(base + ".trace.csv", "w") as f:
                write_trace_csv(f, t)
            with open(base + ".trace.json", "w") as f:
                write_trace_json(f, t)
            sw = res.trace.sweeps
            last = sw[-1] if sw else None
            runs.append({"rep": rep, "trace": base + ".trace.csv", "sweeps": len(sw),
                         "mean_sweep_s": last.elapsed_s / len(sw) if sw else 0.0,
                         "final_objective": last.objective if sw else 0.0, "final_fit": last.fit if sw else 0.0})
            paths.append(base + ".trace.csv")
        summary[name] = {"runs": runs, "mean_sweep_s": sum(r["mean_sweep_s"] for r in runs) / len(runs)}
    sp = os.path.join(spec.out_dir, "summary.json")
    with open(sp, "w") as f:
        f.write(json.dumps(summary, indent=2, sort_keys=True) + "\n")
    return ExperimentResult(paths, sp)


@dataclasses.dataclass
class BenchStats:
    """harness.hpp:71-78 (slots = 8-byte device scratch of one call)"""
    repetitions: int
    median_s: float
    min_s: float
    max_s: float
    peak_slots: int
    largest_alloc_slots: int


def bench_kernel(x: SparseTensor, u, mode: int, variant: int = 0, repetitions: int = 5) -> BenchStats:
    """harness.cpp:350-381 with CUDA-event timings of the device TTMcTC call."""
    if repetitions < 1:
        raise ShapeError("repetitions must be at least 1")
    fs = _factors_of(u)
    _check_factors(x, fs)
    ranks = np.array([f.shape[1] for f in fs], np.uint64)
    times = np.empty(repetitions, np.float64)
    scratch = np.zeros(2, np.uint64)
    _check(load_library().hq_bench_ttmctc(x.handle, _ptr_array(fs), ranks, int(mode), int(repetitions), times,
                                          scratch))
    t = np.sort(times)
    mid = len(t) // 2
    med = float(t[mid]) if len(t) % 2 else 0.5 * float(t[mid - 1] + t[mid])
    return BenchStats(repetitions, med, float(t[0]), float(t[-1]), int((scratch[0] + 7) // 8),
                      int((scratch[1] + 7) // 8))
