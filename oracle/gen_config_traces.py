"""Reference trajectories on the BASELINE configs (parity fixtures for N1).

TEST INFRASTRUCTURE ONLY.  Runs the UNMODIFIED reference library
(oracle/_ref/libtucker_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile) on the exact inputs bench.py and the GPU tests generate
(paper_2510_16930_b200/workloads.py: seeded PCG64 COO, duplicates merged by
the reference's own SparseTensor constructor) and the reference's own seeded
initial factors (tucker::random_factors, solvers.cpp:182-195).  It records,
per sweep, what the reference's solve loop (solvers.cpp:50-178, element-wise
kernel with the core kept fresh, :90-91 / :143-144) produces:

* the core G (full, K^N doubles), f = ||G||^2 and fit = ||X||^2 - f
  (solvers.cpp:154-155);
* the per-mode drift (subspace_distance, manifold.cpp:55-60);
* a fingerprint of every factor (tests/sketch.py: a 256-column Rademacher
  sketch + 128 sampled rows) -- the factors themselves are 10^5-10^6 rows.

The sweeps are run with ``ref_hoqri_replay`` one sweep at a time (the same
reference calls, in the same order, as tucker::hoqri's loop: ttmctc_elementwise
with the fresh core, max_abs, qr_orthonormal, subspace_distance, ttmc_core).

config 5 (2e8 nonzeros, N = 4; ~2-3 h per reference sweep) records single
calls instead: the core at the seeded initial factors (ttmc_core) and one
TTMcTC per mode with that core (kernels.cpp:86-163), as fingerprints.

With --variant matrix the same trajectory is run with the reference's other
kernel, ttmctc_matrix (ref_hoqri_replay_matrix; core once per sweep as
solvers.cpp does for that variant): it differs from the element-wise run only
in floating-point summation order, so the spread between the two fixtures is
the reference's own rounding sensitivity on that input -- the yardstick the
GPU tests hold the engine's deviation against on ill-conditioned sweeps.

Usage:  python oracle/gen_config_traces.py CONFIG FACTOR_SEED SWEEPS [--keep DIR] [--variant matrix]
Writes tests/golden/cfg{C}_s{SEED}.npz (rewritten after every sweep, so a
partial run is usable; ``done_sweeps`` says how far it got).
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from oracle_bind import RefLib, RefTensor, ref_random_factors  # noqa: E402
from sketch import fingerprint  # noqa: E402
from paper_2510_16930_b200.workloads import CONFIGS, config_coo  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("seed", type=int)
    ap.add_argument("sweeps", type=int)
    ap.add_argument("--keep", default=None, help="also save full factors per sweep here (local analysis)")
    ap.add_argument("--variant", default="elementwise", choices=["elementwise", "matrix"],
                    help="matrix: the reference's ttmctc_matrix trajectory (its own rounding spread)")
    a = ap.parse_args()
    c = CONFIGS[a.config]
    dims, ranks = list(c["dims"]), list(c["ranks"])
    N = len(dims)
    t0 = time.time()
    coords, vals = config_coo(a.config)
    t_gen = time.time() - t0
    lib = RefLib()
    t0 = time.time()
    x = RefTensor.create(lib, dims, coords, vals)
    t_build = time.time() - t0
    out = dict(config=np.array(a.config), factor_seed=np.array(a.seed, np.uint64),
               tensor_seed=np.array(1000 + a.config), dims=np.asarray(dims, np.uint64),
               ranks=np.asarray(ranks, np.uint64), nnz_merged=np.array(x.nnz),
               input_coords_sha=np.array(sha(coords)), input_vals_sha=np.array(sha(vals)),
               norm_sq=np.array(x.norm_sq()), t_build_s=np.array(t_build),
               source=np.array("oracle/_ref (unmodified reference): SparseTensor ctor, random_factors, "
                               "ttmc_core, ttmctc_elementwise, qr_orthonormal, subspace_distance "
                               "(solvers.cpp:50-178 loop via ref_hoqri_replay)"))
    del coords, vals
    name = os.path.join(OUT, f"cfg{a.config}_s{a.seed}" + ("_matrix" if a.variant == "matrix" else "") + ".npz")
    out["variant"] = np.array(a.variant)
    print(f"cfg{a.config} seed {a.seed}: gen {t_gen:.1f}s build {t_build:.1f}s nnz {x.nnz}", flush=True)

    u = ref_random_factors(lib, dims, ranks, a.seed)
    fp = [fingerprint(f) for f in u]
    for n in range(N):
        out[f"init_sketch{n}"], out[f"rows_idx{n}"], out[f"init_rows{n}"] = fp[n]
    t0 = time.time()
    core0 = x.ttmc_core(ranks, u)
    out["t_core_s"] = np.array(time.time() - t0)
    out["core0"] = core0
    out["objective0"] = np.array(float(np.add.accumulate((core0 * core0).ravel())[-1]))

    if a.sweeps == 0:  # single calls (config 5)
        tt = []
        for n in range(N):
            t0 = time.time()
            an = x.ttmctc(ranks, u, n, core0)
            tt.append(time.time() - t0)
            out[f"A{n}_sketch"], _, out[f"A{n}_rows"] = fingerprint(an)
            out[f"A{n}_rows_idx"] = fp[n][1]
            out[f"A{n}_fro"] = np.array(float(np.sqrt((an * an).sum())))
            out["t_ttmctc_s"] = np.asarray(tt)
            out["done_modes"] = np.array(n + 1)
            np.savez_compressed(name, **out)
            print(f"  mode {n}: ttmctc {tt[-1]:.1f}s", flush=True)
        return

    S = a.sweeps
    cores = np.zeros((S,) + tuple(ranks))
    obj, fit = np.zeros(S), np.zeros(S)
    drift = np.zeros((S, N))
    sk = [np.zeros((S,) + fp[n][0].shape) for n in range(N)]
    rw = [np.zeros((S,) + fp[n][2].shape) for n in range(N)]
    t_sweep = np.zeros(S)
    for s in range(S):
        t0 = time.time()
        cs, fs, dr = x.replay(ranks, u, 1, a.variant)
        t_sweep[s] = time.time() - t0
        u = fs[0]
        cores[s] = cs[0]
        obj[s] = float(np.add.accumulate((cs[0] * cs[0]).ravel())[-1])  # sequential, as norm_sq (dense_core.cpp:110-114)
        fit[s] = float(out["norm_sq"]) - obj[s]
        drift[s] = dr[0]
        for n in range(N):
            sk[n][s], _, rw[n][s] = fingerprint(u[n])
            if a.keep:
                os.makedirs(a.keep, exist_ok=True)
                np.save(os.path.join(a.keep, f"cfg{a.config}_s{a.seed}_sweep{s + 1}_U{n}.npy"), u[n])
        out.update(cores=cores[:s + 1], objective=obj[:s + 1], fit=fit[:s + 1], drift=drift[:s + 1],
                   t_sweep_s=t_sweep[:s + 1], done_sweeps=np.array(s + 1))
        for n in range(N):
            out[f"sketch{n}"] = sk[n][:s + 1]
            out[f"rows{n}"] = rw[n][:s + 1]
        np.savez_compressed(name, **out)
        print(f"  sweep {s + 1}: {t_sweep[s]:.1f}s f {obj[s]:.15g} drift {drift[s]}", flush=True)


if __name__ == "__main__":
    main()
