"""Generate tests/golden/*.npz from the UNMODIFIED reference library.

TEST INFRASTRUCTURE ONLY.  Needs oracle/_ref/libtucker_ref.so (``make -C
oracle ref``), which is compiled from /root/reference/proj/src, so it runs in
the build container.  The fixtures it writes are committed; the GPU box and
the CPU test suite read only the fixtures.

Every fixture records the reference function that produced it.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from oracle_bind import RefLib, RefTensor, ref_qr, ref_random_factors, ref_svd_leading  # noqa: E402
from paper_2510_16930_b200.workloads import uniform_coo  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_rng(lib):
    raw = np.empty(10000, np.uint64)
    lib.L.ref_raw_stream(5489, 10000, raw)
    seeds = np.array([0, 7, 0x48514F5251, 2**63 + 11], np.uint64)
    normals = np.empty((len(seeds), 64))
    for i, s in enumerate(seeds):
        lib.L.ref_normal_stream(int(s), 64, normals[i])
    mix = np.array([[lib.L.ref_mix_seed(s, t) for t in range(5)] for s in (0, 1, 12345, 2**64 - 1)], np.uint64)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), raw_5489_first=raw[:16], raw_5489_10000=raw[-1:],
                        normal_seeds=seeds, normals=normals, mix_seed_args=np.array([0, 1, 12345, 2**64 - 1], np.uint64),
                        mix_seed=mix, source=np.array("tucker::Rng / mix_seed (rng.hpp:13-62)"))


def _tensor_case(lib, name, dims, coords, vals, out):
    t = RefTensor.create(lib, dims, coords, vals)
    c, v = t.export()
    out[f"{name}_dims"] = np.asarray(dims, np.uint64)
    out[f"{name}_in_coords"] = np.asarray(coords, np.uint32)
    out[f"{name}_in_vals"] = np.asarray(vals, np.float64)
    out[f"{name}_coords"] = c
    out[f"{name}_vals"] = v
    out[f"{name}_norm_sq"] = np.array(t.norm_sq())
    for m in range(len(dims)):
        off, ent = t.buckets(m)
        out[f"{name}_off{m}"] = off
        out[f"{name}_ent{m}"] = ent


def gen_tensors(lib):
    out = {}
    # hand case: 2- and 3-fold duplicates, an explicit zero, reversed order
    dims = [4, 5, 6]
    coords = np.array([[3, 4, 5], [0, 0, 0], [1, 2, 3], [0, 0, 0], [2, 2, 2], [1, 2, 3], [0, 0, 0], [3, 0, 1],
                       [2, 2, 2]], np.uint32)
    vals = np.array([1.5, 1.0, -2.0, 2.0, 0.25, 2.0, 0.125, 7.0, -0.25])
    _tensor_case(lib, "hand", dims, coords[::-1], vals[::-1], out)
    # gen_synthetic instances (distinct coords), fed back in reversed order
    for name, dims, nnz, seed in (("gs4", [7, 9, 4, 3], 50, 21), ("gs2", [12, 9], 40, 45), ("gs3", [6, 4, 5], 30, 3)):
        t = RefTensor.gen_synthetic(lib, dims, nnz, seed)
        c, v = t.export()
        _tensor_case(lib, name, dims, c[::-1].copy(), v[::-1].copy(), out)
    # heavy duplicates (multiplicities up to ~10): merged sums
    rng = np.random.Generator(np.random.PCG64(5))
    c = rng.integers(0, 5, size=(400, 3)).astype(np.uint32)
    v = rng.random(400)
    _tensor_case(lib, "dups", [5, 5, 5], c, v, out)
    np.savez_compressed(os.path.join(OUT, "tensors.npz"), **out)


def gen_kernels(lib):
    """Acceptance criterion-1 style instances (acceptance.cpp:157-189) plus the
    kernels_test.cpp KATs, with every kernel output from the reference."""
    out = {}
    meta = np.random.Generator(np.random.PCG64(20240101))
    cases = []
    for trial in range(24):
        order = [2, 3, 4][trial % 3]
        dims = [int(x) for x in meta.integers(2, 13, size=order)]
        ranks = [int(meta.integers(1, min(4, d) + 1)) for d in dims]
        cells = int(np.prod(dims))
        nnz = int(meta.integers(1, min(200, cells) + 1))
        cases.append((f"r{trial}", dims, ranks, nnz, int(meta.integers(1, 2**62)), int(meta.integers(1, 2**62))))
    cases.append(("k6x5x4", [6, 5, 4], [3, 2, 2], 30, 77, 8))
    cases.append(("k20", [20, 18, 16], [3, 3, 3], 200, 41, 5))
    cases.append(("k4d", [10, 9, 8, 7], [2, 3, 2, 2], 120, 44, 17))
    names = []
    for name, dims, ranks, nnz, tseed, fseed in cases:
        t = RefTensor.gen_synthetic(lib, dims, nnz, tseed)
        c, v = t.export()
        u = ref_random_factors(lib, dims, ranks, fseed)
        g = t.ttmc_core(ranks, u)
        out[f"{name}_dims"] = np.asarray(dims, np.uint64)
        out[f"{name}_ranks"] = np.asarray(ranks, np.uint64)
        out[f"{name}_coords"] = c
        out[f"{name}_vals"] = v
        out[f"{name}_core"] = g
        for m in range(len(dims)):
            out[f"{name}_U{m}"] = u[m]
            out[f"{name}_A{m}"] = t.ttmctc(ranks, u, m, g)          # ttmctc_elementwise(x,u,m,&g)
            out[f"{name}_Am{m}"] = t.ttmctc(ranks, u, m, None, 1)   # ttmctc_matrix
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


def gen_qr(lib):
    out = {}
    a = np.array([[3.0], [4.0]])
    out["k34_A"], out["k34_Q"] = a, ref_qr(lib, a)
    normals = np.empty(250)
    lib.L.ref_normal_stream(17, 250, normals)
    a = normals.reshape(50, 5).copy()
    out["r50x5_A"], out["r50x5_Q"] = a, ref_qr(lib, a)
    normals = np.empty(30)
    lib.L.ref_normal_stream(5, 30, normals)
    a = normals.reshape(10, 3).copy()
    a[:, 2] = a[:, 0] + a[:, 1]  # rank 2 (dense_core_test.cpp:80-98)
    out["def10x3_A"], out["def10x3_Q"] = a, ref_qr(lib, a)
    a = np.zeros((6, 2))
    a[:, 0] = 1.0  # second column zero -> seeded fill
    out["def6x2_A"], out["def6x2_Q"] = a, ref_qr(lib, a)
    normals = np.empty(64)
    lib.L.ref_normal_stream(99, 64, normals)
    a = normals.reshape(8, 8).copy()
    out["sq8_A"], out["sq8_Q"] = a, ref_qr(lib, a)
    out["names"] = np.array(["k34", "r50x5", "def10x3", "def6x2", "sq8"])
    np.savez_compressed(os.path.join(OUT, "qr.npz"), **out)


def _hoqri_case(lib, name, t, dims, ranks, sweeps, seed, out, snapshots=True):
    c, v = t.export()
    r = t.hoqri(ranks, sweeps, 0.0, seed)
    out[f"{name}_dims"] = np.asarray(dims, np.uint64)
    out[f"{name}_ranks"] = np.asarray(ranks, np.uint64)
    out[f"{name}_seed"] = np.array(seed, np.uint64)
    out[f"{name}_sweeps"] = np.array(sweeps)
    out[f"{name}_status"] = np.array(r["status"])
    out[f"{name}_payload"] = np.array(r["payload"])
    if r["status"]:
        out[f"{name}_coords"], out[f"{name}_vals"] = c, v
        return
    u0 = ref_random_factors(lib, dims, ranks, seed)
    out[f"{name}_norm_sq"] = np.array(t.norm_sq())
    out[f"{name}_initial_objective"] = np.array(r["initial_objective"])
    out[f"{name}_objective"] = r["objective"]
    out[f"{name}_fit"] = r["fit"]
    out[f"{name}_drift"] = r["drift"]
    out[f"{name}_core"] = r["core"]
    for m in range(len(dims)):
        out[f"{name}_U0_{m}"] = u0[m]
        out[f"{name}_U{m}"] = r["factors"][m]
    if snapshots:
        out[f"{name}_coords"], out[f"{name}_vals"] = c, v
        cs, fs, dr = t.replay(ranks, u0, sweeps)
        out[f"{name}_core_snap"] = cs
        for m in range(len(dims)):
            out[f"{name}_Usnap{m}"] = np.stack([f[m] for f in fs])


def gen_hoqri(lib):
    out = {}
    names = []
    for name, dims, nnz, tseed, ranks, sweeps, seed in (
        ("h3", [20, 18, 16], 200, 41, [3, 3, 3], 25, 5),           # solvers_test.cpp:143-156
        ("h4", [10, 9, 8, 7], 120, 44, [2, 3, 2, 2], 40, 17),     # solvers_test.cpp:325-345
        ("h2", [12, 9], 40, 45, [3, 3], 30, 3),                   # order 2
        ("h50", [50, 50, 50], 500, 31, [5, 5, 5], 30, 8),          # solvers_test.cpp:119-141
    ):
        t = RefTensor.gen_synthetic(lib, dims, nnz, tseed)
        _hoqri_case(lib, name, t, dims, ranks, sweeps, seed, out)
        names.append(name)
    # degenerate: explicit zero entry -> DegenerateStateError(mode 1) (solvers_test.cpp:312-323)
    t = RefTensor.create(lib, [3, 3, 3], np.array([[1, 1, 1]], np.uint32), np.array([0.0]))
    _hoqri_case(lib, "deg", t, [3, 3, 3], [1, 1, 1], 5, 1, out)
    names.append("deg")
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "hoqri.npz"), **out)


def gen_grad(lib):
    """Gradient tracing (trace_gradients / tol_grad, solvers.cpp:58, 126-150,
    165-167) through tucker::hoqri with seeded random init: per-update
    grad_norm_sq, f_before, f_after, sigma, lambda, and the sweep count."""
    out, names = {}, []
    for name, dims, nnz, tseed, ranks, sweeps, seed, tol_grad in (
        ("g3", [20, 18, 16], 200, 41, [3, 3, 3], 12, 5, 0.0),
        ("g4", [10, 9, 8, 7], 120, 44, [2, 3, 2, 2], 10, 17, 0.0),
        ("gk", [60, 50, 40], 3000, 47, [10, 8, 6], 8, 9, 0.0),
        ("gstop", [50, 50, 50], 500, 31, [5, 5, 5], 60, 8, 0.02),
    ):
        t = RefTensor.gen_synthetic(lib, dims, nnz, tseed)
        c, v = t.export()
        r = t.hoqri_traced(ranks, sweeps, 0.0, seed, tol_grad)
        if r["status"]:
            raise RuntimeError(f"{name}: reference status {r['status']}")
        out[f"{name}_dims"] = np.asarray(dims, np.uint64)
        out[f"{name}_ranks"] = np.asarray(ranks, np.uint64)
        out[f"{name}_seed"] = np.array(seed, np.uint64)
        out[f"{name}_max_sweeps"] = np.array(sweeps)
        out[f"{name}_tol_grad"] = np.array(tol_grad)
        out[f"{name}_coords"], out[f"{name}_vals"] = c, v
        for k in ("sweeps", "objective", "fit", "grad", "updates", "f_before", "f_after", "sigma", "lambda_", "core"):
            out[f"{name}_{k}"] = np.asarray(r[k])
        u0 = ref_random_factors(lib, dims, ranks, seed)
        for m in range(len(dims)):
            out[f"{name}_U0_{m}"] = u0[m]
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "grad.npz"), **out)


def gen_trace(lib):
    """harness.cpp:101-161 trace files (CSV + JSON) of a reference hoqri run,
    for the trace-schema tests of the engine's harness."""
    dims, nnz, tseed, ranks, sweeps, seed = [20, 18, 16], 200, 41, [3, 3, 3], 6, 5
    t = RefTensor.gen_synthetic(lib, dims, nnz, tseed)
    csv, js = t.trace_files(ranks, sweeps, seed)
    c, v = t.export()
    np.savez_compressed(os.path.join(OUT, "trace.npz"), dims=np.asarray(dims, np.uint64), nnz=np.array(nnz),
                        tensor_seed=np.array(tseed, np.uint64), ranks=np.asarray(ranks, np.uint64),
                        sweeps=np.array(sweeps), seed=np.array(seed, np.uint64), csv=np.array(csv),
                        json=np.array(js), coords=c, vals=v)


def _planted(dims, ranks, seed):
    """dense planted Tucker tensor (every cell stored), the solvers_test planted_tensor idea"""
    rng = np.random.default_rng(seed)
    us = [np.linalg.qr(rng.standard_normal((d, k)))[0] for d, k in zip(dims, ranks)]
    g = rng.standard_normal(ranks)
    x = g
    for v, u in enumerate(us):
        x = np.moveaxis(np.tensordot(u, np.moveaxis(x, v, 0), axes=(1, 0)), 0, v)
    idx = np.indices(dims).reshape(len(dims), -1).T.astype(np.uint32)
    return idx, x.reshape(-1).copy()


def gen_dense(lib):
    """Desk-scale dense paths of the reference (kernels.cpp:264-348, dense_core.cpp:266-327,
    solvers.cpp:93-122, 202-215): dense unfoldings, svd_leading, HOSVD init, hoqri from HOSVD,
    hooi (random / HOSVD, traced)."""
    out, names = {}, []
    cases = [("s8", "syn", [8, 8, 8], 30, 4, [3, 3, 3], 10, 123),
             ("s15", "syn", [15, 14, 13], 120, 51, [3, 3, 3], 40, 4),
             ("r4", "syn", [6, 5, 4, 3], 60, 9, [2, 2, 2, 2], 8, 3),
             ("pl", "planted", [10, 9, 8], 0, 5, [2, 2, 2], 6, 1)]
    for name, kind, dims, nnz, tseed, ranks, sweeps, seed in cases:
        if kind == "syn":
            t = RefTensor.gen_synthetic(lib, dims, nnz, tseed)
        else:
            c0, v0 = _planted(dims, ranks, tseed)
            t = RefTensor.create(lib, dims, c0, v0)
        c, v = t.export()
        out[f"{name}_dims"], out[f"{name}_ranks"] = np.asarray(dims, np.uint64), np.asarray(ranks, np.uint64)
        out[f"{name}_coords"], out[f"{name}_vals"] = c, v
        out[f"{name}_sweeps"], out[f"{name}_seed"] = np.array(sweeps), np.array(seed, np.uint64)
        for m in range(len(dims)):
            st, d = t.densify(m)
            out[f"{name}_dense{m}"] = d
        st, msg, hs = t.init_factors(ranks, seed, True)
        assert st == 0, msg
        u0 = ref_random_factors(lib, dims, ranks, seed)
        for m in range(len(dims)):
            out[f"{name}_hosvd{m}"] = hs[m]
            st, y = t.unfold_dense(ranks, u0, m)
            out[f"{name}_Y{m}"] = y
            out[f"{name}_U0_{m}"] = u0[m]
        for alg, hosvd, tag in ((0, 1, "hoqri_hosvd"), (1, 0, "hooi_rand"), (1, 1, "hooi_hosvd")):
            r = t.solve(alg, ranks, sweeps, 0.0, seed, hosvd, trace_gradients=(alg == 1 and hosvd == 0))
            assert r["status"] == 0, (name, tag, r["status"])
            for k in ("sweeps", "initial_objective", "objective", "fit", "drift", "grad", "core"):
                out[f"{name}_{tag}_{k}"] = np.asarray(r[k])
            for m in range(len(dims)):
                out[f"{name}_{tag}_U{m}"] = r["factors"][m]
        names.append(name)
    # svd_leading: m > p (Gram on the column side), m <= p, rank-deficient (fill), zero matrix
    rng = np.random.default_rng(3)
    a1 = rng.standard_normal((30, 12))
    a2 = rng.standard_normal((8, 20))
    a3 = rng.standard_normal((25, 6))
    a3[:, 4] = a3[:, 0] - 2 * a3[:, 1]
    a3[:, 5] = 0.0
    svd = [("sv_tall", a1, 4), ("sv_wide", a2, 3), ("sv_def", a3, 6), ("sv_zero", np.zeros((10, 4)), 2)]
    for nm, a, k in svd:
        out[f"{nm}_A"], out[f"{nm}_k"], out[f"{nm}_U"] = a, np.array(k), ref_svd_leading(lib, a, k)
    out["svd_names"] = np.array([nm for nm, _, _ in svd])
    # capacity: HOSVD init beyond the cap (solvers_test.cpp:80-87)
    t = RefTensor.gen_synthetic(lib, [40, 40, 40], 50, 6)
    st, msg, _ = t.init_factors([2, 2, 2], 0, True, cap=1000)
    c, v = t.export()
    out.update(cap_coords=c, cap_vals=v, cap_status=np.array(st), cap_message=np.array(msg))
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "dense.npz"), **out)


def gen_config1(lib):
    """BASELINE config 1 at full size: 10^4 cube, 10^5 uniform draws, U(0,1),
    rank 10^3, 20 sweeps.  Inputs come from workloads.uniform_coo(seed=1001);
    stores layout hashes, the trace, the final core and final factors."""
    dims, draws, ranks, sweeps, seed = [10**4] * 3, 10**5, [10] * 3, 20, 1234
    coords, vals = uniform_coo(dims, draws, 1001)
    t = RefTensor.create(lib, dims, coords, vals)
    c, v = t.export()
    out = dict(dims=np.asarray(dims, np.uint64), ranks=np.asarray(ranks, np.uint64), draws=np.array(draws),
               gen_seed=np.array(1001), seed=np.array(seed, np.uint64), sweeps=np.array(sweeps),
               nnz=np.array(t.nnz), coords_sha=np.array(sha(c)), vals_sha=np.array(sha(v)))
    for m in range(3):
        off, ent = t.buckets(m)
        out[f"off{m}_sha"] = np.array(sha(off))
        out[f"ent{m}_sha"] = np.array(sha(ent))
    r = t.hoqri(ranks, sweeps, 0.0, seed)
    out.update(norm_sq=np.array(t.norm_sq()), initial_objective=np.array(r["initial_objective"]),
               objective=r["objective"], fit=r["fit"], drift=r["drift"], core=r["core"],
               ref_elapsed_s=r["elapsed"])
    for m in range(3):
        out[f"U{m}"] = r["factors"][m]
    np.savez_compressed(os.path.join(OUT, "config1.npz"), **out)


def main():
    if not RefLib.available():
        sys.exit("oracle/_ref/libtucker_ref.so missing: run `make -C oracle ref` first")
    os.makedirs(OUT, exist_ok=True)
    lib = RefLib()
    gen_rng(lib)
    gen_tensors(lib)
    gen_kernels(lib)
    gen_qr(lib)
    gen_hoqri(lib)
    gen_grad(lib)
    gen_trace(lib)
    gen_dense(lib)
    if "--skip-config1" not in sys.argv:
        gen_config1(lib)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
