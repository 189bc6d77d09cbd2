"""Pins the C restatement (oracle/hq_oracle.c) to the reference's own outputs.

The fixtures in tests/golden/ were produced by the unmodified reference
library (oracle/gen_golden.py over oracle/_ref/libtucker_ref.so).  CPU only.
"""
import hashlib

import numpy as np
import pytest

from conftest import golden
from paper_2510_16930_b200.workloads import uniform_coo


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_rng_streams(oracle):
    g = golden("rng.npz")
    raw = oracle.raw_stream(5489, 10000)
    assert (raw[:16] == g["raw_5489_first"]).all()
    assert raw[-1] == g["raw_5489_10000"][0] == 9981545732273789042  # C++ [rand.predef]
    for s, row in zip(g["normal_seeds"], g["normals"]):
        assert (oracle.normal_stream(int(s), 64) == row).all()
    for i, s in enumerate(g["mix_seed_args"]):
        for t in range(5):
            assert oracle.mix_seed(int(s), t) == int(g["mix_seed"][i, t])


@pytest.mark.parametrize("name", ["hand", "gs4", "gs2", "gs3", "dups"])
def test_normalize_and_buckets(oracle, name):
    g = golden("tensors.npz")
    dims = g[f"{name}_dims"]
    c, v = oracle.normalize(dims, g[f"{name}_in_coords"], g[f"{name}_in_vals"])
    assert (c == g[f"{name}_coords"]).all()
    # merged values: exact for <= 2 duplicates, ~m*eps otherwise (sparse_tensor.cpp:49-64)
    np.testing.assert_allclose(v, g[f"{name}_vals"], rtol=1e-14, atol=1e-15)
    for m in range(dims.size):
        off, ent = oracle.buckets(dims, c, m)
        assert (off == g[f"{name}_off{m}"]).all()
        assert (ent == g[f"{name}_ent{m}"]).all()
    assert abs(oracle.norm_sq(v) - float(g[f"{name}_norm_sq"])) <= 1e-13 * max(1.0, float(g[f"{name}_norm_sq"]))


def test_hand_kats():
    g = golden("tensors.npz")
    # duplicates summed (sparse_tensor_test.cpp:24-29) and explicit zeros kept
    c, v = g["hand_coords"], g["hand_vals"]
    row = {tuple(x): y for x, y in zip(c.tolist(), v.tolist())}
    assert row[(0, 0, 0)] == 1.0 + 2.0 + 0.125
    assert row[(2, 2, 2)] == 0.0
    assert row[(1, 2, 3)] == 0.0


def test_kernels(oracle):
    g = golden("kernels.npz")
    for name in g["names"]:
        dims, ranks = g[f"{name}_dims"], g[f"{name}_ranks"]
        c, v = g[f"{name}_coords"], g[f"{name}_vals"]
        u = [g[f"{name}_U{m}"] for m in range(dims.size)]
        core = oracle.ttmc_core(dims, ranks, c, v, u)
        assert np.abs(core - g[f"{name}_core"]).max() <= 1e-13
        for m in range(dims.size):
            a = oracle.ttmctc(dims, ranks, c, v, u, m, g[f"{name}_core"])
            assert np.abs(a - g[f"{name}_A{m}"]).max() <= 1e-13
            # the matrix variant agrees to 1e-11 (kernels_test.cpp:167-190)
            assert np.abs(a - g[f"{name}_Am{m}"]).max() <= 1e-11


def test_qr(oracle):
    g = golden("qr.npz")
    for name in g["names"]:
        q = oracle.qr(g[f"{name}_A"])
        assert np.abs(q - g[f"{name}_Q"]).max() <= 1e-14, name
    np.testing.assert_allclose(g["k34_Q"][:, 0], [0.6, 0.8], rtol=1e-14)


def test_hoqri_traces(oracle):
    g = golden("hoqri.npz")
    for name in g["names"]:
        dims, ranks = g[f"{name}_dims"], g[f"{name}_ranks"]
        sweeps = int(g[f"{name}_sweeps"])
        c, v = g[f"{name}_coords"], g[f"{name}_vals"]
        if int(g[f"{name}_status"]):
            u0 = oracle.random_factors(dims, ranks, int(g[f"{name}_seed"]))
            r = oracle.hoqri(dims, ranks, c, v, u0, sweeps)
            assert r["status"] == 8 and r["degenerate_mode"] == int(g[f"{name}_payload"])
            continue
        u0 = oracle.random_factors(dims, ranks, int(g[f"{name}_seed"]))
        for m in range(dims.size):
            assert np.abs(u0[m] - g[f"{name}_U0_{m}"]).max() == 0.0  # bitwise init (solvers_test.cpp:61-70)
        r = oracle.hoqri(dims, ranks, c, v, u0, sweeps, snapshots=True)
        assert r["sweeps"] == sweeps
        np.testing.assert_allclose(r["objective"], g[f"{name}_objective"], rtol=1e-12)
        np.testing.assert_allclose(r["drift"], g[f"{name}_drift"], atol=1e-12)
        assert np.abs(r["core"] - g[f"{name}_core"]).max() <= 1e-12
        assert np.abs(r["core_snap"] - g[f"{name}_core_snap"]).max() <= 1e-12
        for m in range(dims.size):
            assert np.abs(r["factors"][m] - g[f"{name}_U{m}"]).max() <= 1e-12


def test_config1_layout_and_trace(oracle):
    """BASELINE config 1 at full size (10^4 cube, 10^5 draws, K=10, 20 sweeps)."""
    g = golden("config1.npz")
    dims, ranks = g["dims"], g["ranks"]
    coords, vals = uniform_coo([int(d) for d in dims], int(g["draws"]), int(g["gen_seed"]))
    c, v = oracle.normalize(dims, coords, vals)
    assert c.shape[0] == int(g["nnz"])
    assert sha(c) == str(g["coords_sha"]) and sha(v) == str(g["vals_sha"])
    for m in range(3):
        off, ent = oracle.buckets(dims, c, m)
        assert sha(off) == str(g[f"off{m}_sha"]) and sha(ent) == str(g[f"ent{m}_sha"])
    u0 = oracle.random_factors(dims, ranks, int(g["seed"]))
    r = oracle.hoqri(dims, ranks, c, v, u0, int(g["sweeps"]))
    np.testing.assert_allclose(r["objective"], g["objective"], rtol=1e-12)
    np.testing.assert_allclose(r["fit"], g["fit"], rtol=1e-12)
    assert np.abs(r["core"] - g["core"]).max() <= 1e-12 * np.abs(g["core"]).max()


def test_oracle_gradient_trace_matches_reference(oracle):
    """hqo_hoqri_traced (solvers.cpp:126-150, 165-167; manifold.cpp:37-84)
    against tucker::hoqri with trace_gradients: per-update diagnostics and the
    tol_grad stop."""
    g = golden("grad.npz")
    for n in g["names"]:
        dims = [int(d) for d in g[f"{n}_dims"]]
        ranks = [int(r) for r in g[f"{n}_ranks"]]
        u0 = [g[f"{n}_U0_{m}"] for m in range(len(dims))]
        r = oracle.hoqri_traced(dims, ranks, g[f"{n}_coords"], g[f"{n}_vals"], u0, int(g[f"{n}_max_sweeps"]), 0.0,
                                float(g[f"{n}_tol_grad"]))
        assert r["status"] == 0 and r["sweeps"] == int(g[f"{n}_sweeps"]), n
        for k in ("grad", "f_before", "f_after", "sigma", "lambda_", "objective"):
            np.testing.assert_allclose(r[k], g[f"{n}_{k}"], rtol=1e-13, atol=1e-14, err_msg=f"{n}:{k}")
