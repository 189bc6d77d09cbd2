"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference's public benchmark inputs are synthetic (BASELINE.json
``configs``); there is no dataset.  These generators produce COO arrays
(uint32 AoS coords, float64 values) in the shapes and distributions the
configs name.  Duplicates are NOT merged here: the tensor constructor merges
them by summing, exactly as the reference's ``SparseTensor`` does
(proj/src/sparse_tensor.cpp:43-71), so nnz_merged is reported after building.

Generation is numpy (PCG64, fixed seeds), so every machine produces the same
arrays.  Config 4 (planted model) evaluates its model entries with torch on
the GPU when one is present, in float64, in an operation order that makes
the numpy and torch results bit-identical.
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    1: dict(name="c1_uniform_1e4cube_nnz1e5_K10", dims=(10**4,) * 3, draws=10**5, ranks=(10,) * 3, sweeps=20, values="uniform"),
    2: dict(name="c2_uniform_1e6cube_nnz1e7_K10", dims=(10**6,) * 3, draws=10**7, ranks=(10,) * 3, sweeps=20, values="uniform"),
    3: dict(name="c3_zipf1.1_5e5x2e4x2e3_nnz1e8_K10", dims=(5 * 10**5, 2 * 10**4, 2 * 10**3), draws=10**8, ranks=(10,) * 3,
            sweeps=20, values="lognormal", zipf_s=1.1),
    4: dict(name="c4_planted_1e5cube_nnz5e7_K16", dims=(10**5,) * 3, draws=5 * 10**7, ranks=(16,) * 3, sweeps=20, values="planted",
            noise=0.01),
    5: dict(name="c5_uniform_2e5pow4_nnz2e8_K8", dims=(2 * 10**5,) * 4, draws=2 * 10**8, ranks=(8,) * 4, sweeps=10, values="uniform"),
}


def uniform_coo(dims, draws, seed, values="uniform"):
    """Coordinates uniform over the extents, values U(0,1) (or N(0,1))."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = len(dims)
    coords = np.empty((draws, n), dtype=np.uint32)
    for m, d in enumerate(dims):
        coords[:, m] = rng.integers(0, d, size=draws, dtype=np.uint32)
    if values == "uniform":
        vals = rng.random(draws, dtype=np.float64)
    elif values == "normal":
        vals = rng.standard_normal(draws, dtype=np.float64)
    else:
        raise ValueError(values)
    return coords, vals


def zipf_coo(dims, draws, seed, s=1.1):
    """Each mode index = perm_n[Zipf(s) rank], a seeded permutation per mode;
    values lognormal(0, 1) (config 3)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = len(dims)
    coords = np.empty((draws, n), dtype=np.uint32)
    for m, d in enumerate(dims):
        w = np.arange(1, d + 1, dtype=np.float64) ** (-s)
        cdf = np.cumsum(w)
        cdf /= cdf[-1]
        perm = rng.permutation(d).astype(np.uint32)
        chunk = 1 << 24
        for b in range(0, draws, chunk):
            e = min(draws, b + chunk)
            r = np.searchsorted(cdf, rng.random(e - b), side="right")
            np.minimum(r, d - 1, out=r)
            coords[b:e, m] = perm[r]
    vals = rng.lognormal(0.0, 1.0, size=draws)
    return coords, vals


def planted_coo(dims, draws, ranks, seed, noise=0.01, device=None):
    """Config 4: orthonormal factors (seeded Gaussian + QR), dense Gaussian
    core, uniform coordinates, value = model entry + noise*rms(model)*N(0,1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = len(dims)
    factors = []
    for d, k in zip(dims, ranks):
        factors.append(_mgs2(rng.standard_normal((d, k))))
    core = rng.standard_normal(tuple(ranks))
    coords = np.empty((draws, n), dtype=np.uint32)
    for m, d in enumerate(dims):
        coords[:, m] = rng.integers(0, d, size=draws, dtype=np.uint32)
    model = _model_entries(coords, factors, core, device)
    rms = float(np.sqrt((model * model).sum() / draws)) if draws else 0.0
    vals = model + noise * rms * rng.standard_normal(draws)
    return coords, vals, factors, core


def _mgs2(a):
    """Orthonormal columns by modified Gram-Schmidt, twice (positive R
    diagonal).  Only elementwise ops and numpy's pairwise ``sum`` (plain C, no
    CPU-dispatched BLAS), so every host produces the same bits."""
    q = np.array(a, np.float64).T.copy()  # columns as contiguous rows
    for _ in range(2):
        for j in range(q.shape[0]):
            for i in range(j):
                q[j] -= (q[i] * q[j]).sum() * q[i]
            q[j] /= np.sqrt((q[j] * q[j]).sum())
    return np.ascontiguousarray(q.T)


def _model_entries(coords, factors, core, device):
    """Tucker model entries sum_{p,q,r} G[p,q,r] U1[i,p] U2[j,q] U3[k,r] in a
    FIXED sequence of elementwise IEEE multiplies and adds (no BLAS, no fused
    multiply-add, no library reductions), so numpy on any host and torch on
    the GPU produce bit-identical values: the parity fixtures made from the
    reference on the build host and the GPU tests see the same tensor."""
    xp, conv = np, (lambda a: a)
    try:
        import torch
        if device is not None or torch.cuda.is_available():
            dev = device or "cuda"
            xp = torch
            conv = (lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev))
    except Exception:  # pragma: no cover
        pass
    g = np.asarray(core, np.float64)
    out = np.empty(coords.shape[0])
    chunk = (1 << 24) if xp is not np else (1 << 20)
    for b in range(0, coords.shape[0], chunk):
        rows = [conv(u[coords[b:b + chunk, m]].T.copy()) for m, u in enumerate(factors)]  # (K_m, n) each
        t = _contract(g, rows)
        out[b:b + chunk] = t.cpu().numpy() if xp is not np else t
    return out


def _contract(g, rows):
    """value = sum_{k0} r0[k0] * (sum_{k1} r1[k1] * (... sum_{kl} g[k0..kl] * rl[kl]))
    with each sum taken left to right, one rounding per multiply and per add."""
    if g.ndim == 1:
        acc = rows[0][0] * float(g[0])
        for k in range(1, g.shape[0]):
            acc = acc + rows[0][k] * float(g[k])
        return acc
    acc = None
    for k in range(g.shape[0]):
        term = rows[0][k] * _contract(g[k], rows[1:])
        acc = term if acc is None else acc + term
    return acc


def config_coo(cfg_id, seed=None, scale=1.0):
    """COO arrays for BASELINE config ``cfg_id``; ``scale`` < 1 shrinks the
    draw count (and keeps extents) for bounded parity runs."""
    c = CONFIGS[cfg_id]
    seed = 1000 + cfg_id if seed is None else seed
    draws = max(1, int(c["draws"] * scale))
    if c["values"] == "uniform":
        return uniform_coo(c["dims"], draws, seed)
    if c["values"] == "lognormal":
        return zipf_coo(c["dims"], draws, seed, c["zipf_s"])
    if c["values"] == "planted":
        coords, vals, _, _ = planted_coo(c["dims"], draws, c["ranks"], seed, c["noise"])
        return coords, vals
    raise ValueError(c["values"])
