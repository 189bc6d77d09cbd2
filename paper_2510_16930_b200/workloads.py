"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference's public benchmark inputs are synthetic (BASELINE.json
``configs``); there is no dataset.  These generators produce COO arrays
(uint32 AoS coords, float64 values) in the shapes and distributions the
configs name.  Duplicates are NOT merged here: the tensor constructor merges
them by summing, exactly as the reference's ``SparseTensor`` does
(proj/src/sparse_tensor.cpp:43-71), so nnz_merged is reported after building.

Generation is numpy (PCG64, fixed seeds), so every machine produces the same
arrays.  Config 4 (planted model) evaluates its model entries with torch on
the GPU when one is present, in float64.
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
        q, r = np.linalg.qr(rng.standard_normal((d, k)))
        q *= np.sign(np.diag(r))[None, :]
        factors.append(np.ascontiguousarray(q))
    core = rng.standard_normal(tuple(ranks))
    coords = np.empty((draws, n), dtype=np.uint32)
    for m, d in enumerate(dims):
        coords[:, m] = rng.integers(0, d, size=draws, dtype=np.uint32)
    model = _model_entries(coords, factors, core, device)
    rms = float(np.sqrt(np.mean(model * model))) if draws else 0.0
    vals = model + noise * rms * rng.standard_normal(draws)
    return coords, vals, factors, core


def _model_entries(coords, factors, core, device):
    try:
        import torch
    except Exception:  # pragma: no cover
        torch = None
    if torch is not None and (device is not None or torch.cuda.is_available()):
        dev = device or "cuda"
        g = torch.as_tensor(core, device=dev)
        us = [torch.as_tensor(u, device=dev) for u in factors]
        out = np.empty(coords.shape[0])
        chunk = 1 << 20
        for b in range(0, coords.shape[0], chunk):
            c = torch.as_tensor(coords[b:b + chunk].astype(np.int64), device=dev)
            t = g
            rows = [u[c[:, m]] for m, u in enumerate(us)]
            t = torch.einsum("pqr,np,nq,nr->n", g, *rows) if len(us) == 3 else _einsum_n(torch, g, rows)
            out[b:b + chunk] = t.cpu().numpy()
        return out
    out = np.empty(coords.shape[0])
    chunk = 1 << 16
    for b in range(0, coords.shape[0], chunk):
        rows = [u[coords[b:b + chunk, m]] for m, u in enumerate(factors)]
        t = core
        # contract one mode at a time, batch dim first
        t = np.einsum("p...,np->n...", t, rows[0])
        for r in rows[1:]:
            t = np.einsum("np...,np->n...", t, r)
        out[b:b + chunk] = t
    return out


def _einsum_n(torch, g, rows):
    t = torch.einsum("p...,np->n...", g, rows[0])
    for r in rows[1:]:
        t = torch.einsum("np...,np->n...", t, r)
    return t


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
