"""Compact, exact-to-rounding fingerprints of tall factor matrices.

TEST INFRASTRUCTURE.  The BASELINE configs' factors are 10^5..10^6 rows (80 MB
per factor at config 2), too large to commit per sweep.  A parity fixture
therefore keeps, per factor:

* ``sketch``  S = Omega^T U / sqrt(m), Omega an I x m Rademacher (+-1) matrix
  whose signs come from a counter hash of (row, 64-column block) -- the same
  bits on every machine (numpy uint64 arithmetic here, the same arithmetic on
  the GPU box's host).  For a difference D = U_gpu - U_ref,
  ||Omega^T D||_F^2 / m is an unbiased estimate of ||D||_F^2 with relative
  standard deviation <= sqrt(2/m) (m = 256: 9 %);
* ``rows``    the exact values of a seeded sample of rows.

The parity tests use ||S_gpu - S_ref||_F as the estimate of ||U_gpu - U_ref||_F
and bound the north_star subspace metric ||U_g U_g^T - U_r U_r^T||_F by
2 ||U_g - U_r||_F (both factors orthonormal).
"""
from __future__ import annotations

import numpy as np

M_SKETCH = 256
N_ROWS = 128
_SALT = np.uint64(0x5EED5EED5EED5EED)


def _splitmix(z):
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def sign_bits(row0, rows, m=M_SKETCH):
    """Packed sign bits of Omega[row0:row0+rows, :m] as uint8 (rows, m/8)."""
    blocks = m // 64
    i = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    b = np.arange(blocks, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        h = _splitmix((i * np.uint64(blocks) + b) ^ _SALT)
    return h.astype("<u8").view(np.uint8).reshape(rows, m // 8)


def omega(row0, rows, m=M_SKETCH, dtype=np.float64):
    bits = np.unpackbits(sign_bits(row0, rows, m), axis=1, bitorder="little")
    return (1.0 - 2.0 * bits.astype(dtype))


def sketch(u, m=M_SKETCH, chunk=1 << 16):
    """S = Omega^T U / sqrt(m) (m x K), numpy, chunked over rows."""
    u = np.asarray(u, np.float64)
    s = np.zeros((m, u.shape[1]))
    for r0 in range(0, u.shape[0], chunk):
        r1 = min(u.shape[0], r0 + chunk)
        s += omega(r0, r1 - r0, m).T @ u[r0:r1]
    return s / np.sqrt(m)


def sketch_torch(u, m=M_SKETCH, chunk=1 << 18, cache=None):
    """Same sketch with the product on a torch device (u: torch float64
    tensor).  ``cache`` (a dict) keeps the unpacked Omega per row count."""
    import torch
    rows = u.shape[0]
    key = (rows, m)
    om = None if cache is None else cache.get(key)
    if om is None:
        om = torch.from_numpy(sign_bits(0, rows, m)).to(u.device)
        if cache is not None:
            cache[key] = om
    s = torch.zeros((m, u.shape[1]), dtype=torch.float64, device=u.device)
    shifts = torch.arange(8, device=u.device, dtype=torch.uint8)
    for r0 in range(0, rows, chunk):
        r1 = min(rows, r0 + chunk)
        bits = ((om[r0:r1, :, None] >> shifts) & 1).reshape(r1 - r0, m)
        s += (1.0 - 2.0 * bits.to(torch.float64)).T @ u[r0:r1]
    return (s / np.sqrt(m)).cpu().numpy()


def sample_rows(rows, n=N_ROWS, seed=77):
    rng = np.random.Generator(np.random.PCG64(seed + rows))
    return np.sort(rng.choice(rows, size=min(n, rows), replace=False)).astype(np.int64)


def fingerprint(u):
    """(sketch, sampled row ids, sampled rows) of a factor."""
    u = np.asarray(u, np.float64)
    idx = sample_rows(u.shape[0])
    return sketch(u), idx, u[idx]


def diff_estimate(s_a, s_b):
    """Estimate of ||U_a - U_b||_F from two sketches."""
    return float(np.linalg.norm(np.asarray(s_a) - np.asarray(s_b)))
