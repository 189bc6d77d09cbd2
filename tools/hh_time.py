"""Device time of qr_orthonormal on a rank-deficient tall matrix (Householder path), CUDA events around the call."""
import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
import paper_2510_16930_b200 as hq
m, k = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(5)
a = rng.standard_normal((m, k))
a[:, 3] = a[:, :3] @ rng.standard_normal(3)
a[:, 7] = a[:, :7] @ rng.standard_normal(7)
hq.qr_orthonormal(a)
ts = []
for _ in range(5):
    t = time.perf_counter(); hq.qr_orthonormal(a); ts.append(time.perf_counter() - t)
print(f"qr_orthonormal {m}x{k} (Householder path): median {1e3 * sorted(ts)[2]:.2f} ms wall (incl. H2D/D2H)")
