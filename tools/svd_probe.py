"""Singular values of the TTMcTC output A along a config-2 HOQRI solve (QR conditioning)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import CONFIGS, config_coo
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[cid]
coords, vals = config_coo(cid)
dims, ranks = list(c["dims"]), list(c["ranks"])
x = hq.SparseTensor(dims, coords, vals)
u0 = hq.random_factors(dims, ranks, 1)
for sw in (1, 3, 6, 10, 14, 18):
    r = hq.hoqri(x, hq.SolverConfig(ranks=ranks, max_sweeps=sw, tol_fit_change=0.0), init_factors=u0.factors)
    a = hq.ttmctc_elementwise(x, r.model.factors, 0, r.model.core)
    s = np.linalg.svd(a, compute_uv=False)
    g = np.linalg.svd(r.model.core.data.reshape(ranks[0], -1), compute_uv=False)
    print(sw, "A sv ratio", s[-1] / s[0], "core sv", g[0], g[-1], "fit", r.trace.sweeps[-1].fit, flush=True)
