import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np
import paper_2510_16930_b200 as hq
g = np.load('/root/repo/tests/golden/qr.npz')
for name in g["names"]:
    a = g[f"{name}_A"]
    qs = [hq.qr_orthonormal(a) for _ in range(4)]
    print(name, a.shape, [float(np.abs(q - g[f"{name}_Q"]).max()) for q in qs], [bool((qs[0]==q).all()) for q in qs])
