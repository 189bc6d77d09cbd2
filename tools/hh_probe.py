import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2510_16930_b200 as hq
m, k, dead = int(sys.argv[1]), int(sys.argv[2]), [int(x) for x in sys.argv[3].split(',')]
rng = np.random.default_rng(5)
a = rng.standard_normal((m, k))
for d in dead:
    a[:, d] = a[:, :d] @ rng.standard_normal(d) if d else 0.0
t = time.time()
q = hq.qr_orthonormal(a)
print("qr ok", time.time() - t, np.abs(q.T @ q - np.eye(k)).max(), flush=True)
