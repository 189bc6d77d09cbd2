"""Phase breakdown of one end-to-end solve (bench.py's e2e step) on a BASELINE config."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import CONFIGS, config_coo

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[cfg_id]
coords, vals = config_coo(cfg_id)
dims, ranks = list(c["dims"]), list(c["ranks"])
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
pc = torch.from_numpy(np.ascontiguousarray(coords)).pin_memory()
pv = torch.from_numpy(np.ascontiguousarray(vals)).pin_memory()
u0 = hq.random_factors(dims, ranks, int(os.environ.get("HQ_SEED", "20251016")))
pu = [torch.from_numpy(np.ascontiguousarray(f)).pin_memory() for f in u0.factors]
hc, hv, hu = pc.numpy(), pv.numpy(), [t.numpy() for t in pu]
cfg = hq.SolverConfig(ranks=ranks, max_sweeps=c["sweeps"], tol_fit_change=0.0)
po = [torch.empty((d, k), dtype=torch.float64).pin_memory().numpy() for d, k in zip(dims, ranks)]
pcore = torch.empty(int(np.prod(ranks)), dtype=torch.float64).pin_memory().numpy()
for it in range(int(os.environ.get("HQ_ITERS", "3"))):
    t = [time.perf_counter()]
    x = hq.SparseTensor(dims, hc, hv); torch.cuda.synchronize(); t.append(time.perf_counter())
    sol = hq.Solver(x, cfg, init_factors=hu, stream=s.cuda_stream); torch.cuda.synchronize(); t.append(time.perf_counter())
    sol.run(1); sol.sync(); t.append(time.perf_counter())
    st1 = sol.status()
    sol.run(c["sweeps"] - 1); sol.sync(); t.append(time.perf_counter())
    print("status after sweep 1:", st1, "after all:", sol.status())
    r = sol.download(out=(po, pcore)); t.append(time.perf_counter())
    del sol; torch.cuda.synchronize(); t.append(time.perf_counter())
    del x; torch.cuda.synchronize(); t.append(time.perf_counter())
    names = ["tensor", "solver", "sweep1", "sweeps", "download", "del_solver", "del_tensor"]
    print(it, " ".join(f"{n}={1e3 * (t[i + 1] - t[i]):.1f}ms" for i, n in enumerate(names)), f"total={1e3 * (t[-1] - t[0]):.1f}")
