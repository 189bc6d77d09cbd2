"""Per-phase cycle breakdown of the specialised pass (needs a -DHQ_PHASE_TIMING build via HQ_LIB)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import CONFIGS, config_coo
c = CONFIGS[2]
coords, vals = config_coo(2)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
x = hq.SparseTensor(list(c["dims"]), coords, vals)
u0 = hq.random_factors(list(c["dims"]), list(c["ranks"]), 1)
sol = hq.Solver(x, hq.SolverConfig(ranks=list(c["ranks"]), max_sweeps=4, tol_fit_change=0.0), init_factors=u0.factors, stream=s.cuda_stream)
sol.run(1); sol.sync()
L = hq.load_library()
buf = (C.c_ulonglong * 16)()
L.hq_debug_phase_cycles(buf, 1)
for _ in range(3):
    sol.launch_mode_pass(0)
torch.cuda.synchronize()
L.hq_debug_phase_cycles(buf, 1)
names = ["wait gathers", "kron", "Y write", "issue gathers", "A-GEMM", "A write/max", "M-GEMM+W", "meta+records t+2"]
tot = sum(buf[i] for i in range(8))
for i, n in enumerate(names):
    print(f"{n:18s} {buf[i] / 3 / 296 / 1e3:9.1f} kcycles/CTA/launch  {100 * buf[i] / tot:5.1f}%")
