"""Per-phase cycle breakdown of the K = 10 short-row pass k_pass_np3 (needs a
-DHQ_PHASE_TIMING build selected with HQ_LIB; thread 0 of every CTA adds the
cycles between phase marks).   python tools/phase_timing.py [cfg]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import CONFIGS, config_coo
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[cfg]
coords, vals = config_coo(cfg)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
x = hq.SparseTensor(list(c["dims"]), coords, vals)
u0 = hq.random_factors(list(c["dims"]), list(c["ranks"]), 1)
sol = hq.Solver(x, hq.SolverConfig(ranks=list(c["ranks"]), max_sweeps=4, tol_fit_change=0.0), init_factors=u0.factors, stream=s.cuda_stream)
sol.run(1); sol.sync()
L = hq.load_library()
buf = (C.c_ulonglong * 16)()
L.hq_debug_phase_cycles(buf, 1)
reps = 3
for _ in range(reps):
    sol.launch_mode_pass(0)
torch.cuda.synchronize()
L.hq_debug_phase_cycles(buf, 1)
ctas = 148 * 3
names = ["meta", "records wait", "gather issue", "gather wait", "kron", "Y write", "A-GEMM+epi", "M-GEMM+W"]
tot = sum(buf[i] for i in range(8))
for i, n in enumerate(names):
    print(f"{n:14s} {buf[i] / reps / ctas / 1e3:9.1f} kcycles/CTA/launch  {100 * buf[i] / tot:5.1f}%")
print(f"{'total':14s} {tot / reps / ctas / 1e3:9.1f} kcycles/CTA/launch")
