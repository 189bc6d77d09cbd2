"""Per-phase cycle breakdown of the fiber-unit segment kernel k_fibseg (needs a -DHQ_PHASE_TIMING build
selected with HQ_LIB; thread 0 of every CTA adds the cycles between phase marks).
python tools/fib_phase_timing.py [cfg]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import CONFIGS, config_coo
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = CONFIGS[cfg]
coords, vals = config_coo(cfg)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
x = hq.SparseTensor(list(c["dims"]), coords, vals)
u0 = hq.random_factors(list(c["dims"]), list(c["ranks"]), 1)
sol = hq.Solver(x, hq.SolverConfig(ranks=list(c["ranks"]), max_sweeps=4, tol_fit_change=0.0), init_factors=u0.factors, stream=s.cuda_stream)
sol.run(1); sol.sync()
L = hq.load_library()
buf = (C.c_ulonglong * 16)()
names = ["head (count, records, cursor)", "slice wait", "gather issue", "next slice issue", "gather wait", "unit sums",
         "DMMA k-steps", "segment reduce + end"]
for m in range(len(c["dims"])):
    L.hq_debug_fib_phase_cycles(buf, 1)
    reps = 3
    for _ in range(reps):
        sol.launch_mode_pass(m)
    torch.cuda.synchronize()
    L.hq_debug_fib_phase_cycles(buf, 1)
    tot = sum(buf[i] for i in range(8))
    print(f"mode {m} fiber plan {x.fiber_plan(m)}")
    for i, n in enumerate(names):
        print(f"  {n:30s} {buf[i] / reps / 1e6:9.2f} Mcycles (all CTAs) / launch  {100 * buf[i] / max(tot, 1):5.1f}%")
