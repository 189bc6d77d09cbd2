"""Times the fused mode pass (per mode) and whole sweeps of a BASELINE config
with CUDA events on the solver's stream; one JSON line (HQ_LIB selects a
variant library).   python tools/pass_time.py [cfg] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_16930_b200 as hq  # noqa: E402
from paper_2510_16930_b200.workloads import CONFIGS, config_coo  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = CONFIGS[cfg_id]
coords, vals = config_coo(cfg_id)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
x = hq.SparseTensor(list(c["dims"]), coords, vals)
u0 = hq.random_factors(list(c["dims"]), list(c["ranks"]), 20251016)
sweeps = 4 + 12
sol = hq.Solver(x, hq.SolverConfig(ranks=list(c["ranks"]), max_sweeps=sweeps, tol_fit_change=0.0),
                init_factors=u0.factors, stream=s.cuda_stream)
sol.run(2)
sol.sync()
out = {"cfg": cfg_id, "lib": os.environ.get("HQ_LIB", "default"), "pass_ms": []}
for m in range(len(c["dims"])):
    sol.launch_mode_pass(m)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        sol.launch_mode_pass(m)
    e1.record(s)
    e1.synchronize()
    out["pass_ms"].append(round(e0.elapsed_time(e1) / reps, 4))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
sol.run(10)
e1.record(s)
e1.synchronize()
out["sweep_ms"] = round(e0.elapsed_time(e1) / 10, 4)
st = sol.status() if hasattr(sol, "status") else None
print(json.dumps(out), flush=True)
