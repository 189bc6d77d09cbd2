"""Live per-kernel timeline of steady-state HOQRI sweeps (torch.profiler / CUPTI activity records, no
replay or serialisation): per-kernel device time per sweep and the idle gaps between kernels."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import CONFIGS, config_coo

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
c = CONFIGS[cid]
coords, vals = config_coo(cid)
dims, ranks = list(c["dims"]), list(c["ranks"])
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
x = hq.SparseTensor(dims, coords, vals)
u0 = hq.random_factors(dims, ranks, int(os.environ.get("HQ_SEED", "20251016")))
sol = hq.Solver(x, hq.SolverConfig(ranks=ranks, max_sweeps=1000, tol_fit_change=0.0), init_factors=u0.factors,
                stream=s.cuda_stream)
sol.run(3); sol.sync()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sol.run(sweeps); sol.sync()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
agg = collections.OrderedDict()
busy = 0.0
for e in evs:
    n = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:70]
    d = e.time_range.end - e.time_range.start
    a = agg.setdefault(n, [0, 0.0]); a[0] += 1; a[1] += d
    busy += d
span = evs[-1].time_range.end - evs[0].time_range.start
print(f"config {cid}: {sweeps} sweeps, span {span / sweeps:.1f} us/sweep, kernel-busy {busy / sweeps:.1f} us/sweep, "
      f"{len(evs) / sweeps:.1f} launches/sweep, status {sol.status()}")
for n, (k, d) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{d / sweeps:9.1f} us/sweep {k / sweeps:6.1f}x {d / k:8.1f} us  {n}")
if len(sys.argv) > 3:
    pat = sys.argv[3]
    seq = [(e.name, e.time_range.end - e.time_range.start) for e in evs]
    print("launch sequence of one sweep (us):")
    for nm, d in seq[: len(seq) // sweeps]:
        print(f"  {d:8.1f}  {nm.replace('(anonymous namespace)::', '').replace('void ', '').split('(')[0][:60]}")
