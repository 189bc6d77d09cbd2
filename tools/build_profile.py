"""Phase times of the device layout build (HQ_PROFILE_BUILD=1) for a BASELINE config, three builds in a row."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HQ_PROFILE_BUILD"] = "1"
import numpy as np
import torch
import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import CONFIGS, config_coo

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[cfg_id]
coords, vals = config_coo(cfg_id)
dims = list(c["dims"])
pc = torch.from_numpy(np.ascontiguousarray(coords)).pin_memory().numpy()
pv = torch.from_numpy(np.ascontiguousarray(vals)).pin_memory().numpy()
for it in range(3):
    t0 = time.perf_counter()
    x = hq.SparseTensor(dims, pc, pv)
    torch.cuda.synchronize()
    print(f"--- build {it}: {1e3 * (time.perf_counter() - t0):.1f} ms, nnz {x.nnz()}", file=sys.stderr, flush=True)
    del x
    torch.cuda.synchronize()
