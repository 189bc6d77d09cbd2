"""GPU: the engine's OWN multi-rank path (hq_solver_create_dist) at world
size 2 -- two processes, one rank each, through the host transport
(hq_comm_create_host: collectives are D2H -> host combine in rank order ->
H2D, so no kernel waits on another rank and both ranks may share the one GPU
gpurun provides).  Row-partitioned pass, all-reduced Grams / M / W, owner
row gather of every new factor, the host-driven Householder continuation
with the reference's seeded fill on rank-deficient updates, and the sharded
storage (hq_tensor_shard: each rank keeps only its rows' streams), and the
fused apply + all-gather (the apply kernel stores its rows of U_new into the
other rank's replica, mapped through CUDA IPC; a barrier follows).  Every
sweep is checked against the oracle (the C restatement of the reference's
solve loop, oracle/hq_oracle.c) and the final state against the single-GPU
engine."""
import json
import os
import subprocess
import sys
import textwrap
import uuid

import numpy as np
import pytest

import paper_2510_16930_b200 as hq
from paper_2510_16930_b200.workloads import uniform_coo

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RANK_SCRIPT = textwrap.dedent("""
    import json, sys, numpy as np
    sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
    import paper_2510_16930_b200 as hq
    rank, world, name, case, shard, out = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5], sys.argv[6]
    rank, world, shard = int(rank), int(world), shard == '1'
    z = np.load(case)
    dims, ranks, sweeps = [int(d) for d in z['dims']], [int(r) for r in z['ranks']], int(z['sweeps'])
    u0 = [z['U0_%d' % m] for m in range(len(dims))]
    cap = max(max(d * k for d, k in zip(dims, ranks)), sweeps * len(dims) * max(ranks) ** 2, int(np.prod(ranks)) * 4)
    comm = hq.Comm.host(world, rank, name, cap)
    x = hq.SparseTensor(dims, z['coords'], z['vals'])
    if shard:
        x.shard(comm)
    sol = hq.Solver(x, hq.SolverConfig(ranks=ranks, max_sweeps=sweeps, tol_fit_change=0.0), init_factors=u0, comm=comm)
    res = []
    for s in range(sweeps):
        sol.run(1)
        sol.sync()
        r = sol.download()
        res.append(dict(core=r.model.core.data.tolist(), factors=[f.tolist() for f in r.model.factors.factors],
                        objective=[t.objective for t in r.trace.sweeps], drift=[t.drift for t in r.trace.sweeps]))
    st = sol.status()
    if rank == 0:
        json.dump(dict(res=res, status=st), open(out, 'w'))
    print('ok', st)
""")


def _world2(tmp_path, dims, ranks, coords, vals, u0, sweeps, shard, peer=True):
    case = tmp_path / "case.npz"
    np.savez(case, dims=np.asarray(dims), ranks=np.asarray(ranks), sweeps=sweeps, coords=coords, vals=vals,
             **{f"U0_{m}": u for m, u in enumerate(u0)})
    out = tmp_path / "rank0.json"
    name = "/hq_t_" + uuid.uuid4().hex[:12]
    procs = [subprocess.Popen([sys.executable, "-c", RANK_SCRIPT, str(r), "2", name, str(case), "1" if shard else "0",
                               str(out)], cwd=ROOT, env={**os.environ, "HQ_HOST_BARRIER_S": "90", "HQ_PEER_APPLY": "1" if peer else "0"},
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(2)]
    logs = []
    for p in procs:
        try:
            o, e = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append((p.returncode, o, e))
    if not all(rc == 0 and "ok" in o for rc, o, e in logs):
        raise AssertionError("\n".join(f"--- rank {r}: rc {rc}\n{o}\n{e[-4000:]}" for r, (rc, o, e) in enumerate(logs)))
    return json.load(open(out))


def _deficient_case():
    """Mode 1 has only 6 distinct indices and K = 8, so every mode-1 TTMcTC output has rank <= 6: each mode-1
    update needs the reference's seeded fill (dense_core.cpp:145-157) -- the host-driven Householder
    continuation on both ranks."""
    rng = np.random.default_rng(5)
    dims, k = [300, 240, 200], 8
    n = 6000
    coords = np.empty((n, 3), np.uint32)
    coords[:, 0] = rng.integers(0, dims[0], n)
    coords[:, 1] = rng.choice(np.array([3, 50, 77, 120, 199, 230], np.uint32), n)
    coords[:, 2] = rng.integers(0, dims[2], n)
    vals = rng.random(n)
    return dims, [k] * 3, coords, vals


@pytest.mark.parametrize("shard", [False, True])
@pytest.mark.parametrize("case", ["uniform", "deficient"])
def test_world2_engine_matches_oracle(tmp_path, oracle, case, shard):
    if case == "uniform":
        dims, ranks = [4000, 3000, 2000], [10, 10, 10]
        coords, vals = uniform_coo(dims, 40000, 21)
        sweeps = 6
    else:
        dims, ranks, coords, vals = _deficient_case()
        sweeps = 4
    oc, ov = oracle.normalize(dims, coords, vals)
    u0 = oracle.random_factors(dims, ranks, 13)
    out = _world2(tmp_path, dims, ranks, coords, vals, u0, sweeps, shard)
    ref = oracle.hoqri(dims, ranks, oc, ov, u0, sweeps, snapshots=True)
    N = len(dims)
    if case == "deficient":
        assert out["status"]["dist_householder"] >= sweeps, out["status"]  # every mode-1 update at least
    for s, r in enumerate(out["res"]):
        np.testing.assert_allclose(np.array(r["objective"]), ref["objective"][:s + 1], rtol=1e-9)
        np.testing.assert_allclose(np.array(r["drift"]), ref["drift"][:s + 1], atol=1e-10)
        for m in range(N):
            ug, ur = np.array(r["factors"][m]), ref["factor_snap"][s][m]
            assert np.linalg.norm(ug @ ug.T - ur @ ur.T) <= 1e-8, (s, m)
        g, gr = np.array(r["core"]), ref["core_snap"][s].reshape(-1)
        assert np.linalg.norm(g - gr) <= 1e-9 * np.linalg.norm(gr), s
    # the apply stored U_new straight into the other rank's replica (CUDA IPC peer memory; fused apply +
    # all-gather), and the all-gather path (HQ_PEER_APPLY=0) gives the same bits
    assert out["status"]["peer_apply"] == 1, out["status"]
    if case == "uniform" and not shard:
        out0 = _world2(tmp_path, dims, ranks, coords, vals, u0, sweeps, shard, peer=False)
        assert out0["status"]["peer_apply"] == 0
        for m in range(N):
            assert np.array_equal(np.array(out0["res"][-1]["factors"][m]), np.array(out["res"][-1]["factors"][m]))
        assert np.array_equal(np.array(out0["res"][-1]["core"]), np.array(out["res"][-1]["core"]))
    # the single-GPU engine on the same inputs ends in the same state
    x = hq.SparseTensor(dims, coords, vals)
    r1 = hq.hoqri(x, hq.SolverConfig(ranks=ranks, max_sweeps=sweeps, tol_fit_change=0.0), init_factors=u0)
    g2 = np.array(out["res"][-1]["core"])
    assert np.linalg.norm(g2 - r1.model.core.data) <= 1e-9 * np.linalg.norm(r1.model.core.data)
