"""CPU tests of the multi-GPU path with torch.distributed/gloo.

* the engine's row partition planner (hq_partition_rows, host code in the
  CUDA library — callable without a GPU);
* the row-partitioned mode update the engine runs per rank (local pass over
  the owned rows; all-reduce of M = A^T Y, W = A^T A, the CholeskyQR2 Gram
  and the drift product; owner broadcast of new factor rows), restated in
  numpy on world_size 2 and checked against the single-process oracle
  (the C restatement of the reference's solve loop).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2510_16930_b200 as hq
from conftest import golden


def test_partition_rows_balanced_and_whole():
    rng = np.random.default_rng(0)
    lens = rng.poisson(10, size=1000).astype(np.uint64)
    lens[17] = 3000  # one heavy row
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
    for world in (1, 2, 3, 8):
        b = hq.partition_rows(off, world)
        assert b[0] == 0 and b[-1] == 1000 and (np.diff(b.astype(np.int64)) >= 0).all()
        nnz = int(off[-1])
        per = [int(off[b[r + 1]] - off[b[r]]) for r in range(world)]
        assert sum(per) == nnz
        assert max(per) <= nnz / world + lens.max()  # ideal + one row
    # empty tensor and fewer rows than ranks
    assert hq.partition_rows(np.zeros(4, np.uint64), 4).tolist() == [0, 0, 0, 0, 3]
    b = hq.partition_rows(np.array([0, 5, 5, 9], np.uint64), 8)
    assert b[0] == 0 and b[-1] == 3


# ---------------------------------------------------------------- numpy rank --
def _kron_rows(x_vals, other_rows):
    # other_rows: list of (nnz x K_v) gathered factor rows, ascending v != n
    k = other_rows[0] * x_vals[:, None]
    for r in other_rows[1:]:
        k = (k[:, :, None] * r[:, None, :]).reshape(k.shape[0], -1)
    return k


def _core_unfold(core, n):
    return np.moveaxis(core, n, 0).reshape(core.shape[n], -1)


def _core_fold(gn, ranks, n):
    other = [ranks[v] for v in range(len(ranks)) if v != n]
    return np.moveaxis(gn.reshape([ranks[n]] + other), 0, n)


def _rank_solve(rank, world, port, dims, ranks, coords, vals, u0, sweeps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N = len(dims)
    u = [f.copy() for f in u0]
    # initial core: each rank its mode-0 rows, then all-reduce
    core = None

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        return t.numpy()

    def owned(n):
        order = np.argsort(coords[:, n], kind="stable")  # mode-n buckets keep the lexicographic order
        cn = coords[order]
        off = np.zeros(dims[n] + 1, np.uint64)
        np.add.at(off, cn[:, n].astype(np.int64) + 1, 1)
        off = np.cumsum(off).astype(np.uint64)
        b = hq.partition_rows(off, world)
        lo, hi = int(off[b[rank]]), int(off[b[rank + 1]])
        return order[lo:hi], int(b[rank]), int(b[rank + 1])

    def local_y(n, sel):
        others = [v for v in range(N) if v != n]
        rows = [u[v][coords[sel, v]] for v in others]
        kr = _kron_rows(vals[sel], rows)
        y = np.zeros((dims[n], kr.shape[1]))
        np.add.at(y, coords[sel, n].astype(np.int64), kr)
        return y

    sel0, _, _ = owned(0)
    y0 = local_y(0, sel0)
    core = _core_fold(allreduce(u[0].T @ y0), ranks, 0)
    objs = []
    for _ in range(sweeps):
        for n in range(N):
            sel, r0, r1 = owned(n)
            y = local_y(n, sel)[r0:r1]
            a = y @ _core_unfold(core, n).T                    # TTMcTC rows this rank owns
            m = allreduce(a.T @ y)                             # M = A^T Y_(n)
            w = allreduce(a.T @ a)                             # W = A^T A
            r1c = np.linalg.cholesky(w).T
            q1 = np.linalg.solve(r1c.T, a.T).T                 # A R1^-1
            w2 = allreduce(q1.T @ q1)
            r2c = np.linalg.cholesky(w2).T
            rinv = np.linalg.inv(r2c @ r1c)
            unew_loc = a @ rinv
            p = allreduce(unew_loc.T @ u[n][r0:r1])            # drift product
            full = np.zeros_like(u[n])
            full[r0:r1] = unew_loc
            u[n] = allreduce(full)                             # owner rows -> everyone
            core = _core_fold(rinv.T @ m, ranks, n)            # G_(n) = R^-T M
            assert p.shape == (ranks[n], ranks[n])
        objs.append(float(np.sum(core * core)))
    if rank == 0:
        np.savez(out, core=core, objs=np.array(objs), **{f"U{v}": u[v] for v in range(N)})
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", ["h3", "h4"])
def test_row_partitioned_solve_matches_oracle(tmp_path, oracle, name):
    g = golden("hoqri.npz")
    dims = [int(d) for d in g[f"{name}_dims"]]
    ranks = [int(r) for r in g[f"{name}_ranks"]]
    coords = g[f"{name}_coords"].astype(np.int64)
    vals = g[f"{name}_vals"]
    u0 = [g[f"{name}_U0_{m}"] for m in range(len(dims))]
    sweeps = 6
    out = str(tmp_path / "rank0.npz")
    mp.spawn(_rank_solve, args=(2, _free_port(), dims, ranks, coords, vals, u0, sweeps, out), nprocs=2, join=True)
    r = np.load(out)
    ref = oracle.hoqri(dims, ranks, coords.astype(np.uint32), vals, u0, sweeps)
    np.testing.assert_allclose(r["objs"], ref["objective"], rtol=1e-9)
    assert np.linalg.norm(r["core"] - ref["core"]) <= 1e-9 * np.linalg.norm(ref["core"])
    for m in range(len(dims)):
        ug, ur = r[f"U{m}"], ref["factors"][m]
        assert np.sqrt(2) * np.linalg.norm(ug - ur @ (ur.T @ ug)) <= 1e-8
