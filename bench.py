"""HOQRI benchmark (BASELINE.json metric: HOQRI iter/s & TTMcTC nnz/s, FP64).

Workload: BASELINE config 2 — a 10^6 x 10^6 x 10^6 sparse tensor with 10^7
uniform int32 coordinates (duplicates merged), U(0,1) values, Tucker rank
10x10x10 — the largest configuration the north_star scores on one GPU.
A step is one HOQRI sweep (N mode updates: TTMcTC, CholeskyQR2, drift, core
update, objective/fit).  Data is synthetic (seeded PCG64), as the reference's
benchmarks are.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]

engine arm: `value` = sweeps/s with every operand resident in HBM, timed with
CUDA events on the solver's stream; `e2e` = the same metric through the public
API (SparseTensor build from pinned host COO + hoqri() with host init factors,
results copied back), `roofline` for the dominant kernel (the fused sparse
mode pass), `cpu_baseline` = the reference library (oracle/_ref) timed on the
host on a bounded sample.  reference arm: the reference CPU implementation on
all host threads (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CONFIG_ID = 2
SEED_INIT = 20251016
METRIC = "HOQRI iter/s (FP64) — BASELINE config {cfg}"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="engine", choices=["engine", "reference"])
    p.add_argument("--config", type=int, default=CONFIG_ID)
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=1_000_000)
    return p.parse_args()


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload(cfg_id):
    from paper_2510_16930_b200.workloads import CONFIGS, config_coo
    c = CONFIGS[cfg_id]
    coords, vals = config_coo(cfg_id)
    return c, coords, vals


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: an NVML
    polling thread (2 ms period, one sample at start and one at stop, so even a
    30 ms region has samples); nvidia-smi -lms 100 if NVML is unavailable."""
    REASON_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
                   "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.nv = None
        self.samples, self.reasons = [], set()
        self.max_mhz = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = "%08x:%02x:%02x.0" % (getattr(pr, "pci_domain_id", 0), pr.pci_bus_id, pr.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _sample(self):
        nv, h = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        for name, b in self.REASON_BITS.items():
            if bits & b:
                self.reasons.add(name)

    def start(self):
        import threading
        try:
            self.nv = self._handle()
            nv, h = self.nv
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self._sample()
            self._stop = threading.Event()

            def loop():
                while not self._stop.wait(0.002):
                    try:
                        self._sample()
                    except Exception:
                        return
            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.nv is not None:
            self._stop.set()
            self.thread.join(timeout=1)
            try:
                self._sample()
            except Exception:
                pass
            return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx = [], None
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": [],
                "samples": len(sm), "source": "nvidia-smi"}


# ------------------------------------------------------------- FP64 peak --
def fp64_peak_tflops():
    """cuBLAS DGEMM (torch.matmul float64, 8192^3) best of 5: the FP64
    roofline denominator (MEASURED_PEAKS.json carries no FP64 figure)."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn_like(a)
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * n ** 3 / best / 1e9


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {"hbm_gbs": 6650.0, "fallback": True}


# --------------------------------------------------------------- CPU side --
def cpu_reference_sample(x_coords, x_vals, dims, ranks, factors, core, sample, threads, reps=1):
    """Times the UNMODIFIED reference kernels (oracle/_ref) on the first
    `sample` lexicographic nonzeros, split over `threads` host threads, and the
    reference QR at full size once.  Returns per-sweep seconds extrapolated to
    the full nnz, plus the pieces."""
    from oracle_bind import RefLib, RefTensor, Oracle
    nnz = x_vals.size
    S = min(sample, nnz)
    if RefLib.available():
        lib = RefLib()
        kind = "reference"
        t = RefTensor.create(lib, dims, x_coords[:S], x_vals[:S])
        sl = lib.L.ref_slices_create(t.h, threads)
        fl = np.ascontiguousarray(np.concatenate([f.reshape(-1) for f in factors]))
        rk = np.asarray(ranks, np.uint64)
        cd = np.ascontiguousarray(core.reshape(-1))
        t_ttm = min(lib.L.ref_slices_time(sl, rk, fl, cd, 0, 0, 1) for _ in range(reps))
        t_core = min(lib.L.ref_slices_time(sl, rk, fl, cd, 0, 1, 1) for _ in range(reps))
        lib.L.ref_slices_destroy(sl)
        a = np.ascontiguousarray(factors[0])
        t_qr = lib.L.ref_time_qr(a.shape[0], a.shape[1], a.reshape(-1), 1)
    else:  # the C restatement (oracle/hq_oracle.c), single thread
        o = Oracle()
        kind = "port"
        threads = 1
        t0 = time.perf_counter()
        o.ttmctc(dims, ranks, x_coords[:S], x_vals[:S], factors, 0, core)
        t_ttm = time.perf_counter() - t0
        t0 = time.perf_counter()
        o.ttmc_core(dims, ranks, x_coords[:S], x_vals[:S], factors)
        t_core = time.perf_counter() - t0
        t0 = time.perf_counter()
        o.qr(factors[0])
        t_qr = time.perf_counter() - t0
    N = len(dims)
    scale = nnz / S
    sweep_s = N * ((t_ttm + t_core) * scale + t_qr)
    return dict(kind=kind, threads=threads, sample=S, t_ttm=t_ttm, t_core=t_core, t_qr=t_qr, sweep_s=sweep_s,
                ttmctc_nnz_per_s=S / t_ttm)


def host_desc():
    try:
        model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except Exception:
        model = "unknown"
    return model, os.cpu_count()


# ------------------------------------------------------------------ arms --
def run_reference(args, ws, rank):
    if rank != 0:
        return
    c, coords, vals = workload(args.config)
    from oracle_bind import Oracle
    o = Oracle()
    oc, ov = o.normalize(c["dims"], coords, vals) if len(vals) <= 2_000_000 else _merge_numpy(coords, vals)
    factors = _numpy_orthonormal(c["dims"], c["ranks"])
    core = np.random.default_rng(1).standard_normal(int(np.prod(c["ranks"])))
    threads = os.cpu_count() or 1
    sample = max(1, min(args.cpu_sample * max(1, threads // 2), ov.size))
    res = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference_sample(oc, ov, list(c["dims"]), list(c["ranks"]), factors, core, sample, threads)
        if i >= args.warmup:
            res.append(r)
    sweep_s = statistics.median(r["sweep_s"] for r in res)
    value = 1.0 / sweep_s
    model, ncpu = host_desc()
    line = {"impl": "reference", "metric": METRIC.format(cfg=args.config), "value": value, "unit": "iter/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sweep_s * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",  # same fixed workload as the engine arm
            "data": "synthetic (BASELINE config %d, seeded PCG64)" % args.config,
            "config": {"workload": c["name"], "dims": list(c["dims"]), "ranks": list(c["ranks"]),
                       "nnz_merged": int(ov.size)},
            "cpu_baseline": {"value": value, "unit": "iter/s", "cores": res[0]["threads"], "kind": res[0]["kind"],
                             "sample": f"{res[0]['sample']} of {ov.size} nonzeros per step, ttmctc_elementwise + "
                                       f"ttmc_core on {res[0]['threads']} threads (lexicographic slices, one "
                                       f"reference call per thread), qr_orthonormal at full size; sweep = N x "
                                       f"(kernels scaled to full nnz + QR); host: {model}, {ncpu} cores"},
            "ttmctc": {"value": statistics.median(r["ttmctc_nnz_per_s"] for r in res) * res[0]["threads"],
                       "unit": "nnz/s"},
            "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _merge_numpy(coords, vals):
    """Lexicographic sort + duplicate merge with numpy (host, reference-arm
    setup only)."""
    order = np.lexsort(coords.T[::-1])
    c = coords[order]
    v = vals[order]
    head = np.ones(len(c), bool)
    head[1:] = (c[1:] != c[:-1]).any(axis=1)
    idx = np.flatnonzero(head)
    return np.ascontiguousarray(c[head]), np.add.reduceat(v, idx)


def _numpy_orthonormal(dims, ranks, seed=SEED_INIT):
    rng = np.random.default_rng(seed)
    out = []
    for d, k in zip(dims, ranks):
        q, _ = np.linalg.qr(rng.standard_normal((d, k)))
        out.append(np.ascontiguousarray(q))
    return out


def run_engine(args, ws, rank, local):
    import torch
    import torch.distributed as dist
    import paper_2510_16930_b200 as hq

    torch.cuda.set_device(local)
    comm = None
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [hq.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = hq.Comm(ws, rank, uid[0])
    elif os.environ.get("HQ_BENCH_DIST_PATH") == "1":  # test hook: the distributed path on one rank
        comm = hq.Comm(1, 0, hq.nccl_unique_id())
    c, coords, vals = workload(args.config)
    dims, ranks = list(c["dims"]), list(c["ranks"])
    N = len(dims)
    stream = torch.cuda.Stream()  # a real stream: the solver launches (and is timed) on it
    torch.cuda.set_stream(stream)
    x = hq.SparseTensor(dims, coords, vals)
    nnz = x.nnz()
    u0 = hq.random_factors(dims, ranks, SEED_INIT)
    W, K = max(1, args.warmup), max(1, args.steps)
    cfg = hq.SolverConfig(ranks=ranks, max_sweeps=W + K + 1, tol_fit_change=0.0)
    solver = hq.Solver(x, cfg, init_factors=u0.factors, stream=stream.cuda_stream, comm=comm)
    solver.run(W)
    solver.sync()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    solver.run(K)
    # (status read after the timed region)
    e1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    solver.sync()
    dev_status = solver.status()
    if ws > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = K / (ms / 1e3)  # whole-job sweeps of the one tensor (rows partitioned over the ranks)

    # ---- dominant kernel: the fused sparse mode pass, timed per launch
    reps = 10
    pass_ms, flops, bytes_ = [], [], []
    for m in range(N):
        solver.launch_mode_pass(m)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(reps):
            solver.launch_mode_pass(m)
        a1.record(stream)
        torch.cuda.synchronize()
        pass_ms.append(a0.elapsed_time(a1) / reps)
        f, b = solver.mode_pass_work(m)
        flops.append(f)
        bytes_.append(b)
    avg_pass_ms = sum(pass_ms) / N
    avg_flops = sum(flops) / N
    avg_bytes = sum(bytes_) / N
    tflops = avg_flops / (avg_pass_ms * 1e-3) / 1e12
    peak64 = fp64_peak_tflops()
    peaks = measured_peaks()
    ttm_f, ttm_b = solver.ttmctc_work(0)
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = json.load(open(tr_path)).get("configs", {}).get(str(args.config), {}).get("mode_pass_dram_bytes")
        except Exception:
            traffic = None

    # ---- e2e through the public API, host buffers (pinned), 20-sweep solves
    e2e = None
    if args.e2e_steps > 0:
        pc = torch.from_numpy(np.ascontiguousarray(coords)).pin_memory()
        pv = torch.from_numpy(np.ascontiguousarray(vals)).pin_memory()
        pu = [torch.from_numpy(np.ascontiguousarray(f)).pin_memory() for f in u0.factors]
        hc, hv, hu = pc.numpy(), pv.numpy(), [t.numpy() for t in pu]
        sweeps = c["sweeps"]
        ecfg = hq.SolverConfig(ranks=ranks, max_sweeps=sweeps, tol_fit_change=0.0)

        # page-locked result buffers, like the inputs (the D2H is a DMA either way)
        po = [torch.empty((d, k), dtype=torch.float64).pin_memory() for d, k in zip(dims, ranks)]
        pcore = torch.empty(int(np.prod(ranks)), dtype=torch.float64).pin_memory()
        hout = ([t.numpy() for t in po], pcore.numpy())

        def e2e_step():
            xe = hq.SparseTensor(dims, hc, hv)  # H2D of the COO + device layout build
            se = hq.Solver(xe, ecfg, init_factors=hu, stream=stream.cuda_stream, comm=comm)  # H2D of the factors
            se.run(sweeps)
            r = se.download(out=hout)  # D2H of factors, core, trace
            del se, xe
            return r

        for _ in range(2):  # warm: the first solves also grow the device memory pool to its working set
            r = e2e_step()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        t0 = time.perf_counter()
        step_s = []
        for _ in range(args.e2e_steps):
            ts = time.perf_counter()
            r = e2e_step()
            step_s.append(time.perf_counter() - ts)
        dt = time.perf_counter() - t0
        if ws > 1:
            t = torch.tensor([dt], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        h2d = hc.nbytes + hv.nbytes + sum(a.nbytes for a in hu)
        d2h = sum(f.nbytes for f in r.model.factors.factors) + r.model.core.data.nbytes + 8 * (2 + N) * sweeps
        e2e = {"value": args.e2e_steps * sweeps / dt, "unit": "iter/s", "h2d_bytes_per_step": int(h2d),
               "solve_s": [round(x, 4) for x in step_s],
               "d2h_bytes_per_step": int(d2h),
               "step": f"one full {sweeps}-sweep solve through the C-ABI from pinned host buffers: SparseTensor "
                       f"build (COO upload, device sort/merge/buckets) + init factors upload + {sweeps} sweeps + "
                       f"factors/core/trace download (wall clock, max over ranks)"}

    cpu = None
    if rank == 0 and not args.no_cpu:
        st = solver.download()
        core = st.model.core.data
        cpu = cpu_reference_sample(x.coords(), x.values(), dims, ranks, st.model.factors.factors, core,
                                   args.cpu_sample, 1)

    if rank != 0:
        return
    model, ncpu = host_desc()
    line = {
        "metric": METRIC.format(cfg=args.config), "value": value, "unit": "iter/s", "n_gpus": ws, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config %d: uniform int32 coords, U(0,1) values, seeded PCG64; duplicates "
                "merged on device)" % args.config,
        "config": {"workload": c["name"], "dims": dims, "ranks": ranks, "draws": c["draws"], "nnz_merged": nnz,
                   "step": "one HOQRI sweep (N mode updates)",
                   "parallelism": f"row-partitioned x{ws} (NCCL all-reduce + owner broadcast)" if ws > 1 else "single GPU",
                   "l2": "inputs larger than L2 (mode streams %.0f MB + factors %.0f MB vs 126 MB L2)" %
                         (nnz * (4 * (N - 1) + 8) * N / 1e6, sum(d * k for d, k in zip(dims, ranks)) * 8 * 2 / 1e6)},
        "ttmctc": {"value": nnz / (avg_pass_ms * 1e-3), "unit": "nnz/s",
                   "note": "fused mode pass (TTMcTC + Gram + core projection) per launch, mean over modes"},
        "roofline": {"bound": "tensor", "achieved": tflops, "peak": peak64, "unit": "TFLOP/s",
                     "frac": tflops / peak64, "traffic": traffic,
                     "kernel": "fused sparse mode pass (hq_pass: short-row tiles + long-row segment/fix-up kernels)",
                     "flops_per_launch": avg_flops, "bytes_per_launch": avg_bytes, "launch_ms": avg_pass_ms,
                     "per_mode_ms": pass_ms,
                     "hbm": {"achieved_gbs": avg_bytes / (avg_pass_ms * 1e-3) / 1e9, "peak_gbs": peaks.get("hbm_gbs"),
                             "frac": avg_bytes / (avg_pass_ms * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6535.7)},
                     "peak_source": "FP64: cuBLAS DGEMM 8192^3 measured in this run (MEASURED_PEAKS.json has no "
                                    "FP64 entry); HBM: MEASURED_PEAKS.json",
                     "ttmctc_canonical": {"flops": ttm_f, "bytes": ttm_b,
                                          "frac_of_fp64_peak": ttm_f / (avg_pass_ms * 1e-3) / 1e12 / peak64}},
        "solver_status": dev_status,
        "gpu_launches": solver.launches_per_sweep() * K,
        "clocks": clk,
    }
    if e2e:
        line["e2e"] = e2e
    if cpu:
        line["cpu_baseline"] = {
            "value": 1.0 / cpu["sweep_s"], "unit": "iter/s", "cores": cpu["threads"], "kind": cpu["kind"],
            "sample": f"reference ttmctc_elementwise + ttmc_core on the first {cpu['sample']} of {nnz} nonzeros "
                      f"({cpu['t_ttm']:.2f} s + {cpu['t_core']:.2f} s), qr_orthonormal+drift at full size "
                      f"({cpu['t_qr']:.2f} s); sweep = N x (kernels x nnz/sample + QR) = {cpu['sweep_s']:.1f} s; "
                      f"1 thread of {ncpu} ({model})",
            "ttmctc_nnz_per_s": cpu["ttmctc_nnz_per_s"]}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_engine(args, ws, rank, local)


if __name__ == "__main__":
    main()
