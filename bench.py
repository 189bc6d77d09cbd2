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
mode pass), `ttmctc` = SURVEY 8(d)'s standalone TTMcTC nnz/s, `sweep_roofline`
= the sweep against SURVEY 8(d)'s canonical T_iter, `cpu_baseline` = one
full-size mode update of the unmodified reference (oracle/_ref), 1 thread.
reference arm (rank 0 only): K full-size mode updates of the unmodified
reference's solve loop, each timed as it runs.  `--gpus N` without torchrun
re-launches itself with N ranks.
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
def cpu_baseline_measure(coords, vals, dims, ranks, factors):
    """cpu_baseline: ONE full-size mode update (mode 0) of the reference's solve
    loop, timed as it runs (oracle/_ref, 1 thread; see reference_mode_updates);
    sweep = N x that (the configs' modes have equal nnz; the reference arm times
    every mode).  Without oracle/_ref: the C restatement (oracle/hq_oracle.c) of
    the same calls at full size ("port")."""
    from oracle_bind import RefLib, Oracle
    N = len(dims)
    if RefLib.available():
        r = reference_mode_updates(coords, vals, dims, ranks, factors, 1, 0)
        t = r["steps_s"][0]
        return dict(kind="reference", sweep_s=N * t, step_s=t, phases=r["phases"][0], nnz=r["nnz"],
                    ttmctc_nnz_per_s=r["nnz"] / r["phases"][0]["ttmctc"])
    o = Oracle()
    t0 = time.perf_counter()
    core = o.ttmc_core(dims, ranks, coords, vals, factors)
    t1 = time.perf_counter()
    a = o.ttmctc(dims, ranks, coords, vals, factors, 0, core)
    t2 = time.perf_counter()
    o.qr(a)
    t3 = time.perf_counter()
    t = t3 - t0
    return dict(kind="port", sweep_s=N * t, step_s=t, nnz=len(vals),
                phases={"ttmctc": t2 - t1, "qr": t3 - t2, "core": t1 - t0}, ttmctc_nnz_per_s=len(vals) / (t2 - t1))


def sweep_roofline(solver, dims, ranks, nnz, bw_gbs, p64_tflops):
    """T_iter,roof = sum_n [T(TTMcTC_n) + T(core_n) + T(QR_n)],
    T = max(B / BW, F / P64) with the canonical (minimal) F and B."""
    N = len(dims)
    bw, p64 = bw_gbs * 1e9, p64_tflops * 1e12
    tot, parts = 0.0, []
    for n in range(N):
        f, b = solver.ttmctc_work(n)  # F = 2 nnz L + 2 R_n prod K, B = nnz(4N+8) + 8 sum_{v!=n} I_v K_v + 8 I_n K_n
        t_ttm = max(b / bw, f / p64)
        b_core = b - 8.0 * dims[n] * ranks[n] + 8.0 * dims[n] * ranks[n] + 8.0 * float(np.prod(ranks))
        t_core = max(b_core / bw, f / p64)
        t_qr = max(24.0 * dims[n] * ranks[n] / bw, 8.0 * dims[n] * ranks[n] ** 2 / p64)
        parts.append({"ttmctc_us": t_ttm * 1e6, "core_us": t_core * 1e6, "qr_us": t_qr * 1e6})
        tot += t_ttm + t_core + t_qr
    return tot, parts


def host_desc():
    try:
        model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except Exception:
        model = "unknown"
    return model, os.cpu_count()


# ------------------------------------------------------------------ arms --
def reference_mode_updates(coords, vals, dims, ranks, factors, steps, warmup, sample_warm=100_000):
    """The UNMODIFIED reference (oracle/_ref) on the GPU box's host: `steps`
    full-size mode updates of tucker::hoqri's loop (ref_capi.cpp
    ref_state_mode_update: ttmctc_elementwise with the fresh core, max_abs,
    qr_orthonormal, subspace_distance, ttmc_core -- solvers.cpp:86-146), mode
    n = step mod N, one thread.  Nothing is sampled or extrapolated: each step
    is timed as it runs.  The `warmup` steps run on a prefix of the nonzeros
    (they only fault pages in).  Returns per-step seconds and phase times."""
    from oracle_bind import RefLib, RefTensor, RefSolveState
    lib = RefLib()
    N = len(dims)
    if warmup:
        tw = RefTensor.create(lib, dims, coords[:sample_warm], vals[:sample_warm])
        sw = RefSolveState(tw, ranks, factors)
        for i in range(warmup):
            sw.mode_update(i % N)
        del sw, tw
    t0 = time.perf_counter()
    t = RefTensor.create(lib, dims, coords, vals)  # the reference's SparseTensor ctor (sort + merge + buckets)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    st = RefSolveState(t, ranks, factors)  # initial core, solvers.cpp:66
    t_init = time.perf_counter() - t0
    steps_s, phases = [], []
    for i in range(steps):
        t0 = time.perf_counter()
        _, ph = st.mode_update(i % N)
        steps_s.append(time.perf_counter() - t0)
        phases.append(ph)
    return dict(steps_s=steps_s, phases=phases, t_build=t_build, t_init=t_init, nnz=t.nnz)


def bench_config(c, dims, ranks, nnz, ws):
    """The `config` / `data` entries of the JSON line -- the same for both arms (the reference arm measures the
    engine arm's workload; what one of its timed steps covers is its `sample_step`)."""
    N = len(dims)
    config = {"workload": c["name"], "dims": dims, "ranks": ranks, "draws": c["draws"], "nnz_merged": int(nnz),
              "step": "one HOQRI sweep (N mode updates)",
              "parallelism": (f"row-partitioned x{ws} (NCCL all-reduces; QR apply + all-gather of the new factor "
                              f"fused over peer memory)") if ws > 1 else "single GPU",
              "l2": "%s (mode streams %.0f MB + factors %.0f MB vs 126 MB L2)" %
                    ("inputs larger than L2" if nnz * (4 * (N - 1) + 8) * N > 126e6 else
                     "inputs SMALLER than L2: a parity-test size, not a bench configuration",
                     nnz * (4 * (N - 1) + 8) * N / 1e6, sum(d * k for d, k in zip(dims, ranks)) * 8 * 2 / 1e6)}
    kind = {"uniform": "uniform int32 coords, U(0,1) values",
            "lognormal": "Zipf(%s) mode indices over seeded permutations, lognormal(0,1) values" % c.get("zipf_s"),
            "planted": "uniform int32 coords, planted rank-%d Tucker model + %g Gaussian noise" %
                       (ranks[0], c.get("noise", 0.0))}[c["values"]]
    data = "synthetic (BASELINE %s: %s; seeded PCG64; duplicates merged)" % (c["name"].split("_")[0], kind)
    return config, data


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref = the unmodified reference library), rank 0 only.  A step is
    ONE full-size mode update of the reference's solve loop (1/N of a sweep);
    value = sweeps/s = K / (N x the K steps' wall time)."""
    if rank != 0:
        return
    c, coords, vals = workload(args.config)
    from oracle_bind import RefLib, ref_random_factors
    dims, ranks = list(c["dims"]), list(c["ranks"])
    N = len(dims)
    K, W = max(1, args.steps), max(0, args.warmup)
    u0 = ref_random_factors(RefLib(), dims, ranks, SEED_INIT)  # tucker::random_factors, the engine arm's init
    r = reference_mode_updates(coords, vals, dims, ranks, u0, K, W)
    total = sum(r["steps_s"])
    value = (K / N) / total
    model, ncpu = host_desc()
    ttm = [p["ttmctc"] for p in r["phases"]]
    config, data = bench_config(c, dims, ranks, r["nnz"], ws)
    line = {"impl": "reference", "metric": METRIC.format(cfg=args.config), "value": value, "unit": "iter/s",
            "n_gpus": ws, "steps": K, "warmup": W, "ms_per_step": total / K * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": data, "config": config,
            "sample_step": f"a timed step of this arm is one full-size mode update of tucker::hoqri's loop (1/{N} of "
                           "a sweep): ttmctc_elementwise(core given) + max_abs + qr_orthonormal + "
                           "subspace_distance + ttmc_core on every nonzero; value = sweeps/s over the timed steps",
            "cpu_baseline": {"value": value, "unit": "iter/s", "cores": 1, "kind": "reference",
                             "sample": f"none: {K} full-size mode updates ({K / N:.2f} sweeps) of the unmodified "
                                       f"reference, each timed as it ran (steady_clock); the reference is "
                                       f"single-threaded (kernels.cpp has no threading), so 1 thread of {ncpu} "
                                       f"host cores ({model}); warm-up steps ran on a 1e5-nonzero prefix",
                             "phase_s_mean": {k: statistics.mean(p[k] for p in r["phases"]) for k in r["phases"][0]},
                             "setup_s": {"sparse_tensor_ctor": r["t_build"], "initial_ttmc_core": r["t_init"]}},
            "ttmctc": {"value": r["nnz"] / statistics.median(ttm), "unit": "nnz/s",
                       "note": "median of the timed steps' ttmctc_elementwise calls (core given), full nnz"},
            "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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
    if comm is not None and ws > 1:
        x.shard(comm)  # each rank keeps only its rows' streams (SPEC.md:247 row partition)
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
    if ws > 1:
        # a multi-GPU update that is not plain CholeskyQR2 (shifted / rank-deficient) is finished by a
        # host-driven continuation inside sync(): it belongs to the timed sweeps
        solver.sync()
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
    # ---- SURVEY 8(d) TTMcTC nnz/s: the standalone TTMcTC call with the core given (kernels.cpp:86-163 with
    # precomputed_core), median of 10 CUDA-event-timed calls per mode
    ttm_ms = []
    for m in range(N):
        for _ in range(2):
            solver.launch_ttmctc(m)
        ts = []
        for _ in range(10):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            solver.launch_ttmctc(m)
            a1.record(stream)
            a1.synchronize()
            ts.append(a0.elapsed_time(a1))
        ttm_ms.append(statistics.median(ts))
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
            if comm is not None and ws > 1:
                xe.shard(comm)
            se = hq.Solver(xe, ecfg, init_factors=hu, stream=stream.cuda_stream, comm=comm)  # H2D of the factors
            se.run(sweeps)
            r = se.download(out=hout)  # D2H of factors, core, trace
            del se, xe
            return r

        for _ in range(2):  # warm: the first solves also fill the engine's device block cache with the working set
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
        cpu = cpu_baseline_measure(coords, vals, dims, ranks, st.model.factors.factors)  # the reference merges
    t_roof, roof_parts = sweep_roofline(solver, dims, ranks, nnz, peaks.get("hbm_gbs", 6535.7), peak64)
    ttm_canon = [solver.ttmctc_work(m) for m in range(N)]

    if rank != 0:
        return
    model, ncpu = host_desc()
    config, data = bench_config(c, dims, ranks, nnz, ws)
    line = {
        "metric": METRIC.format(cfg=args.config), "value": value, "unit": "iter/s", "n_gpus": ws, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": data, "config": config,
        "ttmctc": {"value": nnz / (statistics.mean(ttm_ms) * 1e-3), "unit": "nnz/s",
                   "per_mode_ms": ttm_ms,
                   "note": "SURVEY 8(d): standalone TTMcTC (core given; G_(n)^T unfold + A only), median of 10 "
                           "CUDA-event-timed calls per mode; value = nnz / mean of the per-mode medians",
                   "roofline_frac_per_mode": [max(b / (peaks.get("hbm_gbs", 6535.7) * 1e9), f / (peak64 * 1e12)) /
                                              (t * 1e-3) for (f, b), t in zip(ttm_canon, ttm_ms)],
                   "fp64_frac_per_mode": [f / (t * 1e-3) / 1e12 / peak64 for (f, b), t in zip(ttm_canon, ttm_ms)]},
        "fused_pass": {"value": nnz / (avg_pass_ms * 1e-3), "unit": "nnz/s", "per_mode_ms": pass_ms,
                       "note": "the solver's fused mode pass (TTMcTC + M = A^T Y + W = A^T A + max|A|) per launch"},
        "sweep_roofline": {"t_roof_us": t_roof * 1e6, "iter_per_s_roof": 1.0 / t_roof,
                           "frac": value * t_roof, "per_mode": roof_parts,
                           "note": "SURVEY 8(d): sum over modes of max(B/BW, F/P64) for TTMcTC + core + QR, "
                                   "canonical minimal F and B; BW = MEASURED_PEAKS hbm_gbs, P64 = live DGEMM"},
        "drift_note": "the drift's K x K nuclear norms (Jacobi SVD) are evaluated at download, outside the timed "
                      "region (< 0.2 % of a sweep); P = U_new^T U_old itself is computed inside every sweep",
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
            "value": 1.0 / cpu["sweep_s"], "unit": "iter/s", "cores": 1, "kind": cpu["kind"],
            "sample": f"one full-size mode update (mode 0, all {cpu['nnz']} nonzeros) of the reference's solve "
                      f"loop, timed as it ran: " + ", ".join(f"{k} {v:.2f} s" for k, v in cpu["phases"].items()) +
                      f"; sweep = {N} x {cpu['step_s']:.1f} s; 1 thread of {ncpu} ({model}); the reference is "
                      f"single-threaded",
            "ttmctc_nnz_per_s": cpu["ttmctc_nnz_per_s"]}
    print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """`--gpus N` without a launcher: re-exec this script under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args)
    ws, rank, local = dist_setup(args)
    if ws != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch with --nproc-per-node {args.gpus}")
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_engine(args, ws, rank, local)


if __name__ == "__main__":
    main()
