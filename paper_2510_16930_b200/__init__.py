"""B200-native HOQRI engine: Python mirror of the reference's `tucker::` API.

The reference (arxiv 2510.16930, /root/reference/proj) is a C++ library whose
public API is proj/include/tucker/*.hpp.  This module binds the engine's C-ABI
(include/hoqri_b200.h, lib/libhoqri_b200.so) with ctypes and exposes the same
names, argument meanings and error types, so the parity tests read like the
reference's own tests:

    SparseTensor(dims, coords, values)        sparse_tensor.hpp:37-57
    load_tns / write_tns                      sparse_tensor.hpp:76-83
    norm_sq(SparseTensor | CoreTensor)        sparse_tensor.hpp:69, dense_core.hpp:48
    ttmc_core(x, u)                           kernels.hpp:46
    ttmctc_elementwise(x, u, mode, core)      kernels.hpp:52-54
    ttmctc_matrix(x, u, mode)                 kernels.hpp:59-60
    qr_orthonormal(a)                         dense_core.hpp:60
    subspace_distance(u, v)                   manifold.hpp:34-36
    random_factors(dims, ranks, seed)         solvers.hpp:72-73
    hoqri(x, config)                          solvers.hpp:80
    fit_error(x, model)                       solvers.hpp:87

All compute runs in the CUDA engine.  There is no CPU fallback: importing
works without a GPU (so the C-ABI can be inspected), but every compute call
raises when the engine cannot run.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import List, Optional, Sequence

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libhoqri_b200.so")

# ---------------------------------------------------------------- errors --
# errors.hpp:9-70


class Error(RuntimeError):
    pass


class ShapeError(Error):
    pass


class RangeError(Error):
    pass


class ValueError_(Error):
    pass


class ParseError(Error):
    def __init__(self, what, line_number=0):
        super().__init__(f"line {line_number}: {what}" if line_number else what)
        self.line_number = line_number


class CapacityError(Error):
    pass


class ContractError(Error):
    pass


class DiagnosticError(Error):
    pass


class DegenerateStateError(Error):
    def __init__(self, mode_1based, what=None):
        super().__init__(what or f"degenerate state: TTMcTC output is identically zero for mode {mode_1based}")
        self.mode = mode_1based


class InfeasibleError(Error):
    pass


class DeviceError(Error):
    """CUDA / NCCL failure inside the engine."""


_STATUS = {1: ShapeError, 2: RangeError, 3: ValueError_, 5: CapacityError, 6: ContractError, 7: DiagnosticError,
           9: InfeasibleError, 10: DeviceError, 11: DeviceError, 12: Error}

# ----------------------------------------------------------------- C-ABI --
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class HqConfig(C.Structure):
    _fields_ = [("order", C.c_int), ("ranks", C.c_uint64 * 8), ("max_sweeps", C.c_uint64),
                ("tol_fit_change", C.c_double), ("seed", C.c_uint64), ("init", C.c_int), ("kernel", C.c_int),
                ("trace_gradients", C.c_int), ("tol_grad", C.c_double), ("capacity_cap", C.c_uint64)]


class HqTrace(C.Structure):
    _fields_ = [("data_norm_sq", C.c_double), ("initial_objective", C.c_double), ("sweeps", C.c_uint64),
                ("objective", C.c_void_p), ("fit", C.c_void_p), ("drift", C.c_void_p),
                ("grad_norm_sq", C.c_void_p), ("elapsed_s", C.c_void_p),
                ("upd_f_before", C.c_void_p), ("upd_f_after", C.c_void_p), ("upd_elapsed_s", C.c_void_p),
                ("upd_sigma", C.c_void_p), ("upd_lambda", C.c_void_p), ("sigma_stride", C.c_uint64),
                ("updates", C.c_uint64)]


EXPORTED_SYMBOLS = [
    "hq_last_error", "hq_last_error_payload", "hq_version", "hq_release_cached_memory",
    "hq_tensor_create", "hq_tensor_create_dev", "hq_tensor_destroy", "hq_tensor_info", "hq_tensor_mode_plan",
    "hq_tensor_fiber_plan", "hq_tensor_export",
    "hq_tensor_buckets", "hq_tensor_norm_sq",
    "hq_ttmc_core", "hq_ttmctc", "hq_qr_orthonormal", "hq_subspace_distance", "hq_random_factors",
    "hq_config_default", "hq_hoqri", "hq_fit_error",
    "hq_solver_create", "hq_solver_destroy", "hq_solver_run", "hq_solver_sync", "hq_solver_status", "hq_solver_launch_mode_pass",
    "hq_solver_launch_ttmctc", "hq_solver_launches_per_sweep", "hq_solver_download", "hq_solver_mode_pass_work",
    "hq_solver_ttmctc_work", "hq_nccl_unique_id", "hq_comm_create", "hq_comm_destroy", "hq_partition_rows",
    "hq_comm_create_host", "hq_tensor_shard",
    "hq_solver_create_dist", "hq_bench_ttmctc", "hq_gen_synthetic",
    "hq_tns_parse", "hq_tns_parse_file", "hq_tns_info", "hq_tns_copy", "hq_tns_tensor", "hq_tns_destroy",
    "hq_densify_unfold", "hq_ttmc_unfold_dense", "hq_svd_leading", "hq_init_factors", "hq_hooi",
    "hq_sym_eig",
]

_lib = None


def load_library(path: str = None) -> C.CDLL:
    """Loads lib/libhoqri_b200.so (builds it in-tree first if it is missing).
    HQ_LIB overrides the path (kernel-variant experiments)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("HQ_LIB") or LIB_PATH
    if not os.path.exists(path):
        from . import build
        build.build_engine()
    L = C.CDLL(path)
    vp, pp = C.c_void_p, C.POINTER(C.c_void_p)
    L.hq_last_error.restype = C.c_char_p
    L.hq_last_error_payload.restype = C.c_int64
    L.hq_version.restype = C.c_char_p
    L.hq_tensor_create.argtypes = [C.c_int, _u64p, C.c_uint64, vp, vp, vp, pp]
    L.hq_tensor_create_dev.argtypes = [C.c_int, _u64p, C.c_uint64, vp, vp, vp, pp]
    L.hq_tensor_destroy.argtypes = [vp]
    L.hq_tensor_info.argtypes = [vp, C.POINTER(C.c_int), _u64p, C.POINTER(C.c_uint64)]
    L.hq_tensor_mode_plan.argtypes = [vp, C.c_int] + [C.POINTER(C.c_uint64)] * 4 + [C.POINTER(C.c_int),
                                                                                    C.POINTER(C.c_uint64)]
    L.hq_tensor_fiber_plan.argtypes = [vp, C.c_int] + [C.POINTER(C.c_uint64)] * 4
    L.hq_tensor_export.argtypes = [vp, vp, vp]
    L.hq_tensor_buckets.argtypes = [vp, C.c_int, _u64p, vp]
    L.hq_tensor_norm_sq.argtypes = [vp, C.POINTER(C.c_double)]
    L.hq_ttmc_core.argtypes = [vp, vp, _u64p, _f64p]
    L.hq_ttmctc.argtypes = [vp, vp, _u64p, C.c_int, vp, C.c_int, _f64p]
    L.hq_qr_orthonormal.argtypes = [C.c_uint64, C.c_uint64, _f64p, _f64p]
    L.hq_subspace_distance.argtypes = [C.c_uint64, C.c_uint64, _f64p, _f64p, C.POINTER(C.c_double)]
    L.hq_random_factors.argtypes = [C.c_int, _u64p, _u64p, C.c_uint64, vp]
    L.hq_config_default.argtypes = [C.POINTER(HqConfig)]
    L.hq_config_default.restype = None
    L.hq_hoqri.argtypes = [vp, C.POINTER(HqConfig), vp, vp, vp, C.POINTER(HqTrace)]
    L.hq_fit_error.argtypes = [C.c_double, C.c_uint64, _f64p, C.POINTER(C.c_double)]
    L.hq_bench_ttmctc.argtypes = [vp, pp, _u64p, C.c_int, C.c_uint64, _f64p, _u64p]
    L.hq_gen_synthetic.argtypes = [C.c_int, _u64p, C.c_uint64, C.c_uint64, C.c_void_p, _f64p]
    L.hq_tns_parse.argtypes = [C.c_char_p, C.c_uint64, C.c_int, vp, pp]
    L.hq_tns_parse_file.argtypes = [C.c_char_p, C.c_int, vp, pp]
    L.hq_tns_info.argtypes = [vp, C.POINTER(C.c_int), vp, C.POINTER(C.c_uint64)]
    L.hq_tns_copy.argtypes = [vp, vp, vp]
    L.hq_tns_tensor.argtypes = [vp, vp, pp]
    L.hq_tns_destroy.argtypes = [vp]
    L.hq_densify_unfold.argtypes = [vp, C.c_int, C.c_uint64, _f64p]
    L.hq_ttmc_unfold_dense.argtypes = [vp, vp, _u64p, C.c_int, C.c_uint64, _f64p]
    L.hq_svd_leading.argtypes = [C.c_uint64, C.c_uint64, _f64p, C.c_uint64, _f64p]
    L.hq_init_factors.argtypes = [vp, C.POINTER(HqConfig), vp]
    L.hq_sym_eig.argtypes = [C.c_uint64, _f64p, _f64p, vp]
    L.hq_hooi.argtypes = [vp, C.POINTER(HqConfig), vp, vp, vp, C.POINTER(HqTrace)]
    L.hq_solver_create.argtypes = [vp, C.POINTER(HqConfig), vp, vp, pp]
    L.hq_solver_destroy.argtypes = [vp]
    L.hq_solver_run.argtypes = [vp, C.c_uint64]
    L.hq_solver_sync.argtypes = [vp]
    L.hq_solver_status.argtypes = [vp, C.POINTER(C.c_int64)]
    L.hq_solver_launch_mode_pass.argtypes = [vp, C.c_int]
    L.hq_solver_launch_ttmctc.argtypes = [vp, C.c_int]
    L.hq_solver_launches_per_sweep.argtypes = [vp, C.POINTER(C.c_uint64)]
    L.hq_solver_download.argtypes = [vp, vp, vp, C.POINTER(HqTrace)]
    L.hq_solver_mode_pass_work.argtypes = [vp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.hq_solver_ttmctc_work.argtypes = [vp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.hq_nccl_unique_id.argtypes = [vp]
    L.hq_comm_create.argtypes = [C.c_int, C.c_int, vp, pp]
    L.hq_comm_destroy.argtypes = [vp]
    L.hq_comm_create_host.argtypes = [C.c_int, C.c_int, C.c_char_p, C.c_uint64, pp]
    L.hq_tensor_shard.argtypes = [vp, vp]
    L.hq_partition_rows.argtypes = [_u64p, C.c_uint64, C.c_int, _u64p]
    L.hq_solver_create_dist.argtypes = [vp, C.POINTER(HqConfig), vp, vp, vp, pp]
    _lib = L
    return L


def _check(status: int):
    if status == 0:
        return
    L = load_library()
    msg = L.hq_last_error().decode(errors="replace")
    payload = int(L.hq_last_error_payload())
    if status == 8:
        raise DegenerateStateError(payload, msg)
    if status == 4:
        raise ParseError(msg, payload)
    raise _STATUS.get(status, Error)(msg)


def _ptr_array(arrs):
    a = (C.c_void_p * max(1, len(arrs)))()
    for i, x in enumerate(arrs):
        a[i] = x.ctypes.data
    return a


# ----------------------------------------------------------------- types --
@dataclasses.dataclass
class CoreTensor:
    """Dense core, lexicographic layout with the last mode fastest (dense_core.hpp:33-43)."""
    ranks: List[int]
    data: np.ndarray

    def order(self):
        return len(self.ranks)

    def size(self):
        return int(self.data.size)

    def as_array(self):
        return self.data.reshape(tuple(self.ranks))


@dataclasses.dataclass
class FactorSet:
    """Per-mode factors, factor n of shape I_n x K_n (dense_core.hpp:45-54)."""
    factors: List[np.ndarray]

    def order(self):
        return len(self.factors)

    def orthonormality_defect(self):
        worst = 0.0
        for u in self.factors:
            g = u.T @ u
            worst = max(worst, float(np.abs(g - np.eye(g.shape[0])).max()) if g.size else 0.0)
        return worst


class SparseTensor:
    """Device-resident COO tensor (sparse_tensor.hpp:20-66).  Construction
    validates, sorts, merges duplicates and builds all mode layouts on the GPU."""

    def __init__(self, dims: Sequence[int], coords, values, *, _handle=None):
        L = load_library()
        self._dims = [int(d) for d in dims]
        if _handle is not None:
            self._h = _handle
        else:
            d = np.ascontiguousarray(np.asarray(self._dims, dtype=np.uint64))
            c = np.ascontiguousarray(np.asarray(coords, dtype=np.uint32)).reshape(-1)
            v = np.ascontiguousarray(np.asarray(values, dtype=np.float64)).reshape(-1)
            n = len(self._dims)
            if n == 0:
                raise ShapeError("sparse tensor needs at least one mode")
            if c.size != v.size * n:
                raise ShapeError("coordinate array does not match entry count")
            h = C.c_void_p()
            _check(L.hq_tensor_create(n, d, v.size, c.ctypes.data if c.size else None,
                                      v.ctypes.data if v.size else None, None, C.byref(h)))
            self._h = h
        order = C.c_int(0)
        nnz = C.c_uint64(0)
        dd = np.zeros(8, np.uint64)
        _check(L.hq_tensor_info(self._h, C.byref(order), dd, C.byref(nnz)))
        self._nnz = int(nnz.value)
        self._coords = None
        self._values = None

    @classmethod
    def from_device(cls, dims, coords_ptr: int, values_ptr: int, nnz: int, stream: int = 0):
        """Builds from COO already in device memory (e.g. torch tensors' data_ptr())."""
        L = load_library()
        d = np.ascontiguousarray(np.asarray(dims, dtype=np.uint64))
        h = C.c_void_p()
        _check(L.hq_tensor_create_dev(d.size, d, nnz, coords_ptr, values_ptr, stream or None, C.byref(h)))
        return cls(dims, None, None, _handle=h)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                load_library().hq_tensor_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def order(self):
        return len(self._dims)

    def dims(self):
        return list(self._dims)

    def nnz(self):
        return self._nnz

    def shard(self, comm: "Comm"):
        """Keep only this rank's rows of every mode stream (the distributed solver's row partition); the
        tensor is then usable only with a Solver on `comm`."""
        _check(load_library().hq_tensor_shard(self.handle, comm._h))
        self._sharded = True
        return self

    def mode_plan(self, mode):
        """Engine work plan of one mode's unfolding: rows, nonempty_rows, long_rows (> 256 nonzeros),
        long_segments, hot (skewed mode: its factor is gathered L1-allocating by the other passes), max_tile32
        (most short-row nonzeros in one 32-row tile)."""
        v = [C.c_uint64() for _ in range(5)]
        hot = C.c_int()
        _check(load_library().hq_tensor_mode_plan(self._h, int(mode), *[C.byref(x) for x in v[:4]], C.byref(hot),
                                                  C.byref(v[4])))
        return dict(rows=v[0].value, nonempty_rows=v[1].value, long_rows=v[2].value, long_segments=v[3].value,
                    hot=bool(hot.value), max_tile32=v[4].value)

    def fiber_plan(self, mode):
        """Fiber units of one mode's long rows (order 3, skewed tensors): units (0 = not used), long_nnz (the
        long rows' nonzeros the units cover), the derived stream's segments, and short_max (the mode's
        long-row threshold)."""
        v = [C.c_uint64() for _ in range(4)]
        _check(load_library().hq_tensor_fiber_plan(self._h, int(mode), *[C.byref(x) for x in v]))
        return dict(units=v[0].value, long_nnz=v[1].value, segments=v[2].value, short_max=v[3].value)

    def _export(self):
        if self._coords is None:
            c = np.empty(max(1, self._nnz * self.order()), np.uint32)
            v = np.empty(max(1, self._nnz), np.float64)
            _check(load_library().hq_tensor_export(self._h, c.ctypes.data, v.ctypes.data))
            self._coords = c[: self._nnz * self.order()].reshape(self._nnz, self.order())
            self._values = v[: self._nnz]
        return self._coords, self._values

    def values(self):
        return self._export()[1]

    def coords(self):
        return self._export()[0]

    def value(self, e):
        return float(self.values()[e])

    def coord(self, e, mode):
        return int(self.coords()[e, mode])

    def coord_row(self, e):
        return self.coords()[e]

    def buckets_built(self):
        return True

    def mode_bucket(self, mode):
        """(offsets[I_n + 1], entries[nnz]) as in ModeBuckets (sparse_tensor.hpp:25-32)."""
        off = np.empty(self._dims[mode] + 1, np.uint64)
        ent = np.empty(max(1, self._nnz), np.uint64)
        _check(load_library().hq_tensor_buckets(self._h, mode, off, ent.ctypes.data))
        return off, ent[: self._nnz]


def release_cached_memory() -> int:
    """Returns the device buffers the engine keeps for its next solve to the driver; the bytes freed
    (hq_release_cached_memory)."""
    L = load_library()
    freed = C.c_uint64(0)
    _check(L.hq_release_cached_memory(C.byref(freed)))
    return int(freed.value)


def norm_sq(x):
    if isinstance(x, SparseTensor):
        out = C.c_double(0)
        _check(load_library().hq_tensor_norm_sq(x.handle, C.byref(out)))
        return out.value
    if isinstance(x, CoreTensor):
        return float(np.dot(x.data, x.data))
    raise TypeError("norm_sq expects a SparseTensor or CoreTensor")


def _factors_of(u):
    fs = u.factors if isinstance(u, FactorSet) else list(u)
    return [np.ascontiguousarray(np.asarray(f, dtype=np.float64)) for f in fs]


def _check_factors(x: SparseTensor, fs):
    # kernels.cpp:12-22
    if len(fs) != x.order():
        raise ShapeError("factor count does not match tensor order")
    for n, f in enumerate(fs):
        if f.ndim != 2 or f.shape[0] != x.dims()[n]:
            raise ShapeError(f"factor {n + 1} has {f.shape[0]} rows, tensor extent is {x.dims()[n]}")
        if f.shape[1] == 0:
            raise ShapeError("factor with zero columns")


def ttmc_core(x: SparseTensor, u) -> CoreTensor:
    fs = _factors_of(u)
    _check_factors(x, fs)
    ranks = np.array([f.shape[1] for f in fs], np.uint64)
    out = np.empty(int(np.prod(ranks)), np.float64)
    _check(load_library().hq_ttmc_core(x.handle, _ptr_array(fs), ranks, out))
    return CoreTensor([int(r) for r in ranks], out)


def ttmctc_elementwise(x: SparseTensor, u, mode: int, precomputed_core: Optional[CoreTensor] = None,
                       ws=None) -> np.ndarray:
    fs = _factors_of(u)
    _check_factors(x, fs)
    if mode < 0 or mode >= x.order():
        raise RangeError("ttmctc: mode out of range")
    ranks = np.array([f.shape[1] for f in fs], np.uint64)
    core_ptr = None
    if precomputed_core is not None:
        if list(precomputed_core.ranks) != [int(r) for r in ranks]:
            raise ShapeError("precomputed core ranks do not match the factors")
        cd = np.ascontiguousarray(precomputed_core.data, dtype=np.float64)
        core_ptr = cd.ctypes.data
    a = np.empty((x.dims()[mode], int(ranks[mode])), np.float64)
    _check(load_library().hq_ttmctc(x.handle, _ptr_array(fs), ranks, mode, core_ptr, 0, a.reshape(-1)))
    return a


def ttmctc_matrix(x: SparseTensor, u, mode: int, ws=None) -> np.ndarray:
    fs = _factors_of(u)
    _check_factors(x, fs)
    if mode < 0 or mode >= x.order():
        raise RangeError("ttmctc: mode out of range")
    ranks = np.array([f.shape[1] for f in fs], np.uint64)
    a = np.empty((x.dims()[mode], int(ranks[mode])), np.float64)
    _check(load_library().hq_ttmctc(x.handle, _ptr_array(fs), ranks, mode, None, 1, a.reshape(-1)))
    return a


def qr_orthonormal(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2:
        raise ShapeError("qr_orthonormal: matrix expected")
    q = np.empty_like(a)
    if a.shape[1] == 0:
        if a.shape[0] < a.shape[1]:
            raise ShapeError("qr_orthonormal: need rows >= cols")
        return q
    _check(load_library().hq_qr_orthonormal(a.shape[0], a.shape[1], a.reshape(-1), q.reshape(-1)))
    return q


def subspace_distance(u, v) -> float:
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
    v = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
    if u.shape != v.shape:
        raise ShapeError("subspace_distance: shapes differ")
    out = C.c_double(0)
    _check(load_library().hq_subspace_distance(u.shape[0], u.shape[1], u.reshape(-1), v.reshape(-1), C.byref(out)))
    return out.value


def random_factors(dims, ranks, seed) -> FactorSet:
    if len(dims) != len(ranks):
        raise ShapeError("random_factors: dims/ranks length mismatch")
    d = np.ascontiguousarray(np.asarray(dims, np.uint64))
    r = np.ascontiguousarray(np.asarray(ranks, np.uint64))
    fs = [np.empty((int(a), int(b)), np.float64) for a, b in zip(d, r)]
    _check(load_library().hq_random_factors(d.size, d, r, int(seed) & (2**64 - 1), _ptr_array(fs)))
    return FactorSet(fs)


# ---------------------------------------------------------------- solver --
INIT_RANDOM, INIT_HOSVD, INIT_GIVEN = 0, 1, 2
KERNEL_ELEMENTWISE, KERNEL_MATRIX = 0, 1


@dataclasses.dataclass
class SolverConfig:
    """solvers.hpp:17-28"""
    ranks: List[int]
    max_sweeps: int = 100
    tol_fit_change: float = 1e-12
    seed: int = 0
    init: int = INIT_RANDOM
    trace_gradients: bool = False
    kernel: int = KERNEL_ELEMENTWISE
    tol_grad: float = 0.0
    capacity_cap: int = 1 << 31  # kernels.hpp:62 (dense unfoldings of the desk-scale paths)

    def to_c(self, order):
        c = HqConfig()
        load_library().hq_config_default(C.byref(c))
        c.order = order
        for i, k in enumerate(self.ranks):
            c.ranks[i] = int(k)
        c.max_sweeps = int(self.max_sweeps)
        c.tol_fit_change = float(self.tol_fit_change)
        c.seed = int(self.seed) & (2**64 - 1)
        c.init = int(self.init)
        c.kernel = int(self.kernel)
        c.trace_gradients = int(bool(self.trace_gradients))
        c.tol_grad = float(self.tol_grad)
        c.capacity_cap = int(self.capacity_cap)
        return c


@dataclasses.dataclass
class TuckerModel:
    factors: FactorSet
    core: CoreTensor
    data_norm_sq: float = 0.0


@dataclasses.dataclass
class SweepRecord:
    sweep: int
    elapsed_s: float
    objective: float
    fit: float
    total_grad_norm_sq: float
    grad_norm_sq: List[float]
    drift: List[float]


@dataclasses.dataclass
class ModeUpdateRecord:
    """solvers.hpp:40-49 (filled only when gradients are traced)"""
    sweep: int
    mode: int
    f_before: float
    f_after: float
    grad_norm_sq: float
    sigma: List[float]
    lambda_: List[float]
    elapsed_s: float


@dataclasses.dataclass
class IterationTrace:
    data_norm_sq: float
    initial_objective: float
    sweeps: List[SweepRecord]
    updates: list


@dataclasses.dataclass
class SolveResult:
    model: TuckerModel
    trace: IterationTrace


def _check_ranks(x: SparseTensor, ranks):
    # solvers.cpp:22-30
    if len(ranks) != x.order():
        raise ShapeError("rank count does not match tensor order")
    for n, k in enumerate(ranks):
        if k < 1 or k > x.dims()[n]:
            raise ShapeError(f"rank for mode {n + 1} must lie in [1, {x.dims()[n]}]")


class _TraceBuffers:
    def __init__(self, sweeps, order, ranks=None):
        self.ranks = [int(k) for k in ranks] if ranks is not None else [1] * order
        nu = max(1, sweeps * order)
        self.ks = max(self.ranks)
        self.obj = np.zeros(max(1, sweeps))
        self.fit = np.zeros(max(1, sweeps))
        self.drift = np.zeros(nu)
        self.grad = np.zeros(nu)
        self.el = np.zeros(max(1, sweeps))
        self.fb = np.zeros(nu)
        self.fa = np.zeros(nu)
        self.uel = np.zeros(nu)
        self.sig = np.zeros(nu * self.ks)
        self.lam = np.zeros(nu * self.ks)
        self.c = HqTrace(0.0, 0.0, 0, self.obj.ctypes.data, self.fit.ctypes.data, self.drift.ctypes.data,
                         self.grad.ctypes.data, self.el.ctypes.data, self.fb.ctypes.data, self.fa.ctypes.data,
                         self.uel.ctypes.data, self.sig.ctypes.data, self.lam.ctypes.data, self.ks, 0)

    def to_trace(self, order):
        s = int(self.c.sweeps)
        recs = []
        for i in range(s):
            g = [float(v) for v in self.grad[i * order:(i + 1) * order]]
            recs.append(SweepRecord(i + 1, float(self.el[i]), float(self.obj[i]), float(self.fit[i]), float(sum(g)), g,
                                    [float(v) for v in self.drift[i * order:(i + 1) * order]]))
        ups = []
        for i in range(int(self.c.updates)):
            n = i % order
            k = self.ranks[n]
            ups.append(ModeUpdateRecord(i // order + 1, n, float(self.fb[i]), float(self.fa[i]), float(self.grad[i]),
                                        [float(v) for v in self.sig[i * self.ks:i * self.ks + k]],
                                        [float(v) for v in self.lam[i * self.ks:i * self.ks + k]], float(self.uel[i])))
        return IterationTrace(float(self.c.data_norm_sq), float(self.c.initial_objective), recs, ups)


def hoqri(x: SparseTensor, config: SolverConfig, init_factors: Optional[Sequence[np.ndarray]] = None) -> SolveResult:
    """tucker::hoqri (solvers.hpp:80; solvers.cpp:50-178, 217-219), on the device."""
    _check_ranks(x, config.ranks)
    if config.max_sweeps < 1:
        raise ShapeError("max_sweeps must be at least 1")
    if config.tol_fit_change < 0:
        raise ShapeError("tolerance must be nonnegative")
    L = load_library()
    n = x.order()
    cfg = config.to_c(n)
    init_arr = None
    if init_factors is not None:
        fs0 = _factors_of(init_factors)
        _check_factors(x, fs0)
        cfg.init = INIT_GIVEN
        init_arr = _ptr_array(fs0)
    fs = [np.empty((x.dims()[v], int(config.ranks[v])), np.float64) for v in range(n)]
    core = np.empty(int(np.prod(config.ranks)), np.float64)
    tb = _TraceBuffers(int(config.max_sweeps), n, config.ranks)
    _check(L.hq_hoqri(x.handle, C.byref(cfg), init_arr, _ptr_array(fs), core.ctypes.data, C.byref(tb.c)))
    trace = tb.to_trace(n)
    model = TuckerModel(FactorSet(fs), CoreTensor([int(k) for k in config.ranks], core), trace.data_norm_sq)
    return SolveResult(model, trace)


def hooi(x: SparseTensor, config: SolverConfig, init_factors: Optional[Sequence[np.ndarray]] = None) -> SolveResult:
    """tucker::hooi (solvers.hpp:82-83; solvers.cpp:93-178): desk-scale, every step on the device
    (dense Y_(n), cuSOLVER eigen-solve of the smaller Gram side)."""
    _check_ranks(x, config.ranks)
    if config.max_sweeps < 1:
        raise ShapeError("max_sweeps must be at least 1")
    if config.tol_fit_change < 0:
        raise ShapeError("tolerance must be nonnegative")
    n = x.order()
    cfg = config.to_c(n)
    init_arr = None
    if init_factors is not None:
        fs0 = _factors_of(init_factors)
        _check_factors(x, fs0)
        cfg.init = INIT_GIVEN
        init_arr = _ptr_array(fs0)
    fs = [np.empty((x.dims()[v], int(config.ranks[v])), np.float64) for v in range(n)]
    core = np.empty(int(np.prod(config.ranks)), np.float64)
    tb = _TraceBuffers(int(config.max_sweeps), n, config.ranks)
    _check(load_library().hq_hooi(x.handle, C.byref(cfg), init_arr, _ptr_array(fs), core.ctypes.data, C.byref(tb.c)))
    trace = tb.to_trace(n)
    model = TuckerModel(FactorSet(fs), CoreTensor([int(k) for k in config.ranks], core), trace.data_norm_sq)
    return SolveResult(model, trace)


def init_factors(x: SparseTensor, config: SolverConfig) -> FactorSet:
    """solvers.hpp:69-70 / solvers.cpp:197-215: seeded random, or HOSVD (desk-scale) on the device."""
    _check_ranks(x, config.ranks)
    n = x.order()
    fs = [np.empty((x.dims()[v], int(config.ranks[v])), np.float64) for v in range(n)]
    cfg = config.to_c(n)
    _check(load_library().hq_init_factors(x.handle, C.byref(cfg), _ptr_array(fs)))
    return FactorSet(fs)


def svd_leading(y, k: int) -> np.ndarray:
    """dense_core.hpp:64: leading k left singular vectors (device eigen-solve; a subspace match of the
    reference, column signs may differ)."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    if y.ndim != 2:
        raise ShapeError("svd_leading: matrix expected")
    m, p = y.shape
    if k > min(m, p):
        raise ShapeError("svd_leading: k exceeds min(rows, cols)")
    u = np.zeros((m, int(k)), np.float64)
    if k:
        _check(load_library().hq_svd_leading(m, p, y.reshape(-1), int(k), u.reshape(-1)))
    return u


def jacobi_eig_sym(m):
    """dense_core.hpp:85-90: eigenpairs of the symmetrised matrix, values descending, vectors in columns
    (device eigen-solve; vector signs may differ from the reference's Jacobi rotations)."""
    m = np.ascontiguousarray(m, dtype=np.float64)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ShapeError("jacobi_eig_sym: square matrix required")
    n = m.shape[0]
    vals, vecs = np.zeros(n, np.float64), np.zeros((n, n), np.float64)
    if n:
        _check(load_library().hq_sym_eig(n, m.reshape(-1), vals, vecs.ctypes.data))
    return vals, vecs


def densify_unfold(x: SparseTensor, mode: int, capacity_cap: int = 1 << 31) -> np.ndarray:
    """kernels.hpp:70-71 on the device"""
    if not 0 <= mode < x.order():
        raise RangeError("densify_unfold: mode out of range")
    cols = 1
    for v, d in enumerate(x.dims()):
        if v != mode:
            cols *= d
    rows = x.dims()[mode]
    if cols and rows > capacity_cap // cols:
        raise CapacityError(f"dense unfolding of {rows} x {cols} exceeds the capacity cap; this path is desk-scale only")
    out = np.empty(rows * cols, np.float64)
    _check(load_library().hq_densify_unfold(x.handle, int(mode), int(capacity_cap), out))
    return out.reshape(rows, cols)


def ttmc_unfold_dense(x: SparseTensor, u, mode: int, capacity_cap: int = 1 << 31) -> np.ndarray:
    """kernels.hpp:66-67 on the device"""
    fs = _factors_of(u)
    _check_factors(x, fs)
    if not 0 <= mode < x.order():
        raise RangeError("ttmc_unfold_dense: mode out of range")
    ranks = np.array([f.shape[1] for f in fs], np.uint64)
    cols = int(np.prod([int(r) for v, r in enumerate(ranks) if v != mode]))
    rows = x.dims()[mode]
    if cols and rows > capacity_cap // cols:
        raise CapacityError(f"dense unfolding of {rows} x {cols} exceeds the capacity cap; this path is desk-scale only")
    out = np.empty(rows * cols, np.float64)
    _check(load_library().hq_ttmc_unfold_dense(x.handle, _ptr_array(fs), ranks, int(mode), int(capacity_cap), out))
    return out.reshape(rows, cols)


def fit_error(x: SparseTensor, model: TuckerModel) -> float:
    """solvers.cpp:225-236"""
    if model.factors.order() != x.order():
        raise ShapeError("fit_error: model order does not match the tensor")
    out = C.c_double(0)
    d = np.ascontiguousarray(model.core.data, dtype=np.float64)
    _check(load_library().hq_fit_error(float(model.data_norm_sq), d.size, d, C.byref(out)))
    return out.value


# ---------------------------------------------------- device-resident API --
def partition_rows(offsets, world: int) -> np.ndarray:
    """Row partition of one mode (rank r owns rows [b[r], b[r+1])): contiguous
    whole rows with ~nnz/world nonzeros each.  Host code, no GPU needed."""
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64))
    b = np.zeros(world + 1, np.uint64)
    _check(load_library().hq_partition_rows(off, off.size - 1, world, b))
    return b


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(load_library().hq_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


class Comm:
    """Communicator of one rank: NCCL (one process per GPU, current device), or
    with ``Comm.host(...)`` the host transport (ranks exchange through a POSIX
    shared-memory segment; several ranks may share one GPU)."""

    def __init__(self, world: int, rank: int, uid: bytes = b"\0" * 128, _handle=None):
        if _handle is None:
            buf = (C.c_uint8 * 128).from_buffer_copy(uid)
            h = C.c_void_p()
            _check(load_library().hq_comm_create(world, rank, C.cast(buf, C.c_void_p), C.byref(h)))
            _handle = h
        self._h = _handle
        self.world, self.rank = world, rank

    @classmethod
    def host(cls, world: int, rank: int, name: str, capacity: int) -> "Comm":
        """Host transport over the shared-memory segment `name` (starts with '/'; every rank passes the same
        name); `capacity` = the largest collective in doubles (>= max I_n K_n)."""
        h = C.c_void_p()
        _check(load_library().hq_comm_create_host(world, rank, name.encode(), int(capacity), C.byref(h)))
        return cls(world, rank, _handle=h)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                load_library().hq_comm_destroy(self._h)
                self._h = None
        except Exception:
            pass


class Solver:
    """Device-resident solve for benchmarks: every operand stays in HBM; sweeps
    and single kernels are launched on `stream` (a cudaStream_t as int).  With
    `comm`, the rows of every mode are partitioned over the ranks."""

    def __init__(self, x: SparseTensor, config: SolverConfig, init_factors=None, stream: int = 0, comm: "Comm" = None):
        L = load_library()
        self.x = x
        self.n = x.order()
        self.config = config
        cfg = config.to_c(self.n)
        arr = None
        if init_factors is not None:
            fs0 = _factors_of(init_factors)
            cfg.init = INIT_GIVEN
            arr = _ptr_array(fs0)
            self._keep = fs0
        h = C.c_void_p()
        if comm is not None:
            self._comm = comm
            _check(L.hq_solver_create_dist(x.handle, C.byref(cfg), arr, stream or None, comm._h, C.byref(h)))
        else:
            _check(L.hq_solver_create(x.handle, C.byref(cfg), arr, stream or None, C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                load_library().hq_solver_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def run(self, sweeps):
        _check(load_library().hq_solver_run(self._h, int(sweeps)))

    def sync(self):
        _check(load_library().hq_solver_sync(self._h))

    def status(self):
        """Device status word: sweeps done, Householder fallbacks, abort code, degenerate mode, shifted
        CholeskyQR3 updates, (multi-GPU) updates finished by the host-driven Householder continuation, and
        whether the multi-GPU apply writes U_new into the other ranks' replicas over peer memory."""
        out = (C.c_int64 * 8)()
        _check(load_library().hq_solver_status(self._h, out))
        return {"sweeps": out[0], "fallbacks": out[1], "abort": out[2], "degenerate_mode": out[3],
                "shifted": out[4], "dist_householder": out[5], "peer_apply": out[6]}

    def launch_mode_pass(self, mode):
        """The fused sparse pass of a mode update (A, M, W, max|A|), on the solver's stream."""
        _check(load_library().hq_solver_launch_mode_pass(self._h, mode))

    def launch_ttmctc(self, mode):
        """The standalone TTMcTC of `mode` with the current core (kernels.cpp:86-163): A only."""
        _check(load_library().hq_solver_launch_ttmctc(self._h, mode))

    def launches_per_sweep(self):
        out = C.c_uint64(0)
        _check(load_library().hq_solver_launches_per_sweep(self._h, C.byref(out)))
        return int(out.value)

    def mode_pass_work(self, mode):
        f, b = C.c_double(0), C.c_double(0)
        _check(load_library().hq_solver_mode_pass_work(self._h, mode, C.byref(f), C.byref(b)))
        return f.value, b.value

    def ttmctc_work(self, mode):
        f, b = C.c_double(0), C.c_double(0)
        _check(load_library().hq_solver_ttmctc_work(self._h, mode, C.byref(f), C.byref(b)))
        return f.value, b.value

    def download(self, out=None):
        """Factors, core and trace to the host.  `out` = (factor arrays, core array) lets the caller supply
        (e.g. page-locked) C-contiguous float64 destinations of the right shapes."""
        if out is None:
            fs = [np.empty((self.x.dims()[v], int(self.config.ranks[v])), np.float64) for v in range(self.n)]
            core = np.empty(int(np.prod(self.config.ranks)), np.float64)
        else:
            fs, core = list(out[0]), out[1]
            for v, f in enumerate(fs):
                if (f.dtype != np.float64 or not f.flags.c_contiguous
                        or f.shape != (self.x.dims()[v], int(self.config.ranks[v]))):
                    raise ShapeError(f"download: factor {v} destination has the wrong shape/dtype/layout")
            if core.dtype != np.float64 or not core.flags.c_contiguous or core.size != int(np.prod(self.config.ranks)):
                raise ShapeError("download: core destination has the wrong size/dtype/layout")
            core = core.reshape(-1)
        tb = _TraceBuffers(int(self.config.max_sweeps), self.n, self.config.ranks)
        _check(load_library().hq_solver_download(self._h, _ptr_array(fs), core.ctypes.data, C.byref(tb.c)))
        trace = tb.to_trace(self.n)
        return SolveResult(TuckerModel(FactorSet(fs), CoreTensor(list(self.config.ranks), core), trace.data_norm_sq),
                           trace)


# ------------------------------------------------------------- .tns I/O --
def gen_synthetic_coo(dims, nnz: int, seed: int):
    """harness.cpp:62-98 (gen_synthetic) as raw COO: nnz distinct uniform
    coordinates, standard-normal values, the reference's Rng stream."""
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.uint64))
    if d.size == 0:
        raise ShapeError("gen_synthetic: need at least one mode")
    coords = np.empty((int(nnz), d.size), np.uint32)
    vals = np.empty(int(nnz), np.float64)
    _check(load_library().hq_gen_synthetic(d.size, d, int(nnz), int(seed) & (2**64 - 1), coords.ctypes.data, vals))
    return coords, vals


def gen_synthetic(dims, nnz: int, seed: int) -> SparseTensor:
    """tucker::gen_synthetic (harness.hpp:27-31)"""
    coords, vals = gen_synthetic_coo(dims, nnz, seed)
    return SparseTensor([int(v) for v in dims], coords, vals)


def load_tns(source, dims_override: Optional[Sequence[int]] = None) -> SparseTensor:
    """sparse_tensor.cpp:136-215: native threaded text parse, build on the device."""
    from .tns import load_tns_tensor
    return load_tns_tensor(source, dims_override)


def write_tns(out, x: SparseTensor):
    """sparse_tensor.cpp:224-235"""
    c, v = x._export()
    lines = ["dims: " + " ".join(str(d) for d in x.dims())]
    for e in range(x.nnz()):
        lines.append(" ".join(str(int(i) + 1) for i in c[e]) + " " + ("%.17g" % v[e]))
    text = "\n".join(lines) + "\n"
    if hasattr(out, "write"):
        out.write(text)
    else:
        with open(out, "w") as f:
            f.write(text)
