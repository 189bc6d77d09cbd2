"""ctypes bindings for the test-side checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  -> oracle/liboracle.so, the C restatement (oracle/hq_oracle.c)
* ``RefLib``  -> oracle/_ref/libtucker_ref.so, the unmodified reference library
  compiled from /root/reference/proj/src (present only where it was built).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtucker_ref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def _u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _u32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def build_oracle():
    if not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "liboracle.so")])


class Oracle:
    """The C restatement of the reference hot path."""

    def __init__(self):
        build_oracle()
        L = C.CDLL(ORACLE_SO)
        self.L = L
        L.hqo_raw_stream.argtypes = [C.c_uint64, C.c_uint64, u64p]
        L.hqo_normal_stream.argtypes = [C.c_uint64, C.c_uint64, f64p]
        L.hqo_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.hqo_mix_seed.restype = C.c_uint64
        L.hqo_normalize.argtypes = [C.c_int, u64p, C.c_uint64, u32p, f64p, u32p, f64p, C.POINTER(C.c_uint64)]
        L.hqo_buckets.argtypes = [C.c_int, u64p, C.c_uint64, u32p, C.c_int, u64p, u64p]
        L.hqo_norm_sq.argtypes = [C.c_uint64, f64p]
        L.hqo_norm_sq.restype = C.c_double
        L.hqo_ttmc_core.argtypes = [C.c_int, u64p, u64p, C.c_uint64, u32p, f64p, f64p, f64p]
        L.hqo_ttmctc.argtypes = [C.c_int, u64p, u64p, C.c_uint64, u32p, f64p, f64p, C.c_int, f64p, f64p]
        L.hqo_qr.argtypes = [C.c_uint64, C.c_uint64, f64p, f64p]
        L.hqo_subspace_distance.argtypes = [C.c_uint64, C.c_uint64, f64p, f64p]
        L.hqo_subspace_distance.restype = C.c_double
        L.hqo_random_factors.argtypes = [C.c_int, u64p, u64p, C.c_uint64, f64p]
        L.hqo_orthonormality_defect.argtypes = [C.c_int, u64p, u64p, f64p]
        L.hqo_orthonormality_defect.restype = C.c_double
        L.hqo_hoqri.argtypes = [C.c_int, u64p, u64p, C.c_uint64, u32p, f64p, f64p, C.c_uint64, C.c_double,
                                f64p, C.POINTER(C.c_uint64), C.POINTER(C.c_double), f64p, f64p, f64p,
                                C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]
        L.hqo_fit_error.argtypes = [C.c_double, C.c_uint64, f64p, C.POINTER(C.c_double)]
        L.hqo_hoqri_traced.argtypes = [C.c_int, u64p, u64p, C.c_uint64, u32p, f64p, f64p, C.c_uint64, C.c_double,
                                       C.c_double, C.c_uint64, f64p, C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                       f64p, f64p, f64p, f64p, f64p, f64p, f64p, f64p, C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_int), C.POINTER(C.c_int)]

    # rng
    def raw_stream(self, seed, n):
        out = np.empty(n, np.uint64)
        self.L.hqo_raw_stream(seed, n, out)
        return out

    def normal_stream(self, seed, n):
        out = np.empty(n, np.float64)
        self.L.hqo_normal_stream(seed, n, out)
        return out

    def mix_seed(self, seed, salt):
        return int(self.L.hqo_mix_seed(seed, salt))

    # tensor
    def normalize(self, dims, coords, vals):
        dims = _u64(dims)
        coords = _u32(coords).reshape(-1)
        vals = _f64(vals)
        nnz = vals.size
        oc = np.empty(max(nnz * dims.size, 1), np.uint32)
        ov = np.empty(max(nnz, 1), np.float64)
        out_nnz = C.c_uint64(0)
        st = self.L.hqo_normalize(dims.size, dims, nnz, coords, vals, oc, ov, C.byref(out_nnz))
        if st:
            raise RuntimeError(f"normalize status {st}")
        u = out_nnz.value
        return oc[: u * dims.size].reshape(u, dims.size).copy(), ov[:u].copy()

    def buckets(self, dims, coords, mode):
        dims = _u64(dims)
        coords = _u32(coords).reshape(-1)
        nnz = coords.size // dims.size
        off = np.empty(int(dims[mode]) + 1, np.uint64)
        ent = np.empty(max(nnz, 1), np.uint64)
        self.L.hqo_buckets(dims.size, dims, nnz, coords, mode, off, ent)
        return off, ent[:nnz]

    def norm_sq(self, vals):
        vals = _f64(vals)
        return self.L.hqo_norm_sq(vals.size, vals)

    def ttmc_core(self, dims, ranks, coords, vals, factors):
        dims, ranks = _u64(dims), _u64(ranks)
        coords, vals = _u32(coords).reshape(-1), _f64(vals)
        f = _f64(np.concatenate([np.asarray(u, np.float64).reshape(-1) for u in factors]))
        core = np.empty(int(np.prod(ranks)), np.float64)
        self.L.hqo_ttmc_core(dims.size, dims, ranks, vals.size, coords, vals, f, core)
        return core.reshape(tuple(int(r) for r in ranks))

    def ttmctc(self, dims, ranks, coords, vals, factors, mode, core):
        dims, ranks = _u64(dims), _u64(ranks)
        coords, vals = _u32(coords).reshape(-1), _f64(vals)
        f = _f64(np.concatenate([np.asarray(u, np.float64).reshape(-1) for u in factors]))
        a = np.empty(int(dims[mode] * ranks[mode]), np.float64)
        self.L.hqo_ttmctc(dims.size, dims, ranks, vals.size, coords, vals, f, mode, _f64(core).reshape(-1), a)
        return a.reshape(int(dims[mode]), int(ranks[mode]))

    def qr(self, a):
        a = _f64(a)
        q = np.empty_like(a)
        st = self.L.hqo_qr(a.shape[0], a.shape[1], a.reshape(-1), q.reshape(-1))
        if st:
            raise ValueError("qr: rows < cols")
        return q

    def subspace_distance(self, u, v):
        u, v = _f64(u), _f64(v)
        return self.L.hqo_subspace_distance(u.shape[0], u.shape[1], u.reshape(-1), v.reshape(-1))

    def random_factors(self, dims, ranks, seed):
        dims, ranks = _u64(dims), _u64(ranks)
        out = np.empty(int(np.sum(dims * ranks)), np.float64)
        st = self.L.hqo_random_factors(dims.size, dims, ranks, seed, out)
        if st:
            raise ValueError("random_factors: rank exceeds extent")
        return _split(out, dims, ranks)

    def orthonormality_defect(self, dims, ranks, factors):
        dims, ranks = _u64(dims), _u64(ranks)
        f = _f64(np.concatenate([np.asarray(u).reshape(-1) for u in factors]))
        return self.L.hqo_orthonormality_defect(dims.size, dims, ranks, f)

    def hoqri(self, dims, ranks, coords, vals, init_factors, max_sweeps, tol=0.0, snapshots=False):
        """Normalised inputs.  Returns dict with factors, core, trace, snapshots."""
        dims, ranks = _u64(dims), _u64(ranks)
        coords, vals = _u32(coords).reshape(-1), _f64(vals)
        N = dims.size
        f = _f64(np.concatenate([np.asarray(u).reshape(-1) for u in init_factors]))
        pk = int(np.prod(ranks))
        core = np.empty(pk, np.float64)
        sd = C.c_uint64(0)
        f0 = C.c_double(0)
        obj = np.zeros(max_sweeps, np.float64)
        fit = np.zeros(max_sweeps, np.float64)
        drift = np.zeros(max_sweeps * N, np.float64)
        deg = C.c_int(0)
        csnap = fsnap = None
        if snapshots:
            csnap = np.zeros(max_sweeps * pk, np.float64)
            fsnap = np.zeros(max_sweeps * f.size, np.float64)
        st = self.L.hqo_hoqri(N, dims, ranks, vals.size, coords, vals, f, max_sweeps, tol, core,
                              C.byref(sd), C.byref(f0), obj, fit, drift,
                              csnap.ctypes.data if snapshots else None,
                              fsnap.ctypes.data if snapshots else None, C.byref(deg))
        s = sd.value
        out = dict(status=st, degenerate_mode=deg.value, sweeps=s, initial_objective=f0.value,
                   objective=obj[:s], fit=fit[:s], drift=drift[: s * N].reshape(s, N),
                   factors=_split(f, dims, ranks), core=core.reshape(tuple(int(r) for r in ranks)))
        if snapshots:
            out["core_snap"] = csnap[: s * pk].reshape((s,) + tuple(int(r) for r in ranks))
            out["factor_snap"] = [_split(fsnap[i * f.size:(i + 1) * f.size], dims, ranks) for i in range(s)]
        return out


def _oracle_hoqri_traced(self, dims, ranks, coords, vals, init_factors, max_sweeps, tol=0.0, tol_grad=0.0):
    """hqo_hoqri_traced: the oracle solve with per-update gradient diagnostics."""
    dims, ranks = _u64(dims), _u64(ranks)
    coords, vals = _u32(coords).reshape(-1), _f64(vals)
    N = dims.size
    ks = int(ranks.max())
    f = _f64(np.concatenate([np.asarray(u).reshape(-1) for u in init_factors]))
    core = np.empty(int(np.prod(ranks)), np.float64)
    sd, nu = C.c_uint64(0), C.c_uint64(0)
    f0 = C.c_double(0)
    obj, fit = np.zeros(max_sweeps), np.zeros(max_sweeps)
    drift, grad = np.zeros(max_sweeps * N), np.zeros(max_sweeps * N)
    fb, fa = np.zeros(max_sweeps * N), np.zeros(max_sweeps * N)
    sig, lam = np.zeros(max_sweeps * N * ks), np.zeros(max_sweeps * N * ks)
    deg, bad = C.c_int(0), C.c_int(0)
    st = self.L.hqo_hoqri_traced(N, dims, ranks, vals.size, coords, vals, f, max_sweeps, tol, tol_grad, ks, core,
                                 C.byref(sd), C.byref(f0), obj, fit, drift, grad, fb, fa, sig, lam, C.byref(nu),
                                 C.byref(deg), C.byref(bad))
    s, u = int(sd.value), int(nu.value)
    return dict(status=st, bad_k=bad.value, sweeps=s, objective=obj[:s], fit=fit[:s], grad=grad[:u], updates=u,
                f_before=fb[:u], f_after=fa[:u], sigma=sig[:u * ks].reshape(u, ks),
                lambda_=lam[:u * ks].reshape(u, ks), core=core)


Oracle.hoqri_traced = _oracle_hoqri_traced


def _split(flat, dims, ranks):
    out, o = [], 0
    for d, r in zip(dims, ranks):
        d, r = int(d), int(r)
        out.append(np.array(flat[o:o + d * r]).reshape(d, r))
        o += d * r
    return out


class RefLib:
    """The unmodified reference library (oracle/_ref), via oracle/ref_capi.cpp."""

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self):
        L = C.CDLL(REF_SO)
        self.L = L
        vp = C.c_void_p
        L.ref_tensor_create.argtypes = [C.c_int, u64p, C.c_uint64, u32p, f64p, C.POINTER(vp)]
        L.ref_gen_synthetic.argtypes = [C.c_int, u64p, C.c_uint64, C.c_uint64, C.POINTER(vp)]
        L.ref_tensor_destroy.argtypes = [vp]
        L.ref_tensor_nnz.argtypes = [vp]
        L.ref_tensor_nnz.restype = C.c_uint64
        L.ref_tensor_export.argtypes = [vp, u32p, f64p]
        L.ref_tensor_buckets.argtypes = [vp, C.c_int, u64p, u64p]
        L.ref_norm_sq.argtypes = [vp]
        L.ref_norm_sq.restype = C.c_double
        L.ref_ttmc_core.argtypes = [vp, u64p, f64p, f64p]
        L.ref_ttmctc.argtypes = [vp, u64p, f64p, C.c_int, C.c_void_p, C.c_int, f64p]
        L.ref_qr.argtypes = [C.c_uint64, C.c_uint64, f64p, f64p]
        L.ref_subspace_distance.argtypes = [C.c_uint64, C.c_uint64, f64p, f64p]
        L.ref_subspace_distance.restype = C.c_double
        L.ref_random_factors.argtypes = [C.c_int, u64p, u64p, C.c_uint64, f64p]
        L.ref_raw_stream.argtypes = [C.c_uint64, C.c_uint64, u64p]
        L.ref_normal_stream.argtypes = [C.c_uint64, C.c_uint64, f64p]
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_hoqri.argtypes = [vp, u64p, C.c_uint64, C.c_double, C.c_uint64, C.c_int, f64p, f64p,
                                C.POINTER(C.c_uint64), C.POINTER(C.c_double), f64p, f64p, f64p, f64p]
        L.ref_hoqri_replay.argtypes = [vp, u64p, f64p, C.c_uint64, f64p, f64p, f64p]
        L.ref_hoqri_replay_matrix.argtypes = [vp, u64p, f64p, C.c_uint64, f64p, f64p, f64p]
        L.ref_tensor_dims.argtypes = [vp, u64p]
        L.ref_densify_unfold.argtypes = [vp, C.c_int, C.c_uint64, f64p]
        L.ref_ttmc_unfold_dense.argtypes = [vp, u64p, f64p, C.c_int, C.c_uint64, f64p]
        L.ref_svd_leading.argtypes = [C.c_uint64, C.c_uint64, f64p, C.c_uint64, f64p]
        L.ref_init_factors.argtypes = [vp, u64p, C.c_uint64, C.c_int, C.c_uint64, f64p]
        L.ref_solve.argtypes = [vp, C.c_int, u64p, C.c_uint64, C.c_double, C.c_uint64, C.c_int, C.c_int, f64p, f64p,
                                C.POINTER(C.c_uint64), C.POINTER(C.c_double), f64p, f64p, f64p, f64p]
        L.ref_tns_parse.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_void_p, C.POINTER(vp)]
        L.ref_last_message.restype = C.c_char_p
        L.ref_trace_files.argtypes = [vp, u64p, C.c_uint64, C.c_uint64, C.c_char_p, C.c_char_p, C.c_uint64]
        L.ref_hoqri_traced.argtypes = [vp, u64p, C.c_uint64, C.c_double, C.c_uint64, C.c_double, C.c_uint64, f64p,
                                       f64p, C.POINTER(C.c_uint64), f64p, f64p, f64p, C.POINTER(C.c_uint64), f64p,
                                       f64p, f64p, f64p]
        L.ref_last_payload.restype = C.c_int64
        L.ref_slices_create.argtypes = [vp, C.c_int]
        L.ref_slices_create.restype = vp
        L.ref_slices_destroy.argtypes = [vp]
        L.ref_slices_time.argtypes = [vp, u64p, f64p, f64p, C.c_int, C.c_int, C.c_int]
        L.ref_slices_time.restype = C.c_double
        L.ref_time_qr.argtypes = [C.c_uint64, C.c_uint64, f64p, C.c_int]
        L.ref_time_qr.restype = C.c_double
        L.ref_state_create.argtypes = [vp, u64p, f64p]
        L.ref_state_create.restype = vp
        L.ref_state_destroy.argtypes = [vp]
        L.ref_state_mode_update.argtypes = [vp, vp, C.c_int, C.POINTER(C.c_double), f64p]


def ref_svd_leading(lib, y, k):
    y = _f64(y)
    out = np.empty(y.shape[0] * k, np.float64)
    st = lib.L.ref_svd_leading(y.shape[0], y.shape[1], y.reshape(-1), k, out)
    if st:
        raise RuntimeError(f"ref svd_leading status {st}")
    return out.reshape(y.shape[0], k)


def ref_load_tns(lib, text: bytes, dims_override=None):
    """tucker::load_tns on a text buffer -> (status, message, payload, RefTensor or None)."""
    h = C.c_void_p()
    ov = None if dims_override is None else _u64(dims_override)
    st = lib.L.ref_tns_parse(text, len(text), 0 if ov is None else ov.size, None if ov is None else ov.ctypes.data,
                             C.byref(h))
    if st:
        return st, lib.L.ref_last_message().decode(), int(lib.L.ref_last_payload()), None
    d = np.zeros(16, np.uint64)
    n = lib.L.ref_tensor_dims(h, d)
    return 0, "", 0, RefTensor(lib, h, [int(v) for v in d[:n]])


class RefTensor:
    def __init__(self, lib: RefLib, handle, dims):
        self.lib, self.h, self.dims = lib, handle, [int(d) for d in dims]

    @classmethod
    def create(cls, lib, dims, coords, vals):
        dims = _u64(dims)
        h = C.c_void_p()
        st = lib.L.ref_tensor_create(dims.size, dims, _f64(vals).size, _u32(coords).reshape(-1), _f64(vals), C.byref(h))
        if st:
            raise RuntimeError(f"ref tensor create status {st}")
        return cls(lib, h, dims)

    @classmethod
    def gen_synthetic(cls, lib, dims, nnz, seed):
        dims = _u64(dims)
        h = C.c_void_p()
        st = lib.L.ref_gen_synthetic(dims.size, dims, nnz, seed, C.byref(h))
        if st:
            raise RuntimeError(f"gen_synthetic status {st}")
        return cls(lib, h, dims)

    def __del__(self):
        try:
            self.lib.L.ref_tensor_destroy(self.h)
        except Exception:
            pass

    @property
    def nnz(self):
        return int(self.lib.L.ref_tensor_nnz(self.h))

    def export(self):
        n = self.nnz
        c = np.empty(max(n * len(self.dims), 1), np.uint32)
        v = np.empty(max(n, 1), np.float64)
        self.lib.L.ref_tensor_export(self.h, c, v)
        return c[: n * len(self.dims)].reshape(n, len(self.dims)), v[:n]

    def buckets(self, mode):
        off = np.empty(self.dims[mode] + 1, np.uint64)
        ent = np.empty(max(self.nnz, 1), np.uint64)
        self.lib.L.ref_tensor_buckets(self.h, mode, off, ent)
        return off, ent[: self.nnz]

    def norm_sq(self):
        return self.lib.L.ref_norm_sq(self.h)

    def ttmc_core(self, ranks, factors):
        ranks = _u64(ranks)
        f = _f64(np.concatenate([np.asarray(u).reshape(-1) for u in factors]))
        core = np.empty(int(np.prod(ranks)), np.float64)
        st = self.lib.L.ref_ttmc_core(self.h, ranks, f, core)
        if st:
            raise RuntimeError(f"ttmc_core status {st}")
        return core.reshape(tuple(int(r) for r in ranks))

    def ttmctc(self, ranks, factors, mode, core=None, variant=0):
        ranks = _u64(ranks)
        f = _f64(np.concatenate([np.asarray(u).reshape(-1) for u in factors]))
        a = np.empty(self.dims[mode] * int(ranks[mode]), np.float64)
        cp = None if core is None else _f64(core).reshape(-1)
        st = self.lib.L.ref_ttmctc(self.h, ranks, f, mode, None if cp is None else cp.ctypes.data, variant, a)
        if st:
            raise RuntimeError(f"ttmctc status {st}")
        return a.reshape(self.dims[mode], int(ranks[mode]))

    def hoqri(self, ranks, max_sweeps, tol, seed, kernel=0):
        ranks = _u64(ranks)
        N = len(self.dims)
        f = np.empty(int(sum(d * int(r) for d, r in zip(self.dims, ranks))), np.float64)
        core = np.empty(int(np.prod(ranks)), np.float64)
        sd, f0 = C.c_uint64(0), C.c_double(0)
        obj, fit, el = (np.zeros(max_sweeps) for _ in range(3))
        drift = np.zeros(max_sweeps * N)
        st = self.lib.L.ref_hoqri(self.h, ranks, max_sweeps, tol, seed, kernel, f, core, C.byref(sd), C.byref(f0),
                                  obj, fit, drift, el)
        s = sd.value
        return dict(status=st, payload=int(self.lib.L.ref_last_payload()), sweeps=s, initial_objective=f0.value,
                    objective=obj[:s], fit=fit[:s], drift=drift[: s * N].reshape(s, N), elapsed=el[:s],
                    factors=_split(f, self.dims, ranks), core=core.reshape(tuple(int(r) for r in ranks)))

    def densify(self, mode, cap=1 << 31):
        cols = int(np.prod([d for v, d in enumerate(self.dims) if v != mode]))
        out = np.empty(self.dims[mode] * cols, np.float64)
        st = self.lib.L.ref_densify_unfold(self.h, mode, cap, out)
        return st, (out.reshape(self.dims[mode], cols) if not st else None)

    def unfold_dense(self, ranks, factors, mode, cap=1 << 31):
        ranks = _u64(ranks)
        f = _f64(np.concatenate([np.asarray(u).reshape(-1) for u in factors]))
        cols = int(np.prod([int(r) for v, r in enumerate(ranks) if v != mode]))
        out = np.empty(self.dims[mode] * cols, np.float64)
        st = self.lib.L.ref_ttmc_unfold_dense(self.h, ranks, f, mode, cap, out)
        return st, (out.reshape(self.dims[mode], cols) if not st else None)

    def init_factors(self, ranks, seed, hosvd, cap=1 << 31):
        ranks = _u64(ranks)
        out = np.empty(sum(d * int(k) for d, k in zip(self.dims, ranks)), np.float64)
        st = self.lib.L.ref_init_factors(self.h, ranks, seed, int(hosvd), cap, out)
        msg = self.lib.L.ref_last_message().decode() if st else ""
        return st, msg, (_split(out, self.dims, ranks) if not st else None)

    def solve(self, hooi, ranks, sweeps, tol, seed, hosvd, trace_gradients=False):
        ranks = _u64(ranks)
        n = len(self.dims)
        fs = np.empty(sum(d * int(k) for d, k in zip(self.dims, ranks)), np.float64)
        core = np.empty(int(np.prod(ranks)), np.float64)
        sw, f0 = C.c_uint64(0), C.c_double(0)
        obj, fit = np.zeros(sweeps), np.zeros(sweeps)
        drift, grad = np.zeros(sweeps * n), np.zeros(sweeps * n)
        st = self.lib.L.ref_solve(self.h, int(hooi), ranks, sweeps, tol, seed, int(hosvd), int(trace_gradients), fs,
                                  core, C.byref(sw), C.byref(f0), obj, fit, drift, grad)
        s_ = int(sw.value)
        return dict(status=st, sweeps=s_, initial_objective=f0.value, objective=obj[:s_], fit=fit[:s_],
                    drift=drift[:s_ * n], grad=grad[:s_ * n], core=core,
                    factors=_split(fs, self.dims, ranks) if not st else None)

    def trace_files(self, ranks, sweeps, seed, cap=1 << 20):
        """make_trace_file + write_trace_csv / write_trace_json of a reference hoqri run."""
        c, j = C.create_string_buffer(cap), C.create_string_buffer(cap)
        st = self.lib.L.ref_trace_files(self.h, _u64(ranks), sweeps, seed, c, j, cap)
        if st:
            raise RuntimeError(f"ref_trace_files status {st}")
        return c.value.decode(), j.value.decode()

    def hoqri_traced(self, ranks, sweeps, tol, seed, tol_grad=0.0):
        """tucker::hoqri with trace_gradients (per-update ModeUpdateRecords)."""
        ranks = _u64(ranks)
        n = len(self.dims)
        ks = int(ranks.max())
        fs = np.empty(sum(d * int(k) for d, k in zip(self.dims, ranks)), np.float64)
        core = np.empty(int(np.prod(ranks)), np.float64)
        sw, nu = C.c_uint64(0), C.c_uint64(0)
        obj, fit = np.zeros(sweeps), np.zeros(sweeps)
        grad = np.zeros(sweeps * n)
        fb, fa = np.zeros(sweeps * n), np.zeros(sweeps * n)
        sig, lam = np.zeros(sweeps * n * ks), np.zeros(sweeps * n * ks)
        st = self.lib.L.ref_hoqri_traced(self.h, ranks, sweeps, tol, seed, tol_grad, ks, fs, core, C.byref(sw), obj,
                                         fit, grad, C.byref(nu), fb, fa, sig, lam)
        s, u = int(sw.value), int(nu.value)
        return dict(status=st, sweeps=s, objective=obj[:s], fit=fit[:s], grad=grad[:u], updates=u, f_before=fb[:u],
                    f_after=fa[:u], sigma=sig[:u * ks].reshape(u, ks), lambda_=lam[:u * ks].reshape(u, ks),
                    core=core)

    def replay(self, ranks, init_factors, sweeps, variant="elementwise"):
        ranks = _u64(ranks)
        f = _f64(np.concatenate([np.asarray(u).reshape(-1) for u in init_factors]))
        pk = int(np.prod(ranks))
        cs = np.zeros(sweeps * pk)
        fs = np.zeros(sweeps * f.size)
        dr = np.zeros(sweeps * len(self.dims))
        fn = self.lib.L.ref_hoqri_replay if variant == "elementwise" else self.lib.L.ref_hoqri_replay_matrix
        st = fn(self.h, ranks, f, sweeps, cs, fs, dr)
        if st:
            raise RuntimeError(f"replay status {st}")
        return (cs.reshape((sweeps,) + tuple(int(r) for r in ranks)),
                [_split(fs[i * f.size:(i + 1) * f.size], self.dims, ranks) for i in range(sweeps)],
                dr.reshape(sweeps, len(self.dims)))


class RefSolveState:
    """The factors + fresh core tucker::hoqri carries between mode updates
    (ref_capi.cpp ref_state_*); mode_update(n) runs one full-size mode update of
    the reference's solve loop and returns (drift, seconds per phase)."""

    def __init__(self, t: "RefTensor", ranks, factors):
        self.t = t
        self.ranks = _u64(ranks)
        f = _f64(np.concatenate([np.asarray(u).reshape(-1) for u in factors]))
        self.h = t.lib.L.ref_state_create(t.h, self.ranks, f)

    def mode_update(self, mode):
        d = C.c_double(0)
        tm = np.zeros(4)
        st = self.t.lib.L.ref_state_mode_update(self.t.h, self.h, int(mode), C.byref(d), tm)
        if st:
            raise RuntimeError(f"reference mode update status {st}")
        return d.value, dict(ttmctc=tm[0], qr=tm[1], drift=tm[2], core=tm[3])

    def __del__(self):
        try:
            self.t.lib.L.ref_state_destroy(self.h)
        except Exception:
            pass


def ref_random_factors(lib: RefLib, dims, ranks, seed):
    dims, ranks = _u64(dims), _u64(ranks)
    out = np.empty(int(np.sum(dims * ranks)), np.float64)
    st = lib.L.ref_random_factors(dims.size, dims, ranks, seed, out)
    if st:
        raise RuntimeError(f"random_factors status {st}")
    return _split(out, dims, ranks)


def ref_qr(lib: RefLib, a):
    a = _f64(a)
    q = np.empty_like(a)
    st = lib.L.ref_qr(a.shape[0], a.shape[1], a.reshape(-1), q.reshape(-1))
    if st:
        raise RuntimeError(f"qr status {st}")
    return q
