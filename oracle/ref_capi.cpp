// ref_capi.cpp — extern "C" wrapper around the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources under /root/reference/proj/src into oracle/_ref/ (git
// ignored).  Used to (1) generate the golden vectors in tests/golden/,
// (2) cross-check the C restatement oracle/hq_oracle.c, and (3) time the
// reference CPU path for bench.py's cpu_baseline / --impl reference leg.
// The product never links or loads this.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <sstream>
#include <thread>
#include <vector>

#include "tucker/errors.hpp"
#include "tucker/harness.hpp"
#include "tucker/kernels.hpp"
#include "tucker/manifold.hpp"
#include "tucker/rng.hpp"
#include "tucker/solvers.hpp"
#include "tucker/sparse_tensor.hpp"

using namespace tucker;

namespace {

int code_of(const std::exception& e) {
    if (dynamic_cast<const ShapeError*>(&e)) return 1;
    if (dynamic_cast<const RangeError*>(&e)) return 2;
    if (dynamic_cast<const ValueError*>(&e)) return 3;
    if (dynamic_cast<const ParseError*>(&e)) return 4;
    if (dynamic_cast<const CapacityError*>(&e)) return 5;
    if (dynamic_cast<const ContractError*>(&e)) return 6;
    if (dynamic_cast<const DiagnosticError*>(&e)) return 7;
    if (dynamic_cast<const DegenerateStateError*>(&e)) return 8;
    if (dynamic_cast<const InfeasibleError*>(&e)) return 9;
    return 12;
}

struct RefTensor {
    SparseTensor x;
};

FactorSet to_factors(int n, const uint64_t* dims, const uint64_t* ranks, const double* f) {
    FactorSet u;
    std::size_t o = 0;
    for (int v = 0; v < n; ++v) {
        Matrix m(dims[v], ranks[v]);
        std::memcpy(m.data.data(), f + o, sizeof(double) * dims[v] * ranks[v]);
        o += dims[v] * ranks[v];
        u.factors.push_back(std::move(m));
    }
    return u;
}

void from_factors(const FactorSet& u, double* out) {
    std::size_t o = 0;
    for (const Matrix& m : u.factors) {
        std::memcpy(out + o, m.data.data(), sizeof(double) * m.data.size());
        o += m.data.size();
    }
}

thread_local int64_t g_payload = 0;

}  // namespace

extern "C" {

int64_t ref_last_payload() { return g_payload; }
thread_local std::string g_msg;
int ref_tensor_dims(void* h, uint64_t* dims) {
    const SparseTensor& x = static_cast<RefTensor*>(h)->x;
    for (std::size_t m = 0; m < x.order(); ++m) dims[m] = x.dims()[m];
    return static_cast<int>(x.order());
}
const char* ref_last_message() { return g_msg.c_str(); }

// SparseTensor ctor (sparse_tensor.cpp:18-41).  Handle owns the tensor.
int ref_tensor_create(int n, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                      const double* vals, void** out) {
    try {
        std::vector<std::size_t> d(dims, dims + n);
        std::vector<index_t> c(coords, coords + nnz * n);
        std::vector<double> v(vals, vals + nnz);
        *out = new RefTensor{SparseTensor(std::move(d), std::move(c), std::move(v))};
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_gen_synthetic(int n, const uint64_t* dims, uint64_t nnz, uint64_t seed, void** out) {
    try {
        std::vector<std::size_t> d(dims, dims + n);
        *out = new RefTensor{gen_synthetic(d, nnz, seed)};
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

void ref_tensor_destroy(void* h) { delete static_cast<RefTensor*>(h); }

uint64_t ref_tensor_nnz(void* h) { return static_cast<RefTensor*>(h)->x.nnz(); }

void ref_tensor_export(void* h, uint32_t* coords, double* vals) {
    const SparseTensor& x = static_cast<RefTensor*>(h)->x;
    for (std::size_t e = 0; e < x.nnz(); ++e) {
        vals[e] = x.value(e);
        for (std::size_t m = 0; m < x.order(); ++m) coords[e * x.order() + m] = x.coord(e, m);
    }
}

void ref_tensor_buckets(void* h, int mode, uint64_t* offsets, uint64_t* entries) {
    const SparseTensor& x = static_cast<RefTensor*>(h)->x;
    const auto& b = x.mode_bucket(mode);
    for (std::size_t i = 0; i < b.offsets.size(); ++i) offsets[i] = b.offsets[i];
    for (std::size_t i = 0; i < b.entries.size(); ++i) entries[i] = b.entries[i];
}

double ref_norm_sq(void* h) { return norm_sq(static_cast<RefTensor*>(h)->x); }

int ref_ttmc_core(void* h, const uint64_t* ranks, const double* factors, double* core) {
    try {
        const SparseTensor& x = static_cast<RefTensor*>(h)->x;
        const int n = static_cast<int>(x.order());
        std::vector<uint64_t> dims(x.dims().begin(), x.dims().end());
        CoreTensor g = ttmc_core(x, to_factors(n, dims.data(), ranks, factors));
        std::memcpy(core, g.data.data(), sizeof(double) * g.data.size());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// variant 0: ttmctc_elementwise with precomputed core (or none if core==NULL)
// variant 1: ttmctc_matrix
int ref_ttmctc(void* h, const uint64_t* ranks, const double* factors, int mode,
               const double* core, int variant, double* a_out) {
    try {
        const SparseTensor& x = static_cast<RefTensor*>(h)->x;
        const int n = static_cast<int>(x.order());
        std::vector<uint64_t> dims(x.dims().begin(), x.dims().end());
        FactorSet u = to_factors(n, dims.data(), ranks, factors);
        Matrix a;
        if (variant == 1) {
            a = ttmctc_matrix(x, u, mode);
        } else if (core) {
            CoreTensor g(std::vector<std::size_t>(ranks, ranks + n));
            std::memcpy(g.data.data(), core, sizeof(double) * g.data.size());
            a = ttmctc_elementwise(x, u, mode, &g);
        } else {
            a = ttmctc_elementwise(x, u, mode);
        }
        std::memcpy(a_out, a.data.data(), sizeof(double) * a.data.size());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int ref_qr(uint64_t rows, uint64_t cols, const double* a, double* q) {
    try {
        Matrix m(rows, cols);
        std::memcpy(m.data.data(), a, sizeof(double) * rows * cols);
        Matrix r = qr_orthonormal(m);
        std::memcpy(q, r.data.data(), sizeof(double) * rows * cols);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

double ref_subspace_distance(uint64_t rows, uint64_t cols, const double* u, const double* v) {
    Matrix a(rows, cols), b(rows, cols);
    std::memcpy(a.data.data(), u, sizeof(double) * rows * cols);
    std::memcpy(b.data.data(), v, sizeof(double) * rows * cols);
    return subspace_distance(a, b);
}

int ref_random_factors(int n, const uint64_t* dims, const uint64_t* ranks, uint64_t seed,
                       double* out) {
    try {
        FactorSet u = random_factors(std::vector<std::size_t>(dims, dims + n),
                                     std::vector<std::size_t>(ranks, ranks + n), seed);
        from_factors(u, out);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

void ref_raw_stream(uint64_t seed, uint64_t n, uint64_t* out) {
    Rng r(seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.raw();
}

void ref_normal_stream(uint64_t seed, uint64_t n, double* out) {
    Rng r(seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.normal();
}

uint64_t ref_mix_seed(uint64_t seed, uint64_t salt) { return mix_seed(seed, salt); }

// tucker::hoqri (solvers.cpp:217-219) with random init from `seed`.  Fills the
// final model and the per-sweep trace.  kernel: 0 element-wise, 1 matrix.
int ref_hoqri(void* h, const uint64_t* ranks, uint64_t max_sweeps, double tol, uint64_t seed,
              int kernel, double* factors_out, double* core_out, uint64_t* sweeps_done,
              double* initial_objective, double* objective, double* fit, double* drift,
              double* elapsed_s) {
    try {
        const SparseTensor& x = static_cast<RefTensor*>(h)->x;
        SolverConfig cfg;
        cfg.ranks.assign(ranks, ranks + x.order());
        cfg.max_sweeps = max_sweeps;
        cfg.tol_fit_change = tol;
        cfg.seed = seed;
        cfg.kernel = kernel ? KernelVariant::kMatrix : KernelVariant::kElementwise;
        SolveResult r = hoqri(x, cfg);
        from_factors(r.model.factors, factors_out);
        std::memcpy(core_out, r.model.core.data.data(), sizeof(double) * r.model.core.size());
        *sweeps_done = r.trace.sweeps.size();
        *initial_objective = r.trace.initial_objective;
        for (std::size_t s = 0; s < r.trace.sweeps.size(); ++s) {
            objective[s] = r.trace.sweeps[s].objective;
            fit[s] = r.trace.sweeps[s].fit;
            elapsed_s[s] = r.trace.sweeps[s].elapsed_s;
            for (std::size_t m = 0; m < x.order(); ++m)
                drift[s * x.order() + m] = r.trace.sweeps[s].drift[m];
        }
        return 0;
    } catch (const DegenerateStateError& e) {
        g_payload = static_cast<int64_t>(e.mode);
        return 8;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// tucker::hoqri with gradient tracing (trace_gradients, tol_grad: solvers.cpp:58,
// 126-150, 165-167), random init from `seed`: the per-sweep trace plus every
// ModeUpdateRecord (sigma / lambda rows of stride ks).
int ref_hoqri_traced(void* h, const uint64_t* ranks, uint64_t max_sweeps, double tol, uint64_t seed, double tol_grad,
                     uint64_t ks, double* factors_out, double* core_out, uint64_t* sweeps_done, double* objective,
                     double* fit, double* grad, uint64_t* updates, double* f_before, double* f_after, double* sigma,
                     double* lambda) {
    try {
        const SparseTensor& x = static_cast<RefTensor*>(h)->x;
        SolverConfig cfg;
        cfg.ranks.assign(ranks, ranks + x.order());
        cfg.max_sweeps = max_sweeps;
        cfg.tol_fit_change = tol;
        cfg.seed = seed;
        cfg.trace_gradients = true;
        cfg.tol_grad = tol_grad;
        SolveResult r = hoqri(x, cfg);
        from_factors(r.model.factors, factors_out);
        std::memcpy(core_out, r.model.core.data.data(), sizeof(double) * r.model.core.size());
        const std::size_t n = x.order();
        *sweeps_done = r.trace.sweeps.size();
        for (std::size_t s = 0; s < r.trace.sweeps.size(); ++s) {
            objective[s] = r.trace.sweeps[s].objective;
            fit[s] = r.trace.sweeps[s].fit;
            for (std::size_t m = 0; m < n; ++m) grad[s * n + m] = r.trace.sweeps[s].grad_norm_sq[m];
        }
        *updates = r.trace.updates.size();
        for (std::size_t i = 0; i < r.trace.updates.size(); ++i) {
            const ModeUpdateRecord& up = r.trace.updates[i];
            f_before[i] = up.f_before;
            f_after[i] = up.f_after;
            for (std::size_t k = 0; k < up.sigma.size() && k < ks; ++k) sigma[i * ks + k] = up.sigma[k];
            for (std::size_t k = 0; k < up.lambda.size() && k < ks; ++k) lambda[i * ks + k] = up.lambda[k];
        }
        return 0;
    } catch (const DegenerateStateError& e) {
        g_payload = static_cast<int64_t>(e.mode);
        return 8;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// harness.cpp:101-161: the trace of a reference hoqri run (random init from
// `seed`) rendered by make_trace_file + write_trace_csv / write_trace_json.
// Writes NUL-terminated text into csv_out / json_out (capacity cap each).
int ref_trace_files(void* h, const uint64_t* ranks, uint64_t max_sweeps, uint64_t seed, char* csv_out,
                    char* json_out, uint64_t cap) {
    try {
        const SparseTensor& x = static_cast<RefTensor*>(h)->x;
        SolverConfig cfg;
        cfg.ranks.assign(ranks, ranks + x.order());
        cfg.max_sweeps = max_sweeps;
        cfg.tol_fit_change = 0.0;
        cfg.seed = seed;
        SolveResult r = hoqri(x, cfg);
        TraceFile t = make_trace_file("hoqri", cfg, x, r.trace);
        std::ostringstream c, j;
        write_trace_csv(c, t);
        write_trace_json(j, t);
        const std::string cs = c.str(), js = j.str();
        if (cs.size() + 1 > cap || js.size() + 1 > cap) return 5;
        std::memcpy(csv_out, cs.c_str(), cs.size() + 1);
        std::memcpy(json_out, js.c_str(), js.size() + 1);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// tucker::load_tns (sparse_tensor.cpp:136-215) on a text buffer: the tensor
// handle, or the exception's status, message (ref_last_message) and, for
// ParseError, the line (ref_last_payload).
int ref_tns_parse(const char* text, uint64_t len, int ovr_n, const uint64_t* ovr, void** out) {
    try {
        std::istringstream in(std::string(text, len));
        std::optional<std::vector<std::size_t>> o;
        if (ovr_n > 0) o = std::vector<std::size_t>(ovr, ovr + ovr_n);
        auto* t = new RefTensor{load_tns(in, o)};
        *out = t;
        return 0;
    } catch (const ParseError& e) {
        g_payload = static_cast<int64_t>(e.line_number);
        g_msg = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return code_of(e);
    }
}

// desk-scale paths of the reference: dense unfoldings, svd_leading, init_factors (random / HOSVD), hooi
int ref_densify_unfold(void* h, int mode, uint64_t cap, double* out) {
    try {
        Matrix m = densify_unfold(static_cast<RefTensor*>(h)->x, mode, cap);
        std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
        return 0;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return code_of(e);
    }
}

int ref_ttmc_unfold_dense(void* h, const uint64_t* ranks, const double* factors, int mode, uint64_t cap, double* out) {
    try {
        const SparseTensor& x = static_cast<RefTensor*>(h)->x;
        std::vector<uint64_t> dims(x.dims().begin(), x.dims().end());
        FactorSet u = to_factors(static_cast<int>(x.order()), dims.data(), ranks, factors);
        Matrix m = ttmc_unfold_dense(x, u, mode, cap);
        std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
        return 0;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return code_of(e);
    }
}

int ref_svd_leading(uint64_t rows, uint64_t cols, const double* y, uint64_t k, double* out) {
    try {
        Matrix a(rows, cols);
        std::memcpy(a.data.data(), y, sizeof(double) * rows * cols);
        Matrix u = svd_leading(a, k);
        std::memcpy(out, u.data.data(), sizeof(double) * u.data.size());
        return 0;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return code_of(e);
    }
}

int ref_init_factors(void* h, const uint64_t* ranks, uint64_t seed, int hosvd, uint64_t cap, double* out) {
    try {
        const SparseTensor& x = static_cast<RefTensor*>(h)->x;
        SolverConfig cfg;
        cfg.ranks.assign(ranks, ranks + x.order());
        cfg.seed = seed;
        cfg.init = hosvd ? InitMode::kHosvd : InitMode::kRandom;
        cfg.capacity_cap = cap;
        from_factors(init_factors(x, cfg), out);
        return 0;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return code_of(e);
    }
}

// hoqri / hooi with random or HOSVD init (and optional gradient tracing): the trace and final model
int ref_solve(void* h, int algorithm_hooi, const uint64_t* ranks, uint64_t max_sweeps, double tol, uint64_t seed,
              int hosvd, int trace_gradients, double* factors_out, double* core_out, uint64_t* sweeps_done,
              double* initial_objective, double* objective, double* fit, double* drift, double* grad) {
    try {
        const SparseTensor& x = static_cast<RefTensor*>(h)->x;
        SolverConfig cfg;
        cfg.ranks.assign(ranks, ranks + x.order());
        cfg.max_sweeps = max_sweeps;
        cfg.tol_fit_change = tol;
        cfg.seed = seed;
        cfg.init = hosvd ? InitMode::kHosvd : InitMode::kRandom;
        cfg.trace_gradients = trace_gradients != 0;
        SolveResult r = algorithm_hooi ? hooi(x, cfg) : hoqri(x, cfg);
        from_factors(r.model.factors, factors_out);
        std::memcpy(core_out, r.model.core.data.data(), sizeof(double) * r.model.core.size());
        *sweeps_done = r.trace.sweeps.size();
        *initial_objective = r.trace.initial_objective;
        const std::size_t n = x.order();
        for (std::size_t s2 = 0; s2 < r.trace.sweeps.size(); ++s2) {
            objective[s2] = r.trace.sweeps[s2].objective;
            fit[s2] = r.trace.sweeps[s2].fit;
            for (std::size_t m = 0; m < n; ++m) {
                drift[s2 * n + m] = r.trace.sweeps[s2].drift[m];
                grad[s2 * n + m] = r.trace.sweeps[s2].grad_norm_sq[m];
            }
        }
        return 0;
    } catch (const DegenerateStateError& e) {
        g_payload = static_cast<int64_t>(e.mode);
        g_msg = e.what();
        return 8;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return code_of(e);
    }
}

// Per-update replay with the reference's own kernels (the acceptance.cpp:268-304
// pattern), recording the core and factors after every sweep.  Starts from the
// given factors.
int ref_hoqri_replay(void* h, const uint64_t* ranks, const double* init_factors,
                     uint64_t sweeps, double* core_snap, double* factor_snap, double* drift) {
    try {
        const SparseTensor& x = static_cast<RefTensor*>(h)->x;
        const int n = static_cast<int>(x.order());
        std::vector<uint64_t> dims(x.dims().begin(), x.dims().end());
        FactorSet u = to_factors(n, dims.data(), ranks, init_factors);
        CoreTensor core = ttmc_core(x, u);
        std::size_t ftotal = 0;
        for (int v = 0; v < n; ++v) ftotal += dims[v] * ranks[v];
        for (uint64_t s = 0; s < sweeps; ++s) {
            for (int m = 0; m < n; ++m) {
                Matrix a = ttmctc_elementwise(x, u, m, &core);
                if (max_abs(a) == 0.0) {
                    g_payload = m + 1;
                    return 8;
                }
                Matrix old = std::move(u.factors[m]);
                u.factors[m] = qr_orthonormal(a);
                drift[s * n + m] = subspace_distance(u.factors[m], old);
                core = ttmc_core(x, u);
            }
            std::memcpy(core_snap + s * core.size(), core.data.data(),
                        sizeof(double) * core.size());
            from_factors(u, factor_snap + s * ftotal);
        }
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// ---- timing helpers for the CPU baseline (bench.py) -------------------------
// Times `reps` calls of ttmctc_elementwise(x, u, mode, &g) and of ttmc_core on
// `threads` host threads.  With threads > 1 the nonzeros are split into
// contiguous lexicographic slices, one reference SparseTensor per thread
// (built before timing), and each thread calls the unmodified reference
// kernel on its slice: the row/entry partitioning the reference's parallelism
// contract allows.  Returns seconds per call (wall clock).
struct RefSlices {
    std::vector<SparseTensor> parts;
};

void* ref_slices_create(void* h, int threads) {
    const SparseTensor& x = static_cast<RefTensor*>(h)->x;
    auto* s = new RefSlices;
    const std::size_t n = x.order(), nnz = x.nnz();
    for (int t = 0; t < threads; ++t) {
        std::size_t b = nnz * t / threads, e = nnz * (t + 1) / threads;
        std::vector<index_t> c;
        std::vector<double> v;
        c.reserve((e - b) * n);
        v.reserve(e - b);
        for (std::size_t i = b; i < e; ++i) {
            for (std::size_t m = 0; m < n; ++m) c.push_back(x.coord(i, m));
            v.push_back(x.value(i));
        }
        s->parts.emplace_back(x.dims(), std::move(c), std::move(v));
    }
    return s;
}

void ref_slices_destroy(void* s) { delete static_cast<RefSlices*>(s); }

// what: 0 = ttmctc_elementwise(mode, core given), 1 = ttmc_core
double ref_slices_time(void* s, const uint64_t* ranks, const double* factors,
                       const double* core, int mode, int what, int reps) {
    auto* sl = static_cast<RefSlices*>(s);
    const SparseTensor& x0 = sl->parts[0];
    const int n = static_cast<int>(x0.order());
    std::vector<uint64_t> dims(x0.dims().begin(), x0.dims().end());
    FactorSet u = to_factors(n, dims.data(), ranks, factors);
    CoreTensor g(std::vector<std::size_t>(ranks, ranks + n));
    std::memcpy(g.data.data(), core, sizeof(double) * g.data.size());
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) {
        std::vector<std::thread> th;
        for (std::size_t t = 0; t < sl->parts.size(); ++t)
            th.emplace_back([&, t] {
                if (what == 0)
                    (void)ttmctc_elementwise(sl->parts[t], u, mode, &g);
                else
                    (void)ttmc_core(sl->parts[t], u);
            });
        for (auto& t : th) t.join();
    }
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count() / reps;
}

double ref_time_qr(uint64_t rows, uint64_t cols, const double* a, int reps) {
    Matrix m(rows, cols);
    std::memcpy(m.data.data(), a, sizeof(double) * rows * cols);
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) {
        Matrix q = qr_orthonormal(m);
        Matrix d = matmul_tn(q, m);  // the drift product of subspace_distance
        (void)nuclear_norm(d);
    }
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count() / reps;
}

// ---- one mode update of the reference's solve loop, at full size -----------
// State = the factors and the fresh core that tucker::hoqri carries from one
// mode update to the next (solvers.cpp:66, 86-146, element-wise kernel with
// core_per_update).  ref_state_mode_update runs exactly that loop body:
//   A = ttmctc_elementwise(x, u, n, &core, &ws)   (solvers.cpp:90-91)
//   max_abs(A) == 0 -> DegenerateStateError      (:124)
//   U_n = qr_orthonormal(A); drift = subspace_distance(U_n, U_old)   (:139-141)
//   core = ttmc_core(x, u)                        (:143-144)
// and returns each phase's wall time (t_out: ttmctc, qr, drift, core).  Used
// by bench.py's reference arm and cpu_baseline: every timed step is one real,
// full-size mode update -- nothing is sampled or extrapolated.
struct RefState {
    FactorSet u;
    CoreTensor core;
    KernelWorkspace ws;
};

void* ref_state_create(void* h, const uint64_t* ranks, const double* factors) {
    const SparseTensor& x = static_cast<RefTensor*>(h)->x;
    const int n = static_cast<int>(x.order());
    std::vector<uint64_t> dims(x.dims().begin(), x.dims().end());
    auto* st = new RefState{to_factors(n, dims.data(), ranks, factors), CoreTensor{}, KernelWorkspace{}};
    st->core = ttmc_core(x, st->u);  // solvers.cpp:66
    return st;
}

void ref_state_destroy(void* s) { delete static_cast<RefState*>(s); }

int ref_state_mode_update(void* h, void* s, int mode, double* drift, double* t_out) {
    try {
        const SparseTensor& x = static_cast<RefTensor*>(h)->x;
        RefState& st = *static_cast<RefState*>(s);
        using clk = std::chrono::steady_clock;
        auto sec = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
        auto t0 = clk::now();
        Matrix a = ttmctc_elementwise(x, st.u, mode, &st.core, &st.ws);
        if (max_abs(a) == 0.0) {
            g_payload = mode + 1;
            return 8;
        }
        auto t1 = clk::now();
        Matrix old = std::move(st.u.factors[mode]);
        st.u.factors[mode] = qr_orthonormal(a);
        auto t2 = clk::now();
        *drift = subspace_distance(st.u.factors[mode], old);
        auto t3 = clk::now();
        st.core = ttmc_core(x, st.u);
        auto t4 = clk::now();
        t_out[0] = sec(t0, t1);
        t_out[1] = sec(t1, t2);
        t_out[2] = sec(t2, t3);
        t_out[3] = sec(t3, t4);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// The same per-sweep replay with the reference's OTHER kernel variant,
// KernelVariant::kMatrix (ttmctc_matrix, Alg. 4, kernels.cpp:165-262): per mode
// A = ttmctc_matrix(x, u, n, &ws), QR, drift, and -- as solve() does for the
// matrix variant without tracing (solvers.cpp:80-81, 153) -- the core only at
// the end of the sweep.  Its trajectory differs from the element-wise one only
// by floating-point summation order: the spread between the two is the
// reference's own rounding sensitivity on a given input.
int ref_hoqri_replay_matrix(void* h, const uint64_t* ranks, const double* init_factors, uint64_t sweeps,
                            double* core_snap, double* factor_snap, double* drift) {
    try {
        const SparseTensor& x = static_cast<RefTensor*>(h)->x;
        const int n = static_cast<int>(x.order());
        std::vector<uint64_t> dims(x.dims().begin(), x.dims().end());
        FactorSet u = to_factors(n, dims.data(), ranks, init_factors);
        KernelWorkspace ws;
        std::size_t ftotal = 0;
        for (int v = 0; v < n; ++v) ftotal += dims[v] * ranks[v];
        for (uint64_t s = 0; s < sweeps; ++s) {
            for (int m = 0; m < n; ++m) {
                Matrix a = ttmctc_matrix(x, u, m, &ws);
                if (max_abs(a) == 0.0) {
                    g_payload = m + 1;
                    return 8;
                }
                Matrix old = std::move(u.factors[m]);
                u.factors[m] = qr_orthonormal(a);
                drift[s * n + m] = subspace_distance(u.factors[m], old);
            }
            CoreTensor core = ttmc_core(x, u);
            std::memcpy(core_snap + s * core.size(), core.data.data(), sizeof(double) * core.size());
            from_factors(u, factor_snap + s * ftotal);
        }
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

}  // extern "C"
