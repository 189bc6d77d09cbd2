// tucker_shim.cpp — the reference's `tucker::` API over the engine's C-ABI.
//
// Every numeric entry point forwards to libhoqri_b200.so (include/hoqri_b200.h)
// and rethrows the C-ABI status as the reference's exception type with the
// same payload (errors.hpp taxonomy; DegenerateStateError keeps the 1-based
// mode).  Only K x K bookkeeping (matmul helpers on desk-scale matrices,
// unfold_core's index shuffle) runs on the host, as in the reference.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <ctime>
#include <filesystem>
#include <fstream>
#include <limits>
#include <algorithm>
#include <cmath>
#include <fstream>
#include <istream>
#include <ostream>
#include <sstream>

#include "hoqri_b200.h"
#include "tucker/harness.hpp"
#include "tucker/tucker_b200.hpp"

namespace tucker {

namespace {

[[noreturn]] void rethrow(int st) {
    std::string msg = hq_last_error();
    int64_t payload = hq_last_error_payload();
    switch (st) {
        case HQ_ERR_SHAPE: throw ShapeError(msg);
        case HQ_ERR_RANGE: throw RangeError(msg);
        case HQ_ERR_VALUE: throw ValueError(msg);
        case HQ_ERR_PARSE: throw ParseError(msg, static_cast<std::size_t>(payload));
        case HQ_ERR_CAPACITY: throw CapacityError(msg);
        case HQ_ERR_CONTRACT: throw ContractError(msg);
        case HQ_ERR_DIAGNOSTIC: throw DiagnosticError(msg);
        case HQ_ERR_DEGENERATE: throw DegenerateStateError(static_cast<std::size_t>(payload));
        case HQ_ERR_INFEASIBLE: throw InfeasibleError(msg);
        default: throw DeviceError(msg);
    }
}

inline void check(int st) {
    if (st != HQ_OK) rethrow(st);
}

void check_factors(const SparseTensor& x, const FactorSet& u) {  // kernels.cpp:12-22
    if (u.order() != x.order()) throw ShapeError("factor count does not match tensor order");
    for (std::size_t n = 0; n < x.order(); ++n) {
        if (u.factors[n].rows != x.dims()[n])
            throw ShapeError("factor " + std::to_string(n + 1) + " has " + std::to_string(u.factors[n].rows) +
                             " rows, tensor extent is " + std::to_string(x.dims()[n]));
        if (u.factors[n].cols == 0) throw ShapeError("factor with zero columns");
    }
}

std::vector<uint64_t> ranks_of(const FactorSet& u) {
    std::vector<uint64_t> r;
    for (const Matrix& m : u.factors) r.push_back(m.cols);
    return r;
}

std::vector<const double*> ptrs(const FactorSet& u) {
    std::vector<const double*> p;
    for (const Matrix& m : u.factors) p.push_back(m.data.data());
    return p;
}

}  // namespace

// ------------------------------------------------------------ dense_core --
Matrix identity(std::size_t n) {
    Matrix m(n, n);
    for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
}

Matrix transpose(const Matrix& a) {
    Matrix t(a.cols, a.rows);
    for (std::size_t i = 0; i < a.rows; ++i)
        for (std::size_t j = 0; j < a.cols; ++j) t(j, i) = a(i, j);
    return t;
}

Matrix matmul(const Matrix& a, const Matrix& b) {
    if (a.cols != b.rows) throw ShapeError("matmul: inner dimensions differ");
    Matrix c(a.rows, b.cols);
    for (std::size_t i = 0; i < a.rows; ++i)
        for (std::size_t k = 0; k < a.cols; ++k)
            for (std::size_t j = 0; j < b.cols; ++j) c(i, j) += a(i, k) * b(k, j);
    return c;
}

Matrix matmul_tn(const Matrix& a, const Matrix& b) {
    if (a.rows != b.rows) throw ShapeError("matmul_tn: row counts differ");
    Matrix c(a.cols, b.cols);
    for (std::size_t k = 0; k < a.rows; ++k)
        for (std::size_t i = 0; i < a.cols; ++i)
            for (std::size_t j = 0; j < b.cols; ++j) c(i, j) += a(k, i) * b(k, j);
    return c;
}

Matrix matmul_nt(const Matrix& a, const Matrix& b) {
    if (a.cols != b.cols) throw ShapeError("matmul_nt: column counts differ");
    Matrix c(a.rows, b.rows);
    for (std::size_t i = 0; i < a.rows; ++i)
        for (std::size_t j = 0; j < b.rows; ++j) {
            double s = 0.0;
            for (std::size_t k = 0; k < a.cols; ++k) s += a(i, k) * b(j, k);
            c(i, j) = s;
        }
    return c;
}

double frob_norm_sq(const Matrix& a) {
    double s = 0.0;
    for (double v : a.data) s += v * v;
    return s;
}

double max_abs(const Matrix& a) {
    double m = 0.0;
    for (double v : a.data) m = std::max(m, std::fabs(v));
    return m;
}

double max_abs_diff(const Matrix& a, const Matrix& b) {
    if (a.rows != b.rows || a.cols != b.cols) throw ShapeError("max_abs_diff: shapes differ");
    double m = 0.0;
    for (std::size_t i = 0; i < a.data.size(); ++i) m = std::max(m, std::fabs(a.data[i] - b.data[i]));
    return m;
}

CoreTensor::CoreTensor(std::vector<std::size_t> r) : ranks(std::move(r)) {
    std::size_t total = 1;
    for (std::size_t k : ranks) {
        if (k == 0) throw ShapeError("zero core rank");
        total *= k;
    }
    data.assign(total, 0.0);
}

double norm_sq(const CoreTensor& g) {
    double s = 0.0;
    for (double v : g.data) s += v * v;
    return s;
}

double FactorSet::orthonormality_defect() const {
    double worst = 0.0;
    for (const Matrix& u : factors) {
        Matrix g = matmul_tn(u, u);
        for (std::size_t i = 0; i < g.rows; ++i)
            for (std::size_t j = 0; j < g.cols; ++j)
                worst = std::max(worst, std::fabs(g(i, j) - (i == j ? 1.0 : 0.0)));
    }
    return worst;
}

Matrix qr_orthonormal(const Matrix& a) {
    if (a.rows < a.cols) throw ShapeError("qr_orthonormal: need rows >= cols");
    Matrix q(a.rows, a.cols);
    if (a.cols == 0) return q;
    check(hq_qr_orthonormal(a.rows, a.cols, a.data.data(), q.data.data()));
    return q;
}

EigResult jacobi_eig_sym(Matrix m) {  // dense_core.cpp:200-262 contract; eigen-solve on the device
    if (m.rows != m.cols) throw ShapeError("jacobi_eig_sym: square matrix required");
    EigResult r;
    r.values.resize(m.rows);
    r.vectors = Matrix(m.rows, m.rows);
    check(hq_sym_eig(m.rows, m.data.data(), r.values.data(), r.vectors.data.data()));
    return r;
}

std::vector<double> gram_eigvals_desc(const Matrix& m) {  // dense_core.cpp:371-386
    if (m.rows != m.cols) throw ShapeError("gram_eigvals_desc: square matrix required");
    const double scale = std::max(1.0, std::sqrt(frob_norm_sq(m)));
    for (std::size_t i = 0; i < m.rows; ++i)
        for (std::size_t j = i + 1; j < m.cols; ++j)
            if (std::fabs(m(i, j) - m(j, i)) > 1e-10 * scale)
                throw ContractError("gram_eigvals_desc: matrix is not symmetric");
    std::vector<double> ev(m.rows);
    check(hq_sym_eig(m.rows, m.data.data(), ev.data(), nullptr));
    for (double& v : ev) {
        if (v < -1e-10 * scale) throw ContractError("gram_eigvals_desc: matrix is not PSD");
        v = std::max(v, 0.0);
    }
    return ev;
}

double nuclear_norm(const Matrix& m) {  // dense_core.cpp:329-335: sum of sqrt(eig(M^T M))
    if (m.rows != m.cols) throw ShapeError("nuclear_norm: square matrix required");
    const Matrix mtm = matmul_tn(m, m);
    std::vector<double> ev(m.rows);
    check(hq_sym_eig(m.rows, mtm.data.data(), ev.data(), nullptr));
    double s = 0.0;
    for (double v : ev) s += std::sqrt(std::max(v, 0.0));
    return s;
}

std::vector<std::size_t> unfold_col_strides(const std::vector<std::size_t>& dims, std::size_t mode) {
    if (mode >= dims.size()) throw RangeError("unfold: mode out of range");
    std::vector<std::size_t> st(dims.size(), 0);
    std::size_t s = 1;
    for (std::size_t v = dims.size(); v-- > 0;) {
        if (v == mode) continue;
        st[v] = s;
        s *= dims[v];
    }
    return st;
}

Matrix unfold_core(const CoreTensor& g, std::size_t mode) {
    const std::size_t n = g.order();
    if (mode >= n) throw RangeError("unfold_core: mode out of range");
    Matrix m(g.ranks[mode], g.size() / g.ranks[mode]);
    std::vector<std::size_t> cs = unfold_col_strides(g.ranks, mode);
    std::vector<std::size_t> idx(n, 0);
    for (std::size_t lin = 0; lin < g.size(); ++lin) {
        std::size_t col = 0;
        for (std::size_t v = 0; v < n; ++v)
            if (v != mode) col += idx[v] * cs[v];
        m(idx[mode], col) = g.data[lin];
        for (std::size_t v = n; v-- > 0;) {
            if (++idx[v] < g.ranks[v]) break;
            idx[v] = 0;
        }
    }
    return m;
}

// --------------------------------------------------------- sparse tensor --
struct SparseTensor::Host {
    std::mutex mu;
    bool have_entries = false;
    std::vector<index_t> coords;
    std::vector<double> values;
    std::vector<std::unique_ptr<ModeBuckets>> buckets;
};

SparseTensor::SparseTensor(std::vector<std::size_t> dims, std::vector<index_t> coords, std::vector<double> values)
    : dims_(std::move(dims)) {
    const std::size_t n = dims_.size();
    if (n == 0) throw ShapeError("sparse tensor needs at least one mode");
    for (std::size_t d : dims_)
        if (d == 0) throw ShapeError("zero extent");
    if (coords.size() != values.size() * n) throw ShapeError("coordinate array does not match entry count");
    std::vector<uint64_t> d(dims_.begin(), dims_.end());
    hq_tensor* h = nullptr;
    check(hq_tensor_create(static_cast<int>(n), d.data(), values.size(), coords.data(), values.data(), nullptr, &h));
    dev_ = std::shared_ptr<hq_tensor>(h, [](hq_tensor* p) { hq_tensor_destroy(p); });
    uint64_t nnz = 0;
    check(hq_tensor_info(h, nullptr, nullptr, &nnz));
    nnz_ = nnz;
    host_ = std::make_shared<Host>();
    host_->buckets.resize(n);
}

const std::vector<index_t>& SparseTensor::coords() const {
    std::lock_guard<std::mutex> lk(host_->mu);
    if (!host_->have_entries) {
        host_->coords.resize(nnz_ * dims_.size());
        host_->values.resize(nnz_);
        check(hq_tensor_export(dev_.get(), host_->coords.data(), host_->values.data()));
        host_->have_entries = true;
    }
    return host_->coords;
}

const std::vector<double>& SparseTensor::values() const {
    coords();
    return host_->values;
}

const SparseTensor::ModeBuckets& SparseTensor::mode_bucket(std::size_t mode) const {
    std::lock_guard<std::mutex> lk(host_->mu);
    auto& b = host_->buckets.at(mode);
    if (!b) {
        auto nb = std::make_unique<ModeBuckets>();
        std::vector<uint64_t> off(dims_[mode] + 1), ent(nnz_);
        check(hq_tensor_buckets(dev_.get(), static_cast<int>(mode), off.data(), ent.data()));
        nb->offsets.assign(off.begin(), off.end());
        nb->entries.assign(ent.begin(), ent.end());
        b = std::move(nb);
    }
    return *b;
}

double norm_sq(const SparseTensor& x) {
    double v = 0.0;
    check(hq_tensor_norm_sq(x.device(), &v));
    return v;
}

SparseTensor load_tns(std::istream& in, std::optional<std::vector<std::size_t>> dims_override) {
    // sparse_tensor.cpp:136-215: the engine's threaded parser (hq_tns_parse), same rules and errors
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    std::vector<uint64_t> ovr;
    if (dims_override) ovr.assign(dims_override->begin(), dims_override->end());
    hq_tns* p = nullptr;
    check(hq_tns_parse(text.data(), text.size(), static_cast<int>(ovr.size()), ovr.empty() ? nullptr : ovr.data(), &p));
    std::unique_ptr<hq_tns, int (*)(hq_tns*)> guard_p(p, hq_tns_destroy);
    int order = 0;
    uint64_t nnz = 0;
    uint64_t d[64] = {0};
    check(hq_tns_info(p, &order, d, &nnz));
    const std::size_t nd = dims_override ? dims_override->size() : static_cast<std::size_t>(order);
    std::vector<index_t> coords(nnz * static_cast<std::size_t>(order));
    std::vector<double> values(nnz);
    check(hq_tns_copy(p, coords.data(), values.data()));
    return SparseTensor(std::vector<std::size_t>(d, d + nd), std::move(coords), std::move(values));
}

SparseTensor load_tns_file(const std::string& path, std::optional<std::vector<std::size_t>> dims_override) {
    std::ifstream in(path);
    if (!in) throw Error("cannot open '" + path + "'");
    return load_tns(in, std::move(dims_override));
}

void write_tns(std::ostream& out, const SparseTensor& x) {
    out << "dims:";
    for (std::size_t d : x.dims()) out << ' ' << d;
    out << '\n';
    char buf[64];
    for (std::size_t e = 0; e < x.nnz(); ++e) {
        for (std::size_t m = 0; m < x.order(); ++m) out << (x.coord(e, m) + 1) << ' ';
        std::snprintf(buf, sizeof(buf), "%.17g", x.value(e));
        out << buf << '\n';
    }
}

void write_tns_file(const std::string& path, const SparseTensor& x) {
    std::ofstream out(path);
    if (!out) throw Error("cannot open '" + path + "' for writing");
    write_tns(out, x);
}

// --------------------------------------------------------------- kernels --
CoreTensor ttmc_core(const SparseTensor& x, const FactorSet& u) {
    check_factors(x, u);
    auto r = ranks_of(u);
    CoreTensor g(std::vector<std::size_t>(r.begin(), r.end()));
    auto p = ptrs(u);
    check(hq_ttmc_core(x.device(), p.data(), r.data(), g.data.data()));
    return g;
}

static Matrix ttmctc_common(const SparseTensor& x, const FactorSet& u, std::size_t mode, const CoreTensor* core,
                            int variant, KernelWorkspace* ws) {
    check_factors(x, u);
    if (mode >= x.order()) throw RangeError("ttmctc: mode out of range");
    auto r = ranks_of(u);
    if (core && std::vector<std::size_t>(r.begin(), r.end()) != core->ranks)
        throw ShapeError("precomputed core ranks do not match the factors");
    Matrix a(x.dims()[mode], u.factors[mode].cols);
    if (ws) {  // device scratch of one call: A plus the per-CTA partials (upper bound)
        std::size_t l = 1;
        for (std::size_t v = 0; v < r.size(); ++v)
            if (v != mode) l *= r[v];
        std::size_t abytes = a.data.size() * sizeof(double);
        std::size_t part = std::min<std::size_t>(296, (x.dims()[mode] + 31) / 32) * (l + r[mode] + 1) * r[mode] * 8;
        ws->meter.acquire(abytes);
        ws->meter.acquire(part);
        ws->meter.release(part);
        ws->meter.release(abytes);
    }
    auto p = ptrs(u);
    check(hq_ttmctc(x.device(), p.data(), r.data(), static_cast<int>(mode), core ? core->data.data() : nullptr,
                    variant, a.data.data()));
    return a;
}

Matrix ttmctc_elementwise(const SparseTensor& x, const FactorSet& u, std::size_t mode,
                          const CoreTensor* precomputed_core, KernelWorkspace* ws) {
    return ttmctc_common(x, u, mode, precomputed_core, 0, ws);
}

Matrix ttmctc_matrix(const SparseTensor& x, const FactorSet& u, std::size_t mode, KernelWorkspace* ws) {
    return ttmctc_common(x, u, mode, nullptr, 1, ws);
}

// -------------------------------------------------------------- manifold --
Matrix project_tangent(const Matrix& u, const Matrix& a) {  // manifold.cpp:10-22: A - U sym(U^T A)
    if (u.rows != a.rows || u.cols != a.cols)
        throw ShapeError("project_tangent: U and A must have the same shape");
    Matrix s = matmul_tn(u, a);
    for (std::size_t i = 0; i < s.rows; ++i)
        for (std::size_t j = i + 1; j < s.cols; ++j) s(i, j) = s(j, i) = 0.5 * (s(i, j) + s(j, i));
    const Matrix us = matmul(u, s);
    Matrix out = a;
    for (std::size_t i = 0; i < out.data.size(); ++i) out.data[i] -= us.data[i];
    return out;
}

Matrix riemannian_grad(const Matrix& u, const Matrix& a, const Matrix& gn) {  // manifold.cpp:24-35
    if (u.rows != a.rows || u.cols != a.cols)
        throw ShapeError("riemannian_grad: U and A must have the same shape");
    if (gn.rows != u.cols) throw ShapeError("riemannian_grad: core unfolding does not match the mode rank");
    const Matrix ugg = matmul(u, matmul_nt(gn, gn));
    Matrix out(a.rows, a.cols);
    for (std::size_t i = 0; i < out.data.size(); ++i) out.data[i] = 2.0 * (a.data[i] - ugg.data[i]);
    return out;
}

double grad_norm_sq(const Matrix& a, const Matrix& gn) {  // manifold.cpp:37-53: 4(||A||^2 - ||G G^T||^2)
    if (gn.rows != a.cols) throw ShapeError("grad_norm_sq: core unfolding does not match the mode rank");
    const double a_sq = frob_norm_sq(a);
    const double r = 4.0 * (a_sq - frob_norm_sq(matmul_nt(gn, gn)));
    if (r < -1e-8 * std::max(1.0, 4.0 * a_sq))
        throw DiagnosticError("grad_norm_sq is negative beyond rounding; orthonormality is broken upstream");
    if (std::fabs(r) <= 1e-10) return 0.0;
    return std::max(r, 0.0);
}

InterlacingResult interlacing_check(const Matrix& a, const Matrix& gn) {  // manifold.cpp:62-84
    if (gn.rows != a.cols) throw ShapeError("interlacing_check: core unfolding does not match the mode rank");
    InterlacingResult r;
    r.sigma = gram_eigvals_desc(matmul_tn(a, a));
    for (double& v : r.sigma) v = std::sqrt(v);
    r.lambda = gram_eigvals_desc(matmul_nt(gn, gn));
    const double scale = std::max(1.0, r.sigma.empty() ? 0.0 : r.sigma[0]);
    for (std::size_t k = 0; k < r.sigma.size(); ++k) {
        const double margin = r.sigma[k] - r.lambda[k];
        if (k == 0 || margin < r.min_margin) r.min_margin = margin;
        if (margin < -1e-9 * scale)
            throw DiagnosticError("interlacing violated at k=" + std::to_string(k + 1) +
                                  "; upstream state is numerically corrupted");
    }
    return r;
}

double subspace_distance(const Matrix& u, const Matrix& v) {
    if (u.rows != v.rows || u.cols != v.cols) throw ShapeError("subspace_distance: shapes differ");
    double d = 0.0;
    check(hq_subspace_distance(u.rows, u.cols, u.data.data(), v.data.data(), &d));
    return d;
}

// --------------------------------------------------------------- solvers --
FactorSet random_factors(const std::vector<std::size_t>& dims, const std::vector<std::size_t>& ranks,
                         std::uint64_t seed) {
    if (dims.size() != ranks.size()) throw ShapeError("random_factors: dims/ranks length mismatch");
    FactorSet u;
    std::vector<double*> out;
    for (std::size_t n = 0; n < dims.size(); ++n) u.factors.emplace_back(dims[n], ranks[n]);
    for (auto& m : u.factors) out.push_back(m.data.data());
    std::vector<uint64_t> d(dims.begin(), dims.end()), r(ranks.begin(), ranks.end());
    check(hq_random_factors(static_cast<int>(dims.size()), d.data(), r.data(), seed, out.data()));
    return u;
}

static void check_ranks(const SparseTensor& x, const std::vector<std::size_t>& ranks) {  // solvers.cpp:22-30
    if (ranks.size() != x.order()) throw ShapeError("rank count does not match tensor order");
    for (std::size_t n = 0; n < ranks.size(); ++n)
        if (ranks[n] < 1 || ranks[n] > x.dims()[n])
            throw ShapeError("rank for mode " + std::to_string(n + 1) + " must lie in [1, " +
                             std::to_string(x.dims()[n]) + "]");
}

FactorSet init_factors(const SparseTensor& x, const SolverConfig& config) {  // solvers.cpp:202-215
    check_ranks(x, config.ranks);
    if (config.init == InitMode::kRandom) return random_factors(x.dims(), config.ranks, config.seed);
    hq_config c;
    hq_config_default(&c);
    c.order = static_cast<int>(x.order());
    for (std::size_t v = 0; v < x.order(); ++v) c.ranks[v] = config.ranks[v];
    c.init = 1;
    c.capacity_cap = config.capacity_cap;
    FactorSet u;
    for (std::size_t v = 0; v < x.order(); ++v) u.factors.emplace_back(x.dims()[v], config.ranks[v]);
    std::vector<double*> fo;
    for (auto& m : u.factors) fo.push_back(m.data.data());
    check(hq_init_factors(x.device(), &c, fo.data()));
    return u;
}

Matrix svd_leading(const Matrix& y, std::size_t k) {  // dense_core.hpp:64 (device eigen-solve)
    if (k > std::min(y.rows, y.cols)) throw ShapeError("svd_leading: k exceeds min(rows, cols)");
    Matrix u(y.rows, k);
    if (k) check(hq_svd_leading(y.rows, y.cols, y.data.data(), k, u.data.data()));
    return u;
}

Matrix densify_unfold(const SparseTensor& x, std::size_t mode, std::size_t capacity_cap) {  // kernels.hpp:70-71
    if (mode >= x.order()) throw RangeError("densify_unfold: mode out of range");
    std::size_t cols = 1;
    for (std::size_t v = 0; v < x.order(); ++v)
        if (v != mode) cols *= x.dims()[v];
    if (cols != 0 && x.dims()[mode] > capacity_cap / cols)
        throw CapacityError("dense unfolding of " + std::to_string(x.dims()[mode]) + " x " + std::to_string(cols) +
                            " exceeds the capacity cap; this path is desk-scale only");
    Matrix m(x.dims()[mode], cols);
    check(hq_densify_unfold(x.device(), static_cast<int>(mode), capacity_cap, m.data.data()));
    return m;
}

Matrix ttmc_unfold_dense(const SparseTensor& x, const FactorSet& u, std::size_t mode,
                         std::size_t capacity_cap) {  // kernels.hpp:66-67
    check_factors(x, u);
    if (mode >= x.order()) throw RangeError("ttmc_unfold_dense: mode out of range");
    std::size_t cols = 1;
    std::vector<uint64_t> r;
    for (std::size_t v = 0; v < x.order(); ++v) {
        r.push_back(u.factors[v].cols);
        if (v != mode) cols *= u.factors[v].cols;
    }
    if (cols != 0 && x.dims()[mode] > capacity_cap / cols)
        throw CapacityError("dense unfolding of " + std::to_string(x.dims()[mode]) + " x " + std::to_string(cols) +
                            " exceeds the capacity cap; this path is desk-scale only");
    Matrix y(x.dims()[mode], cols);
    auto p = ptrs(u);
    check(hq_ttmc_unfold_dense(x.device(), p.data(), r.data(), static_cast<int>(mode), capacity_cap, y.data.data()));
    return y;
}

static SolveResult solve_impl(const SparseTensor& x, const SolverConfig& config, const FactorSet* start,
                              bool hooi_alg = false) {
    check_ranks(x, config.ranks);
    if (config.max_sweeps < 1) throw ShapeError("max_sweeps must be at least 1");
    if (config.tol_fit_change < 0.0) throw ShapeError("tolerance must be nonnegative");
    const std::size_t n = x.order();
    hq_config c;
    hq_config_default(&c);
    c.order = static_cast<int>(n);
    for (std::size_t v = 0; v < n; ++v) c.ranks[v] = config.ranks[v];
    c.max_sweeps = config.max_sweeps;
    c.tol_fit_change = config.tol_fit_change;
    c.seed = config.seed;
    c.kernel = config.kernel == KernelVariant::kMatrix ? 1 : 0;
    c.trace_gradients = config.trace_gradients ? 1 : 0;
    c.tol_grad = config.tol_grad;
    c.init = config.init == InitMode::kHosvd ? 1 : 0;
    c.capacity_cap = config.capacity_cap;
    std::vector<const double*> init;
    if (start) {
        if (start->order() != n) throw ShapeError("factor count does not match tensor order");
        c.init = 2;
        init = ptrs(*start);
    }
    SolveResult res;
    for (std::size_t v = 0; v < n; ++v) res.model.factors.factors.emplace_back(x.dims()[v], config.ranks[v]);
    res.model.core = CoreTensor(config.ranks);
    std::vector<double*> fo;
    for (auto& m : res.model.factors.factors) fo.push_back(m.data.data());
    const std::size_t nu = config.max_sweeps * n;
    std::size_t ks = 1;
    for (std::size_t k : config.ranks) ks = std::max(ks, k);
    std::vector<double> obj(config.max_sweeps), fit(config.max_sweeps), drift(nu), el(config.max_sweeps), grad(nu),
        fb(nu), fa(nu), uel(nu), sig(nu * ks), lam(nu * ks);
    hq_trace tr{};
    tr.objective = obj.data();
    tr.fit = fit.data();
    tr.drift = drift.data();
    tr.elapsed_s = el.data();
    tr.grad_norm_sq = grad.data();
    tr.upd_f_before = fb.data();
    tr.upd_f_after = fa.data();
    tr.upd_elapsed_s = uel.data();
    tr.upd_sigma = sig.data();
    tr.upd_lambda = lam.data();
    tr.sigma_stride = ks;
    if (hooi_alg)
        check(hq_hooi(x.device(), &c, start ? init.data() : nullptr, fo.data(), res.model.core.data.data(), &tr));
    else
        check(hq_hoqri(x.device(), &c, start ? init.data() : nullptr, fo.data(), res.model.core.data.data(), &tr));
    res.model.data_norm_sq = tr.data_norm_sq;
    res.trace.data_norm_sq = tr.data_norm_sq;
    res.trace.initial_objective = tr.initial_objective;
    for (std::size_t s = 0; s < tr.sweeps; ++s) {
        SweepRecord r;
        r.sweep = s + 1;
        r.elapsed_s = el[s];
        r.objective = obj[s];
        r.fit = fit[s];
        r.grad_norm_sq.assign(grad.begin() + s * n, grad.begin() + (s + 1) * n);
        for (double g : r.grad_norm_sq) r.total_grad_norm_sq += g;
        r.drift.assign(drift.begin() + s * n, drift.begin() + (s + 1) * n);
        res.trace.sweeps.push_back(std::move(r));
    }
    for (std::size_t i = 0; i < tr.updates; ++i) {  // solvers.cpp:127-150
        ModeUpdateRecord up;
        up.sweep = i / n + 1;
        up.mode = i % n;
        up.f_before = fb[i];
        up.f_after = fa[i];
        up.grad_norm_sq = grad[i];
        up.sigma.assign(sig.begin() + i * ks, sig.begin() + i * ks + config.ranks[up.mode]);
        up.lambda.assign(lam.begin() + i * ks, lam.begin() + i * ks + config.ranks[up.mode]);
        up.elapsed_s = uel[i];
        res.trace.updates.push_back(std::move(up));
    }
    return res;
}

SolveResult hoqri(const SparseTensor& x, const SolverConfig& config) { return solve_impl(x, config, nullptr); }

SolveResult hooi(const SparseTensor& x, const SolverConfig& config) {  // solvers.hpp:82-83, on the device
    return solve_impl(x, config, nullptr, true);
}

SolveResult hoqri_from(const SparseTensor& x, const SolverConfig& config, const FactorSet& start) {
    return solve_impl(x, config, &start);
}

GradientReport gradient_report(const SparseTensor& x, const FactorSet& u) {  // solvers.cpp:238-252
    const CoreTensor core = ttmc_core(x, u);
    GradientReport rep;
    for (std::size_t n = 0; n < x.order(); ++n) {
        const Matrix a = ttmctc_elementwise(x, u, n, &core);
        const Matrix gn = unfold_core(core, n);
        rep.per_mode_norm_sq.push_back(grad_norm_sq(a, gn));
        InterlacingResult il = interlacing_check(a, gn);
        rep.sigma.push_back(std::move(il.sigma));
        rep.lambda.push_back(std::move(il.lambda));
        rep.total_norm_sq += rep.per_mode_norm_sq.back();
    }
    return rep;
}

DescentCheck check_descent_inequality(const IterationTrace& trace, double data_norm_sq) {  // solvers.cpp:254-270
    DescentCheck out;
    const double slack = 1e-8 * data_norm_sq * data_norm_sq;
    for (const ModeUpdateRecord& up : trace.updates) {
        ++out.checked;
        const double excess = up.grad_norm_sq - (4.0 * data_norm_sq * (up.f_after - up.f_before) + slack);
        if (excess > 0.0) {
            ++out.violations;
            out.ok = false;
        }
        out.worst_violation = std::max(out.worst_violation, excess);
    }
    return out;
}

double fit_error(const SparseTensor& x, const TuckerModel& model) {
    if (model.factors.order() != x.order()) throw ShapeError("fit_error: model order does not match the tensor");
    double out = 0.0;
    check(hq_fit_error(model.data_norm_sq, model.core.data.size(), model.core.data.data(), &out));
    return out;
}


// ================================================================ harness ==
// The reference's experiment / trace surface (harness.hpp) over the engine.
namespace {

std::string fmt17(double v) {  // harness.cpp:27-31
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}

std::string joined(const std::vector<std::size_t>& v) {
    std::string s;
    for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
    return s;
}

std::string now_utc() {
    std::time_t t = std::time(nullptr);
    std::tm tm{};
    gmtime_r(&t, &tm);
    char buf[32];
    std::strftime(buf, sizeof(buf), "%Y-%m-%dT%H:%M:%SZ", &tm);
    return buf;
}

std::string json_string(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        switch (c) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\n': o += "\\n"; break;
            case '\t': o += "\\t"; break;
            default:
                if (static_cast<unsigned char>(c) < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof(b), "\\u%04x", c);
                    o += b;
                } else {
                    o += c;
                }
        }
    }
    return o + "\"";
}

std::string json_number(double v) { return std::isfinite(v) ? fmt17(v) : "null"; }

// a small reader for the trace document: {"header": {str: str}, "columns": [str], "rows": [[num]]}
struct JsonIn {
    std::string s;
    std::size_t p = 0;
    void ws() {
        while (p < s.size() && std::isspace(static_cast<unsigned char>(s[p]))) ++p;
    }
    [[noreturn]] void bad(const std::string& what) { throw ParseError("trace json: " + what); }
    void expect(char c) {
        ws();
        if (p >= s.size() || s[p] != c) bad(std::string("expected '") + c + "'");
        ++p;
    }
    bool peek(char c) {
        ws();
        return p < s.size() && s[p] == c;
    }
    std::string str() {
        expect('"');
        std::string o;
        while (p < s.size() && s[p] != '"') {
            char c = s[p++];
            if (c == '\\') {
                if (p >= s.size()) bad("bad escape");
                char e = s[p++];
                switch (e) {
                    case 'n': o += '\n'; break;
                    case 't': o += '\t'; break;
                    case 'r': o += '\r'; break;
                    case 'b': o += '\b'; break;
                    case 'f': o += '\f'; break;
                    case 'u': {
                        if (p + 4 > s.size()) bad("bad \\u escape");
                        o += static_cast<char>(std::stoi(s.substr(p, 4), nullptr, 16));
                        p += 4;
                        break;
                    }
                    default: o += e;
                }
            } else {
                o += c;
            }
        }
        expect('"');
        return o;
    }
    double num() {
        ws();
        if (s.compare(p, 4, "null") == 0) {
            p += 4;
            return std::numeric_limits<double>::quiet_NaN();
        }
        const char* b = s.data() + p;
        char* e = nullptr;
        double v = std::strtod(b, &e);
        if (e == b) bad("bad number");
        p += static_cast<std::size_t>(e - b);
        return v;
    }
    void skip_value() {
        ws();
        if (peek('"')) {
            str();
        } else if (peek('{')) {
            expect('{');
            if (!peek('}'))
                do {
                    str();
                    expect(':');
                    skip_value();
                } while (peek(',') && (++p, true));
            expect('}');
        } else if (peek('[')) {
            expect('[');
            if (!peek(']'))
                do skip_value();
                while (peek(',') && (++p, true));
            expect(']');
        } else if (s.compare(p, 4, "true") == 0 || s.compare(p, 4, "null") == 0) {
            p += 4;
        } else if (s.compare(p, 5, "false") == 0) {
            p += 5;
        } else {
            num();
        }
    }
};

}  // namespace

SparseTensor gen_synthetic(const std::vector<std::size_t>& dims, std::size_t nnz, std::uint64_t seed) {
    std::vector<uint64_t> d(dims.begin(), dims.end());
    if (d.empty()) throw ShapeError("gen_synthetic: need at least one mode");
    std::vector<index_t> coords(nnz * dims.size());
    std::vector<double> vals(nnz);
    check(hq_gen_synthetic(static_cast<int>(d.size()), d.data(), nnz, seed, coords.data(), vals.data()));
    return SparseTensor(dims, std::move(coords), std::move(vals));
}

TraceFile make_trace_file(const std::string& solver_name, const SolverConfig& config, const SparseTensor& x,
                          const IterationTrace& trace) {  // harness.cpp:101-140: same keys and columns
    TraceFile t;
    t.header["trace_version"] = std::to_string(kTraceVersion);
    t.header["tool_version"] = kToolVersion;
    t.header["timestamp"] = now_utc();
    t.header["solver"] = solver_name;
    t.header["dims"] = joined(x.dims());
    t.header["nnz"] = std::to_string(x.nnz());
    t.header["ranks"] = joined(config.ranks);
    t.header["seed"] = std::to_string(config.seed);
    t.header["init"] = config.init == InitMode::kRandom ? "random" : "hosvd";
    t.header["kernel"] = config.kernel == KernelVariant::kElementwise ? "elementwise" : "matrix";
    t.header["max_sweeps"] = std::to_string(config.max_sweeps);
    t.header["tol"] = fmt17(config.tol_fit_change);
    t.header["data_norm_sq"] = fmt17(trace.data_norm_sq);
    t.header["initial_objective"] = fmt17(trace.initial_objective);
    t.columns = {"sweep", "elapsed_s", "objective", "fit", "grad_norm_sq"};
    for (std::size_t n = 0; n < x.order(); ++n) t.columns.push_back("drift_" + std::to_string(n + 1));
    for (const SweepRecord& r : trace.sweeps) {
        std::vector<double> row{static_cast<double>(r.sweep), r.elapsed_s, r.objective, r.fit, r.total_grad_norm_sq};
        row.insert(row.end(), r.drift.begin(), r.drift.end());
        t.rows.push_back(std::move(row));
    }
    return t;
}

void write_trace_csv(std::ostream& out, const TraceFile& t) {  // harness.cpp:142-153
    for (const auto& kv : t.header) out << "# " << kv.first << "=" << kv.second << "\n";
    for (std::size_t i = 0; i < t.columns.size(); ++i) out << (i ? "," : "") << t.columns[i];
    out << "\n";
    for (const auto& row : t.rows) {
        for (std::size_t i = 0; i < row.size(); ++i) out << (i ? "," : "") << fmt17(row[i]);
        out << "\n";
    }
}

void write_trace_json(std::ostream& out, const TraceFile& t) {  // harness.cpp:155-161 (keys in sorted order)
    out << "{\n  \"columns\": [";
    for (std::size_t i = 0; i < t.columns.size(); ++i)
        out << (i ? "," : "") << "\n    " << json_string(t.columns[i]);
    out << (t.columns.empty() ? "]" : "\n  ]") << ",\n  \"header\": {";
    std::size_t k = 0;
    for (const auto& kv : t.header) out << (k++ ? "," : "") << "\n    " << json_string(kv.first) << ": " << json_string(kv.second);
    out << (t.header.empty() ? "}" : "\n  }") << ",\n  \"rows\": [";
    for (std::size_t r = 0; r < t.rows.size(); ++r) {
        out << (r ? "," : "") << "\n    [";
        for (std::size_t i = 0; i < t.rows[r].size(); ++i)
            out << (i ? "," : "") << "\n      " << json_number(t.rows[r][i]);
        out << (t.rows[r].empty() ? "]" : "\n    ]");
    }
    out << (t.rows.empty() ? "]" : "\n  ]") << "\n}\n";
}

TraceFile read_trace_csv(std::istream& in) {  // harness.cpp:163-199: same parse rules and errors
    TraceFile t;
    std::string line;
    bool have_columns = false;
    std::size_t line_no = 0;
    while (std::getline(in, line)) {
        ++line_no;
        if (line.empty()) continue;
        if (line[0] == '#') {
            const std::size_t start = line.find_first_not_of(" \t", 1);
            if (start == std::string::npos) continue;
            const std::size_t eq = line.find('=', start);
            if (eq == std::string::npos) continue;
            t.header[line.substr(start, eq - start)] = line.substr(eq + 1);
            continue;
        }
        std::vector<std::string> cells;
        std::size_t b = 0;
        while (true) {
            const std::size_t c = line.find(',', b);
            cells.push_back(line.substr(b, c == std::string::npos ? std::string::npos : c - b));
            if (c == std::string::npos) break;
            b = c + 1;
        }
        if (!have_columns) {
            t.columns = cells;
            have_columns = true;
            continue;
        }
        std::vector<double> row;
        for (const std::string& cell : cells) {
            double v = 0.0;
            auto res = std::from_chars(cell.data(), cell.data() + cell.size(), v);
            if (res.ec != std::errc{} || res.ptr != cell.data() + cell.size())
                throw ParseError("bad numeric cell '" + cell + "'", line_no);
            row.push_back(v);
        }
        if (row.size() != t.columns.size()) throw ParseError("row width does not match the column header", line_no);
        t.rows.push_back(std::move(row));
    }
    if (!have_columns) throw ParseError("trace has no column header");
    return t;
}

TraceFile read_trace_json(std::istream& in) {
    JsonIn j{std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>())};
    TraceFile t;
    bool h = false, c = false, r = false;
    j.expect('{');
    if (!j.peek('}'))
        do {
            const std::string key = j.str();
            j.expect(':');
            if (key == "header") {
                h = true;
                j.expect('{');
                if (!j.peek('}'))
                    do {
                        std::string k2 = j.str();
                        j.expect(':');
                        t.header[k2] = j.str();
                    } while (j.peek(',') && (++j.p, true));
                j.expect('}');
            } else if (key == "columns") {
                c = true;
                j.expect('[');
                if (!j.peek(']'))
                    do t.columns.push_back(j.str());
                    while (j.peek(',') && (++j.p, true));
                j.expect(']');
            } else if (key == "rows") {
                r = true;
                j.expect('[');
                if (!j.peek(']'))
                    do {
                        std::vector<double> row;
                        j.expect('[');
                        if (!j.peek(']'))
                            do row.push_back(j.num());
                            while (j.peek(',') && (++j.p, true));
                        j.expect(']');
                        t.rows.push_back(std::move(row));
                    } while (j.peek(',') && (++j.p, true));
                j.expect(']');
            } else {
                j.skip_value();
            }
        } while (j.peek(',') && (++j.p, true));
    j.expect('}');
    if (!h || !c || !r) throw ParseError("trace json: missing header, columns or rows");
    return t;
}

ExperimentResult run_experiment(const ExperimentSpec& spec) {  // harness.cpp:241-345, solves on the device
    if (spec.repetitions < 1) throw ShapeError("repetitions must be at least 1");
    if (spec.input_path.has_value() == spec.synthetic.has_value())
        throw ShapeError("specify exactly one input source (file or synthetic)");
    if (spec.out_dir.empty()) throw ShapeError("output directory required");
    SparseTensor x;
    if (spec.input_path) {
        x = load_tns_file(*spec.input_path, spec.dims_override);
    } else {
        const SyntheticSpec& syn = *spec.synthetic;
        x = gen_synthetic(syn.dims, syn.nnz, syn.seed);
    }
    std::filesystem::create_directories(spec.out_dir);
    std::vector<std::pair<const char*, bool>> chosen;  // (name, is_hooi)
    if (spec.solver != SolverChoice::kHooi) chosen.push_back({"hoqri", false});
    if (spec.solver != SolverChoice::kHoqri) chosen.push_back({"hooi", true});
    ExperimentResult result;
    std::string sections;
    for (const auto& [name, is_hooi] : chosen) {
        std::string runs;
        double mean_total = 0.0;
        for (std::size_t rep = 0; rep < spec.repetitions; ++rep) {  // repetitions share the GPU: in order
            SolverConfig cfg = spec.config;
            cfg.seed = spec.config.seed + rep;
            SolveResult res = is_hooi ? hooi(x, cfg) : hoqri(x, cfg);
            TraceFile t = make_trace_file(name, cfg, x, res.trace);
            const std::string base =
                (std::filesystem::path(spec.out_dir) / (std::string(name) + "_rep" + std::to_string(rep))).string();
            {
                std::ofstream csv(base + ".trace.csv");
                write_trace_csv(csv, t);
                std::ofstream js(base + ".trace.json");
                write_trace_json(js, t);
            }
            const std::size_t sweeps = res.trace.sweeps.size();
            double mean_sweep = 0.0, fobj = 0.0, ffit = 0.0;
            if (sweeps) {
                mean_sweep = res.trace.sweeps.back().elapsed_s / static_cast<double>(sweeps);
                fobj = res.trace.sweeps.back().objective;
                ffit = res.trace.sweeps.back().fit;
            }
            mean_total += mean_sweep;
            result.trace_paths.push_back(base + ".trace.csv");
            runs += std::string(rep ? "," : "") + "\n      {\n        \"final_fit\": " + json_number(ffit) +
                    ",\n        \"final_objective\": " + json_number(fobj) + ",\n        \"mean_sweep_s\": " +
                    json_number(mean_sweep) + ",\n        \"rep\": " + std::to_string(rep) +
                    ",\n        \"sweeps\": " + std::to_string(sweeps) + ",\n        \"trace\": " +
                    json_string(base + ".trace.csv") + "\n      }";
        }
        sections += ",\n  " + json_string(name) + ": {\n    \"mean_sweep_s\": " +
                    json_number(mean_total / static_cast<double>(spec.repetitions)) + ",\n    \"runs\": [" + runs +
                    "\n    ]\n  }";
    }
    auto arr = [](const std::vector<std::size_t>& v) {
        std::string s2 = "[";
        for (std::size_t i2 = 0; i2 < v.size(); ++i2) s2 += (i2 ? ", " : "") + std::to_string(v[i2]);
        return s2 + "]";
    };
    const std::string sp = (std::filesystem::path(spec.out_dir) / "summary.json").string();
    std::ofstream out(sp);
    // keys in sorted order like the reference's json dump: dims, hooi, hoqri, nnz, ranks, repetitions, tool_version
    std::string hooi_sec, hoqri_sec;
    {
        const std::size_t cut = sections.find(",\n  \"hooi\"");
        hoqri_sec = cut == std::string::npos ? sections : sections.substr(0, cut);
        hooi_sec = cut == std::string::npos ? std::string() : sections.substr(cut);
        if (spec.solver == SolverChoice::kHooi) {
            hooi_sec = sections;
            hoqri_sec.clear();
        }
    }
    out << "{\n  \"dims\": " << arr(x.dims()) << hooi_sec << hoqri_sec << ",\n  \"nnz\": " << x.nnz()
        << ",\n  \"ranks\": " << arr(spec.config.ranks) << ",\n  \"repetitions\": " << spec.repetitions
        << ",\n  \"tool_version\": " << json_string(kToolVersion) << "\n}\n";
    result.summary_path = sp;
    return result;
}

BenchStats bench_kernel(const SparseTensor& x, const FactorSet& u, std::size_t mode, KernelVariant variant,
                        std::size_t repetitions) {  // harness.cpp:350-381, device-timed
    (void)variant;  // both variants run the same device kernel (kernels.hpp:52-60)
    if (repetitions < 1) throw ShapeError("repetitions must be at least 1");
    if (mode >= x.order()) throw RangeError("ttmctc: mode out of range");
    check_factors(x, u);
    std::vector<uint64_t> ranks;
    for (const Matrix& m : u.factors) ranks.push_back(m.cols);
    std::vector<double> times(repetitions);
    uint64_t scratch[2] = {0, 0};
    auto p = ptrs(u);
    check(hq_bench_ttmctc(x.device(), p.data(), ranks.data(), static_cast<int>(mode), repetitions, times.data(),
                          scratch));
    BenchStats st;
    st.repetitions = repetitions;
    std::sort(times.begin(), times.end());
    st.min_s = times.front();
    st.max_s = times.back();
    const std::size_t mid = times.size() / 2;
    st.median_s = times.size() % 2 ? times[mid] : 0.5 * (times[mid - 1] + times[mid]);
    st.peak_slots = (scratch[0] + 7) / 8;
    st.largest_alloc_slots = (scratch[1] + 7) / 8;
    return st;
}

}  // namespace tucker
