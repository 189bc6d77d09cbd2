// tucker_shim.cpp — the reference's `tucker::` API over the engine's C-ABI.
//
// Every numeric entry point forwards to libhoqri_b200.so (include/hoqri_b200.h)
// and rethrows the C-ABI status as the reference's exception type with the
// same payload (errors.hpp taxonomy; DegenerateStateError keeps the 1-based
// mode).  Only K x K bookkeeping (matmul helpers on desk-scale matrices,
// unfold_core's index shuffle) runs on the host, as in the reference.
#include <algorithm>
#include <cmath>
#include <fstream>
#include <istream>
#include <ostream>
#include <sstream>

#include "hoqri_b200.h"
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
    // sparse_tensor.cpp:136-215 (text parse on the host, build on the device)
    std::vector<std::size_t> header;
    std::vector<index_t> coords;
    std::vector<double> values;
    std::vector<std::size_t> seen;
    std::size_t order = dims_override ? dims_override->size() : 0;
    std::string line;
    std::size_t line_no = 0;
    bool content = false;
    auto parse_u = [&](const std::string& t) -> uint64_t {
        if (t.empty() || !std::all_of(t.begin(), t.end(), ::isdigit))
            throw ParseError("expected an integer index, got '" + t + "'", line_no);
        return std::stoull(t);
    };
    while (std::getline(in, line)) {
        ++line_no;
        if (line.empty() || line[0] == '#' ||
            std::all_of(line.begin(), line.end(), [](unsigned char c) { return std::isspace(c); }))
            continue;
        std::istringstream ls(line);
        std::vector<std::string> tok;
        if (!content && line.rfind("dims:", 0) == 0) {
            content = true;
            std::istringstream hs(line.substr(5));
            for (std::string t; hs >> t;) tok.push_back(t);
            if (tok.empty()) throw ParseError("empty dims header", line_no);
            for (auto& t : tok) {
                uint64_t d = parse_u(t);
                if (d == 0) throw RangeError("line " + std::to_string(line_no) + ": extent must be at least 1");
                header.push_back(d);
            }
            if (order && header.size() != order) throw ParseError("dims header order does not match override", line_no);
            if (!order) order = header.size();
            seen.assign(order, 0);
            continue;
        }
        content = true;
        for (std::string t; ls >> t;) tok.push_back(t);
        if (!order) {
            if (tok.size() < 2) throw ParseError("entry line needs at least one index and a value", line_no);
            order = tok.size() - 1;
            seen.assign(order, 0);
        }
        if (tok.size() != order + 1)
            throw ParseError("expected " + std::to_string(order + 1) + " fields, got " + std::to_string(tok.size()),
                             line_no);
        if (seen.empty()) seen.assign(order, 0);
        for (std::size_t m = 0; m < order; ++m) {
            uint64_t idx = parse_u(tok[m]);
            if (idx < 1)
                throw RangeError("line " + std::to_string(line_no) + ": indices are 1-based, got " + std::to_string(idx));
            if (idx - 1 > 0xFFFFFFFFull)
                throw RangeError("line " + std::to_string(line_no) + ": index " + std::to_string(idx) + " too large");
            coords.push_back(static_cast<index_t>(idx - 1));
            seen[m] = std::max<std::size_t>(seen[m], idx);
        }
        char* end = nullptr;
        double v = std::strtod(tok[order].c_str(), &end);
        if (end != tok[order].c_str() + tok[order].size())
            throw ParseError("expected a real value, got '" + tok[order] + "'", line_no);
        if (!std::isfinite(v)) throw ValueError("line " + std::to_string(line_no) + ": non-finite value");
        values.push_back(v);
    }
    std::vector<std::size_t> dims;
    if (dims_override)
        dims = *dims_override;
    else if (!header.empty())
        dims = header;
    else if (!seen.empty())
        dims = seen;
    else
        throw ParseError("no entries and no dims header; cannot infer tensor order");
    for (auto& d : dims)
        if (d == 0) d = 1;
    return SparseTensor(std::move(dims), std::move(coords), std::move(values));
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

FactorSet init_factors(const SparseTensor& x, const SolverConfig& config) {
    check_ranks(x, config.ranks);
    if (config.init != InitMode::kRandom)
        throw CapacityError("HOSVD initialisation is desk-scale only and outside the B200 engine; use random init");
    return random_factors(x.dims(), config.ranks, config.seed);
}

static SolveResult solve_impl(const SparseTensor& x, const SolverConfig& config, const FactorSet* start) {
    check_ranks(x, config.ranks);
    if (config.max_sweeps < 1) throw ShapeError("max_sweeps must be at least 1");
    if (config.tol_fit_change < 0.0) throw ShapeError("tolerance must be nonnegative");
    if (!start && config.init != InitMode::kRandom)
        throw CapacityError("HOSVD initialisation is desk-scale only and outside the B200 engine; use random init");
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

SolveResult hoqri_from(const SparseTensor& x, const SolverConfig& config, const FactorSet& start) {
    return solve_impl(x, config, &start);
}

double fit_error(const SparseTensor& x, const TuckerModel& model) {
    if (model.factors.order() != x.order()) throw ShapeError("fit_error: model order does not match the tensor");
    double out = 0.0;
    check(hq_fit_error(model.data_norm_sq, model.core.data.size(), model.core.data.data(), &out));
    return out;
}

}  // namespace tucker
