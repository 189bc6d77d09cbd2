// tucker_b200.hpp — the reference's `tucker::` hot-path API, served by the
// B200 engine (libtucker_b200.so over libhoqri_b200.so).
//
// Callers of the reference library (/root/reference/proj) include
// "tucker/<name>.hpp" and link `tucker`; with this tree on the include path
// and libtucker_b200.so on the link line they get the same names, types,
// argument meanings and exceptions, with every numeric step on the GPU.
// Each declaration cites the reference declaration it stands in for
// (paths relative to /root/reference/proj/include/tucker/).
//
// Scope: the HOQRI hot path plus its section 8(f)
// neighbours: gradient diagnostics, .tns ingestion, the harness (harness.hpp)
// and the desk-scale HOSVD initialisation / HOOI, all on the device.
#pragma once

#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

struct hq_tensor;

namespace tucker {

// ---------------------------------------------------------- errors.hpp ---
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : Error {
    ParseError(const std::string& what, std::size_t line = 0)
        : Error(line ? "line " + std::to_string(line) + ": " + what : what), line_number(line) {}
    std::size_t line_number;
};
struct RangeError : Error { using Error::Error; };
struct ValueError : Error { using Error::Error; };
struct ShapeError : Error { using Error::Error; };
struct CapacityError : Error { using Error::Error; };
struct ContractError : Error { using Error::Error; };
struct DiagnosticError : Error { using Error::Error; };
struct InfeasibleError : Error { using Error::Error; };
struct DegenerateStateError : Error {
    explicit DegenerateStateError(std::size_t mode_1based)
        : Error("degenerate state: TTMcTC output is identically zero for mode " +
                std::to_string(mode_1based)),
          mode(mode_1based) {}
    std::size_t mode;
};
// CUDA / NCCL failures surface as this (not part of the reference taxonomy)
struct DeviceError : Error { using Error::Error; };

// ------------------------------------------------------ dense_core.hpp ---
struct Matrix {  // dense_core.hpp:10-22, row-major
    std::size_t rows = 0, cols = 0;
    std::vector<double> data;
    Matrix() = default;
    Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
    double& operator()(std::size_t i, std::size_t j) { return data[i * cols + j]; }
    double operator()(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
    double* row(std::size_t i) { return data.data() + i * cols; }
    const double* row(std::size_t i) const { return data.data() + i * cols; }
};

Matrix identity(std::size_t n);
Matrix transpose(const Matrix& a);
Matrix matmul(const Matrix& a, const Matrix& b);
Matrix matmul_tn(const Matrix& a, const Matrix& b);
Matrix matmul_nt(const Matrix& a, const Matrix& b);
double frob_norm_sq(const Matrix& a);
double max_abs(const Matrix& a);
double max_abs_diff(const Matrix& a, const Matrix& b);

struct CoreTensor {  // dense_core.hpp:33-43, last mode fastest
    std::vector<std::size_t> ranks;
    std::vector<double> data;
    CoreTensor() = default;
    explicit CoreTensor(std::vector<std::size_t> r);
    std::size_t order() const { return ranks.size(); }
    std::size_t size() const { return data.size(); }
};
double norm_sq(const CoreTensor& g);

struct FactorSet {  // dense_core.hpp:45-54
    std::vector<Matrix> factors;
    std::size_t order() const { return factors.size(); }
    double orthonormality_defect() const;
};

Matrix qr_orthonormal(const Matrix& a);                          // dense_core.hpp:60 (device)
Matrix unfold_core(const CoreTensor& g, std::size_t mode);       // dense_core.hpp:72
std::vector<std::size_t> unfold_col_strides(const std::vector<std::size_t>& dims,
                                            std::size_t mode);   // dense_core.hpp:77-78
double nuclear_norm(const Matrix& m);                             // dense_core.hpp:67 (device eigen-solve)
std::vector<double> gram_eigvals_desc(const Matrix& m);          // dense_core.hpp:82 (device eigen-solve)
struct EigResult {                                               // dense_core.hpp:86-89
    std::vector<double> values;
    Matrix vectors;
};
EigResult jacobi_eig_sym(Matrix m);  // dense_core.hpp:90: same pairs (device syevd; vector signs may differ)

// -------------------------------------------------- sparse_tensor.hpp ----
using index_t = std::uint32_t;

// sparse_tensor.hpp:20-66.  The tensor lives on the GPU (layout built there);
// host views of the sorted entries and buckets are materialised on first use.
class SparseTensor {
public:
    struct ModeBuckets {
        std::vector<std::size_t> offsets;
        std::vector<std::size_t> entries;
        std::size_t bucket_size(std::size_t i) const { return offsets[i + 1] - offsets[i]; }
    };

    SparseTensor() = default;
    SparseTensor(std::vector<std::size_t> dims, std::vector<index_t> coords,
                 std::vector<double> values);

    std::size_t order() const { return dims_.size(); }
    const std::vector<std::size_t>& dims() const { return dims_; }
    std::size_t nnz() const { return nnz_; }
    double value(std::size_t e) const { return values()[e]; }
    const std::vector<double>& values() const;
    index_t coord(std::size_t e, std::size_t mode) const { return coords()[e * dims_.size() + mode]; }
    const index_t* coord_row(std::size_t e) const { return coords().data() + e * dims_.size(); }
    void build_mode_buckets() {}
    bool buckets_built() const { return !dims_.empty(); }
    const ModeBuckets& mode_bucket(std::size_t mode) const;

    hq_tensor* device() const { return dev_.get(); }

private:
    const std::vector<index_t>& coords() const;
    struct Host;
    std::vector<std::size_t> dims_;
    std::size_t nnz_ = 0;
    std::shared_ptr<hq_tensor> dev_;
    std::shared_ptr<Host> host_;
};

double norm_sq(const SparseTensor& x);  // sparse_tensor.hpp:69
SparseTensor load_tns(std::istream& in, std::optional<std::vector<std::size_t>> dims_override = {});
SparseTensor load_tns_file(const std::string& path,
                           std::optional<std::vector<std::size_t>> dims_override = {});
void write_tns(std::ostream& out, const SparseTensor& x);
void write_tns_file(const std::string& path, const SparseTensor& x);

// ---------------------------------------------------------- kernels.hpp ---
struct WorkspaceMeter {  // kernels.hpp:15-36: here it meters transient device scratch
    std::size_t current_bytes = 0, peak_bytes = 0, largest_single_bytes = 0;
    void acquire(std::size_t bytes) {
        current_bytes += bytes;
        if (current_bytes > peak_bytes) peak_bytes = current_bytes;
        if (bytes > largest_single_bytes) largest_single_bytes = bytes;
    }
    void release(std::size_t bytes) { current_bytes -= bytes < current_bytes ? bytes : current_bytes; }
    void reset() { *this = WorkspaceMeter{}; }
    std::size_t peak_slots() const { return (peak_bytes + 7) / 8; }
    std::size_t largest_single_slots() const { return (largest_single_bytes + 7) / 8; }
};
struct KernelWorkspace {  // kernels.hpp:38-41
    std::vector<double> column;
    std::vector<std::uint32_t> stamp;
    std::vector<std::size_t> touched;
    WorkspaceMeter meter;
};

CoreTensor ttmc_core(const SparseTensor& x, const FactorSet& u);                    // kernels.hpp:46
Matrix ttmctc_elementwise(const SparseTensor& x, const FactorSet& u, std::size_t mode,
                          const CoreTensor* precomputed_core = nullptr,
                          KernelWorkspace* ws = nullptr);                           // kernels.hpp:52-54
Matrix ttmctc_matrix(const SparseTensor& x, const FactorSet& u, std::size_t mode,
                     KernelWorkspace* ws = nullptr);                                // kernels.hpp:59-60
constexpr std::size_t kDefaultCapacityCap = std::size_t{1} << 31;

// ---------------------------------------------------------- manifold.hpp --
struct GradientReport {  // manifold.hpp:14-19
    std::vector<double> per_mode_norm_sq;
    double total_norm_sq = 0.0;
    std::vector<std::vector<double>> sigma;
    std::vector<std::vector<double>> lambda;
};
Matrix project_tangent(const Matrix& u, const Matrix& a);                  // manifold.hpp:23
Matrix riemannian_grad(const Matrix& u, const Matrix& a, const Matrix& gn);  // manifold.hpp:27
double grad_norm_sq(const Matrix& a, const Matrix& gn);                    // manifold.hpp:31
double subspace_distance(const Matrix& u, const Matrix& v);  // manifold.hpp:34-36 (device)
struct InterlacingResult {  // manifold.hpp:38-42
    std::vector<double> sigma, lambda;
    double min_margin = 0.0;
};
InterlacingResult interlacing_check(const Matrix& a, const Matrix& gn);     // manifold.hpp:46

// ----------------------------------------------------------- solvers.hpp --
enum class InitMode { kRandom, kHosvd };
enum class KernelVariant { kElementwise, kMatrix };

struct SolverConfig {  // solvers.hpp:17-28
    std::vector<std::size_t> ranks;
    std::size_t max_sweeps = 100;
    double tol_fit_change = 1e-12;
    std::uint64_t seed = 0;
    InitMode init = InitMode::kRandom;
    bool trace_gradients = false;
    KernelVariant kernel = KernelVariant::kElementwise;
    double tol_grad = 0.0;
    std::size_t capacity_cap = kDefaultCapacityCap;
};

struct TuckerModel {
    FactorSet factors;
    CoreTensor core;
    double data_norm_sq = 0.0;
};

struct ModeUpdateRecord {
    std::size_t sweep = 0, mode = 0;
    double f_before = 0.0, f_after = 0.0, grad_norm_sq = 0.0;
    std::vector<double> sigma, lambda;
    double elapsed_s = 0.0;
};

struct SweepRecord {
    std::size_t sweep = 0;
    double elapsed_s = 0.0, objective = 0.0, fit = 0.0, total_grad_norm_sq = 0.0;
    std::vector<double> grad_norm_sq, drift;
};

struct IterationTrace {
    double data_norm_sq = 0.0, initial_objective = 0.0;
    std::vector<SweepRecord> sweeps;
    std::vector<ModeUpdateRecord> updates;
};

struct SolveResult {
    TuckerModel model;
    IterationTrace trace;
};

FactorSet random_factors(const std::vector<std::size_t>& dims, const std::vector<std::size_t>& ranks,
                         std::uint64_t seed);                    // solvers.hpp:72-73
FactorSet init_factors(const SparseTensor& x, const SolverConfig& config);  // solvers.hpp:77 (random or HOSVD)
SolveResult hooi(const SparseTensor& x, const SolverConfig& config);         // solvers.hpp:82-83 (device)
Matrix svd_leading(const Matrix& y, std::size_t k);                          // dense_core.hpp:64 (device)
Matrix densify_unfold(const SparseTensor& x, std::size_t mode,
                      std::size_t capacity_cap = kDefaultCapacityCap);       // kernels.hpp:70-71 (device)
Matrix ttmc_unfold_dense(const SparseTensor& x, const FactorSet& u, std::size_t mode,
                         std::size_t capacity_cap = kDefaultCapacityCap);    // kernels.hpp:66-67 (device)
SolveResult hoqri(const SparseTensor& x, const SolverConfig& config);        // solvers.hpp:80
// B200 extension: start from caller-supplied factors (init_factors result)
SolveResult hoqri_from(const SparseTensor& x, const SolverConfig& config, const FactorSet& start);
double fit_error(const SparseTensor& x, const TuckerModel& model);           // solvers.hpp:87
GradientReport gradient_report(const SparseTensor& x, const FactorSet& u);   // solvers.hpp:91 (device TTMcTC)
struct DescentCheck {                                                       // solvers.hpp:93-98
    bool ok = true;
    std::size_t checked = 0, violations = 0;
    double worst_violation = 0.0;
};
DescentCheck check_descent_inequality(const IterationTrace& trace, double data_norm_sq);  // solvers.hpp:102-103

}  // namespace tucker
