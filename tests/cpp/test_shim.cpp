// C++ checks of the tucker:: drop-in (libtucker_b200.so over the CUDA engine),
// written the way the reference's own tests are (proj/tests/*.cpp): same
// calls, same known answers, same exception types.  Needs a GPU.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <string>

#include <filesystem>
#include <fstream>

#include "tucker/harness.hpp"
#include "tucker/kernels.hpp"
#include "tucker/solvers.hpp"
#include "tucker/sparse_tensor.hpp"

using namespace tucker;

static int failures = 0;
#define CHECK(c)                                                               \
    do {                                                                       \
        if (!(c)) {                                                            \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);           \
            ++failures;                                                        \
        }                                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                               \
    do {                                                                       \
        bool thrown_ = false;                                                     \
        try {                                                                  \
            (void)(expr);                                                      \
        } catch (const T&) {                                                   \
            thrown_ = true;                                                     \
        } catch (...) {                                                        \
        }                                                                      \
        if (!thrown_) {                                                         \
            std::printf("FAIL %s:%d: %s did not throw %s\n", __FILE__, __LINE__, #expr, #T); \
            ++failures;                                                        \
        }                                                                      \
    } while (0)

static FactorSet identity_factors(const std::vector<std::size_t>& dims) {
    FactorSet u;
    for (std::size_t d : dims) u.factors.push_back(identity(d));
    return u;
}

int main() {
    // sparse_tensor_test.cpp:24-29 — duplicates summed; lexicographic order restored
    {
        std::istringstream in("1 1 1 1.0\n1 1 1 2.0\n2 1 1 0.5\n");
        SparseTensor x = load_tns(in);
        CHECK(x.nnz() == 2);
        CHECK(std::fabs(x.value(0) - 3.0) < 1e-15);
        CHECK(x.coord(1, 0) == 1);
        const auto& b = x.mode_bucket(0);
        CHECK(b.offsets.size() == 3 && b.offsets[1] == 1 && b.entries[1] == 1);
        CHECK(std::fabs(norm_sq(x) - 9.25) < 1e-15);
    }
    // kernels_test.cpp:34-45 indicator core = 2
    {
        SparseTensor x({2, 2, 2}, {0, 0, 0}, {2.0});
        FactorSet u;
        for (int n = 0; n < 3; ++n) {
            Matrix e0(2, 1);
            e0(0, 0) = 1.0;
            u.factors.push_back(e0);
        }
        CoreTensor g = ttmc_core(x, u);
        CHECK(g.size() == 1 && std::fabs(g.data[0] - 2.0) < 1e-15);
        // kernels_test.cpp:64-73 identity factors: A(0,0) = 4, the rest exactly 0
        Matrix a = ttmctc_elementwise(x, identity_factors(x.dims()), 0);
        CHECK(std::fabs(a(0, 0) - 4.0) < 1e-14);
        double off = 0.0;
        for (std::size_t i = 1; i < a.data.size(); ++i) off += std::fabs(a.data[i]);
        CHECK(off == 0.0);
    }
    // kernels_test.cpp:100-116 rank-1 matrix variant
    {
        SparseTensor x({2, 2, 2}, {1, 0, 1}, {3.0});
        FactorSet u;
        for (int n = 0; n < 3; ++n) {
            Matrix c(2, 1);
            c(0, 0) = 0.6;
            c(1, 0) = 0.8;
            u.factors.push_back(c);
        }
        double y1 = 3.0 * 0.6 * 0.8;
        Matrix a = ttmctc_matrix(x, u, 0);
        CHECK(std::fabs(a(0, 0)) < 1e-15);
        CHECK(std::fabs(a(1, 0) - y1 * (y1 * 0.8)) < 1e-13 * y1 * y1);
    }
    // dense_core_test.cpp:50-57 QR sign convention
    {
        Matrix a(2, 1);
        a(0, 0) = 3.0;
        a(1, 0) = 4.0;
        Matrix q = qr_orthonormal(a);
        CHECK(std::fabs(q(0, 0) - 0.6) < 1e-14 && std::fabs(q(1, 0) - 0.8) < 1e-14);
        CHECK_THROWS_AS(qr_orthonormal(Matrix(2, 3)), ShapeError);
    }
    // kernels_test.cpp:273-281 shape / range errors
    {
        SparseTensor x({4, 4, 4}, {0, 1, 2, 3, 3, 3}, {1.0, 2.0});
        FactorSet bad = random_factors({5, 4, 4}, {2, 2, 2}, 1);
        CHECK_THROWS_AS(ttmctc_elementwise(x, bad, 0), ShapeError);
        CHECK_THROWS_AS(ttmc_core(x, bad), ShapeError);
        FactorSet ok = random_factors(x.dims(), {2, 2, 2}, 1);
        CHECK_THROWS_AS(ttmctc_elementwise(x, ok, 3), RangeError);
        CHECK_THROWS_AS(SparseTensor({2, 2}, {0, 2}, {1.0}), RangeError);
        CHECK_THROWS_AS(SparseTensor({2, 2}, {0, 1}, {NAN}), ValueError);
    }
    // solvers_test.cpp:312-323 degenerate zero state -> mode 1
    {
        SparseTensor x({3, 3, 3}, {1, 1, 1}, {0.0});
        SolverConfig cfg;
        cfg.ranks = {1, 1, 1};
        cfg.seed = 1;
        bool caught = false;
        try {
            hoqri(x, cfg);
        } catch (const DegenerateStateError& e) {
            caught = (e.mode == 1);
        }
        CHECK(caught);
    }
    // solvers_test.cpp:119-141 / 275-293 — monotone objective, fit identity, fresh core
    {
        std::vector<std::size_t> dims{50, 50, 50};
        std::vector<index_t> coords;
        std::vector<double> vals;
        uint64_t s = 88172645463325252ull;
        for (int e = 0; e < 500; ++e) {
            for (int m = 0; m < 3; ++m) {
                s ^= s << 13; s ^= s >> 7; s ^= s << 17;
                coords.push_back(static_cast<index_t>(s % 50));
            }
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            vals.push_back((double)(s >> 11) * 0x1.0p-53 - 0.5);
        }
        SparseTensor x(dims, coords, vals);
        SolverConfig cfg;
        cfg.ranks = {5, 5, 5};
        cfg.max_sweeps = 60;
        cfg.tol_fit_change = 0.0;
        cfg.seed = 8;
        SolveResult r = hoqri(x, cfg);
        CHECK(r.trace.sweeps.size() == 60);
        double prev = r.trace.initial_objective;
        for (const SweepRecord& sw : r.trace.sweeps) {
            CHECK(sw.objective >= prev - 1e-9 * std::max(prev, 1.0));
            CHECK(std::fabs(sw.fit - (r.trace.data_norm_sq - sw.objective)) <= 1e-8 * r.trace.data_norm_sq);
            prev = sw.objective;
        }
        CHECK(r.model.factors.orthonormality_defect() <= 1e-10);
        CoreTensor fresh = ttmc_core(x, r.model.factors);
        double worst = 0.0;
        for (std::size_t i = 0; i < fresh.size(); ++i) worst = std::max(worst, std::fabs(fresh.data[i] - r.model.core.data[i]));
        CHECK(worst <= 1e-10);
        CHECK(fit_error(x, r.model) >= 0.0);
        // bitwise determinism (solvers_test.cpp:295-310)
        SolveResult r2 = hoqri(x, cfg);
        for (std::size_t i = 0; i < r.trace.sweeps.size(); ++i) CHECK(r.trace.sweeps[i].objective == r2.trace.sweeps[i].objective);
    }
    // harness.hpp surface: gen_synthetic, run_experiment traces, bench_kernel (device-timed)
    {
        SparseTensor x = gen_synthetic({20, 18, 16}, 200, 41);
        CHECK(x.nnz() == 200);
        const std::string dir = (std::filesystem::temp_directory_path() / "hq_shim_harness").string();
        std::filesystem::remove_all(dir);
        ExperimentSpec spec;
        spec.synthetic = SyntheticSpec{{20, 18, 16}, 200, 41};
        spec.config.ranks = {3, 3, 3};
        spec.config.max_sweeps = 6;
        spec.config.tol_fit_change = 0.0;
        spec.config.seed = 5;
        spec.repetitions = 2;
        spec.out_dir = dir;
        ExperimentResult er = run_experiment(spec);
        CHECK(er.trace_paths.size() == 2);
        CHECK(std::filesystem::exists(er.summary_path));
        std::ifstream fc(er.trace_paths[0]);
        TraceFile tc = read_trace_csv(fc);
        std::ifstream fj(er.trace_paths[0].substr(0, er.trace_paths[0].size() - 4) + ".json");
        TraceFile tj = read_trace_json(fj);
        CHECK(tc.columns.size() == 8 && tc.rows.size() == 6);
        CHECK(tj.columns == tc.columns && tj.header == tc.header && tj.rows.size() == tc.rows.size());
        for (std::size_t i = 0; i < tc.rows.size(); ++i) CHECK(tj.rows[i] == tc.rows[i]);
        CHECK(tc.header["solver"] == "hoqri" && tc.header["seed"] == "5" && tc.header["dims"] == "20,18,16");
        for (std::size_t i = 1; i < tc.rows.size(); ++i) CHECK(tc.rows[i][1] >= tc.rows[i - 1][1]);  // elapsed
        spec.solver = SolverChoice::kBoth;
        spec.repetitions = 1;
        ExperimentResult eb = run_experiment(spec);
        CHECK(eb.trace_paths.size() == 2);
        CHECK(eb.trace_paths[1].find("hooi_rep0.trace.csv") != std::string::npos);
        // HOOI and HOSVD init on the device (solvers_test.cpp:71-79, 158-170)
        SolverConfig hc;
        hc.ranks = {3, 3, 3};
        hc.max_sweeps = 10;
        hc.tol_fit_change = 0.0;
        hc.init = InitMode::kHosvd;
        SolveResult ra = hoqri(x, hc), rb = hooi(x, hc);
        CHECK(rb.trace.sweeps.size() == 10);
        double prev = rb.trace.initial_objective;
        for (const SweepRecord& sw : rb.trace.sweeps) {
            CHECK(sw.objective >= prev - 1e-9 * std::max(prev, 1.0));
            prev = sw.objective;
        }
        CHECK(rb.model.factors.orthonormality_defect() <= 1e-10);
        FactorSet hs = init_factors(x, hc);
        CHECK(hs.factors.size() == 3 && hs.orthonormality_defect() <= 1e-10);
        Matrix yd = densify_unfold(x, 0);
        CHECK(yd.rows == 20 && yd.cols == 18 * 16);
        Matrix ul = svd_leading(yd, 3);
        CHECK(ul.rows == 20 && ul.cols == 3);
        hc.capacity_cap = 100;
        CHECK_THROWS_AS(init_factors(x, hc), CapacityError);
        FactorSet u = random_factors(x.dims(), {3, 3, 3}, 7);
        BenchStats bs = bench_kernel(x, u, 1, KernelVariant::kElementwise, 5);
        CHECK(bs.repetitions == 5 && bs.min_s > 0.0 && bs.min_s <= bs.median_s && bs.median_s <= bs.max_s);
        CHECK(bs.peak_slots >= 18 * 3 && bs.largest_alloc_slots <= bs.peak_slots);
        std::istringstream bad("a,b\n1,2\n1,x\n");
        CHECK_THROWS_AS(read_trace_csv(bad), ParseError);
        std::filesystem::remove_all(dir);
    }
    // gradient tracing (solvers.cpp:126-150): every update recorded, interlacing holds
    {
        SparseTensor x = gen_synthetic({20, 18, 16}, 200, 41);
        SolverConfig cfg;
        cfg.ranks = {3, 3, 3};
        cfg.max_sweeps = 5;
        cfg.tol_fit_change = 0.0;
        cfg.seed = 5;
        cfg.trace_gradients = true;
        SolveResult r = hoqri(x, cfg);
        CHECK(r.trace.updates.size() == 15);
        for (const ModeUpdateRecord& up : r.trace.updates) {
            CHECK(up.grad_norm_sq >= 0.0 && up.sigma.size() == 3 && up.lambda.size() == 3);
            for (std::size_t k = 0; k < 3; ++k) CHECK(up.sigma[k] - up.lambda[k] >= -1e-9 * std::max(1.0, up.sigma[0]));
        }
        double tot = 0.0;
        for (double g : r.trace.sweeps[0].grad_norm_sq) tot += g;
        CHECK(std::fabs(tot - r.trace.sweeps[0].total_grad_norm_sq) <= 1e-12 * std::max(1.0, tot));
    }
    if (failures) {
        std::printf("%d check(s) failed\n", failures);
        return 1;
    }
    std::printf("test_shim: all checks passed\n");
    return 0;
}
