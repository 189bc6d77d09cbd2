// hq_solver.cu — the device-resident HOQRI driver and the C-ABI.
//
// Mirrors tucker::solve for HOQRI (proj/src/solvers.cpp:50-178): initial core
// (solvers.cpp:66), then per sweep and mode n: TTMcTC (solvers.cpp:90-91),
// degeneracy test (:124), QR (:139-140), drift (:141), core update
// (:143-144); objective, fit and the stop rule per sweep (:153-168); the
// orthonormality-defect check at the end (:171-172).
//
// B200 shape of one mode update (all device, no host round trip):
//   gt      G_(n)^T from the core                                   (tiny)
//   pass    one sparse pass: Y_i, a_i = Y_i G_(n)^T -> A, and the partials of
//           W = A^T A, M = A^T Y_(n), max|A|                      (dominant)
//   reduce  fixed-order sums of the partials
//   chol1   degeneracy test, R1 = chol(W)
//   gram2   W2 = (A R1^-1)^T (A R1^-1)
//   chol2   R2 = chol(W2), Rinv = R1^-1 R2^-1, core: G_(n) = Rinv^T M
//           (U_new = A Rinv => U_new^T Y_(n) = Rinv^T A^T Y_(n); this replaces
//           the reference's second sparse pass ttmc_core)
//   apply   U_new = A Rinv, P = U_new^T U_old
//   drift   2K - 2||P||_*, and at the end of a sweep f, fit, stop rule
// The Householder branch (householder -> drift product -> sparse core pass)
// runs instead of gram2..apply only when chol1/chol2 flag it on the device.
// A whole sweep is captured once per factor-buffer parity as a CUDA graph.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_set>
#include <vector>
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <thread>

#include "hq_comm.cuh"
#include "hq_dense.cuh"
#include "hq_fast.cuh"
#include "hq_long.cuh"
#include "hq_tns.cuh"
#include "hq_hooi.cuh"

namespace hq {

namespace {

thread_local std::string g_err;
thread_local int64_t g_payload = 0;

template <class F>
int guard(F&& f) {
    try {
        f();
        return HQ_OK;
    } catch (const Error& e) {
        g_err = e.what();
        g_payload = e.payload;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        g_payload = 0;
        return HQ_ERR_CAPACITY;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_payload = 0;
        return HQ_ERR_INTERNAL;
    }
}

inline cudaStream_t as_stream(void* p) { return reinterpret_cast<cudaStream_t>(p); }

}  // namespace

// ---- host Gaussian stream, bit-exact with tucker::Rng::normal (rng.hpp:24-35):
// raw mt19937_64 draws are sequential; the Box-Muller transform of each pair
// is independent, so it is spread over host threads.
uint64_t mix_seed(uint64_t seed, uint64_t salt) {  // rng.hpp:57-62
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (salt + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void gaussian_stream(uint64_t seed, uint64_t count, double* out) {
    if (!count) return;
    const uint64_t pairs = (count + 1) / 2;
    std::vector<uint64_t> raw(2 * pairs);
    std::mt19937_64 gen(seed);
    for (auto& r : raw) r = gen();
    unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (pairs < 65536) nt = 1;
    auto work = [&](uint64_t pb, uint64_t pe) {
        for (uint64_t k = pb; k < pe; ++k) {
            double u1 = 1.0 - static_cast<double>(raw[2 * k] >> 11) * 0x1.0p-53;
            double u2 = static_cast<double>(raw[2 * k + 1] >> 11) * 0x1.0p-53;
            double r = std::sqrt(-2.0 * std::log(u1));
            double theta = 6.283185307179586476925286766559 * u2;
            out[2 * k] = r * std::cos(theta);
            if (2 * k + 1 < count) out[2 * k + 1] = r * std::sin(theta);
        }
    };
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) th.emplace_back(work, pairs * t / nt, pairs * (t + 1) / nt);
    for (auto& t : th) t.join();
}

std::shared_ptr<const FillTable> fill_table(uint64_t count) {
    if (count == 0 || count > kFillTableCap) return nullptr;
    static std::mutex mu;
    static std::map<int, std::shared_ptr<FillTable>> cache;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    HQ_CUDA(cudaGetDevice(&dev));
    auto& t = cache[dev];
    if (!t || t->len < count) {
        const uint64_t len = std::min<uint64_t>(kFillTableCap, std::max<uint64_t>(count, t ? 2 * t->len : 0));
        std::vector<double> h(len);
        gaussian_stream(0x48514F5251ull, len, h.data());
        auto nt = std::make_shared<FillTable>();
        nt->buf.alloc(len);
        HQ_CUDA(cudaMemcpy(nt->buf.get(), h.data(), sizeof(double) * len, cudaMemcpyHostToDevice));
        nt->len = len;
        t = nt;  // holders of the previous table keep it alive
    }
    return t;
}

// ---------------------------------------------------------------- QR -----
void QrWork::ensure(uint64_t rows, int K) {
    size_t sl = dense_slots();
    if (wpart.n < sl * K * K) wpart.alloc(sl * K * K);
    if (ppart.n < sl * K * K) ppart.alloc(sl * K * K);
    if (maxpart.n < sl) maxpart.alloc(sl);
    if (w.n < (size_t)K * K) w.alloc(K * K);
    if (r1inv.n < (size_t)K * K) r1inv.alloc(K * K);
    if (rinv.n < (size_t)K * K) rinv.alloc(K * K);
    if (rc.n < (size_t)K * K) rc.alloc(K * K);
    if (!maxv.n) maxv.alloc(1);
    const size_t hw = householder_work_doubles(rows, K);
    if (hh.n < hw) {
        hh.alloc(hw);
        householder_reset(hh.get(), 0);
        HQ_CUDA(cudaDeviceSynchronize());
    }
    if (!st.n) st.alloc(1);
}

// Q = qr_orthonormal(A) on the device (A, Q device, rows x K).  Returns the
// fallback flag (1 when the Householder path ran).
void qr_device(const double* A, uint64_t rows, int K, double* Q, QrWork& w, cudaStream_t s) {
    w.ensure(rows, K);
    HQ_CUDA(cudaMemsetAsync(w.st.get(), 0, sizeof(DevStatus), s));
    DevStatus* st = w.st.get();
    launch_gram(A, rows, K, w.wpart.get(), w.maxpart.get(), st, kAlways, s);
    launch_reduce_pass(nullptr, 0, w.wpart.get(), K * K, w.maxpart.get(), dense_slots(), nullptr, w.w.get(),
                       w.maxv.get(), st, kAlways, s);
    launch_chol1(w.w.get(), w.maxv.get(), K, w.r1inv.get(), st, 0, rows, s);
    launch_gram2(A, rows, K, w.r1inv.get(), w.wpart.get(), st, s);
    launch_chol2(w.wpart.get(), dense_slots(), K, w.r1inv.get(), w.rinv.get(), w.rc.get(), nullptr, nullptr, nullptr,
                 st, s);
    launch_gram3(A, rows, K, w.r1inv.get(), w.rinv.get(), Q, w.wpart.get(), st, s);  // shifted: Q <- Q2
    launch_chol3(w.wpart.get(), dense_slots(), K, w.rc.get(), w.rinv.get(), w.w.get(), st, s);
    launch_apply_qr(A, rows, K, w.r1inv.get(), w.rinv.get(), Q, nullptr, nullptr, true, st, kOnlyCholQR, s);
    DevStatus h{};
    HQ_CUDA(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    if (h.fallback) {  // Householder with the reference's fill (its normal stream built only when needed)
        auto table = fill_table(rows * (uint64_t)K);
        launch_householder(A, rows, K, Q, w.hh.get(), table ? table->buf.get() : nullptr, table ? table->len : 0, st,
                           kOnlyFallback, s);
        HQ_CUDA(cudaStreamSynchronize(s));
    }
}

void check_rank_limits(int K) {
    if (K > kMaxRank) fail(HQ_ERR_CAPACITY, "rank " + std::to_string(K) + " above the engine limit of 32");
}

// ---------------------------------------------- helpers for hq_hooi.cu ----
void ttmc_core_dev(const DeviceTensor& T, const FactorPtrs& f, const int* ranks, double* core, cudaStream_t s) {
    ModeShape sh = make_mode_shape(T.order, ranks, 0);
    const ModeLayout& L = T.modes[0];
    const int sl = pass_slots(L, sh);
    DBuf<double> mpart, wpart, maxpart, ypart;
    mpart.alloc((size_t)sl * sh.kn * sh.L);
    wpart.alloc((size_t)sl * sh.kn * sh.kn);
    maxpart.alloc(sl);
    ypart.alloc(std::max<size_t>(1, pass_ypart_doubles(L, sh)));
    PassOut out{nullptr, mpart.get(), wpart.get(), maxpart.get(), ypart.get()};
    launch_pass(T, 0, sh, f, kCore, nullptr, out, nullptr, kAlways, s);
    launch_reduce_core(mpart.get(), sl, (uint64_t)sh.kn * sh.L, core, nullptr, kAlways, s);
    HQ_CUDA(cudaStreamSynchronize(s));
}

double subspace_distance_dev(const double* u, const double* v, uint64_t rows, int k, cudaStream_t s) {
    DBuf<double> pp, d, obj, fit, fp;
    DBuf<DevStatus> st;
    pp.alloc((size_t)dense_slots() * k * k);
    d.alloc(1);
    obj.alloc(1);
    fit.alloc(1);
    fp.alloc(1);
    st.alloc(1);
    HQ_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(DevStatus), s));
    launch_apply(nullptr, rows, k, nullptr, const_cast<double*>(u), v, pp.get(), false, nullptr, kAlways, s);
    SweepTrace tr{obj.get(), fit.get(), d.get(), fp.get(), nullptr, 1, 0.0, nullptr};
    launch_drift(pp.get(), dense_slots(), k, nullptr, 0, 0.0, 1, 0, false, 0.0, 1, tr, st.get(), s);
    double out = 0.0;
    HQ_CUDA(cudaMemcpyAsync(&out, d.get(), 8, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    return out;
}

double orthonormality_defect_dev(const double* u, uint64_t rows, int k, cudaStream_t s) {
    DBuf<double> wp, mx;
    wp.alloc((size_t)dense_slots() * k * k);
    mx.alloc(1);
    launch_defect(u, rows, k, wp.get(), mx.get(), s);
    double out = 0.0;
    HQ_CUDA(cudaMemcpyAsync(&out, mx.get(), 8, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    return out;
}

// init_factors (solvers.cpp:182-215): 0 random (seeded Gaussian + QR), 1 HOSVD, 2 caller's factors
void init_factors_dev(const DeviceTensor& T, const hq_config& cfg, const double* const* init_host, double* const* U,
                      cudaStream_t s) {
    const int N = T.order;
    int ranks[kMaxOrder];
    for (int v = 0; v < N; ++v) ranks[v] = (int)cfg.ranks[v];
    if (cfg.init == 2) {
        for (int v = 0; v < N; ++v)
            HQ_CUDA(cudaMemcpyAsync(U[v], init_host[v], sizeof(double) * T.dims[v] * ranks[v], cudaMemcpyHostToDevice,
                                    s));
        HQ_CUDA(cudaStreamSynchronize(s));
    } else if (cfg.init == 0) {
        QrWork qw;
        for (int v = 0; v < N; ++v) {
            std::vector<double> g((size_t)T.dims[v] * ranks[v]);
            gaussian_stream(mix_seed(cfg.seed, (uint64_t)v), g.size(), g.data());
            DBuf<double> a;
            a.alloc(std::max<size_t>(1, g.size()));
            HQ_CUDA(cudaMemcpyAsync(a.get(), g.data(), sizeof(double) * g.size(), cudaMemcpyHostToDevice, s));
            qr_device(a.get(), T.dims[v], ranks[v], U[v], qw, s);
            HQ_CUDA(cudaStreamSynchronize(s));
        }
    } else if (cfg.init == 1) {
        hosvd_init_dev(T, ranks, cfg.capacity_cap ? cfg.capacity_cap : (1ull << 31), U, s);
    } else {
        fail(HQ_ERR_SHAPE, "unknown init mode");
    }
}

// ------------------------------------------------------------- solver ----
struct Solver {
    const DeviceTensor* T = nullptr;
    cudaStream_t s = nullptr;
    int N = 0;
    int ranks[kMaxOrder] = {0};
    uint64_t dims[kMaxOrder] = {0};
    uint64_t core_size = 1;
    hq_config cfg{};
    double dns = 0.0;
    double initial_objective = 0.0;

    DBuf<double> U[kMaxOrder][2];
    DBuf<double> core, gt, A, mpart, wpart, maxpart, ypart, red3, r1inv, rinv, rc, w2part, hh;
    DBuf<double> ppart[kMaxOrder];  // per-mode drift products (their drift kernels run on the side stream)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork[kMaxOrder] = {nullptr};
    cudaEvent_t ev_join = nullptr;
    DBuf<double> tr_obj, tr_fit, tr_drift, fit_prev;
    DBuf<double> tr_p;      // P = U_new^T U_old per (sweep, mode): drifts evaluated at download
    DBuf<double> tr_pr;     // multi-GPU: tr_p summed over the ranks (each rank stores its rows' partial)
    // gradient tracing (trace_gradients / tol_grad > 0, solvers.cpp:58): per-update diagnostics
    bool tracing = false;
    DBuf<double> tr_grad, tr_fb, tr_sig, tr_lam;
    DBuf<unsigned long long> tr_t, tr_tend;
    DBuf<int> dranks;
    int kmax_ = 1;
    // multi-GPU: this rank owns rows [bnd[n][rank], bnd[n][rank+1]) of every mode n
    const Comm* comm = nullptr;
    std::vector<uint64_t> bnd[kMaxOrder];
    DBuf<double> w2red, pred;  // all-reduced K x K Gram / drift product (distributed path)
    DBuf<double> core_alt;     // conditional core recompute (distributed path)
    std::shared_ptr<const FillTable> fill;  // Householder fill stream (rank-deficient QR)
    // multi-GPU: the other ranks' replicas of every factor buffer, mapped through CUDA IPC (peer_u[n][q][i] is
    // U[n][q] of the i-th other rank).  When every rank could map every peer, the apply stores its rows of U_new
    // into all replicas itself (k_rowgemm's peer_out) and a barrier replaces the all-gather.
    std::vector<double*> peer_u[kMaxOrder][2];
    std::vector<void*> peer_maps;  // cudaIpcOpenMemHandle results (closed in the destructor)
    bool peer_apply = false;
    uint64_t rb(int n) const { return comm ? bnd[n][comm->rank] : 0; }
    uint64_t re(int n) const { return comm ? bnd[n][comm->rank + 1] : dims[n]; }
    DBuf<DevStatus> st;
    ModeShape sh[kMaxOrder];
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    int host_parity = 0;
    uint64_t launched = 0;
    std::vector<cudaEvent_t> ev;  // ev[0] start, ev[i] after sweep i
    QrWork qw;
    // opt-in step profiler (HQ_PROFILE_SWEEP=1): events after every launch of one eager sweep
    bool prof = false;
    std::vector<std::pair<std::string, cudaEvent_t>> prof_ev;
    void mark(const char* what) {
        if (!prof) return;
        cudaEvent_t e;
        HQ_CUDA(cudaEventCreate(&e));
        HQ_CUDA(cudaEventRecord(e, s));
        prof_ev.emplace_back(what, e);
    }

    ~Solver() {
        if (!peer_maps.empty()) {
            cudaDeviceSynchronize();  // no kernel of this rank may still be storing into a peer's replica
            close_peers();
        }
        for (auto& g : graph)
            if (g) cudaGraphExecDestroy(g);
        for (auto e : ev) cudaEventDestroy(e);
        for (auto e : ev_fork)
            if (e) cudaEventDestroy(e);
        if (ev_join) cudaEventDestroy(ev_join);
        if (side) cudaStreamDestroy(side);
    }

    FactorPtrs factors_for_mode(int n, int p) const {
        FactorPtrs f{};
        for (int v = 0; v < N; ++v) {
            f.u[v] = U[v][(v < n) ? 1 - p : p].get();
            f.k[v] = ranks[v];
        }
        return f;
    }

    PassOut pass_out(double* a) {
        return PassOut{a, mpart.get(), wpart.get(), maxpart.get(), ypart.get()};
    }

    void setup(const DeviceTensor* t, const hq_config* c, const double* const* init, cudaStream_t stream,
               const Comm* cm = nullptr) {
        T = t;
        comm = cm;  // a one-rank communicator runs the distributed path with identity collectives
        s = stream;
        cfg = *c;
        N = t->order;
        if (cfg.order != N) fail(HQ_ERR_SHAPE, "rank count does not match tensor order");
        for (int v = 0; v < N; ++v) {  // solvers.cpp:22-30
            if (cfg.ranks[v] < 1 || cfg.ranks[v] > t->dims[v])
                fail(HQ_ERR_SHAPE, "rank for mode " + std::to_string(v + 1) + " must lie in [1, " +
                                       std::to_string(t->dims[v]) + "]");
            ranks[v] = (int)cfg.ranks[v];
            dims[v] = t->dims[v];
            check_rank_limits(ranks[v]);
            core_size *= (uint64_t)ranks[v];
        }
        if (cfg.max_sweeps < 1) fail(HQ_ERR_SHAPE, "max_sweeps must be at least 1");
        if (cfg.tol_fit_change < 0.0) fail(HQ_ERR_SHAPE, "tolerance must be nonnegative");
        dns = t->norm_sq;
        size_t maxIK = 0, maxML = 0, maxslots = 0, maxy = 0, maxLK = 0, maxGT = 0;
        for (int v = 0; v < N; ++v) {
            sh[v] = make_mode_shape(N, ranks, v);
            maxIK = std::max(maxIK, (size_t)dims[v] * ranks[v]);
            int sl = pass_slots(t->modes[v], sh[v]);
            maxslots = std::max(maxslots, (size_t)sl);
            maxML = std::max(maxML, (size_t)sl * sh[v].kn * sh[v].L);
            maxy = std::max(maxy, pass_ypart_doubles(t->modes[v], sh[v]));
            maxLK = std::max(maxLK, (size_t)sh[v].kn * sh[v].L);
            maxGT = std::max(maxGT, gt_doubles(sh[v]));
        }
        int kmax = 1;
        for (int v = 0; v < N; ++v) kmax = std::max(kmax, ranks[v]);
        for (int v = 0; v < N; ++v)
            for (int p = 0; p < 2; ++p) U[v][p].alloc((size_t)dims[v] * ranks[v]);
        core.alloc(core_size);
        gt.alloc(maxGT);
        A.alloc(maxIK);
        mpart.alloc(maxML);
        wpart.alloc(maxslots * kmax * kmax);
        maxpart.alloc(maxslots);
        ypart.alloc(std::max<size_t>(maxy, 1));
        // M, W and max|A| of a mode update in one buffer (per mode: M at 0, W at K_n L, max after W) so
        // the distributed path all-reduces them in one call (max|A| >= 0 per rank: its sum is zero
        // exactly when every rank's is, which is all the degeneracy test reads)
        red3.alloc(maxLK + (size_t)kmax * kmax + 1);
        r1inv.alloc(kmax * kmax);
        rinv.alloc(kmax * kmax);
        rc.alloc(kmax * kmax);
        w2part.alloc((size_t)dense_slots() * kmax * kmax);
        for (int v = 0; v < N; ++v) ppart[v].alloc((size_t)dense_slots() * ranks[v] * ranks[v]);
        {
            size_t hw = 0;
            for (int v = 0; v < N; ++v) hw = std::max(hw, householder_work_doubles(dims[v], ranks[v]));
            hh.alloc(hw);
            householder_reset(hh.get(), s);
            // the reference's fill stream for the largest Householder this solve can run
            fill = fill_table(maxIK);
        }
        w2red.alloc(kmax * kmax);
        if (comm) core_alt.alloc(core_size);
        pred.alloc(kmax * kmax);
        if (t->shard_world > 1 && (!comm || comm->world != t->shard_world || comm->rank != t->shard_rank))
            fail(HQ_ERR_SHAPE, "the tensor is sharded for rank " + std::to_string(t->shard_rank) + " of " +
                                   std::to_string(t->shard_world) + "; the solver's communicator does not match");
        if (t->shard_world > 1 && cfg.init == 1)
            fail(HQ_ERR_SHAPE, "HOSVD initialisation needs the whole tensor on every rank (hq_tensor_shard frees it)");
        if (comm) {
            for (int v = 0; v < N; ++v) {
                if (t->shard_world > 1) {
                    bnd[v] = t->shard_bounds[v];
                    continue;
                }
                std::vector<int64_t> off(dims[v] + 1);
                HQ_CUDA(cudaMemcpyAsync(off.data(), t->modes[v].rowptr.get(), sizeof(int64_t) * off.size(),
                                        cudaMemcpyDeviceToHost, s));
                HQ_CUDA(cudaStreamSynchronize(s));
                std::vector<uint64_t> uo(off.begin(), off.end());
                bnd[v].assign(comm->world + 1, 0);
                partition_rows(uo.data(), dims[v], comm->world, bnd[v].data());
            }
        }
        HQ_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        for (int v = 0; v < N; ++v) HQ_CUDA(cudaEventCreateWithFlags(&ev_fork[v], cudaEventDisableTiming));
        HQ_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        tr_obj.alloc(cfg.max_sweeps);
        tr_fit.alloc(cfg.max_sweeps);
        tr_drift.alloc(cfg.max_sweeps * N);
        kmax_ = kmax;
        tracing = cfg.trace_gradients || cfg.tol_grad > 0.0;
        if (tracing) {
            tr_grad.alloc(cfg.max_sweeps * N);
            tr_fb.alloc(cfg.max_sweeps * N);
            tr_sig.alloc(cfg.max_sweeps * N * kmax);
            tr_lam.alloc(cfg.max_sweeps * N * kmax);
            tr_t.alloc(cfg.max_sweeps * N);
            tr_tend.alloc(cfg.max_sweeps);
        }
        tr_p.alloc((size_t)cfg.max_sweeps * N * kmax * kmax);
        dranks.alloc(N);
        HQ_CUDA(cudaMemcpyAsync(dranks.get(), ranks, sizeof(int) * N, cudaMemcpyHostToDevice, s));
        fit_prev.alloc(1);
        st.alloc(1);
        HQ_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(DevStatus), s));

        setup_peers();
        // ---- initial factors (solvers.cpp:182-215)
        {
            double* u0[kMaxOrder];
            for (int v = 0; v < N; ++v) u0[v] = U[v][0].get();
            init_factors_dev(*T, cfg, init, u0, s);
        }
        // ---- initial core (solvers.cpp:66) and objective
        compute_core(0, kAlways);
        DBuf<double> f0;
        f0.alloc(1);
        launch_core_normsq(core.get(), core_size, f0.get(), s);
        HQ_CUDA(cudaMemcpyAsync(&initial_objective, f0.get(), 8, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        double fp = dns - initial_objective;
        HQ_CUDA(cudaMemcpyAsync(fit_prev.get(), &fp, 8, cudaMemcpyHostToDevice, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        host_parity = 0;
    }

    // Multi-GPU: exchange CUDA IPC handles of the factor buffers and map every other rank's replicas.  The
    // handles travel through the communicator's own all-reduce (each byte as a double in the rank's segment of
    // a zeroed array: exact sums), so both transports carry them.  HQ_PEER_APPLY=0 keeps the all-gather.
    void setup_peers() {
        peer_apply = false;
        if (!comm || comm->world <= 1 || comm->world - 1 > kMaxPeers) return;
        const char* e = std::getenv("HQ_PEER_APPLY");
        const int W = comm->world, R = comm->rank;
        const int nb = 2 * N, hb = (int)sizeof(cudaIpcMemHandle_t);
        const size_t len = (size_t)W * nb * hb + W;  // handles, then one "mapped all peers" flag per rank
        std::vector<double> h(len, 0.0);
        bool ok = !(e && e[0] == '0');
        for (int v = 0; v < N && ok; ++v)
            for (int q = 0; q < 2 && ok; ++q) {
                cudaIpcMemHandle_t mh;
                if (cudaIpcGetMemHandle(&mh, U[v][q].p) != cudaSuccess) {
                    cudaGetLastError();
                    ok = false;
                    break;
                }
                const unsigned char* b = reinterpret_cast<const unsigned char*>(&mh);
                for (int i = 0; i < hb; ++i) h[((size_t)R * nb + 2 * v + q) * hb + i] = (double)b[i];
            }
        DBuf<double> d;
        d.alloc(len);
        auto exchange = [&] {
            HQ_CUDA(cudaMemcpyAsync(d.get(), h.data(), sizeof(double) * len, cudaMemcpyHostToDevice, s));
            comm->allreduce_sum(d.get(), len, s);
            HQ_CUDA(cudaMemcpyAsync(h.data(), d.get(), sizeof(double) * len, cudaMemcpyDeviceToHost, s));
            HQ_CUDA(cudaStreamSynchronize(s));
        };
        h[(size_t)W * nb * hb + R] = ok ? 1.0 : 0.0;
        exchange();
        bool all = true;
        for (int r = 0; r < W; ++r) all = all && h[(size_t)W * nb * hb + r] == 1.0;
        std::vector<double*> maps[kMaxOrder][2];
        bool mapped = all;
        for (int r = 0; r < W && mapped; ++r) {
            if (r == R) continue;
            for (int v = 0; v < N && mapped; ++v)
                for (int q = 0; q < 2 && mapped; ++q) {
                    cudaIpcMemHandle_t mh;
                    unsigned char* b = reinterpret_cast<unsigned char*>(&mh);
                    for (int i = 0; i < hb; ++i) b[i] = (unsigned char)h[((size_t)r * nb + 2 * v + q) * hb + i];
                    void* ptr = nullptr;
                    if (cudaIpcOpenMemHandle(&ptr, mh, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                        cudaGetLastError();
                        mapped = false;
                        break;
                    }
                    peer_maps.push_back(ptr);
                    maps[v][q].push_back(static_cast<double*>(ptr));
                }
        }
        // second round: every rank mapped every replica, or nobody uses them
        std::fill(h.begin(), h.end(), 0.0);
        h[(size_t)W * nb * hb + R] = mapped ? 1.0 : 0.0;
        exchange();
        for (int r = 0; r < W; ++r) mapped = mapped && h[(size_t)W * nb * hb + r] == 1.0;
        if (mapped) {
            for (int v = 0; v < N; ++v)
                for (int q = 0; q < 2; ++q) peer_u[v][q] = maps[v][q];
            peer_apply = true;
        } else {
            close_peers();
        }
    }
    void close_peers() {
        for (void* m : peer_maps) cudaIpcCloseMemHandle(m);
        peer_maps.clear();
    }

    // core = X x {U^T} with the parity-p factors, via the mode-0 pass
    // core = X x {U^T} by a kCore sparse pass over mode 0 (setup; after a
    // Householder fallback or a shifted CholeskyQR3 update, where R^-T M would
    // carry the Gram matrix's conditioning into the core).  Multi-GPU: the
    // all-reduce runs unconditionally in the captured graph, so a conditional
    // recompute goes through core_alt and is copied into place only when it ran.
    // the mode whose kCore pass is cheapest: the longest rows (fewest non-empty rows) run on the
    // DMMA long-row path; ties keep the lowest mode
    int core_mode() const {
        int best = 0;
        for (int v = 1; v < N; ++v)
            if (T->modes[v].nonempty_rows < T->modes[best].nonempty_rows) best = v;
        return best;
    }

    void compute_core(int p, int run_if, int updated_mode = -1) {
        FactorPtrs f{};
        for (int v = 0; v < N; ++v) {
            int q = (updated_mode >= 0 && v <= updated_mode) ? 1 - p : p;
            f.u[v] = U[v][q].get();
            f.k[v] = ranks[v];
        }
        const int cm = core_mode();
        launch_pass(*T, cm, sh[cm], f, kCore, nullptr, pass_out(nullptr), st.get(), run_if, s, rb(cm), re(cm));
        const int slots = pass_slots(T->modes[cm], sh[cm]);
        if (comm && run_if != kAlways) {
            launch_reduce_core_mode(mpart.get(), slots, sh[cm], core_alt.get(), st.get(), run_if, s);
            comm->allreduce_sum(core_alt.get(), core_size, s);
            launch_reduce_core(core_alt.get(), 1, core_size, core.get(), st.get(), run_if, s);
        } else {
            launch_reduce_core_mode(mpart.get(), slots, sh[cm], core.get(), st.get(), run_if, s);
            if (comm) comm->allreduce_sum(core.get(), core_size, s);
        }
    }

    void mode_update(int n, int p) {
        const ModeShape& m = sh[n];
        const int K = ranks[n];
        const uint64_t r0 = rb(n), r1 = re(n), lrows = r1 - r0;
        FactorPtrs f = factors_for_mode(n, p);
        DevStatus* S = st.get();
        launch_gt(core.get(), m, ranks, gt.get(), S, s);
        mark("gt");
        launch_pass(*T, n, m, f, kTTMcTC, gt.get(), pass_out(A.get()), S, kAlways, s, r0, r1);
        mark("pass");
        const int slots = pass_slots(T->modes[n], m);
        double* mred = red3.get();
        double* wred = mred + (size_t)m.kn * m.L;
        double* maxv = wred + (size_t)K * K;
        launch_reduce_pass(mpart.get(), m.kn * m.L, wpart.get(), K * K, maxpart.get(), slots, mred, wred, maxv, S,
                           kAlways, s);
        mark("reduce");
        if (comm) {  // M, W, max|A| over all ranks' rows
            comm->allreduce_sum(mred, (size_t)m.kn * m.L + (size_t)K * K + 1, s);
        }
        if (tracing) {  // pre-update diagnostics (solvers.cpp:126-137): W = A^T A and G_(n) at hand
            UpdTrace ut{tr_grad.get(), tr_fb.get(), tr_sig.get(), tr_lam.get(), tr_t.get(), kmax_};
            launch_update_diag(wred, gt.get(), K, m.L, n, N, ut, S, s);
        }
        launch_chol1(wred, maxv, K, r1inv.get(), S, n + 1, dims[n], s, comm != nullptr);
        mark("chol1");
        const double* a_loc = A.get() + r0 * K;
        double* unew = U[n][1 - p].get();
        const double* uold = U[n][p].get();
        double* pp = ppart[n].get();
        int pslots = dense_slots();
        if (!comm) {
            launch_gram2(a_loc, lrows, K, r1inv.get(), w2part.get(), S, s);
            mark("gram2");
            launch_chol2(w2part.get(), dense_slots(), K, r1inv.get(), rinv.get(), rc.get(), mred, &m, core.get(),
                         S, s);
            mark("chol2");
            // shifted CholeskyQR3 branch (device flag): U_new <- Q2, R3
            launch_gram3(a_loc, lrows, K, r1inv.get(), rinv.get(), unew, w2part.get(), S, s);
            launch_chol3(w2part.get(), dense_slots(), K, rc.get(), rinv.get(), wred, S, s);
            mark("cholqr3(no-op)");
            // U_new = (A R1^-1) R2^-1 (shifted: Q2 R3^-1), P partials
            launch_apply_qr(a_loc, lrows, K, r1inv.get(), rinv.get(), unew, uold, pp, true, S, kOnlyCholQR, s);
            mark("apply");
            // Householder branch (device flag)
            launch_householder(A.get(), dims[n], K, unew, hh.get(), fill ? fill->buf.get() : nullptr,
                               fill ? fill->len : 0, S, kOnlyFallback, s);
            launch_apply(nullptr, dims[n], K, nullptr, unew, uold, pp, false, S, kOnlyFallback, s);
            compute_core(p, kFallbackOrShifted, n);
            mark("fallback(no-op)");
        } else {
            // distributed: plain CholeskyQR2 over this rank's rows with all-reduced Grams.  Any update that is
            // not plain (shifted or rank-deficient) stops the graph at chol1 / chol2 (abort 3) and is finished
            // by dist_continuation (the reference's Householder with its seeded fill, on the gathered A).
            double* uloc = unew + r0 * K;
            launch_gram2(a_loc, lrows, K, r1inv.get(), w2part.get(), S, s);
            launch_reduce_pass(nullptr, 0, w2part.get(), K * K, nullptr, dense_slots(), nullptr, w2red.get(), nullptr, S,
                               kOnlyCholQR, s);
            comm->allreduce_sum(w2red.get(), (size_t)K * K, s);
            launch_chol2(w2red.get(), 1, K, r1inv.get(), rinv.get(), rc.get(), mred, &m, core.get(), S, s, true, n + 1);
            // U_new rows = Q R^-1, P partials of this rank's rows (tr_p is all-reduced once, at download)
            if (peer_apply) {
                // the apply stores its rows into every rank's replica of U_new over peer memory; the barrier
                // orders those stores before the next pass's gathers on every rank
                double* po[kMaxPeers];
                const auto& pu = peer_u[n][1 - p];
                for (size_t i = 0; i < pu.size(); ++i) po[i] = pu[i] + r0 * K;
                launch_apply_qr(a_loc, lrows, K, r1inv.get(), rinv.get(), uloc, uold + r0 * K, pp, false, S,
                                kOnlyCholQR, s, po, (int)pu.size());
                comm->barrier(s);
            } else {
                launch_apply_qr(a_loc, lrows, K, r1inv.get(), rinv.get(), uloc, uold + r0 * K, pp, false, S,
                                kOnlyCholQR, s);
                comm->allgather_rows(unew, bnd[n].data(), (size_t)K, s);
            }
        }
        mode_tail(n, pp, pslots);
    }

    // P stored for the lazy drift (side stream); after the last mode, f, fit and the stop rules
    void mode_tail(int n, const double* pp, int pslots) {
        const int K = ranks[n];
        DevStatus* S = st.get();
        // the drift feeds only the trace: P is stored beside the next mode update (side stream) and the
        // drifts are evaluated in one batch at download
        HQ_CUDA(cudaEventRecord(ev_fork[n], s));
        HQ_CUDA(cudaStreamWaitEvent(side, ev_fork[n], 0));
        launch_store_p(pp, pslots, K, N, n, kmax_, cfg.max_sweeps, tr_p.get(), S, side);
        if (n == N - 1) {
            HQ_CUDA(cudaEventRecord(ev_join, side));
            HQ_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
            SweepTrace tr{tr_obj.get(), tr_fit.get(), tr_drift.get(), fit_prev.get(),
                          tracing ? tr_grad.get() : nullptr, N, cfg.tol_grad, tracing ? tr_tend.get() : nullptr};
            launch_sweep_end(core.get(), core_size, dns, cfg.tol_fit_change, cfg.max_sweeps, tr, S, s);
            mark("sweep_end");
        }
    }

    // Multi-GPU: finish the update the sweep graph stopped at (abort 3: its Gram matrix was not fit for plain
    // CholeskyQR2) as the reference does every update -- Householder QR with the seeded rank-deficiency fill
    // (dense_core.cpp:127-198) -- on the all-gathered A, redundantly on every rank (the same bits everywhere:
    // same A, same deterministic kernel, same fill stream), then the core by a sparse pass over this rank's
    // rows (all-reduced), then the rest of the sweep eagerly.  Every rank reaches the same decision from the
    // same all-reduced Gram matrix, so all ranks run the continuation together.
    void dist_continuation(const DevStatus& h) {
        const int n = h.pending_mode - 1;
        if (n < 0 || n >= N) fail(HQ_ERR_INTERNAL, "distributed continuation: no pending mode");
        const int p = h.sweep & 1;  // parity of the sweep in progress (sweep h.sweep + 1)
        const int K = ranks[n];
        DevStatus* S = st.get();
        double* unew = U[n][1 - p].get();
        const double* uold = U[n][p].get();
        launch_dist_resume(S, s);
        comm->allgather_rows(A.get(), bnd[n].data(), (size_t)K, s);
        launch_householder(A.get(), dims[n], K, unew, hh.get(), fill ? fill->buf.get() : nullptr,
                           fill ? fill->len : 0, S, kOnlyFallback, s);
        double* pp = ppart[n].get();
        launch_apply(nullptr, dims[n], K, nullptr, unew, uold, pp, false, S, kOnlyFallback, s);
        if (comm->rank != 0)  // P over all rows on every rank: one copy enters the download all-reduce
            HQ_CUDA(cudaMemsetAsync(pp, 0, sizeof(double) * (size_t)dense_slots() * K * K, s));
        compute_core(p, kAlways, n);
        mode_tail(n, pp, dense_slots());
        for (int m = n + 1; m < N; ++m) mode_update(m, p);
    }

    // Multi-GPU: run host-driven continuations until the sweeps requested so far are done (the graphs queued
    // behind a stopped update ran as no-ops: every kernel skips while abort is set, and the collectives in them
    // only re-send identical replicated data).
    void settle() {
        if (!comm) return;
        for (;;) {
            DevStatus h = status();
            if (h.abort != 3) return;
            dist_continuation(h);
            DevStatus h2 = status();
            if (h2.abort == 3) continue;
            if (h2.abort) return;
            host_parity = h2.sweep & 1;
            launched = (uint64_t)h2.sweep;
            const uint64_t done = (uint64_t)h2.sweep;
            for (uint64_t i = done; i < target && i < cfg.max_sweeps; ++i) {
                HQ_CUDA(cudaGraphLaunch(graph[host_parity], s));
                host_parity ^= 1;
                ++launched;
                if (launched < ev.size()) HQ_CUDA(cudaEventRecord(ev[launched], s));
            }
        }
    }

    void issue_sweep(int p) {
        for (int n = 0; n < N; ++n) mode_update(n, p);
    }

    int launches_per_sweep() const {
        int c = 0;
        const int core_pass = pass_launch_count(T->modes[core_mode()], sh[core_mode()]);
        for (int n = 0; n < N; ++n) {
            const int pass = pass_launch_count(T->modes[n], sh[n]);
            if (tracing) c += 1;  // update diagnostics
            if (!comm)  // gt, pass, reduce, chol1, gram2, chol2, gram3, chol3, apply, householder, apply-P,
                        // core pass + reduce, store_p
                c += 1 + pass + 1 + 1 + 1 + 1 + 1 + 1 + 1 + 1 + 1 + core_pass + 1 + 1;
            else        // gt, pass, reduce, chol1, gram2, reduce, chol2, apply, store_p (collective kernels not counted)
                c += 1 + pass + 1 + 1 + 1 + 1 + 1 + 1 + 1;
        }
        return c + 1;  // sweep_end
    }

    void build_graphs() {
        for (int p = 0; p < 2; ++p) {
            cudaGraph_t g;
            HQ_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
            issue_sweep(p);
            HQ_CUDA(cudaStreamEndCapture(s, &g));
            HQ_CUDA(cudaGraphInstantiate(&graph[p], g, 0));
            cudaGraphDestroy(g);
        }
    }

    void profile_one_sweep() {
        prof = true;
        mark("start");
        issue_sweep(host_parity);
        host_parity ^= 1;
        ++launched;
        HQ_CUDA(cudaStreamSynchronize(s));
        prof = false;
        std::map<std::string, double> tot;
        for (size_t i = 1; i < prof_ev.size(); ++i) {
            float ms = 0.f;
            HQ_CUDA(cudaEventElapsedTime(&ms, prof_ev[i - 1].second, prof_ev[i].second));
            tot[prof_ev[i].first] += ms * 1e3;
        }
        double all = 0.0;
        for (auto& kv : tot) all += kv.second;
        std::fprintf(stderr, "[hq] sweep profile (us, warm, eager):");
        for (auto& kv : tot) std::fprintf(stderr, " %s=%.1f", kv.first.c_str(), kv.second);
        std::fprintf(stderr, " total=%.1f\n", all);
        for (auto& pe : prof_ev) cudaEventDestroy(pe.second);
        prof_ev.clear();
    }

    uint64_t target = 0;  // sweeps requested so far (settle() relaunches what a stopped update skipped)

    void run(uint64_t sweeps) {
        target += sweeps;
        if (!graph[0] && std::getenv("HQ_PROFILE_SWEEP") && sweeps > 1) {
            profile_one_sweep();
            --sweeps;
        }
        if (!graph[0]) {
            // first sweep eagerly (sets kernel attributes), then capture
            ensure_events();
            issue_sweep(host_parity);
            host_parity ^= 1;
            ++launched;
            HQ_CUDA(cudaEventRecord(ev[std::min<size_t>(launched, ev.size() - 1)], s));
            build_graphs();
            if (sweeps) --sweeps;
        }
        ensure_events();
        for (uint64_t i = 0; i < sweeps; ++i) {
            HQ_CUDA(cudaGraphLaunch(graph[host_parity], s));
            host_parity ^= 1;
            ++launched;
            if (launched < ev.size()) HQ_CUDA(cudaEventRecord(ev[launched], s));
        }
    }

    void ensure_events() {
        if (ev.empty()) {
            ev.resize(cfg.max_sweeps + 1);
            for (auto& e : ev) HQ_CUDA(cudaEventCreate(&e));
            HQ_CUDA(cudaEventRecord(ev[0], s));
        }
    }

    DevStatus status() {
        DevStatus h{};
        HQ_CUDA(cudaMemcpyAsync(&h, st.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        return h;
    }

    void check_status(const DevStatus& h) {
        if (h.abort == 5 && h.diag_code == 1)  // manifold.cpp:45-47
            fail(HQ_ERR_DIAGNOSTIC, "grad_norm_sq is negative beyond rounding; orthonormality is broken upstream");
        if (h.abort == 5)  // manifold.cpp:79-81
            fail(HQ_ERR_DIAGNOSTIC, "interlacing violated at k=" + std::to_string(h.diag_k) +
                                        "; upstream state is numerically corrupted");
        if (h.abort == 6) fail(HQ_ERR_CONTRACT, "gram_eigvals_desc: matrix is not PSD");  // dense_core.cpp:381-382
        if (h.abort == 3)  // settle() finishes these; reaching here means a caller skipped it
            fail(HQ_ERR_INTERNAL, "distributed solve stopped at a pending Householder update (mode " +
                                      std::to_string(h.pending_mode) + ") that was not continued");
        if (h.abort == 1)
            fail(HQ_ERR_DEGENERATE,
                 "degenerate state: TTMcTC output is identically zero for mode " + std::to_string(h.degenerate_mode),
                 h.degenerate_mode);
    }

    // solve loop: launch sweeps in batches, stop once the device reports the
    // stop rule (or max_sweeps)
    void solve() {
        uint64_t remaining = cfg.max_sweeps;
        const uint64_t batch = cfg.tol_fit_change > 0.0 ? 2 : remaining;
        while (remaining) {
            uint64_t b = std::min(batch, remaining);
            run(b);
            remaining -= b;
            settle();
            DevStatus h = status();
            check_status(h);
            if (h.abort || (uint64_t)h.sweep >= cfg.max_sweeps) break;
        }
    }

    void download(double* const* factors_out, double* core_out, hq_trace* tr) {
        DevStatus h = status();
        check_status(h);
        const int parity = h.sweep & 1;
        if (factors_out)
            for (int v = 0; v < N; ++v)
                if (factors_out[v])
                    HQ_CUDA(cudaMemcpyAsync(factors_out[v], U[v][parity].get(), sizeof(double) * dims[v] * ranks[v],
                                            cudaMemcpyDeviceToHost, s));
        if (core_out)
            HQ_CUDA(cudaMemcpyAsync(core_out, core.get(), sizeof(double) * core_size, cudaMemcpyDeviceToHost, s));
        if (comm && h.sweep) {  // every rank, trace requested or not: the per-rank P partials, summed
            const size_t np = (size_t)h.sweep * N * kmax_ * kmax_;
            if (!tr_pr.p) tr_pr.alloc(tr_p.n);
            HQ_CUDA(cudaMemcpyAsync(tr_pr.get(), tr_p.get(), sizeof(double) * np, cudaMemcpyDeviceToDevice, s));
            comm->allreduce_sum(tr_pr.get(), np, s);
        }
        if (tr) {
            tr->data_norm_sq = dns;
            tr->initial_objective = initial_objective;
            tr->sweeps = (uint64_t)h.sweep;
            if (h.sweep) {
                if (tr->objective)
                    HQ_CUDA(cudaMemcpyAsync(tr->objective, tr_obj.get(), 8 * h.sweep, cudaMemcpyDeviceToHost, s));
                if (tr->fit) HQ_CUDA(cudaMemcpyAsync(tr->fit, tr_fit.get(), 8 * h.sweep, cudaMemcpyDeviceToHost, s));
                if (tr->drift) {
                    launch_drift_batch(comm ? tr_pr.get() : tr_p.get(), h.sweep * N, N, dranks.get(), kmax_,
                                       tr_drift.get(), s);
                    HQ_CUDA(cudaMemcpyAsync(tr->drift, tr_drift.get(), 8 * h.sweep * N, cudaMemcpyDeviceToHost, s));
                }
            }
            HQ_CUDA(cudaStreamSynchronize(s));
            if (tr->elapsed_s && !ev.empty()) {
                for (uint64_t i = 1; i <= (uint64_t)h.sweep && i < ev.size(); ++i) {
                    float ms = 0.f;
                    HQ_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[i]));
                    tr->elapsed_s[i - 1] = ms * 1e-3;
                }
            }
            const uint64_t nu = (uint64_t)h.sweep * N;
            if (tr->grad_norm_sq) {
                if (tracing && nu)
                    HQ_CUDA(cudaMemcpy(tr->grad_norm_sq, tr_grad.get(), 8 * nu, cudaMemcpyDeviceToHost));
                else
                    for (uint64_t i = 0; i < nu; ++i) tr->grad_norm_sq[i] = 0.0;  // solvers.cpp:82
            }
            tr->updates = 0;
            if (tracing && nu) {
                // ModeUpdateRecords (solvers.hpp:40-49): f_after of update n is f_before of update n+1, the
                // sweep's objective for the last mode; elapsed between successive diagnostics points
                std::vector<double> fb(nu), obj(h.sweep), sig(nu * kmax_), lam(nu * kmax_);
                std::vector<unsigned long long> t(nu), tend(h.sweep);
                HQ_CUDA(cudaMemcpy(fb.data(), tr_fb.get(), 8 * nu, cudaMemcpyDeviceToHost));
                HQ_CUDA(cudaMemcpy(obj.data(), tr_obj.get(), 8 * h.sweep, cudaMemcpyDeviceToHost));
                HQ_CUDA(cudaMemcpy(sig.data(), tr_sig.get(), 8 * nu * kmax_, cudaMemcpyDeviceToHost));
                HQ_CUDA(cudaMemcpy(lam.data(), tr_lam.get(), 8 * nu * kmax_, cudaMemcpyDeviceToHost));
                HQ_CUDA(cudaMemcpy(t.data(), tr_t.get(), 8 * nu, cudaMemcpyDeviceToHost));
                HQ_CUDA(cudaMemcpy(tend.data(), tr_tend.get(), 8 * h.sweep, cudaMemcpyDeviceToHost));
                tr->updates = nu;
                for (uint64_t i = 0; i < nu; ++i) {
                    const uint64_t sw = i / N;
                    const int n = (int)(i % N);
                    const bool last = n == N - 1;
                    if (tr->upd_f_before) tr->upd_f_before[i] = fb[i];
                    if (tr->upd_f_after) tr->upd_f_after[i] = last ? obj[sw] : fb[i + 1];
                    if (tr->upd_elapsed_s) {
                        const unsigned long long t1 = last ? tend[sw] : t[i + 1];
                        tr->upd_elapsed_s[i] = t1 > t[i] ? (double)(t1 - t[i]) * 1e-9 : 0.0;
                    }
                    const uint64_t ks = tr->sigma_stride;
                    for (int k = 0; k < ranks[n] && ks; ++k) {
                        if (tr->upd_sigma && (uint64_t)k < ks) tr->upd_sigma[i * ks + k] = sig[i * kmax_ + k];
                        if (tr->upd_lambda && (uint64_t)k < ks) tr->upd_lambda[i * ks + k] = lam[i * kmax_ + k];
                    }
                }
            }
        }
        HQ_CUDA(cudaStreamSynchronize(s));
        // solvers.cpp:171-172
        DBuf<double> wp, mx;
        int kmax = 1;
        for (int v = 0; v < N; ++v) kmax = std::max(kmax, ranks[v]);
        wp.alloc((size_t)dense_slots() * kmax * kmax);
        mx.alloc(N);
        for (int v = 0; v < N; ++v) launch_defect(U[v][parity].get(), dims[v], ranks[v], wp.get(), mx.get() + v, s);
        std::vector<double> hm(N);
        HQ_CUDA(cudaMemcpyAsync(hm.data(), mx.get(), 8 * N, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        for (double d : hm)
            if (d > 1e-10) fail(HQ_ERR_DIAGNOSTIC, "solver produced factors with orthonormality defect above 1e-10");
    }
};

}  // namespace hq

struct hq_solver {
    std::unique_ptr<hq::Solver> impl;
};

using namespace hq;

// ====================================================================== C-ABI
extern "C" {

const char* hq_last_error(void) { return g_err.c_str(); }
int64_t hq_last_error_payload(void) { return g_payload; }
const char* hq_version(void) { return "hoqri_b200 0.1 (sm_100a)"; }

static int tensor_create_impl(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                              const double* values, bool on_device, void* stream, hq_tensor** out) {
    return guard([&] {
        if (!out) fail(HQ_ERR_SHAPE, "null output handle");
        if (order <= 0) fail(HQ_ERR_SHAPE, "sparse tensor needs at least one mode");
        if (nnz && (!coords || !values)) fail(HQ_ERR_SHAPE, "coordinate array does not match entry count");
        auto h = std::make_unique<hq_tensor>();
        h->stream = as_stream(stream);
        if (!h->stream) {
            HQ_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
            h->own_stream = true;
        }
        cudaStream_t s = h->stream;
        if (on_device || !nnz) {
            build_tensor(h->t, order, dims, nnz, coords, values, s);
        } else {
            DBuf<uint32_t> c;
            DBuf<double> v;
            c.alloc(nnz * order);
            v.alloc(nnz);
            // coordinates first at full link bandwidth; the values follow on a second stream while the
            // coordinate-only part of the build (range check, key packing, lexicographic sort) runs
            cudaStream_t s2 = nullptr;
            cudaEvent_t ev_c = nullptr, ev_v = nullptr;
            HQ_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
            HQ_CUDA(cudaEventCreateWithFlags(&ev_c, cudaEventDisableTiming));
            HQ_CUDA(cudaEventCreateWithFlags(&ev_v, cudaEventDisableTiming));
            struct Cleanup {
                cudaStream_t s2;
                cudaEvent_t a, b;
                ~Cleanup() {
                    cudaStreamSynchronize(s2);
                    cudaEventDestroy(a);
                    cudaEventDestroy(b);
                    cudaStreamDestroy(s2);
                }
            } cleanup{s2, ev_c, ev_v};
            HQ_CUDA(cudaMemcpyAsync(c.get(), coords, sizeof(uint32_t) * nnz * order, cudaMemcpyHostToDevice, s));
            HQ_CUDA(cudaEventRecord(ev_c, s));
            HQ_CUDA(cudaStreamWaitEvent(s2, ev_c, 0));
            HQ_CUDA(cudaMemcpyAsync(v.get(), values, sizeof(double) * nnz, cudaMemcpyHostToDevice, s2));
            HQ_CUDA(cudaEventRecord(ev_v, s2));
            if (std::getenv("HQ_PROFILE_BUILD")) {
                const auto t0 = std::chrono::steady_clock::now();
                HQ_CUDA(cudaStreamSynchronize(s));
                std::fprintf(stderr, "[build] upload wait     %8.2f ms (coordinates)\n",
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
            }
            build_tensor(h->t, order, dims, nnz, c.get(), v.get(), s, ev_v);
        }
        *out = h.release();
    });
}

int hq_tensor_create(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords, const double* values,
                     void* stream, hq_tensor** out) {
    return tensor_create_impl(order, dims, nnz, coords, values, false, stream, out);
}

int hq_tensor_create_dev(int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords_dev,
                         const double* values_dev, void* stream, hq_tensor** out) {
    return tensor_create_impl(order, dims, nnz, coords_dev, values_dev, true, stream, out);
}

int hq_tns_parse(const char* text, uint64_t len, int override_order, const uint64_t* override_dims, hq_tns** out) {
    return guard([&] {
        auto p = std::make_unique<hq_tns>();
        tns_parse(text, len, override_order, override_dims, *p);
        *out = p.release();
    });
}

int hq_tns_parse_file(const char* path, int override_order, const uint64_t* override_dims, hq_tns** out) {
    return guard([&] {
        FILE* f = std::fopen(path, "rb");
        if (!f) fail(HQ_ERR_VALUE, std::string("cannot open '") + path + "'");
        std::string buf;
        std::fseek(f, 0, SEEK_END);
        const long n = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        buf.resize(n > 0 ? (size_t)n : 0);
        const size_t got = n > 0 ? std::fread(&buf[0], 1, (size_t)n, f) : 0;
        std::fclose(f);
        buf.resize(got);
        auto p = std::make_unique<hq_tns>();
        tns_parse(buf.data(), buf.size(), override_order, override_dims, *p);
        *out = p.release();
    });
}

int hq_tns_info(const hq_tns* p, int* order, uint64_t* dims, uint64_t* nnz) {
    return guard([&] {
        if (order) *order = p->order;
        if (dims)
            for (size_t m = 0; m < p->dims.size(); ++m) dims[m] = p->dims[m];
        if (nnz) *nnz = p->values.size();
    });
}

int hq_tns_copy(const hq_tns* p, uint32_t* coords, double* values) {
    return guard([&] {
        if (coords) std::copy(p->coords.begin(), p->coords.end(), coords);
        if (values) std::copy(p->values.begin(), p->values.end(), values);
    });
}

int hq_tns_tensor(const hq_tns* p, void* stream, hq_tensor** out) {
    return tensor_create_impl((int)p->dims.size(), p->dims.data(), p->values.size(), p->coords.data(),
                              p->values.data(), false, stream, out);
}

int hq_tns_destroy(hq_tns* p) {
    return guard([&] { delete p; });
}

int hq_tensor_destroy(hq_tensor* t) {
    return guard([&] { delete t; });
}

int hq_tensor_info(const hq_tensor* t, int* order, uint64_t* dims, uint64_t* nnz) {
    return guard([&] {
        if (order) *order = t->t.order;
        if (dims)
            for (int m = 0; m < t->t.order; ++m) dims[m] = t->t.dims[m];
        if (nnz) *nnz = t->t.nnz;
    });
}

int hq_tensor_mode_plan(const hq_tensor* t, int mode, uint64_t* rows, uint64_t* nonempty_rows, uint64_t* long_rows,
                        uint64_t* long_segments, int* hot, uint64_t* max_tile32) {
    return guard([&] {
        if (mode < 0 || mode >= t->t.order)
            fail(HQ_ERR_RANGE, "mode " + std::to_string(mode) + " out of range for order " + std::to_string(t->t.order));
        const ModeLayout& L = t->t.modes[mode];
        if (rows) *rows = L.rows;
        if (nonempty_rows) *nonempty_rows = L.nonempty_rows;
        if (long_rows) *long_rows = L.long_rows;
        if (long_segments) *long_segments = L.long_segments;
        if (hot) *hot = L.hot ? 1 : 0;
        if (max_tile32) *max_tile32 = L.max_tile32;
    });
}

int hq_tensor_fiber_plan(const hq_tensor* t, int mode, uint64_t* units, uint64_t* long_nnz, uint64_t* segments,
                         uint64_t* short_max) {
    return guard([&] {
        if (mode < 0 || mode >= t->t.order)
            fail(HQ_ERR_RANGE, "mode " + std::to_string(mode) + " out of range for order " + std::to_string(t->t.order));
        const FiberLayout& F = t->t.modes[mode].fib;
        if (units) *units = F.on ? F.units : 0;
        if (long_nnz) *long_nnz = F.on ? F.long_nnz : 0;
        if (segments) *segments = F.on ? F.long_segments : 0;
        if (short_max) *short_max = (uint64_t)t->t.modes[mode].short_max;
    });
}

int hq_tensor_export(const hq_tensor* t, uint32_t* coords, double* values) {
    return guard([&] {
        require_unsharded(t->t, "hq_tensor_export");
        cudaStream_t s = t->stream;
        if (t->t.nnz) {
            if (coords)
                HQ_CUDA(cudaMemcpyAsync(coords, t->t.coords.get(), sizeof(uint32_t) * t->t.nnz * t->t.order,
                                        cudaMemcpyDeviceToHost, s));
            if (values)
                HQ_CUDA(cudaMemcpyAsync(values, t->t.vals.get(), sizeof(double) * t->t.nnz, cudaMemcpyDeviceToHost, s));
        }
        HQ_CUDA(cudaStreamSynchronize(s));
    });
}

int hq_tensor_buckets(const hq_tensor* t, int mode, uint64_t* offsets, uint64_t* entries) {
    return guard([&] {
        require_unsharded(t->t, "hq_tensor_buckets");
        if (mode < 0 || mode >= t->t.order) fail(HQ_ERR_RANGE, "mode out of range");
        export_buckets(t->t, mode, offsets, entries, t->stream);
    });
}

int hq_tensor_norm_sq(const hq_tensor* t, double* out) {
    return guard([&] { *out = t->t.norm_sq; });
}

namespace {

struct UploadedFactors {
    DBuf<double> u[kMaxOrder];
    FactorPtrs f{};
    int ranks[kMaxOrder] = {0};
};

void upload_factors(const DeviceTensor& T, const double* const* factors, const uint64_t* ranks, UploadedFactors& uf,
                    cudaStream_t s) {
    for (int v = 0; v < T.order; ++v) {
        if (ranks[v] == 0) fail(HQ_ERR_SHAPE, "factor with zero columns");
        check_rank_limits((int)ranks[v]);
        uf.ranks[v] = (int)ranks[v];
        uf.u[v].alloc(T.dims[v] * ranks[v]);
        HQ_CUDA(cudaMemcpyAsync(uf.u[v].get(), factors[v], sizeof(double) * T.dims[v] * ranks[v],
                                cudaMemcpyHostToDevice, s));
        uf.f.u[v] = uf.u[v].get();
        uf.f.k[v] = (int)ranks[v];
    }
}

struct PassBuffers {
    DBuf<double> mpart, wpart, maxpart, ypart, core;
    void ensure(const ModeLayout& L, const ModeShape& sh) {
        int sl = pass_slots(L, sh);
        mpart.alloc((size_t)sl * sh.kn * sh.L);
        wpart.alloc((size_t)sl * sh.kn * sh.kn);
        maxpart.alloc(sl);
        ypart.alloc(std::max<size_t>(1, pass_ypart_doubles(L, sh)));
    }
};

void core_device(const DeviceTensor& T, const UploadedFactors& uf, double* core_dev, cudaStream_t s) {
    ModeShape sh = make_mode_shape(T.order, uf.ranks, 0);
    PassBuffers pb;
    pb.ensure(T.modes[0], sh);
    PassOut out{nullptr, pb.mpart.get(), pb.wpart.get(), pb.maxpart.get(), pb.ypart.get()};
    launch_pass(T, 0, sh, uf.f, kCore, nullptr, out, nullptr, kAlways, s);
    uint64_t size = (uint64_t)sh.kn * sh.L;
    launch_reduce_core(pb.mpart.get(), pass_slots(T.modes[0], sh), size, core_dev, nullptr, kAlways, s);
    HQ_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

int hq_ttmc_core(const hq_tensor* t, const double* const* factors, const uint64_t* ranks, double* core_out) {
    return guard([&] {
        require_unsharded(t->t, "hq_ttmc_core");
        cudaStream_t s = t->stream;
        UploadedFactors uf;
        upload_factors(t->t, factors, ranks, uf, s);
        uint64_t size = 1;
        for (int v = 0; v < t->t.order; ++v) size *= ranks[v];
        DBuf<double> core;
        core.alloc(size);
        core_device(t->t, uf, core.get(), s);
        HQ_CUDA(cudaMemcpyAsync(core_out, core.get(), sizeof(double) * size, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
    });
}

int hq_ttmctc(const hq_tensor* t, const double* const* factors, const uint64_t* ranks, int mode, const double* core,
              int variant, double* a_out) {
    (void)variant;
    return guard([&] {
        require_unsharded(t->t, "hq_ttmctc");
        if (mode < 0 || mode >= t->t.order) fail(HQ_ERR_RANGE, "ttmctc: mode out of range");
        cudaStream_t s = t->stream;
        const DeviceTensor& T = t->t;
        UploadedFactors uf;
        upload_factors(T, factors, ranks, uf, s);
        uint64_t size = 1;
        for (int v = 0; v < T.order; ++v) size *= ranks[v];
        DBuf<double> dcore;
        dcore.alloc(size);
        if (core)
            HQ_CUDA(cudaMemcpyAsync(dcore.get(), core, sizeof(double) * size, cudaMemcpyHostToDevice, s));
        else
            core_device(T, uf, dcore.get(), s);
        ModeShape sh = make_mode_shape(T.order, uf.ranks, mode);
        DBuf<double> gt, A;
        gt.alloc(gt_doubles(sh));
        A.alloc(T.dims[mode] * sh.kn);
        launch_gt(dcore.get(), sh, uf.ranks, gt.get(), nullptr, s);
        PassBuffers pb;
        pb.ensure(T.modes[mode], sh);
        PassOut out{A.get(), pb.mpart.get(), pb.wpart.get(), pb.maxpart.get(), pb.ypart.get()};
        launch_pass(T, mode, sh, uf.f, kTTMcTCOnly, gt.get(), out, nullptr, kAlways, s);
        HQ_CUDA(cudaMemcpyAsync(a_out, A.get(), sizeof(double) * T.dims[mode] * sh.kn, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
    });
}

int hq_bench_ttmctc(const hq_tensor* t, const double* const* factors, const uint64_t* ranks, int mode,
                    uint64_t repetitions, double* seconds_out, uint64_t* transient_bytes) {
    return guard([&] {
        require_unsharded(t->t, "hq_bench_ttmctc");
        if (mode < 0 || mode >= t->t.order) fail(HQ_ERR_RANGE, "ttmctc: mode out of range");
        if (repetitions < 1) fail(HQ_ERR_SHAPE, "repetitions must be at least 1");
        cudaStream_t s = t->stream;
        const DeviceTensor& T = t->t;
        UploadedFactors uf;
        upload_factors(T, factors, ranks, uf, s);
        uint64_t size = 1;
        for (int v = 0; v < T.order; ++v) size *= ranks[v];
        DBuf<double> dcore;
        dcore.alloc(size);
        core_device(T, uf, dcore.get(), s);
        ModeShape sh = make_mode_shape(T.order, uf.ranks, mode);
        DBuf<double> gt, A;
        gt.alloc(gt_doubles(sh));
        A.alloc(T.dims[mode] * sh.kn);
        PassBuffers pb;
        pb.ensure(T.modes[mode], sh);
        PassOut out{A.get(), pb.mpart.get(), pb.wpart.get(), pb.maxpart.get(), pb.ypart.get()};
        // per call: G_(n)^T and the fused pass (the kernel a TTMcTC call runs), timed on the device
        cudaEvent_t e0, e1;
        HQ_CUDA(cudaEventCreate(&e0));
        HQ_CUDA(cudaEventCreate(&e1));
        launch_gt(dcore.get(), sh, uf.ranks, gt.get(), nullptr, s);  // warm-up call
        launch_pass(T, mode, sh, uf.f, kTTMcTCOnly, gt.get(), out, nullptr, kAlways, s);
        for (uint64_t r = 0; r < repetitions; ++r) {
            HQ_CUDA(cudaEventRecord(e0, s));
            launch_gt(dcore.get(), sh, uf.ranks, gt.get(), nullptr, s);
            launch_pass(T, mode, sh, uf.f, kTTMcTCOnly, gt.get(), out, nullptr, kAlways, s);
            HQ_CUDA(cudaEventRecord(e1, s));
            HQ_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            HQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            seconds_out[r] = ms * 1e-3;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (transient_bytes) {  // the call's device scratch: A, G^T, partial slots, long-row partials
            const size_t parts[6] = {A.bytes(), gt.bytes(), pb.mpart.bytes(), pb.wpart.bytes(), pb.maxpart.bytes(),
                                     pb.ypart.bytes()};
            transient_bytes[0] = transient_bytes[1] = 0;
            for (size_t b : parts) {
                transient_bytes[0] += b;
                transient_bytes[1] = std::max<uint64_t>(transient_bytes[1], b);
            }
        }
    });
}

// harness.cpp:62-98 gen_synthetic: nnz distinct uniform coordinates (rejection
// of duplicates), standard-normal values, one tucker::Rng stream (rng.hpp)
int hq_gen_synthetic(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed, uint32_t* coords_out,
                     double* values_out) {
    return guard([&] {
        if (order < 1) fail(HQ_ERR_SHAPE, "gen_synthetic: need at least one mode");
        unsigned __int128 total = 1;
        for (int m = 0; m < order; ++m) {
            if (dims[m] == 0) fail(HQ_ERR_SHAPE, "gen_synthetic: zero extent");
            total *= dims[m];
        }
        if ((unsigned __int128)nnz > total)
            fail(HQ_ERR_INFEASIBLE, "gen_synthetic: nnz " + std::to_string(nnz) + " exceeds the number of cells");
        std::mt19937_64 gen(seed);
        bool has_spare = false;
        double spare = 0.0;
        auto uniform01 = [&] { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
        auto normal = [&] {
            if (has_spare) {
                has_spare = false;
                return spare;
            }
            const double u1 = 1.0 - uniform01(), u2 = uniform01();
            const double r = std::sqrt(-2.0 * std::log(u1));
            const double theta = 6.283185307179586476925286766559 * u2;
            spare = r * std::sin(theta);
            has_spare = true;
            return r * std::cos(theta);
        };
        auto uniform_below = [&](uint64_t n) -> uint64_t {
            if (n <= 1) return 0;
            const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
            uint64_t x;
            do {
                x = gen();
            } while (x >= limit);
            return x % n;
        };
        struct KeyHash {
            size_t operator()(const std::pair<uint64_t, uint64_t>& k) const {
                return std::hash<uint64_t>()(k.first * 0x9E3779B97F4A7C15ull ^ k.second);
            }
        };
        std::unordered_set<std::pair<uint64_t, uint64_t>, KeyHash> seen;
        seen.reserve(nnz * 2);
        std::vector<uint32_t> tuple(order);
        uint64_t have = 0;
        while (have < nnz) {
            unsigned __int128 linear = 0;
            for (int m = 0; m < order; ++m) {
                tuple[m] = static_cast<uint32_t>(uniform_below(dims[m]));
                linear = linear * dims[m] + tuple[m];
            }
            if (!seen.insert({(uint64_t)(linear >> 64), (uint64_t)linear}).second) continue;  // duplicate: resample
            for (int m = 0; m < order; ++m) coords_out[have * order + m] = tuple[m];
            values_out[have] = normal();
            ++have;
        }
    });
}

// ------------------------------------------------------------ desk-scale --
int hq_densify_unfold(const hq_tensor* t, int mode, uint64_t capacity_cap, double* out) {
    return guard([&] {
        require_unsharded(t->t, "hq_densify_unfold");
        DBuf<double> d;
        densify_unfold_dev(t->t, mode, capacity_cap, d, t->stream);
        const uint64_t n = t->t.dims[mode] * densify_cols(t->t, mode);
        HQ_CUDA(cudaMemcpyAsync(out, d.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, t->stream));
        HQ_CUDA(cudaStreamSynchronize(t->stream));
    });
}

int hq_ttmc_unfold_dense(const hq_tensor* t, const double* const* factors, const uint64_t* ranks, int mode,
                         uint64_t capacity_cap, double* out) {
    return guard([&] {
        require_unsharded(t->t, "hq_ttmc_unfold_dense");
        if (mode < 0 || mode >= t->t.order) fail(HQ_ERR_RANGE, "ttmc_unfold_dense: mode out of range");
        UploadedFactors uf;
        upload_factors(t->t, factors, ranks, uf, t->stream);
        DBuf<double> y;
        ttmc_unfold_dense_dev(t->t, mode, uf.f, uf.ranks, capacity_cap, y, t->stream);
        ModeShape sh = make_mode_shape(t->t.order, uf.ranks, mode);
        HQ_CUDA(cudaMemcpyAsync(out, y.get(), sizeof(double) * t->t.dims[mode] * sh.L, cudaMemcpyDeviceToHost,
                                t->stream));
        HQ_CUDA(cudaStreamSynchronize(t->stream));
    });
}

int hq_svd_leading(uint64_t rows, uint64_t cols, const double* y, uint64_t k, double* u_out) {
    return guard([&] {
        if (k > std::min(rows, cols)) fail(HQ_ERR_SHAPE, "svd_leading: k exceeds min(rows, cols)");
        if (k == 0) return;
        check_rank_limits((int)k);
        cudaStream_t s = nullptr;
        DBuf<double> Y, U;
        Y.alloc(rows * cols);
        U.alloc(rows * k);
        HQ_CUDA(cudaMemcpyAsync(Y.get(), y, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, s));
        svd_leading_dev(Y.get(), rows, cols, (int)k, U.get(), s);
        HQ_CUDA(cudaMemcpyAsync(u_out, U.get(), sizeof(double) * rows * k, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
    });
}

int hq_sym_eig(uint64_t n, const double* m, double* values_desc, double* vectors) {
    return guard([&] { sym_eig_host(n, m, values_desc, vectors, nullptr); });
}

int hq_init_factors(const hq_tensor* t, const hq_config* cfg, double* const* factors_out) {
    return guard([&] {
        require_unsharded(t->t, "hq_init_factors");
        const DeviceTensor& T = t->t;
        if (cfg->order != T.order) fail(HQ_ERR_SHAPE, "rank count does not match tensor order");
        DBuf<double> U[kMaxOrder];
        double* up[kMaxOrder];
        for (int v = 0; v < T.order; ++v) {
            if (cfg->ranks[v] < 1 || cfg->ranks[v] > T.dims[v])
                fail(HQ_ERR_SHAPE, "rank for mode " + std::to_string(v + 1) + " must lie in [1, " +
                                       std::to_string(T.dims[v]) + "]");
            check_rank_limits((int)cfg->ranks[v]);
            U[v].alloc(T.dims[v] * cfg->ranks[v]);
            up[v] = U[v].get();
        }
        init_factors_dev(T, *cfg, nullptr, up, t->stream);
        for (int v = 0; v < T.order; ++v)
            HQ_CUDA(cudaMemcpyAsync(factors_out[v], up[v], sizeof(double) * T.dims[v] * cfg->ranks[v],
                                    cudaMemcpyDeviceToHost, t->stream));
        HQ_CUDA(cudaStreamSynchronize(t->stream));
    });
}

int hq_hooi(const hq_tensor* t, const hq_config* cfg, const double* const* init_factors, double* const* factors_out,
            double* core_out, hq_trace* trace) {
    return guard([&] {
        require_unsharded(t->t, "hq_hooi");
        if (cfg->order != t->t.order) fail(HQ_ERR_SHAPE, "rank count does not match tensor order");
        hq_config c = *cfg;
        if (init_factors) c.init = 2;
        hooi_solve(t->t, c, init_factors, factors_out, core_out, trace, t->stream);
    });
}

int hq_qr_orthonormal(uint64_t rows, uint64_t cols, const double* a, double* q_out) {
    return guard([&] {
        if (rows < cols) fail(HQ_ERR_SHAPE, "qr_orthonormal: need rows >= cols");
        if (cols == 0) return;
        check_rank_limits((int)cols);
        cudaStream_t s = nullptr;
        DBuf<double> A, Q;
        A.alloc(rows * cols);
        Q.alloc(rows * cols);
        HQ_CUDA(cudaMemcpyAsync(A.get(), a, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, s));
        QrWork w;
        qr_device(A.get(), rows, (int)cols, Q.get(), w, s);
        HQ_CUDA(cudaMemcpyAsync(q_out, Q.get(), sizeof(double) * rows * cols, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
    });
}

int hq_subspace_distance(uint64_t rows, uint64_t cols, const double* u, const double* v, double* out) {
    return guard([&] {
        if (cols == 0) {
            *out = 0.0;
            return;
        }
        check_rank_limits((int)cols);
        cudaStream_t s = nullptr;
        DBuf<double> U, V, pp, d, obj, fit, fp;
        DBuf<DevStatus> st;
        U.alloc(rows * cols);
        V.alloc(rows * cols);
        pp.alloc((size_t)dense_slots() * cols * cols);
        d.alloc(1);
        obj.alloc(1);
        fit.alloc(1);
        fp.alloc(1);
        st.alloc(1);
        HQ_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(DevStatus), s));
        HQ_CUDA(cudaMemcpyAsync(U.get(), u, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, s));
        HQ_CUDA(cudaMemcpyAsync(V.get(), v, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, s));
        launch_apply(nullptr, rows, (int)cols, nullptr, U.get(), V.get(), pp.get(), false, nullptr, kAlways, s);
        SweepTrace tr{obj.get(), fit.get(), d.get(), fp.get(), nullptr, 1, 0.0, nullptr};
        launch_drift(pp.get(), dense_slots(), (int)cols, nullptr, 0, 0.0, 1, 0, false, 0.0, 1, tr, st.get(), s);
        HQ_CUDA(cudaMemcpyAsync(out, d.get(), 8, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
    });
}

int hq_random_factors(int order, const uint64_t* dims, const uint64_t* ranks, uint64_t seed,
                      double* const* factors_out) {
    return guard([&] {
        cudaStream_t s = nullptr;
        QrWork w;
        for (int v = 0; v < order; ++v) {
            if (ranks[v] > dims[v]) fail(HQ_ERR_SHAPE, "qr_orthonormal: need rows >= cols");
            if (ranks[v] == 0) continue;
            check_rank_limits((int)ranks[v]);
            std::vector<double> g(dims[v] * ranks[v]);
            gaussian_stream(mix_seed(seed, (uint64_t)v), g.size(), g.data());
            DBuf<double> A, Q;
            A.alloc(g.size());
            Q.alloc(g.size());
            HQ_CUDA(cudaMemcpyAsync(A.get(), g.data(), sizeof(double) * g.size(), cudaMemcpyHostToDevice, s));
            qr_device(A.get(), dims[v], (int)ranks[v], Q.get(), w, s);
            HQ_CUDA(cudaMemcpyAsync(factors_out[v], Q.get(), sizeof(double) * g.size(), cudaMemcpyDeviceToHost, s));
            HQ_CUDA(cudaStreamSynchronize(s));
        }
    });
}

void hq_config_default(hq_config* cfg) {
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->max_sweeps = 100;
    cfg->tol_fit_change = 1e-12;
    cfg->capacity_cap = 1ull << 31;  // kernels.hpp:62
}

int hq_solver_create(const hq_tensor* t, const hq_config* cfg, const double* const* init_factors, void* stream,
                     hq_solver** out) {
    return guard([&] {
        require_unsharded(t->t, "hq_solver_create");
        auto h = std::make_unique<hq_solver>();
        h->impl = std::make_unique<Solver>();
        cudaStream_t s = stream ? as_stream(stream) : t->stream;
        h->impl->setup(&t->t, cfg, init_factors, s);
        *out = h.release();
    });
}

int hq_release_cached_memory(uint64_t* freed_bytes) {
    return guard([&] {
        HQ_CUDA(cudaDeviceSynchronize());
        const size_t f = device_cache().release_all();
        if (freed_bytes) *freed_bytes = (uint64_t)f;
    });
}

// debug: per-phase cycle counters of the specialised pass (zeros unless built
// with -DHQ_PHASE_TIMING); not part of the public header
int hq_debug_phase_cycles(unsigned long long* out16, int reset) {
    return guard([&] { debug_phase_cycles(out16, reset); });
}

int hq_debug_fib_phase_cycles(unsigned long long* out16, int reset) {
    return guard([&] { debug_fib_phase_cycles(out16, reset); });
}

int hq_nccl_unique_id(uint8_t* id_out) {
    return guard([&] { nccl_unique_id(id_out); });
}

int hq_comm_create(int world, int rank, const uint8_t* id, hq_comm** out) {
    return guard([&] {
        auto c = std::make_unique<hq_comm>();
        c->impl = comm_create(world, rank, id);
        *out = c.release();
    });
}

int hq_comm_create_host(int world, int rank, const char* name, uint64_t capacity, hq_comm** out) {
    return guard([&] {
        auto c = std::make_unique<hq_comm>();
        c->impl = comm_create_host(world, rank, name, capacity);
        *out = c.release();
    });
}

int hq_tensor_shard(hq_tensor* t, const hq_comm* comm) {
    return guard([&] {
        if (!comm) fail(HQ_ERR_SHAPE, "hq_tensor_shard: null communicator");
        shard_tensor(t->t, comm->impl->world, comm->impl->rank, t->stream);
    });
}

int hq_comm_destroy(hq_comm* c) {
    return guard([&] { delete c; });
}

int hq_partition_rows(const uint64_t* offsets, uint64_t rows, int world, uint64_t* bounds) {
    return guard([&] {
        if (world < 1) fail(HQ_ERR_SHAPE, "world size must be positive");
        partition_rows(offsets, rows, world, bounds);
    });
}

int hq_solver_create_dist(const hq_tensor* t, const hq_config* cfg, const double* const* init_factors, void* stream,
                          const hq_comm* comm, hq_solver** out) {
    return guard([&] {
        auto h = std::make_unique<hq_solver>();
        h->impl = std::make_unique<Solver>();
        cudaStream_t s = stream ? as_stream(stream) : t->stream;
        h->impl->setup(&t->t, cfg, init_factors, s, comm ? comm->impl : nullptr);
        *out = h.release();
    });
}

int hq_solver_destroy(hq_solver* s) {
    return guard([&] { delete s; });
}

int hq_solver_run(hq_solver* s, uint64_t sweeps) {
    return guard([&] { s->impl->run(sweeps); });
}

int hq_solver_sync(hq_solver* s) {
    return guard([&] {
        s->impl->settle();
        s->impl->check_status(s->impl->status());
    });
}

int hq_solver_launch_mode_pass(hq_solver* sv, int mode) {
    return guard([&] {
        Solver& S = *sv->impl;
        if (mode < 0 || mode >= S.N) fail(HQ_ERR_RANGE, "mode out of range");
        FactorPtrs f = S.factors_for_mode(mode, S.host_parity);
        launch_pass(*S.T, mode, S.sh[mode], f, kTTMcTC, S.gt.get(), S.pass_out(S.A.get()), nullptr, kAlways, S.s,
                    S.rb(mode), S.re(mode));
    });
}

// the standalone TTMcTC (kernels.cpp:86-163 with precomputed_core): A = Y_(n) G_(n)^T only
int hq_solver_launch_ttmctc(hq_solver* sv, int mode) {
    return guard([&] {
        Solver& S = *sv->impl;
        if (mode < 0 || mode >= S.N) fail(HQ_ERR_RANGE, "mode out of range");
        FactorPtrs f = S.factors_for_mode(mode, S.host_parity);
        launch_gt(S.core.get(), S.sh[mode], S.ranks, S.gt.get(), nullptr, S.s);  // G_(n)^T of the current core
        launch_pass(*S.T, mode, S.sh[mode], f, kTTMcTCOnly, S.gt.get(), S.pass_out(S.A.get()), nullptr, kAlways,
                    S.s, S.rb(mode), S.re(mode));
    });
}

int hq_solver_status(hq_solver* s, int64_t* out) {
    return guard([&] {
        DevStatus h = s->impl->status();
        out[0] = h.sweep;
        out[1] = h.fallback_count;
        out[2] = h.abort;
        out[3] = h.degenerate_mode;
        out[4] = h.shifted_count;
        out[5] = h.dist_hh_count;
        out[6] = s->impl->peer_apply ? 1 : 0;
        out[7] = 0;
    });
}

int hq_solver_launches_per_sweep(const hq_solver* s, uint64_t* out) {
    return guard([&] { *out = (uint64_t)s->impl->launches_per_sweep(); });
}

int hq_solver_download(hq_solver* s, double* const* factors_out, double* core_out, hq_trace* trace) {
    return guard([&] { s->impl->download(factors_out, core_out, trace); });
}

int hq_solver_mode_pass_work(const hq_solver* sv, int mode, double* flops, double* bytes) {
    return guard([&] {
        const Solver& S = *sv->impl;
        const ModeShape& m = S.sh[mode];
        const ModeLayout& L = S.T->modes[mode];
        double nnz = (double)S.T->nnz, R = (double)L.nonempty_rows;
        // kron rows (L per nonzero, built as (L/K_last) products + L FMAs),
        // a_i = Y_i G^T, M += a_i^T Y_i, W += a_i^T a_i
        *flops = 2.0 * nnz * m.L + 2.0 * R * m.L * m.kn * 2.0 + 2.0 * R * m.kn * m.kn;
        double fb = 0.0;
        for (int v = 0; v < S.N; ++v)
            if (v != mode) fb += 8.0 * (double)S.dims[v] * S.ranks[v];
        *bytes = nnz * (4.0 * (S.N - 1) + 8.0) + 8.0 * (double)(L.rows + 1) + fb + 8.0 * (double)S.dims[mode] * m.kn;
    });
}

int hq_solver_ttmctc_work(const hq_solver* sv, int mode, double* flops, double* bytes) {
    return guard([&] {
        const Solver& S = *sv->impl;
        const ModeShape& m = S.sh[mode];
        const ModeLayout& L = S.T->modes[mode];
        double nnz = (double)S.T->nnz, R = (double)L.nonempty_rows;
        // F = 2 nnz prod_{v!=n} K_v + 2 R_n prod_v K_v
        *flops = 2.0 * nnz * m.L + 2.0 * R * m.L * m.kn;
        double fb = 0.0;
        for (int v = 0; v < S.N; ++v)
            if (v != mode) fb += 8.0 * (double)S.dims[v] * S.ranks[v];
        // B = nnz (4N + 8) + 8 sum_{v!=n} I_v K_v + 8 I_n K_n
        *bytes = nnz * (4.0 * S.N + 8.0) + fb + 8.0 * (double)S.dims[mode] * m.kn;
    });
}

int hq_hoqri(const hq_tensor* t, const hq_config* cfg, const double* const* init_factors, double* const* factors_out,
             double* core_out, hq_trace* trace) {
    return guard([&] {
        require_unsharded(t->t, "hq_hoqri");
        Solver S;
        S.setup(&t->t, cfg, init_factors, t->stream);
        S.solve();
        S.download(factors_out, core_out, trace);
    });
}

int hq_fit_error(double data_norm_sq, uint64_t core_size, const double* core, double* out) {
    return guard([&] {  // solvers.cpp:225-236
        double f = 0.0;
        for (uint64_t i = 0; i < core_size; ++i) f += core[i] * core[i];
        double r = data_norm_sq - f;
        double scale = std::max(1.0, data_norm_sq);
        if (r < -1e-8 * scale)
            fail(HQ_ERR_CONTRACT,
                 "fit_error: core energy exceeds the data norm; core is inconsistent with the factors");
        *out = (std::fabs(r) <= 1e-10 * scale) ? 0.0 : std::max(r, 0.0);
    });
}

}  // extern "C"
