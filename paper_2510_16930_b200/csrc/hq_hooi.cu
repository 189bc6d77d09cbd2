// hq_hooi.cu — desk-scale dense paths of the reference, on the device
// (SURVEY 8(f) rank 4): HOSVD initialisation and HOOI.
//
//   densify_unfold      (kernels.cpp:326-348)  X_(n) dense, one store per merged entry
//   ttmc_unfold_dense   (kernels.cpp:264-324)  Y_(n) = X_(n) (x) U_v dense, one warp per row
//   svd_leading         (dense_core.cpp:266-327) leading K left singular vectors from the
//                       eigenvectors of the smaller Gram matrix (cuSOLVER syevd; Gram by
//                       cuBLAS DGEMM); the rank-deficient fill uses the reference's stream
//                       Rng(0x48514F5251 ^ 0x5544); the final Gram-Schmidt pass is the
//                       device qr_orthonormal (same Q for a full-rank input)
//   init_factors HOSVD  (solvers.cpp:202-215)
//   hooi                (solvers.cpp:93-122, 152-178) host-sequenced, every step on the device
//
// Both dense unfoldings are capacity-capped exactly like the reference
// (rows > cap / cols -> CapacityError).  These paths are not the HOQRI hot
// path; the eigen-solver is a library call, so eigenvector signs (and the basis
// inside a repeated eigenvalue) may differ from the reference's cyclic Jacobi:
// results agree as subspaces (tests compare subspace distance, f and fit).
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "hq_dense.cuh"
#include "hq_hooi.cuh"

namespace hq {

namespace {

struct DenseLib {
    cublasHandle_t blas = nullptr;
    cusolverDnHandle_t sol = nullptr;
};

DenseLib& dense_lib(cudaStream_t s) {
    static std::mutex mu;
    static std::map<int, DenseLib> libs;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    HQ_CUDA(cudaGetDevice(&dev));
    DenseLib& d = libs[dev];
    if (!d.blas && cublasCreate(&d.blas) != CUBLAS_STATUS_SUCCESS) fail(HQ_ERR_CUDA, "cublasCreate failed");
    if (!d.sol && cusolverDnCreate(&d.sol) != CUSOLVER_STATUS_SUCCESS) fail(HQ_ERR_CUDA, "cusolverDnCreate failed");
    cublasSetStream(d.blas, s);
    cusolverDnSetStream(d.sol, s);
    return d;
}

// row-major C (M x N) = op(A) op(B): the column-major call on the transposes
void gemm_rm(cudaStream_t s, bool ta, bool tb, int M, int N, int K, const double* A, int lda, const double* B, int ldb,
             double* C, int ldc) {
    const double one = 1.0, zero = 0.0;
    DenseLib& d = dense_lib(s);
    if (cublasDgemm(d.blas, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, N, M, K, &one, B, ldb, A,
                    lda, &zero, C, ldc) != CUBLAS_STATUS_SUCCESS)
        fail(HQ_ERR_CUDA, "cublasDgemm failed");
}

__global__ void k_densify(const uint32_t* __restrict__ coords, const double* __restrict__ vals, uint64_t nnz,
                          int order, int mode, const uint64_t* __restrict__ stride, uint64_t ncols, double* out) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz; e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t col = 0;
        for (int v = 0; v < order; ++v)
            if (v != mode) col += (uint64_t)coords[e * order + v] * stride[v];
        out[(uint64_t)coords[e * order + mode] * ncols + col] += vals[e];  // merged entries: one writer per cell
    }
}

struct UnfoldArgs {
    const int64_t* rowptr;
    const double* val;
    const uint32_t* idx[kMaxOrder - 1];
    const double* u[kMaxOrder - 1];
    ModeShape sh;
    uint64_t rows;
};

// Y_i[l] = sum_e x_e prod_j U_j[idx_j(e)][digit_j(l)], nonzeros of row i in stream order
__global__ void k_unfold_dense(UnfoldArgs a, double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int L = a.sh.L;
    for (uint64_t i = warp; i < a.rows; i += nw) {
        const int64_t b = a.rowptr[i], e1 = a.rowptr[i + 1];
        for (int l = lane; l < L; l += 32) {
            int dig[kMaxOrder - 1];
            for (int j = 0; j < a.sh.nothers; ++j) dig[j] = (l / a.sh.cstride[j]) % a.sh.ko[j];
            double acc = 0.0;
            for (int64_t p = b; p < e1; ++p) {
                double t = a.val[p];
                for (int j = 0; j < a.sh.nothers; ++j) t *= a.u[j][(size_t)a.idx[j][p] * a.sh.ko[j] + dig[j]];
                acc += t;
            }
            y[i * (uint64_t)L + l] = acc;
        }
    }
}

__global__ void k_scale_col(double* u, uint64_t m, int k, int j, double inv) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        u[i * k + j] *= inv;
}

// jacobi_eig_sym symmetrises its input first (dense_core.cpp:204-210)
__global__ void k_symmetrize(double* m, uint64_t n) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n * n; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = t / n, j = t % n;
        if (j <= i) continue;
        const double avg = 0.5 * (m[i * n + j] + m[j * n + i]);
        m[i * n + j] = avg;
        m[j * n + i] = avg;
    }
}

__global__ void k_max_abs(const double* __restrict__ v, uint64_t n, double* out) {
    __shared__ double red[32];
    double m = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs(v[i]));
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) out[blockIdx.x] = m;
    }
}

int grid_for(uint64_t n) { return (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, num_sms() * 8)); }

void check_capacity(uint64_t rows, uint64_t cols, uint64_t cap) {  // kernels.cpp:275-279, 331-335
    if (cols != 0 && rows > cap / cols)
        fail(HQ_ERR_CAPACITY, "dense unfolding of " + std::to_string(rows) + " x " + std::to_string(cols) +
                                  " exceeds the capacity cap; this path is desk-scale only");
}

}  // namespace

double max_abs_dev(const double* v, uint64_t n, cudaStream_t s) {
    const int g = grid_for(n);
    DBuf<double> part;
    part.alloc(g);
    k_max_abs<<<g, 256, 0, s>>>(v, n, part.get());
    HQ_CHECK_LAUNCH();
    std::vector<double> h(g);
    HQ_CUDA(cudaMemcpyAsync(h.data(), part.get(), sizeof(double) * g, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    double m = 0.0;
    for (double x : h) m = std::max(m, x);
    return m;
}

uint64_t densify_cols(const DeviceTensor& T, int mode) {
    uint64_t c = 1;
    for (int v = 0; v < T.order; ++v)
        if (v != mode) {
            if (T.dims[v] && c > UINT64_MAX / T.dims[v]) fail(HQ_ERR_CAPACITY, "dense unfolding size overflows");
            c *= T.dims[v];
        }
    return c;
}

void densify_unfold_dev(const DeviceTensor& T, int mode, uint64_t cap, DBuf<double>& out, cudaStream_t s) {
    if (mode < 0 || mode >= T.order) fail(HQ_ERR_RANGE, "densify_unfold: mode out of range");
    const uint64_t rows = T.dims[mode], cols = densify_cols(T, mode);
    check_capacity(rows, cols, cap);
    std::vector<uint64_t> stride(T.order, 0);  // unfold_col_strides(dims, mode): last other mode fastest
    uint64_t acc = 1;
    for (int v = T.order - 1; v >= 0; --v)
        if (v != mode) {
            stride[v] = acc;
            acc *= T.dims[v];
        }
    DBuf<uint64_t> dstride;
    dstride.alloc(T.order);
    HQ_CUDA(cudaMemcpyAsync(dstride.get(), stride.data(), 8 * T.order, cudaMemcpyHostToDevice, s));
    out.alloc(std::max<uint64_t>(1, rows * cols));
    HQ_CUDA(cudaMemsetAsync(out.get(), 0, sizeof(double) * rows * cols, s));
    if (T.nnz) {
        k_densify<<<grid_for(T.nnz), 256, 0, s>>>(T.coords.get(), T.vals.get(), T.nnz, T.order, mode, dstride.get(), cols,
                                                  out.get());
        HQ_CHECK_LAUNCH();
    }
    HQ_CUDA(cudaStreamSynchronize(s));
}

void ttmc_unfold_dense_dev(const DeviceTensor& T, int mode, const FactorPtrs& f, const int* ranks, uint64_t cap,
                           DBuf<double>& y, cudaStream_t s) {
    if (mode < 0 || mode >= T.order) fail(HQ_ERR_RANGE, "ttmc_unfold_dense: mode out of range");
    ModeShape sh = make_mode_shape(T.order, ranks, mode);
    const uint64_t rows = T.dims[mode];
    check_capacity(rows, (uint64_t)sh.L, cap);
    const ModeLayout& L = T.modes[mode];
    UnfoldArgs a{};
    a.rowptr = L.rowptr.get();
    a.val = L.val.get();
    for (int j = 0; j < sh.nothers; ++j) {
        a.idx[j] = L.idx[j].get();
        a.u[j] = f.u[L.others[j]];
    }
    a.sh = sh;
    a.rows = rows;
    y.alloc(std::max<uint64_t>(1, rows * (uint64_t)sh.L));
    if (rows) {
        const int blocks = (int)std::max<uint64_t>(1, std::min<uint64_t>((rows + 7) / 8, num_sms() * 16));
        k_unfold_dense<<<blocks, 256, 0, s>>>(a, y.get());
        HQ_CHECK_LAUNCH();
    }
    HQ_CUDA(cudaStreamSynchronize(s));
}

void svd_leading_dev(const double* y, uint64_t m, uint64_t p, int k, double* u_out, cudaStream_t s) {
    if ((uint64_t)k > std::min(m, p)) fail(HQ_ERR_SHAPE, "svd_leading: k exceeds min(rows, cols)");
    if (k == 0) return;
    const uint64_t n = std::min(m, p);
    if (n > 46340) fail(HQ_ERR_CAPACITY, "svd_leading: Gram side above the dense eigen-solver limit");
    DenseLib& d = dense_lib(s);
    DBuf<double> g, w;
    g.alloc(n * n);
    w.alloc(n);
    if (m <= p)
        gemm_rm(s, false, true, (int)m, (int)m, (int)p, y, (int)p, y, (int)p, g.get(), (int)m);  // Y Y^T
    else
        gemm_rm(s, true, false, (int)p, (int)p, (int)m, y, (int)p, y, (int)p, g.get(), (int)p);  // Y^T Y
    int lwork = 0;
    if (cusolverDnDsyevd_bufferSize(d.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, g.get(), (int)n,
                                    w.get(), &lwork) != CUSOLVER_STATUS_SUCCESS)
        fail(HQ_ERR_CUDA, "cusolverDnDsyevd_bufferSize failed");
    DBuf<double> work;
    work.alloc(std::max(1, lwork));
    DBuf<int> info;
    info.alloc(1);
    if (cusolverDnDsyevd(d.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, g.get(), (int)n, w.get(),
                         work.get(), lwork, info.get()) != CUSOLVER_STATUS_SUCCESS)
        fail(HQ_ERR_CUDA, "cusolverDnDsyevd failed");
    int hinfo = 0;
    HQ_CUDA(cudaMemcpyAsync(&hinfo, info.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    if (hinfo != 0) fail(HQ_ERR_DIAGNOSTIC, "svd_leading: the symmetric eigen-solver did not converge");
    // eigenvalues ascending, eigenvector j = column j of g (column-major): descending order = n-1-j
    if (m <= p) {  // dense_core.cpp:272-278: U = leading eigenvectors of Y Y^T
        for (int j = 0; j < k; ++j)
            HQ_CUDA(cudaMemcpy2DAsync(u_out + j, sizeof(double) * k, g.get() + (n - 1 - j) * n, sizeof(double),
                                      sizeof(double), m, cudaMemcpyDeviceToDevice, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        return;
    }
    // dense_core.cpp:280-326: V_k (p x k) -> U = Y V_k / sigma, deficient columns filled, then Gram-Schmidt
    std::vector<double> lam(n);
    HQ_CUDA(cudaMemcpyAsync(lam.data(), w.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    DBuf<double> vk, uu;
    vk.alloc(p * k);
    uu.alloc(m * k);
    for (int j = 0; j < k; ++j)
        HQ_CUDA(cudaMemcpy2DAsync(vk.get() + j, sizeof(double) * k, g.get() + (n - 1 - j) * n, sizeof(double),
                                  sizeof(double), p, cudaMemcpyDeviceToDevice, s));
    gemm_rm(s, false, false, (int)m, k, (int)p, y, (int)p, vk.get(), k, uu.get(), k);
    HQ_CUDA(cudaStreamSynchronize(s));
    const double lam_max = std::max(lam[n - 1], 0.0), sigma_max = std::sqrt(lam_max);
    uint64_t drawn = 0;
    for (int j = 0; j < k; ++j) {
        const double sigma = std::sqrt(std::max(lam[n - 1 - j], 0.0));
        if (sigma > 1e-12 * (sigma_max > 0.0 ? sigma_max : 1.0)) {
            k_scale_col<<<grid_for(m), 256, 0, s>>>(uu.get(), m, k, j, 1.0 / sigma);
            HQ_CHECK_LAUNCH();
        } else {  // the reference's deficiency stream, continued across deficient columns
            std::vector<double> all(drawn + m);
            gaussian_stream(0x48514F5251ull ^ 0x5544ull, drawn + m, all.data());
            HQ_CUDA(cudaMemcpy2DAsync(uu.get() + j, sizeof(double) * k, all.data() + drawn, sizeof(double),
                                      sizeof(double), m, cudaMemcpyHostToDevice, s));
            HQ_CUDA(cudaStreamSynchronize(s));
            drawn += m;
        }
    }
    QrWork qw;
    qr_device(uu.get(), m, k, u_out, qw, s);
}

void sym_eig_host(uint64_t n, const double* m, double* values_desc, double* vectors, cudaStream_t s) {
    if (n == 0) return;
    if (n > 46340) fail(HQ_ERR_CAPACITY, "sym_eig: matrix above the dense eigen-solver limit");
    DenseLib& d = dense_lib(s);
    DBuf<double> g, w;
    g.alloc(n * n);
    w.alloc(n);
    HQ_CUDA(cudaMemcpyAsync(g.get(), m, sizeof(double) * n * n, cudaMemcpyHostToDevice, s));
    k_symmetrize<<<grid_for(n * n), 256, 0, s>>>(g.get(), n);
    HQ_CHECK_LAUNCH();
    int lwork = 0;
    if (cusolverDnDsyevd_bufferSize(d.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, g.get(), (int)n,
                                    w.get(), &lwork) != CUSOLVER_STATUS_SUCCESS)
        fail(HQ_ERR_CUDA, "cusolverDnDsyevd_bufferSize failed");
    DBuf<double> work;
    work.alloc(std::max(1, lwork));
    DBuf<int> info;
    info.alloc(1);
    if (cusolverDnDsyevd(d.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, g.get(), (int)n, w.get(),
                         work.get(), lwork, info.get()) != CUSOLVER_STATUS_SUCCESS)
        fail(HQ_ERR_CUDA, "cusolverDnDsyevd failed");
    std::vector<double> lam(n), vec(n * n);
    int hinfo = 0;
    HQ_CUDA(cudaMemcpyAsync(&hinfo, info.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaMemcpyAsync(lam.data(), w.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaMemcpyAsync(vec.data(), g.get(), sizeof(double) * n * n, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    if (hinfo != 0) fail(HQ_ERR_DIAGNOSTIC, "sym_eig: the symmetric eigen-solver did not converge");
    // ascending pairs, vector j = column j (column-major) -> descending, vectors as row-major columns
    for (uint64_t j = 0; j < n; ++j) {
        const uint64_t src = n - 1 - j;
        values_desc[j] = lam[src];
        if (vectors)
            for (uint64_t i = 0; i < n; ++i) vectors[i * n + j] = vec[src * n + i];
    }
}

void hosvd_init_dev(const DeviceTensor& T, const int* ranks, uint64_t cap, double* const* U, cudaStream_t s) {
    for (int n = 0; n < T.order; ++n) {  // solvers.cpp:202-215
        DBuf<double> xn;
        try {
            densify_unfold_dev(T, n, cap, xn, s);
        } catch (const Error& e) {
            if (e.code != HQ_ERR_CAPACITY) throw;
            fail(HQ_ERR_CAPACITY, std::string(e.what()) + "; HOSVD initialization is desk-scale only, use random init");
        }
        svd_leading_dev(xn.get(), T.dims[n], densify_cols(T, n), ranks[n], U[n], s);
    }
}

namespace {

__global__ void k_set_sweep(DevStatus* st, int sweep) {
    st->sweep = sweep;
    st->abort = 0;
}

double core_norm_sq_dev(const double* core, uint64_t size, cudaStream_t s) {
    DBuf<double> f;
    f.alloc(1);
    launch_core_normsq(core, size, f.get(), s);
    double h = 0.0;
    HQ_CUDA(cudaMemcpyAsync(&h, f.get(), 8, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    return h;
}

}  // namespace

void hooi_solve(const DeviceTensor& T, const hq_config& cfg, const double* const* init_host,
                double* const* factors_out, double* core_out, hq_trace* tr, cudaStream_t s) {
    using Clock = std::chrono::steady_clock;
    const int N = T.order;
    if (cfg.max_sweeps < 1) fail(HQ_ERR_SHAPE, "max_sweeps must be at least 1");
    if (cfg.tol_fit_change < 0.0) fail(HQ_ERR_SHAPE, "tolerance must be nonnegative");
    int ranks[kMaxOrder];
    uint64_t core_size = 1;
    int kmax = 1;
    for (int v = 0; v < N; ++v) {
        ranks[v] = (int)cfg.ranks[v];
        if (ranks[v] < 1 || (uint64_t)ranks[v] > T.dims[v])
            fail(HQ_ERR_SHAPE, "rank for mode " + std::to_string(v + 1) + " must lie in [1, " +
                                   std::to_string(T.dims[v]) + "]");
        check_rank_limits(ranks[v]);
        core_size *= ranks[v];
        kmax = std::max(kmax, ranks[v]);
    }
    const uint64_t cap = cfg.capacity_cap ? cfg.capacity_cap : (1ull << 31);
    const bool tracing = cfg.trace_gradients || cfg.tol_grad > 0.0;
    DBuf<double> U[kMaxOrder], Uold;
    double* up[kMaxOrder];
    uint64_t maxik = 0;
    for (int v = 0; v < N; ++v) {
        U[v].alloc((uint64_t)T.dims[v] * ranks[v]);
        up[v] = U[v].get();
        maxik = std::max<uint64_t>(maxik, (uint64_t)T.dims[v] * ranks[v]);
    }
    Uold.alloc(maxik);
    init_factors_dev(T, cfg, init_host, up, s);
    FactorPtrs f{};
    for (int v = 0; v < N; ++v) {
        f.u[v] = U[v].get();
        f.k[v] = ranks[v];
    }
    const double dns = T.norm_sq;
    DBuf<double> core;
    core.alloc(core_size);
    ttmc_core_dev(T, f, ranks, core.get(), s);
    const double f0 = core_norm_sq_dev(core.get(), core_size, s);
    double fit_prev = dns - f0;
    // per-update diagnostics on the device (k_update_diag), trace kept on the host
    const uint64_t nu = cfg.max_sweeps * (uint64_t)N;
    DBuf<double> dgrad, dfb, dsig, dlam, gt, a, w;
    DBuf<unsigned long long> dt;
    DBuf<DevStatus> st;
    if (tracing) {
        dgrad.alloc(nu);
        dfb.alloc(nu);
        dsig.alloc(nu * kmax);
        dlam.alloc(nu * kmax);
        dt.alloc(nu);
        st.alloc(1);
        HQ_CUDA(cudaMemsetAsync(st.get(), 0, sizeof(DevStatus), s));
    }
    std::vector<double> obj, fit, drift, grad(nu, 0.0), fb(nu, 0.0), fa(nu, 0.0), uel(nu, 0.0), el;
    uint64_t sweeps = 0;
    const auto t0 = Clock::now();
    for (uint64_t sweep = 1; sweep <= cfg.max_sweeps; ++sweep) {
        double total_g = 0.0;
        for (int n = 0; n < N; ++n) {
            const auto tu0 = Clock::now();
            const uint64_t I = T.dims[n];
            const int K = ranks[n];
            DBuf<double> y;
            ttmc_unfold_dense_dev(T, n, f, ranks, cap, y, s);
            ModeShape sh = make_mode_shape(N, ranks, n);
            const int L = sh.L;
            if (max_abs_dev(y.get(), I * (uint64_t)L, s) == 0.0)  // solvers.cpp:98
                fail(HQ_ERR_DEGENERATE,
                     "degenerate state: TTMcTC output is identically zero for mode " + std::to_string(n + 1), n + 1);
            const uint64_t u_idx = (sweep - 1) * N + n;
            if (tracing) {  // solvers.cpp:101-109: G_(n) = U_n^T Y, A = Y G_(n)^T, diagnostics
                gt.alloc((uint64_t)L * K);
                a.alloc(I * K);
                w.alloc((uint64_t)K * K);
                gemm_rm(s, true, false, L, K, (int)I, y.get(), L, U[n].get(), K, gt.get(), K);
                gemm_rm(s, false, false, (int)I, K, L, y.get(), L, gt.get(), K, a.get(), K);
                gemm_rm(s, true, false, K, K, (int)I, a.get(), K, a.get(), K, w.get(), K);
                k_set_sweep<<<1, 1, 0, s>>>(st.get(), (int)sweep - 1);
                UpdTrace ut{dgrad.get(), dfb.get(), dsig.get(), dlam.get(), dt.get(), kmax};
                launch_update_diag(w.get(), gt.get(), K, L, n, N, ut, st.get(), s);
                DevStatus h{};
                HQ_CUDA(cudaMemcpyAsync(&h, st.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
                HQ_CUDA(cudaMemcpyAsync(&grad[u_idx], dgrad.get() + u_idx, 8, cudaMemcpyDeviceToHost, s));
                HQ_CUDA(cudaStreamSynchronize(s));
                if (h.abort == 5 && h.diag_code == 1)
                    fail(HQ_ERR_DIAGNOSTIC, "grad_norm_sq is negative beyond rounding; orthonormality is broken upstream");
                if (h.abort == 5)
                    fail(HQ_ERR_DIAGNOSTIC, "interlacing violated at k=" + std::to_string(h.diag_k) +
                                                "; upstream state is numerically corrupted");
                if (h.abort == 6) fail(HQ_ERR_CONTRACT, "gram_eigvals_desc: matrix is not PSD");
                fb[u_idx] = core_norm_sq_dev(core.get(), core_size, s);  // f_before = ||core||^2 (solvers.cpp:102)
                total_g += grad[u_idx];
            }
            HQ_CUDA(cudaMemcpyAsync(Uold.get(), U[n].get(), sizeof(double) * I * K, cudaMemcpyDeviceToDevice, s));
            svd_leading_dev(y.get(), I, (uint64_t)L, K, U[n].get(), s);  // solvers.cpp:112
            drift.resize(sweep * N, 0.0);
            drift[u_idx] = subspace_distance_dev(U[n].get(), Uold.get(), I, K, s);
            if (tracing) {  // solvers.cpp:115-120
                ttmc_core_dev(T, f, ranks, core.get(), s);
                fa[u_idx] = core_norm_sq_dev(core.get(), core_size, s);
                uel[u_idx] = std::chrono::duration<double>(Clock::now() - tu0).count();
            }
        }
        if (!tracing) ttmc_core_dev(T, f, ranks, core.get(), s);
        const double ob = core_norm_sq_dev(core.get(), core_size, s);
        obj.push_back(ob);
        fit.push_back(dns - ob);
        el.push_back(std::chrono::duration<double>(Clock::now() - t0).count());
        sweeps = sweep;
        if (std::fabs(fit_prev - (dns - ob)) < cfg.tol_fit_change) break;  // solvers.cpp:163-167
        if (cfg.tol_grad > 0.0 && std::sqrt(total_g) <= cfg.tol_grad * std::max(ob, 1e-300)) break;
        fit_prev = dns - ob;
    }
    for (int v = 0; v < N; ++v)  // solvers.cpp:171-172
        if (orthonormality_defect_dev(U[v].get(), T.dims[v], ranks[v], s) > 1e-10)
            fail(HQ_ERR_DIAGNOSTIC, "solver produced factors with orthonormality defect above 1e-10");
    if (factors_out)
        for (int v = 0; v < N; ++v)
            if (factors_out[v])
                HQ_CUDA(cudaMemcpyAsync(factors_out[v], U[v].get(), sizeof(double) * T.dims[v] * ranks[v],
                                        cudaMemcpyDeviceToHost, s));
    if (core_out) HQ_CUDA(cudaMemcpyAsync(core_out, core.get(), sizeof(double) * core_size, cudaMemcpyDeviceToHost, s));
    std::vector<double> sig, lam;
    if (tracing && sweeps) {
        const uint64_t nd = sweeps * N;
        sig.resize(nd * kmax);
        lam.resize(nd * kmax);
        HQ_CUDA(cudaMemcpyAsync(sig.data(), dsig.get(), 8 * nd * kmax, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaMemcpyAsync(lam.data(), dlam.get(), 8 * nd * kmax, cudaMemcpyDeviceToHost, s));
    }
    HQ_CUDA(cudaStreamSynchronize(s));
    if (!tr) return;
    tr->data_norm_sq = dns;
    tr->initial_objective = f0;
    tr->sweeps = sweeps;
    tr->updates = tracing ? sweeps * N : 0;
    for (uint64_t i = 0; i < sweeps; ++i) {
        if (tr->objective) tr->objective[i] = obj[i];
        if (tr->fit) tr->fit[i] = fit[i];
        if (tr->elapsed_s) tr->elapsed_s[i] = el[i];
    }
    for (uint64_t i = 0; i < sweeps * N; ++i) {
        if (tr->drift) tr->drift[i] = drift[i];
        if (tr->grad_norm_sq) tr->grad_norm_sq[i] = grad[i];
        if (!tracing) continue;
        if (tr->upd_f_before) tr->upd_f_before[i] = fb[i];
        if (tr->upd_f_after) tr->upd_f_after[i] = fa[i];
        if (tr->upd_elapsed_s) tr->upd_elapsed_s[i] = uel[i];
        const int K = ranks[i % N];
        for (int k = 0; k < K && (uint64_t)k < tr->sigma_stride; ++k) {
            if (tr->upd_sigma) tr->upd_sigma[i * tr->sigma_stride + k] = sig[i * kmax + k];
            if (tr->upd_lambda) tr->upd_lambda[i * tr->sigma_stride + k] = lam[i * kmax + k];
        }
    }
}

}  // namespace hq
