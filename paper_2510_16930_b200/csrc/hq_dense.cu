// hq_dense.cu — orthogonalisation and K x K steps of a mode update.
//
// The reference orthonormalises A^(n) with Householder QR (R_kk >= 0,
// proj/src/dense_core.cpp:127-198).  The thin QR with positive diag(R) is
// unique, so CholeskyQR2 yields the same Q (to rounding) at a fraction of the
// passes: W = A^T A (fused into the sparse pass), R1 = chol(W),
// W2 = (A R1^-1)^T (A R1^-1), R2 = chol(W2), U = A (R2 R1)^-1.  When the first
// Cholesky shows a column with less than 1e-6 of its norm outside the span of
// the previous ones (kappa too large for CholeskyQR2, or the reference's
// rank-deficient branch, dense_core.cpp:146-157) the device Householder path
// runs instead.
//
// The drift (manifold.cpp:55-60) is 2K - 2 ||U_new^T U_old||_* with the
// nuclear norm from the reference's cyclic Jacobi (dense_core.cpp:200-264,
// 329-335), evaluated on the device by one thread (K x K).
#include <algorithm>
#include <cmath>

#include "hq_dense.cuh"

namespace hq {

int dense_slots() { return num_sms() * 4; }

namespace {


// deterministic block sum (fixed tree)
__device__ double block_sum(double v, double* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
        if (threadIdx.x == 0) red[32] = t;
    }
    __syncthreads();
    return red[32];
}

#include "hq_small.inc"

// ---- Householder fallback (dense_core.cpp:127-198) ------------------------
struct DevRng {
    unsigned long long mt[312];
    int idx;
    int has_spare;
    double spare;
};

__device__ void rng_seed(DevRng* r, unsigned long long seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i) r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + i;
    r->idx = 312;
    r->has_spare = 0;
    r->spare = 0.0;
}

__device__ unsigned long long rng_raw(DevRng* r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            unsigned long long y = (r->mt[i] & 0xFFFFFFFF80000000ull) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            unsigned long long v = r->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1ull) v ^= 0xB5026F5AA96619E9ull;
            r->mt[i] = v;
        }
        r->idx = 0;
    }
    unsigned long long y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= (y >> 43);
    return y;
}

__device__ double rng_normal(DevRng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = 1.0 - (double)(rng_raw(r) >> 11) * 0x1.0p-53;
    double u2 = (double)(rng_raw(r) >> 11) * 0x1.0p-53;
    double rad = sqrt(-2.0 * log(u1));
    double theta = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(theta);
    r->has_spare = 1;
    return rad * cos(theta);
}

constexpr int kHhThreads = 1024;

__global__ void __launch_bounds__(kHhThreads) k_householder(const double* __restrict__ A, uint64_t m, int n,
                                                            double* __restrict__ q, double* __restrict__ work,
                                                            const DevStatus* st, int run_if) {
    if (skip_kernel(st, run_if)) return;
    __shared__ DevRng rng;
    __shared__ double red[33];
    __shared__ double betas[kMaxRank];
    __shared__ int flip[kMaxRank];
    double* w = work;                       // m x n
    double* refl = work + m * (uint64_t)n;  // n reflectors of length m
    const uint64_t tid = threadIdx.x, nt = blockDim.x;
    double part = 0.0;
    for (uint64_t i = tid; i < m * (uint64_t)n; i += nt) {
        double v = A[i];
        w[i] = v;
        part += v * v;
    }
    const double anorm = sqrt(block_sum(part, red));
    const double pivot_tol = 1e-12 * anorm;
    if (tid == 0) rng_seed(&rng, 0x48514F5251ull);
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        part = 0.0;
        for (uint64_t i = k + tid; i < m; i += nt) part += w[i * n + k] * w[i * n + k];
        double normx = sqrt(block_sum(part, red));
        if (normx <= pivot_tol) {
            do {
                if (tid == 0)
                    for (uint64_t i = k; i < m; ++i) w[i * n + k] = rng_normal(&rng);
                __syncthreads();
                part = 0.0;
                for (uint64_t i = k + tid; i < m; i += nt) part += w[i * n + k] * w[i * n + k];
                normx = sqrt(block_sum(part, red));
            } while (normx == 0.0);
        }
        const double x0 = w[(uint64_t)k * n + k];
        const double alpha = (x0 >= 0.0) ? -normx : normx;
        double* v = refl + (uint64_t)k * m;
        part = 0.0;
        for (uint64_t i = k + tid; i < m; i += nt) {
            double vi = (i == (uint64_t)k) ? x0 - alpha : w[i * n + k];
            v[i - k] = vi;
            part += vi * vi;
        }
        const double vn2 = block_sum(part, red);
        const double beta = (vn2 > 0.0) ? 2.0 / vn2 : 0.0;
        for (int j = k; j < n; ++j) {
            part = 0.0;
            for (uint64_t i = k + tid; i < m; i += nt) part += v[i - k] * w[i * n + j];
            const double dot = block_sum(part, red) * beta;
            for (uint64_t i = k + tid; i < m; i += nt) w[i * n + j] -= dot * v[i - k];
            __syncthreads();
        }
        if (tid == 0) {
            w[(uint64_t)k * n + k] = alpha;
            flip[k] = alpha < 0.0;
            betas[k] = beta;
        }
        __syncthreads();
    }
    for (uint64_t i = tid; i < m * (uint64_t)n; i += nt) q[i] = 0.0;
    __syncthreads();
    for (int k = (int)tid; k < n; k += nt) q[(uint64_t)k * n + k] = 1.0;
    __syncthreads();
    for (int kk = n - 1; kk >= 0; --kk) {
        const double beta = betas[kk];
        if (beta == 0.0) continue;
        const double* v = refl + (uint64_t)kk * m;
        for (int j = kk; j < n; ++j) {
            part = 0.0;
            for (uint64_t i = kk + tid; i < m; i += nt) part += v[i - kk] * q[i * n + j];
            const double dot = block_sum(part, red) * beta;
            for (uint64_t i = kk + tid; i < m; i += nt) q[i * n + j] -= dot * v[i - kk];
            __syncthreads();
        }
    }
    for (uint64_t i = tid; i < m * (uint64_t)n; i += nt) {
        int col = (int)(i % n);
        if (flip[col]) q[i] = -q[i];
    }
}

__global__ void k_gt(const double* __restrict__ core, ModeShape sh, int order, const int* __restrict__ dranks_unused,
                     double* __restrict__ gt, const DevStatus* st) {
    if (skip_kernel(st, kAlways)) return;
    int ks[kMaxOrder], gstride[kMaxOrder];
    {
        int j = 0;
        for (int v = 0; v < order; ++v) ks[v] = (v == sh.n) ? sh.kn : sh.ko[j++];
        int s = 1;
        for (int v = order - 1; v >= 0; --v) {
            gstride[v] = s;
            s *= ks[v];
        }
    }
    const int L = sh.L, Kn = sh.kn;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < L * Kn; q += gridDim.x * blockDim.x) {
        int l = q / Kn, r = q - l * Kn;
        size_t lin = (size_t)r * gstride[sh.n];
        int j = 0;
        for (int v = 0; v < order; ++v) {
            if (v == sh.n) continue;
            lin += (size_t)((l / sh.cstride[j]) % sh.ko[j]) * gstride[v];
            ++j;
        }
        gt[q] = core[lin];
    }
    (void)dranks_unused;
}

__global__ void k_reduce_core(const double* __restrict__ mpart, int nslots, uint64_t size, double* core_out,
                              const DevStatus* st, int run_if) {
    if (skip_kernel(st, run_if)) return;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < size; q += (uint64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int c = 0; c < nslots; ++c) acc += mpart[(size_t)c * size + q];
        core_out[q] = acc;
    }
}

__global__ void k_normsq_one(const double* __restrict__ core, uint64_t size, double* out) {
    __shared__ double red[33];
    double part = 0.0;
    for (uint64_t q = threadIdx.x; q < size; q += blockDim.x) part += core[q] * core[q];
    double f = block_sum(part, red);
    if (threadIdx.x == 0) *out = f;
}

__global__ void k_defect(const double* __restrict__ wpart, int nslots, int K, double* out) {
    __shared__ double red[33];
    double mx = 0.0;
    for (int q = threadIdx.x; q < K * K; q += blockDim.x) {
        double acc = 0.0;
        for (int c = 0; c < nslots; ++c) acc += wpart[(size_t)c * K * K + q];
        int i = q / K, j = q - i * K;
        mx = fmax(mx, fabs(acc - (i == j ? 1.0 : 0.0)));
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
        *out = m;
    }
}

}  // namespace

void launch_reduce_pass(const double* mpart, int mlen, const double* wpart, int wlen, const double* maxpart,
                        int nslots, double* m_out, double* w_out, double* max_out, const DevStatus* st, int run_if,
                        cudaStream_t s) {
    const int tot = mlen + wlen;
    const int blocks = std::max(1, (tot + 7) / 8);
    k_reduce_pass<<<blocks, 256, 0, s>>>(mpart, mlen, wpart, wlen, maxpart, nslots, m_out, w_out, max_out, st, run_if);
    HQ_CHECK_LAUNCH();
}

void launch_gram(const double* A, uint64_t rows, int K, double* wpart, double* maxpart, const DevStatus* st,
                 int run_if, cudaStream_t s) {
    launch_rowgemm(K, A, rows, nullptr, nullptr, nullptr, wpart, maxpart, st, run_if, s);
}

void launch_chol1(const double* w, const double* maxv, int K, double* r1inv, DevStatus* st, int degenerate_mode,
                  cudaStream_t s, bool abort_on_fallback) {
    k_chol1<<<1, 32, 0, s>>>(w, maxv, K, r1inv, st, degenerate_mode, abort_on_fallback ? 1 : 0);
    HQ_CHECK_LAUNCH();
}

void launch_gram2(const double* A, uint64_t rows, int K, const double* r1inv, double* wpart, const DevStatus* st,
                  cudaStream_t s) {
    launch_rowgemm(K, A, rows, r1inv, nullptr, nullptr, wpart, nullptr, st, kOnlyCholQR, s);
}

void launch_chol2(const double* wpart, int nslots, int K, const double* r1inv, double* rinv, const double* m,
                  const ModeShape* sh, double* core_out, DevStatus* st, cudaStream_t s, bool abort_on_fallback) {
    ModeShape z{};
    k_chol2<<<1, 1024, 0, s>>>(wpart, nslots, K, r1inv, rinv, m, sh ? *sh : z, m != nullptr, core_out, st,
                               abort_on_fallback ? 1 : 0);
    HQ_CHECK_LAUNCH();
}

void launch_apply(const double* A, uint64_t rows, int K, const double* rinv, double* u_out, const double* u_old,
                  double* ppart, bool apply, const DevStatus* st, int run_if, cudaStream_t s) {
    if (apply)
        launch_rowgemm(K, A, rows, rinv, u_out, u_old, ppart, nullptr, st, run_if, s);
    else
        launch_rowgemm(K, u_out, rows, nullptr, nullptr, u_old, ppart, nullptr, st, run_if, s);
}

void launch_drift(const double* ppart, int nslots, int K, const double* core, uint64_t core_size, double dns,
                  int order, int mode, bool end_of_sweep, double tol, uint64_t max_sweeps, const SweepTrace& tr,
                  DevStatus* st, cudaStream_t s) {
    k_drift<<<1, 1024, 0, s>>>(ppart, nslots, K, core, core_size, dns, order, mode, end_of_sweep ? 1 : 0, tol,
                              max_sweeps, tr, st);
    HQ_CHECK_LAUNCH();
}

void launch_store_p(const double* ppart, int nslots, int K, int order, int mode, int kmax, uint64_t max_sweeps,
                    double* trp, const DevStatus* st, cudaStream_t s) {
    const int blocks = std::max(1, (K * K + 7) / 8);
    k_store_p<<<blocks, 256, 0, s>>>(ppart, nslots, K, order, mode, kmax, max_sweeps, trp, st);
    HQ_CHECK_LAUNCH();
}

void launch_sweep_end(const double* core, uint64_t core_size, double dns, double tol, uint64_t max_sweeps,
                      const SweepTrace& tr, DevStatus* st, cudaStream_t s) {
    k_sweep_end<<<1, 1024, 0, s>>>(core, core_size, dns, tol, max_sweeps, tr, st);
    HQ_CHECK_LAUNCH();
}

void launch_drift_batch(const double* trp, int pairs, int order, const int* ranks_dev, int kmax, double* drift,
                        cudaStream_t s) {
    if (pairs <= 0) return;
    k_drift_batch<<<pairs, 32, 0, s>>>(trp, pairs, order, ranks_dev, kmax, drift);
    HQ_CHECK_LAUNCH();
}

void launch_householder(const double* A, uint64_t rows, int K, double* q_out, double* work, const DevStatus* st,
                        int run_if, cudaStream_t s) {
    k_householder<<<1, kHhThreads, 0, s>>>(A, rows, K, q_out, work, st, run_if);
    HQ_CHECK_LAUNCH();
}

void launch_gt(const double* core, const ModeShape& sh, const int* ranks, double* gt, const DevStatus* st,
               cudaStream_t s) {
    (void)ranks;
    int tot = sh.L * sh.kn;
    int blocks = std::max(1, std::min((tot + 255) / 256, num_sms()));
    k_gt<<<blocks, 256, 0, s>>>(core, sh, sh.order, nullptr, gt, st);
    HQ_CHECK_LAUNCH();
}

void launch_reduce_core(const double* mpart, int nslots, uint64_t size, double* core_out, const DevStatus* st,
                        int run_if, cudaStream_t s) {
    int blocks = (int)std::max<uint64_t>(1, std::min<uint64_t>((size + 255) / 256, (uint64_t)num_sms() * 4));
    k_reduce_core<<<blocks, 256, 0, s>>>(mpart, nslots, size, core_out, st, run_if);
    HQ_CHECK_LAUNCH();
}

void launch_core_normsq(const double* core, uint64_t size, double* out, cudaStream_t s) {
    k_normsq_one<<<1, 256, 0, s>>>(core, size, out);
    HQ_CHECK_LAUNCH();
}

void launch_defect(const double* u, uint64_t rows, int K, double* wpart, double* out_max, cudaStream_t s) {
    launch_rowgemm(K, u, rows, nullptr, nullptr, nullptr, wpart, nullptr, nullptr, kAlways, s);
    k_defect<<<1, 256, 0, s>>>(wpart, dense_slots(), K, out_max);
    HQ_CHECK_LAUNCH();
}

}  // namespace hq
