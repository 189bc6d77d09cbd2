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

int dense_slots() { return num_sms() * 2; }

namespace {

constexpr int kDenseThreads = 256;
constexpr int kChunk = 32;

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

__global__ void k_reduce_pass(const double* __restrict__ mpart, int mlen, const double* __restrict__ wpart, int wlen,
                              const double* __restrict__ maxpart, int nslots, double* m_out, double* w_out,
                              double* max_out, const DevStatus* st, int run_if) {
    if (skip_kernel(st, run_if)) return;
    int tot = mlen + wlen;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += gridDim.x * blockDim.x) {
        double acc = 0.0;
        if (q < mlen) {
            for (int c = 0; c < nslots; ++c) acc += mpart[(size_t)c * mlen + q];
            m_out[q] = acc;
        } else {
            int r = q - mlen;
            for (int c = 0; c < nslots; ++c) acc += wpart[(size_t)c * wlen + r];
            w_out[r] = acc;
        }
    }
    if (max_out && blockIdx.x == 0 && threadIdx.x == 0) {
        double m = 0.0;
        for (int c = 0; c < nslots; ++c) m = fmax(m, maxpart[c]);
        *max_out = m;
    }
}

// Gram partials of a row-major rows x K matrix, optionally transformed by an
// upper-triangular T (rows of A T), plus max|A|.
__global__ void __launch_bounds__(kDenseThreads) k_gram(const double* __restrict__ A, uint64_t rows, int K,
                                                        const double* __restrict__ T, double* __restrict__ wpart,
                                                        double* __restrict__ maxpart, const DevStatus* st, int run_if) {
    if (skip_kernel(st, run_if)) return;
    __shared__ double sA[kChunk * kMaxRank];
    __shared__ double sU[kChunk * kMaxRank];
    __shared__ double sT[kMaxRank * kMaxRank];
    __shared__ double red[33];
    const int G = gridDim.x, c = blockIdx.x;
    const uint64_t rb = rows * c / G, re = rows * (c + 1) / G;
    if (T)
        for (int q = threadIdx.x; q < K * K; q += blockDim.x) sT[q] = T[q];
    double acc[kAcc];
#pragma unroll
    for (int j = 0; j < kAcc; ++j) acc[j] = 0.0;
    double mx = 0.0;
    for (uint64_t r0 = rb; r0 < re; r0 += kChunk) {
        const int nr = (int)min((uint64_t)kChunk, re - r0);
        __syncthreads();
        for (int q = threadIdx.x; q < nr * K; q += blockDim.x) {
            double v = A[r0 * K + q];
            sA[q] = v;
            mx = fmax(mx, fabs(v));
        }
        __syncthreads();
        const double* src = sA;
        if (T) {
            for (int q = threadIdx.x; q < nr * K; q += blockDim.x) {
                int r = q / K, j = q - r * K;
                double s = 0.0;
                for (int k = 0; k <= j; ++k) s += sA[r * K + k] * sT[k * K + j];
                sU[q] = s;
            }
            __syncthreads();
            src = sU;
        }
#pragma unroll
        for (int j = 0; j < kAcc; ++j) {
            int e = threadIdx.x + j * kDenseThreads;
            if (e < K * K) {
                int p = e / K, q = e - p * K;
                double a = acc[j];
                for (int r = 0; r < nr; ++r) a += src[r * K + p] * src[r * K + q];
                acc[j] = a;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < kAcc; ++j) {
        int e = threadIdx.x + j * kDenseThreads;
        if (e < K * K) wpart[(size_t)c * K * K + e] = acc[j];
    }
    if (maxpart) {
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
        __syncthreads();
        if (threadIdx.x == 0) {
            double m = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
            maxpart[c] = m;
        }
    }
}

// upper-triangular Cholesky W = R^T R; false when a pivot keeps less than
// 1e-12 of its diagonal (column nearly in the span of the previous ones)
__device__ bool chol_upper(const double* W, int K, double* R) {
    for (int q = 0; q < K * K; ++q) R[q] = 0.0;
    for (int k = 0; k < K; ++k) {
        double d = W[k * K + k];
        for (int j = 0; j < k; ++j) d -= R[j * K + k] * R[j * K + k];
        if (!(d > 1e-12 * W[k * K + k]) || !isfinite(d)) return false;
        double rkk = sqrt(d);
        R[k * K + k] = rkk;
        for (int c = k + 1; c < K; ++c) {
            double s = W[k * K + c];
            for (int j = 0; j < k; ++j) s -= R[j * K + k] * R[j * K + c];
            R[k * K + c] = s / rkk;
        }
    }
    return true;
}

__device__ void inv_upper(const double* R, int K, double* X) {
    for (int q = 0; q < K * K; ++q) X[q] = 0.0;
    for (int j = 0; j < K; ++j) {
        X[j * K + j] = 1.0 / R[j * K + j];
        for (int i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int k = i + 1; k <= j; ++k) s += R[i * K + k] * X[k * K + j];
            X[i * K + j] = -s / R[i * K + i];
        }
    }
}

__global__ void k_chol1(const double* __restrict__ w, const double* __restrict__ maxv, int K, double* r1inv,
                        DevStatus* st, int degenerate_mode) {
    if (skip_kernel(st, kAlways)) return;
    __shared__ double sW[kMaxRank * kMaxRank];
    __shared__ double sR[kMaxRank * kMaxRank];
    __shared__ double sX[kMaxRank * kMaxRank];
    for (int q = threadIdx.x; q < K * K; q += blockDim.x) sW[q] = w[q];
    __syncthreads();
    if (threadIdx.x != 0) return;
    st->fallback = 0;
    if (*maxv == 0.0) {
        if (degenerate_mode > 0) {  // solvers.cpp:124: DegenerateStateError(n + 1)
            st->abort = 1;
            st->degenerate_mode = degenerate_mode;
            st->degenerate_sweep = st->sweep + 1;
            return;
        }
        st->fallback = 1;  // zero matrix: the reference fills every column (dense_core.cpp:146-157)
        return;
    }
    if (!chol_upper(sW, K, sR)) {
        st->fallback = 1;
        return;
    }
    inv_upper(sR, K, sX);
    for (int q = 0; q < K * K; ++q) r1inv[q] = sX[q];
}

__global__ void k_chol2(const double* __restrict__ wpart, int nslots, int K, const double* __restrict__ r1inv,
                        double* rinv, const double* __restrict__ m, ModeShape sh, int has_m, double* core_out,
                        DevStatus* st) {
    if (skip_kernel(st, kOnlyCholQR)) return;
    __shared__ double sW[kMaxRank * kMaxRank];
    __shared__ double sR[kMaxRank * kMaxRank];
    __shared__ double sX[kMaxRank * kMaxRank];
    __shared__ double sY[kMaxRank * kMaxRank];
    __shared__ int ok;
    for (int q = threadIdx.x; q < K * K; q += blockDim.x) {
        double acc = 0.0;
        for (int c = 0; c < nslots; ++c) acc += wpart[(size_t)c * K * K + q];
        sW[q] = acc;
        sY[q] = r1inv[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ok = chol_upper(sW, K, sR);
        if (ok) {
            for (int k = 0; k < K; ++k)  // R2 ~ I after one CholQR pass
                if (!(sR[k * K + k] > 0.5 && sR[k * K + k] < 2.0)) ok = 0;
        }
        if (ok) {
            inv_upper(sR, K, sX);
            // Rinv = R1inv * R2inv (both upper)
            for (int i = 0; i < K; ++i)
                for (int j = 0; j < K; ++j) {
                    double s = 0.0;
                    for (int k = i; k <= j; ++k) s += sY[i * K + k] * sX[k * K + j];
                    sW[i * K + j] = (j >= i) ? s : 0.0;
                }
        } else {
            st->fallback = 1;
        }
    }
    __syncthreads();
    if (!ok) return;
    for (int q = threadIdx.x; q < K * K; q += blockDim.x) rinv[q] = sW[q];
    if (has_m) {
        // G_(n) = Rinv^T M, refolded into the core (dense_core.cpp:350-369 layout)
        const int L = sh.L;
        int gstride[kMaxOrder];
        int ks[kMaxOrder];
        {
            int j = 0;
            for (int v = 0; v < sh.order; ++v) ks[v] = (v == sh.n) ? sh.kn : sh.ko[j++];
            int s = 1;
            for (int v = sh.order - 1; v >= 0; --v) {
                gstride[v] = s;
                s *= ks[v];
            }
        }
        for (int q = threadIdx.x; q < K * L; q += blockDim.x) {
            int r = q / L, l = q - r * L;
            double acc = 0.0;
            for (int k = 0; k <= r; ++k) acc += sW[k * K + r] * m[(size_t)k * L + l];
            size_t lin = (size_t)r * gstride[sh.n];
            int j = 0;
            for (int v = 0; v < sh.order; ++v) {
                if (v == sh.n) continue;
                int kv = (l / sh.cstride[j]) % sh.ko[j];
                lin += (size_t)kv * gstride[v];
                ++j;
            }
            core_out[lin] = acc;
        }
    }
}

__global__ void __launch_bounds__(kDenseThreads) k_apply(const double* __restrict__ A, uint64_t rows, int K,
                                                         const double* __restrict__ rinv, double* u_out,
                                                         const double* __restrict__ u_old, double* __restrict__ ppart,
                                                         int apply, const DevStatus* st, int run_if) {
    if (skip_kernel(st, run_if)) return;
    __shared__ double sA[kChunk * kMaxRank];
    __shared__ double sU[kChunk * kMaxRank];
    __shared__ double sO[kChunk * kMaxRank];
    __shared__ double sT[kMaxRank * kMaxRank];
    const int G = gridDim.x, c = blockIdx.x;
    const uint64_t rb = rows * c / G, re = rows * (c + 1) / G;
    if (apply)
        for (int q = threadIdx.x; q < K * K; q += blockDim.x) sT[q] = rinv[q];
    double acc[kAcc];
#pragma unroll
    for (int j = 0; j < kAcc; ++j) acc[j] = 0.0;
    for (uint64_t r0 = rb; r0 < re; r0 += kChunk) {
        const int nr = (int)min((uint64_t)kChunk, re - r0);
        __syncthreads();
        for (int q = threadIdx.x; q < nr * K; q += blockDim.x) {
            if (apply)
                sA[q] = A[r0 * K + q];
            else
                sU[q] = u_out[r0 * K + q];
            if (u_old) sO[q] = u_old[r0 * K + q];
        }
        __syncthreads();
        if (apply) {
            for (int q = threadIdx.x; q < nr * K; q += blockDim.x) {
                int r = q / K, j = q - r * K;
                double s = 0.0;
                for (int k = 0; k <= j; ++k) s += sA[r * K + k] * sT[k * K + j];
                sU[q] = s;
                u_out[r0 * K + q] = s;
            }
            __syncthreads();
        }
        if (u_old) {
#pragma unroll
            for (int j = 0; j < kAcc; ++j) {
                int e = threadIdx.x + j * kDenseThreads;
                if (e < K * K) {
                    int p = e / K, q = e - p * K;
                    double a = acc[j];
                    for (int r = 0; r < nr; ++r) a += sU[r * K + p] * sO[r * K + q];
                    acc[j] = a;
                }
            }
        }
    }
    if (u_old) {
#pragma unroll
        for (int j = 0; j < kAcc; ++j) {
            int e = threadIdx.x + j * kDenseThreads;
            if (e < K * K) ppart[(size_t)c * K * K + e] = acc[j];
        }
    }
}

// cyclic Jacobi eigenvalues (dense_core.cpp:200-264), single thread
__device__ void jacobi_eigvals(double* m, int n, double* ev) {
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            double avg = 0.5 * (m[i * n + j] + m[j * n + i]);
            m[i * n + j] = m[j * n + i] = avg;
        }
    double fn = 0.0;
    for (int i = 0; i < n * n; ++i) fn += m[i] * m[i];
    fn = sqrt(fn);
    const double stop = 1e-15 * (fn > 0.0 ? fn : 1.0);
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += m[p * n + q] * m[p * n + q];
        if (sqrt(2.0 * off) <= stop) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                double apq = m[p * n + q];
                if (fabs(apq) <= 1e-300) continue;
                double theta = (m[q * n + q] - m[p * n + p]) / (2.0 * apq);
                double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0);
                double s = t * c;
                double tau = s / (1.0 + c);
                double app = m[p * n + p], aqq = m[q * n + q];
                m[p * n + p] = app - t * apq;
                m[q * n + q] = aqq + t * apq;
                m[p * n + q] = m[q * n + p] = 0.0;
                for (int r = 0; r < n; ++r) {
                    if (r != p && r != q) {
                        double arp = m[r * n + p], arq = m[r * n + q];
                        m[r * n + p] = m[p * n + r] = arp - s * (arq + tau * arp);
                        m[r * n + q] = m[q * n + r] = arq + s * (arp - tau * arq);
                    }
                }
            }
    }
    for (int i = 0; i < n; ++i) ev[i] = m[i * n + i];
}

__global__ void k_drift(const double* __restrict__ ppart, int nslots, int K, const double* __restrict__ core,
                        uint64_t core_size, double dns, int order, int mode, int end_of_sweep, double tol,
                        uint64_t max_sweeps, SweepTrace tr, DevStatus* st) {
    if (st->abort || (st->sweep >= (int)max_sweeps)) return;
    __shared__ double sP[kMaxRank * kMaxRank];
    __shared__ double sM[kMaxRank * kMaxRank];
    __shared__ double ev[kMaxRank];
    __shared__ double red[33];
    for (int q = threadIdx.x; q < K * K; q += blockDim.x) {
        double acc = 0.0;
        for (int c = 0; c < nslots; ++c) acc += ppart[(size_t)c * K * K + q];
        sP[q] = acc;
    }
    __syncthreads();
    // M^T M with M = U_new^T U_old (manifold.cpp:57 -> dense_core.cpp:331)
    for (int q = threadIdx.x; q < K * K; q += blockDim.x) {
        int i = q / K, j = q - i * K;
        double s = 0.0;
        for (int r = 0; r < K; ++r) s += sP[r * K + i] * sP[r * K + j];
        sM[q] = s;
    }
    double f = 0.0;
    if (end_of_sweep) {
        double part = 0.0;
        for (uint64_t q = threadIdx.x; q < core_size; q += blockDim.x) part += core[q] * core[q];
        f = block_sum(part, red);
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int sw = st->sweep;
    jacobi_eigvals(sM, K, ev);
    double s = 0.0;
    for (int i = 0; i < K; ++i) s += sqrt(ev[i] > 0.0 ? ev[i] : 0.0);
    double d = 2.0 * (double)K - 2.0 * s;
    tr.drift[(size_t)sw * order + mode] = d > 0.0 ? d : 0.0;
    if (st->fallback) st->fallback_count++;
    st->fallback = 0;
    if (end_of_sweep) {
        double fit = dns - f;
        tr.objective[sw] = f;
        tr.fit[sw] = fit;
        st->sweep = sw + 1;
        // solvers.cpp:164-167 stop rule
        if (fabs(*tr.fit_prev - fit) < tol) st->abort = 2;
        *tr.fit_prev = fit;
    }
}

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
    int tot = mlen + wlen;
    int blocks = std::max(1, std::min((tot + 255) / 256, num_sms() * 4));
    k_reduce_pass<<<blocks, 256, 0, s>>>(mpart, mlen, wpart, wlen, maxpart, nslots, m_out, w_out, max_out, st, run_if);
    HQ_CHECK_LAUNCH();
}

void launch_gram(const double* A, uint64_t rows, int K, double* wpart, double* maxpart, const DevStatus* st,
                 int run_if, cudaStream_t s) {
    k_gram<<<dense_slots(), kDenseThreads, 0, s>>>(A, rows, K, nullptr, wpart, maxpart, st, run_if);
    HQ_CHECK_LAUNCH();
}

void launch_chol1(const double* w, const double* maxv, int K, double* r1inv, DevStatus* st, int degenerate_mode,
                  cudaStream_t s) {
    k_chol1<<<1, 128, 0, s>>>(w, maxv, K, r1inv, st, degenerate_mode);
    HQ_CHECK_LAUNCH();
}

void launch_gram2(const double* A, uint64_t rows, int K, const double* r1inv, double* wpart, const DevStatus* st,
                  cudaStream_t s) {
    k_gram<<<dense_slots(), kDenseThreads, 0, s>>>(A, rows, K, r1inv, wpart, nullptr, st, kOnlyCholQR);
    HQ_CHECK_LAUNCH();
}

void launch_chol2(const double* wpart, int nslots, int K, const double* r1inv, double* rinv, const double* m,
                  const ModeShape* sh, double* core_out, DevStatus* st, cudaStream_t s) {
    ModeShape z{};
    k_chol2<<<1, 256, 0, s>>>(wpart, nslots, K, r1inv, rinv, m, sh ? *sh : z, m != nullptr, core_out, st);
    HQ_CHECK_LAUNCH();
}

void launch_apply(const double* A, uint64_t rows, int K, const double* rinv, double* u_out, const double* u_old,
                  double* ppart, bool apply, const DevStatus* st, int run_if, cudaStream_t s) {
    k_apply<<<dense_slots(), kDenseThreads, 0, s>>>(A, rows, K, rinv, u_out, u_old, ppart, apply ? 1 : 0, st, run_if);
    HQ_CHECK_LAUNCH();
}

void launch_drift(const double* ppart, int nslots, int K, const double* core, uint64_t core_size, double dns,
                  int order, int mode, bool end_of_sweep, double tol, uint64_t max_sweeps, const SweepTrace& tr,
                  DevStatus* st, cudaStream_t s) {
    k_drift<<<1, 256, 0, s>>>(ppart, nslots, K, core, core_size, dns, order, mode, end_of_sweep ? 1 : 0, tol,
                              max_sweeps, tr, st);
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
    k_gram<<<dense_slots(), kDenseThreads, 0, s>>>(u, rows, K, nullptr, wpart, nullptr, nullptr, kAlways);
    k_defect<<<1, 256, 0, s>>>(wpart, dense_slots(), K, out_max);
    HQ_CHECK_LAUNCH();
}

}  // namespace hq
