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
#include <cstdio>

#include "hq_dense.cuh"

namespace hq {

int dense_slots() { return num_sms(); }  // = the tall-skinny pass's grid (one CTA per SM, hq_rowgemm.cu)

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

// Multi-CTA Householder QR (one CTA per SM, co-resident: cooperative launch)
// with the reference's exact step sequence (dense_core.cpp:127-198): for each
// column k, normx over rows >= k, the rank-deficiency fill when
// normx <= 1e-12 ||A||_F, alpha = -sign(x0) normx, v = x - alpha e_k,
// beta = 2 / v^T v, and the reflector applied to columns > k; then Q formed by
// backward accumulation and its columns' signs flipped where alpha < 0
// (R_kk >= 0).  CTA c owns rows [m c / G, m (c + 1) / G); each column needs
// one pass over the rows and one grid barrier: the pass that applies
// reflector k also accumulates, per CTA, T_j = sum_{i > k+1} w_{i,k+1} w_ij for
// the next column, and every CTA reduces the G partials in the same fixed
// order, so all CTAs derive identical alpha / beta / dots.  The fill takes
// its normals from the precomputed stream (fill_table) when one is given,
// else CTA 0 draws them with the device MT19937-64.
constexpr int kHhThreads = 256;
constexpr int kHhSlot = 36;  // partial-slot stride (K <= 32 sums + ||A||^2)
constexpr int kHhGramSlot = 32 * 33 / 2;  // per-CTA partial of V^T V (upper triangle, K <= 32)
constexpr int kHhGramRows = 64;           // rows of V staged per Gram tile

struct HhCtl {
    unsigned int bar_count;
    unsigned int bar_gen;
    unsigned int rng_seeded;
    unsigned int started;  // diagnostics for the barrier watchdog: CTAs that entered / left the kernel
    unsigned int exited;
    unsigned int timeout_cta;   // barrier watchdog: 1 + the CTA that gave up (0: none), read by the host on failure
    unsigned int timeout_gen;
    unsigned int pad;
    DevRng rng;
};

__host__ __device__ inline size_t hh_part_doubles(int G) { return (size_t)2 * G * kHhSlot; }
constexpr size_t kHhCtlDoubles = (sizeof(HhCtl) + 15) / 16 * 2;

__device__ __forceinline__ void hh_grid_sync(HhCtl* ctl, unsigned int& gen) {
    // every thread's global writes of this phase (partial slots, w, reflectors, q) are made visible at GPU
    // scope before thread 0 signals arrival: a fence by thread 0 alone orders only its own stores, and a CTA
    // reading another CTA's partial slot early derives different pivots -> diverging barrier counts (hang)
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int arrived = atomicAdd(&ctl->bar_count, 1u);
        if (arrived == gridDim.x - 1) {
            ctl->bar_count = 0;
            __threadfence();
            atomicExch(&ctl->bar_gen, gen + 1);
        } else {
            const long long t0 = clock64();
            // poll with acquire loads (served by L2 in parallel), not atomics that serialise on one address
            // against the last arriver's release
            auto gen_now = [&]() {
                unsigned int g;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&ctl->bar_gen) : "memory");
                return g;
            };
            while (gen_now() == gen) {
                __nanosleep(64);
                if (clock64() - t0 > (1ll << 33)) {  // ~4 s: a lost arrival -- fail loudly instead of hanging
                    // (no printf: its ABI call would make every inlined barrier save registers to the stack)
                    ctl->timeout_cta = blockIdx.x + 1;
                    ctl->timeout_gen = gen;
                    __threadfence_system();
                    __trap();
                }
            }
        }
        __threadfence();
        gen = gen + 1;
    }
    __syncthreads();
}

// per-CTA sums of acc[0..cnt) (deterministic: warp tree, then warps in order)
template <int KM>
__device__ __forceinline__ void hh_cta_partials(const double (&acc)[KM + 1], int cnt, double* red_w, double* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int j = 0; j <= KM; ++j) {
        double v = acc[j];
        for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) red_w[warp * (KM + 1) + j] = v;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += red_w[w * (KM + 1) + j];
        out[j] = t;
    }
}

// sum over CTAs c = 0, 1, ... (this order, every CTA alike) of p[c * stride]; the loads of a batch of 8
// are issued together (one L2 round trip per batch, not per CTA); L2 reads: other CTAs' slots
__device__ __forceinline__ double hh_sum_slots(const double* p, size_t stride, unsigned G) {
    double t = 0.0;
    unsigned c = 0;
    for (; c + 8 <= G; c += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + (size_t)(c + u) * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) t += v[u];
    }
    for (; c < G; ++c) t += __ldcg(p + (size_t)c * stride);
    return t;
}

// every CTA: T[j] = sum over CTAs (in order) of part[c][j], j < cnt
__device__ __forceinline__ void hh_reduce_all(const double* part, int cnt, double* T) {
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) T[j] = hh_sum_slots(part + j, kHhSlot, gridDim.x);
    __syncthreads();
}

template <int KM>
__device__ __forceinline__ double pick(const double (&row)[KM], int k) {
    double v = 0.0;
#pragma unroll
    for (int j = 0; j < KM; ++j)
        if (j == k) v = row[j];
    return v;
}

template <int KM>
__global__ void __launch_bounds__(kHhThreads, 1) k_householder_mc(const double* __restrict__ A, uint64_t m, int n,
                                                               double* __restrict__ q, double* __restrict__ work,
                                                               const double* __restrict__ table, uint64_t table_len,
                                                               const DevStatus* st, int run_if) {
    if (skip_kernel(st, run_if)) return;
    __shared__ double red_w[(kHhThreads / 32) * (KM + 1)];
    __shared__ double T[KM + 1];
    __shared__ double dots[KM];
    __shared__ double betas[KM];
    __shared__ int flip[KM];
    __shared__ double sc[4];  // normx, pivot_tol, x0 - alpha
    const unsigned G = gridDim.x, c = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
    // work: control block | partials [2][G][kHhSlot] | w (m x n) | reflectors (n x m);
    // fixed offsets, so every (m, n) shares one barrier
    HhCtl* ctl = reinterpret_cast<HhCtl*>(work);
    double* part = work + kHhCtlDoubles;
    double* w = part + hh_part_doubles((int)G);
    double* refl = w + m * (uint64_t)n;  // rows >= k of reflector k used
    const uint64_t r0 = m * c / G, r1 = m * (c + 1) / G;
    unsigned int gen = 0;
    if (tid == 0) {
        gen = atomicAdd(&ctl->bar_gen, 0u);
        atomicAdd(&ctl->started, 1u);
    }
    if (c == 0 && tid == 0) ctl->rng_seeded = 0;  // each QR starts the fill stream afresh (read after a barrier)
    int par = 0;
    uint64_t pos = 0;  // fill-stream position (identical in every CTA)
    auto slot = [&](int pr) { return part + ((size_t)pr * G + c) * kHhSlot; };
    auto slots = [&](int pr) { return part + (size_t)pr * G * kHhSlot; };

    // copy A -> w; partials of T_j for column 0 (rows > 0) and ||A||^2 (slot KM)
    {
        double acc[KM + 1];
#pragma unroll
        for (int j = 0; j <= KM; ++j) acc[j] = 0.0;
        for (uint64_t i = r0 + tid; i < r1; i += nt) {
            double row[KM];
#pragma unroll
            for (int j = 0; j < KM; ++j) row[j] = j < n ? A[i * n + j] : 0.0;
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (j < n) {
                    w[i * n + j] = row[j];
                    acc[KM] += row[j] * row[j];
                    if (i > 0) acc[j] += row[0] * row[j];
                }
        }
        hh_cta_partials<KM>(acc, KM + 1, red_w, slot(par));
    }
    hh_grid_sync(ctl, gen);
    double ptol = 0.0;
    for (int k = 0; k < n; ++k) {
        hh_reduce_all(slots(par), k == 0 ? KM + 1 : n, T);
        if (k == 0) ptol = 1e-12 * sqrt(T[KM]);
        double normx;
        {
            const double x0 = __ldcg(w + (uint64_t)k * n + k);  // pivot row: another CTA's
            normx = sqrt(T[k] + x0 * x0);
        }
        // rank-deficient column: rows >= k replaced by the next normals of the
        // fill stream (dense_core.cpp:146-157), redrawn while the norm is zero
        bool need = normx <= ptol;
        while (need) {
            // every CTA has read the pivot w[k][k] and taken the same decision before the owner of row k
            // overwrites it with the fill: without this barrier a late CTA could read the filled pivot, skip
            // the fill, and run two grid barriers fewer than the others (the kernel then hangs)
            hh_grid_sync(ctl, gen);
            const uint64_t cnt = m - (uint64_t)k;
            if (table && pos + cnt <= table_len) {
                for (uint64_t i = (r0 > (uint64_t)k ? r0 : (uint64_t)k) + tid; i < r1; i += nt)
                    w[i * n + k] = table[pos + (i - k)];
            } else if (c == 0 && tid == 0) {
                if (!ctl->rng_seeded) {
                    rng_seed(&ctl->rng, 0x48514F5251ull);
                    for (uint64_t d = 0; d < pos; ++d) rng_normal(&ctl->rng);  // normals already taken from the table
                    ctl->rng_seeded = 1;
                }
                for (uint64_t i = k; i < m; ++i) w[i * n + k] = rng_normal(&ctl->rng);
            }
            pos += cnt;
            hh_grid_sync(ctl, gen);
            {
                double acc[KM + 1];
#pragma unroll
                for (int j = 0; j <= KM; ++j) acc[j] = 0.0;
                for (uint64_t i = (r0 > (uint64_t)k + 1 ? r0 : (uint64_t)k + 1) + tid; i < r1; i += nt) {
                    const double wk = w[i * n + k];
#pragma unroll
                    for (int j = 0; j < KM; ++j)
                        if (j >= k && j < n) acc[j] += wk * w[i * n + j];
                }
                par ^= 1;
                hh_cta_partials<KM>(acc, n, red_w, slot(par));
            }
            hh_grid_sync(ctl, gen);
            hh_reduce_all(slots(par), n, T);
            const double x0 = __ldcg(w + (uint64_t)k * n + k);  // pivot row: another CTA's
            normx = sqrt(T[k] + x0 * x0);
            need = normx == 0.0;
        }
        // reflector (every CTA derives the same values)
        if (tid == 0) {
            const double x0 = __ldcg(w + (uint64_t)k * n + k);  // pivot row: another CTA's
            const double alpha = (x0 >= 0.0) ? -normx : normx;
            const double vk = x0 - alpha;
            const double vn2 = T[k] + vk * vk;
            sc[2] = vk;
            betas[k] = (vn2 > 0.0) ? 2.0 / vn2 : 0.0;
            flip[k] = alpha < 0.0;
        }
        __syncthreads();
        for (int j = k + 1 + (int)tid; j < n; j += nt) dots[j] = betas[k] * (sc[2] * __ldcg(w + (uint64_t)k * n + j) + T[j]);
        __syncthreads();
        // apply to columns > k over rows >= k; partial T for column k+1 (rows > k+1)
        {
            double acc[KM + 1];
#pragma unroll
            for (int j = 0; j <= KM; ++j) acc[j] = 0.0;
            const double vk = sc[2];
            for (uint64_t i = (r0 > (uint64_t)k ? r0 : (uint64_t)k) + tid; i < r1; i += nt) {
                double row[KM];
#pragma unroll
                for (int j = 0; j < KM; ++j) row[j] = (j >= k && j < n) ? w[i * n + j] : 0.0;
                const double v = (i == (uint64_t)k) ? vk : pick<KM>(row, k);
                refl[(uint64_t)k * m + i] = v;
                // row k becomes R's row k, which no later step reads -- and other CTAs may still be
                // reading it for their dots in this phase, so it is left untouched
                if (i == (uint64_t)k) continue;
#pragma unroll
                for (int j = 0; j < KM; ++j)
                    if (j > k && j < n) {
                        row[j] -= dots[j] * v;
                        w[i * n + j] = row[j];
                    }
                if (i > (uint64_t)k + 1) {
                    const double wn = pick<KM>(row, k + 1);
#pragma unroll
                    for (int j = 0; j < KM; ++j)
                        if (j >= k + 1 && j < n) acc[j] += wn * row[j];
                }
            }
            par ^= 1;
            hh_cta_partials<KM>(acc, n, red_w, slot(par));
        }
        hh_grid_sync(ctl, gen);
    }
    // ---- Q = H_0 ... H_{n-1} [I; 0] in compact WY form (LAPACK dlarft):
    // H_0 ... H_{n-1} = I - V Tw V^T with V = [v_0 ... v_{n-1}] (v_k zero above row k) and Tw upper
    // triangular, Tw[k][k] = beta_k, Tw[0:k, k] = -beta_k Tw[0:k, 0:k] (V[:, 0:k]^T v_k).  Then
    // Q [i, :] = e_i - v(i) C with C = Tw V_top^T (V_top = the first n rows of V), so the whole product is
    // one Gram pass (V^T V, partial per CTA), one barrier, and one pass writing Q -- equal in exact
    // arithmetic to the reference's backward accumulation (dense_core.cpp:183-196).
    {
        constexpr int NP = KM * (KM + 1) / 2;  // upper-triangle pairs of V^T V
        double* gpart = refl + (uint64_t)n * m;  // [G][kHhGramSlot]
        __shared__ double sV[kHhGramRows][KM + 1];
        __shared__ double sG[KM][KM];
        __shared__ double sTw[KM][KM];
        __shared__ double sC[KM][KM];
        const int np = n * (n + 1) / 2;
        double gacc[(NP + kHhThreads - 1) / kHhThreads];
#pragma unroll
        for (int u = 0; u < (NP + kHhThreads - 1) / kHhThreads; ++u) gacc[u] = 0.0;
        for (uint64_t t0 = r0; t0 < r1; t0 += kHhGramRows) {
            const int tr = (int)min((uint64_t)kHhGramRows, r1 - t0);
            __syncthreads();
            for (int e = tid; e < kHhGramRows * n; e += nt) {  // reflector-major: coalesced along rows
                const int k = e / kHhGramRows, r = e - k * kHhGramRows;
                const uint64_t i = t0 + r;
                sV[r][k] = (r < tr && i >= (uint64_t)k) ? refl[(uint64_t)k * m + i] : 0.0;
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < (NP + kHhThreads - 1) / kHhThreads; ++u) {
                const int pi = (int)tid + u * kHhThreads;
                if (pi < np) {
                    int k = 0, rem = pi;  // pair pi -> (k, l), l >= k, row-major upper triangle
                    while (rem >= n - k) {
                        rem -= n - k;
                        ++k;
                    }
                    const int l = k + rem;
                    double sacc = gacc[u];
                    for (int r = 0; r < tr; ++r) sacc = fma(sV[r][k], sV[r][l], sacc);
                    gacc[u] = sacc;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < (NP + kHhThreads - 1) / kHhThreads; ++u) {
            const int pi = (int)tid + u * kHhThreads;
            if (pi < np) gpart[(size_t)c * kHhGramSlot + pi] = gacc[u];
        }
        hh_grid_sync(ctl, gen);
        // V^T V (every CTA, fixed order over the CTAs), then Tw and C on one warp
        for (int pi = tid; pi < np; pi += nt) {
            const double v = hh_sum_slots(gpart + pi, kHhGramSlot, G);
            int k = 0, rem = pi;
            while (rem >= n - k) {
                rem -= n - k;
                ++k;
            }
            sG[k][k + rem] = v;
            sG[k + rem][k] = v;
        }
        // V_top: the first n rows of V (another CTA's rows: read through L2)
        for (int e = tid; e < n * n; e += nt) {
            const int j = e / n, l = e - j * n;  // v_l[j]
            sV[j][l] = ((uint64_t)j < m && j >= l) ? __ldcg(refl + (uint64_t)l * m + j) : 0.0;
        }
        __syncthreads();
        if (tid < 32) {
            const int lane = tid;
            for (int k = 0; k < n; ++k) {
                // Tw[0:k, k] = -beta_k Tw[0:k, 0:k] G[0:k, k]  (lane l computes row l < k)
                double z = 0.0;
                if (lane < k)
                    for (int j = lane; j < k; ++j) z += sTw[lane][j] * sG[j][k];
                __syncwarp();
                if (lane < n) sTw[lane][k] = lane < k ? -betas[k] * z : (lane == k ? betas[k] : 0.0);
                __syncwarp();
            }
            // C = Tw V_top^T: C[k][j] = sum_{l >= k} Tw[k][l] v_l[j]
            for (int e = lane; e < n * n; e += 32) {
                const int k = e / n, j = e - k * n;
                double v = 0.0;
                for (int l = k; l < n; ++l) v += sTw[k][l] * sV[j][l];
                sC[k][j] = v;
            }
        }
        __syncthreads();
        for (uint64_t i = r0 + tid; i < r1; i += nt) {
            double vi[KM];
#pragma unroll
            for (int k = 0; k < KM; ++k) vi[k] = (k < n && i >= (uint64_t)k) ? refl[(uint64_t)k * m + i] : 0.0;
            // (the j loop is left rolled: unrolled, its KM x KM loads of C are hoisted and spill registers)
#pragma unroll 1
            for (int j = 0; j < n; ++j) {
                double v = (i == (uint64_t)j) ? 1.0 : 0.0;
#pragma unroll
                for (int k = 0; k < KM; ++k)
                    if (k < n) v -= vi[k] * sC[k][j];
                q[i * n + j] = v;
            }
        }
    }
    // R_kk >= 0: flip the columns whose alpha was negative
    for (uint64_t i = r0 + tid; i < r1; i += nt)
        for (int j = 0; j < n; ++j)
            if (flip[j]) q[i * n + j] = -q[i * n + j];
    if (tid == 0) atomicAdd(&ctl->exited, 1u);
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
    // order 3, K = 10: the short-row pass's A-GEMM fragments (hq_pass_fast.cu k_pass_np3), pre-permuted after
    // G_(n)^T.  Lane 4g + c of a warp holds the Kronecker block P_c x Q_c of row g (P_c = 5 (c / 2) + .., Q_c =
    // 5 (c % 2) + .., in lds_block's order: for an odd start the first element comes last); k-step ks = 5 p + q
    // takes column pi(ks, c) = P_c[p] 10 + Q_c[q].  Table at gt + L K: [25][32] = G^T[pi(ks, c)][g], then
    // [25][4][2] = G^T[pi(ks, c)][8 + j].
    if (gt_frag_table(sh)) {
        double* tb = gt + (size_t)L * Kn;
        auto blk5 = [](int st, int i) { const int odd = st & 1; return i == 4 ? (odd ? st : st + 4) : st + odd + i; };
        for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 25 * 32 + 25 * 8; q += gridDim.x * blockDim.x) {
            int ks, c, col;
            if (q < 25 * 32) {
                ks = q / 32;
                const int lane = q % 32;
                c = lane & 3;
                col = lane >> 2;
            } else {
                const int t = q - 25 * 32;
                ks = t / 8;
                c = (t / 2) % 4;
                col = 8 + t % 2;
            }
            const int p = ks / 5, qq = ks % 5;
            const int l = blk5(5 * (c / 2), p) * 10 + blk5(5 * (c % 2), qq);
            size_t lin = (size_t)col * gstride[sh.n];
            int j = 0;
            for (int v = 0; v < order; ++v) {
                if (v == sh.n) continue;
                lin += (size_t)((l / sh.cstride[j]) % sh.ko[j]) * gstride[v];
                ++j;
            }
            tb[q] = core[lin];
        }
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

// the same reduction for a pass over mode n != 0: G_(n) (K_n x L) refolded into the core layout
__global__ void k_reduce_core_refold(const double* __restrict__ mpart, int nslots, ModeShape sh, double* core_out,
                                     const DevStatus* st, int run_if) {
    if (skip_kernel(st, run_if)) return;
    int gstride[kMaxOrder];
    {
        int ks[kMaxOrder];
        int j = 0;
        for (int v = 0; v < sh.order; ++v) ks[v] = (v == sh.n) ? sh.kn : sh.ko[j++];
        int acc = 1;
        for (int v = sh.order - 1; v >= 0; --v) {
            gstride[v] = acc;
            acc *= ks[v];
        }
    }
    const uint64_t size = (uint64_t)sh.kn * sh.L;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < size; q += (uint64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int c = 0; c < nslots; ++c) acc += mpart[(size_t)c * size + q];
        const int r = (int)(q / sh.L), l = (int)(q - (uint64_t)r * sh.L);
        size_t lin = (size_t)r * gstride[sh.n];
        int j = 0;
        for (int v = 0; v < sh.order; ++v) {
            if (v == sh.n) continue;
            lin += (size_t)((l / sh.cstride[j]) % sh.ko[j]) * gstride[v];
            ++j;
        }
        core_out[lin] = acc;
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
                  uint64_t m_rows, cudaStream_t s, bool abort_on_fallback) {
    k_chol1<<<1, 32, 0, s>>>(w, maxv, K, r1inv, st, degenerate_mode, abort_on_fallback ? 1 : 0, m_rows);
    HQ_CHECK_LAUNCH();
}

void launch_gram2(const double* A, uint64_t rows, int K, const double* r1inv, double* wpart, const DevStatus* st,
                  cudaStream_t s) {
    // Q1 = A R1^-1 is not written: the later passes recompute it bit for bit from A
    launch_rowgemm(K, A, rows, r1inv, nullptr, nullptr, wpart, nullptr, st, kOnlyCholQR, s);
}

void launch_chol2(const double* wpart, int nslots, int K, const double* r1inv, double* rinv, double* rc,
                  const double* m, const ModeShape* sh, double* core_out, DevStatus* st, cudaStream_t s,
                  bool abort_on_fallback, int mode1) {
    ModeShape z{};
    k_chol2<<<1, 1024, 0, s>>>(wpart, nslots, K, r1inv, rinv, rc, m, sh ? *sh : z, m != nullptr, core_out, st,
                               abort_on_fallback ? 1 : 0, 2, nullptr, mode1);
    HQ_CHECK_LAUNCH();
}

void launch_gram3(const double* A, uint64_t rows, int K, const double* r1inv, const double* r2inv, double* q_out,
                  double* wpart, const DevStatus* st, cudaStream_t s) {
    RowGemm g{};
    g.A = A;
    g.rows = rows;
    g.T = r1inv;
    g.T2 = r2inv;
    g.out = q_out;
    g.part = wpart;
    g.st = st;
    g.run_if = kOnlyShifted;
    launch_rowgemm(K, g, s);
}

void launch_chol3(const double* wpart, int nslots, int K, const double* rc, double* rinv, const double* wfull,
                  DevStatus* st, cudaStream_t s, bool abort_on_fallback) {
    ModeShape z{};
    k_chol2<<<1, 1024, 0, s>>>(wpart, nslots, K, rc, rinv, nullptr, nullptr, z, 0, nullptr, st,
                               abort_on_fallback ? 1 : 0, 3, wfull, 0);
    HQ_CHECK_LAUNCH();
}

void launch_apply(const double* A, uint64_t rows, int K, const double* rinv, double* u_out, const double* u_old,
                  double* ppart, bool apply, const DevStatus* st, int run_if, cudaStream_t s) {
    if (apply)
        launch_rowgemm(K, A, rows, rinv, u_out, u_old, ppart, nullptr, st, run_if, s);
    else
        launch_rowgemm(K, u_out, rows, nullptr, nullptr, u_old, ppart, nullptr, st, run_if, s);
}

void launch_apply_qr(const double* A, uint64_t rows, int K, const double* r1inv, const double* rinv, double* u_out,
                     const double* u_old, double* ppart, bool shifted_alt, const DevStatus* st, int run_if,
                     cudaStream_t s, double* const* peer_out, int npeer) {
    RowGemm g{};
    if (npeer > kMaxPeers) fail(HQ_ERR_CAPACITY, "more peer replicas than the apply kernel takes");
    for (int r = 0; r < npeer; ++r) g.peer_out[r] = peer_out[r];
    g.npeer = npeer;
    g.A = A;
    g.rows = rows;
    g.T = r1inv;
    g.T2 = rinv;
    g.alt = shifted_alt ? u_out : nullptr;
    g.out = u_out;
    g.other = u_old;
    g.part = ppart;
    g.st = st;
    g.run_if = run_if;
    launch_rowgemm(K, g, s);
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

// multi-GPU continuation (hq_solver.cu): clear the abort the chol kernels raised and arm the Householder
// (kOnlyFallback) kernels for the pending update
__global__ void k_dist_resume(DevStatus* st) {
    st->abort = 0;
    st->pending_mode = 0;
    st->fallback = 1;
    st->shifted = 0;
    st->dist_hh_count++;
}

void launch_dist_resume(DevStatus* st, cudaStream_t s) {
    k_dist_resume<<<1, 1, 0, s>>>(st);
    HQ_CHECK_LAUNCH();
}

void launch_sweep_end(const double* core, uint64_t core_size, double dns, double tol, uint64_t max_sweeps,
                      const SweepTrace& tr, DevStatus* st, cudaStream_t s) {
    k_sweep_end<<<1, 1024, 0, s>>>(core, core_size, dns, tol, max_sweeps, tr, st);
    HQ_CHECK_LAUNCH();
}

void launch_update_diag(const double* w, const double* gt, int K, int L, int mode, int order, const UpdTrace& tr,
                        DevStatus* st, cudaStream_t s) {
    k_update_diag<<<1, 256, 0, s>>>(w, gt, K, L, mode, order, tr, st);
    HQ_CHECK_LAUNCH();
}

void launch_drift_batch(const double* trp, int pairs, int order, const int* ranks_dev, int kmax, double* drift,
                        cudaStream_t s) {
    if (pairs <= 0) return;
    k_drift_batch<<<pairs, 32, 0, s>>>(trp, pairs, order, ranks_dev, kmax, drift);
    HQ_CHECK_LAUNCH();
}

size_t householder_work_doubles(uint64_t rows, int K) {
    return kHhCtlDoubles + hh_part_doubles(num_sms()) + 2 * rows * (uint64_t)K + (size_t)num_sms() * kHhGramSlot;
}

void householder_reset(double* work, cudaStream_t s) { HQ_CUDA(cudaMemsetAsync(work, 0, sizeof(HhCtl), s)); }

void launch_householder(const double* A, uint64_t rows, int K, double* q_out, double* work, const double* table,
                        uint64_t table_len, const DevStatus* st, int run_if, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)num_sms());
    cfg.blockDim = dim3(kHhThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (K <= 8)
        HQ_CUDA(cudaLaunchKernelEx(&cfg, k_householder_mc<8>, A, rows, K, q_out, work, table, table_len, st, run_if));
    else if (K <= 16)
        HQ_CUDA(cudaLaunchKernelEx(&cfg, k_householder_mc<16>, A, rows, K, q_out, work, table, table_len, st, run_if));
    else
        HQ_CUDA(cudaLaunchKernelEx(&cfg, k_householder_mc<32>, A, rows, K, q_out, work, table, table_len, st, run_if));
    HQ_CHECK_LAUNCH();
}

void launch_gt(const double* core, const ModeShape& sh, const int* ranks, double* gt, const DevStatus* st,
               cudaStream_t s) {
    (void)ranks;
    int tot = sh.L * sh.kn + (gt_frag_table(sh) ? kGtFragTable : 0);
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

void launch_reduce_core_mode(const double* mpart, int nslots, const ModeShape& sh, double* core_out,
                             const DevStatus* st, int run_if, cudaStream_t s) {
    const uint64_t size = (uint64_t)sh.kn * sh.L;
    if (sh.n == 0) {
        launch_reduce_core(mpart, nslots, size, core_out, st, run_if, s);
        return;
    }
    int blocks = (int)std::max<uint64_t>(1, std::min<uint64_t>((size + 255) / 256, (uint64_t)num_sms() * 4));
    k_reduce_core_refold<<<blocks, 256, 0, s>>>(mpart, nslots, sh, core_out, st, run_if);
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
