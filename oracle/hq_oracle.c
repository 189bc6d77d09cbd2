/*
 * hq_oracle.c — CPU restatement of the reference HOQRI hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2510_16930_b200/,
 * include/) may link, load or call this file.  Only tests/, the smoke check in
 * __graft_entry__.py and bench.py's cpu_baseline leg use it, and only as the
 * checker.  It is pinned against the reference itself: tests/golden/ holds
 * vectors produced by the reference library compiled from
 * /root/reference/proj/src (oracle/Makefile -> oracle/_ref/), and
 * tests/test_oracle_golden.py checks this file against them.
 *
 * Every function cites the reference file:line it restates.  Paths are
 * relative to /root/reference/proj.
 *
 * Conventions (same as the reference):
 *   coords   uint32, AoS, coords[e*N + m]          (include/tucker/sparse_tensor.hpp:46-51)
 *   factors  row-major I_n x K_n, concatenated per mode in mode order
 *   core     K_1 x ... x K_N, last mode fastest   (include/tucker/dense_core.hpp:118-128)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define HQO_OK 0
#define HQO_ERR_SHAPE 1
#define HQO_ERR_RANGE 2
#define HQO_ERR_VALUE 3
#define HQO_ERR_CONTRACT 6
#define HQO_ERR_DIAGNOSTIC 7
#define HQO_ERR_DEGENERATE 8

/* ------------------------------------------------------------------ RNG --
 * include/tucker/rng.hpp:13-54: std::mt19937_64 (standard-specified), then
 * uniform01 = (raw >> 11) * 2^-53, Box-Muller normal with a cached spare,
 * rejection uniform_below.  mt19937_64 is restated from its published
 * definition (Matsumoto & Nishimura 2000; C++ [rand.eng.mers] parameters). */

typedef struct {
    uint64_t mt[312];
    int idx;
    int has_spare;
    double spare;
} hqo_rng;

void hqo_rng_seed(hqo_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
    r->has_spare = 0;
    r->spare = 0.0;
}

uint64_t hqo_rng_raw(hqo_rng* r) {
    const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % 312] & lower);
            uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1ull) v ^= 0xB5026F5AA96619E9ull;
            r->mt[i] = v;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= (y >> 43);
    return y;
}

double hqo_rng_uniform01(hqo_rng* r) {  /* rng.hpp:19-21 */
    return (double)(hqo_rng_raw(r) >> 11) * 0x1.0p-53;
}

double hqo_rng_normal(hqo_rng* r) {  /* rng.hpp:24-35 */
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = 1.0 - hqo_rng_uniform01(r);
    double u2 = hqo_rng_uniform01(r);
    double rad = sqrt(-2.0 * log(u1));
    double theta = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(theta);
    r->has_spare = 1;
    return rad * cos(theta);
}

uint64_t hqo_rng_uniform_below(hqo_rng* r, uint64_t n) {  /* rng.hpp:38-46 */
    if (n <= 1) return 0;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do {
        x = hqo_rng_raw(r);
    } while (x >= limit);
    return x % n;
}

uint64_t hqo_mix_seed(uint64_t seed, uint64_t salt) {  /* rng.hpp:57-62 (splitmix64) */
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (salt + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* n raw draws / normals from a fresh generator (for golden checks) */
void hqo_raw_stream(uint64_t seed, uint64_t n, uint64_t* out) {
    hqo_rng r;
    hqo_rng_seed(&r, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = hqo_rng_raw(&r);
}

void hqo_normal_stream(uint64_t seed, uint64_t n, double* out) {
    hqo_rng r;
    hqo_rng_seed(&r, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = hqo_rng_normal(&r);
}

/* ------------------------------------------------------- sparse tensor --
 * src/sparse_tensor.cpp:18-41 validation, :43-71 lexicographic sort and
 * duplicate merge, :73-89 per-mode buckets (stable counting sort). */

static int g_sort_n;
static const uint32_t* g_sort_c;

static int lex_cmp(const void* pa, const void* pb) {
    uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
    const uint32_t* ca = g_sort_c + a * (uint64_t)g_sort_n;
    const uint32_t* cb = g_sort_c + b * (uint64_t)g_sort_n;
    for (int m = 0; m < g_sort_n; ++m) {
        if (ca[m] < cb[m]) return -1;
        if (ca[m] > cb[m]) return 1;
    }
    return (a < b) ? -1 : (a > b);  /* ties in input order */
}

/* Validates like sparse_tensor.cpp:22-38 and reports the first offending
 * entry through bad_entry/bad_mode.  Returns HQO_ERR_* or HQO_OK. */
int hqo_validate(int N, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                 const double* vals, uint64_t* bad_entry, int* bad_mode) {
    if (N <= 0) return HQO_ERR_SHAPE;
    for (int m = 0; m < N; ++m)
        if (dims[m] == 0) return HQO_ERR_SHAPE;
    for (uint64_t e = 0; e < nnz; ++e) {
        for (int m = 0; m < N; ++m) {
            if ((uint64_t)coords[e * N + m] >= dims[m]) {
                *bad_entry = e;
                *bad_mode = m;
                return HQO_ERR_RANGE;
            }
        }
        if (!isfinite(vals[e])) {
            *bad_entry = e;
            *bad_mode = -1;
            return HQO_ERR_VALUE;
        }
    }
    return HQO_OK;
}

/* sparse_tensor.cpp:43-71.  out_coords/out_vals sized for nnz entries. */
int hqo_normalize(int N, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                  const double* vals, uint32_t* out_coords, double* out_vals,
                  uint64_t* out_nnz) {
    uint64_t be = 0;
    int bm = 0;
    int st = hqo_validate(N, dims, nnz, coords, vals, &be, &bm);
    if (st) return st;
    uint64_t* perm = (uint64_t*)malloc(sizeof(uint64_t) * (nnz ? nnz : 1));
    for (uint64_t i = 0; i < nnz; ++i) perm[i] = i;
    g_sort_n = N;
    g_sort_c = coords;
    qsort(perm, nnz, sizeof(uint64_t), lex_cmp);
    uint64_t u = 0;
    for (uint64_t p = 0; p < nnz; ++p) {
        const uint32_t* row = coords + perm[p] * N;
        int dup = (u > 0) && memcmp(row, out_coords + (u - 1) * N, sizeof(uint32_t) * N) == 0;
        if (dup) {
            out_vals[u - 1] += vals[perm[p]];
        } else {
            memcpy(out_coords + u * N, row, sizeof(uint32_t) * N);
            out_vals[u] = vals[perm[p]];
            ++u;
        }
    }
    free(perm);
    *out_nnz = u;
    return HQO_OK;
}

/* sparse_tensor.cpp:73-89 for one mode; offsets has dims[mode]+1 slots. */
void hqo_buckets(int N, const uint64_t* dims, uint64_t nnz, const uint32_t* coords,
                 int mode, uint64_t* offsets, uint64_t* entries) {
    uint64_t I = dims[mode];
    memset(offsets, 0, sizeof(uint64_t) * (I + 1));
    for (uint64_t e = 0; e < nnz; ++e) ++offsets[coords[e * N + mode] + 1];
    for (uint64_t i = 0; i < I; ++i) offsets[i + 1] += offsets[i];
    uint64_t* cursor = (uint64_t*)malloc(sizeof(uint64_t) * (I ? I : 1));
    memcpy(cursor, offsets, sizeof(uint64_t) * I);
    for (uint64_t e = 0; e < nnz; ++e) entries[cursor[coords[e * N + mode]]++] = e;
    free(cursor);
}

double hqo_norm_sq(uint64_t nnz, const double* vals) {  /* sparse_tensor.cpp:91-95 */
    double s = 0.0;
    for (uint64_t e = 0; e < nnz; ++e) s += vals[e] * vals[e];
    return s;
}

/* ------------------------------------------------------------- kernels -- */

static void factor_offsets(int N, const uint64_t* dims, const uint64_t* ranks, uint64_t* off) {
    uint64_t o = 0;
    for (int v = 0; v < N; ++v) {
        off[v] = o;
        o += dims[v] * ranks[v];
    }
}

static uint64_t prod_ranks(int N, const uint64_t* ranks) {
    uint64_t p = 1;
    for (int v = 0; v < N; ++v) p *= ranks[v];
    return p;
}

/* src/kernels.cpp:40-84: per-nonzero rank-1 outer product over all modes,
 * odometer over the rank tuple with the last mode fastest. */
void hqo_ttmc_core(int N, const uint64_t* dims, const uint64_t* ranks, uint64_t nnz,
                   const uint32_t* coords, const double* vals, const double* factors,
                   double* core) {
    uint64_t off[16], stride[16], idx[16];
    const double* w[16];
    factor_offsets(N, dims, ranks, off);
    uint64_t total = prod_ranks(N, ranks);
    memset(core, 0, sizeof(double) * total);
    stride[N - 1] = 1;
    for (int v = N - 1; v > 0; --v) stride[v - 1] = stride[v] * ranks[v];
    const int last = N - 1;
    for (uint64_t e = 0; e < nnz; ++e) {
        const double xv = vals[e];
        const uint32_t* c = coords + e * N;
        for (int v = 0; v < N; ++v) w[v] = factors + off[v] + (uint64_t)c[v] * ranks[v];
        for (int v = 0; v < N; ++v) idx[v] = 0;
        for (;;) {
            double p = xv;
            uint64_t base = 0;
            for (int v = 0; v < last; ++v) {
                p *= w[v][idx[v]];
                base += idx[v] * stride[v];
            }
            for (uint64_t k = 0; k < ranks[last]; ++k) core[base + k] += p * w[last][k];
            if (N == 1) break;
            int v = last, done = 0;
            while (v-- > 0) {
                if (++idx[v] < ranks[v]) break;
                idx[v] = 0;
                if (v == 0) done = 1;
            }
            if (done) break;
        }
    }
}

/* src/kernels.cpp:86-163 (Alg. 3): nonzeros outermost, rank tuples inner. */
void hqo_ttmctc(int N, const uint64_t* dims, const uint64_t* ranks, uint64_t nnz,
                const uint32_t* coords, const double* vals, const double* factors, int mode,
                const double* core, double* A) {
    uint64_t off[16], stride[16], idx[16];
    const double* w[16];
    factor_offsets(N, dims, ranks, off);
    memset(A, 0, sizeof(double) * dims[mode] * ranks[mode]);
    stride[N - 1] = 1;
    for (int v = N - 1; v > 0; --v) stride[v - 1] = stride[v] * ranks[v];
    const int last = N - 1;
    const uint64_t kn = ranks[mode];
    for (uint64_t e = 0; e < nnz; ++e) {
        const double xv = vals[e];
        const uint32_t* c = coords + e * N;
        for (int v = 0; v < N; ++v) w[v] = factors + off[v] + (uint64_t)c[v] * ranks[v];
        double* arow = A + (uint64_t)c[mode] * kn;
        for (int v = 0; v < N; ++v) idx[v] = 0;
        for (;;) {
            double p = xv;
            uint64_t base = 0;
            for (int v = 0; v < last; ++v) {
                if (v != mode) p *= w[v][idx[v]];
                base += idx[v] * stride[v];
            }
            const double* gb = core + base;
            if (mode == last) {
                for (uint64_t k = 0; k < ranks[last]; ++k) arow[k] += p * gb[k];
            } else {
                double s = 0.0;
                for (uint64_t k = 0; k < ranks[last]; ++k) s += w[last][k] * gb[k];
                arow[idx[mode]] += p * s;
            }
            if (N == 1) break;
            int v = last, done = 0;
            while (v-- > 0) {
                if (++idx[v] < ranks[v]) break;
                idx[v] = 0;
                if (v == 0) done = 1;
            }
            if (done) break;
        }
    }
}

/* --------------------------------------------------------- dense core --
 * src/dense_core.cpp:127-198: Householder thin QR, sign convention R_kk >= 0,
 * pivots <= 1e-12 ||A||_F replaced by seeded random directions
 * (kDeficiencySeed = 0x48514F5251, dense_core.cpp:14). */

#define HQO_DEFICIENCY_SEED 0x48514F5251ull

int hqo_qr(uint64_t m, uint64_t n, const double* a, double* q) {
    if (m < n) return HQO_ERR_SHAPE;
    if (n == 0) return HQO_OK;
    double* w = (double*)malloc(sizeof(double) * m * n);
    memcpy(w, a, sizeof(double) * m * n);
    double anorm = 0.0;
    for (uint64_t i = 0; i < m * n; ++i) anorm += a[i] * a[i];
    anorm = sqrt(anorm);
    const double pivot_tol = 1e-12 * anorm;
    double* refl = (double*)malloc(sizeof(double) * m * n);  /* reflector k in refl[k*m ..] */
    double* betas = (double*)calloc(n, sizeof(double));
    int* flip = (int*)calloc(n, sizeof(int));
    hqo_rng rng;
    hqo_rng_seed(&rng, HQO_DEFICIENCY_SEED);
#define W(i, j) w[(i) * n + (j)]
    for (uint64_t k = 0; k < n; ++k) {
        double normx = 0.0;
        for (uint64_t i = k; i < m; ++i) normx += W(i, k) * W(i, k);
        normx = sqrt(normx);
        if (normx <= pivot_tol) {
            do {
                normx = 0.0;
                for (uint64_t i = k; i < m; ++i) {
                    W(i, k) = hqo_rng_normal(&rng);
                    normx += W(i, k) * W(i, k);
                }
                normx = sqrt(normx);
            } while (normx == 0.0);
        }
        double x0 = W(k, k);
        double alpha = (x0 >= 0.0) ? -normx : normx;
        double* v = refl + k * m;
        v[0] = x0 - alpha;
        for (uint64_t i = k + 1; i < m; ++i) v[i - k] = W(i, k);
        double vn2 = 0.0;
        for (uint64_t i = 0; i < m - k; ++i) vn2 += v[i] * v[i];
        double beta = (vn2 > 0.0) ? 2.0 / vn2 : 0.0;
        for (uint64_t j = k; j < n; ++j) {
            double dot = 0.0;
            for (uint64_t i = k; i < m; ++i) dot += v[i - k] * W(i, j);
            dot *= beta;
            for (uint64_t i = k; i < m; ++i) W(i, j) -= dot * v[i - k];
        }
        W(k, k) = alpha;
        flip[k] = alpha < 0.0;
        betas[k] = beta;
    }
#undef W
#define Q(i, j) q[(i) * n + (j)]
    memset(q, 0, sizeof(double) * m * n);
    for (uint64_t k = 0; k < n; ++k) Q(k, k) = 1.0;
    for (uint64_t kk = n; kk-- > 0;) {
        const double* v = refl + kk * m;
        double beta = betas[kk];
        if (beta == 0.0) continue;
        for (uint64_t j = kk; j < n; ++j) {
            double dot = 0.0;
            for (uint64_t i = kk; i < m; ++i) dot += v[i - kk] * Q(i, j);
            dot *= beta;
            for (uint64_t i = kk; i < m; ++i) Q(i, j) -= dot * v[i - kk];
        }
    }
    for (uint64_t k = 0; k < n; ++k) {
        if (!flip[k]) continue;
        for (uint64_t i = 0; i < m; ++i) Q(i, k) = -Q(i, k);
    }
#undef Q
    free(w);
    free(refl);
    free(betas);
    free(flip);
    return HQO_OK;
}

/* dense_core.cpp:200-264: cyclic Jacobi on a symmetric n x n matrix (in
 * place), eigenvalues returned descending (stable sort). */
void hqo_jacobi_eigvals(uint64_t n, double* m, double* evals) {
#define M(i, j) m[(i) * n + (j)]
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = i + 1; j < n; ++j) {
            double avg = 0.5 * (M(i, j) + M(j, i));
            M(i, j) = M(j, i) = avg;
        }
    double fnorm = 0.0;
    for (uint64_t i = 0; i < n * n; ++i) fnorm += m[i] * m[i];
    fnorm = sqrt(fnorm);
    const double stop = 1e-15 * (fnorm > 0.0 ? fnorm : 1.0);
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0;
        for (uint64_t p = 0; p < n; ++p)
            for (uint64_t q = p + 1; q < n; ++q) off += M(p, q) * M(p, q);
        if (sqrt(2.0 * off) <= stop) break;
        for (uint64_t p = 0; p < n; ++p) {
            for (uint64_t q = p + 1; q < n; ++q) {
                double apq = M(p, q);
                if (fabs(apq) <= 1e-300) continue;
                double theta = (M(q, q) - M(p, p)) / (2.0 * apq);
                double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0);
                double s = t * c;
                double tau = s / (1.0 + c);
                double app = M(p, p), aqq = M(q, q);
                M(p, p) = app - t * apq;
                M(q, q) = aqq + t * apq;
                M(p, q) = M(q, p) = 0.0;
                for (uint64_t r = 0; r < n; ++r) {
                    if (r != p && r != q) {
                        double arp = M(r, p), arq = M(r, q);
                        M(r, p) = M(p, r) = arp - s * (arq + tau * arp);
                        M(r, q) = M(q, r) = arq + s * (arp - tau * arq);
                    }
                }
            }
        }
    }
    for (uint64_t i = 0; i < n; ++i) evals[i] = M(i, i);
    /* stable descending insertion sort (dense_core.cpp:251-254) */
    for (uint64_t i = 1; i < n; ++i) {
        double x = evals[i];
        uint64_t j = i;
        while (j > 0 && evals[j - 1] < x) {
            evals[j] = evals[j - 1];
            --j;
        }
        evals[j] = x;
    }
#undef M
}

/* manifold.cpp:55-60 -> dense_core.cpp:329-335: 2K - 2 * nuclear(U^T V). */
double hqo_subspace_distance(uint64_t m, uint64_t k, const double* u, const double* v) {
    double* p = (double*)calloc(k * k, sizeof(double));
    double* g = (double*)calloc(k * k, sizeof(double));
    double* ev = (double*)calloc(k, sizeof(double));
    for (uint64_t r = 0; r < m; ++r)  /* matmul_tn order (dense_core.cpp:47-61) */
        for (uint64_t i = 0; i < k; ++i) {
            double ui = u[r * k + i];
            if (ui == 0.0) continue;
            for (uint64_t j = 0; j < k; ++j) p[i * k + j] += ui * v[r * k + j];
        }
    for (uint64_t r = 0; r < k; ++r)
        for (uint64_t i = 0; i < k; ++i) {
            double pi = p[r * k + i];
            if (pi == 0.0) continue;
            for (uint64_t j = 0; j < k; ++j) g[i * k + j] += pi * p[r * k + j];
        }
    hqo_jacobi_eigvals(k, g, ev);
    double s = 0.0;
    for (uint64_t i = 0; i < k; ++i) s += sqrt(ev[i] > 0.0 ? ev[i] : 0.0);
    free(p);
    free(g);
    free(ev);
    double d = 2.0 * (double)k - 2.0 * s;
    return d > 0.0 ? d : 0.0;
}

/* max_n max_ij |U^T U - I| (dense_core.cpp:116-125) */
double hqo_orthonormality_defect(int N, const uint64_t* dims, const uint64_t* ranks,
                                 const double* factors) {
    uint64_t off[16];
    factor_offsets(N, dims, ranks, off);
    double worst = 0.0;
    for (int v = 0; v < N; ++v) {
        uint64_t k = ranks[v];
        for (uint64_t i = 0; i < k; ++i)
            for (uint64_t j = 0; j < k; ++j) {
                double s = 0.0;
                for (uint64_t r = 0; r < dims[v]; ++r)
                    s += factors[off[v] + r * k + i] * factors[off[v] + r * k + j];
                double d = fabs(s - (i == j ? 1.0 : 0.0));
                if (d > worst) worst = d;
            }
    }
    return worst;
}

/* solvers.cpp:182-195: per mode Rng(mix_seed(seed, n)), row-major normals,
 * then qr_orthonormal. */
int hqo_random_factors(int N, const uint64_t* dims, const uint64_t* ranks, uint64_t seed,
                       double* out) {
    uint64_t off[16];
    factor_offsets(N, dims, ranks, off);
    for (int n = 0; n < N; ++n) {
        if (ranks[n] > dims[n]) return HQO_ERR_SHAPE;
        hqo_rng r;
        hqo_rng_seed(&r, hqo_mix_seed(seed, (uint64_t)n));
        uint64_t cnt = dims[n] * ranks[n];
        double* g = (double*)malloc(sizeof(double) * (cnt ? cnt : 1));
        for (uint64_t i = 0; i < cnt; ++i) g[i] = hqo_rng_normal(&r);
        int st = hqo_qr(dims[n], ranks[n], g, out + off[n]);
        free(g);
        if (st) return st;
    }
    return HQO_OK;
}

/* ------------------------------------------------- gradient diagnostics --
 * unfold_core (dense_core.cpp:350-369): G_(n) is K_n x L, column
 * sum_{v != n} k_v * stride_v with the last other mode fastest. */
static void unfold_core(int N, const uint64_t* ranks, int n, const double* core, double* gn) {
    uint64_t L = prod_ranks(N, ranks) / ranks[n];
    uint64_t stride[16];
    uint64_t sacc = 1;
    for (int v = N - 1; v >= 0; --v) {
        if (v == n) continue;
        stride[v] = sacc;
        sacc *= ranks[v];
    }
    uint64_t idx[16] = {0};
    uint64_t size = prod_ranks(N, ranks);
    for (uint64_t lin = 0; lin < size; ++lin) {
        uint64_t col = 0;
        for (int v = 0; v < N; ++v)
            if (v != n) col += idx[v] * stride[v];
        gn[idx[n] * L + col] = core[lin];
        for (int v = N - 1; v >= 0; --v) {
            if (++idx[v] < ranks[v]) break;
            idx[v] = 0;
        }
    }
}

/* gram_eigvals_desc (dense_core.cpp:371-386); m is consumed.  Returns
 * HQO_ERR_CONTRACT when not symmetric / not PSD. */
static int gram_eigvals_desc(uint64_t k, double* m, double* ev) {
    double fro = 0.0;
    for (uint64_t i = 0; i < k * k; ++i) fro += m[i] * m[i];
    double scale = sqrt(fro) > 1.0 ? sqrt(fro) : 1.0;
    for (uint64_t i = 0; i < k; ++i)
        for (uint64_t j = i + 1; j < k; ++j)
            if (fabs(m[i * k + j] - m[j * k + i]) > 1e-10 * scale) return HQO_ERR_CONTRACT;
    hqo_jacobi_eigvals(k, m, ev);
    for (uint64_t i = 0; i < k; ++i) {
        if (ev[i] < -1e-10 * scale) return HQO_ERR_CONTRACT;
        if (ev[i] < 0.0) ev[i] = 0.0;
    }
    return HQO_OK;
}

/* diagnose_update (solvers.cpp:39-46) = grad_norm_sq (manifold.cpp:37-55) +
 * interlacing_check (manifold.cpp:63-84) for A (m x k) and G_(n) (k x L). */
int hqo_update_diag(uint64_t m, uint64_t k, const double* a, uint64_t L, const double* gn, double* grad,
                    double* sigma, double* lambda, int* bad_k) {
    *bad_k = 0;
    double a_sq = 0.0;
    for (uint64_t i = 0; i < m * k; ++i) a_sq += a[i] * a[i];
    double* gg = (double*)calloc(k * k, sizeof(double));
    double* ata = (double*)calloc(k * k, sizeof(double));
    for (uint64_t i = 0; i < k; ++i) /* matmul_nt (dense_core.cpp:63-77) */
        for (uint64_t j = 0; j < k; ++j) {
            double acc = 0.0;
            for (uint64_t l = 0; l < L; ++l) acc += gn[i * L + l] * gn[j * L + l];
            gg[i * k + j] = acc;
        }
    double gg_sq = 0.0;
    for (uint64_t i = 0; i < k * k; ++i) gg_sq += gg[i] * gg[i];
    double r = 4.0 * (a_sq - gg_sq);
    double scale = 4.0 * a_sq > 1.0 ? 4.0 * a_sq : 1.0;
    int st = HQO_OK;
    if (r < -1e-8 * scale) {
        st = HQO_ERR_DIAGNOSTIC;
        goto out;
    }
    *grad = (fabs(r) <= 1e-10) ? 0.0 : (r > 0.0 ? r : 0.0);
    for (uint64_t row = 0; row < m; ++row) /* matmul_tn (dense_core.cpp:47-61) */
        for (uint64_t i = 0; i < k; ++i) {
            double ai = a[row * k + i];
            if (ai == 0.0) continue;
            for (uint64_t j = 0; j < k; ++j) ata[i * k + j] += ai * a[row * k + j];
        }
    st = gram_eigvals_desc(k, ata, sigma);
    if (st) goto out;
    for (uint64_t i = 0; i < k; ++i) sigma[i] = sqrt(sigma[i]);
    st = gram_eigvals_desc(k, gg, lambda);
    if (st) goto out;
    {
        double sc = (k && sigma[0] > 1.0) ? sigma[0] : 1.0;
        for (uint64_t i = 0; i < k; ++i)
            if (sigma[i] - lambda[i] < -1e-9 * sc) {
                *bad_k = (int)i + 1;
                st = HQO_ERR_DIAGNOSTIC;
                goto out;
            }
    }
out:
    free(gg);
    free(ata);
    return st;
}

/* ---------------------------------------------------------------- solve --
 * solvers.cpp:50-178 for HOQRI with the element-wise kernel (core kept fresh
 * after every mode update, solvers.cpp:73-74, 143-144), no gradient tracing.
 * Inputs must already be normalised (hqo_normalize).  Outputs:
 *   factors_io   in: initial factors (init_factors result); out: final factors
 *   core_out     final core (fresh, solvers.cpp:174-177)
 *   sweeps_done, objective[s], fit[s], drift[s*N + n]
 *   core_snap    optional, core after each sweep  (max_sweeps * prod K)
 *   factor_snap  optional, factors after each sweep (max_sweeps * sum I_n K_n)
 * Returns HQO_ERR_DEGENERATE with *degenerate_mode (1-based) on A == 0
 * (solvers.cpp:124). */
typedef struct hqo_trace_out {
    double tol_grad;  /* solvers.cpp:165-167 */
    uint64_t ks;      /* row stride of sigma / lambda */
    double* grad;     /* [max_sweeps * N] */
    double* f_before;
    double* f_after;
    double* sigma;    /* [max_sweeps * N * ks] */
    double* lambda;
    uint64_t* updates;
    int* bad_k;
} hqo_trace_out;

static int hoqri_impl(int N, const uint64_t* dims, const uint64_t* ranks, uint64_t nnz, const uint32_t* coords,
                      const double* vals, double* factors_io, uint64_t max_sweeps, double tol_fit_change,
                      double* core_out, uint64_t* sweeps_done, double* initial_objective, double* objective,
                      double* fit, double* drift, double* core_snap, double* factor_snap, int* degenerate_mode,
                      const hqo_trace_out* tr) {
    uint64_t off[16];
    factor_offsets(N, dims, ranks, off);
    uint64_t total_f = off[N - 1] + dims[N - 1] * ranks[N - 1];
    uint64_t pk = prod_ranks(N, ranks);
    uint64_t maxa = 0;
    for (int v = 0; v < N; ++v)
        if (dims[v] * ranks[v] > maxa) maxa = dims[v] * ranks[v];
    double* a = (double*)malloc(sizeof(double) * (maxa ? maxa : 1));
    double* qn = (double*)malloc(sizeof(double) * (maxa ? maxa : 1));
    const double dns = hqo_norm_sq(nnz, vals);
    hqo_ttmc_core(N, dims, ranks, nnz, coords, vals, factors_io, core_out);
    double f0 = hqo_norm_sq(pk, core_out);
    *initial_objective = f0;
    double fit_prev = dns - f0;
    *sweeps_done = 0;
    int st = HQO_OK;
    double* gn = (double*)malloc(sizeof(double) * (pk ? pk : 1));
    if (tr) *tr->updates = 0;
    for (uint64_t sweep = 1; sweep <= max_sweeps; ++sweep) {
        double total_g = 0.0;
        for (int n = 0; n < N; ++n) {
            const uint64_t u = (sweep - 1) * N + n;
            hqo_ttmctc(N, dims, ranks, nnz, coords, vals, factors_io, n, core_out, a);
            double mx = 0.0;
            for (uint64_t i = 0; i < dims[n] * ranks[n]; ++i)
                if (fabs(a[i]) > mx) mx = fabs(a[i]);
            if (mx == 0.0) {
                *degenerate_mode = n + 1;
                st = HQO_ERR_DEGENERATE;
                goto done;
            }
            if (tr) { /* solvers.cpp:126-137: diagnostics at the pre-update state */
                tr->f_before[u] = hqo_norm_sq(pk, core_out);
                unfold_core(N, ranks, n, core_out, gn);
                st = hqo_update_diag(dims[n], ranks[n], a, pk / ranks[n], gn, &tr->grad[u], tr->sigma + u * tr->ks,
                                     tr->lambda + u * tr->ks, tr->bad_k);
                if (st) goto done;
                total_g += tr->grad[u];
            }
            hqo_qr(dims[n], ranks[n], a, qn);
            drift[(sweep - 1) * N + n] =
                hqo_subspace_distance(dims[n], ranks[n], qn, factors_io + off[n]);
            memcpy(factors_io + off[n], qn, sizeof(double) * dims[n] * ranks[n]);
            hqo_ttmc_core(N, dims, ranks, nnz, coords, vals, factors_io, core_out);
            if (tr) {
                tr->f_after[u] = hqo_norm_sq(pk, core_out);
                *tr->updates = u + 1;
            }
        }
        double obj = hqo_norm_sq(pk, core_out);
        objective[sweep - 1] = obj;
        fit[sweep - 1] = dns - obj;
        *sweeps_done = sweep;
        if (core_snap) memcpy(core_snap + (sweep - 1) * pk, core_out, sizeof(double) * pk);
        if (factor_snap)
            memcpy(factor_snap + (sweep - 1) * total_f, factors_io, sizeof(double) * total_f);
        if (fabs(fit_prev - (dns - obj)) < tol_fit_change) break;
        if (tr && tr->tol_grad > 0.0 && sqrt(total_g) <= tr->tol_grad * (obj > 1e-300 ? obj : 1e-300)) break;
        fit_prev = dns - obj;
    }
done:
    free(a);
    free(qn);
    free(gn);
    return st;
}

int hqo_hoqri(int N, const uint64_t* dims, const uint64_t* ranks, uint64_t nnz,
              const uint32_t* coords, const double* vals, double* factors_io,
              uint64_t max_sweeps, double tol_fit_change, double* core_out,
              uint64_t* sweeps_done, double* initial_objective, double* objective,
              double* fit, double* drift, double* core_snap, double* factor_snap,
              int* degenerate_mode) {
    return hoqri_impl(N, dims, ranks, nnz, coords, vals, factors_io, max_sweeps, tol_fit_change, core_out,
                      sweeps_done, initial_objective, objective, fit, drift, core_snap, factor_snap, degenerate_mode,
                      NULL);
}

/* hqo_hoqri with gradient tracing (trace_gradients / tol_grad > 0,
 * solvers.cpp:58, 126-137, 146-150, 165-167): per update u = (sweep-1)*N + n
 * grad, f_before, f_after, sigma / lambda (stride ks).  Returns
 * HQO_ERR_DIAGNOSTIC (bad_k = 1-based interlacing index, 0 for a negative
 * gradient) or HQO_ERR_CONTRACT like the reference. */
int hqo_hoqri_traced(int N, const uint64_t* dims, const uint64_t* ranks, uint64_t nnz, const uint32_t* coords,
                     const double* vals, double* factors_io, uint64_t max_sweeps, double tol_fit_change,
                     double tol_grad, uint64_t ks, double* core_out, uint64_t* sweeps_done,
                     double* initial_objective, double* objective, double* fit, double* drift, double* grad,
                     double* f_before, double* f_after, double* sigma, double* lambda, uint64_t* updates,
                     int* degenerate_mode, int* bad_k) {
    hqo_trace_out tr = {tol_grad, ks, grad, f_before, f_after, sigma, lambda, updates, bad_k};
    return hoqri_impl(N, dims, ranks, nnz, coords, vals, factors_io, max_sweeps, tol_fit_change, core_out,
                      sweeps_done, initial_objective, objective, fit, drift, NULL, NULL, degenerate_mode, &tr);
}

/* solvers.cpp:225-236 */
int hqo_fit_error(double data_norm_sq, uint64_t pk, const double* core, double* out) {
    double r = data_norm_sq - hqo_norm_sq(pk, core);
    double scale = data_norm_sq > 1.0 ? data_norm_sq : 1.0;
    if (r < -1e-8 * scale) return 6; /* ContractError */
    if (fabs(r) <= 1e-10 * scale) {
        *out = 0.0;
        return HQO_OK;
    }
    *out = r > 0.0 ? r : 0.0;
    return HQO_OK;
}
