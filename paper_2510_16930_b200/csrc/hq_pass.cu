// hq_pass.cu — the sparse passes over a mode-sorted stream.
//
// One pass over mode n computes, for every row i of the mode-n unfolding,
//   Y_i = sum_{e in row i} x_e (kron_{v != n} U_v[c_v(e), :])        (1 x L)
// and from it either the TTMcTC output row a_i = Y_i G_(n)^T (Alg. 3 result,
// proj/src/kernels.cpp:86-163) or, for the core update, a_i = U_n[i, :]
// (then sum_i a_i^T Y_i = G_(n), proj/src/kernels.cpp:40-84).  Every pass also
// accumulates M = sum_i a_i^T Y_i, W = sum_i a_i^T a_i and max|a_i| into
// per-CTA partial slots that a fixed-order reduction combines: no float
// atomics anywhere, so results are bitwise run-to-run deterministic
// (kernels_test.cpp:192-203, solvers_test.cpp:295-310).
//
// This file holds the work planner and the generic (any order, any ranks)
// kernels; hq_pass_fast.cu holds the specialised kernels for the benchmark
// shapes.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "hq_fast.cuh"
#include "hq_long.cuh"
#include "hq_plan.cuh"

namespace hq {

ModeShape make_mode_shape(int order, const int* ranks, int n) {
    ModeShape sh{};
    sh.order = order;
    sh.n = n;
    sh.kn = ranks[n];
    sh.nothers = order - 1;
    int j = 0;
    for (int v = 0; v < order; ++v)
        if (v != n) sh.ko[j++] = ranks[v];
    int s = 1;
    for (int q = sh.nothers - 1; q >= 0; --q) {
        sh.cstride[q] = s;
        s *= sh.ko[q];
    }
    sh.L = s;
    return sh;
}

// ------------------------------------------------------------------ plan --
namespace {

__global__ void k_long_flags(const int64_t* __restrict__ rowptr, uint64_t rows, uint32_t* __restrict__ flag,
                             uint32_t* __restrict__ nseg, int64_t hot_len, unsigned long long* __restrict__ hot_nnz) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows; i += (uint64_t)gridDim.x * blockDim.x) {
        int64_t len = rowptr[i + 1] - rowptr[i];
        bool lng = len > kShortMax;
        flag[i] = lng;
        nseg[i] = lng ? (uint32_t)((len + kSegLen - 1) / kSegLen) : 0u;
        if (len > hot_len) atomicAdd(hot_nnz, (unsigned long long)len);  // integer: order-independent
    }
}

__global__ void k_tile_max(const int64_t* __restrict__ rowptr, uint64_t rows, unsigned long long* __restrict__ out) {
    const uint64_t nt = (rows + 31) / 32;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nt; t += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long s = 0;
        const uint64_t e = min(rows, t * 32 + 32);
        for (uint64_t i = t * 32; i < e; ++i) {
            const int64_t len = rowptr[i + 1] - rowptr[i];
            if (len <= kShortMax) s += (unsigned long long)len;
        }
        atomicMax(out, s);
    }
}

__global__ void k_long_compact(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                               const uint32_t* __restrict__ nseg, const uint32_t* __restrict__ segpos, uint64_t rows,
                               uint32_t* __restrict__ ids, int64_t* __restrict__ segptr) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows; i += (uint64_t)gridDim.x * blockDim.x) {
        if (flag[i]) {
            ids[pos[i]] = (uint32_t)i;
            segptr[pos[i]] = segpos[i];
        }
    }
}

__global__ void k_long_segments(const int64_t* __restrict__ rowptr, const uint32_t* __restrict__ ids,
                                const int64_t* __restrict__ segptr, uint64_t nlong, int64_t* __restrict__ seg_begin,
                                uint32_t* __restrict__ seg_row) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nlong; r += (uint64_t)gridDim.x * blockDim.x) {
        int64_t b = rowptr[ids[r]], e = rowptr[ids[r] + 1];
        int64_t s = segptr[r];
        for (int64_t p = b; p < e; p += kSegLen, ++s) {
            seg_begin[s] = p;
            seg_row[s] = (uint32_t)r;
        }
    }
}

template <class T>
void exclusive_scan(const T* in, T* out, uint64_t n, cudaStream_t s) {
    size_t tmp = 0;
    HQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, s));
    DBuf<uint8_t> t;
    t.alloc(tmp ? tmp : 1);
    HQ_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, (int)n, s));
}

inline int grid_for(uint64_t n, int threads = 256) {
    uint64_t b = ceil_div(n ? n : 1, threads);
    return (int)std::min<uint64_t>(std::max<uint64_t>(b, 1), (uint64_t)num_sms() * 16);
}

}  // namespace

void plan_mode(ModeLayout& L, uint64_t nnz, cudaStream_t s) {
    const uint64_t rows = L.rows;
    DBuf<uint32_t> flag, nseg, pos, segpos;
    DBuf<unsigned long long> hot;
    flag.alloc(rows);
    nseg.alloc(rows);
    pos.alloc(rows);
    segpos.alloc(rows);
    hot.alloc(1);
    HQ_CUDA(cudaMemsetAsync(hot.get(), 0, sizeof(unsigned long long), s));
    const int64_t hot_len = std::max<int64_t>(64, (int64_t)(32 * (nnz / std::max<uint64_t>(rows, 1))));
    k_long_flags<<<grid_for(rows), 256, 0, s>>>(L.rowptr.get(), rows, flag.get(), nseg.get(), hot_len, hot.get());
    HQ_CHECK_LAUNCH();
    DBuf<unsigned long long> tmax;
    tmax.alloc(1);
    HQ_CUDA(cudaMemsetAsync(tmax.get(), 0, sizeof(unsigned long long), s));
    k_tile_max<<<grid_for((rows + 31) / 32), 256, 0, s>>>(L.rowptr.get(), rows, tmax.get());
    HQ_CHECK_LAUNCH();
    unsigned long long hot_nnz = 0, tile_max = 0;
    HQ_CUDA(cudaMemcpyAsync(&hot_nnz, hot.get(), sizeof(hot_nnz), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaMemcpyAsync(&tile_max, tmax.get(), sizeof(tile_max), cudaMemcpyDeviceToHost, s));
    exclusive_scan(flag.get(), pos.get(), rows, s);
    exclusive_scan(nseg.get(), segpos.get(), rows, s);
    uint32_t lp = 0, lf = 0, sp = 0, sn = 0;
    HQ_CUDA(cudaMemcpyAsync(&lp, pos.get() + rows - 1, 4, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaMemcpyAsync(&lf, flag.get() + rows - 1, 4, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaMemcpyAsync(&sp, segpos.get() + rows - 1, 4, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaMemcpyAsync(&sn, nseg.get() + rows - 1, 4, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    L.hot = nnz > 0 && (double)hot_nnz >= 0.05 * (double)nnz;
    L.max_tile32 = tile_max;
    L.long_rows = (uint64_t)lp + lf;
    L.long_segments = (uint64_t)sp + sn;
    if (L.long_rows) {
        L.long_row_ids.alloc(L.long_rows);
        L.long_seg_ptr.alloc(L.long_rows + 1);
        L.seg_begin.alloc(L.long_segments);
        L.seg_row.alloc(L.long_segments);
        k_long_compact<<<grid_for(rows), 256, 0, s>>>(flag.get(), pos.get(), nseg.get(), segpos.get(), rows,
                                                     L.long_row_ids.get(), L.long_seg_ptr.get());
        int64_t tail = (int64_t)L.long_segments;
        HQ_CUDA(cudaMemcpyAsync(L.long_seg_ptr.get() + L.long_rows, &tail, 8, cudaMemcpyHostToDevice, s));
        k_long_segments<<<grid_for(L.long_rows), 256, 0, s>>>(L.rowptr.get(), L.long_row_ids.get(),
                                                             L.long_seg_ptr.get(), L.long_rows, L.seg_begin.get(),
                                                             L.seg_row.get());
        HQ_CHECK_LAUNCH();
        HQ_CUDA(cudaStreamSynchronize(s));
    }
}

// ------------------------------------------------------- generic kernels --
namespace {

struct PassArgs {
    ModeShape sh;
    uint64_t rbase;  // first row of the processed range
    uint64_t rows;   // rows in the range
    const int64_t* rowptr;
    const double* val;
    const uint32_t* idx[kMaxOrder - 1];
    const double* uo[kMaxOrder - 1];  // factors of the other modes, ascending v != n
    const double* un;                 // U_n (kCore)
    const double* gt;                 // L x K_n (kTTMcTC)
    PassOut out;
    int kind;
    int R;           // rows per tile
    int64_t ntiles;
    int slot0;       // first partial slot of this kernel
    const DevStatus* st;
    int run_if;
    // long rows
    const uint32_t* long_ids;
    const int64_t* long_segptr;
    const int64_t* seg_begin;
    const uint32_t* seg_row;
    uint64_t nlong;
    uint64_t nseg;
};

constexpr int kGenericThreads = 256;

__device__ __forceinline__ double kron_entry(const PassArgs& a, int64_t p, const int* kidx) {
    double prod = a.val[p];
    for (int j = 0; j < a.sh.nothers; ++j)
        prod *= a.uo[j][(size_t)a.idx[j][p] * a.sh.ko[j] + kidx[j]];
    return prod;
}

__device__ __forceinline__ void col_digits(const ModeShape& sh, int col, int* kidx) {
    for (int j = 0; j < sh.nothers; ++j) kidx[j] = (col / sh.cstride[j]) % sh.ko[j];
}

__device__ int64_t tile_lower(const PassArgs& a, int64_t z) {
    int64_t lo = 0, hi = a.ntiles;
    const int64_t zb = a.rowptr[a.rbase];
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        uint64_t r = a.rbase + min((uint64_t)mid * a.R, a.rows);
        if (a.rowptr[r] - zb >= z)
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo;
}

__device__ __forceinline__ double block_max(double v, double* red) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double m = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    return m;
}

__global__ void __launch_bounds__(kGenericThreads) k_pass_tiles_generic(PassArgs a) {
    if (skip_kernel(a.st, a.run_if)) return;
    extern __shared__ double sm[];
    __shared__ double red[32];
    const int L = a.sh.L, Kn = a.sh.kn, R = a.R;
    double* Y = sm;
    double* as = sm + (size_t)R * L;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t Z = a.rowptr[a.rbase + a.rows] - a.rowptr[a.rbase];
    const int64_t t0 = tile_lower(a, (Z * c) / G);
    const int64_t t1 = (c == G - 1) ? a.ntiles : tile_lower(a, (Z * (c + 1)) / G);
    const int slot = a.slot0 + c;
    double* mp = a.out.mpart + (size_t)slot * Kn * L;
    double* wp = a.out.wpart + (size_t)slot * Kn * Kn;
    for (int q = threadIdx.x; q < Kn * L; q += blockDim.x) mp[q] = 0.0;
    for (int q = threadIdx.x; q < Kn * Kn; q += blockDim.x) wp[q] = 0.0;
    double mx = 0.0;
    for (int64_t t = t0; t < t1; ++t) {
        const uint64_t r0 = a.rbase + (uint64_t)t * R;
        const int nr = (int)min((uint64_t)R, a.rbase + a.rows - r0);
        for (int q = threadIdx.x; q < nr * L; q += blockDim.x) {
            int lr = q / L, col = q - lr * L;
            uint64_t i = r0 + lr;
            int64_t s = a.rowptr[i], e = a.rowptr[i + 1];
            double acc = 0.0;
            if (e - s <= kShortMax) {
                int kidx[kMaxOrder - 1];
                col_digits(a.sh, col, kidx);
                for (int64_t p = s; p < e; ++p) acc += kron_entry(a, p, kidx);
            }
            Y[q] = acc;
        }
        __syncthreads();
        for (int q = threadIdx.x; q < nr * Kn; q += blockDim.x) {
            int lr = q / Kn, r = q - lr * Kn;
            uint64_t i = r0 + lr;
            bool lng = (a.rowptr[i + 1] - a.rowptr[i]) > kShortMax;
            double v = 0.0;
            if (!lng) {
                if (a.kind == kTTMcTC) {
                    const double* y = Y + (size_t)lr * L;
                    for (int l = 0; l < L; ++l) v += y[l] * a.gt[(size_t)l * Kn + r];
                } else {
                    v = a.un[i * Kn + r];
                }
                if (a.out.A) a.out.A[i * Kn + r] = v;
            }
            as[q] = v;
            mx = fmax(mx, fabs(v));
        }
        __syncthreads();
        for (int q = threadIdx.x; q < Kn * L; q += blockDim.x) {
            int r = q / L, l = q - r * L;
            double acc = mp[q];
            for (int lr = 0; lr < nr; ++lr) acc += as[lr * Kn + r] * Y[(size_t)lr * L + l];
            mp[q] = acc;
        }
        for (int q = threadIdx.x; q < Kn * Kn; q += blockDim.x) {
            int r1 = q / Kn, r2 = q - r1 * Kn;
            double acc = wp[q];
            for (int lr = 0; lr < nr; ++lr) acc += as[lr * Kn + r1] * as[lr * Kn + r2];
            wp[q] = acc;
        }
        __syncthreads();
    }
    double m = block_max(mx, red);
    if (threadIdx.x == 0) a.out.maxpart[slot] = m;
}

// one CTA per segment of a long row: partial Kronecker row -> ypart[seg]
__global__ void __launch_bounds__(kGenericThreads) k_pass_longseg_generic(PassArgs a) {
    if (skip_kernel(a.st, a.run_if)) return;
    const int L = a.sh.L;
    for (uint64_t sg = blockIdx.x; sg < a.nseg; sg += gridDim.x) {
        int64_t sb = a.seg_begin[sg];
        uint32_t row = a.long_ids[a.seg_row[sg]];
        if (row < a.rbase || row >= a.rbase + a.rows) continue;
        int64_t se = min(sb + kSegLen, a.rowptr[row + 1]);
        for (int col = threadIdx.x; col < L; col += blockDim.x) {
            int kidx[kMaxOrder - 1];
            col_digits(a.sh, col, kidx);
            double acc = 0.0;
            for (int64_t p = sb; p < se; ++p) acc += kron_entry(a, p, kidx);
            a.out.ypart[sg * L + col] = acc;
        }
    }
}

// sums each long row's segment partials in segment order, then a_i, M, W
__global__ void __launch_bounds__(kGenericThreads) k_pass_longfix_generic(PassArgs a) {
    if (skip_kernel(a.st, a.run_if)) return;
    extern __shared__ double sm[];
    __shared__ double red[32];
    const int L = a.sh.L, Kn = a.sh.kn;
    double* Y = sm;
    double* as = sm + L;
    const int G = gridDim.x, c = blockIdx.x;
    const uint64_t lb = a.nlong * c / G, le = a.nlong * (c + 1) / G;
    const int slot = a.slot0 + c;
    double* mp = a.out.mpart + (size_t)slot * Kn * L;
    double* wp = a.out.wpart + (size_t)slot * Kn * Kn;
    for (int q = threadIdx.x; q < Kn * L; q += blockDim.x) mp[q] = 0.0;
    for (int q = threadIdx.x; q < Kn * Kn; q += blockDim.x) wp[q] = 0.0;
    double mx = 0.0;
    for (uint64_t lr = lb; lr < le; ++lr) {
        const uint32_t row = a.long_ids[lr];
        if (row < a.rbase || row >= a.rbase + a.rows) continue;
        const int64_t s0 = a.long_segptr[lr], s1 = a.long_segptr[lr + 1];
        for (int col = threadIdx.x; col < L; col += blockDim.x) {
            double y = 0.0;
            for (int64_t sg = s0; sg < s1; ++sg) y += a.out.ypart[sg * L + col];
            Y[col] = y;
        }
        __syncthreads();
        for (int r = threadIdx.x; r < Kn; r += blockDim.x) {
            double v = 0.0;
            if (a.kind == kTTMcTC) {
                for (int l = 0; l < L; ++l) v += Y[l] * a.gt[(size_t)l * Kn + r];
            } else {
                v = a.un[(size_t)row * Kn + r];
            }
            if (a.out.A) a.out.A[(size_t)row * Kn + r] = v;
            as[r] = v;
            mx = fmax(mx, fabs(v));
        }
        __syncthreads();
        for (int q = threadIdx.x; q < Kn * L; q += blockDim.x) {
            int r = q / L, l = q - r * L;
            mp[q] += as[r] * Y[l];
        }
        for (int q = threadIdx.x; q < Kn * Kn; q += blockDim.x) {
            int r1 = q / Kn, r2 = q - r1 * Kn;
            wp[q] += as[r1] * as[r2];
        }
        __syncthreads();
    }
    double m = block_max(mx, red);
    if (threadIdx.x == 0) a.out.maxpart[slot] = m;
}

int generic_rows_per_tile(const ModeShape& sh) {
    int r = 12288 / (sh.L + sh.kn);
    return std::max(1, std::min(32, r));
}

int short_grid() { return num_sms() * 2; }

// HQ_FORCE_GENERIC=1 routes every shape through the generic kernels (tests
// compare both paths on the same inputs).
bool force_generic() {
    const char* e = std::getenv("HQ_FORCE_GENERIC");
    return e && e[0] == '1';
}
int long_grid(const ModeLayout& L) { return (int)std::min<uint64_t>(L.long_rows, (uint64_t)num_sms() * 2); }

void set_smem(const void* fn, size_t bytes) {
    if (bytes > 48 * 1024) HQ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace

int tile_grid(const ModeShape& sh) {
    if (fast_supported(sh) && !force_generic()) return fast_grid(sh.ko[0], sh.ko[1], sh.kn);
    return short_grid();
}

// short-row tile kernels run (and own partial slots) only when the mode has short rows
int short_slots(const ModeLayout& L, const ModeShape& sh) {
    return (L.long_rows == 0 || L.nonempty_rows > L.long_rows) ? tile_grid(sh) : 0;
}

int pass_slots(const ModeLayout& L, const ModeShape& sh) {
    return short_slots(L, sh) + (L.long_rows ? long_grid(L) : 0);
}

size_t pass_ypart_doubles(const ModeLayout& L, const ModeShape& sh) { return (size_t)L.long_segments * sh.L; }

int pass_launch_count(const ModeLayout& L, const ModeShape& sh) {
    return (short_slots(L, sh) ? 1 : 0) + (L.long_rows ? 2 : 0);
}

void launch_pass(const DeviceTensor& T, int mode, const ModeShape& sh, const FactorPtrs& f, PassKind kind,
                 const double* gt, const PassOut& out, const DevStatus* st, int run_if, cudaStream_t s,
                 uint64_t row_begin, uint64_t row_end) {
    const ModeLayout& L = T.modes[mode];
    row_end = std::min<uint64_t>(row_end, L.rows);
    row_begin = std::min(row_begin, row_end);
    if ((size_t)sh.L * 8 > 200 * 1024)
        fail(HQ_ERR_CAPACITY, "Kronecker row of " + std::to_string(sh.L) + " entries exceeds the device kernel limit");
    const bool a_only = kind == kTTMcTCOnly;
    if (a_only) kind = kTTMcTC;
    PassArgs a{};
    a.sh = sh;
    a.rbase = row_begin;
    a.rows = row_end - row_begin;
    a.rowptr = L.rowptr.get();
    a.val = L.val.get();
    for (int j = 0; j < sh.nothers; ++j) {
        a.idx[j] = L.idx[j].get();
        a.uo[j] = f.u[L.others[j]];
    }
    a.un = f.u[mode];
    a.gt = gt;
    a.out = out;
    a.kind = kind;
    a.st = st;
    a.run_if = run_if;
    a.long_ids = L.long_row_ids.get();
    a.long_segptr = L.long_seg_ptr.get();
    a.seg_begin = L.seg_begin.get();
    a.seg_row = L.seg_row.get();
    a.nlong = L.long_rows;
    a.nseg = L.long_segments;

    a.R = generic_rows_per_tile(sh);
    a.ntiles = (int64_t)ceil_div(a.rows, a.R);
    a.slot0 = 0;
    if (!short_slots(L, sh)) {
        // every nonempty row is long: no tile kernel, so nothing writes the empty rows' A = 0 -- clear the
        // range first (the long-row kernels overwrite the long rows)
        if (out.A && L.nonempty_rows < L.rows && a.rows)
            HQ_CUDA(cudaMemsetAsync(out.A + (size_t)row_begin * sh.kn, 0, sizeof(double) * a.rows * sh.kn, s));
    } else if (fast_supported(sh) && !force_generic()) {
        FastArgs fa{};
        fa.rbase = a.rbase;
        fa.rows = a.rows;
        fa.rowptr = a.rowptr;
        fa.val = a.val;
        fa.ia = a.idx[0];
        fa.ib = a.idx[1];
        fa.ua = a.uo[0];
        fa.ub = a.uo[1];
        fa.un = a.un;
        fa.gt = gt;
        fa.A = out.A;
        fa.mpart = out.mpart;
        fa.wpart = out.wpart;
        fa.maxpart = out.maxpart;
        fa.kind = kind;
        fa.a_only = a_only;
        fa.slot0 = 0;
        fa.st = st;
        fa.run_if = run_if;
        fa.l1_a = T.modes[L.others[0]].hot;
        fa.l1_b = T.modes[L.others[1]].hot;
        launch_fast(fa, sh, tile_grid(sh), s);
    } else {
        size_t smem = sizeof(double) * ((size_t)a.R * sh.L + (size_t)a.R * sh.kn);
        set_smem((const void*)k_pass_tiles_generic, smem);
        k_pass_tiles_generic<<<short_grid(), kGenericThreads, smem, s>>>(a);
        HQ_CHECK_LAUNCH();
    }
    if (L.long_rows && long_fast_supported(sh) && !force_generic()) {
        LongArgs la{};
        la.rbase = a.rbase;
        la.rows = a.rows;
        la.rowptr = a.rowptr;
        la.val = a.val;
        la.i0 = a.idx[0];
        la.i1 = a.idx[1];
        la.i2 = sh.nothers > 2 ? a.idx[2] : nullptr;
        la.u0 = a.uo[0];
        la.u1 = a.uo[1];
        la.u2 = sh.nothers > 2 ? a.uo[2] : nullptr;
        la.l1_0 = T.modes[L.others[0]].hot;
        la.l1_1 = T.modes[L.others[1]].hot;
        la.l1_2 = sh.nothers > 2 && T.modes[L.others[2]].hot;
        la.un = a.un;
        la.gt = gt;
        la.long_ids = a.long_ids;
        la.long_segptr = a.long_segptr;
        la.seg_begin = a.seg_begin;
        la.seg_row = a.seg_row;
        la.nlong = a.nlong;
        la.nseg = a.nseg;
        la.ypart = out.ypart;
        la.A = out.A;
        la.mpart = out.mpart;
        la.wpart = out.wpart;
        la.maxpart = out.maxpart;
        la.kind = kind;
        la.slot0 = short_slots(L, sh);
        la.st = st;
        la.run_if = run_if;
        launch_long_fast(la, sh, long_grid(L), s);
    } else if (L.long_rows) {
        int segs = (int)std::min<uint64_t>(L.long_segments, (uint64_t)num_sms() * 8);
        k_pass_longseg_generic<<<segs, kGenericThreads, 0, s>>>(a);
        HQ_CHECK_LAUNCH();
        a.slot0 = short_slots(L, sh);
        size_t smem2 = sizeof(double) * ((size_t)sh.L + sh.kn);
        set_smem((const void*)k_pass_longfix_generic, smem2);
        k_pass_longfix_generic<<<long_grid(L), kGenericThreads, smem2, s>>>(a);
        HQ_CHECK_LAUNCH();
    }
}

}  // namespace hq
