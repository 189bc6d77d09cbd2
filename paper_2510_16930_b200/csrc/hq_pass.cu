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

__global__ void k_long_flags(const int64_t* __restrict__ rowptr, uint64_t rows, int64_t short_max,
                             uint32_t* __restrict__ flag, uint32_t* __restrict__ nseg, int64_t hot_len,
                             unsigned long long* __restrict__ hot_nnz) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows; i += (uint64_t)gridDim.x * blockDim.x) {
        int64_t len = rowptr[i + 1] - rowptr[i];
        bool lng = len > short_max;
        flag[i] = lng;
        nseg[i] = lng ? (uint32_t)((len + kSegLen - 1) / kSegLen) : 0u;
        if (len > hot_len) atomicAdd(hot_nnz, (unsigned long long)len);  // integer: order-independent
    }
}

__global__ void k_tile_max(const int64_t* __restrict__ rowptr, uint64_t rows, int64_t short_max,
                           unsigned long long* __restrict__ out) {
    const uint64_t nt = (rows + 31) / 32;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nt; t += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long s = 0;
        const uint64_t e = min(rows, t * 32 + 32);
        for (uint64_t i = t * 32; i < e; ++i) {
            const int64_t len = rowptr[i + 1] - rowptr[i];
            if (len <= short_max) s += (unsigned long long)len;
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


// ---------------------------------------------------------- fiber units --
// One CTA per long-row segment (<= kSegLen = 4096 consecutive nonzeros of one row), 16 positions per thread.
// A position heads a unit when it is the segment's first, when the first other index changes, or every
// kFiberCap positions inside a fiber.  FILL = false counts the units of each segment; FILL = true writes them
// at the segment's base (the exclusive scan of the counts): units come out in stream order.
struct MaxOp {
    __device__ __forceinline__ int operator()(int a, int b) const { return a > b ? a : b; }
};
template <bool FILL>
__global__ void __launch_bounds__(256) k_fib_units(const int64_t* __restrict__ rowptr, const uint32_t* __restrict__ long_ids,
                                                   const int64_t* __restrict__ seg_begin, const uint32_t* __restrict__ seg_row,
                                                   uint64_t nseg, const uint32_t* __restrict__ ia,
                                                   uint32_t* __restrict__ segcount, const uint32_t* __restrict__ segbase,
                                                   int64_t* __restrict__ ustart, uint8_t* __restrict__ ulen,
                                                   uint32_t* __restrict__ outer) {
    static_assert(kSegLen == 256 * 16, "16 positions per thread");
    using ScanI = cub::BlockScan<int, 256>;
    __shared__ typename ScanI::TempStorage tmp;
    const int t = threadIdx.x;
    for (uint64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
        const int64_t b = seg_begin[sg];
        const int64_t rend = rowptr[long_ids[seg_row[sg]] + 1];
        const int n = (int)min((int64_t)kSegLen, rend - b);
        const int p0 = 16 * t;
        uint32_t v[17];
#pragma unroll
        for (int i = 0; i < 17; ++i) {
            const int p = p0 + i - 1;
            v[i] = (p >= 0 && p < n) ? ia[b + p] : 0xffffffffu;
        }
        // last fiber head at or before the end of this thread's range (-1: none in range)
        int last = -1;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int p = p0 + i;
            if (p < n && (p == 0 || v[i + 1] != v[i])) last = p;
        }
        int before;  // last fiber head before this thread's range
        ScanI(tmp).ExclusiveScan(last, before, -1, MaxOp());
        __syncthreads();
        int fstart = before, cnt = 0;
        unsigned heads = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int p = p0 + i;
            if (p < n) {
                if (p == 0 || v[i + 1] != v[i]) fstart = p;
                if ((p - fstart) % kFiberCap == 0) {
                    heads |= 1u << i;
                    ++cnt;
                }
            }
        }
        int base, total;
        ScanI(tmp).ExclusiveSum(cnt, base, total);
        __syncthreads();
        if (!FILL) {
            if (t == 0) segcount[sg] = (uint32_t)total;
        } else {
            // a unit ends at the next head (possibly in a later thread's range) or at the segment end: every
            // thread publishes its first head position, threads without one forward the next thread's
            __shared__ int firsthead[257];
            firsthead[t] = heads ? p0 + (__ffs(heads) - 1) : -1;
            if (t == 0) firsthead[256] = n;
            __syncthreads();
            const size_t ub = (size_t)segbase[sg] + base;
            int k = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (heads >> i & 1) {
                    const int p = p0 + i;
                    int nx = -1;
                    const unsigned later = heads >> (i + 1);
                    if (i < 15 && later) nx = p + __ffs(later);
                    else {
                        for (int tt = t + 1; tt <= 256 && nx < 0; ++tt) nx = firsthead[tt];
                    }
                    ustart[ub + k] = b + p;
                    ulen[ub + k] = (uint8_t)(nx - p);
                    outer[ub + k] = v[i + 1];
                    ++k;
                }
            }
            __syncthreads();
        }
    }
}

__global__ void k_long_nnz(const int64_t* __restrict__ rowptr, const uint32_t* __restrict__ ids, uint64_t nlong,
                           unsigned long long* __restrict__ out) {
    unsigned long long s = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nlong; r += (uint64_t)gridDim.x * blockDim.x)
        s += (unsigned long long)(rowptr[ids[r] + 1] - rowptr[ids[r]]);
    if (s) atomicAdd(out, s);  // integer: order-independent
}

// units of long row r = segbase[ptr[r + 1]] - segbase[ptr[r]] -> cnt[row id]; derived segments per long row
__global__ void k_fib_row_counts(const uint32_t* __restrict__ ids, const int64_t* __restrict__ segptr, uint64_t nlong,
                                 const uint32_t* __restrict__ segbase, int64_t* __restrict__ cnt,
                                 uint32_t* __restrict__ nsegf) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nlong; r += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t c = (int64_t)segbase[segptr[r + 1]] - (int64_t)segbase[segptr[r]];
        cnt[ids[r]] = c;
        nsegf[r] = (uint32_t)((c + kSegLen - 1) / kSegLen);
    }
}
// cost of a derived segment: its units (one DMMA column each) and its nonzeros (one unit-sum term each)
__global__ void k_fib_seg_cost(const int64_t* __restrict__ rowptr_f, const uint32_t* __restrict__ ids,
                               const int64_t* __restrict__ seg_begin, const uint32_t* __restrict__ seg_row, uint64_t nseg,
                               const int64_t* __restrict__ ustart, const uint8_t* __restrict__ ulen,
                               int64_t* __restrict__ cost) {
    for (uint64_t sg = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; sg <= nseg; sg += (uint64_t)gridDim.x * blockDim.x) {
        int64_t c = 0;
        if (sg < nseg) {
            const int64_t first = seg_begin[sg];
            const int64_t last = min(first + (int64_t)kSegLen, rowptr_f[ids[seg_row[sg]] + 1]) - 1;
            const int64_t nz = ustart[last] + ulen[last] - ustart[first];
            c = 4 * (last - first + 1) + 2 * nz;
        }
        cost[sg] = c;
    }
}
__global__ void k_u32_to_i64(const uint32_t* __restrict__ a, uint64_t n, int64_t* __restrict__ b) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = (int64_t)a[i];
}
__global__ void k_fib_fill(uint64_t n, uint32_t* __restrict__ ident, double* __restrict__ ones) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        ident[i] = (uint32_t)i;
        ones[i] = 1.0;
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


// HQ_FIBERS=0 disables the fiber units, =1 builds them whenever a mode has long rows (tests); default: only
// where they shrink the long rows' stream by >= 1.5x
int fibers_mode() {
    const char* e = std::getenv("HQ_FIBERS");
    if (e && (e[0] == '0' || e[0] == '1')) return e[0] - '0';
    return -1;
}

void plan_fibers(ModeLayout& L, cudaStream_t s) {
    FiberLayout& F = L.fib;
    F = FiberLayout{};
    const int fm = fibers_mode();
    if (fm == 0 || !L.long_rows || !L.idx[0].p) return;
    const uint64_t nseg = L.long_segments, nlong = L.long_rows;
    DBuf<uint32_t> segcount, segbase;
    DBuf<unsigned long long> lnz;
    segcount.alloc(nseg + 1);
    segbase.alloc(nseg + 1);
    lnz.alloc(1);
    HQ_CUDA(cudaMemsetAsync(lnz.get(), 0, 8, s));
    HQ_CUDA(cudaMemsetAsync(segcount.get() + nseg, 0, 4, s));
    k_long_nnz<<<grid_for(nlong), 256, 0, s>>>(L.rowptr.get(), L.long_row_ids.get(), nlong, lnz.get());
    const int g = (int)std::min<uint64_t>(nseg, (uint64_t)num_sms() * 8);
    k_fib_units<false><<<g, 256, 0, s>>>(L.rowptr.get(), L.long_row_ids.get(), L.seg_begin.get(), L.seg_row.get(), nseg,
                                         L.idx[0].get(), segcount.get(), nullptr, nullptr, nullptr, nullptr);
    HQ_CHECK_LAUNCH();
    exclusive_scan(segcount.get(), segbase.get(), nseg + 1, s);  // segbase[nseg] = the unit count
    uint32_t units = 0;
    unsigned long long long_nnz = 0;
    HQ_CUDA(cudaMemcpyAsync(&units, segbase.get() + nseg, 4, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaMemcpyAsync(&long_nnz, lnz.get(), 8, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    if (!units || (fm != 1 && (double)long_nnz < 1.5 * (double)units)) return;
    F.units = units;
    F.long_nnz = long_nnz;
    F.start.alloc(units);
    F.len.alloc(units);
    F.outer.alloc((size_t)units + 4);
    F.ident.alloc((size_t)units + 4);
    F.ones.alloc((size_t)units + 2);
    k_fib_units<true><<<g, 256, 0, s>>>(L.rowptr.get(), L.long_row_ids.get(), L.seg_begin.get(), L.seg_row.get(), nseg,
                                        L.idx[0].get(), nullptr, segbase.get(), F.start.get(), F.len.get(),
                                        F.outer.get());
    HQ_CHECK_LAUNCH();
    k_fib_fill<<<grid_for(units), 256, 0, s>>>(units, F.ident.get(), F.ones.get());
    // unit range of every row, and the derived stream's segments
    DBuf<int64_t> cnt;
    DBuf<uint32_t> nsegf, segposf;
    cnt.alloc(L.rows + 1);
    nsegf.alloc(nlong);
    segposf.alloc(nlong);
    HQ_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int64_t) * (L.rows + 1), s));
    k_fib_row_counts<<<grid_for(nlong), 256, 0, s>>>(L.long_row_ids.get(), L.long_seg_ptr.get(), nlong, segbase.get(),
                                                    cnt.get(), nsegf.get());
    HQ_CHECK_LAUNCH();
    F.rowptr.alloc(L.rows + 1);
    exclusive_scan(cnt.get(), F.rowptr.get(), L.rows + 1, s);
    exclusive_scan(nsegf.get(), segposf.get(), nlong, s);
    uint32_t sp = 0, sn = 0;
    HQ_CUDA(cudaMemcpyAsync(&sp, segposf.get() + nlong - 1, 4, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaMemcpyAsync(&sn, nsegf.get() + nlong - 1, 4, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    F.long_segments = (uint64_t)sp + sn;
    F.long_seg_ptr.alloc(nlong + 1);
    F.seg_begin.alloc(F.long_segments);
    F.seg_row.alloc(F.long_segments);
    k_u32_to_i64<<<grid_for(nlong), 256, 0, s>>>(segposf.get(), nlong, F.long_seg_ptr.get());
    const int64_t tail = (int64_t)F.long_segments;
    HQ_CUDA(cudaMemcpyAsync(F.long_seg_ptr.get() + nlong, &tail, 8, cudaMemcpyHostToDevice, s));
    k_long_segments<<<grid_for(nlong), 256, 0, s>>>(F.rowptr.get(), L.long_row_ids.get(), F.long_seg_ptr.get(), nlong,
                                                   F.seg_begin.get(), F.seg_row.get());
    HQ_CHECK_LAUNCH();
    {
        DBuf<int64_t> cost;
        cost.alloc(F.long_segments + 1);
        F.seg_cost.alloc(F.long_segments + 1);
        k_fib_seg_cost<<<grid_for(F.long_segments + 1), 256, 0, s>>>(F.rowptr.get(), L.long_row_ids.get(),
                                                                    F.seg_begin.get(), F.seg_row.get(), F.long_segments,
                                                                    F.start.get(), F.len.get(), cost.get());
        HQ_CHECK_LAUNCH();
        exclusive_scan(cost.get(), F.seg_cost.get(), F.long_segments + 1, s);
        HQ_CUDA(cudaStreamSynchronize(s));
    }
    F.on = true;
}

}  // namespace

namespace {

// long rows (more than short_max nonzeros), their segments, the hot flag and the largest short-row tile
void plan_long_rows(ModeLayout& L, uint64_t nnz, int64_t short_max, cudaStream_t s) {
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
    L.short_max = short_max;
    k_long_flags<<<grid_for(rows), 256, 0, s>>>(L.rowptr.get(), rows, L.short_max, flag.get(), nseg.get(), hot_len,
                                               hot.get());
    HQ_CHECK_LAUNCH();
    DBuf<unsigned long long> tmax;
    tmax.alloc(1);
    HQ_CUDA(cudaMemsetAsync(tmax.get(), 0, sizeof(unsigned long long), s));
    k_tile_max<<<grid_for((rows + 31) / 32), 256, 0, s>>>(L.rowptr.get(), rows, L.short_max, tmax.get());
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
    L.long_row_ids.release();
    L.long_seg_ptr.release();
    L.seg_begin.release();
    L.seg_row.release();
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

}  // namespace

void plan_mode(ModeLayout& L, uint64_t nnz, int order, cudaStream_t s) {
    plan_long_rows(L, nnz, kShortMax, s);
    L.fib = FiberLayout{};
    if (order != 3 || fibers_mode() == 0) return;
    if (L.hot) {
        // a skewed mode: its long rows run through the fiber units where those shrink the stream, and the fiber
        // kernel outruns the tile kernel (tiles of very unequal rows) from ~50 nonzeros per row on -- plan
        // with the lower threshold, and go back to the plain plan when the units do not pay
        plan_long_rows(L, nnz, kSkewedShortMax, s);
        plan_fibers(L, s);
        if (!L.fib.on) plan_long_rows(L, nnz, kShortMax, s);
    } else {
        plan_fibers(L, s);
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
    int64_t short_max;
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
            if (e - s <= a.short_max) {
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
            bool lng = (a.rowptr[i + 1] - a.rowptr[i]) > a.short_max;
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


// ---- fiber unit sums: T[u] = sum_{e in unit u} x_e U_b[b_e]  (one thread per unit, <= kFiberCap nonzeros).
// SM = true: the whole last-mode factor is first copied into shared memory (small extents: every gather
// is a shared-memory read); otherwise rows are read through L1 (hot rows of a skewed factor stay there).
template <int KB, bool SM>
__global__ void __launch_bounds__(SM ? (KB > 10 ? 512 : 1024) : 256)
    k_unit_sums(const int64_t* __restrict__ ustart, const uint8_t* __restrict__ ulen, const int64_t* __restrict__ rowptr_f,
                uint64_t rbase, uint64_t rows, const double* __restrict__ val, const uint32_t* __restrict__ ib,
                const double* __restrict__ ub, uint64_t ub_rows, double* __restrict__ T, const DevStatus* st,
                int run_if) {
    if (skip_kernel(st, run_if)) return;
    extern __shared__ __align__(16) double tab[];
    if (SM) {
        const double2* src = reinterpret_cast<const double2*>(ub);
        double2* dst = reinterpret_cast<double2*>(tab);
        for (size_t q = threadIdx.x; q < ub_rows * KB / 2; q += blockDim.x) dst[q] = src[q];
        __syncthreads();
    }
    const double* base = SM ? tab : ub;
    const int64_t u0 = rowptr_f[rbase], u1 = rowptr_f[rbase + rows];
    for (int64_t u = u0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < u1; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e0 = ustart[u];
        const int n = ulen[u];
        double t[KB];
#pragma unroll
        for (int q = 0; q < KB; ++q) t[q] = 0.0;
        double x = val[e0];
        uint32_t r = ib[e0];
        for (int i = 0; i < n; ++i) {
            const double xc = x;
            const double2* row = reinterpret_cast<const double2*>(base + (size_t)r * KB);
            if (i + 1 < n) {  // next record's stream loads under this record's row loads
                x = val[e0 + i + 1];
                r = ib[e0 + i + 1];
            }
#pragma unroll
            for (int q = 0; q < KB / 2; ++q) {
                const double2 d = SM ? row[q] : __ldg(row + q);
                t[2 * q] = fma(xc, d.x, t[2 * q]);
                t[2 * q + 1] = fma(xc, d.y, t[2 * q + 1]);
            }
        }
        double2* o = reinterpret_cast<double2*>(T + (size_t)u * KB);
#pragma unroll
        for (int q = 0; q < KB / 2; ++q) o[q] = make_double2(t[2 * q], t[2 * q + 1]);
    }
}

template <int KB>
void launch_unit_sums_k(const ModeLayout& L, uint64_t rbase, uint64_t rows, const double* ub, uint64_t ub_rows,
                        double* T, const DevStatus* st, int run_if, cudaStream_t s) {
    const FiberLayout& F = L.fib;
    const size_t tab = (size_t)ub_rows * KB * sizeof(double);
    if (tab <= 200 * 1024) {
        static bool attr = false;
        if (!attr) {
            HQ_CUDA(cudaFuncSetAttribute(k_unit_sums<KB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            attr = true;
        }
        k_unit_sums<KB, true><<<num_sms(), KB > 10 ? 512 : 1024, tab, s>>>(F.start.get(), F.len.get(), F.rowptr.get(), rbase, rows,
                                                          L.val.get(), L.idx[1].get(), ub, ub_rows, T, st, run_if);
    } else {
        k_unit_sums<KB, false><<<num_sms() * 8, 256, 0, s>>>(F.start.get(), F.len.get(), F.rowptr.get(), rbase, rows,
                                                            L.val.get(), L.idx[1].get(), ub, ub_rows, T, st, run_if);
    }
    HQ_CHECK_LAUNCH();
}

bool unit_sums_supported(int kb) { return kb == 8 || kb == 10 || kb == 16; }

void launch_unit_sums(int kb, const ModeLayout& L, uint64_t rbase, uint64_t rows, const double* ub, uint64_t ub_rows,
                      double* T, const DevStatus* st, int run_if, cudaStream_t s) {
    if (kb == 8) launch_unit_sums_k<8>(L, rbase, rows, ub, ub_rows, T, st, run_if, s);
    else if (kb == 10) launch_unit_sums_k<10>(L, rbase, rows, ub, ub_rows, T, st, run_if, s);
    else if (kb == 16) launch_unit_sums_k<16>(L, rbase, rows, ub, ub_rows, T, st, run_if, s);
    else fail(HQ_ERR_INTERNAL, "no unit-sum kernel for this rank");
}

// the long rows go through their fiber units when the layout has them and the shape has the kernels
bool fibers_fit(const ModeLayout& L, const ModeShape& sh) {
    return L.fib.on && sh.order == 3 && long_fast_supported(sh) && unit_sums_supported(sh.ko[1]);
}
bool use_fibers(const ModeLayout& L, const ModeShape& sh) { return fibers_fit(L, sh) && !force_generic(); }

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

// scratch of a pass: the long-row segment partials, then (fiber units) the unit sums T
size_t pass_ypart_doubles(const ModeLayout& L, const ModeShape& sh) {
    return (size_t)L.long_segments * sh.L + (fibers_fit(L, sh) ? (size_t)L.fib.units * sh.ko[1] + 2 : 0);
}

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
    a.short_max = L.short_max;

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
        fa.short_max = (int)L.short_max;
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
        static const bool fused = [] {
            const char* e = std::getenv("HQ_FIB_FUSED");
            return !(e && e[0] == '0');
        }();
        if (use_fibers(L, sh) && fused) {
            // fiber units, fused: the segment kernel forms each unit's sum over the last other mode in
            // shared memory and takes its Kronecker product with the unit's first-other-mode row (k_fibseg)
            la.rowptr_nz = a.rowptr;
            la.rowptr = L.fib.rowptr.get();
            la.i0 = L.fib.outer.get();
            la.ustart = L.fib.start.get();
            la.ulen = L.fib.len.get();
            la.seg_cost = L.fib.seg_cost.get();
            la.long_segptr = L.fib.long_seg_ptr.get();
            la.seg_begin = L.fib.seg_begin.get();
            la.seg_row = L.fib.seg_row.get();
            la.nseg = L.fib.long_segments;
        } else if (use_fibers(L, sh)) {
            // fiber units: T = the unit sums over the last other mode, then the long-row kernels run on the
            // derived stream (value 1, indices (first other index, unit id)) with T as the last factor table
            double* Tu = out.ypart + (size_t)L.long_segments * sh.L;
            launch_unit_sums(sh.ko[1], L, a.rbase, a.rows, a.uo[1], T.dims[L.others[1]], Tu, st, run_if, s);
            la.rowptr = L.fib.rowptr.get();
            la.val = L.fib.ones.get();
            la.i0 = L.fib.outer.get();
            la.i1 = L.fib.ident.get();
            la.u1 = Tu;
            la.l1_1 = false;
            la.long_segptr = L.fib.long_seg_ptr.get();
            la.seg_begin = L.fib.seg_begin.get();
            la.seg_row = L.fib.seg_row.get();
            la.nseg = L.fib.long_segments;
        }
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
