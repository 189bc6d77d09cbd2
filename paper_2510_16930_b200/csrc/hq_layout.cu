// hq_layout.cu — device construction of the sparse tensor layout.
//
// Replaces tucker::SparseTensor's constructor (proj/src/sparse_tensor.cpp:18-89):
//   validate   (sparse_tensor.cpp:22-38)  one pass, first offending entry by atomicMin
//   normalize  (sparse_tensor.cpp:43-71)  pack the N coordinates into a
//              multi-word key (mode 0 most significant, ceil(log2 I_v) bits per
//              mode), stable LSD radix sort of (key, entry) pairs, run heads,
//              run-length merge summing values in input order
//   buckets    (sparse_tensor.cpp:73-89)  per mode a stable radix sort of the
//              merged entries by c_n (== the reference's counting sort), offsets
//              by boundary scatter, and the mode-n SoA streams the kernels read
// Coordinate order, offsets and entries are bit-exact with the reference; a
// merged value of >= 3 duplicates may differ in the last ulp (the reference
// sums them in std::sort's unspecified order among equal keys).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "hq_internal.cuh"
#include "hq_plan.cuh"

namespace hq {

namespace {

constexpr int kMaxWords = 4;  // keys up to 256 bits

__global__ void k_validate(const uint32_t* __restrict__ coords, const double* __restrict__ vals,
                           uint64_t nnz, int order, const uint64_t* __restrict__ dims,
                           unsigned long long* first_bad) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (uint64_t)gridDim.x * blockDim.x) {
        bool bad = vals && !isfinite(vals[e]);  // vals == nullptr: coordinates only
        if (coords)
            for (int m = 0; m < order; ++m) bad |= (uint64_t)coords[e * order + m] >= dims[m];
        if (bad) atomicMin(first_bad, (unsigned long long)e);
    }
}

struct KeySpec {
    int order;
    int nwords;
    int bits[kMaxOrder];
};

__global__ void k_pack_keys(const uint32_t* __restrict__ coords, uint64_t nnz, KeySpec ks,
                            uint64_t* __restrict__ keys /* nwords x nnz, word 0 least significant */) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t w[kMaxWords] = {0, 0, 0, 0};
        for (int m = 0; m < ks.order; ++m) {
            int b = ks.bits[m];
            if (b == 0) continue;
            for (int j = kMaxWords - 1; j > 0; --j) w[j] = (w[j] << b) | (w[j - 1] >> (64 - b));
            w[0] = (w[0] << b) | coords[e * ks.order + m];
        }
        for (int j = 0; j < ks.nwords; ++j) keys[j * nnz + e] = w[j];
    }
}

__global__ void k_iota(uint32_t* p, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

__global__ void k_gather_u64(const uint64_t* __restrict__ src, const uint32_t* __restrict__ perm, uint64_t n,
                             uint64_t* __restrict__ dst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = src[perm[i]];
}

__global__ void k_heads(const uint32_t* __restrict__ coords, const uint32_t* __restrict__ perm, uint64_t n,
                        int order, uint32_t* __restrict__ head) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t h = 1;
        if (i > 0) {
            const uint32_t* a = coords + (uint64_t)perm[i] * order;
            const uint32_t* b = coords + (uint64_t)perm[i - 1] * order;
            h = 0;
            for (int m = 0; m < order; ++m) h |= (a[m] != b[m]);
        }
        head[i] = h;
    }
}

__global__ void k_run_starts(const uint32_t* __restrict__ head, const uint32_t* __restrict__ runid, uint64_t n,
                             uint32_t* __restrict__ start) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        if (head[i]) start[runid[i]] = (uint32_t)i;
}

// sparse_tensor.cpp:58-68: each run's values summed in sorted (= input) order.
// Runs longer than kLongRun (hot cells of skewed inputs: 10^5 duplicates are
// common under Zipf draws) would serialise one thread on a chain of dependent
// gathers; they are queued for k_merge_long instead.
constexpr uint64_t kLongRun = 128;

__global__ void k_merge(const uint32_t* __restrict__ coords, const double* __restrict__ vals,
                        const uint32_t* __restrict__ perm, const uint32_t* __restrict__ start, uint64_t nruns,
                        uint64_t n, int order, uint32_t* __restrict__ out_coords, double* __restrict__ out_vals,
                        uint32_t* __restrict__ long_runs, unsigned int* __restrict__ n_long) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nruns; u += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t s = start[u], e = (u + 1 < nruns) ? start[u + 1] : n;
        uint32_t p0 = perm[s];
        for (int m = 0; m < order; ++m) out_coords[u * order + m] = coords[(uint64_t)p0 * order + m];
        if (e - s > kLongRun) {
            long_runs[atomicAdd(n_long, 1u)] = (uint32_t)u;
            continue;
        }
        double acc = vals[p0];
        for (uint64_t p = s + 1; p < e; ++p) acc += vals[perm[p]];
        out_vals[u] = acc;
    }
}

// one block per long run: thread-strided partial sums in input order, then a
// fixed reduction tree, so the merged value does not depend on scheduling
__global__ void __launch_bounds__(256) k_merge_long(const double* __restrict__ vals, const uint32_t* __restrict__ perm,
                                                    const uint32_t* __restrict__ start, uint64_t nruns, uint64_t n,
                                                    const uint32_t* __restrict__ long_runs,
                                                    const unsigned int* __restrict__ n_long,
                                                    double* __restrict__ out_vals) {
    __shared__ double red[256];
    const unsigned int cnt = *n_long;
    for (unsigned int i = blockIdx.x; i < cnt; i += gridDim.x) {
        const uint32_t u = long_runs[i];
        const uint64_t s = start[u], e = (u + 1 < nruns) ? start[u + 1] : n;
        double acc = 0.0;
        for (uint64_t p = s + threadIdx.x; p < e; p += blockDim.x) acc += vals[perm[p]];
        red[threadIdx.x] = acc;
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) out_vals[u] = red[0];
        __syncthreads();
    }
}

__global__ void k_extract_mode(const uint32_t* __restrict__ coords, uint64_t n, int order, int mode,
                               uint32_t* __restrict__ key) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        key[i] = coords[i * order + mode];
}

// offsets[i] = #entries with key < i  (keys sorted ascending)
__global__ void k_rowptr(const uint32_t* __restrict__ key, uint64_t n, uint64_t rows, int64_t* __restrict__ rowptr) {
    uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t p = tid; p <= n; p += stride) {
        int64_t lo = (p == 0) ? 0 : (int64_t)key[p - 1] + 1;  // first row index > previous key
        int64_t hi = (p == n) ? (int64_t)rows : (int64_t)key[p];
        for (int64_t i = lo; i <= hi && i <= (int64_t)rows; ++i) rowptr[i] = (int64_t)p;
    }
}

__global__ void k_mode_streams(const uint32_t* __restrict__ coords, const double* __restrict__ vals,
                               const uint32_t* __restrict__ entries /* null: identity */, uint64_t n, int order,
                               int mode, double* __restrict__ out_val, uint32_t* o0, uint32_t* o1, uint32_t* o2,
                               uint32_t* o3, uint32_t* o4, uint32_t* o5, uint32_t* o6) {
    uint32_t* outs[7] = {o0, o1, o2, o3, o4, o5, o6};
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t e = entries ? entries[p] : p;
        out_val[p] = vals[e];
        int j = 0;
        for (int v = 0; v < order; ++v) {
            if (v == mode) continue;
            outs[j++][p] = coords[e * order + v];
        }
    }
}

__global__ void k_count_nonempty(const int64_t* __restrict__ rowptr, uint64_t rows, unsigned long long* cnt) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows; i += (uint64_t)gridDim.x * blockDim.x)
        c += rowptr[i + 1] > rowptr[i];
    for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

// deterministic sum of squares: fixed grid, per-block partials, one final block
__global__ void k_sumsq_partial(const double* __restrict__ v, uint64_t n, double* part) {
    __shared__ double sh[32];
    double s = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        s += v[i] * v[i];
    for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
        part[blockIdx.x] = t;
    }
}

__global__ void k_sum_serial(const double* part, int n, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += part[i];
        *out = t;
    }
}

inline int grid_for(uint64_t n, int threads = 256) {
    uint64_t b = ceil_div(n ? n : 1, threads);
    uint64_t cap = (uint64_t)num_sms() * 16;
    return (int)std::min<uint64_t>(std::max<uint64_t>(b, 1), cap);
}

template <class K, class V>
void radix_sort_pairs(const K* kin, K* kout, const V* vin, V* vout, uint64_t n, int end_bit, cudaStream_t s) {
    if (n == 0) return;
    if (n > 0x7fffffffull) fail(HQ_ERR_CAPACITY, "tensor too large for the device sort (nnz >= 2^31)");
    size_t tmp = 0;
    HQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)n, 0, end_bit, s));
    DBuf<uint8_t> t;
    t.alloc(tmp ? tmp : 1);
    HQ_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kin, kout, vin, vout, (int)n, 0, end_bit, s));
}

int bit_width(uint64_t extent) {
    uint64_t m = extent - 1;
    int b = 0;
    while (m) { ++b; m >>= 1; }
    return b;
}

// HQ_PROFILE_BUILD=1: per-phase wall times of the layout build (stream-synchronised; diagnostics only)
struct PhaseClock {
    cudaStream_t s;
    bool on;
    std::chrono::steady_clock::time_point t;
    explicit PhaseClock(cudaStream_t st) : s(st), on(std::getenv("HQ_PROFILE_BUILD") != nullptr) {
        if (on) {
            cudaStreamSynchronize(s);
            t = std::chrono::steady_clock::now();
        }
    }
    void mark(const char* what, int mode = -1) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[build] %-14s%s%d %8.2f ms\n", what, mode >= 0 ? " mode " : "", mode >= 0 ? mode : 0,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

}  // namespace

double device_sum_sq(const double* v, uint64_t n, cudaStream_t s) {
    const int blocks = 256;
    DBuf<double> part, out;
    part.alloc(blocks);
    out.alloc(1);
    k_sumsq_partial<<<blocks, 256, 0, s>>>(v, n, part.get());
    k_sum_serial<<<1, 32, 0, s>>>(part.get(), blocks, out.get());
    HQ_CHECK_LAUNCH();
    double h = 0.0;
    HQ_CUDA(cudaMemcpyAsync(&h, out.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    return h;
}

void build_tensor(DeviceTensor& T, int order, const uint64_t* dims, uint64_t nnz, const uint32_t* coords_in,
                  const double* vals_in, cudaStream_t s, cudaEvent_t vals_ready) {
    if (order <= 0) fail(HQ_ERR_SHAPE, "sparse tensor needs at least one mode");
    if (order > kMaxOrder) fail(HQ_ERR_SHAPE, "tensor order above the engine limit of 8");
    for (int m = 0; m < order; ++m)
        if (dims[m] == 0) fail(HQ_ERR_SHAPE, "zero extent");
    for (int m = 0; m < order; ++m)
        if (dims[m] > 0x100000000ull) fail(HQ_ERR_CAPACITY, "extent above 2^32");
    T.order = order;
    for (int m = 0; m < order; ++m) T.dims[m] = dims[m];
    PhaseClock clk(s);

    // ---- validation (sparse_tensor.cpp:29-38): the first bad entry in entry order decides the error (its
    // coordinates are checked before its value).  With vals_ready the coordinate check runs now and the value
    // check after the lexicographic sort (the values' upload overlaps the sort); the sort never indexes
    // memory by coordinate, so a bad coordinate is harmless until the check below.
    DBuf<uint64_t> ddims;
    DBuf<unsigned long long> bad;
    auto check_entries = [&]() {
        unsigned long long hb = 0;
        HQ_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(hb), cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        if (hb != ~0ull) {
            uint32_t c[kMaxOrder];
            double v;
            HQ_CUDA(cudaMemcpy(c, coords_in + hb * order, sizeof(uint32_t) * order, cudaMemcpyDeviceToHost));
            HQ_CUDA(cudaMemcpy(&v, vals_in + hb, sizeof(double), cudaMemcpyDeviceToHost));
            for (int m = 0; m < order; ++m)
                if (c[m] >= dims[m])
                    fail(HQ_ERR_RANGE, "coordinate " + std::to_string(c[m]) + " out of range for mode " +
                                           std::to_string(m + 1) + " (extent " + std::to_string(dims[m]) + ")");
            fail(HQ_ERR_VALUE, "non-finite value at entry " + std::to_string(hb));
        }
    };
    if (nnz) {
        ddims.alloc(order);
        HQ_CUDA(cudaMemcpyAsync(ddims.get(), dims, sizeof(uint64_t) * order, cudaMemcpyHostToDevice, s));
        bad.alloc(1);
        HQ_CUDA(cudaMemsetAsync(bad.get(), 0xff, sizeof(unsigned long long), s));
        k_validate<<<grid_for(nnz), 256, 0, s>>>(coords_in, vals_ready ? nullptr : vals_in, nnz, order, ddims.get(),
                                                 bad.get());
        HQ_CHECK_LAUNCH();
        if (!vals_ready) check_entries();
    }
    clk.mark("validate");

    // ---- lexicographic sort (sparse_tensor.cpp:43-53)
    KeySpec ks{};
    ks.order = order;
    int total_bits = 0;
    for (int m = 0; m < order; ++m) {
        ks.bits[m] = bit_width(dims[m]);
        total_bits += ks.bits[m];
    }
    ks.nwords = std::max(1, (total_bits + 63) / 64);
    if (ks.nwords > kMaxWords) fail(HQ_ERR_CAPACITY, "coordinate key wider than 256 bits");

    DBuf<uint32_t> perm;
    uint64_t nruns = 0;
    DBuf<uint32_t> start;
    if (nnz) {
        DBuf<uint64_t> keys, kg, kout;
        keys.alloc((size_t)ks.nwords * nnz);
        kg.alloc(nnz);
        kout.alloc(nnz);
        k_pack_keys<<<grid_for(nnz), 256, 0, s>>>(coords_in, nnz, ks, keys.get());
        DBuf<uint32_t> p0, p1;
        p0.alloc(nnz);
        p1.alloc(nnz);
        k_iota<<<grid_for(nnz), 256, 0, s>>>(p0.get(), nnz);
        HQ_CHECK_LAUNCH();
        clk.mark("sort buffers");
        for (int w = 0; w < ks.nwords; ++w) {
            int wbits = (w < ks.nwords - 1) ? 64 : total_bits - 64 * (ks.nwords - 1);
            if (wbits <= 0) continue;
            const uint64_t* kin = keys.get() + (size_t)w * nnz;
            if (w > 0) {
                k_gather_u64<<<grid_for(nnz), 256, 0, s>>>(kin, p0.get(), nnz, kg.get());
                kin = kg.get();
            }
            radix_sort_pairs(kin, kout.get(), p0.get(), p1.get(), nnz, wbits, s);
            std::swap(p0, p1);
        }
        perm = std::move(p0);
        clk.mark("radix sort");
        if (vals_ready) {  // the values have landed: their check, then the first bad entry (if any) is reported
            HQ_CUDA(cudaStreamWaitEvent(s, vals_ready, 0));
            k_validate<<<grid_for(nnz), 256, 0, s>>>(nullptr, vals_in, nnz, order, ddims.get(), bad.get());
            HQ_CHECK_LAUNCH();
            check_entries();
        }
        clk.mark("lexsort");

        // ---- run heads and merge (sparse_tensor.cpp:54-70)
        DBuf<uint32_t> head, runid;
        head.alloc(nnz);
        runid.alloc(nnz);
        k_heads<<<grid_for(nnz), 256, 0, s>>>(coords_in, perm.get(), nnz, order, head.get());
        size_t tmp = 0;
        HQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, head.get(), runid.get(), (int)nnz, s));
        DBuf<uint8_t> t;
        t.alloc(tmp ? tmp : 1);
        HQ_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, head.get(), runid.get(), (int)nnz, s));
        uint32_t last_id = 0, last_head = 0;
        HQ_CUDA(cudaMemcpyAsync(&last_id, runid.get() + nnz - 1, 4, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaMemcpyAsync(&last_head, head.get() + nnz - 1, 4, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        nruns = (uint64_t)last_id + last_head;
        start.alloc(nruns);
        k_run_starts<<<grid_for(nnz), 256, 0, s>>>(head.get(), runid.get(), nnz, start.get());
        T.coords.alloc(nruns * order);
        T.vals.alloc(nruns);
        DBuf<uint32_t> long_runs;
        long_runs.alloc(std::max<uint64_t>(1, std::min<uint64_t>(nruns, nnz / (kLongRun + 1))));
        DBuf<unsigned int> n_long;
        n_long.alloc(1);
        HQ_CUDA(cudaMemsetAsync(n_long.get(), 0, sizeof(unsigned int), s));
        k_merge<<<grid_for(nruns), 256, 0, s>>>(coords_in, vals_in, perm.get(), start.get(), nruns, nnz, order,
                                               T.coords.get(), T.vals.get(), long_runs.get(), n_long.get());
        k_merge_long<<<num_sms() * 4, 256, 0, s>>>(vals_in, perm.get(), start.get(), nruns, nnz, long_runs.get(),
                                                  n_long.get(), T.vals.get());
        HQ_CHECK_LAUNCH();
    }
    clk.mark("merge");
    T.nnz = nruns;
    const uint64_t n = nruns;
    T.norm_sq = n ? device_sum_sq(T.vals.get(), n, s) : 0.0;

    // ---- per-mode buckets and streams (sparse_tensor.cpp:73-89)
    for (int m = 0; m < order; ++m) {
        ModeLayout& L = T.modes[m];
        L.mode = m;
        L.rows = dims[m];
        L.rowptr.alloc(dims[m] + 1);
        int j = 0;
        for (int v = 0; v < order; ++v)
            if (v != m) L.others[j++] = v;
        // 16 bytes of tail padding: the pass stages a tile's contiguous stream slice with 16-byte copies from its
        // aligned base, which may read up to one 16-byte unit past the last nonzero
        L.val.alloc(n + 2);
        for (int q = 0; q < order - 1; ++q) L.idx[q].alloc(n + 4);
        DBuf<uint32_t> key, skey;
        key.alloc(n);
        if (n) k_extract_mode<<<grid_for(n), 256, 0, s>>>(T.coords.get(), n, order, m, key.get());
        const uint32_t* sorted_keys = key.get();
        if (m > 0 && n) {
            DBuf<uint32_t> io;
            io.alloc(n);
            k_iota<<<grid_for(n), 256, 0, s>>>(io.get(), n);
            skey.alloc(n);
            L.entries.alloc(n);
            radix_sort_pairs(key.get(), skey.get(), io.get(), L.entries.get(), n, std::max(1, ks.bits[m]), s);
            sorted_keys = skey.get();
        }
        clk.mark("mode sort", m);
        k_rowptr<<<grid_for(n + 1), 256, 0, s>>>(sorted_keys, n, dims[m], L.rowptr.get());
        if (n) {
            uint32_t* o[7] = {nullptr};
            for (int q = 0; q < order - 1; ++q) o[q] = L.idx[q].get();
            k_mode_streams<<<grid_for(n), 256, 0, s>>>(T.coords.get(), T.vals.get(), m > 0 ? L.entries.get() : nullptr,
                                                      n, order, m, L.val.get(), o[0], o[1], o[2], o[3], o[4], o[5],
                                                      o[6]);
        }
        DBuf<unsigned long long> cnt;
        cnt.alloc(1);
        HQ_CUDA(cudaMemsetAsync(cnt.get(), 0, 8, s));
        k_count_nonempty<<<grid_for(dims[m]), 256, 0, s>>>(L.rowptr.get(), dims[m], cnt.get());
        HQ_CHECK_LAUNCH();
        unsigned long long hc = 0;
        HQ_CUDA(cudaMemcpyAsync(&hc, cnt.get(), 8, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        L.nonempty_rows = hc;
        clk.mark("mode streams", m);
        plan_mode(L, n, order, s);
        clk.mark("mode plan", m);
    }
    HQ_CUDA(cudaStreamSynchronize(s));
}

// ---- exports (for the bit-exact layout checks)
__global__ void k_iota64(uint64_t* p, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = i;
}
__global__ void k_u32_to_u64(const uint32_t* a, uint64_t n, uint64_t* b) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}
__global__ void k_i64_to_u64(const int64_t* a, uint64_t n, uint64_t* b) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = (uint64_t)a[i];
}

void export_buckets(const DeviceTensor& T, int mode, uint64_t* offsets, uint64_t* entries, cudaStream_t s) {
    const ModeLayout& L = T.modes[mode];
    DBuf<uint64_t> tmp;
    tmp.alloc(std::max<uint64_t>(L.rows + 1, T.nnz) + 1);
    k_i64_to_u64<<<grid_for(L.rows + 1), 256, 0, s>>>(L.rowptr.get(), L.rows + 1, tmp.get());
    HQ_CUDA(cudaMemcpyAsync(offsets, tmp.get(), sizeof(uint64_t) * (L.rows + 1), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    if (T.nnz) {
        if (mode == 0)
            k_iota64<<<grid_for(T.nnz), 256, 0, s>>>(tmp.get(), T.nnz);
        else
            k_u32_to_u64<<<grid_for(T.nnz), 256, 0, s>>>(L.entries.get(), T.nnz, tmp.get());
        HQ_CHECK_LAUNCH();
        HQ_CUDA(cudaMemcpyAsync(entries, tmp.get(), sizeof(uint64_t) * T.nnz, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
    }
}

}  // namespace hq
