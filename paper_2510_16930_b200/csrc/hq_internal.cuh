// hq_internal.cuh — shared types, error plumbing and device helpers of the
// B200 HOQRI engine.  No exception escapes the C-ABI (hq_capi.cu catches
// hq::Error and maps it to hq_status + a thread-local message).
#pragma once

#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <iterator>
#include <map>
#include <mutex>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hoqri_b200.h"

namespace hq {

constexpr int kMaxOrder = 8;

struct Error : std::runtime_error {
    int code;
    int64_t payload;
    Error(int c, const std::string& m, int64_t p = 0) : std::runtime_error(m), code(c), payload(p) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg, int64_t payload = 0) {
    throw Error(code, msg, payload);
}

#define HQ_CUDA(call)                                                                       \
    do {                                                                                    \
        cudaError_t _e = (call);                                                            \
        if (_e != cudaSuccess)                                                              \
            ::hq::fail(HQ_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define HQ_CHECK_LAUNCH() HQ_CUDA(cudaGetLastError())

// ---------------------------------------------------------------- memory --
// Device buffers come from a size-keyed cache of cudaMalloc blocks (a caching allocator, like the host
// frameworks'): a freed block goes onto a free list and the next request of (nearly) the same size takes it, so
// a solve that follows another of the same shape makes no driver allocation at all.  The CUDA stream-ordered
// pool this replaced re-used blocks only most of the time: about one config-2 solve in three paid a fresh
// 40-160 MB mapping (1-450 ms inside cudaMallocAsync, measured with HQ_ALLOC_TIMING on this pool's boxes),
// which was the whole of the end-to-end variance.  HQ_POOL_RELEASE_GB caps the bytes kept on the free lists;
// hq_release_cached_memory() returns them to the driver; an out-of-memory cudaMalloc frees them and retries.
struct DeviceCache {
    std::mutex mu;
    std::multimap<size_t, void*> blocks[16];  // per device: free blocks by size
    size_t cached = 0;
    size_t cap = ~size_t(0);
    DeviceCache() {
        if (const char* e = std::getenv("HQ_POOL_RELEASE_GB")) cap = (size_t)std::strtoull(e, nullptr, 10) << 30;
    }
    static size_t round_up(size_t bytes) { return (bytes + 511) & ~size_t(511); }
    static int device() {
        int dev = 0;
        cudaGetDevice(&dev);
        return dev & 15;
    }
    // a free block of at least `bytes` and at most 1/8 more (so odd-sized leftovers do not pin large blocks)
    void* take(size_t bytes, size_t* got) {
        std::lock_guard<std::mutex> g(mu);
        auto& m = blocks[device()];
        auto it = m.lower_bound(bytes);
        if (it == m.end() || it->first > bytes + bytes / 8) return nullptr;
        void* p = it->second;
        *got = it->first;
        cached -= it->first;
        m.erase(it);
        return p;
    }
    void put(void* p, size_t bytes) {
        std::lock_guard<std::mutex> g(mu);
        auto& m = blocks[device()];
        m.emplace(bytes, p);
        cached += bytes;
        while (cached > cap && !m.empty()) {  // over the cap: the largest blocks go back to the driver
            auto it = std::prev(m.end());
            cudaFree(it->second);
            cached -= it->first;
            m.erase(it);
        }
    }
    size_t release_all() {
        std::lock_guard<std::mutex> g(mu);
        size_t freed = 0;
        for (auto& m : blocks) {
            for (auto& kv : m) {
                cudaFree(kv.second);
                freed += kv.first;
            }
            m.clear();
        }
        cached = 0;
        return freed;
    }
};
inline DeviceCache& device_cache() {
    static DeviceCache* c = new DeviceCache();  // never destroyed: the CUDA context may be gone at exit
    return *c;
}

// RAII device buffer.
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    // a rank's slice [off, off + n) of a conceptually longer array (sharded mode streams): get() returns the
    // base the kernels index with global positions, p - off; only the slice is allocated
    size_t off = 0;
    size_t cap = 0;  // bytes of the underlying block
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), off(o.off), cap(o.cap) { o.p = nullptr; o.n = 0; o.off = 0; o.cap = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p; n = o.n; off = o.off; cap = o.cap;
            o.p = nullptr; o.n = 0; o.off = 0; o.cap = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        off = 0;
        n = count;
        if (count) {
            const size_t want = DeviceCache::round_up(sizeof(T) * count);
            DeviceCache& c = device_cache();
            void* q = c.take(want, &cap);
            if (!q) {
#ifdef HQ_ALLOC_TIMING
                const auto t0 = std::chrono::steady_clock::now();
#endif
                cudaError_t e = cudaMalloc(&q, want);
                if (e == cudaErrorMemoryAllocation) {  // give the cached blocks back and try once more
                    cudaGetLastError();
                    cudaDeviceSynchronize();
                    c.release_all();
                    e = cudaMalloc(&q, want);
                }
                HQ_CUDA(e);
                cap = want;
#ifdef HQ_ALLOC_TIMING
                std::fprintf(stderr, "[alloc] %zu bytes from the driver: %.2f ms\n", want,
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
#endif
            }
            p = static_cast<T*>(q);
        }
    }
    void release() {
        if (p) {
            cudaDeviceSynchronize();  // like cudaFree: no pending work may still use the block
            device_cache().put(p, cap);
        }
        p = nullptr;
        n = 0;
        off = 0;
        cap = 0;
    }
    T* get() const { return p ? p - off : nullptr; }
    size_t bytes() const { return sizeof(T) * n; }
};

inline int num_sms() {
    static int sms = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    return sms;
}

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// ----------------------------------------------------------- device tensor --
// One mode's view of the tensor: nonzeros in mode-n order (stable counting
// sort of the lexicographic order == the reference's ModeBuckets.entries,
// sparse_tensor.cpp:73-89), as SoA streams.
// Fiber units of a mode's long rows (order 3; hq_pass.cu plan_fibers).  Within a row the stream is sorted by
// (first other mode, last other mode), so nonzeros sharing the first other index a are contiguous -- a fiber
// (row, a).  Y_row = sum_fibers U_a[a] (x) t_fiber with t_fiber = sum_{e in fiber} x_e U_b[b_e]: the Kronecker
// product is formed once per fiber instead of once per nonzero.  Fibers are cut into units of at most
// kFiberCap nonzeros (bounded work per thread in the unit-sum kernel); the units of a mode form a derived
// stream (value 1, indices (a, unit id)) that the long-row kernels consume with T = the unit sums as the
// last factor table.  Built only where it shrinks the long rows' stream by >= 1.5x (skewed tensors).
#ifndef HQ_FIBER_CAP
#define HQ_FIBER_CAP 16
#endif
constexpr int kFiberCap = HQ_FIBER_CAP;
struct FiberLayout {
    bool on = false;
    uint64_t units = 0;
    uint64_t long_nnz = 0;   // nonzeros of the long rows (units cover exactly these)
    DBuf<int64_t> start;     // units: stream position of the unit's first nonzero
    DBuf<uint8_t> len;       // units: nonzeros in the unit (1..kFiberCap)
    DBuf<int64_t> rowptr;    // rows + 1: unit range of each row (short rows: empty)
    DBuf<uint32_t> outer;    // units: index into the first other mode's factor
    DBuf<uint32_t> ident;    // units: 0, 1, 2, ... (the unit's own row of T)
    DBuf<double> ones;       // units: 1.0
    uint64_t long_segments = 0;  // the derived stream's long-row plan (same long rows, segments over units)
    DBuf<int64_t> seg_begin;
    DBuf<uint32_t> seg_row;
    DBuf<int64_t> long_seg_ptr;
    DBuf<int64_t> seg_cost;  // segments + 1: prefix sums of the segments' cost (units and nonzeros) -- CTA ranges
};

struct ModeLayout {
    int mode = 0;
    uint64_t rows = 0;                 // I_n
    DBuf<int64_t> rowptr;              // I_n + 1  (== ModeBuckets.offsets)
    DBuf<uint32_t> entries;            // nnz      (== ModeBuckets.entries; mode 0: identity, not stored)
    DBuf<double> val;                  // nnz, values in mode order
    DBuf<uint32_t> idx[kMaxOrder - 1];  // nnz each: index of the j-th other mode (ascending v != n)
    int others[kMaxOrder - 1] = {0};
    uint64_t nonempty_rows = 0;        // R_n
    // skewed: rows longer than 32x the mean hold >= 5% of the nonzeros.  Row i of this mode's unfolding is
    // how often U_n[i] is gathered by the other modes' passes, so a skewed mode's factor has hot rows that
    // pile onto single L2 slices: its gathers are made L1-allocating (cp.async.ca) to absorb the repeats.
    bool hot = false;
    uint64_t max_tile32 = 0;  // most short-row nonzeros in one 32-row tile (the pass kernels' tile)
    // work plan (see hq_pass.cu)
    int64_t short_max = 256;           // rows with more nonzeros are long (kShortMax; lower where fiber units run)
    uint64_t long_rows = 0;
    DBuf<uint32_t> long_row_ids;       // rows with more than kShortMax nonzeros
    uint64_t long_segments = 0;
    DBuf<int64_t> seg_begin;           // long-row segments: [seg_begin, seg_end) positions
    DBuf<uint32_t> seg_row;            // owning long row (index into long_row_ids)
    DBuf<int64_t> long_seg_ptr;        // long row r owns segments [ptr[r], ptr[r+1])
    FiberLayout fib;                   // fiber units of the long rows (order 3, skewed tensors)
};

struct DeviceTensor {
    int order = 0;
    uint64_t dims[kMaxOrder] = {0};
    uint64_t nnz = 0;
    DBuf<uint32_t> coords;   // lexicographically sorted, merged, AoS nnz x order
    DBuf<double> vals;       // merged values
    double norm_sq = 0.0;
    ModeLayout modes[kMaxOrder];
    // row-partitioned storage (hq_tensor_shard): this rank keeps, per mode, only the stream slice of its rows
    // [shard_bounds[n][rank], shard_bounds[n][rank + 1]); the lexicographic copy and the buckets' entries are freed
    int shard_world = 1, shard_rank = 0;
    std::vector<uint64_t> shard_bounds[kMaxOrder];
};

// ------------------------------------------------------------ kernel args --
struct FactorPtrs {
    const double* u[kMaxOrder];
    int k[kMaxOrder];
};

// Rank bookkeeping for mode n: the Kronecker row of the other modes has
// length L = prod_{v != n} K_v, column index = sum_v k_v * cstride[v] with the
// last other mode fastest (unfold_col_strides, dense_core.cpp:337-348).
struct ModeShape {
    int order;
    int n;
    int kn;          // K_n
    int L;           // prod_{v != n} K_v
    int nothers;     // order - 1
    int ko[kMaxOrder - 1];       // K of each other mode, ascending v != n
    int cstride[kMaxOrder - 1];  // column stride of each other mode
};

ModeShape make_mode_shape(int order, const int* ranks, int n);

}  // namespace hq

struct hq_tensor {
    hq::DeviceTensor t;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    ~hq_tensor() {
        if (own_stream && stream) cudaStreamDestroy(stream);
    }
};
