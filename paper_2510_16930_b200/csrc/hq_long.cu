// hq_long.cu — long rows (more than kShortMax nonzeros) on the FP64 tensor path.
//
// A long row's Kronecker row is a small GEMM over its nonzeros:
//   Y_i = sum_e x_e (U_a[j_e] (x) ... ) (x) U_last[l_e]  =  S^T V,
//   S[e] = x_e * (kron of all other factor rows but the last)   (LS wide)
//   V[e] = U_last[l_e]                                          (KL wide)
// so DMMA m8n8k4 (k = 4 nonzeros) computes it with full tiles whenever LS and
// KL are multiples of 8 (K = 16 at order 3, K = 8 at order 4: configs 4, 5).
//
// k_longseg_mma : one segment (<= kSegLen nonzeros of one row) at a time per
//                 CTA; 128-nonzero chunks staged in shared memory with
//                 cp.async (double-buffered), four warps split the k-steps,
//                 fixed-order cross-warp sum -> ypart[segment].
// k_longfix_mma : tiles of 16 long rows: Y = sum of the row's segment
//                 partials in segment order, then A = Y G^T, M += A^T Y
//                 (DMMA), W += A^T A, max|A| -> the per-CTA partial slots.
// Same results contract as the generic long-row kernels in hq_pass.cu
// (deterministic: static work assignment, fixed summation orders).
#include <algorithm>
#include <cstdlib>

#include "hq_long.cuh"

// Debug instrumentation: -DHQ_PHASE_TIMING accumulates per-phase cycles of thread 0 of every k_fibseg CTA
// (read back with hq_debug_fib_phase_cycles); compiled out otherwise.
#ifdef HQ_PHASE_TIMING
__device__ unsigned long long hq_fib_phase_cycles[16];
#define HQ_FPHASE(i)                                                                   \
    do {                                                                               \
        if (threadIdx.x == 0) {                                                        \
            long long _now = clock64();                                                \
            atomicAdd(&hq_fib_phase_cycles[i], (unsigned long long)(_now - _ph_t));    \
            _ph_t = _now;                                                              \
        }                                                                              \
    } while (0)
#else
#define HQ_FPHASE(i) do { } while (0)
#endif

// k-steps per unrolled step of a warp's share of a full chunk (4 = all of it: the fragment loads of the next
// k-steps behind the DMMAs of this one; config 4 pass 2.197 -> 2.173 ms, config 5 11.67 -> 11.52 ms)
#ifndef HQ_LS_KU
#define HQ_LS_KU 4
#endif
#define HQ_PRAGMA_(x) _Pragma(#x)
#define HQ_UNROLL(n) HQ_PRAGMA_(unroll n)
#ifndef HQ_FIB_DIVFREE
#define HQ_FIB_DIVFREE 1
#endif
#ifndef HQ_FIB_UNROLL
#define HQ_FIB_UNROLL 0
#endif

namespace hq {

namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cpa16(void* d, const void* s) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(d)), "l"(s));
}
// L1-allocating variant for the rows of a hot factor (repeats served by L1, not one L2 slice)
__device__ __forceinline__ void cpa16_l1(void* d, const void* s) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(saddr(d)), "l"(s));
}
__device__ __forceinline__ void cpa8(void* d, const void* s) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(saddr(d)), "l"(s));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// shape of the Kronecker row: other-mode ranks K0, K1, (K2 = 0 at order 3)
template <int K0, int K1, int K2>
struct LS_ {
    static constexpr int NO = K2 ? 3 : 2;           // other modes
    static constexpr int LS = K2 ? K0 * K1 : K0;  // S width
    static constexpr int KL = K2 ? K2 : K1;       // V width (last other mode)
    static constexpr int L = LS * KL;
    static constexpr int MT = (LS + 7) / 8, NTL = (KL + 7) / 8;
    static constexpr int RW = K0 + K1 + K2;        // staged factor doubles per nonzero
    // + x; row stride = 4 mod 8 doubles: the 4 nonzeros of a k-step land on disjoint banks
    static constexpr int FW = (RW + 4) / 8 * 8 + 4;
    static constexpr int CH = 128;                  // nonzeros per chunk
    static constexpr int WARPS = 8, THREADS = 256;
    static constexpr size_t row_doubles = (size_t)CH * FW;           // one gathered-row buffer
    static constexpr size_t red_doubles = (size_t)WARPS * MT * NTL * 64;
    static constexpr size_t rec_words = (size_t)NO * CH;             // one index-record buffer
    static constexpr size_t smem = (2 * row_doubles + red_doubles) * 8 + 3 * rec_words * 4;
    static_assert(K0 % 2 == 0 && K1 % 2 == 0 && K2 % 2 == 0, "16-byte factor rows");
};

// Walks a CTA's chunks: segments [sg, se) of the rank's rows, each cut into
// CH-nonzero chunks (a chunk never straddles two segments).
struct ChunkCursor {
    uint64_t sg, se;
    int64_t z0, zend;
    __device__ bool valid() const { return sg < se; }
    __device__ void seek(const LongArgs& a, uint64_t rend) {  // first in-range segment at or after sg
        for (; sg < se; ++sg) {
            const uint32_t row = a.long_ids[a.seg_row[sg]];
            if (row < a.rbase || row >= rend) continue;  // another rank's row
            z0 = a.seg_begin[sg];
            zend = min(z0 + (int64_t)kSegLen, a.rowptr[row + 1]);
            return;
        }
    }
    __device__ int n(int ch) const { return (int)min((int64_t)ch, zend - z0); }
    __device__ bool last(int ch) const { return z0 + ch >= zend; }
    __device__ void advance(const LongArgs& a, uint64_t rend, int ch) {
        z0 += ch;
        if (z0 >= zend) {
            ++sg;
            seek(a, rend);
        }
    }
};

// One k-step (4 nonzeros) of Y_seg += S^T V on the DMMA pipe.  Lane (gid, tig)
// supplies S[e][8 mt + gid] and V[e][8 nt + gid] for nonzero e = 4 ks + tig.
template <int K0, int K1, int K2, class S, bool FULL>
__device__ __forceinline__ void kstep(const double* f, int ks, int n, int gid, int tig,
                                      double (&acc)[S::MT][S::NTL][2]) {
    const int e = ks * 4 + tig;
    const bool ev = FULL || e < n;
    const double* fe = f + (size_t)e * S::FW;
    const double x = ev ? fe[S::RW] : 0.0;
    double bv[S::NTL];
#pragma unroll
    for (int nt = 0; nt < S::NTL; ++nt) {
        const int col = nt * 8 + gid;
        bv[nt] = (ev && col < S::KL) ? fe[(K2 ? K0 + K1 : K0) + col] : 0.0;
    }
    if constexpr (K2 != 0) {
        static_assert(K1 == 8 && K0 % 2 == 0, "order-4 layout: column = 8 * (U_a index) + U_b index");
        // S[e][8 mt + gid] = x U_a[mt] U_b[gid]: one product per lane, then U_a pairs (16-byte loads)
        const double xb = ev ? x * fe[K0 + gid] : 0.0;
#pragma unroll
        for (int mp = 0; mp < S::MT / 2; ++mp) {
            const double2 ap = *reinterpret_cast<const double2*>(fe + 2 * mp);
            const double a0 = ap.x * xb, a1 = ap.y * xb;
#pragma unroll
            for (int nt = 0; nt < S::NTL; ++nt) {
                dmma(acc[2 * mp][nt][0], acc[2 * mp][nt][1], a0, bv[nt]);
                dmma(acc[2 * mp + 1][nt][0], acc[2 * mp + 1][nt][1], a1, bv[nt]);
            }
        }
    } else {
#pragma unroll
        for (int mt = 0; mt < S::MT; ++mt) {
            const int col = mt * 8 + gid;
            const double av = (ev && col < S::LS) ? x * fe[col] : 0.0;
#pragma unroll
            for (int nt = 0; nt < S::NTL; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], av, bv[nt]);
        }
    }
}

// 16-byte pieces of one factor's rows for n staged nonzeros: four (K/2)
// consecutive lanes copy one row; full chunks run a fixed-trip loop.
template <int KM, int OFF, class S>
__device__ __forceinline__ void gather_mode(const double* __restrict__ u, const uint32_t* r, double* dst, int n,
                                            int tid, int l1) {
    constexpr int PM = KM / 2;
    auto cp = [&](void* d, const void* src) {
        if (l1) cpa16_l1(d, src);
        else cpa16(d, src);
    };
    if (n == S::CH) {
        constexpr int TOT = S::CH * PM, IT = (TOT + S::THREADS - 1) / S::THREADS;
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int q = tid + it * S::THREADS;
            if (TOT % S::THREADS == 0 || q < TOT) {
                const int e = q / PM, p = q - e * PM;
                cp(dst + (size_t)e * S::FW + OFF + 2 * p, u + (size_t)r[e] * KM + 2 * p);
            }
        }
    } else {
        for (int q = tid; q < n * PM; q += S::THREADS) {
            const int e = q / PM, p = q - e * PM;
            cp(dst + (size_t)e * S::FW + OFF + 2 * p, u + (size_t)r[e] * KM + 2 * p);
        }
    }
}

// Three-stage pipeline per CTA over a flat chunk sequence:
//   iteration c: index records of chunk c+2 (coalesced 4-byte cp.async),
//                factor-row gathers of chunk c+1 (16-byte cp.async pieces,
//                row indices read from the staged records), DMMA on chunk c.
// Warps split a chunk's k-steps; at a segment's last chunk the eight warps'
// fragments are summed in warp order into ypart[segment].
template <int K0, int K1, int K2>
__global__ void __launch_bounds__(256) k_longseg_mma(LongArgs a) {
    using S = LS_<K0, K1, K2>;
    if (skip_kernel(a.st, a.run_if)) return;
    extern __shared__ __align__(16) double sm[];
    double* rowbuf = sm;                                   // [2][CH][FW]
    double* red = sm + 2 * S::row_doubles;                 // [WARPS][MT*NTL][64]
    uint32_t* rec = reinterpret_cast<uint32_t*>(red + S::red_doubles);  // [3][NO][CH]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const uint64_t G = gridDim.x, c = blockIdx.x;
    const uint64_t rend = a.rbase + a.rows;
    const uint32_t* idx[3] = {a.i0, a.i1, a.i2};

    ChunkCursor cr{a.nseg * c / G, a.nseg * (c + 1) / G, 0, 0};
    cr.seek(a, rend);
    ChunkCursor cg = cr, cc = cr;  // gathers / compute cursors trail the records cursor

    auto issue_records = [&](int slot) {
        if (cr.valid()) {
            const int n = cr.n(S::CH);
            uint32_t* r = rec + (size_t)slot * S::rec_words;
#pragma unroll
            for (int m = 0; m < S::NO; ++m)
                for (int e = tid; e < n; e += S::THREADS) {
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr(r + m * S::CH + e)),
                                 "l"(idx[m] + cr.z0 + e));
                }
            cr.advance(a, rend, S::CH);
        }
        cpa_commit();
    };
    auto issue_gathers = [&](int rslot, int bslot) {
        if (cg.valid()) {
            const int n = cg.n(S::CH);
            const uint32_t* r = rec + (size_t)rslot * S::rec_words;
            double* dst = rowbuf + (size_t)bslot * S::row_doubles;
            gather_mode<K0, 0, S>(a.u0, r, dst, n, tid, a.l1_0);
            gather_mode<K1, K0, S>(a.u1, r + S::CH, dst, n, tid, a.l1_1);
            if constexpr (K2 != 0) gather_mode<K2, K0 + K1, S>(a.u2, r + 2 * S::CH, dst, n, tid, a.l1_2);
            if (tid < n) cpa8(dst + (size_t)tid * S::FW + S::RW, a.val + cg.z0 + tid);
            cg.advance(a, rend, S::CH);
        }
        cpa_commit();
    };

    double acc[S::MT][S::NTL][2];
#pragma unroll
    for (int i = 0; i < S::MT; ++i)
#pragma unroll
        for (int j = 0; j < S::NTL; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    issue_records(0);
    issue_records(1);
    cpa_wait<1>();
    __syncthreads();
    issue_gathers(0, 0);
    for (int ch = 0; cc.valid(); ++ch) {
        issue_records((ch + 2) % 3);
        cpa_wait<1>();  // gathers of chunk ch and records of chunk ch+1 have landed
        __syncthreads();
        issue_gathers((ch + 1) % 3, (ch + 1) & 1);
        const int n = cc.n(S::CH);
        const double* f = rowbuf + (size_t)(ch & 1) * S::row_doubles;
        if (n == S::CH) {
HQ_UNROLL(HQ_LS_KU)
            for (int ks = warp; ks < S::CH / 4; ks += S::WARPS) kstep<K0, K1, K2, S, true>(f, ks, n, gid, tig, acc);
        } else {
            for (int ks = warp; ks < (n + 3) / 4; ks += S::WARPS) kstep<K0, K1, K2, S, false>(f, ks, n, gid, tig, acc);
        }
        if (cc.last(S::CH)) {
            // fixed-order sum of the warps' fragments -> ypart[segment]
            double* rw = red + (size_t)warp * S::MT * S::NTL * 64;
#pragma unroll
            for (int mt = 0; mt < S::MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < S::NTL; ++nt) {
                    rw[(mt * S::NTL + nt) * 64 + gid * 8 + 2 * tig] = acc[mt][nt][0];
                    rw[(mt * S::NTL + nt) * 64 + gid * 8 + 2 * tig + 1] = acc[mt][nt][1];
                    acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
                }
            __syncthreads();
            const uint64_t sg = cc.sg;
            for (int q = tid; q < S::L; q += S::THREADS) {
                const int sidx = q / S::KL, t = q - sidx * S::KL;  // Kronecker column q = s * KL + t
                const int o = ((sidx / 8) * S::NTL + t / 8) * 64 + (sidx % 8) * 8 + (t % 8);
                double v = 0.0;
#pragma unroll
                for (int w = 0; w < S::WARPS; ++w) v += red[(size_t)w * S::MT * S::NTL * 64 + o];
                a.ypart[sg * S::L + q] = v;
            }
        }
        cc.advance(a, rend, S::CH);
    }
    cpa_wait<0>();
}

// Synchronous variant (default for K = 16 at order 3; HQ_LONG_SYNC=0/1 forces): one chunk at a time per
// CTA (records, then rows, then the
// k-steps), one row buffer and one record buffer -- less shared memory per CTA, so more CTAs (warps) per SM
// overlap each other's phases instead of one CTA overlapping its own.  Same arithmetic and order.
template <int K0, int K1, int K2>
__global__ void __launch_bounds__(256) k_longseg_sync(LongArgs a) {
    using S = LS_<K0, K1, K2>;
    if (skip_kernel(a.st, a.run_if)) return;
    extern __shared__ __align__(16) double sm[];
    double* rowbuf = sm;                                   // [CH][FW]
    double* red = sm + S::row_doubles;                     // [WARPS][MT*NTL][64]
    uint32_t* rec = reinterpret_cast<uint32_t*>(red + S::red_doubles);  // [NO][CH]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const uint64_t G = gridDim.x, c = blockIdx.x;
    const uint64_t rend = a.rbase + a.rows;
    const uint32_t* idx[3] = {a.i0, a.i1, a.i2};
    ChunkCursor cc{a.nseg * c / G, a.nseg * (c + 1) / G, 0, 0};
    cc.seek(a, rend);
    double acc[S::MT][S::NTL][2];
#pragma unroll
    for (int i = 0; i < S::MT; ++i)
#pragma unroll
        for (int j = 0; j < S::NTL; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    while (cc.valid()) {
        const int n = cc.n(S::CH);
#pragma unroll
        for (int m = 0; m < S::NO; ++m)
            for (int e = tid; e < n; e += S::THREADS)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr(rec + m * S::CH + e)),
                             "l"(idx[m] + cc.z0 + e));
        cpa_commit();
        cpa_wait<0>();
        __syncthreads();
        gather_mode<K0, 0, S>(a.u0, rec, rowbuf, n, tid, a.l1_0);
        gather_mode<K1, K0, S>(a.u1, rec + S::CH, rowbuf, n, tid, a.l1_1);
        if constexpr (K2 != 0) gather_mode<K2, K0 + K1, S>(a.u2, rec + 2 * S::CH, rowbuf, n, tid, a.l1_2);
        if (tid < n) cpa8(rowbuf + (size_t)tid * S::FW + S::RW, a.val + cc.z0 + tid);
        cpa_commit();
        cpa_wait<0>();
        __syncthreads();
        if (n == S::CH) {
HQ_UNROLL(HQ_LS_KU)
            for (int ks = warp; ks < S::CH / 4; ks += S::WARPS) kstep<K0, K1, K2, S, true>(rowbuf, ks, n, gid, tig, acc);
        } else {
            for (int ks = warp; ks < (n + 3) / 4; ks += S::WARPS)
                kstep<K0, K1, K2, S, false>(rowbuf, ks, n, gid, tig, acc);
        }
        if (cc.last(S::CH)) {
            double* rw = red + (size_t)warp * S::MT * S::NTL * 64;
#pragma unroll
            for (int mt = 0; mt < S::MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < S::NTL; ++nt) {
                    rw[(mt * S::NTL + nt) * 64 + gid * 8 + 2 * tig] = acc[mt][nt][0];
                    rw[(mt * S::NTL + nt) * 64 + gid * 8 + 2 * tig + 1] = acc[mt][nt][1];
                    acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
                }
            __syncthreads();
            const uint64_t sg = cc.sg;
            for (int q = tid; q < S::L; q += S::THREADS) {
                const int sidx = q / S::KL, t = q - sidx * S::KL;
                const int o = ((sidx / 8) * S::NTL + t / 8) * 64 + (sidx % 8) * 8 + (t % 8);
                double v = 0.0;
#pragma unroll
                for (int w = 0; w < S::WARPS; ++w) v += red[(size_t)w * S::MT * S::NTL * 64 + o];
                a.ypart[sg * S::L + q] = v;
            }
        }
        __syncthreads();  // rows, records and the reduction buffer are free for the next chunk
        cc.advance(a, rend, S::CH);
    }
}


// ------------------------------------------------------------ fiber units --
// Segment kernel over a mode's fiber units (FiberLayout, hq_internal.cuh): a unit is <= kFiberCap consecutive
// nonzeros of one row that share the first other index a, so
//   Y_row = sum_units U_a[a] (x) t_unit,   t_unit = sum_{e in unit} x_e U_b[b_e].
// The Kronecker product costs one DMMA column per unit instead of one per nonzero.  A chunk is the next
// <= CH units of a segment holding <= NCAP nonzeros (cold fibers: 128 units, hot fibers: NCAP / 16); one
// chunk at a time per CTA, three CTAs per SM overlap each other's phases:
//   1. the chunk's nonzeros are one contiguous slice of the value / last-index streams, already staged (it
//      was requested a chunk ahead, as were the unit records, held in registers);
//   2. gathers: the units' U_a rows and the nonzeros' U_b rows, all in flight at once (16-byte cp.async);
//      the next chunk's slice behind them;
//   3. unit sums from shared memory (one thread per unit and column pair) into the row buffer next to U_a;
//   4. the DMMA k-steps of k_longseg (S^T V, k = 4 units per step) and its fixed-order reduction into
//      ypart[segment] at a segment's last chunk.
template <int K0, int K1>
struct FS_ {
    using S = LS_<K0, K1, 0>;
    static constexpr int CH = 128;    // most units of a chunk
    static constexpr int NCAP = kFiberCap <= 4 ? 512 : 448;  // most nonzeros of a chunk (three CTAs per SM at K = 10)
    static constexpr int RW = K0 + K1;
    static constexpr int FW = RW + (12 - RW % 8) % 8;  // row stride = 4 mod 8 doubles (conflict-free k-step loads)
    static constexpr int PM0 = K0 / 2, PM1 = K1 / 2;
    static constexpr size_t row_doubles = (size_t)CH * FW, ub_doubles = (size_t)NCAP * K1;
    static_assert(NCAP >= kFiberCap && FW % 8 == 4, "chunk / row layout");
    static_assert(S::red_doubles <= ub_doubles, "the reduction buffer aliases the staged U_b rows");
    static constexpr size_t smem = (row_doubles + ub_doubles + 2 * (size_t)NCAP) * 8 + 2 * (size_t)NCAP * 4 +
                                   (size_t)CH * 4 + (size_t)(CH + 4) * 4;
};

template <int K0, int K1>
__device__ __forceinline__ void kstep_fib(const double* f, int ks, int n, int gid, int tig,
                                          double (&acc)[LS_<K0, K1, 0>::MT][LS_<K0, K1, 0>::NTL][2]) {
    using S = LS_<K0, K1, 0>;
    constexpr int FW = FS_<K0, K1>::FW;
    const int e = ks * 4 + tig;
    const bool ev = e < n;
    const double* fe = f + (size_t)e * FW;
    double bv[S::NTL];
#pragma unroll
    for (int nt = 0; nt < S::NTL; ++nt) {
        const int col = nt * 8 + gid;
        bv[nt] = (ev && col < K1) ? fe[K0 + col] : 0.0;
    }
#pragma unroll
    for (int mt = 0; mt < S::MT; ++mt) {
        const int col = mt * 8 + gid;
        const double av = (ev && col < K0) ? fe[col] : 0.0;
#pragma unroll
        for (int nt = 0; nt < S::NTL; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], av, bv[nt]);
    }
}

template <int K0, int K1>
__global__ void __launch_bounds__(256) k_fibseg(LongArgs a) {
    using S = LS_<K0, K1, 0>;
    using F = FS_<K0, K1>;
    if (skip_kernel(a.st, a.run_if)) return;
    extern __shared__ __align__(16) double sm[];
    double* rowbuf = sm;                                   // [CH][FW]: U_a row, t
    double* ubuf = rowbuf + F::row_doubles;                // [NCAP][K1] staged U_b rows; then the reduction buffer
    double* red = ubuf;
    double* nzx = ubuf + F::ub_doubles;                    // [2][NCAP] staged values
    uint32_t* nzi = reinterpret_cast<uint32_t*>(nzx + 2 * F::NCAP);  // [2][NCAP] staged last-mode indices
    uint32_t* rec = nzi + 2 * F::NCAP;                     // [CH] first other index of each unit
    int* uoff = reinterpret_cast<int*>(rec + F::CH);       // [CH + 1] unit offsets into the staged slice
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const uint64_t G = gridDim.x, c = blockIdx.x;
    const uint64_t rend = a.rbase + a.rows;
    const int64_t nz_end = a.rowptr_nz[rend];
    // CTAs take contiguous segment ranges of equal cost (units + nonzeros: segments of hot fibers carry up
    // to kFiberCap times the nonzeros of cold ones)
    auto lower = [&](int64_t z) {
        uint64_t lo = 0, hi = a.nseg;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (a.seg_cost[mid] >= z) hi = mid; else lo = mid + 1;
        }
        return lo;
    };
    const int64_t Z = a.seg_cost[a.nseg], Zq = Z / (int64_t)G, Zr = Z % (int64_t)G;
    ChunkCursor cc{lower(Zq * (int64_t)c + Zr * (int64_t)c / (int64_t)G),
                   c + 1 == G ? a.nseg : lower(Zq * (int64_t)(c + 1) + Zr * (int64_t)(c + 1) / (int64_t)G), 0, 0};
    cc.seek(a, rend);
    double acc[S::MT][S::NTL][2];
#pragma unroll
    for (int i = 0; i < S::MT; ++i)
#pragma unroll
        for (int j = 0; j < S::NTL; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // unit records of a chunk's candidate units (threads < CH), held in registers a chunk ahead
    struct Units {
        uint32_t out;
        int64_t st, base;
        int ln;
    };
    auto load_units = [&](const ChunkCursor& k) {
        Units r{0u, 0, 0, 0};
        if (k.valid()) {
            r.base = a.ustart[k.z0];
            if (tid < k.n(F::CH)) {
                r.out = a.i0[k.z0 + tid];
                r.st = a.ustart[k.z0 + tid];
                r.ln = a.ulen[k.z0 + tid];
            }
        }
        return r;
    };
    auto stage_slice = [&](int64_t base, int b) {  // the next NCAP stream positions from base (clamped to the rows)
        const int lim = (int)min((int64_t)F::NCAP, nz_end - base);
        double* x = nzx + (size_t)b * F::NCAP;
        uint32_t* ix = nzi + (size_t)b * F::NCAP;
        for (int q = tid; q < lim; q += S::THREADS) {
            cpa8(x + q, a.val + base + q);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(saddr(ix + q)), "l"(a.i1 + base + q));
        }
    };
    Units cur = load_units(cc);
    if (cc.valid()) stage_slice(cur.base, 0);
    cpa_commit();
    int buf = 0;
#ifdef HQ_PHASE_TIMING
    long long _ph_t = clock64();
#endif
    while (cc.valid()) {
        const int cand = cc.n(F::CH);
        const int off_end = (int)(cur.st + cur.ln - cur.base);
        const int n = __syncthreads_count(tid < cand && off_end <= F::NCAP);  // >= 1: a unit has <= kFiberCap nonzeros
        if (tid < n) {
            rec[tid] = cur.out;
            uoff[tid] = (int)(cur.st - cur.base);
            if (tid == n - 1) uoff[n] = off_end;
        }
        const bool seg_last = cc.last(n);
        const uint64_t sg = cc.sg;
        ChunkCursor nx = cc;
        nx.advance(a, rend, n);
        const Units nxt = load_units(nx);
        HQ_FPHASE(0);
        cpa_wait<0>();  // this chunk's slice (requested a chunk ahead)
        __syncthreads();
        HQ_FPHASE(1);
        const int nn = uoff[n];
        const double* x = nzx + (size_t)buf * F::NCAP;
        const uint32_t* ix = nzi + (size_t)buf * F::NCAP;
#if HQ_FIB_DIVFREE
        {  // 16-byte pieces, PM consecutive threads per row; (row, piece) advanced without divisions
            constexpr int DE0 = S::THREADS / F::PM0, DP0 = S::THREADS % F::PM0;
            int e = tid / F::PM0, p = tid - e * F::PM0;
            while (e < n) {
                double* d = rowbuf + (size_t)e * F::FW + 2 * p;
                const double* src = a.u0 + (size_t)rec[e] * K0 + 2 * p;
                if (a.l1_0) cpa16_l1(d, src);
                else cpa16(d, src);
                e += DE0;
                p += DP0;
                if (p >= F::PM0) {
                    p -= F::PM0;
                    ++e;
                }
            }
            constexpr int DE1 = S::THREADS / F::PM1, DP1 = S::THREADS % F::PM1;
            e = tid / F::PM1;
            p = tid - e * F::PM1;
            while (e < nn) {
                double* d = ubuf + (size_t)e * K1 + 2 * p;
                const double* src = a.u1 + (size_t)ix[e] * K1 + 2 * p;
                if (a.l1_1) cpa16_l1(d, src);
                else cpa16(d, src);
                e += DE1;
                p += DP1;
                if (p >= F::PM1) {
                    p -= F::PM1;
                    ++e;
                }
            }
        }
#else
        for (int q = tid; q < n * F::PM0; q += S::THREADS) {
            const int e = q / F::PM0, p = q - e * F::PM0;
            double* d = rowbuf + (size_t)e * F::FW + 2 * p;
            const double* src = a.u0 + (size_t)rec[e] * K0 + 2 * p;
            if (a.l1_0) cpa16_l1(d, src);
            else cpa16(d, src);
        }
        for (int q = tid; q < nn * F::PM1; q += S::THREADS) {
            const int e = q / F::PM1, p = q - e * F::PM1;
            double* d = ubuf + (size_t)e * K1 + 2 * p;
            const double* src = a.u1 + (size_t)ix[e] * K1 + 2 * p;
            if (a.l1_1) cpa16_l1(d, src);
            else cpa16(d, src);
        }
#endif
        cpa_commit();
        HQ_FPHASE(2);
        if (nx.valid()) stage_slice(nxt.base, buf ^ 1);
        cpa_commit();
        HQ_FPHASE(3);
        cpa_wait<1>();  // the gathers; the next slice stays in flight
        __syncthreads();
        HQ_FPHASE(4);
        for (int w = tid; w < n * F::PM1; w += S::THREADS) {
            const int u = w / F::PM1, p = w - u * F::PM1;
            double t0 = 0.0, t1 = 0.0;
            const int e1 = uoff[u + 1];
#if HQ_FIB_UNROLL
            for (int e = uoff[u]; e < e1; e += 4) {  // four nonzeros' loads in flight, summed in stream order
                double xs[4];
                double2 ds[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (e + i < e1) {
                        xs[i] = x[e + i];
                        ds[i] = *reinterpret_cast<const double2*>(ubuf + (size_t)(e + i) * K1 + 2 * p);
                    }
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (e + i < e1) {
                        t0 = fma(xs[i], ds[i].x, t0);
                        t1 = fma(xs[i], ds[i].y, t1);
                    }
            }
#else
            for (int e = uoff[u]; e < e1; ++e) {
                const double xe = x[e];
                const double2 d = *reinterpret_cast<const double2*>(ubuf + (size_t)e * K1 + 2 * p);
                t0 = fma(xe, d.x, t0);
                t1 = fma(xe, d.y, t1);
            }
#endif
            *reinterpret_cast<double2*>(rowbuf + (size_t)u * F::FW + K0 + 2 * p) = make_double2(t0, t1);
        }
        __syncthreads();
        HQ_FPHASE(5);
        for (int ks = warp; ks < (n + 3) / 4; ks += S::WARPS) kstep_fib<K0, K1>(rowbuf, ks, n, gid, tig, acc);
        HQ_FPHASE(6);
        if (seg_last) {
            double* rw = red + (size_t)warp * S::MT * S::NTL * 64;
#pragma unroll
            for (int mt = 0; mt < S::MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < S::NTL; ++nt) {
                    rw[(mt * S::NTL + nt) * 64 + gid * 8 + 2 * tig] = acc[mt][nt][0];
                    rw[(mt * S::NTL + nt) * 64 + gid * 8 + 2 * tig + 1] = acc[mt][nt][1];
                    acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
                }
            __syncthreads();
            for (int q = tid; q < S::L; q += S::THREADS) {
                const int sidx = q / S::KL, t = q - sidx * S::KL;
                const int o = ((sidx / 8) * S::NTL + t / 8) * 64 + (sidx % 8) * 8 + (t % 8);
                double v = 0.0;
#pragma unroll
                for (int w = 0; w < S::WARPS; ++w) v += red[(size_t)w * S::MT * S::NTL * 64 + o];
                a.ypart[sg * S::L + q] = v;
            }
        }
        __syncthreads();  // row buffer, staged rows and the reduction buffer are free for the next chunk
        HQ_FPHASE(7);
        cc = nx;
        cur = nxt;
        buf ^= 1;
    }
    cpa_wait<0>();
}

// ---------------------------------------------------------------- fix-up --
template <int L, int KN>
struct LF_ {
    static constexpr int RT = 16;                   // long rows per tile
    static constexpr int WARPS = 4, THREADS = 128;
    static constexpr int LP = (L + 7) / 8 * 8, LDY = LP + 4;
    static constexpr int NT = (KN + 7) / 8, ALD = NT * 8 + 4;
    static constexpr int AB = (RT / 8) * NT, ABW = (AB + WARPS - 1) / WARPS;
    static constexpr int NLT = LP / 8, MB = NT * NLT, MBW = (MB + WARPS - 1) / WARPS;
    static constexpr int WQ = (KN * KN + THREADS - 1) / THREADS;
    static constexpr int KSPLIT = AB >= WARPS ? 1 : WARPS / AB;  // A-GEMM k split over idle warps
    static constexpr int L2 = L / 2, YU = 4;                     // Y loads: double2, 4 in flight
    static constexpr size_t smem = (size_t)RT * LDY * 8 + (size_t)(KSPLIT + 1) * RT * ALD * 8 + 64;
    static_assert(L % 2 == 0 && LDY % 2 == 0, "16-byte Y loads");
    static_assert(L % 4 == 0, "k-steps");
};

template <int L, int KN>
__global__ void __launch_bounds__(128, 1) k_longfix_mma(LongArgs a) {
    using F = LF_<L, KN>;
    if (skip_kernel(a.st, a.run_if)) return;
    extern __shared__ __align__(16) double sm[];
    double* sY = sm;
    double* sA = sm + (size_t)F::RT * F::LDY;
    double* sAp = sA + (size_t)F::RT * F::ALD;  // [KSPLIT][RT][ALD] A-GEMM partials
    __shared__ double red[F::WARPS];
    __shared__ uint32_t srow[F::RT];
    __shared__ int64_t ss0[F::RT], ss1[F::RT];  // segment range; empty when not this rank's row
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const uint64_t G = gridDim.x, c = blockIdx.x;
    const uint64_t lb = a.nlong * c / G, le = a.nlong * (c + 1) / G;
    const uint64_t rend = a.rbase + a.rows;
    for (int q = tid; q < F::RT * F::LDY; q += F::THREADS) sY[q] = 0.0;
    for (int q = tid; q < F::RT * F::ALD; q += F::THREADS) sA[q] = 0.0;
    double macc[F::MBW][2];
#pragma unroll
    for (int b = 0; b < F::MBW; ++b) macc[b][0] = macc[b][1] = 0.0;
    double wacc[F::WQ];
#pragma unroll
    for (int b = 0; b < F::WQ; ++b) wacc[b] = 0.0;
    double mx = 0.0;
    __syncthreads();
    for (uint64_t t0 = lb; t0 < le; t0 += F::RT) {
        const int nr = (int)min((uint64_t)F::RT, le - t0);
        if (tid < F::RT) {
            uint32_t row = 0;
            int64_t s0 = 0, s1 = 0;
            if (tid < nr) {
                row = a.long_ids[t0 + tid];
                if (row >= a.rbase && row < rend) {
                    s0 = a.long_segptr[t0 + tid];
                    s1 = a.long_segptr[t0 + tid + 1];
                }
            }
            srow[tid] = row;
            ss0[tid] = s0;
            ss1[tid] = s1;
        }
        __syncthreads();
        // Y rows: segment partials summed in segment order; first segments of
        // YU elements loaded together, further segments (rows > kSegLen) after
        for (int q0 = tid; q0 < F::RT * F::L2; q0 += F::THREADS * F::YU) {
            double2 v[F::YU];
#pragma unroll
            for (int u = 0; u < F::YU; ++u) {
                const int q = q0 + u * F::THREADS;
                v[u] = make_double2(0.0, 0.0);
                if (q < F::RT * F::L2) {
                    const int r = q / F::L2, l = 2 * (q - r * F::L2);
                    if (ss1[r] > ss0[r]) v[u] = *reinterpret_cast<const double2*>(a.ypart + ss0[r] * L + l);
                }
            }
#pragma unroll
            for (int u = 0; u < F::YU; ++u) {
                const int q = q0 + u * F::THREADS;
                if (q < F::RT * F::L2) {
                    const int r = q / F::L2, l = 2 * (q - r * F::L2);
                    for (int64_t sg = ss0[r] + 1; sg < ss1[r]; ++sg) {
                        const double2 w = *reinterpret_cast<const double2*>(a.ypart + sg * L + l);
                        v[u].x += w.x;
                        v[u].y += w.y;
                    }
                    *reinterpret_cast<double2*>(sY + (size_t)r * F::LDY + l) = v[u];
                }
            }
        }
        __syncthreads();
        if (a.kind == kTTMcTC) {
            constexpr int KS = L / 4;
#pragma unroll
            for (int bi = 0; bi < F::ABW; ++bi) {
                const int b = (warp % (F::WARPS / F::KSPLIT)) + bi * (F::WARPS / F::KSPLIT);
                const int kp = warp / (F::WARPS / F::KSPLIT);
                if (b < F::AB) {
                    const int mt = b / F::NT, nt = b - mt * F::NT;
                    const int gcol = nt * 8 + gid;
                    double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
                    const int k0 = kp * KS / F::KSPLIT, k1 = (kp + 1) * KS / F::KSPLIT;
                    for (int ks = k0; ks < k1; ks += 2) {
                        const double y0 = sY[(size_t)(mt * 8 + gid) * F::LDY + ks * 4 + tig];
                        const double g0 = gcol < KN ? __ldg(a.gt + (size_t)(ks * 4 + tig) * KN + gcol) : 0.0;
                        dmma(c0, c1, y0, g0);
                        if (ks + 1 < k1) {
                            const double y1 = sY[(size_t)(mt * 8 + gid) * F::LDY + (ks + 1) * 4 + tig];
                            const double g1 = gcol < KN ? __ldg(a.gt + (size_t)((ks + 1) * 4 + tig) * KN + gcol) : 0.0;
                            dmma(d0, d1, y1, g1);
                        }
                    }
                    const int row = mt * 8 + gid, col = nt * 8 + 2 * tig;
                    double* dst = sAp + (size_t)kp * F::RT * F::ALD;
                    dst[row * F::ALD + col] = c0 + d0;
                    dst[row * F::ALD + col + 1] = c1 + d1;
                }
            }
        }
        __syncthreads();
        for (int q = tid; q < F::RT * KN; q += F::THREADS) {
            const int r = q / KN, k = q - r * KN;
            double v = 0.0;
            if (ss1[r] > ss0[r]) {
                if (a.kind == kTTMcTC) {
#pragma unroll
                    for (int kp = 0; kp < F::KSPLIT; ++kp) v += sAp[(size_t)kp * F::RT * F::ALD + r * F::ALD + k];
                } else {
                    v = a.un[(size_t)srow[r] * KN + k];
                }
                if (a.A) a.A[(size_t)srow[r] * KN + k] = v;
                mx = fmax(mx, fabs(v));
            }
            sA[r * F::ALD + k] = v;
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < F::RT / 4; ++ks)
#pragma unroll
            for (int bi = 0; bi < F::MBW; ++bi) {
                const int b = warp + bi * F::WARPS;
                if (b < F::MB) {
                    const int mt = b / F::NLT, nt = b - mt * F::NLT;
                    const double av = sA[(size_t)(ks * 4 + tig) * F::ALD + mt * 8 + gid];
                    const double yv = sY[(size_t)(ks * 4 + tig) * F::LDY + nt * 8 + gid];
                    dmma(macc[bi][0], macc[bi][1], av, yv);
                }
            }
#pragma unroll
        for (int wi = 0; wi < F::WQ; ++wi) {
            const int q = tid + wi * F::THREADS;
            if (q < KN * KN) {
                const int r1 = q / KN, r2 = q - r1 * KN;
                double sacc = wacc[wi];
                for (int r = 0; r < F::RT; ++r) sacc = fma(sA[r * F::ALD + r1], sA[r * F::ALD + r2], sacc);
                wacc[wi] = sacc;
            }
        }
        __syncthreads();
    }
    const int slot = a.slot0 + (int)c;
    double* mp = a.mpart + (size_t)slot * KN * L;
#pragma unroll
    for (int bi = 0; bi < F::MBW; ++bi) {
        const int b = warp + bi * F::WARPS;
        if (b < F::MB) {
            const int mt = b / F::NLT, nt = b - mt * F::NLT;
            const int r = mt * 8 + gid, l = nt * 8 + 2 * tig;
            if (r < KN) {
                if (l < L) mp[(size_t)r * L + l] = macc[bi][0];
                if (l + 1 < L) mp[(size_t)r * L + l + 1] = macc[bi][1];
            }
        }
    }
#pragma unroll
    for (int wi = 0; wi < F::WQ; ++wi) {
        const int q = tid + wi * F::THREADS;
        if (q < KN * KN) a.wpart[(size_t)slot * KN * KN + q] = wacc[wi];
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < F::WARPS; ++w) m = fmax(m, red[w]);
        a.maxpart[slot] = m;
    }
}

void set_smem_attr(const void* fn, size_t smem) {
    if (smem > 48 * 1024) HQ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}

template <int K0, int K1, int K2, int KN>
void launch_long_t(const LongArgs& a, int fix_grid, cudaStream_t s) {
    using S = LS_<K0, K1, K2>;
    using F = LF_<S::L, KN>;
    // the synchronous kernel wins where the pipelined one is held to two CTAs per SM by its buffers
    // (K = 16, order 3: 1.10 -> 1.00 ms per config-4 pass); it loses at K = 10 (config 3) and order 4
    // (config 5).  HQ_LONG_SYNC=0/1 forces either.
    static const bool sync_var = [] {
        const char* e = std::getenv("HQ_LONG_SYNC");
        if (e && (e[0] == '0' || e[0] == '1')) return e[0] == '1';
        return K0 == 16 && K1 == 16 && K2 == 0;
    }();
    constexpr size_t sync_smem = (S::row_doubles + S::red_doubles) * 8 + S::rec_words * 4;
    static int per_sm = 0;
    if (!per_sm) {
        set_smem_attr((const void*)k_longseg_mma<K0, K1, K2>, S::smem);
        set_smem_attr((const void*)k_longseg_sync<K0, K1, K2>, sync_smem);
        set_smem_attr((const void*)k_longfix_mma<S::L, KN>, F::smem);
        if (sync_var)
            HQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_longseg_sync<K0, K1, K2>, S::THREADS,
                                                                  sync_smem));
        else
            HQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_longseg_mma<K0, K1, K2>, S::THREADS,
                                                                  S::smem));
        per_sm = std::max(per_sm, 1);
    }
    if constexpr (K2 == 0) {
        if (a.ustart) {  // fiber units
            using FS = FS_<K0, K1>;
            static int fib_per_sm = 0;
            if (!fib_per_sm) {
                set_smem_attr((const void*)k_fibseg<K0, K1>, FS::smem);
                HQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fib_per_sm, k_fibseg<K0, K1>, S::THREADS, FS::smem));
                if (const char* e = std::getenv("HQ_FIB_CTAS")) fib_per_sm = std::min(fib_per_sm, std::atoi(e));
                fib_per_sm = std::max(fib_per_sm, 1);
            }
            const int g = (int)std::min<uint64_t>(a.nseg, (uint64_t)num_sms() * fib_per_sm);
            k_fibseg<K0, K1><<<g, S::THREADS, FS::smem, s>>>(a);
            HQ_CHECK_LAUNCH();
            k_longfix_mma<S::L, KN><<<fix_grid, F::THREADS, F::smem, s>>>(a);
            HQ_CHECK_LAUNCH();
            return;
        }
    }
    const int seg_grid = (int)std::min<uint64_t>(a.nseg, (uint64_t)num_sms() * per_sm);
    if (sync_var)
        k_longseg_sync<K0, K1, K2><<<seg_grid, S::THREADS, sync_smem, s>>>(a);
    else
        k_longseg_mma<K0, K1, K2><<<seg_grid, S::THREADS, S::smem, s>>>(a);
    HQ_CHECK_LAUNCH();
    k_longfix_mma<S::L, KN><<<fix_grid, F::THREADS, F::smem, s>>>(a);
    HQ_CHECK_LAUNCH();
}

}  // namespace

#ifdef HQ_PHASE_TIMING
void debug_fib_phase_cycles(unsigned long long* out, int reset) {
    HQ_CUDA(cudaDeviceSynchronize());
    HQ_CUDA(cudaMemcpyFromSymbol(out, hq_fib_phase_cycles, sizeof(unsigned long long) * 16));
    if (reset) {
        unsigned long long z[16] = {0};
        HQ_CUDA(cudaMemcpyToSymbol(hq_fib_phase_cycles, z, sizeof(z)));
    }
}
#else
void debug_fib_phase_cycles(unsigned long long* out, int) {
    for (int i = 0; i < 16; ++i) out[i] = 0;
}
#endif

bool long_fast_supported(const ModeShape& sh) {
    if (sh.order == 3) {
        const int a = sh.ko[0], b = sh.ko[1], n = sh.kn;
        return (a == 10 && b == 10 && n == 10) || (a == 16 && b == 16 && n == 16) || (a == 8 && b == 8 && n == 8);
    }
    if (sh.order == 4) return sh.ko[0] == 8 && sh.ko[1] == 8 && sh.ko[2] == 8 && sh.kn == 8;
    return false;
}

void launch_long_fast(const LongArgs& a, const ModeShape& sh, int fix_grid, cudaStream_t s) {
    if (sh.order == 3 && sh.ko[0] == 10) launch_long_t<10, 10, 0, 10>(a, fix_grid, s);
    else if (sh.order == 3 && sh.ko[0] == 16) launch_long_t<16, 16, 0, 16>(a, fix_grid, s);
    else if (sh.order == 3 && sh.ko[0] == 8) launch_long_t<8, 8, 0, 8>(a, fix_grid, s);
    else if (sh.order == 4) launch_long_t<8, 8, 8, 8>(a, fix_grid, s);
    else fail(HQ_ERR_INTERNAL, "no specialised long-row path for this shape");
}

}  // namespace hq
