// hq_pass_fast.cu — specialised fused mode pass for order-3 tensors with
// compile-time ranks (the BASELINE shapes: K = 10, 16, 8).
//
// Same contract as the generic tile kernel in hq_pass.cu (per row i of the
// mode-n unfolding: Y_i, a_i = Y_i G_(n)^T or U_n[i], partials of
// M = sum a_i^T Y_i, W = sum a_i^T a_i, max|a_i|), mapped onto B200:
//
//  * FP64 datapath: DFMA and DMMA share it (35.4 / 37.1 TFLOP/s alone, 36.7
//    mixed; tools/microbench_mix.cu), so the pass minimises issue slots:
//    DFMA for the per-nonzero Kronecker rows, DMMA m8n8k4 for the per-row
//    GEMMs.
//  * Memory: the only random traffic is two factor rows per nonzero.  A
//    tile's rows are gathered in bulk with cp.async (every row of the tile in
//    flight at once, no registers held), factor rows with an L2 evict_last
//    policy and the nonzero streams with evict_first; small CTAs (128
//    threads, 3 per SM at K = 10) let one CTA's gathers overlap another's
//    arithmetic.
//
// Per tile of R consecutive short rows (rows with <= kShortMax nonzeros):
//   1. row lengths, virtual offsets (scan), rows ranked by length and dealt to
//      lanes in that order (equal loop lengths per warp);
//   2. records (x, j, k) of the tile -> smem (cp.async), then the two factor
//      rows of every record -> smem (cp.async 16 B), CAP records per round;
//   3. Kronecker rows: lane (row, pb, qb) accumulates a BP x BQ block of
//      Y_i = sum_e x_e U_a[j_e, :] (x) U_b[k_e, :] (DFMA);
//   4. Y tile -> smem (aliasing the gather buffer); A_tile = Y_tile G_(n)^T
//      (DMMA, G_(n)^T fragments from L1) or U_n rows; A written; max|A|;
//   5. M += A_tile^T Y_tile (DMMA, C fragments resident in registers for the
//      CTA's whole tile range), W += A^T A (DFMA).
// Deterministic: fixed row->lane assignment per tile, fixed tile->CTA
// assignment, per-CTA partial slots reduced in fixed order.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "hq_fast.cuh"

// Debug instrumentation: -DHQ_PHASE_TIMING accumulates per-phase cycles of
// thread 0 of every CTA into hq_phase_cycles[] (read back with
// hq_debug_phase_cycles); compiled out otherwise.
#ifdef HQ_PHASE_TIMING
__device__ unsigned long long hq_phase_cycles[16];
#define HQ_PHASE(i)                                                   \
    do {                                                              \
        if (threadIdx.x == 0) {                                       \
            long long _now = clock64();                               \
            atomicAdd(&hq_phase_cycles[i], (unsigned long long)(_now - _ph_t)); \
            _ph_t = _now;                                             \
        }                                                             \
    } while (0)
#else
#define HQ_PHASE(i) do { } while (0)
#endif

#ifndef HQ_CAP
#define HQ_CAP 384
#endif
#ifndef HQ_MINB
#define HQ_MINB 2
#endif
#ifndef HQ_CAP16
#define HQ_CAP16 192
#endif
#ifndef HQ_MINB16
#define HQ_MINB16 2
#endif

namespace hq {

namespace {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// factor-row pieces: a miss fetches the 64-byte pair of sectors (.L2::64B) -- the row's next piece usually needs
// the other one; 20 % less DRAM read traffic on random 80-byte rows in isolation (tools/microbench_fetch.cu
// -DPF=64) and the config-2 pass 0.609 -> 0.605 ms
#ifndef HQ_CP_PF64
#define HQ_CP_PF64 1
#endif
__device__ __forceinline__ void cp16(void* dst, const void* src, uint64_t pol) {
#if HQ_CP_PF64
    asm volatile("cp.async.cg.shared.global.L2::cache_hint.L2::64B [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "l"(pol));
#else
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "l"(pol));
#endif
}
// L1-allocating variant for the rows of a hot (skewed) factor: repeats are served by L1 instead of one L2 slice
__device__ __forceinline__ void cp16_l1(void* dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "l"(pol));
}
__device__ __forceinline__ void cp8(void* dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "l"(pol));
}
__device__ __forceinline__ void cp4(void* dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "l"(pol));
}
__device__ __forceinline__ void cp_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Loads the B doubles of a lane's block starting at element `st` of a staged
// factor row with 16-byte shared loads and no selects: for odd B the element
// that breaks 16-byte alignment is loaded last and the lane keeps its own
// local->global index map (blk_index) for the write-back.
template <int B>
__device__ __forceinline__ void lds_block(const double* f, int st, double (&v)[B]) {
    const int odd = st & 1;
    const double* pr = f + st + odd;
#pragma unroll
    for (int i = 0; i < B / 2; ++i) {
        const double2 d = *reinterpret_cast<const double2*>(pr + 2 * i);
        v[2 * i] = d.x;
        v[2 * i + 1] = d.y;
    }
    if constexpr (B & 1) v[B - 1] = f[odd ? st : st + B - 1];
}
template <int B>
__device__ __forceinline__ int blk_index(int st, int i) {
    const int odd = st & 1;
    if constexpr (B & 1) {
        if (i == B - 1) return odd ? st : st + B - 1;
    }
    return st + odd + i;
}

struct Rec {
    double x;
    uint32_t j, k;
};

template <int KA, int KB, int KN>
struct Cfg {
    static constexpr int L = KA * KB;
    static constexpr int TP = 2;
    static constexpr int TQ = (KB >= 16) ? 4 : 2;
    static constexpr int TR = TP * TQ;           // lanes per row
    static constexpr int BP = KA / TP;
    static constexpr int BQ = KB / TQ;
#ifndef HQ_WARPS
#define HQ_WARPS 4
#endif
    static constexpr int WARPS = HQ_WARPS;
    static constexpr int THREADS = 32 * WARPS;
    static constexpr int R = THREADS / TR;       // rows per tile
    static constexpr int RPW = 32 / TR;          // rows per warp
    static constexpr int LP = (L + 7) / 8 * 8;   // Y columns padded to whole n-tiles
    static constexpr int LDY = LP + 4;           // Y row stride (== 4 mod 8 doubles)
    static constexpr int NT = (KN + 7) / 8;      // A n-tiles / M m-tiles
    static constexpr int ALD = NT * 8 + 4;       // A tile row stride
    static constexpr int NLT = LP / 8;           // M n-tiles
    static constexpr int MB = NT * NLT;          // M blocks
    static constexpr int MBW = (MB + WARPS - 1) / WARPS;
    static constexpr int AB = (R / 8) * NT;      // A blocks
    static constexpr int ABW = (AB + WARPS - 1) / WARPS;
    static constexpr int WQ = (KN * KN + THREADS - 1) / THREADS;
    static constexpr int FW = KA + KB + ((KA + KB) % 8 == 4 ? 2 : ((KA + KB) % 8 == 0 ? 4 : 0));  // staged doubles per
    // record: the two factor rows, padded so consecutive records start 8 banks apart (conflict-free 16 B loads)
    static constexpr int CAP = (KB >= 16) ? HQ_CAP16 : HQ_CAP;  // records per gather round
    static constexpr int MINB = (KB >= 16) ? HQ_MINB16 : HQ_MINB;  // CTAs per SM the register budget targets
    static_assert(KA % TP == 0 && KB % TQ == 0, "rank split");
    static_assert(KA % 2 == 0 && KB % 2 == 0, "16-byte factor rows");
    static_assert(L % 4 == 0, "k-steps of 4");
    static_assert(R % 8 == 0, "m-tiles of 8 rows");
    // shared memory: gather buffer, Y tile, two record buffers, A tile, three row-meta slots
    static constexpr size_t META = (size_t)R * (8 + 4 + 4 + 4) + 16;  // start, len, off, perm, total
    // a record buffer: x[CAP + 2] (f64), j[CAP + 4], k[CAP + 4] (u32) -- SoA, so a tile whose records are one
    // contiguous stream slice is staged with 16-byte copies at the slice's 16-byte-aligned base
    static constexpr size_t RECB = (size_t)(CAP + 2) * 8 + 2 * (size_t)(CAP + 4) * 4;
    static_assert(RECB % 16 == 0, "record buffer alignment");
    static constexpr size_t smem_bytes = (size_t)CAP * FW * 8 + (size_t)R * LDY * 8 + 2 * RECB +
                                         (size_t)R * ALD * 8 + 3 * META + 64;
};

template <int KA, int KB, int KN>
__global__ void __launch_bounds__(Cfg<KA, KB, KN>::THREADS, Cfg<KA, KB, KN>::MINB)
    k_pass_fast3(FastArgs a) {
    using C = Cfg<KA, KB, KN>;
    if (skip_kernel(a.st, a.run_if)) return;
#ifdef HQ_PHASE_TIMING
    long long _ph_t = clock64();
#endif
    extern __shared__ __align__(16) double sm[];
    double* sF = sm;                                          // CAP x FW gathered factor rows
    double* sY = sF + (size_t)C::CAP * C::FW;                 // R x LDY Kronecker rows
    char* sRecB = reinterpret_cast<char*>(sY + (size_t)C::R * C::LDY);  // 2 record buffers (SoA)
    double* sA = reinterpret_cast<double*>(sRecB + 2 * C::RECB);       // R x ALD a_i rows
    auto rx = [&](int rb) { return reinterpret_cast<double*>(sRecB + rb * C::RECB); };
    auto rj = [&](int rb) { return reinterpret_cast<uint32_t*>(sRecB + rb * C::RECB + (C::CAP + 2) * 8); };
    auto rk = [&](int rb) { return rj(rb) + C::CAP + 4; };
    char* sMetaB = reinterpret_cast<char*>(sA + (size_t)C::R * C::ALD);
    // row meta of a tile: start position, length (-1: long row), virtual offset, lane slot -> row, total
    auto m_start = [&](int mb) { return reinterpret_cast<int64_t*>(sMetaB + mb * C::META); };
    auto m_len = [&](int mb) { return reinterpret_cast<int*>(sMetaB + mb * C::META + 8 * C::R); };
    auto m_off = [&](int mb) { return m_len(mb) + C::R; };
    auto m_perm = [&](int mb) { return m_len(mb) + 2 * C::R; };
    auto m_tot = [&](int mb) { return m_len(mb) + 3 * C::R; };
    __shared__ double red[C::WARPS];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    const uint64_t pol_stream = policy_evict_first();
    // with a persisting window on U_a its gathers carry no explicit hint and
    // U_b streams; without one both factors are asked to stay (evict_last)
    const uint64_t pol_a = policy_evict_last();
    const uint64_t pol_b = policy_evict_last();
    for (int q = tid; q < C::R * C::ALD; q += C::THREADS) sA[q] = 0.0;

    // ---- tile range of this CTA (nnz-balanced, static)
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t ntiles = (int64_t)((a.rows + C::R - 1) / C::R);
    const uint64_t rend = a.rbase + a.rows;
    const int64_t zb = a.rowptr[a.rbase];
    const int64_t Z = a.rowptr[rend] - zb;
    auto lower = [&](int64_t z) {
        int64_t lo = 0, hi = ntiles;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            uint64_t r = a.rbase + min((uint64_t)mid * C::R, a.rows);
            if (a.rowptr[r] - zb >= z) hi = mid; else lo = mid + 1;
        }
        return lo;
    };
    const int64_t t0 = lower((Z * c) / G);
    const int64_t t1 = (c == G - 1) ? ntiles : lower((Z * (c + 1)) / G);

    double macc[C::MBW][2];
#pragma unroll
    for (int b = 0; b < C::MBW; ++b) macc[b][0] = macc[b][1] = 0.0;
    // W = A^T A on DMMA: warp w < NT (NT + 1) / 2 owns the upper block (wmA, wmB) of W; its A fragments are
    // the M-GEMM's (same operand layout), so W costs NT (NT + 1) / 2 DMMAs per k-step and no extra loads
    constexpr int NWB = C::NT * (C::NT + 1) / 2;
    static_assert(NWB <= C::WARPS, "one W block per warp");
    const int wmA = (C::NT == 1 || warp < 2) ? 0 : 1, wmB = (C::NT == 1 || warp == 0) ? 0 : 1;
    double wfr0 = 0.0, wfr1 = 0.0;
    double mx = 0.0;

    const double* __restrict__ Ua = a.ua;
    const double* __restrict__ Ub = a.ub;
    const double* __restrict__ gt = a.gt;

    // G_(n)^T fragments of this warp's n-tile, resident for the whole kernel (L1 is nearly all smem here)
    static_assert(C::WARPS % C::NT == 0, "warp -> n-tile mapping");
    constexpr bool kGReg = C::L / 4 <= 32;  // K = 10, 8: fragments fit in registers; K = 16: reloaded per tile
    double gfr[kGReg ? C::L / 4 : 1];
    const int gcolidx = (warp % C::NT) * 8 + (lane >> 2);
    const bool gvalid = a.kind == kTTMcTC && gcolidx < KN;
    if constexpr (kGReg) {
#pragma unroll
        for (int ks = 0; ks < C::L / 4; ++ks)
            gfr[ks] = gvalid ? __ldg(gt + (size_t)(ks * 4 + (lane & 3)) * KN + gcolidx) : 0.0;
    }
    // lane roles in the Kronecker phase
    const int rslot = warp * C::RPW + lane / C::TR;
    const int pb = (lane % C::TR) / C::TQ, qb = lane % C::TQ;
    const int p0 = pb * C::BP, q0 = qb * C::BQ;
    const int sub = lane % C::TR;

    // ---- pipeline helpers (all collective over the CTA unless noted)
    // row meta of tile t from its rowptr slice (st[0..R] already loaded by threads <= R)
    auto meta_from = [&](int64_t t, int mb, int64_t st_lo, int64_t st_hi) {
        const uint64_t r0 = a.rbase + (uint64_t)t * C::R;
        const int nr = (int)min((uint64_t)C::R, rend - r0);
        if (tid < C::R) {
            int len = 0;
            if (tid < nr) {
                const int64_t l = st_hi - st_lo;
                len = (l > a.short_max) ? -1 : (int)l;
            }
            m_len(mb)[tid] = len;
            m_start(mb)[tid] = st_lo;
        }
        const int any_long = __syncthreads_or(tid < C::R && tid < nr && st_hi - st_lo > a.short_max);
        if (tid < C::R) {
            const int* ln = m_len(mb);
            const int me = max(ln[tid], 0);
            int rank = 0, off = 0;
            for (int r = 0; r < C::R; ++r) {
                const int o = max(ln[r], 0);
                rank += (o > me) || (o == me && r < tid);
                off += (r < tid) ? o : 0;
            }
            m_perm(mb)[rank] = tid;
            m_off(mb)[tid] = off;
            if (tid == C::R - 1) {
                m_tot(mb)[0] = off + me;
                // contiguous: the tile's records are the stream slice [start of row 0, + total)
                m_tot(mb)[1] = !any_long && off + me <= C::CAP;
            }
        }
        __syncthreads();
    };
    auto load_starts = [&](int64_t t, int64_t& lo, int64_t& hi) {  // per thread, tid < R
        lo = hi = 0;
        if (t < t1 && tid < C::R) {
            const uint64_t r = a.rbase + (uint64_t)t * C::R + tid;
            if (r < rend) {
                lo = a.rowptr[r];
                hi = a.rowptr[r + 1];
            }
        }
    };
    // records of virtual positions [cv, cv + CAP) of tile (meta mb) -> record buffer rb (per row lanes)
    auto records_issue = [&](int mb, int rb, int cv) {
        if (cv == 0 && m_tot(mb)[1]) {  // one contiguous slice: 16-byte copies from its aligned base
            const int64_t p0 = m_start(mb)[0];
            const int tot = m_tot(mb)[0];
            const int64_t bx = p0 & ~(int64_t)1, bj = p0 & ~(int64_t)3;
            const int nx = (int)((p0 + tot - bx + 1) >> 1), nj = (int)((p0 + tot - bj + 3) >> 2);
            for (int q = tid; q < nx; q += C::THREADS) cp16(rx(rb) + 2 * q, a.val + bx + 2 * q, pol_stream);
            for (int q = tid; q < nj; q += C::THREADS) {
                cp16(rj(rb) + 4 * q, a.ia + bj + 4 * q, pol_stream);
                cp16(rk(rb) + 4 * q, a.ib + bj + 4 * q, pol_stream);
            }
        } else {
            const int lr = m_perm(mb)[rslot];
            const int len = max(m_len(mb)[lr], 0);
            const int voff = m_off(mb)[lr];
            const int64_t pbase = m_start(mb)[lr] - voff;
            const int lo = max(voff, cv), hi = min(voff + len, cv + C::CAP);
            for (int v = lo + sub; v < hi; v += C::TR) {
                const int64_t pz = pbase + v;
                cp8(rx(rb) + (v - cv), a.val + pz, pol_stream);
                cp4(rj(rb) + (v - cv), a.ia + pz, pol_stream);
                cp4(rk(rb) + (v - cv), a.ib + pz, pol_stream);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    // element offsets of record 0 in a record buffer (non-zero only for a contiguous slice)
    auto rec_ox = [&](int mb, int cv) { return (cv == 0 && m_tot(mb)[1]) ? (int)(m_start(mb)[0] & 1) : 0; };
    auto rec_oj = [&](int mb, int cv) { return (cv == 0 && m_tot(mb)[1]) ? (int)(m_start(mb)[0] & 3) : 0; };
    // both factor rows of records [0, cn) -> sF with cp.async, piece-major: consecutive lanes copy
    // consecutive 16-byte pieces of one record's rows.  (Register-staged LDG.128 needs ~100 registers per
    // thread for a whole tile: measured, spills; record-per-thread issue measured 15% slower.)
    constexpr int PA = KA / 2, PP = (KA + KB) / 2;
    auto gathers_issue = [&](int rb, int cn, int oj) {
        // each of the first (THREADS / PP) * PP threads owns one fixed piece slot of every record it copies:
        // no per-piece slot arithmetic, one record index load per piece
        constexpr int RPI = C::THREADS / PP;  // records per iteration
        if (tid < RPI * PP) {
            const int pc = tid % PP;
            const bool isa = pc < PA;
            const double* base = isa ? Ua + 2 * pc : Ub + 2 * (pc - PA);
            const int kk = isa ? KA : KB;
            const int off = isa ? 2 * pc : KA + 2 * (pc - PA);
            const uint64_t pol = isa ? pol_a : pol_b;
            const uint32_t* idxp = (isa ? rj(rb) : rk(rb)) + oj;
            if (isa ? a.l1_a : a.l1_b) {
                for (int e = tid / PP; e < cn; e += RPI)
                    cp16_l1(sF + (size_t)e * C::FW + off, base + (size_t)idxp[e] * kk, pol);
            } else {
                for (int e = tid / PP; e < cn; e += RPI)
                    cp16(sF + (size_t)e * C::FW + off, base + (size_t)idxp[e] * kk, pol);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    __syncthreads();
    if (t0 < t1) {  // prologue: tile t0 gathered, tile t0+1 records in flight
        int64_t lo, hi;
        load_starts(t0, lo, hi);
        meta_from(t0, 0, lo, hi);
        records_issue(0, 0, 0);
        cp_wait_all();
        __syncthreads();
        gathers_issue(0, min(C::CAP, m_tot(0)[0]), rec_oj(0, 0));
        if (t0 + 1 < t1) {
            load_starts(t0 + 1, lo, hi);
            meta_from(t0 + 1, 1, lo, hi);
            records_issue(1, 1, 0);
        }
    }
    for (int64_t t = t0; t < t1; ++t) {
        const int it = (int)(t - t0);
        const int mb = it % 3, rb = it & 1;
        const uint64_t r0 = a.rbase + (uint64_t)t * C::R;
        const int nr = (int)min((uint64_t)C::R, rend - r0);
        int64_t pf_lo, pf_hi;  // tile t+2's rowptr slice, prefetched into registers
        load_starts(t + 2, pf_lo, pf_hi);
        cp_wait_all();  // gathers(t), records(t+1)
        __syncthreads();
        HQ_PHASE(0);
        const int total = m_tot(mb)[0];
        const int lr = m_perm(mb)[rslot];
        const int len = max(m_len(mb)[lr], 0);
        const int voff = m_off(mb)[lr];
        const double* recx = rx(rb) + rec_ox(mb, 0);

        double acc[C::BP][C::BQ];
#pragma unroll
        for (int p = 0; p < C::BP; ++p)
#pragma unroll
            for (int q = 0; q < C::BQ; ++q) acc[p][q] = 0.0;
        auto kron = [&](int e0, int e1) {
#pragma unroll 2
            for (int e = e0; e < e1; ++e) {
                const double x = recx[e];
                const double* f = sF + (size_t)e * C::FW;
                double sa[C::BP], vb[C::BQ];
                lds_block<C::BP>(f, p0, sa);
                lds_block<C::BQ>(f + KA, q0, vb);
#pragma unroll
                for (int p = 0; p < C::BP; ++p) {
                    const double sx = x * sa[p];
#pragma unroll
                    for (int q = 0; q < C::BQ; ++q) acc[p][q] = fma(sx, vb[q], acc[p][q]);
                }
            }
        };
        kron(min(voff, C::CAP), min(voff + len, C::CAP));
        for (int cv = C::CAP; cv < total; cv += C::CAP) {  // tiles above CAP records: extra synchronous rounds
            __syncthreads();
            records_issue(mb, rb, cv);
            cp_wait_all();
            __syncthreads();
            gathers_issue(rb, min(C::CAP, total - cv), 0);
            cp_wait_all();
            __syncthreads();
            kron(max(voff, cv) - cv, min(voff + len, cv + C::CAP) - cv);
        }
        HQ_PHASE(1);
        // Y tile
        {
            double* y = sY + (size_t)lr * C::LDY;
#pragma unroll
            for (int p = 0; p < C::BP; ++p)
#pragma unroll
                for (int q = 0; q < C::BQ; ++q) y[blk_index<C::BP>(p0, p) * KB + blk_index<C::BQ>(q0, q)] = acc[p][q];
            if (C::LP > C::L && pb == 0 && qb == 0)
                for (int l = C::L; l < C::LP; ++l) y[l] = 0.0;
        }
        __syncthreads();  // sF and this tile's record buffer are free
        HQ_PHASE(2);
        if (t + 1 < t1) gathers_issue(rb ^ 1, min(C::CAP, m_tot((mb + 1) % 3)[0]), rec_oj((mb + 1) % 3, 0));
        HQ_PHASE(3);
        const int* ln = m_len(mb);
        if (a.kind == kTTMcTC) {
            // all of this warp's A blocks share one n-tile (b = warp + WARPS*bi, WARPS % NT == 0):
            // interleave the blocks and split the k-chain in two for ILP; G^T fragments are in gfr[]
            const int nt = warp % C::NT;
            constexpr int KSN = C::L / 4;
            double c[C::ABW][2][2];
#pragma unroll
            for (int bi = 0; bi < C::ABW; ++bi) c[bi][0][0] = c[bi][0][1] = c[bi][1][0] = c[bi][1][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < KSN; ++ks)
#pragma unroll
                for (int bi = 0; bi < C::ABW; ++bi) {
                    const int b = warp + bi * C::WARPS;
                    if (b < C::AB) {
                        const int mt = b / C::NT;
                        const double yv = sY[(size_t)(mt * 8 + (lane >> 2)) * C::LDY + (lane & 3) + ks * 4];
                        double gv;
                        if constexpr (kGReg)
                            gv = gfr[ks];
                        else
                            gv = gvalid ? __ldg(gt + (size_t)(ks * 4 + (lane & 3)) * KN + gcolidx) : 0.0;
                        dmma884(c[bi][ks & 1][0], c[bi][ks & 1][1], yv, gv);
                    }
                }
            // epilogue straight from the fragments: long / absent rows zeroed, A written (16-byte stores),
            // max|A|, and the A tile for the M / W products
#pragma unroll
            for (int bi = 0; bi < C::ABW; ++bi) {
                const int b = warp + bi * C::WARPS;
                if (b < C::AB) {
                    const int mt = b / C::NT;
                    const int row = mt * 8 + (lane >> 2);
                    const int col = nt * 8 + 2 * (lane & 3);
                    const bool valid = row < nr && ln[row] >= 0;
                    const double v0 = valid ? c[bi][0][0] + c[bi][1][0] : 0.0;
                    const double v1 = valid ? c[bi][0][1] + c[bi][1][1] : 0.0;
                    sA[row * C::ALD + col] = v0;
                    sA[row * C::ALD + col + 1] = v1;
                    mx = fmax(mx, fmax(fabs(v0), fabs(v1)));  // padding columns are exactly 0
                    if (valid && a.A && col < KN) {
                        double* dst = a.A + (r0 + row) * KN + col;
                        if constexpr (KN % 2 == 0)
                            *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
                        else {
                            dst[0] = v0;
                            if (col + 1 < KN) dst[1] = v1;
                        }
                    }
                }
            }
            __syncthreads();
            HQ_PHASE(4);
        } else {
            for (int q = tid; q < C::R * KN; q += C::THREADS) {
                const int row = q / KN, r = q - row * KN;
                sA[row * C::ALD + r] = (row < nr && ln[row] >= 0) ? a.un[(r0 + row) * KN + r] : 0.0;
            }
            __syncthreads();
            HQ_PHASE(4);
        }
        if (a.kind != kTTMcTC) {
        for (int q = tid; q < C::R * KN; q += C::THREADS) {
            const int row = q / KN, r = q - row * KN;
            const double v = sA[row * C::ALD + r];
            if (row < nr && ln[row] >= 0) {
#ifdef HQ_A_STCS
                if (a.A) __stcs(&a.A[(r0 + row) * KN + r], v);
#else
                if (a.A) a.A[(r0 + row) * KN + r] = v;
#endif
                mx = fmax(mx, fabs(v));
            } else {
                sA[row * C::ALD + r] = 0.0;  // long / absent rows contribute nothing
            }
        }
        __syncthreads();
        }
        HQ_PHASE(5);
        // M += A_tile^T Y_tile (DMMA), W += A^T A (DFMA)
        if (!a.a_only) {
#pragma unroll
        for (int ks = 0; ks < C::R / 4; ++ks)
#pragma unroll
            for (int bi = 0; bi < C::MBW; ++bi) {
                const int b = warp + bi * C::WARPS;
                if (b < C::MB) {
                    const int mt = b / C::NLT, nt = b - mt * C::NLT;
                    const double av = sA[(size_t)(ks * 4 + (lane & 3)) * C::ALD + mt * 8 + (lane >> 2)];
                    const double yv = sY[(size_t)(ks * 4 + (lane & 3)) * C::LDY + nt * 8 + (lane >> 2)];
                    dmma884(macc[bi][0], macc[bi][1], av, yv);
                }
            }
        }
        if (warp < NWB && !a.a_only) {
#pragma unroll
            for (int ks = 0; ks < C::R / 4; ++ks) {
                const double* ar = sA + (size_t)(ks * 4 + (lane & 3)) * C::ALD + (lane >> 2);
                dmma884(wfr0, wfr1, ar[wmA * 8], ar[wmB * 8]);
            }
        }
        __syncthreads();
        HQ_PHASE(6);
        if (t + 2 < t1) {  // tile t+2: meta from the prefetched slice, records into this tile's buffer
            meta_from(t + 2, (mb + 2) % 3, pf_lo, pf_hi);
            records_issue((mb + 2) % 3, rb, 0);
        }
        HQ_PHASE(7);
    }

    // ---- partial slots
    const int slot = a.slot0 + c;
    double* mp = a.mpart + (size_t)slot * KN * C::L;
#pragma unroll
    for (int bi = 0; bi < C::MBW; ++bi) {
        const int b = warp + bi * C::WARPS;
        if (b < C::MB) {
            const int mt = b / C::NLT, nt = b - mt * C::NLT;
            const int r = mt * 8 + (lane >> 2);
            const int l = nt * 8 + 2 * (lane & 3);
            if (r < KN) {
                if (l < C::L) mp[(size_t)r * C::L + l] = macc[bi][0];
                if (l + 1 < C::L) mp[(size_t)r * C::L + l + 1] = macc[bi][1];
            }
        }
    }
    if (warp < NWB) {  // C fragment: W[8 wmA + gid][8 wmB + 2 tig + {0, 1}], mirrored below the diagonal blocks
        double* wp = a.wpart + (size_t)slot * KN * KN;
        const int r = wmA * 8 + (lane >> 2);
        const int c0 = wmB * 8 + 2 * (lane & 3);
        const double v[2] = {wfr0, wfr1};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int cc = c0 + e;
            if (r < KN && cc < KN) {
                wp[r * KN + cc] = v[e];
                if (wmA != wmB) wp[cc * KN + r] = v[e];
            }
        }
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < C::WARPS; ++w) m = fmax(m, red[w]);
        a.maxpart[slot] = m;
    }
}


// ============================================================================
// Three-CTAs-per-SM pass (K = 10): no intra-CTA pipelining -- a tile's
// meta, records, gathers and Kronecker rows run in sequence and the Y tile is
// written over the staged rows -- so a CTA needs ~74 KB of shared memory and
// twelve compute warps share an SM (three independent CTAs overlap each
// other's phases instead of one CTA overlapping its own).
// Records per gather round.  368 is what three CTAs per SM leave room for (3 x (76.7 KB + 1 KB reserved) of the
// SM's 228 KB, 96 bytes to spare): a config-2 tile holds 320 +- 18 records, so 0.4 % of the tiles need a second
// round (3.6 % at 352: pass 0.617 -> 0.609 ms; the rows' sums keep their stream order, same bits).  If the
// device grants fewer than three CTAs per SM at 368, the 352-record instance is used.
#ifndef HQ_NP_CAP
#define HQ_NP_CAP 368
#endif
#ifndef HQ_NP_CAP_SMALL
#define HQ_NP_CAP_SMALL 352
#endif
// records per unrolled step of the Kronecker-row loop (shared loads of the next records behind the DFMAs of this
// one; 2 -> 4: config-2 pass 0.605 -> 0.598 ms; 8 spills)
#ifndef HQ_NP_KU
#define HQ_NP_KU 4
#endif
#define HQ_PRAGMA_(x) _Pragma(#x)
#define HQ_UNROLL(n) HQ_PRAGMA_(unroll n)
#ifndef HQ_NP_MINB
#define HQ_NP_MINB 3
#endif
template <int KA, int KB, int KN, int CAPV>
struct CfgNP : Cfg<KA, KB, KN> {
    static constexpr int CAP = CAPV;
    static constexpr int FW = KA + KB;
    static constexpr int ALD = 12;  // A tile row stride: columns 0..K_n-1 (the M-GEMM reads 8..15 only for K_n > 8)
    static constexpr int GTAB = kGtFragTable;  // the A-GEMM's pre-permuted G_(n)^T fragments (k_gt)
    static constexpr size_t RECB = (size_t)(CAP + 2) * 8 + 2 * (size_t)(CAP + 4) * 4;
    static constexpr size_t SF = (size_t)CAP * FW * 8;
    static constexpr size_t SY = (size_t)Cfg<KA, KB, KN>::R * Cfg<KA, KB, KN>::LDY * 8;
    static_assert(SY <= SF, "the Y tile is written over the staged rows");
    static_assert(KN <= ALD, "A tile row");
    static constexpr size_t smem = SF + RECB + (size_t)Cfg<KA, KB, KN>::R * ALD * 8 + (size_t)GTAB * 8 +
                                   Cfg<KA, KB, KN>::META + Cfg<KA, KB, KN>::R * 4 + 64;
};

template <int KA, int KB, int KN, int CAPV>
__global__ void __launch_bounds__(128, HQ_NP_MINB) k_pass_np3(FastArgs a) {
    using C = CfgNP<KA, KB, KN, CAPV>;
    if (skip_kernel(a.st, a.run_if)) return;
#ifdef HQ_PHASE_TIMING
    long long _ph_t = clock64();
#endif
    extern __shared__ __align__(16) double sm[];
    double* sF = sm;                                                   // staged rows; then the Y tile
    double* sY = sm;
    char* recb = reinterpret_cast<char*>(sm) + C::SF;
    double* rxp = reinterpret_cast<double*>(recb);
    uint32_t* rjp = reinterpret_cast<uint32_t*>(recb + (C::CAP + 2) * 8);
    uint32_t* rkp = rjp + C::CAP + 4;
    double* sA = reinterpret_cast<double*>(recb + C::RECB);
    double* sG = sA + (size_t)C::R * C::ALD;  // fragment table (kTTMcTC)
    char* metab = reinterpret_cast<char*>(sG + C::GTAB);
    int64_t* m_start = reinterpret_cast<int64_t*>(metab);
    int* m_len = reinterpret_cast<int*>(metab + 8 * C::R);
    int* m_off = m_len + C::R;
    int* m_perm = m_len + 2 * C::R;
    int* m_tot = m_len + 3 * C::R;
    __shared__ double red[C::WARPS];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_f = policy_evict_last();
    for (int q = tid; q < C::R * C::ALD; q += C::THREADS) sA[q] = 0.0;
    if (a.kind == kTTMcTC)
        for (int q = tid; q < C::GTAB; q += C::THREADS) sG[q] = a.gt[(size_t)C::L * KN + q];

    const int G = gridDim.x, c = blockIdx.x;
    const int64_t ntiles = (int64_t)((a.rows + C::R - 1) / C::R);
    const uint64_t rend = a.rbase + a.rows;
    const int64_t zb = a.rowptr[a.rbase];
    // CTAs take contiguous tile ranges of equal cost: records + a fixed per-tile cost (meta, barriers, the
    // per-row GEMMs) worth kTileCost records, so ranges of sparse tiles (skewed modes) are not overloaded
    constexpr int64_t kTileCost = 320;
    auto tile_cost = [&](int64_t t) {
        return a.rowptr[a.rbase + min((uint64_t)t * C::R, a.rows)] - zb + kTileCost * t;
    };
    const int64_t Z = tile_cost(ntiles);
    auto lower = [&](int64_t z) {
        int64_t lo = 0, hi = ntiles;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (tile_cost(mid) >= z) hi = mid; else lo = mid + 1;
        }
        return lo;
    };
    const int64_t t0 = lower((Z * c) / G);
    const int64_t t1 = (c == G - 1) ? ntiles : lower((Z * (c + 1)) / G);

    static_assert(KN == 10 && KA == 10 && KB == 10 && C::TR == 4 && C::RPW == 8 && C::BP == 5 && C::BQ == 5,
                  "fragment table layout (gt_frag_table)");
    // M = 13 n-tiles x 2 m-tiles and W's three upper 8 x 8 blocks over 4 warps: warp w owns n-tiles w, w + 4,
    // w + 8 (both m-tiles); n-tile 12 goes to warps 0 (m-tile 0) and 1 (m-tile 1); W_00 and W_11 to warp 2,
    // W_01 to warp 3 -- 7 / 7 / 8 / 7 DMMAs per k-step
    static_assert(C::NLT == 13 && C::WARPS == 4, "M block map");
    constexpr int NTW = 3;
    double macc[NTW][2][2];
#pragma unroll
    for (int j = 0; j < NTW; ++j) macc[j][0][0] = macc[j][0][1] = macc[j][1][0] = macc[j][1][1] = 0.0;
    double xacc0 = 0.0, xacc1 = 0.0, wacc0 = 0.0, wacc1 = 0.0;  // n-tile 12 (warps 0, 1) or W_00 / W_01 (warps 2, 3)
    double w11a = 0.0, w11b = 0.0;                               // W_11 (warp 2)
    double mx = 0.0;
    const double* __restrict__ gt = a.gt;
    const int g8 = lane >> 2;  // the A-GEMM's B-fragment column
    const int rslot = warp * C::RPW + lane / C::TR;
    const int pb = (lane % C::TR) / C::TQ, qb = lane % C::TQ;
    const int p0 = pb * C::BP, q0 = qb * C::BQ, sub = lane % C::TR;
    constexpr int PA = KA / 2, PP = (KA + KB) / 2, RPI = C::THREADS / PP;

    int64_t nlo = 0, nhi = 0;  // rowptr slice of the next tile (threads < R)
    auto load_rp = [&](int64_t t, int64_t& lo, int64_t& hi) {
        lo = hi = 0;
        if (t < t1 && tid < C::R) {
            const uint64_t r = a.rbase + (uint64_t)t * C::R + tid;
            if (r < rend) {
                lo = a.rowptr[r];
                hi = a.rowptr[r + 1];
            }
        }
    };
    load_rp(t0, nlo, nhi);
    for (int64_t t = t0; t < t1; ++t) {
        const uint64_t r0 = a.rbase + (uint64_t)t * C::R;
        const int nr = (int)min((uint64_t)C::R, rend - r0);
        // ---- meta
        // row lengths (-1: long row), exclusive offsets, and ranks by (length desc, row asc): warp 0, one lane
        // per row, with a shuffle scan and a 9-bit ballot radix rank (lengths <= short_max <= kShortMax = 256)
        static_assert(C::R == 32 && kShortMax < 512, "one lane per tile row, 9-bit lengths");
        if (warp == 0) {
            const int ln = (lane < nr) ? ((nhi - nlo > a.short_max) ? -1 : (int)(nhi - nlo)) : 0;
            m_len[lane] = ln;
            m_start[lane] = nlo;
            const int me = max(ln, 0);
            int inc = me;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            m_off[lane] = inc - me;
            if (lane == 31) m_tot[0] = inc;
            unsigned gtm = 0u, eqm = 0xffffffffu;
#pragma unroll
            for (int b = 8; b >= 0; --b) {
                const bool bit = (me >> b) & 1;
                const unsigned B = __ballot_sync(0xffffffffu, bit);
                if (bit) eqm &= B;
                else {
                    gtm |= eqm & B;
                    eqm &= ~B;
                }
            }
            m_perm[__popc(gtm) + __popc(eqm & ((1u << lane) - 1u))] = lane;
        }
        load_rp(t + 1, nlo, nhi);
        __syncthreads();
        HQ_PHASE(0);
        const int total = m_tot[0];
        const int lr = m_perm[rslot];
        const int len = max(m_len[lr], 0);
        const int voff = m_off[lr];
        double acc[C::BP][C::BQ];
#pragma unroll
        for (int p = 0; p < C::BP; ++p)
#pragma unroll
            for (int q = 0; q < C::BQ; ++q) acc[p][q] = 0.0;
        for (int cv = 0; cv < max(total, 1); cv += C::CAP) {
            const int cn = min(C::CAP, total - cv);
            // records of virtual positions [cv, cv + cn): the row's lanes
            {
                const int64_t pbase = m_start[lr] - voff;
                const int lo = max(voff, cv), hi = min(voff + len, cv + C::CAP);
                for (int v = lo + sub; v < hi; v += C::TR) {
                    const int64_t pz = pbase + v;
                    cp8(rxp + (v - cv), a.val + pz, pol_stream);
                    cp4(rjp + (v - cv), a.ia + pz, pol_stream);
                    cp4(rkp + (v - cv), a.ib + pz, pol_stream);
                }
            }
            cp_wait_all();
            __syncthreads();
            HQ_PHASE(1);
            if (tid < RPI * PP) {
                const int pc = tid % PP;
                const bool isa = pc < PA;
                const double* fb = isa ? a.ua + 2 * pc : a.ub + 2 * (pc - PA);
                const int kk = isa ? KA : KB;
                const int off = isa ? 2 * pc : KA + 2 * (pc - PA);
                const uint32_t* idxp = isa ? rjp : rkp;
                if (isa ? a.l1_a : a.l1_b) {
                    for (int e = tid / PP; e < cn; e += RPI)
                        cp16_l1(sF + (size_t)e * C::FW + off, fb + (size_t)idxp[e] * kk, pol_f);
                } else {
                    for (int e = tid / PP; e < cn; e += RPI)
                        cp16(sF + (size_t)e * C::FW + off, fb + (size_t)idxp[e] * kk, pol_f);
                }
            }
            HQ_PHASE(2);
            cp_wait_all();
            __syncthreads();
            HQ_PHASE(3);
            const int e0 = max(voff, cv) - cv, e1 = min(voff + len, cv + C::CAP) - cv;
HQ_UNROLL(HQ_NP_KU)
            for (int e = e0; e < e1; ++e) {
                const double x = rxp[e];
                const double* f = sF + (size_t)e * C::FW;
                double sa[C::BP], vb[C::BQ];
                lds_block<C::BP>(f, p0, sa);
                lds_block<C::BQ>(f + KA, q0, vb);
#pragma unroll
                for (int p = 0; p < C::BP; ++p) {
                    const double sx = x * sa[p];
#pragma unroll
                    for (int q = 0; q < C::BQ; ++q) acc[p][q] = fma(sx, vb[q], acc[p][q]);
                }
            }
            // staged rows / records consumed: before the next round overwrites them (the last round's barrier is
            // after the A-GEMM, which needs only registers, so warps with shorter rows go on to it)
            if (cv + C::CAP < total) __syncthreads();
            HQ_PHASE(4);
        }
        // ---- A_tile = Y_tile G_(n)^T straight from the Kronecker registers.  Lane (g, c) holds the block
        // Y[row g][P_c x Q_c] (the 4 lanes of a row own its four 5 x 5 blocks), which is exactly the DMMA
        // m8n8k4 A-fragment of the warp's 8 rows under a column permutation: k-step ks = 5 p + q takes column
        // pi(ks, c) = P_c[p] K_b + Q_c[q] from lane c.  So output columns 0..7 are 25 DMMAs whose B-fragment is
        // G_(n)^T[pi(ks, c)][g], and columns 8..K_n-1 are per-lane DFMA partials summed over the row's 4 lanes.
        {
            const bool valid = lr < nr && m_len[lr] >= 0;
            if (a.kind == kTTMcTC) {
                // fragments pre-permuted by k_gt (gt_frag_table): gpm[ks][lane] = G_(n)^T[pi(ks, c)][g],
                // gtl[ks][c][0..1] = G_(n)^T[pi(ks, c)][8..9] -- constant offsets, no index arithmetic
                const double* gpm = sG + lane;
                const double* gtl = sG + 32 * (C::BP * C::BQ) + 2 * sub;
                double cc[4][2], ex[2][KN - 8];
#pragma unroll
                for (int u = 0; u < 4; ++u) cc[u][0] = cc[u][1] = 0.0;
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int j = 0; j < KN - 8; ++j) ex[u][j] = 0.0;
#pragma unroll
                for (int p = 0; p < C::BP; ++p)
#pragma unroll
                    for (int q = 0; q < C::BQ; ++q) {
                        const int ks = p * C::BQ + q;
                        const double y = acc[p][q];
                        dmma884(cc[ks & 3][0], cc[ks & 3][1], y, gpm[32 * ks]);
                        const double2 t = *reinterpret_cast<const double2*>(gtl + 8 * ks);
                        ex[ks & 1][0] = fma(y, t.x, ex[ks & 1][0]);
                        ex[ks & 1][1] = fma(y, t.y, ex[ks & 1][1]);
                    }
                const double c0 = (cc[0][0] + cc[1][0]) + (cc[2][0] + cc[3][0]);
                const double c1 = (cc[0][1] + cc[1][1]) + (cc[2][1] + cc[3][1]);
                const double d0 = 0.0, d1 = 0.0;
                double exs[KN - 8];
#pragma unroll
                for (int j = 0; j < KN - 8; ++j) {
                    exs[j] = ex[0][j] + ex[1][j];
                    exs[j] += __shfl_xor_sync(0xffffffffu, exs[j], 1);
                    exs[j] += __shfl_xor_sync(0xffffffffu, exs[j], 2);
                }
                // C fragment: lane (g, c) holds columns 2c, 2c + 1 of row g (= this lane's row lr)
                const double v0 = valid ? c0 + d0 : 0.0, v1 = valid ? c1 + d1 : 0.0;
                double* sa = sA + lr * C::ALD;
                sa[2 * sub] = v0;
                sa[2 * sub + 1] = v1;
                mx = fmax(mx, fmax(fabs(v0), fabs(v1)));
                double* dst = a.A ? a.A + (r0 + lr) * KN : nullptr;
                if (valid && dst) *reinterpret_cast<double2*>(dst + 2 * sub) = make_double2(v0, v1);
                if (sub == 0) {
#pragma unroll
                    for (int j = 0; j < KN - 8; ++j) {
                        const double v = valid ? exs[j] : 0.0;
                        sa[8 + j] = v;
                        mx = fmax(mx, fabs(v));
                    }
                    if (valid && dst) {
                        static_assert((KN - 8) % 2 == 0, "column tail in 16-byte pieces");
#pragma unroll
                        for (int j = 0; j < KN - 8; j += 2)
                            *reinterpret_cast<double2*>(dst + 8 + j) = make_double2(exs[j], exs[j + 1]);
                    }
                }
            } else {  // kCore: a_i = U_n[i]
                for (int r = sub; r < KN; r += C::TR) {
                    const double v = valid ? a.un[(r0 + lr) * KN + r] : 0.0;
                    sA[lr * C::ALD + r] = v;
                    mx = fmax(mx, fabs(v));
                }
            }
        }
        __syncthreads();  // every warp's Kronecker rows done with the staged rows
        if (!a.a_only) {  // Y tile over the staged rows (the M-GEMM's B operand; the standalone TTMcTC needs none)
            double* y = sY + (size_t)lr * C::LDY;
#pragma unroll
            for (int p = 0; p < C::BP; ++p)
#pragma unroll
                for (int q = 0; q < C::BQ; ++q) y[blk_index<C::BP>(p0, p) * KB + blk_index<C::BQ>(q0, q)] = acc[p][q];
            if (C::LP > C::L && pb == 0 && qb == 0)
                for (int l = C::L; l < C::LP; ++l) y[l] = 0.0;
            __syncthreads();
        }
        HQ_PHASE(5);
        HQ_PHASE(6);
        // ---- M += A_tile^T Y_tile, W += A_tile^T A_tile: warp w owns M's n-tiles w, w + 4, ... for both m-tiles,
        // so each k-step loads the two A-fragments once and each Y-fragment once for two DMMAs; W's three
        // upper 8 x 8 blocks reuse the same A-fragments (warps 0-2)
        if (!a.a_only) {
#pragma unroll
            for (int ks = 0; ks < C::R / 4; ++ks) {
                const double* ar = sA + (size_t)(ks * 4 + (lane & 3)) * C::ALD + (lane >> 2);
                const double av0 = ar[0], av1 = (lane >> 2) < KN - 8 ? ar[8] : 0.0;
                const double* yr = sY + (size_t)(ks * 4 + (lane & 3)) * C::LDY + (lane >> 2);
#pragma unroll
                for (int j = 0; j < NTW; ++j) {
                    const double yv = yr[(warp + j * C::WARPS) * 8];
                    dmma884(macc[j][0][0], macc[j][0][1], av0, yv);
                    dmma884(macc[j][1][0], macc[j][1][1], av1, yv);
                }
                if (warp < 2) {
                    dmma884(xacc0, xacc1, warp == 0 ? av0 : av1, yr[12 * 8]);
                } else {
                    dmma884(wacc0, wacc1, av0, warp == 2 ? av0 : av1);
                    if (warp == 2) dmma884(w11a, w11b, av1, av1);
                }
            }
        }
        __syncthreads();
        HQ_PHASE(7);
    }

    const int slot = a.slot0 + c;
    double* mp = a.mpart + (size_t)slot * KN * C::L;
    auto put_m = [&](int mt, int nt, double v0, double v1) {
        const int r = mt * 8 + (lane >> 2), l = nt * 8 + 2 * (lane & 3);
        if (r < KN) {
            if (l < C::L) mp[(size_t)r * C::L + l] = v0;
            if (l + 1 < C::L) mp[(size_t)r * C::L + l + 1] = v1;
        }
    };
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
        put_m(0, warp + j * C::WARPS, macc[j][0][0], macc[j][0][1]);
        put_m(1, warp + j * C::WARPS, macc[j][1][0], macc[j][1][1]);
    }
    if (warp < 2) put_m(warp, 12, xacc0, xacc1);
    else {
        double* wp = a.wpart + (size_t)slot * KN * KN;
        auto put_w = [&](int bA, int bB, double v0, double v1) {
            const int r = bA * 8 + (lane >> 2), c0 = bB * 8 + 2 * (lane & 3);
            const double v[2] = {v0, v1};
#pragma unroll
            for (int e = 0; e < 2; ++e)
                if (r < KN && c0 + e < KN) {
                    wp[r * KN + c0 + e] = v[e];
                    if (bA != bB) wp[(c0 + e) * KN + r] = v[e];
                }
        };
        if (warp == 2) {
            put_w(0, 0, wacc0, wacc1);
            put_w(1, 1, w11a, w11b);
        } else {
            put_w(0, 1, wacc0, wacc1);
        }
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < C::WARPS; ++w) m = fmax(m, red[w]);
        a.maxpart[slot] = m;
    }
}

template <int KA, int KB, int KN>
void launch_fast3(const FastArgs& a, int grid, cudaStream_t s) {
    if constexpr (KA == 10 && KB == 10 && KN == 10) {  // grid = 3 CTAs per SM (fast_grid), one partial slot per CTA
        using CL = CfgNP<KA, KB, KN, HQ_NP_CAP>;
        using CS = CfgNP<KA, KB, KN, HQ_NP_CAP_SMALL>;
        static int large = -1;  // which instance: decided once from the device's occupancy answer
        if (large < 0) {
            HQ_CUDA(cudaFuncSetAttribute(k_pass_np3<KA, KB, KN, HQ_NP_CAP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CL::smem));
            HQ_CUDA(cudaFuncSetAttribute(k_pass_np3<KA, KB, KN, HQ_NP_CAP_SMALL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CS::smem));
            int per_sm = 0;  // the grid (fast_grid) plans HQ_NP_MINB resident CTAs per SM
            HQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pass_np3<KA, KB, KN, HQ_NP_CAP>, 128,
                                                                  CL::smem));
            large = per_sm >= HQ_NP_MINB ? 1 : 0;
        }
        if (large) k_pass_np3<KA, KB, KN, HQ_NP_CAP><<<grid, 128, CL::smem, s>>>(a);
        else k_pass_np3<KA, KB, KN, HQ_NP_CAP_SMALL><<<grid, 128, CS::smem, s>>>(a);
        HQ_CHECK_LAUNCH();
        return;
    } else {  // K = 16 / 8: the software-pipelined two-CTAs-per-SM kernel
        using C = Cfg<KA, KB, KN>;
        static bool attr = false;
        if (!attr) {
            HQ_CUDA(cudaFuncSetAttribute(k_pass_fast3<KA, KB, KN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::smem_bytes));
            attr = true;
        }
        k_pass_fast3<KA, KB, KN><<<grid, C::THREADS, C::smem_bytes, s>>>(a);
        HQ_CHECK_LAUNCH();
    }
}

template <int KA, int KB, int KN>
int grid_fast3() {
    if constexpr (KA == 10 && KB == 10 && KN == 10) return num_sms() * HQ_NP_MINB;
    return num_sms() * Cfg<KA, KB, KN>::MINB;
}

}  // namespace

#ifdef HQ_PHASE_TIMING
void debug_phase_cycles(unsigned long long* out, int reset) {
    HQ_CUDA(cudaMemcpyFromSymbol(out, hq_phase_cycles, sizeof(unsigned long long) * 16));
    if (reset) {
        unsigned long long z[16] = {0};
        HQ_CUDA(cudaMemcpyToSymbol(hq_phase_cycles, z, sizeof(z)));
    }
}
#else
void debug_phase_cycles(unsigned long long* out, int) {
    for (int i = 0; i < 16; ++i) out[i] = 0;
}
#endif

int fast_grid(int ka, int kb, int kn) {
    if (ka == 10 && kb == 10 && kn == 10) return grid_fast3<10, 10, 10>();
    if (ka == 16 && kb == 16 && kn == 16) return grid_fast3<16, 16, 16>();
    if (ka == 8 && kb == 8 && kn == 8) return grid_fast3<8, 8, 8>();
    return num_sms() * 2;
}

bool fast_supported(const ModeShape& sh) {
    if (sh.order != 3) return false;
    const int ka = sh.ko[0], kb = sh.ko[1], kn = sh.kn;
    return (ka == 10 && kb == 10 && kn == 10) || (ka == 16 && kb == 16 && kn == 16) || (ka == 8 && kb == 8 && kn == 8);
}

void launch_fast(const FastArgs& a, const ModeShape& sh, int grid, cudaStream_t s) {
    const int ka = sh.ko[0], kb = sh.ko[1], kn = sh.kn;
    if (ka == 10 && kb == 10 && kn == 10) launch_fast3<10, 10, 10>(a, grid, s);
    else if (ka == 16 && kb == 16 && kn == 16) launch_fast3<16, 16, 16>(a, grid, s);
    else if (ka == 8 && kb == 8 && kn == 8) launch_fast3<8, 8, 8>(a, grid, s);
    else fail(HQ_ERR_INTERNAL, "no specialised pass for this shape");
}

}  // namespace hq
