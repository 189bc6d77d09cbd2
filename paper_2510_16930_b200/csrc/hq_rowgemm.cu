// hq_rowgemm.cu — tall-skinny passes of CholeskyQR2 and the drift product on
// the FP64 tensor path.
//
// One kernel covers every dense I_n x K pass of a mode update:
//   X = A T        (T = R1^-1, R^-1, or the identity)
//   out <- X       (optional; may alias A: each warp reads a row group before
//                   writing it and owns its groups, so in-place is safe)
//   part[c] += X^T Y over the CTA's rows, Y = X (Gram) or another matrix
//              (U_old, for the drift product P = U_new^T U_old)
//   max|A|         (optional)
// Each warp walks groups of 8 rows: the X = A T product and the X^T Y
// accumulation are DMMA m8n8k4 (f64), X is re-laid out through a per-warp
// shared-memory tile.  The K x K accumulators stay in registers; warps are
// combined in fixed order into one partial slot per CTA (deterministic).
// Two kernels share that structure: k_rowgemm_tma (default) stages chunks of
// contiguous rows in a shared-memory ring filled by a producer warp with
// cp.async.bulk; k_rowgemm loads row groups through registers and is kept for
// sources that are not 16-byte aligned (a multi-GPU row slice of A).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "hq_dense.cuh"

namespace hq {

namespace {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

constexpr int kRgWarps = 8;

// B fragments of a K x K transform T (null: none / zero) for X = A T: lane (gid, tig) holds T[4 ks + tig][8 nt + gid]
template <int K, int KS, int NT>
__device__ __forceinline__ void rg_frags(const double* T, double (&tf)[KS][NT], int gid, int tig) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int k = 4 * ks + tig, n = 8 * nt + gid;
            tf[ks][nt] = (T && k < K && n < K) ? T[k * K + n] : 0.0;
        }
}

// a B fragment of T: from the register copy (K <= 16) or from L1 (larger ranks: register budget)
template <int K>
__device__ __forceinline__ double rg_b(double reg, const double* T, int ks, int nt, int gid, int tig) {
    if constexpr (K <= 16) return reg;
    const int k = 4 * ks + tig, n = 8 * nt + gid;
    return (k < K && n < K) ? (T ? __ldg(T + k * K + n) : (k == n ? 1.0 : 0.0)) : 0.0;
}

// Every transform of a mode update (R1^-1, R2^-1, R3^-1, their products, the identity) is upper triangular, so
// T[k][n] = 0 for k > n: the 8-column tile nt of X = A T needs only the k-steps with 4 ks <= 8 nt + 7.  The
// skipped products are exact zeros, so the result has the same bits.
__device__ __forceinline__ constexpr int rg_ksteps(int KS, int nt) { return KS < 2 * (nt + 1) ? KS : 2 * (nt + 1); }

// second stage of a two-stage product, in place on the warp's 8-row X tile: X <- fl(X T2).  The first stage's
// rounded X is exactly what a materialised pass would have written and re-read (CholeskyQR's Q1 / Q2).
template <int K, int KS, int NT, int LD>
__device__ __forceinline__ void rg_stage2(double* sx, const double (&tf2)[KS][NT], const double* T2, int gid,
                                          int tig) {
    constexpr bool kRegs = K <= 16;  // larger ranks read T2's fragments from L1 (register budget)
    double a[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) a[ks] = (4 * ks + tig < K) ? sx[gid * LD + 4 * ks + tig] : 0.0;
    __syncwarp();
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < rg_ksteps(KS, nt); ++ks) {
            const int k = 4 * ks + tig, n = 8 * nt + gid;
            const double b = kRegs ? tf2[ks][nt] : ((k < K && n < K) ? __ldg(T2 + k * K + n) : 0.0);
            dmma884(c0, c1, a[ks], b);
        }
        const int col = 8 * nt + 2 * tig;
        sx[gid * LD + col] = c0;
        sx[gid * LD + col + 1] = c1;
    }
    __syncwarp();
}

template <int K>
struct RG {
    static constexpr int NT = (K + 7) / 8;  // 8-wide tiles of the K dimension
    static constexpr int KP = NT * 8;
    static constexpr int KS = (K + 3) / 4;  // k-steps of X = A T
    static constexpr int LD = KP + 4;       // smem row stride (= 4 mod 8 doubles: fragment reads conflict-free)
};

// the shifted apply (RowGemm::alt): one stage over the materialised Q2 with T2 = R3^-1
__device__ __forceinline__ void rg_select(const RowGemm& g, const double*& A, const double*& T, const double*& T2) {
    const bool alt = g.alt && g.st && g.st->shifted;
    A = alt ? g.alt : g.A;
    T = alt ? g.T2 : g.T;
    T2 = alt ? nullptr : g.T2;
}

template <int K>
__global__ void __launch_bounds__(kRgWarps * 32) k_rowgemm(RowGemm g) {
    using C = RG<K>;
    if (skip_kernel(g.st, g.run_if)) return;
    const double* A;
    const double* T;
    const double* T2;
    rg_select(g, A, T, T2);
    const uint64_t rows = g.rows;
    double* out = g.out;
    const int npeer = out ? g.npeer : 0;
    const RowGemm& gp = g;
    const double* __restrict__ other = g.other;
    double* __restrict__ part = g.part;
    double* __restrict__ maxpart = g.maxpart;
    __shared__ double sX[kRgWarps][8 * C::LD];
    __shared__ double sY[kRgWarps][8 * C::LD];
    __shared__ double sRed[C::KP * C::KP];
    __shared__ double sMax[kRgWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gid = lane >> 2, tig = lane & 3;

    double tf[C::KS][C::NT];
#pragma unroll
    for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt) {
            const int k = 4 * ks + tig, n = 8 * nt + gid;
            double v = 0.0;
            if (K <= 16 && k < K && n < K) v = T ? T[k * K + n] : (k == n ? 1.0 : 0.0);
            tf[ks][nt] = v;
        }
    double tf2[C::KS][C::NT];
    rg_frags<K, C::KS, C::NT>(K <= 16 ? T2 : nullptr, tf2, gid, tig);
    double acc[C::NT][C::NT][2];
#pragma unroll
    for (int i = 0; i < C::NT; ++i)
#pragma unroll
        for (int j = 0; j < C::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int q = lane; q < 8 * C::LD; q += 32) {
        sX[warp][q] = 0.0;
        sY[warp][q] = 0.0;
    }
    __syncwarp();

    const uint64_t groups = (rows + 7) / 8;
    const uint64_t W = (uint64_t)gridDim.x * kRgWarps, w = (uint64_t)blockIdx.x * kRgWarps + warp;
    const uint64_t gb = groups * w / W, ge = groups * (w + 1) / W;
    double mx = 0.0;
    double* sx = sX[warp];
    double* sa = sx;  // the A tile and the X tile share storage (A read into fragments first)
    double* sy = sY[warp];
    // an 8-row group of A / `other` is 8K contiguous doubles: loaded coalesced
    // (lane-strided), re-laid out through shared memory
    constexpr int OQ = (8 * K + 31) / 32;
    auto load_g = [&](uint64_t g, double (&ad)[OQ], double (&od)[OQ]) {
#pragma unroll
        for (int i = 0; i < OQ; ++i) {
            const int q = lane + 32 * i;
            const uint64_t e = g * 8 * K + q;
            const bool v = g < ge && q < 8 * K && e < rows * K;
            ad[i] = v ? A[e] : 0.0;
            od[i] = (other && v) ? other[e] : 0.0;
        }
    };
    auto process = [&](uint64_t g, const double (&ad)[OQ], const double (&od)[OQ]) {
#pragma unroll
        for (int i = 0; i < OQ; ++i) {
            const int q = lane + 32 * i;
            if (q < 8 * K) {
                const int r = q / K, cc = q - r * K;
                sa[r * C::LD + cc] = ad[i];
                mx = fmax(mx, fabs(ad[i]));
                if (other) sy[r * C::LD + cc] = od[i];
            }
        }
        __syncwarp();
        double a[C::KS];
#pragma unroll
        for (int ks = 0; ks < C::KS; ++ks) a[ks] = sa[gid * C::LD + 4 * ks + tig];
        __syncwarp();
        // X = A T (C fragment: row gid, cols 8nt + 2 tig + {0,1})
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt) {
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < rg_ksteps(C::KS, nt); ++ks)
                dmma884(c0, c1, a[ks], rg_b<K>(tf[ks][nt], T, ks, nt, gid, tig));
            const int col = 8 * nt + 2 * tig;
            sx[gid * C::LD + col] = c0;
            sx[gid * C::LD + col + 1] = c1;
        }
        __syncwarp();
        if (T2) rg_stage2<K, C::KS, C::NT, C::LD>(sx, tf2, T2, gid, tig);
        if (out) {
#pragma unroll
            for (int i = 0; i < OQ; ++i) {
                const int q = lane + 32 * i;
                const uint64_t e = g * 8 * K + q;
                if (q < 8 * K && e < rows * K) {
                    const int r = q / K, cc = q - r * K;
                    const double v = sx[r * C::LD + cc];
                    out[e] = v;
                    for (int pr = 0; pr < npeer; ++pr) gp.peer_out[pr][e] = v;
                }
            }
        }
        const double* y = other ? sy : sx;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int mt = 0; mt < C::NT; ++mt) {
                const double av = sx[(4 * ks + tig) * C::LD + 8 * mt + gid];
#pragma unroll
                for (int nt = 0; nt < C::NT; ++nt)
                    if (other || nt >= mt)  // a Gram is symmetric: its lower tiles are mirrored at the end
                        dmma884(acc[mt][nt][0], acc[mt][nt][1], av, y[(4 * ks + tig) * C::LD + 8 * nt + gid]);
            }
        __syncwarp();
    };
    // two row groups in flight ahead of the one being multiplied
    double a0[OQ], o0[OQ], a1[OQ], o1[OQ];
    load_g(gb, a0, o0);
    load_g(gb + 1, a1, o1);
    for (uint64_t g = gb; g < ge; g += 2) {
        process(g, a0, o0);
        load_g(g + 2, a0, o0);
        if (g + 1 < ge) {
            process(g + 1, a1, o1);
            load_g(g + 3, a1, o1);
        }
    }
    // fixed-order combination of the warps' fragments: ((w0 + w1) + w2) + ...
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if (lane == 0) sMax[warp] = mx;
    for (int ww = 0; ww < kRgWarps; ++ww) {
        if (warp == ww) {
#pragma unroll
            for (int mt = 0; mt < C::NT; ++mt)
#pragma unroll
                for (int nt = 0; nt < C::NT; ++nt) {
                    const int p = 8 * mt + gid, q = 8 * nt + 2 * tig;
                    double* d = sRed + p * C::KP + q;
                    d[0] = (ww == 0 ? 0.0 : d[0]) + acc[mt][nt][0];
                    d[1] = (ww == 0 ? 0.0 : d[1]) + acc[mt][nt][1];
                }
        }
        __syncthreads();
    }
    if (part)
        for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
            const int p = e / K, q = e - p * K;
            const bool mirror = !other && (p >> 3) > (q >> 3);
            part[(size_t)blockIdx.x * K * K + e] = mirror ? sRed[q * C::KP + p] : sRed[p * C::KP + q];
        }
    if (maxpart && threadIdx.x == 0) {
        double m = 0.0;
        for (int ww = 0; ww < kRgWarps; ++ww) m = fmax(m, sMax[ww]);
        maxpart[blockIdx.x] = m;
    }
}

// ============================================================================
// Bulk-copy pipelined variant (the default; one CTA per SM, grid = dense_slots()).
//
// The pass streams A (and `other`) once, so it is an HBM pass whose speed is
// set by how many bytes are in flight.  A CTA owns a contiguous range of
// 8*CW-row chunks; a producer warp moves each chunk (contiguous rows*K
// doubles) into a kTStages-deep shared-memory ring with cp.async.bulk (TMA
// engine, completion counted in bytes on a per-stage mbarrier), so 3-4 chunks
// per SM are always in flight without holding registers.  CW consumer warps
// each take one 8-row group of a chunk, with the same DMMA m8n8k4 products as
// above (X = A T, X^T Y), write X coalesced, and release the stage.

__device__ __forceinline__ uint32_t s_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_addr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(s_addr(b)) : "memory");
}
__device__ __forceinline__ void mb_arrive_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(s_addr(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mb_try(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(s_addr(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// bounded wait: a lost arrival traps (a CUDA error the host reports) instead of hanging the device
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
    if (mb_try(b, parity)) return;
    const long long t0 = clock64();
    while (!mb_try(b, parity)) {
        if (clock64() - t0 > (1ll << 33)) {
            printf("hq: rowgemm pipeline barrier timeout: cta %d thread %d\n", (int)blockIdx.x, (int)threadIdx.x);
            __trap();
        }
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s_addr(dst)),
                 "l"(src), "r"(bytes), "r"(s_addr(b))
                 : "memory");
}
__device__ __forceinline__ void cbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int K>
struct RT {
    static constexpr int CW = K <= 16 ? 16 : 8;  // consumer warps (K > 16: register budget of the K x K fragments)
    static constexpr int ROWS = 8 * CW;           // rows per chunk
    static constexpr int NT = (K + 7) / 8;
    static constexpr int KP = NT * 8;
    static constexpr int KS = (K + 3) / 4;
    static constexpr int LD = KP + 4;
    static constexpr int CHD = ROWS * K;  // doubles per chunk per array
    // ring of chunk buffers: S2 stages of (A, other) pairs, or 2 S2 stages of A alone -- as many bytes in
    // flight as ~190 KB of shared memory holds (the pass is bound by bytes in flight x latency)
    static constexpr int SB = 190 * 1024;
    static constexpr int S2 = SB / (2 * CHD * 8) < 8 ? SB / (2 * CHD * 8) : 8;
    static_assert(S2 >= 2, "chunk ring");
    static constexpr int MAXS = 2 * S2;
    static constexpr size_t smem = (size_t)2 * S2 * CHD * 8 + (size_t)CW * 8 * LD * 8 + (size_t)KP * KP * 8 +
                                   CW * 8 + 2 * MAXS * 8 + 64;
};

template <int K>
__global__ void __launch_bounds__((RT<K>::CW + 1) * 32, 1) k_rowgemm_tma(RowGemm g) {
    using C = RT<K>;
    constexpr int kTcW = C::CW, kTRows = C::ROWS;
    if (skip_kernel(g.st, g.run_if)) return;
    const double* A;
    const double* T;
    const double* T2;
    rg_select(g, A, T, T2);
    const uint64_t rows = g.rows;
    double* out = g.out;
    const int npeer = out ? g.npeer : 0;
    const RowGemm& gp = g;
    const double* __restrict__ other = g.other;
    double* __restrict__ part = g.part;
    double* __restrict__ maxpart = g.maxpart;
    extern __shared__ __align__(128) double rsm[];
    const int NS = other ? C::S2 : C::MAXS;                   // stages
    double* sA = rsm;                                         // NS x CHD
    double* sO = sA + (size_t)NS * C::CHD;                    // NS x CHD (other)
    double* sXall = rsm + (size_t)2 * C::S2 * C::CHD;         // kTcW x 8 x LD
    double* sRed = sXall + (size_t)kTcW * 8 * C::LD;          // KP x KP
    double* sMax = sRed + C::KP * C::KP;                      // kTcW
    uint64_t* full = reinterpret_cast<uint64_t*>(sMax + kTcW);
    uint64_t* empty = full + C::MAXS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gid = lane >> 2, tig = lane & 3;

    const uint64_t nch = (rows + kTRows - 1) / kTRows;
    const uint64_t cb = nch * blockIdx.x / gridDim.x, ce = nch * (blockIdx.x + 1) / gridDim.x;
    const int my = (int)(ce - cb);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mb_init(&full[s], 1);
            mb_init(&empty[s], kTcW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kTcW) {  // ---------------- producer
        if (lane == 0) {
            for (int j = 0; j < my; ++j) {
                const int s = j % NS;
                if (j >= NS) mb_wait(&empty[s], ((j / NS) - 1) & 1);
                const uint64_t r0 = (cb + j) * kTRows;
                const uint64_t nr = min((uint64_t)kTRows, rows - r0);
                const uint32_t n = (uint32_t)(nr * K);  // doubles
                const uint32_t n2 = n & ~1u;            // bulk copies move whole 16-byte units
                if (n2 != n) {                          // odd tail: the last double by hand, before the arrive
                    sA[(size_t)s * C::CHD + n - 1] = A[r0 * K + n - 1];
                    if (other) sO[(size_t)s * C::CHD + n - 1] = other[r0 * K + n - 1];
                }
                mb_arrive_tx(&full[s], n2 * 8 * (other ? 2 : 1));
                if (n2) {
                    bulk_g2s(sA + (size_t)s * C::CHD, A + r0 * K, n2 * 8, &full[s]);
                    if (other) bulk_g2s(sO + (size_t)s * C::CHD, other + r0 * K, n2 * 8, &full[s]);
                }
            }
        }
        return;
    }

    // ---------------- consumers: warp w owns rows [8w, 8w + 8) of every chunk
    double tf[C::KS][C::NT];
#pragma unroll
    for (int ks = 0; ks < C::KS; ++ks)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt) {
            const int k = 4 * ks + tig, n = 8 * nt + gid;
            double v = 0.0;
            if (K <= 16 && k < K && n < K) v = T ? T[k * K + n] : (k == n ? 1.0 : 0.0);
            tf[ks][nt] = v;
        }
    double tf2[C::KS][C::NT];
    rg_frags<K, C::KS, C::NT>(K <= 16 ? T2 : nullptr, tf2, gid, tig);
    double acc[C::NT][C::NT][2];
#pragma unroll
    for (int i = 0; i < C::NT; ++i)
#pragma unroll
        for (int j = 0; j < C::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    double* sx = sXall + (size_t)warp * 8 * C::LD;
    for (int q = lane; q < 8 * C::LD; q += 32) sx[q] = 0.0;
    __syncwarp();
    double mx = 0.0;
    const int grow = 8 * warp + gid;  // this lane's row within a chunk (A fragments)

    for (int j = 0; j < my; ++j) {
        const int s = j % NS;
        const uint64_t r0 = (cb + j) * kTRows;
        const int nr = (int)min((uint64_t)kTRows, rows - r0);
        mb_wait(&full[s], (j / NS) & 1);
        const double* ca = sA + (size_t)s * C::CHD;
        const double* co = sO + (size_t)s * C::CHD;
        double a[C::KS];
#pragma unroll
        for (int ks = 0; ks < C::KS; ++ks) {
            const int col = 4 * ks + tig;
            a[ks] = (grow < nr && col < K) ? ca[grow * K + col] : 0.0;
            mx = fmax(mx, fabs(a[ks]));
        }
        // X = A T (C fragment: row gid, cols 8nt + 2 tig + {0,1}) -> sx
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt) {
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < rg_ksteps(C::KS, nt); ++ks)
                dmma884(c0, c1, a[ks], rg_b<K>(tf[ks][nt], T, ks, nt, gid, tig));
            const int col = 8 * nt + 2 * tig;
            sx[gid * C::LD + col] = c0;
            sx[gid * C::LD + col + 1] = c1;
        }
        __syncwarp();
        if (T2) rg_stage2<K, C::KS, C::NT, C::LD>(sx, tf2, T2, gid, tig);
        const int gr0 = 8 * warp;
        if (out) {
            const int lim = max(0, min(8, nr - gr0)) * K;
            double* og = out + (r0 + gr0) * K;
            const uint64_t ob = (r0 + gr0) * K;
            for (int q = lane; q < lim; q += 32) {
                const int r = q / K, cc = q - r * K;
                const double v = sx[r * C::LD + cc];
                og[q] = v;
                for (int pr = 0; pr < npeer; ++pr) gp.peer_out[pr][ob + q] = v;
            }
        }
        // X^T Y: k = the group's rows.  Rows past the chunk end are zero in sx (A fragments were zeroed).
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
            const int rr = 4 * ks + tig;  // row within the group
#pragma unroll
            for (int mt = 0; mt < C::NT; ++mt) {
                const double av = sx[rr * C::LD + 8 * mt + gid];
#pragma unroll
                for (int nt = 0; nt < C::NT; ++nt) {
                    if (other) {
                        const int col = 8 * nt + gid;
                        const double yv = (gr0 + rr < nr && col < K) ? co[(gr0 + rr) * K + col] : 0.0;
                        dmma884(acc[mt][nt][0], acc[mt][nt][1], av, yv);
                    } else if (nt >= mt) {  // a Gram is symmetric: its lower tiles are mirrored at the end
                        dmma884(acc[mt][nt][0], acc[mt][nt][1], av, sx[rr * C::LD + 8 * nt + gid]);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mb_arrive(&empty[s]);
    }

    // fixed-order combination of the consumer warps' fragments
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if (lane == 0) sMax[warp] = mx;
    constexpr int CT = kTcW * 32;
    for (int ww = 0; ww < kTcW; ++ww) {
        if (warp == ww) {
#pragma unroll
            for (int mt = 0; mt < C::NT; ++mt)
#pragma unroll
                for (int nt = 0; nt < C::NT; ++nt) {
                    const int p = 8 * mt + gid, q = 8 * nt + 2 * tig;
                    double* d = sRed + p * C::KP + q;
                    d[0] = (ww == 0 ? 0.0 : d[0]) + acc[mt][nt][0];
                    d[1] = (ww == 0 ? 0.0 : d[1]) + acc[mt][nt][1];
                }
        }
        cbar(1, CT);
    }
    if (part)
        for (int e = threadIdx.x; e < K * K; e += CT) {
            const int p = e / K, q = e - p * K;
            const bool mirror = !other && (p >> 3) > (q >> 3);
            part[(size_t)blockIdx.x * K * K + e] = mirror ? sRed[q * C::KP + p] : sRed[p * C::KP + q];
        }
    if (maxpart && threadIdx.x == 0) {
        double m = 0.0;
        for (int ww = 0; ww < kTcW; ++ww) m = fmax(m, sMax[ww]);
        maxpart[blockIdx.x] = m;
    }
}

template <int K>
void launch_rg(const RowGemm& g, cudaStream_t s) {
    // bulk copies need 16-byte aligned sources (a row-range slice of A in the multi-GPU path may start
    // mid-unit): those take the register-staged kernel
    auto al = [](const double* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
    const bool aligned = al(g.A) && (!g.other || al(g.other)) && (!g.alt || al(g.alt));
    if (aligned) {
        using C = RT<K>;
        static bool attr = false;
        if (!attr) {
            HQ_CUDA(cudaFuncSetAttribute(k_rowgemm_tma<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem));
            attr = true;
        }
        k_rowgemm_tma<K><<<dense_slots(), (C::CW + 1) * 32, C::smem, s>>>(g);
    } else {
        k_rowgemm<K><<<dense_slots(), kRgWarps * 32, 0, s>>>(g);
    }
    HQ_CHECK_LAUNCH();
}

}  // namespace

bool rowgemm_supported(int K) { return K >= 1 && K <= 32; }

void launch_rowgemm(int K, const RowGemm& g, cudaStream_t s) {
    switch (K) {
#define HQ_K(KK) case KK: launch_rg<KK>(g, s); return;
        HQ_K(1) HQ_K(2) HQ_K(3) HQ_K(4) HQ_K(5) HQ_K(6) HQ_K(7) HQ_K(8) HQ_K(9) HQ_K(10) HQ_K(11) HQ_K(12)
        HQ_K(13) HQ_K(14) HQ_K(15) HQ_K(16) HQ_K(17) HQ_K(18) HQ_K(19) HQ_K(20) HQ_K(21) HQ_K(22) HQ_K(23)
        HQ_K(24) HQ_K(25) HQ_K(26) HQ_K(27) HQ_K(28) HQ_K(29) HQ_K(30) HQ_K(31) HQ_K(32)
#undef HQ_K
        default: fail(HQ_ERR_CAPACITY, "rank above 32");
    }
}

void launch_rowgemm(int K, const double* A, uint64_t rows, const double* T, double* out, const double* other,
                    double* part, double* maxpart, const DevStatus* st, int run_if, cudaStream_t s) {
    RowGemm g{};
    g.A = A;
    g.rows = rows;
    g.T = T;
    g.out = out;
    g.other = other;
    g.part = part;
    g.maxpart = maxpart;
    g.st = st;
    g.run_if = run_if;
    launch_rowgemm(K, g, s);
}

}  // namespace hq
