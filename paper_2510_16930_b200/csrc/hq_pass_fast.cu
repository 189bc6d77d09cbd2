// hq_pass_fast.cu — specialised fused mode pass for order-3 tensors with
// compile-time ranks (the BASELINE shapes: K = 10, 16, 8).
//
// Same contract as the generic tile kernel in hq_pass.cu (per row i of the
// mode-n unfolding: Y_i, a_i = Y_i G_(n)^T or U_n[i], partials of
// M = sum a_i^T Y_i, W = sum a_i^T a_i, max|a_i|), mapped onto the B200 FP64
// datapath, which DFMA and DMMA share (measured: 35.4 / 37.1 TFLOP/s alone,
// 36.7 mixed — tools/microbench_mix.cu):
//
//  * tile = R consecutive short rows; rows are ranked by length inside the
//    tile and dealt to warps in that order, so the TR lanes of a row and the
//    rows sharing a warp run loops of near-equal length.
//  * Kronecker phase (DFMA): lane (row, pb, qb) owns a BP x BQ block of
//    Y_i = sum_e x_e U_a[j_e, :] (x) U_b[k_e, :]; factor rows are gathered
//    straight from L2 with 16-byte loads (two 80-byte rows per nonzero is the
//    whole of this pass's random traffic).
//  * GEMM phase (DMMA m8n8k4 f64): A_tile = Y_tile G_(n)^T and
//    M += A_tile^T Y_tile with G^T and Y_tile in shared memory; M's C
//    fragments live in registers across all tiles of the CTA.
//  * W += A^T A and max|A| with DFMA on the A tile in shared memory.
// Deterministic: fixed row->lane assignment per tile, fixed tile->CTA
// assignment, per-CTA partial slots reduced in fixed order.
#include <algorithm>

#include "hq_fast.cuh"

namespace hq {

namespace {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

// Loads B consecutive doubles starting at p (8-byte aligned; 16-byte aligned
// when `odd` is false) with 16-byte loads and no divergence: always reads the
// aligned window [p - odd, p - odd + 2*ceil((B+1)/2)) and shifts.
template <int B>
__device__ __forceinline__ void load_part(const double* p, bool odd, double (&v)[B]) {
    constexpr int W = (B + 2) / 2;  // double2 words covering B+1 doubles
    double w[2 * W];
    const double* base = p - (odd ? 1 : 0);
#pragma unroll
    for (int i = 0; i < W; ++i) {
        double2 d = ldg2(base + 2 * i);
        w[2 * i] = d.x;
        w[2 * i + 1] = d.y;
    }
#pragma unroll
    for (int i = 0; i < B; ++i) v[i] = odd ? w[i + 1] : w[i];
}

// Exact-width loads when every block start is 16-byte aligned.
template <int B>
__device__ __forceinline__ void load_part_aligned(const double* p, double (&v)[B]) {
#pragma unroll
    for (int i = 0; i < B / 2; ++i) {
        double2 d = ldg2(p + 2 * i);
        v[2 * i] = d.x;
        v[2 * i + 1] = d.y;
    }
    if (B & 1) v[B - 1] = __ldg(p + B - 1);
}

template <int KA, int KB, int KN>
struct Cfg {
    static constexpr int L = KA * KB;
    static constexpr int TP = 2;
    static constexpr int TQ = (KB >= 16) ? 4 : 2;
    static constexpr int TR = TP * TQ;          // lanes per row
    static constexpr int BP = KA / TP;
    static constexpr int BQ = KB / TQ;
    static constexpr int RPW = 32 / TR;         // rows per warp
    static constexpr int WARPS = 8;
    static constexpr int THREADS = 32 * WARPS;
    static constexpr int R = RPW * WARPS;       // rows per tile
    static constexpr int LP = (L + 7) / 8 * 8;  // Y columns padded to whole n-tiles
    static constexpr int LDY = LP + 4;          // Y row stride (doubles)
    static constexpr int NT = (KN + 7) / 8;     // A n-tiles
    static constexpr int GLD = NT * 8;          // G^T row stride
    static constexpr int ALD = NT * 8 + 1;      // A tile row stride
    static constexpr int MT = NT;               // M m-tiles
    static constexpr int NLT = LP / 8;          // M n-tiles
    static constexpr int MB = MT * NLT;         // M blocks
    static constexpr int MBW = (MB + WARPS - 1) / WARPS;
    static constexpr int AB = (R / 8) * NT;     // A blocks
    static constexpr int ABW = (AB + WARPS - 1) / WARPS;
    static constexpr int WQ = (KN * KN + THREADS - 1) / THREADS;
    static_assert(KA % TP == 0 && KB % TQ == 0, "rank split");
    static_assert(L % 4 == 0, "k-steps of 4");
    static_assert(R % 8 == 0, "m-tiles of 8 rows");
    static constexpr size_t smem_doubles = (size_t)L * GLD + (size_t)R * LDY + (size_t)R * ALD;
    static constexpr size_t smem_bytes = smem_doubles * 8 + 2 * R * sizeof(int);
};

template <int KA, int KB, int KN>
__global__ void __launch_bounds__(Cfg<KA, KB, KN>::THREADS)
    k_pass_fast3(FastArgs a) {
    using C = Cfg<KA, KB, KN>;
    if (skip_kernel(a.st, a.run_if)) return;
    extern __shared__ double sm[];
    double* sG = sm;                                  // L x GLD   (G_(n)^T, zero-padded)
    double* sY = sG + (size_t)C::L * C::GLD;          // R x LDY   (Kronecker rows)
    double* sA = sY + (size_t)C::R * C::LDY;          // R x ALD   (a_i rows)
    int* sLen = reinterpret_cast<int*>(sA + (size_t)C::R * C::ALD);
    int* sPerm = sLen + C::R;
    __shared__ double red[C::WARPS];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int q = tid; q < C::L * C::GLD; q += C::THREADS) {
        int l = q / C::GLD, r = q - l * C::GLD;
        sG[q] = (a.kind == kTTMcTC && r < KN) ? a.gt[(size_t)l * KN + r] : 0.0;
    }
    for (int q = tid; q < C::R * C::LDY; q += C::THREADS) sY[q] = 0.0;
    for (int q = tid; q < C::R * C::ALD; q += C::THREADS) sA[q] = 0.0;

    // ---- tile range of this CTA (nnz-balanced, static)
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t ntiles = (int64_t)((a.rows + C::R - 1) / C::R);
    const int64_t Z = a.rowptr[a.rows];
    auto lower = [&](int64_t z) {
        int64_t lo = 0, hi = ntiles;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            uint64_t r = min((uint64_t)mid * C::R, a.rows);
            if (a.rowptr[r] >= z) hi = mid; else lo = mid + 1;
        }
        return lo;
    };
    const int64_t t0 = lower((Z * c) / G);
    const int64_t t1 = (c == G - 1) ? ntiles : lower((Z * (c + 1)) / G);

    double macc[C::MBW][2];
#pragma unroll
    for (int b = 0; b < C::MBW; ++b) macc[b][0] = macc[b][1] = 0.0;
    double wacc[C::WQ];
#pragma unroll
    for (int b = 0; b < C::WQ; ++b) wacc[b] = 0.0;
    double mx = 0.0;

    const double* __restrict__ Ua = a.ua;
    const double* __restrict__ Ub = a.ub;
    const double* __restrict__ val = a.val;
    const uint32_t* __restrict__ ia = a.ia;
    const uint32_t* __restrict__ ib = a.ib;

    // lane roles in the Kronecker phase
    const int rslot = warp * C::RPW + lane / C::TR;
    const int pb = (lane % C::TR) / C::TQ, qb = lane % C::TQ;
    const int p0 = pb * C::BP, q0 = qb * C::BQ;

    __syncthreads();
    for (int64_t t = t0; t < t1; ++t) {
        const uint64_t r0 = (uint64_t)t * C::R;
        const int nr = (int)min((uint64_t)C::R, a.rows - r0);
        if (tid < C::R) {
            int len = 0;
            if (tid < nr) {
                int64_t l = a.rowptr[r0 + tid + 1] - a.rowptr[r0 + tid];
                len = (l > kShortMax) ? -1 : (int)l;  // -1: long row (segmented path)
            }
            sLen[tid] = len;
        }
        __syncthreads();
        if (tid < C::R) {  // rank rows by length, descending, ties by index
            const int me = max(sLen[tid], 0);
            int rank = 0;
            for (int r = 0; r < C::R; ++r) {
                int o = max(sLen[r], 0);
                rank += (o > me) || (o == me && r < tid);
            }
            sPerm[rank] = tid;
        }
        __syncthreads();

        // ---- Kronecker rows (DFMA)
        {
            const int lr = sPerm[rslot];
            const int len = max(sLen[lr], 0);
            const int64_t zb = len ? a.rowptr[r0 + lr] : 0;
            double acc[C::BP][C::BQ];
#pragma unroll
            for (int p = 0; p < C::BP; ++p)
#pragma unroll
                for (int q = 0; q < C::BQ; ++q) acc[p][q] = 0.0;
            for (int e = 0; e < len; ++e) {
                const int64_t z = zb + e;
                const double x = __ldg(val + z);
                const uint32_t j = __ldg(ia + z), k = __ldg(ib + z);
                double sa[C::BP], vb[C::BQ];
                if constexpr (C::BP % 2 == 0) {
                    load_part_aligned<C::BP>(Ua + (size_t)j * KA + p0, sa);
                } else {
                    load_part<C::BP>(Ua + (size_t)j * KA + p0, (p0 & 1) != 0, sa);
                }
                if constexpr (C::BQ % 2 == 0) {
                    load_part_aligned<C::BQ>(Ub + (size_t)k * KB + q0, vb);
                } else {
                    load_part<C::BQ>(Ub + (size_t)k * KB + q0, (q0 & 1) != 0, vb);
                }
#pragma unroll
                for (int p = 0; p < C::BP; ++p) {
                    const double s = x * sa[p];
#pragma unroll
                    for (int q = 0; q < C::BQ; ++q) acc[p][q] = fma(s, vb[q], acc[p][q]);
                }
            }
            double* y = sY + (size_t)lr * C::LDY;
#pragma unroll
            for (int p = 0; p < C::BP; ++p)
#pragma unroll
                for (int q = 0; q < C::BQ; ++q) y[(p0 + p) * KB + q0 + q] = acc[p][q];
        }
        __syncthreads();

        // ---- a_i rows: A_tile = Y_tile G^T (DMMA) or U_n rows
        if (a.kind == kTTMcTC) {
#pragma unroll
            for (int bi = 0; bi < C::ABW; ++bi) {
                const int b = warp + bi * C::WARPS;
                if (b < C::AB) {
                    const int mt = b / C::NT, nt = b - mt * C::NT;
                    const double* yrow = sY + (size_t)(mt * 8 + (lane >> 2)) * C::LDY + (lane & 3);
                    const double* gcol = sG + (size_t)(lane & 3) * C::GLD + nt * 8 + (lane >> 2);
                    double c0 = 0.0, c1 = 0.0;
#pragma unroll 5
                    for (int ks = 0; ks < C::L / 4; ++ks) dmma884(c0, c1, yrow[ks * 4], gcol[(size_t)ks * 4 * C::GLD]);
                    const int row = mt * 8 + (lane >> 2);
                    const int col = nt * 8 + 2 * (lane & 3);
                    sA[row * C::ALD + col] = c0;
                    sA[row * C::ALD + col + 1] = c1;
                }
            }
        } else {
            for (int q = tid; q < C::R * KN; q += C::THREADS) {
                int row = q / KN, r = q - row * KN;
                sA[row * C::ALD + r] = (row < nr && sLen[row] >= 0) ? a.un[(r0 + row) * KN + r] : 0.0;
            }
        }
        __syncthreads();
        // write A (short rows only), max|A|
        for (int q = tid; q < C::R * KN; q += C::THREADS) {
            int row = q / KN, r = q - row * KN;
            double v = sA[row * C::ALD + r];
            if (row < nr && sLen[row] >= 0) {
                if (a.A) a.A[(r0 + row) * KN + r] = v;
                mx = fmax(mx, fabs(v));
            } else {
                sA[row * C::ALD + r] = 0.0;  // long / absent rows contribute nothing
            }
        }
        __syncthreads();

        // ---- M += A_tile^T Y_tile (DMMA, C fragments in registers)
#pragma unroll
        for (int bi = 0; bi < C::MBW; ++bi) {
            const int b = warp + bi * C::WARPS;
            if (b < C::MB) {
                const int mt = b / C::NLT, nt = b - mt * C::NLT;
                const double* acol = sA + (size_t)(lane & 3) * C::ALD + mt * 8 + (lane >> 2);
                const double* ycol = sY + (size_t)(lane & 3) * C::LDY + nt * 8 + (lane >> 2);
#pragma unroll 4
                for (int ks = 0; ks < C::R / 4; ++ks)
                    dmma884(macc[bi][0], macc[bi][1], acol[(size_t)ks * 4 * C::ALD], ycol[(size_t)ks * 4 * C::LDY]);
            }
        }
        // ---- W += A^T A (DFMA)
#pragma unroll
        for (int wi = 0; wi < C::WQ; ++wi) {
            const int q = tid + wi * C::THREADS;
            if (q < KN * KN) {
                const int r1 = q / KN, r2 = q - r1 * KN;
                double s = wacc[wi];
                for (int row = 0; row < C::R; ++row) s = fma(sA[row * C::ALD + r1], sA[row * C::ALD + r2], s);
                wacc[wi] = s;
            }
        }
        __syncthreads();
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
#pragma unroll
    for (int wi = 0; wi < C::WQ; ++wi) {
        const int q = tid + wi * C::THREADS;
        if (q < KN * KN) a.wpart[(size_t)slot * KN * KN + q] = wacc[wi];
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
bool launch_fast3(const FastArgs& a, int grid, cudaStream_t s) {
    using C = Cfg<KA, KB, KN>;
    auto fn = k_pass_fast3<KA, KB, KN>;
    static bool attr = false;
    if (!attr) {
        HQ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes));
        attr = true;
    }
    fn<<<grid, C::THREADS, C::smem_bytes, s>>>(a);
    HQ_CHECK_LAUNCH();
    return true;
}

}  // namespace

int fast_grid(int ka, int kb, int kn) {
    (void)ka; (void)kb; (void)kn;
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
