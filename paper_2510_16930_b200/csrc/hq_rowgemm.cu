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
// Each warp walks groups of 8 rows: A fragments come straight from HBM, the
// X = A T product and the X^T Y accumulation are DMMA m8n8k4 (f64), X is
// re-laid out through a per-warp shared-memory tile.  The K x K accumulators
// stay in registers; warps are combined in fixed order into one partial slot
// per CTA (deterministic).
#include <algorithm>

#include "hq_dense.cuh"

namespace hq {

namespace {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

constexpr int kRgWarps = 8;

template <int K>
struct RG {
    static constexpr int NT = (K + 7) / 8;  // 8-wide tiles of the K dimension
    static constexpr int KP = NT * 8;
    static constexpr int KS = (K + 3) / 4;  // k-steps of X = A T
    static constexpr int LD = KP + 4;       // smem row stride (= 4 mod 8 doubles: fragment reads conflict-free)
};

template <int K>
__global__ void __launch_bounds__(kRgWarps * 32)
    k_rowgemm(const double* A, uint64_t rows, const double* __restrict__ T, double* out,
              const double* __restrict__ other, double* __restrict__ part, double* __restrict__ maxpart,
              const DevStatus* st, int run_if) {
    using C = RG<K>;
    if (skip_kernel(st, run_if)) return;
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
            if (k < K && n < K) v = T ? T[k * K + n] : (k == n ? 1.0 : 0.0);
            tf[ks][nt] = v;
        }
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
            for (int ks = 0; ks < C::KS; ++ks) dmma884(c0, c1, a[ks], tf[ks][nt]);
            const int col = 8 * nt + 2 * tig;
            sx[gid * C::LD + col] = c0;
            sx[gid * C::LD + col + 1] = c1;
        }
        __syncwarp();
        if (out) {
#pragma unroll
            for (int i = 0; i < OQ; ++i) {
                const int q = lane + 32 * i;
                const uint64_t e = g * 8 * K + q;
                if (q < 8 * K && e < rows * K) {
                    const int r = q / K, cc = q - r * K;
                    out[e] = sx[r * C::LD + cc];
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

template <int K>
void launch_rg(const double* A, uint64_t rows, const double* T, double* out, const double* other, double* part,
               double* maxpart, const DevStatus* st, int run_if, cudaStream_t s) {
    k_rowgemm<K><<<dense_slots(), kRgWarps * 32, 0, s>>>(A, rows, T, out, other, part, maxpart, st, run_if);  // dense_slots() = 4 CTAs/SM
    HQ_CHECK_LAUNCH();
}

}  // namespace

bool rowgemm_supported(int K) { return K >= 1 && K <= 32; }

void launch_rowgemm(int K, const double* A, uint64_t rows, const double* T, double* out, const double* other,
                    double* part, double* maxpart, const DevStatus* st, int run_if, cudaStream_t s) {
    switch (K) {
#define HQ_K(KK) case KK: launch_rg<KK>(A, rows, T, out, other, part, maxpart, st, run_if, s); return;
        HQ_K(1) HQ_K(2) HQ_K(3) HQ_K(4) HQ_K(5) HQ_K(6) HQ_K(7) HQ_K(8) HQ_K(9) HQ_K(10) HQ_K(11) HQ_K(12)
        HQ_K(13) HQ_K(14) HQ_K(15) HQ_K(16) HQ_K(17) HQ_K(18) HQ_K(19) HQ_K(20) HQ_K(21) HQ_K(22) HQ_K(23)
        HQ_K(24) HQ_K(25) HQ_K(26) HQ_K(27) HQ_K(28) HQ_K(29) HQ_K(30) HQ_K(31) HQ_K(32)
#undef HQ_K
        default: fail(HQ_ERR_CAPACITY, "rank above 32");
    }
}

}  // namespace hq
