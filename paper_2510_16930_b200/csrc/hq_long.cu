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

#include "hq_long.cuh"

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
    static constexpr int LS = K2 ? K0 * K1 : K0;  // S width
    static constexpr int KL = K2 ? K2 : K1;       // V width (last other mode)
    static constexpr int L = LS * KL;
    static constexpr int MT = (LS + 7) / 8, NTL = (KL + 7) / 8;
    static constexpr int RW = K0 + K1 + K2;        // staged factor doubles per nonzero
    // + x; row stride = 4 mod 8 doubles: the 4 nonzeros of a k-step land on disjoint banks
    static constexpr int FW = (RW + 4) / 8 * 8 + 4;
    static constexpr int CH = 128;                  // nonzeros per chunk
    static constexpr int WARPS = 4, THREADS = 128;
    static constexpr size_t smem = 2 * (size_t)CH * FW * 8 + (size_t)WARPS * MT * NTL * 64 * 8;
    static_assert(K0 % 2 == 0 && K1 % 2 == 0 && K2 % 2 == 0, "16-byte factor rows");
};

template <int K0, int K1, int K2>
__global__ void __launch_bounds__(128) k_longseg_mma(LongArgs a) {
    using S = LS_<K0, K1, K2>;
    if (skip_kernel(a.st, a.run_if)) return;
    extern __shared__ __align__(16) double sm[];
    double* red = sm + 2 * (size_t)S::CH * S::FW;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const uint64_t G = gridDim.x, c = blockIdx.x;
    const uint64_t sb = a.nseg * c / G, se = a.nseg * (c + 1) / G;
    const uint64_t rend = a.rbase + a.rows;
    constexpr int P0 = K0 / 2, P1 = K1 / 2, P2 = K2 / 2, PP = P0 + P1 + P2;

    // stage nonzeros [z0, z0 + n) into buffer b: factor rows piece-major, then x
    auto stage = [&](int b, int64_t z0, int n) {
        double* dst = sm + (size_t)b * S::CH * S::FW;
        for (int q = tid; q < n * PP; q += S::THREADS) {
            const int e = q / PP, pc = q - e * PP;
            const int64_t z = z0 + e;
            const double* src;
            int off;
            if (pc < P0) {
                src = a.u0 + (size_t)a.i0[z] * K0 + 2 * pc;
                off = 2 * pc;
            } else if (pc < P0 + P1) {
                src = a.u1 + (size_t)a.i1[z] * K1 + 2 * (pc - P0);
                off = K0 + 2 * (pc - P0);
            } else {
                src = a.u2 + (size_t)a.i2[z] * K2 + 2 * (pc - P0 - P1);
                off = K0 + K1 + 2 * (pc - P0 - P1);
            }
            cpa16(dst + (size_t)e * S::FW + off, src);
        }
        for (int e = tid; e < n; e += S::THREADS) cpa8(dst + (size_t)e * S::FW + S::RW, a.val + z0 + e);
        cpa_commit();
    };

    for (uint64_t sg = sb; sg < se; ++sg) {
        const uint32_t row = a.long_ids[a.seg_row[sg]];
        if (row < a.rbase || row >= rend) continue;  // another rank's row
        const int64_t zs = a.seg_begin[sg];
        const int64_t ze = min(zs + (int64_t)kSegLen, a.rowptr[row + 1]);
        const int nch = (int)((ze - zs + S::CH - 1) / S::CH);
        double acc[S::MT][S::NTL][2];
#pragma unroll
        for (int i = 0; i < S::MT; ++i)
#pragma unroll
            for (int j = 0; j < S::NTL; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        __syncthreads();  // buffers free (previous segment done)
        stage(0, zs, (int)min((int64_t)S::CH, ze - zs));
        for (int ch = 0; ch < nch; ++ch) {
            const int64_t z0 = zs + (int64_t)ch * S::CH;
            const int n = (int)min((int64_t)S::CH, ze - z0);
            if (ch + 1 < nch) {
                stage((ch + 1) & 1, z0 + S::CH, (int)min((int64_t)S::CH, ze - z0 - S::CH));
                cpa_wait<1>();
            } else {
                cpa_wait<0>();
            }
            __syncthreads();
            const double* f = sm + (size_t)(ch & 1) * S::CH * S::FW;
            const int ks_n = (n + 3) / 4;
            for (int ks = warp; ks < ks_n; ks += S::WARPS) {
                const int e = ks * 4 + tig;
                const bool ev = e < n;
                const double* fe = f + (size_t)e * S::FW;
                const double x = ev ? fe[S::RW] : 0.0;
                double bv[S::NTL];
#pragma unroll
                for (int nt = 0; nt < S::NTL; ++nt) {
                    const int col = nt * 8 + gid;
                    bv[nt] = (ev && col < S::KL) ? fe[(K2 ? K0 + K1 : K0) + col] : 0.0;
                }
#pragma unroll
                for (int mt = 0; mt < S::MT; ++mt) {
                    const int col = mt * 8 + gid;
                    double av = 0.0;
                    if (ev && col < S::LS) {
                        if constexpr (K2 != 0)
                            av = x * fe[col / K1] * fe[K0 + col % K1];
                        else
                            av = x * fe[col];
                    }
#pragma unroll
                    for (int nt = 0; nt < S::NTL; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], av, bv[nt]);
                }
            }
            __syncthreads();  // buffer ch&1 is refilled at ch+2
        }
        // fixed-order sum of the four warps' fragments -> ypart[sg]
        double* rw = red + (size_t)warp * S::MT * S::NTL * 64;
#pragma unroll
        for (int mt = 0; mt < S::MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < S::NTL; ++nt) {
                rw[(mt * S::NTL + nt) * 64 + gid * 8 + 2 * tig] = acc[mt][nt][0];
                rw[(mt * S::NTL + nt) * 64 + gid * 8 + 2 * tig + 1] = acc[mt][nt][1];
            }
        __syncthreads();
        for (int q = tid; q < S::L; q += S::THREADS) {
            const int sidx = q / S::KL, t = q - sidx * S::KL;  // Kronecker column q = s * KL + t
            const int mt = sidx / 8, nt = t / 8, o = (sidx % 8) * 8 + (t % 8);
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < S::WARPS; ++w) v += red[(size_t)w * S::MT * S::NTL * 64 + (mt * S::NTL + nt) * 64 + o];
            a.ypart[sg * S::L + q] = v;
        }
    }
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
    static constexpr size_t smem = (size_t)RT * LDY * 8 + (size_t)RT * ALD * 8 + 64;
    static_assert(L % 4 == 0, "k-steps");
};

template <int L, int KN>
__global__ void __launch_bounds__(128) k_longfix_mma(LongArgs a) {
    using F = LF_<L, KN>;
    if (skip_kernel(a.st, a.run_if)) return;
    extern __shared__ __align__(16) double sm[];
    double* sY = sm;
    double* sA = sm + (size_t)F::RT * F::LDY;
    __shared__ double red[F::WARPS];
    __shared__ uint32_t srow[F::RT];
    __shared__ int sval[F::RT];
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
            int v = 0;
            if (tid < nr) {
                row = a.long_ids[t0 + tid];
                v = (row >= a.rbase && row < rend);
            }
            srow[tid] = row;
            sval[tid] = v;
        }
        __syncthreads();
        // Y rows: segment partials summed in segment order
        for (int q = tid; q < F::RT * L; q += F::THREADS) {
            const int r = q / L, l = q - r * L;
            double y = 0.0;
            if (r < nr && sval[r]) {
                const int64_t s0 = a.long_segptr[t0 + r], s1 = a.long_segptr[t0 + r + 1];
                for (int64_t sg = s0; sg < s1; ++sg) y += a.ypart[sg * L + l];
            }
            sY[(size_t)r * F::LDY + l] = y;
        }
        __syncthreads();
        if (a.kind == kTTMcTC) {
#pragma unroll
            for (int bi = 0; bi < F::ABW; ++bi) {
                const int b = warp + bi * F::WARPS;
                if (b < F::AB) {
                    const int mt = b / F::NT, nt = b - mt * F::NT;
                    const int gcol = nt * 8 + gid;
                    double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
                    for (int ks = 0; ks < L / 4; ks += 2) {
                        const double y0 = sY[(size_t)(mt * 8 + gid) * F::LDY + ks * 4 + tig];
                        const double g0 = gcol < KN ? __ldg(a.gt + (size_t)(ks * 4 + tig) * KN + gcol) : 0.0;
                        dmma(c0, c1, y0, g0);
                        if (ks + 1 < L / 4) {
                            const double y1 = sY[(size_t)(mt * 8 + gid) * F::LDY + (ks + 1) * 4 + tig];
                            const double g1 = gcol < KN ? __ldg(a.gt + (size_t)((ks + 1) * 4 + tig) * KN + gcol) : 0.0;
                            dmma(d0, d1, y1, g1);
                        }
                    }
                    const int row = mt * 8 + gid, col = nt * 8 + 2 * tig;
                    sA[row * F::ALD + col] = c0 + d0;
                    sA[row * F::ALD + col + 1] = c1 + d1;
                }
            }
        } else {
            for (int q = tid; q < F::RT * KN; q += F::THREADS) {
                const int r = q / KN, k = q - r * KN;
                sA[r * F::ALD + k] = (r < nr && sval[r]) ? a.un[(size_t)srow[r] * KN + k] : 0.0;
            }
        }
        __syncthreads();
        for (int q = tid; q < F::RT * KN; q += F::THREADS) {
            const int r = q / KN, k = q - r * KN;
            if (r < nr && sval[r]) {
                const double v = sA[r * F::ALD + k];
                if (a.A) a.A[(size_t)srow[r] * KN + k] = v;
                mx = fmax(mx, fabs(v));
            } else {
                sA[r * F::ALD + k] = 0.0;
            }
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
    static int per_sm = 0;
    if (!per_sm) {
        set_smem_attr((const void*)k_longseg_mma<K0, K1, K2>, S::smem);
        set_smem_attr((const void*)k_longfix_mma<S::L, KN>, F::smem);
        HQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_longseg_mma<K0, K1, K2>, S::THREADS,
                                                              S::smem));
        per_sm = std::max(per_sm, 1);
    }
    const int seg_grid = (int)std::min<uint64_t>(a.nseg, (uint64_t)num_sms() * per_sm);
    k_longseg_mma<K0, K1, K2><<<seg_grid, S::THREADS, S::smem, s>>>(a);
    HQ_CHECK_LAUNCH();
    k_longfix_mma<S::L, KN><<<fix_grid, F::THREADS, F::smem, s>>>(a);
    HQ_CHECK_LAUNCH();
}

}  // namespace

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
