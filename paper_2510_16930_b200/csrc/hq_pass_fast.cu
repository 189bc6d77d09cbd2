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

#include "hq_fast.cuh"

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
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
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
__device__ __forceinline__ void cp16(void* dst, const void* src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
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
    static constexpr int WARPS = 4;
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
    static constexpr int FW = KA + KB;           // staged doubles per record (two factor rows)
    static constexpr int CAP = (KB >= 16) ? 192 : 384;  // records per gather round
    static constexpr int MINB = (KB >= 16) ? 2 : 3;     // CTAs per SM the register budget targets
    static_assert(KA % TP == 0 && KB % TQ == 0, "rank split");
    static_assert(KA % 2 == 0 && KB % 2 == 0, "16-byte factor rows");
    static_assert(L % 4 == 0, "k-steps of 4");
    static_assert(R % 8 == 0, "m-tiles of 8 rows");
    // shared memory: gather buffer (aliased by the Y tile), records, A tile, row info
    static constexpr size_t GBUF = (size_t)CAP * FW > (size_t)R * LDY ? (size_t)CAP * FW : (size_t)R * LDY;
    static constexpr size_t smem_bytes =
        GBUF * 8 + (size_t)CAP * sizeof(Rec) + (size_t)R * ALD * 8 + 4 * R * sizeof(int) + 64;
};

template <int KA, int KB, int KN>
__global__ void __launch_bounds__(Cfg<KA, KB, KN>::THREADS, Cfg<KA, KB, KN>::MINB)
    k_pass_fast3(FastArgs a) {
    using C = Cfg<KA, KB, KN>;
    if (skip_kernel(a.st, a.run_if)) return;
    extern __shared__ __align__(16) double sm[];
    double* sF = sm;                                        // CAP x FW gathered factor rows
    double* sY = sm;                                        // R x LDY Kronecker rows (after the gather)
    Rec* sRec = reinterpret_cast<Rec*>(sm + C::GBUF);       // CAP records
    double* sA = reinterpret_cast<double*>(sRec + C::CAP);  // R x ALD a_i rows
    int* sLen = reinterpret_cast<int*>(sA + (size_t)C::R * C::ALD);
    int* sOff = sLen + C::R;   // virtual record offset of each row
    int* sPerm = sOff + C::R;  // lane slot -> row
    int* sTot = sPerm + C::R;  // [0] records in the tile
    __shared__ double red[C::WARPS];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t pol_stream = policy_evict_first();
    // with a persisting window on U_a its gathers carry no explicit hint and
    // U_b streams; without one both factors are asked to stay (evict_last)
    const uint64_t pol_a = a.l2_bytes ? policy_evict_normal() : policy_evict_last();
    const uint64_t pol_b = a.l2_bytes ? pol_stream : policy_evict_last();
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
    double wacc[C::WQ];
#pragma unroll
    for (int b = 0; b < C::WQ; ++b) wacc[b] = 0.0;
    double mx = 0.0;

    const double* __restrict__ Ua = a.ua;
    const double* __restrict__ Ub = a.ub;
    const double* __restrict__ gt = a.gt;

    // lane roles in the Kronecker phase
    const int rslot = warp * C::RPW + lane / C::TR;
    const int pb = (lane % C::TR) / C::TQ, qb = lane % C::TQ;
    const int p0 = pb * C::BP, q0 = qb * C::BQ;
    const int sub = lane % C::TR;

    __syncthreads();
    for (int64_t t = t0; t < t1; ++t) {
        const uint64_t r0 = a.rbase + (uint64_t)t * C::R;
        const int nr = (int)min((uint64_t)C::R, rend - r0);
        // 1. lengths (-1: long row, handled by the segmented path), offsets, ranking
        if (tid < C::R) {
            int len = 0;
            if (tid < nr) {
                const int64_t l = a.rowptr[r0 + tid + 1] - a.rowptr[r0 + tid];
                len = (l > kShortMax) ? -1 : (int)l;
            }
            sLen[tid] = len;
        }
        __syncthreads();
        if (tid < C::R) {
            const int me = max(sLen[tid], 0);
            int rank = 0, off = 0;
            for (int r = 0; r < C::R; ++r) {
                const int o = max(sLen[r], 0);
                rank += (o > me) || (o == me && r < tid);
                off += (r < tid) ? o : 0;
            }
            sPerm[rank] = tid;
            sOff[tid] = off;
            if (tid == C::R - 1) sTot[0] = off + me;
        }
        __syncthreads();
        const int total = sTot[0];
        const int lr = sPerm[rslot];
        const int len = max(sLen[lr], 0);
        const int voff = sOff[lr];
        const int64_t rbase = (len ? a.rowptr[r0 + lr] : 0) - voff;  // physical position = rbase + virtual

        double acc[C::BP][C::BQ];
#pragma unroll
        for (int p = 0; p < C::BP; ++p)
#pragma unroll
            for (int q = 0; q < C::BQ; ++q) acc[p][q] = 0.0;

        for (int cv = 0; cv < total; cv += C::CAP) {
            const int cn = min(C::CAP, total - cv);
            // 2a. records of virtual positions [cv, cv + cn): each row's lanes copy their row
            {
                const int lo = max(voff, cv), hi = min(voff + len, cv + cn);
                for (int v = lo + sub; v < hi; v += C::TR) {
                    const int64_t pz = rbase + v;
                    cp8(&sRec[v - cv].x, a.val + pz, pol_stream);
                    cp4(&sRec[v - cv].j, a.ia + pz, pol_stream);
                    cp4(&sRec[v - cv].k, a.ib + pz, pol_stream);
                }
            }
            cp_wait_all();
            __syncthreads();
            // 2b. both factor rows of every record (16-byte pieces)
            for (int e = tid; e < cn; e += C::THREADS) {
                const Rec r = sRec[e];
                const double* ua = Ua + (size_t)r.j * KA;
                const double* ub = Ub + (size_t)r.k * KB;
                double* dst = sF + (size_t)e * C::FW;
#pragma unroll
                for (int pc = 0; pc < KA / 2; ++pc) cp16(dst + 2 * pc, ua + 2 * pc, pol_a);
#pragma unroll
                for (int pc = 0; pc < KB / 2; ++pc) cp16(dst + KA + 2 * pc, ub + 2 * pc, pol_b);
            }
            cp_wait_all();
            __syncthreads();
            // 3. Kronecker rows from shared memory
            const int e0 = max(voff, cv) - cv, e1 = min(voff + len, cv + cn) - cv;
            for (int e = e0; e < e1; ++e) {
                const double x = sRec[e].x;
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
            __syncthreads();
        }
        // 4. Y tile (aliases the gather buffer)
        {
            double* y = sY + (size_t)lr * C::LDY;
#pragma unroll
            for (int p = 0; p < C::BP; ++p)
#pragma unroll
                for (int q = 0; q < C::BQ; ++q) y[blk_index<C::BP>(p0, p) * KB + blk_index<C::BQ>(q0, q)] = acc[p][q];
            if (C::LP > C::L && pb == 0 && qb == 0)
                for (int l = C::L; l < C::LP; ++l) y[l] = 0.0;
        }
        __syncthreads();
        if (a.kind == kTTMcTC) {
            // all of this warp's A blocks share one n-tile (b = warp + WARPS*bi, WARPS % NT == 0):
            // interleave the blocks and split the k-chain in two for ILP
            static_assert(C::WARPS % C::NT == 0, "warp -> n-tile mapping");
            const int nt = warp % C::NT;
            const int gcolidx = nt * 8 + (lane >> 2);
            const bool gvalid = gcolidx < KN;
            const double* gcol = gt + (size_t)(lane & 3) * KN + (gvalid ? gcolidx : 0);
            constexpr int KSN = C::L / 4;
            double g[KSN];
#pragma unroll
            for (int ks = 0; ks < KSN; ++ks) g[ks] = gvalid ? __ldg(gcol + (size_t)ks * 4 * KN) : 0.0;
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
                        dmma884(c[bi][ks & 1][0], c[bi][ks & 1][1], yv, g[ks]);
                    }
                }
#pragma unroll
            for (int bi = 0; bi < C::ABW; ++bi) {
                const int b = warp + bi * C::WARPS;
                if (b < C::AB) {
                    const int mt = b / C::NT;
                    const int row = mt * 8 + (lane >> 2);
                    const int col = nt * 8 + 2 * (lane & 3);
                    sA[row * C::ALD + col] = c[bi][0][0] + c[bi][1][0];
                    sA[row * C::ALD + col + 1] = c[bi][0][1] + c[bi][1][1];
                }
            }
        } else {
            for (int q = tid; q < C::R * KN; q += C::THREADS) {
                const int row = q / KN, r = q - row * KN;
                sA[row * C::ALD + r] = (row < nr && sLen[row] >= 0) ? a.un[(r0 + row) * KN + r] : 0.0;
            }
        }
        __syncthreads();
        for (int q = tid; q < C::R * KN; q += C::THREADS) {
            const int row = q / KN, r = q - row * KN;
            const double v = sA[row * C::ALD + r];
            if (row < nr && sLen[row] >= 0) {
                if (a.A) a.A[(r0 + row) * KN + r] = v;
                mx = fmax(mx, fabs(v));
            } else {
                sA[row * C::ALD + r] = 0.0;  // long / absent rows contribute nothing
            }
        }
        __syncthreads();
        // 5. M += A_tile^T Y_tile (DMMA), W += A^T A (DFMA)
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
void launch_fast3(const FastArgs& a, int grid, cudaStream_t s) {
    using C = Cfg<KA, KB, KN>;
    auto fn = k_pass_fast3<KA, KB, KN>;
    static bool attr = false;
    if (!attr) {
        HQ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::smem_bytes));
        attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = C::smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr_l2[1];
    if (a.l2_bytes) {
        attr_l2[0].id = cudaLaunchAttributeAccessPolicyWindow;
        attr_l2[0].val.accessPolicyWindow.base_ptr = const_cast<double*>(a.ua);
        attr_l2[0].val.accessPolicyWindow.num_bytes = a.l2_bytes;
        attr_l2[0].val.accessPolicyWindow.hitRatio = a.l2_hit;
        attr_l2[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr_l2[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.attrs = attr_l2;
        cfg.numAttrs = 1;
    }
    HQ_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
}

template <int KA, int KB, int KN>
int grid_fast3() {
    return num_sms() * Cfg<KA, KB, KN>::MINB;
}

}  // namespace

size_t l2_persist_budget() {
    static size_t budget = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess || v <= 0) return (size_t)0;
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)v) != cudaSuccess) {
            cudaGetLastError();
            return (size_t)0;
        }
        return (size_t)v;
    }();
    return budget;
}

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
