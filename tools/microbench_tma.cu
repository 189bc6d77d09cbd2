// TMA tile::gather4 for factor-row gathers: correctness of the smem layout and
// throughput (one elected thread per CTA issues all gathers of a batch).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void g4(uint32_t dst, const CUtensorMap* m, int r0, int r1, int r2, int r3, uint32_t mb) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 :: "r"(dst), "l"(m), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(mb) : "memory");
}
__device__ __forceinline__ void mwait(uint32_t mb, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" :: "r"(mb), "r"(ph));
}
__global__ void check(const __grid_constant__ CUtensorMap tm, double* out) {
    __shared__ __align__(128) double buf[4 * 10];
    __shared__ __align__(8) uint64_t mbar;
    uint32_t mb = sa(&mbar);
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb)); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(320));
        g4(sa(buf), &tm, 5, 999999, 17, 123456, mb);
    }
    mwait(mb, 0);
    for (int i = threadIdx.x; i < 40; i += blockDim.x) out[i] = buf[i];
}
// CAP records per round, both tables; thread 0 issues CAP/4 gather4 per table
__global__ void bench(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, const uint2* idx, long n, double* out) {
    extern __shared__ __align__(128) double sm[];
    const int CAP = 384;
    double* fa = sm; double* fb = sm + (CAP / 4) * 48;  // 4-row blocks padded to 384 B (128 B aligned)
    __shared__ __align__(8) uint64_t mbar;
    uint32_t mb = sa(&mbar);
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb)); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    long per = (n + gridDim.x - 1) / gridDim.x; long b = per * blockIdx.x, e = min(n, b + per);
    double acc = 0; uint32_t ph = 0;
    __shared__ uint2 sidx[384];
    for (long r0 = b; r0 < e; r0 += CAP) {
        int cn = (int)min((long)CAP, e - r0); int cn4 = cn & ~3;
        for (int t = threadIdx.x; t < cn; t += blockDim.x) sidx[t] = idx[r0 + t];
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(cn4 * 160));
            for (int q = 0; q < cn4; q += 4) {
                uint2 i0 = sidx[q], i1 = sidx[q + 1], i2 = sidx[q + 2], i3 = sidx[q + 3];
                g4(sa(fa + (q / 4) * 48), &ta, i0.x, i1.x, i2.x, i3.x, mb);
                g4(sa(fb + (q / 4) * 48), &tb, i0.y, i1.y, i2.y, i3.y, mb);
            }
        }
        mwait(mb, ph); ph ^= 1;
        for (int t = threadIdx.x; t < cn4; t += blockDim.x) acc += fa[(t / 4) * 48 + (t % 4) * 10] + fb[(t / 4) * 48 + (t % 4) * 10 + 9];
        __syncthreads();
    }
    if (acc == 1234.5) out[0] = acc;
}
int main() {
    const long rows = 1000000, n = 10000000;
    std::vector<double> h(rows * 10);
    for (long r = 0; r < rows; ++r) for (int c = 0; c < 10; ++c) h[r * 10 + c] = r * 100.0 + c;
    double *A, *B, *out; uint2* idx;
    CK(cudaMalloc(&A, rows * 80)); CK(cudaMalloc(&B, rows * 80)); CK(cudaMalloc(&out, 4096)); CK(cudaMalloc(&idx, n * 8));
    CK(cudaMemcpy(A, h.data(), rows * 80, cudaMemcpyHostToDevice)); CK(cudaMemcpy(B, h.data(), rows * 80, cudaMemcpyHostToDevice));
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    for (int boxrows : {1}) {
        CUtensorMap ta, tb;
        cuuint64_t gd[2] = {10, (cuuint64_t)rows}; cuuint64_t gs[1] = {80}; cuuint32_t bd[2] = {10, (cuuint32_t)boxrows}; cuuint32_t es[2] = {1, 1};
        CUresult ra = enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        CUresult rb = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, B, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("boxrows %d encode %d %d\n", boxrows, (int)ra, (int)rb);
        if (ra || rb) continue;
        CK(cudaMemset(out, 0, 4096));
        check<<<1, 64>>>(ta, out);
        cudaError_t err = cudaDeviceSynchronize();
        if (err != cudaSuccess) { printf("check failed: %s\n", cudaGetErrorString(err)); return 1; }
        double ho[40]; CK(cudaMemcpy(ho, out, 320, cudaMemcpyDeviceToHost));
        printf("  rows got: %.0f %.0f %.0f %.0f | last of row1: %.0f\n", ho[0], ho[10], ho[20], ho[30], ho[19]);
        if (boxrows != 1) continue;
        std::vector<uint2> hi(n); uint64_t s = 88172645463325252ull;
        for (long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; hi[i].x = s % rows; s ^= s << 13; s ^= s >> 7; s ^= s << 17; hi[i].y = s % rows; }
        CK(cudaMemcpy(idx, hi.data(), n * 8, cudaMemcpyHostToDevice));
        int smem = 2 * 96 * 48 * 8; CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int bps : {2, 3, 4}) for (int thr : {32, 128}) {
            bench<<<148 * bps, thr, smem>>>(ta, tb, idx, n, out);
            cudaEventRecord(e0);
            for (int r = 0; r < 3; ++r) bench<<<148 * bps, thr, smem>>>(ta, tb, idx, n, out);
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
            printf("  gather4 blocks/SM %d threads %d: %.1f us  %.1f G rows/s\n", bps, thr, ms * 1e3, 2.0 * n / ms / 1e6);
        }
    }
    return 0;
}
