// Hybrid factor-row gather: table A rows through TMA tile::gather4 (one elected
// thread, TMA unit) and table B rows through cp.async 16-byte pieces (LSU),
// concurrently, vs cp.async for both -- does splitting the two gathers over the
// two copy engines beat the LSU's piece rate?
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
__device__ __forceinline__ void cp16(void* d, const void* s) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa(d)), "l"(s));
}
// mode 0: both tables cp.async (piece-major, fixed slot per thread); mode 1: A by gather4, B by cp.async
__global__ void bench(const __grid_constant__ CUtensorMap ta, const double* A, const double* B, const uint2* idx, long n,
                      int mode, double* out) {
    extern __shared__ __align__(128) double sm[];
    const int CAP = 384;
    double* fa = sm;                       // gather4 blocks: 4 rows x 80 B padded to 384 B
    double* fb = sm + (CAP / 4) * 48;      // cp.async rows, 80 B each (10 doubles) + pad
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint2 sidx[384];
    const uint32_t mb = sa(&mbar);
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb)); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    long per = (n + gridDim.x - 1) / gridDim.x; long b = per * blockIdx.x, e = min(n, b + per);
    double acc = 0; uint32_t ph = 0;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (long r0 = b; r0 < e; r0 += CAP) {
        int cn = (int)min((long)CAP, e - r0); int cn4 = cn & ~3;
        for (int t = tid; t < cn; t += nt) sidx[t] = idx[r0 + t];
        __syncthreads();
        if (mode == 1) {
            if (tid == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(cn4 * 80));
                for (int q = 0; q < cn4; q += 4) {
                    uint2 i0 = sidx[q], i1 = sidx[q + 1], i2 = sidx[q + 2], i3 = sidx[q + 3];
                    g4(sa(fa + (q / 4) * 48), &ta, i0.x, i1.x, i2.x, i3.x, mb);
                }
            }
            // B rows: 5 pieces per row, fixed slot per thread (first 125 threads of 128)
            const int RPI = nt / 5;
            if (tid < RPI * 5) {
                const int pc = tid % 5;
                for (int r = tid / 5; r < cn4; r += RPI) cp16(fb + r * 12 + 2 * pc, B + (size_t)sidx[r].y * 10 + 2 * pc);
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
            mwait(mb, ph); ph ^= 1;
        } else {
            const int RPI = nt / 10;
            if (tid < RPI * 10) {
                const int pc = tid % 10;
                for (int r = tid / 10; r < cn4; r += RPI) {
                    if (pc < 5) cp16(fa + r * 12 + 2 * pc, A + (size_t)sidx[r].x * 10 + 2 * pc);
                    else cp16(fb + r * 12 + 2 * (pc - 5), B + (size_t)sidx[r].y * 10 + 2 * (pc - 5));
                }
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        for (int t = tid; t < cn4; t += nt) acc += fa[(t / 4) * 48 + (t % 4) * 10] + fb[t * 12 + 9];
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
    CUtensorMap ta;
    cuuint64_t gd[2] = {10, (cuuint64_t)rows}; cuuint64_t gs[1] = {80}; cuuint32_t bd[2] = {10, 1}; cuuint32_t es[2] = {1, 1};
    if (enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) { printf("encode failed\n"); return 1; }
    std::vector<uint2> hi(n); uint64_t s = 88172645463325252ull;
    for (long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; hi[i].x = s % rows; s ^= s << 13; s ^= s >> 7; s ^= s << 17; hi[i].y = s % rows; }
    CK(cudaMemcpy(idx, hi.data(), n * 8, cudaMemcpyHostToDevice));
    int smem = (384 / 4) * 48 * 8 + 384 * 12 * 8; CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode : {0, 1}) for (int bps : {2, 3, 4}) for (int thr : {128, 256}) {
        bench<<<148 * bps, thr, smem>>>(ta, A, B, idx, n, mode, out);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) bench<<<148 * bps, thr, smem>>>(ta, A, B, idx, n, mode, out);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
        printf("mode %d (%s) blocks/SM %d threads %d: %.1f us  %.1f G rows/s\n", mode, mode ? "A gather4 + B cp.async" : "both cp.async",
               bps, thr, ms * 1e3, 2.0 * n / ms / 1e6);
    }
    return 0;
}
