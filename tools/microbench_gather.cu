// Two-table random row gather (the fused pass's memory pattern): per record
// one 80-byte row from table A and one from table B, cp.async into shared
// memory in rounds of 384 records per CTA.  Variants of L2 policy:
//   0 plain  1 evict_last both  2 window(A persisting)+plain  3 window(A)+B evict_first
//   4 ld.global (registers) plain, 8 records in flight per thread
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ void cp16h(void* d, const void* s, uint64_t p) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" :: "r"((uint32_t)__cvta_generic_to_shared(d)), "l"(s), "l"(p));
}
__device__ __forceinline__ void cp16(void* d, const void* s) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"((uint32_t)__cvta_generic_to_shared(d)), "l"(s));
}
__global__ void gather(const double* A, const double* B, const uint2* idx, long n, int mode, double* out) {
    extern __shared__ double sm[];
    const int CAP = 384;
    uint64_t pl = pol_last(), pf = pol_first();
    long per = (n + gridDim.x - 1) / gridDim.x;
    long b = per * blockIdx.x, e = min(n, b + per);
    double acc = 0;
    for (long r0 = b; r0 < e; r0 += CAP) {
        int cn = (int)min((long)CAP, e - r0);
        if (mode >= 4) {  // piece-major: consecutive lanes copy consecutive 16-byte pieces of one row
            for (int q = threadIdx.x; q < cn * 10; q += blockDim.x) {
                int t = q / 10, pc = q - t * 10;
                uint2 jk = idx[r0 + t];
                const double* src = pc < 5 ? A + (size_t)jk.x * 10 + 2 * pc : B + (size_t)jk.y * 10 + 2 * (pc - 5);
                if (mode == 4) cp16(sm + (size_t)t * 20 + 2 * pc, src);
                else cp16h(sm + (size_t)t * 20 + 2 * pc, src, pl);
            }
        } else
        for (int t = threadIdx.x; t < cn; t += blockDim.x) {
            uint2 jk = idx[r0 + t];
            const double* a = A + (size_t)jk.x * 10; const double* bb = B + (size_t)jk.y * 10;
            double* d = sm + (size_t)t * 20;
            for (int p = 0; p < 5; ++p) {
                if (mode == 0 || mode == 2) { cp16(d + 2 * p, a + 2 * p); cp16(d + 10 + 2 * p, bb + 2 * p); }
                else if (mode == 1) { cp16h(d + 2 * p, a + 2 * p, pl); cp16h(d + 10 + 2 * p, bb + 2 * p, pl); }
                else { cp16(d + 2 * p, a + 2 * p); cp16h(d + 10 + 2 * p, bb + 2 * p, pf); }
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        for (int t = threadIdx.x; t < cn; t += blockDim.x) acc += sm[t * 20] + sm[t * 20 + 19];
        __syncthreads();
    }
    if (acc == 1234.5) out[0] = acc;
}
int main() {
    const long rows = 1000000, n = 10000000;
    double *A, *B, *out; uint2* idx;
    CK(cudaMalloc(&A, rows * 80)); CK(cudaMalloc(&B, rows * 80)); CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&idx, n * 8));
    cudaMemset(A, 0, rows * 80); cudaMemset(B, 0, rows * 80);
    std::vector<uint2> h(n); uint64_t s = 88172645463325252ull;
    for (long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i].x = s % rows; s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i].y = s % rows; }
    CK(cudaMemcpy(idx, h.data(), n * 8, cudaMemcpyHostToDevice));
    int maxp = 0; cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp));
    int smem = 384 * 20 * 8;
    CK(cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaStream_t st; cudaStreamCreate(&st);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (float hr : {0.9f}) for (int blocksPerSM : {3, 6}) for (int threads : {128, 256}) for (int mode = 0; mode < 6; ++mode) {
        if (mode == 2 || mode == 3) continue;
        cudaStreamAttrValue v{};
        if (mode >= 2) { v.accessPolicyWindow.base_ptr = A; v.accessPolicyWindow.num_bytes = rows * 80; v.accessPolicyWindow.hitRatio = hr;
            v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting; v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming; }
        CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v));
        cudaCtxResetPersistingL2Cache();
        int grid = 148 * blocksPerSM;
        for (int w = 0; w < 2; ++w) gather<<<grid, threads, smem, st>>>(A, B, idx, n, mode, out);
        cudaEventRecord(e0, st);
        for (int w = 0; w < 3; ++w) gather<<<grid, threads, smem, st>>>(A, B, idx, n, mode, out);
        cudaEventRecord(e1, st); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
        printf("hitRatio %.2f blocks/SM %d threads %d mode %d: %.1f us  %.1f G rows/s\n", hr, blocksPerSM, threads, mode, ms * 1e3, 2.0 * n / ms / 1e6);
    }
    return 0;
}
