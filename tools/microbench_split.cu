// Two-table random gathers of K = 10 factor rows (80 B) vs a split layout:
// columns 0..7 in a 64-byte-row table (one DRAM granule per row) and columns
// 8..9 in a 16-byte-row table small enough to stay in L2 (evict_last).  Same
// cp.async piece count; fewer DRAM bytes per gathered row.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ void cp16h(void* d, const void* s, uint64_t p) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" :: "r"(sa(d)), "l"(s), "l"(p));
}
// mode 0: A, B plain 80 B rows (evict_last both); mode 1: split P (64 B, evict_first) + Q (16 B, evict_last)
__global__ void bench(const double* A, const double* B, const double* PA, const double* QA, const double* PB,
                      const double* QB, const uint2* idx, long n, int mode, double* out) {
    extern __shared__ __align__(128) double sm[];
    const int CAP = 384;
    __shared__ uint2 sidx[384];
    const uint64_t pl = pol_last(), pf = pol_first();
    long per = (n + gridDim.x - 1) / gridDim.x; long b = per * blockIdx.x, e = min(n, b + per);
    double acc = 0;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int RPI = nt / 10;
    for (long r0 = b; r0 < e; r0 += CAP) {
        int cn = (int)min((long)CAP, e - r0);
        for (int t = tid; t < cn; t += nt) sidx[t] = idx[r0 + t];
        __syncthreads();
        if (tid < RPI * 10) {
            const int pc = tid % 10;
            for (int r = tid / 10; r < cn; r += RPI) {
                double* d = sm + r * 22 + (pc < 5 ? 2 * pc : 10 + 2 * (pc - 5));
                const uint32_t j = pc < 5 ? sidx[r].x : sidx[r].y;
                const int q = pc % 5;
                if (mode == 0) {
                    cp16h(d, (pc < 5 ? A : B) + (size_t)j * 10 + 2 * q, pl);
                } else {
                    if (q < 4) cp16h(d, (pc < 5 ? PA : PB) + (size_t)j * 8 + 2 * q, pf);
                    else cp16h(d, (pc < 5 ? QA : QB) + (size_t)j * 2, pl);
                }
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        for (int t = tid; t < cn; t += nt) acc += sm[t * 22] + sm[t * 22 + 19];
        __syncthreads();
    }
    if (acc == 1234.5) out[0] = acc;
}
int main() {
    const long rows = 1000000, n = 10000000;
    double *A, *B, *PA, *QA, *PB, *QB, *out; uint2* idx;
    CK(cudaMalloc(&A, rows * 80)); CK(cudaMalloc(&B, rows * 80)); CK(cudaMalloc(&PA, rows * 64)); CK(cudaMalloc(&QA, rows * 16));
    CK(cudaMalloc(&PB, rows * 64)); CK(cudaMalloc(&QB, rows * 16)); CK(cudaMalloc(&out, 4096)); CK(cudaMalloc(&idx, n * 8));
    cudaMemset(A, 0, rows * 80); cudaMemset(B, 0, rows * 80); cudaMemset(PA, 0, rows * 64); cudaMemset(PB, 0, rows * 64);
    cudaMemset(QA, 0, rows * 16); cudaMemset(QB, 0, rows * 16);
    std::vector<uint2> hi(n); uint64_t s = 88172645463325252ull;
    for (long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; hi[i].x = s % rows; s ^= s << 13; s ^= s >> 7; s ^= s << 17; hi[i].y = s % rows; }
    CK(cudaMemcpy(idx, hi.data(), n * 8, cudaMemcpyHostToDevice));
    int smem = 384 * 22 * 8; CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode : {0, 1}) for (int bps : {2, 3}) for (int thr : {128, 256}) {
        bench<<<148 * bps, thr, smem>>>(A, B, PA, QA, PB, QB, idx, n, mode, out);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) bench<<<148 * bps, thr, smem>>>(A, B, PA, QA, PB, QB, idx, n, mode, out);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
        printf("mode %d (%s) blocks/SM %d threads %d: %.1f us  %.1f G rows/s\n", mode, mode ? "split 64+16" : "80 B rows",
               bps, thr, ms * 1e3, 2.0 * n / ms / 1e6);
    }
    return 0;
}
