// What does an L2 miss on a random factor-row gather cost in DRAM bytes?  One- and two-table random gathers
// at cudaLimitMaxL2FetchGranularity = 32 / 64 / 128 (argv[1]), table size argv[2] rows (default 10^6):
//   0: two tables, 80 B rows                    1: two tables, 64 B heads only (64-byte aligned rows)
//   2: two tables, 16 B tails only (2 x 16 MB)   3: one table, 80 B rows (both gathers from table A)
//   4: two tables, 32 B rows (one sector)
// -DPF=64/128/256 adds the L2 prefetch-size qualifier to the copies.
// Run under ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct for the bytes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_fetch tools/microbench_fetch.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
#ifndef PF
#define PF 0
#endif
__device__ __forceinline__ void cp16(void* d, const void* s) {
#if PF == 64
    asm volatile("cp.async.cg.shared.global.L2::64B [%0], [%1], 16;" :: "r"(sa(d)), "l"(s));
#elif PF == 128
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" :: "r"(sa(d)), "l"(s));
#elif PF == 256
    asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" :: "r"(sa(d)), "l"(s));
#else
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa(d)), "l"(s));
#endif
}
template <int MODE>
__global__ void __launch_bounds__(128) bench(const double* A, const double* B, const uint2* idx, long n, double* out) {
    extern __shared__ __align__(128) double sm[];
    constexpr int CAP = 352;
    constexpr int PIECES = (MODE == 0 || MODE == 3) ? 5 : (MODE == 1 ? 4 : (MODE == 2 ? 1 : 2));  // per row
    constexpr int PITCH = (MODE == 0 || MODE == 3) ? 10 : (MODE == 1 ? 8 : (MODE == 2 ? 2 : 4));  // doubles
    __shared__ uint2 sidx[CAP];
    long per = (n + gridDim.x - 1) / gridDim.x; long b = per * blockIdx.x, e = min(n, b + per);
    double acc = 0;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (long r0 = b; r0 < e; r0 += CAP) {
        int cn = (int)min((long)CAP, e - r0);
        for (int q = tid; q < cn; q += nt) sidx[q] = idx[r0 + q];
        __syncthreads();
        for (int s = tid; s < cn * 2 * PIECES; s += nt) {
            const int r = s / (2 * PIECES), pc = s - r * 2 * PIECES;
            double* d = sm + r * 20 + 2 * pc;
            const bool first = pc < PIECES;
            const uint32_t j = first ? sidx[r].x : sidx[r].y;
            const int q = first ? pc : pc - PIECES;
            const double* t = (first || MODE == 3) ? A : B;
            cp16(d, t + (size_t)j * PITCH + 2 * q);
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        for (int q = tid; q < cn; q += nt) acc += sm[q * 20] + sm[q * 20 + 2 * PIECES];
        __syncthreads();
    }
    if (acc == 1234.5) out[0] = acc;
}
int main(int argc, char** argv) {
    const int gran = argc > 1 ? atoi(argv[1]) : 0;
    const long rows = argc > 2 ? atol(argv[2]) : 1000000, n = 10000000;
    if (gran) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran));
    size_t g = 0; CK(cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity));
    printf("cudaLimitMaxL2FetchGranularity = %zu (asked %d), %ld-row tables\n", g, gran, rows);
    double *A, *B, *out; uint2* idx;
    CK(cudaMalloc(&A, rows * 80)); CK(cudaMalloc(&B, rows * 80)); CK(cudaMalloc(&out, 4096)); CK(cudaMalloc(&idx, n * 8));
    CK(cudaMemset(A, 0, rows * 80)); CK(cudaMemset(B, 0, rows * 80));
    double* flush; const size_t fl = 512ull << 20; CK(cudaMalloc(&flush, fl));
    std::vector<uint2> hi(n); uint64_t s = 88172645463325252ull;
    for (long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; hi[i].x = s % rows; s ^= s << 13; s ^= s >> 7; s ^= s << 17; hi[i].y = s % rows; }
    CK(cudaMemcpy(idx, hi.data(), n * 8, cudaMemcpyHostToDevice));
    const int smem = 352 * 20 * 8;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* nm[] = {"2 tables 80B rows", "2 tables 64B heads", "2 tables 16B tails", "1 table 80B rows", "2 tables 32B rows"};
    void (*ks[])(const double*, const double*, const uint2*, long, double*) = {bench<0>, bench<1>, bench<2>, bench<3>, bench<4>};
    for (int mode = 0; mode < 5; ++mode) {
        CK(cudaFuncSetAttribute(ks[mode], cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        float tot = 0;
        for (int r = 0; r < 4; ++r) {
            cudaMemsetAsync(flush, r, fl);
            cudaEventRecord(e0);
            ks[mode]<<<148 * 3, 128, smem>>>(A, B, idx, n, out);
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) tot += ms;
        }
        const float ms = tot / 3;
        printf("mode %d %-22s: %7.1f us  %6.1f G rows/s\n", mode, nm[mode], ms * 1e3, 2.0 * n / ms / 1e6);
    }
    return 0;
}
