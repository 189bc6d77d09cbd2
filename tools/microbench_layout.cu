// Factor-row layouts for the pass's two-table random gathers (K = 10, 10^6-row tables, 10^7 pairs):
// L2 capacity is allocated in 128-byte lines, and an 80-byte row straddles two lines half of the time
// (1.5 lines = 192 B of L2 per row), so the L2 holds only ~40 % of the two 80 MB tables.  Layouts tried:
//   0: 80 B rows, no hint          1: 80 B rows, evict_last
//   2: split 64 B head + 16 B tail tables (no straddling; 8 tails per line), no hint
//   3: split, tails evict_last     4: split, both evict_last
//   5: 128 B padded rows (one line per row)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_layout tools/microbench_layout.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_normal() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ void cp16h(void* d, const void* s, uint64_t p) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" :: "r"(sa(d)), "l"(s), "l"(p));
}
struct Tabs { const double *A, *B, *PA, *QA, *PB, *QB, *WA, *WB; };
__global__ void __launch_bounds__(128) bench(Tabs t, const uint2* idx, long n, int mode, double* out) {
    extern __shared__ __align__(128) double sm[];
    const int CAP = 352;
    __shared__ uint2 sidx[352];
    const uint64_t pl = pol_last(), pn = pol_normal();
    const uint64_t ph = (mode == 1 || mode == 4) ? pl : pn;  // head / whole-row policy
    const uint64_t pt = (mode == 3 || mode == 4 || mode == 1) ? pl : pn;  // tail policy
    long per = (n + gridDim.x - 1) / gridDim.x; long b = per * blockIdx.x, e = min(n, b + per);
    double acc = 0;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (long r0 = b; r0 < e; r0 += CAP) {
        int cn = (int)min((long)CAP, e - r0);
        for (int q = tid; q < cn; q += nt) sidx[q] = idx[r0 + q];
        __syncthreads();
        // 10 pieces of 16 B per pair (5 per row), piece slots strided over the CTA
        for (int s = tid; s < cn * 10; s += nt) {
            const int r = s / 10, pc = s - r * 10;
            double* d = sm + r * 20 + 2 * pc;
            const bool first = pc < 5;
            const uint32_t j = first ? sidx[r].x : sidx[r].y;
            const int q = first ? pc : pc - 5;
            if (mode <= 1) cp16h(d, (first ? t.A : t.B) + (size_t)j * 10 + 2 * q, ph);
            else if (mode <= 4) {
                if (q < 4) cp16h(d, (first ? t.PA : t.PB) + (size_t)j * 8 + 2 * q, ph);
                else cp16h(d, (first ? t.QA : t.QB) + (size_t)j * 2, pt);
            } else cp16h(d, (first ? t.WA : t.WB) + (size_t)j * 16 + 2 * q, pn);
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        for (int q = tid; q < cn; q += nt) acc += sm[q * 20] + sm[q * 20 + 19];
        __syncthreads();
    }
    if (acc == 1234.5) out[0] = acc;
}
int main() {
    const long rows = 1000000, n = 10000000;
    double *A, *B, *PA, *QA, *PB, *QB, *WA, *WB, *out; uint2* idx;
    CK(cudaMalloc(&A, rows * 80)); CK(cudaMalloc(&B, rows * 80)); CK(cudaMalloc(&PA, rows * 64)); CK(cudaMalloc(&QA, rows * 16));
    CK(cudaMalloc(&PB, rows * 64)); CK(cudaMalloc(&QB, rows * 16)); CK(cudaMalloc(&WA, rows * 128)); CK(cudaMalloc(&WB, rows * 128));
    CK(cudaMalloc(&out, 4096)); CK(cudaMalloc(&idx, n * 8));
    double* flush; const size_t fl = 512ull << 20; CK(cudaMalloc(&flush, fl));
    for (double* p : {A, B, PA, PB, QA, QB, WA, WB}) cudaMemset(p, 0, rows * 16);
    std::vector<uint2> hi(n); uint64_t s = 88172645463325252ull;
    for (long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; hi[i].x = s % rows; s ^= s << 13; s ^= s >> 7; s ^= s << 17; hi[i].y = s % rows; }
    CK(cudaMemcpy(idx, hi.data(), n * 8, cudaMemcpyHostToDevice));
    int smem = 352 * 20 * 8; CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    Tabs t{A, B, PA, QA, PB, QB, WA, WB};
    const char* nm[] = {"80B rows", "80B rows evict_last", "split 64+16", "split, tails evict_last", "split, both evict_last", "128B padded rows"};
    for (int mode = 0; mode < 6; ++mode) for (int bps : {3, 4}) {
        bench<<<148 * bps, 128, smem>>>(t, idx, n, mode, out);
        CK(cudaDeviceSynchronize());
        float tot = 0;
        for (int r = 0; r < 5; ++r) {
            cudaMemsetAsync(flush, r, fl);  // L2 flush between timed runs (the solver's other work evicts too)
            cudaEventRecord(e0);
            bench<<<148 * bps, 128, smem>>>(t, idx, n, mode, out);
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1); tot += ms;
        }
        const float ms = tot / 5;
        printf("mode %d %-26s CTAs/SM %d: %7.1f us  %6.1f G rows/s\n", mode, nm[mode], bps, ms * 1e3, 2.0 * n / ms / 1e6);
    }
    return 0;
}
