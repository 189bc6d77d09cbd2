// Two-table random row gather (the fused pass's pattern: per record one
// 80-byte row of A and one of B), double-buffered rounds of CAP records per
// CTA, comparing the issue mechanisms:
//   mode 0: cp.async 16-byte pieces, piece-major (the pass's current scheme)
//   mode 1: cp.async.bulk (TMA engine) of each whole 80-byte row, one row per
//           thread, completion counted in bytes on a per-buffer mbarrier
// Reports G rows/s and the issue cycles per round (thread 0's clock).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_bulkrow tools/microbench_bulkrow.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int CAP = 384, FW = 22;
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp16(void* d, const void* s) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa(d)), "l"(s));
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" :: "r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("{\n.reg .b64 s;\nmbarrier.arrive.shared::cta.b64 s, [%0];\n}" :: "r"(sa(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nL_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra L_%=;\n}" :: "r"(sa(b)), "r"(ph) : "memory");
}

// row indices from a hash of the record id (the pass reads them from shared memory; a global load here
// would put one DRAM latency inside every issue loop)
__device__ __forceinline__ uint2 rec_idx(long r, long rows) {
    uint64_t x = (uint64_t)r * 0x9E3779B97F4A7C15ull;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    return make_uint2((uint32_t)((x & 0xffffffffull) % rows), (uint32_t)((x >> 32) % rows));
}
__global__ void gather(const double* A, const double* B, const uint2* idx, long n, int mode, double* out,
                       unsigned long long* issue_cyc, int pitch) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bar[2];
    double* buf[2] = {sm, sm + CAP * FW};
    if (threadIdx.x == 0) { mb_init(&bar[0], blockDim.x); mb_init(&bar[1], blockDim.x); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    long per = (n + gridDim.x - 1) / gridDim.x;
    long b = per * blockIdx.x, e = min(n, b + per);
    int rounds = (int)((e - b + CAP - 1) / CAP);
    double acc = 0;
    unsigned long long ic = 0;
    auto issue = [&](int r) {
        long r0 = b + (long)r * CAP;
        int cn = (int)min((long)CAP, e - r0);
        double* d = buf[r & 1];
        long long t0 = clock64();
        if (mode == 0 || mode == 3) {
            // mode 3: each table split into a 64-byte head (8 values, pitch 8) and a 16-byte tail (pitch 2)
            const double* At = A + 8ull * 1000000;  // tails after the heads
            const double* Bt = B + 8ull * 1000000;
            for (int q = threadIdx.x; q < cn * 10; q += blockDim.x) {
                int t = q / 10, pc = q - t * 10;
                uint2 jk = rec_idx(r0 + t, 1000000);
                const double* src;
                if (mode == 0) src = pc < 5 ? A + (size_t)jk.x * pitch + 2 * pc : B + (size_t)jk.y * pitch + 2 * (pc - 5);
                else if (pc < 4) src = A + (size_t)jk.x * 8 + 2 * pc;
                else if (pc == 4) src = At + (size_t)jk.x * 2;
                else if (pc < 9) src = B + (size_t)jk.y * 8 + 2 * (pc - 5);
                else src = Bt + (size_t)jk.y * 2;
                cp16(d + (size_t)t * FW + 2 * pc, src);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        } else if (mode == 2) {  // A rows on the TMA engine (bulk), B rows as cp.async pieces on the LSU
            int mine = 0;
            for (int t = threadIdx.x; t < cn; t += blockDim.x) mine += 1;
            mb_expect(&bar[r & 1], mine * 80);
            for (int t = threadIdx.x; t < cn; t += blockDim.x) {
                uint2 jk = rec_idx(r0 + t, 1000000);
                bulk(d + (size_t)t * FW, A + (size_t)jk.x * 10, 80, &bar[r & 1]);
            }
            mb_arrive(&bar[r & 1]);
            for (int q = threadIdx.x; q < cn * 5; q += blockDim.x) {
                int t = q / 5, pc = q - t * 5;
                uint2 jk = rec_idx(r0 + t, 1000000);
                cp16(d + (size_t)t * FW + 10 + 2 * pc, B + (size_t)jk.y * 10 + 2 * pc);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        } else {
            int mine = 0;
            for (int t = threadIdx.x; t < cn; t += blockDim.x) mine += 2;
            mb_expect(&bar[r & 1], mine * 80);
            for (int t = threadIdx.x; t < cn; t += blockDim.x) {
                uint2 jk = rec_idx(r0 + t, 1000000);
                bulk(d + (size_t)t * FW, A + (size_t)jk.x * 10, 80, &bar[r & 1]);
                bulk(d + (size_t)t * FW + 10, B + (size_t)jk.y * 10, 80, &bar[r & 1]);
            }
            mb_arrive(&bar[r & 1]);
        }
        if (threadIdx.x == 0) ic += clock64() - t0;
    };
    if (rounds > 0) issue(0);
    for (int r = 0; r < rounds; ++r) {
        __syncthreads();  // buffer (r + 1) & 1 free (consumed in round r - 1)
        if (r + 1 < rounds) issue(r + 1);
        if (mode != 1) {
            if (r + 1 < rounds) asm volatile("cp.async.wait_group 1;" ::: "memory");
            else asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        if (mode == 1 || mode == 2) mb_wait(&bar[r & 1], (r >> 1) & 1);
        __syncthreads();
        long r0 = b + (long)r * CAP;
        int cn = (int)min((long)CAP, e - r0);
        double* d = buf[r & 1];
        for (int t = threadIdx.x; t < cn; t += blockDim.x) acc += d[t * FW] + d[t * FW + 19];
    }
    if (acc == 1234.5) out[0] = acc;
    if (threadIdx.x == 0) atomicAdd(issue_cyc, ic);
}

int main() {
    const long rows = 1000000, n = 10000000;
    double *A, *B, *out; uint2* idx; unsigned long long* ic;
    CK(cudaMalloc(&A, rows * 128)); CK(cudaMalloc(&B, rows * 128)); CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&idx, n * 8));
    CK(cudaMalloc(&ic, 8));
    cudaMemset(A, 0, rows * 128); cudaMemset(B, 0, rows * 128);
    std::vector<uint2> h(n); uint64_t s = 88172645463325252ull;
    for (long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i].x = s % rows; s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i].y = s % rows; }
    CK(cudaMemcpy(idx, h.data(), n * 8, cudaMemcpyHostToDevice));
    int smem = 2 * CAP * FW * 8;  // 135 KB: one CTA per SM
    CK(cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int pitch : {10}) for (int threads : {256, 512}) for (int mode : {0, 3}) {
        const int bps = 1;
        int grid = 148 * bps;
        for (int w = 0; w < 2; ++w) gather<<<grid, threads, smem>>>(A, B, idx, n, mode, out, ic, pitch);
        CK(cudaMemset(ic, 0, 8));
        cudaEventRecord(e0);
        for (int w = 0; w < 3; ++w) gather<<<grid, threads, smem>>>(A, B, idx, n, mode, out, ic, pitch);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 3;
        unsigned long long hc; cudaMemcpy(&hc, ic, 8, cudaMemcpyDeviceToHost);
        double rounds = 3.0 * ((double)n / grid / CAP) * grid;
        printf("pitch %2d threads %3d mode %d (%s): %7.1f us  %6.1f G rows/s  issue %7.0f cycles/round\n", pitch, threads,
               mode, mode == 3 ? "split 64+16 " : mode == 2 ? "A bulk+B cp16" : mode ? "bulk/row    " : "cp16        ", ms * 1e3, 2.0 * n / ms / 1e6, hc / rounds);
    }
    return 0;
}
