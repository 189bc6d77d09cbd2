// Microbenchmarks that decide the TTMcTC kernel shape on B200 (sm_100a):
//   (1) DFMA throughput, (2) DMMA (mma.sync f64) throughput for the shapes
//   ptxas accepts on sm_100a, (3) random 80-byte factor-row gathers from
//   working sets below and above L2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_fp64 microbench_fp64.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 1234.5) out[0] = s;
}

__global__ void dmma884_kernel(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    if (s == 1234.5) out[0] = s;
}

__global__ void dmma1684_kernel(double* out, int iters) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
    double c[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 1234.5) out[0] = s;
}

__global__ void dmma1688_kernel(double* out, int iters) {
    double a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
    b[0] = 1.0; b[1] = 0.5;
    double c[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 1234.5) out[0] = s;
}

// each thread gathers `per` random rows of 10 doubles (80 B) from a table of
// `rows` rows; 5 lanes cooperate per row with 16-byte loads.
__global__ void gather_kernel(const double* __restrict__ tab, const uint32_t* __restrict__ idx, long n, double* out) {
    long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    long g = t / 5;
    int part = t % 5;
    double s = 0;
    long stride = (long)gridDim.x * blockDim.x / 5;
    for (long e = g; e < n; e += stride) {
        uint32_t r = __ldg(idx + e);
        double2 v = __ldg(reinterpret_cast<const double2*>(tab + (size_t)r * 10) + part);
        s += v.x + v.y;
    }
    if (s == 1234.5) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SMs %d  L2 %d MB  clock %d MHz\n", sms, l2 >> 20, clk / 1000);
    double* out;
    CK(cudaMalloc(&out, 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    const int iters = 20000;
    for (int threads : {256, 512}) {
        for (int bps : {2, 4, 8}) {
            int blocks = sms * bps;
            dfma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
            cudaEventRecord(e0);
            dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            cudaEventElapsedTime(&ms, e0, e1);
            double fl = 2.0 * 8 * iters * (double)blocks * threads;
            printf("DFMA   threads %d blocks/SM %d : %.2f TFLOP/s\n", threads, bps, fl / ms / 1e9);
        }
    }
    for (int bps : {2, 4, 8}) {
        int blocks = sms * bps, threads = 256;
        dmma884_kernel<<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        dmma884_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * 8 * 4 * 4 * (double)iters * blocks * (threads / 32);
        printf("DMMA m8n8k4   blocks/SM %d : %.2f TFLOP/s\n", bps, fl / ms / 1e9);
        dmma1684_kernel<<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        dmma1684_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 16 * 8 * 4 * 4 * (double)iters * blocks * (threads / 32);
        printf("DMMA m16n8k4  blocks/SM %d : %.2f TFLOP/s\n", bps, fl / ms / 1e9);
        dmma1688_kernel<<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        dmma1688_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 16 * 8 * 8 * 4 * (double)iters * blocks * (threads / 32);
        printf("DMMA m16n8k8  blocks/SM %d : %.2f TFLOP/s\n", bps, fl / ms / 1e9);
    }
    // gathers
    for (long rows : {100000L, 1000000L, 2000000L, 4000000L}) {
        long n = 20000000;
        double* tab;
        uint32_t* idx;
        CK(cudaMalloc(&tab, rows * 80));
        CK(cudaMalloc(&idx, n * 4));
        CK(cudaMemset(tab, 0, rows * 80));
        std::vector<uint32_t> h(n);
        uint64_t s = 88172645463325252ull;
        for (long i = 0; i < n; ++i) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            h[i] = (uint32_t)(s % rows);
        }
        CK(cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice));
        int blocks = sms * 8, threads = 320;
        gather_kernel<<<blocks, threads>>>(tab, idx, n, out);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) gather_kernel<<<blocks, threads>>>(tab, idx, n, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double t = ms / 5 / 1e3;
        printf("gather 80B rows: table %.0f MB: %.3f G rows/s (%.0f GB/s row bytes, idx stream %.0f GB/s)\n",
               rows * 80 / 1e6, n / t / 1e9, n * 80 / t / 1e9, n * 4 / t / 1e9);
        cudaFree(tab);
        cudaFree(idx);
    }
    return 0;
}
