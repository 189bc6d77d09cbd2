// Do DMMA (FP64 tensor) and DFMA (FP64 ALU) issue to separate pipes on B200?
// Half the warps of each CTA run DMMA m8n8k4, half DFMA; compare the mix's
// combined FLOP rate with each alone.
#include <cstdio>
#include <cuda_runtime.h>
__device__ void dfma_loop(double* out, int iters) {
    double acc[8];
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], 1.0000001, 1e-9);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 1234.5) out[0] = s;
}
__device__ void dmma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0;
    double c[4][2] = {};
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    double s = 0;
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    if (s == 1234.5) out[0] = s;
}
// mode 0: all DFMA, 1: all DMMA, 2: even warps DMMA / odd DFMA
__global__ void mix(double* out, int it_f, int it_m, int mode) {
    int w = threadIdx.x / 32;
    bool mm = (mode == 1) || (mode == 2 && (w & 1) == 0);
    if (mm) dmma_loop(out, it_m); else dfma_loop(out, it_f);
}
int main() {
    double* out; cudaMalloc(&out, 8);
    int blocks = 148 * 4, threads = 256;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int itf = 20000, itm = 20000;
    double fl_f = 2.0 * 8 * itf, fl_m_warp = 2.0 * 256 * 4 * itm;  // per thread / per warp
    for (int mode = 0; mode < 3; ++mode) {
        mix<<<blocks, threads>>>(out, 100, 100, mode);
        cudaEventRecord(e0);
        mix<<<blocks, threads>>>(out, itf, itm, mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        int warps = blocks * threads / 32;
        double fl = 0;
        if (mode == 0) fl = fl_f * blocks * threads;
        if (mode == 1) fl = fl_m_warp * warps;
        if (mode == 2) fl = fl_m_warp * warps / 2 + fl_f * blocks * threads / 2;
        printf("mode %d (%s): %.3f ms  %.2f TFLOP/s\n", mode, mode == 0 ? "DFMA" : mode == 1 ? "DMMA" : "half/half",
               ms, fl / ms / 1e9);
    }
    return 0;
}
