// Latency of the K x K Cholesky + triangular inverse of a mode update (one warp), K = 10:
// (a) the engine's shared-memory left-looking warp_chol / warp_inv_upper (runtime K),
// (b) the same with compile-time K,
// (c) registers: lane a owns column a, right-looking updates with shuffles, fast reciprocal square roots.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_chol tools/microbench_chol.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ bool chol_a(const double* W, int K, double* R, int lane) {
    for (int q = lane; q < K * K; q += 32) R[q] = 0.0;
    __syncwarp();
    for (int k = 0; k < K; ++k) {
        double d = W[k * K + k];
        for (int j = 0; j < k; ++j) d -= R[j * K + k] * R[j * K + k];
        if (!(d > 1e-12 * W[k * K + k]) || !isfinite(d)) return false;
        const double rkk = sqrt(d);
        if (lane > k && lane < K) {
            double s = W[k * K + lane];
            for (int j = 0; j < k; ++j) s -= R[j * K + k] * R[j * K + lane];
            R[k * K + lane] = s / rkk;
        }
        if (lane == 0) R[k * K + k] = rkk;
        __syncwarp();
    }
    return true;
}
__device__ void inv_a(const double* R, int K, double* X, int lane) {
    if (lane < K) {
        const int j = lane;
        for (int i = 0; i < K; ++i) X[i * K + j] = 0.0;
        X[j * K + j] = 1.0 / R[j * K + j];
        for (int i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int k = i + 1; k <= j; ++k) s += R[i * K + k] * X[k * K + j];
            X[i * K + j] = -s / R[i * K + i];
        }
    }
    __syncwarp();
}
template <int K>
__device__ bool chol_b(const double* W, double* R, int lane) {
#pragma unroll
    for (int q = lane; q < K * K; q += 32) R[q] = 0.0;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double d = W[k * K + k];
#pragma unroll
        for (int j = 0; j < k; ++j) d -= R[j * K + k] * R[j * K + k];
        if (!(d > 1e-12 * W[k * K + k]) || !isfinite(d)) return false;
        const double rkk = sqrt(d);
        if (lane > k && lane < K) {
            double s = W[k * K + lane];
#pragma unroll
            for (int j = 0; j < k; ++j) s -= R[j * K + k] * R[j * K + lane];
            R[k * K + lane] = s / rkk;
        }
        if (lane == 0) R[k * K + k] = rkk;
        __syncwarp();
    }
    return true;
}
template <int K>
__device__ void inv_b(const double* R, double* X, int lane) {
    if (lane < K) {
        const int j = lane;
#pragma unroll
        for (int i = 0; i < K; ++i) X[i * K + j] = 0.0;
        X[j * K + j] = 1.0 / R[j * K + j];
        for (int i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int k = i + 1; k <= j; ++k) s += R[i * K + k] * X[k * K + j];
            X[i * K + j] = -s / R[i * K + i];
        }
    }
    __syncwarp();
}
// (c) lane a holds column a of W (w[b] = W[b][a]); after the loop w[k] = R[k][a] for k <= a
template <int K, int FAST>
__device__ bool chol_c(const double* W, double* R, double* X, int lane) {
    double w[K];
#pragma unroll
    for (int b = 0; b < K; ++b) w[b] = (lane < K) ? W[b * K + lane] : 0.0;
    const double d0 = (lane < K) ? W[lane * K + lane] : 1.0;
    bool ok = true;
    double rinv_diag = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double piv = __shfl_sync(0xffffffffu, w[k], k);  // W'[k][k] (lane k's w[k])
        const double dk = __shfl_sync(0xffffffffu, d0, k);
        ok = ok && (piv > 1e-12 * dk) && isfinite(piv);
        double rkk, inv;
        if (FAST) { inv = rsqrt(piv); rkk = piv * inv; }
        else { rkk = sqrt(piv); inv = 1.0 / rkk; }
        // row k of R: R[k][a] = W'[k][a] / rkk for a >= k
        double rka = (lane > k) ? w[k] * inv : (lane == k ? rkk : 0.0);
        if (lane == k) rinv_diag = inv;
        w[k] = rka;
        // trailing update W'[b][a] -= R[k][b] R[k][a] for b > k, a > k
#pragma unroll
        for (int b = k + 1; b < K; ++b) {
            const double rkb = __shfl_sync(0xffffffffu, rka, b);
            if (lane > k) w[b] -= rkb * rka;
        }
    }
    // R to smem (row k col a = w[k])
    if (lane < K)
#pragma unroll
        for (int k = 0; k < K; ++k) R[k * K + lane] = (k <= lane) ? w[k] : 0.0;
    __syncwarp();
    // X = R^-1 column j = lane: back substitution, rows i = j-1..0 ; x[i] = -(sum_{k>i} R[i][k] x[k]) / R[i][i]
    double dinv[K];
#pragma unroll
    for (int i = 0; i < K; ++i) dinv[i] = __shfl_sync(0xffffffffu, rinv_diag, i);
    if (lane < K) {
        double x[K];
#pragma unroll
        for (int i = 0; i < K; ++i) x[i] = 0.0;
        const int j = lane;
        x[0] = 0.0;
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
            if (i == j) x[i] = rinv_diag;
            else if (i < j) {
                double s = 0.0;
#pragma unroll
                for (int k = i + 1; k < K; ++k) s += R[i * K + k] * x[k];
                x[i] = -s * dinv[i];
            }
        }
#pragma unroll
        for (int i = 0; i < K; ++i) X[i * K + j] = x[i];
    }
    __syncwarp();
    return ok;
}

template <int V>
__global__ void bench(const double* W, double* out, long long* cyc, int K, int reps) {
    __shared__ double sW[100], sR[100], sX[100];
    const int lane = threadIdx.x;
    for (int q = lane; q < 100; q += 32) sW[q] = W[q];
    __syncwarp();
    long long t0 = clock64();
    bool ok = true;
    for (int r = 0; r < reps; ++r) {
        if (V == 0) { ok = chol_a(sW, K, sR, lane); inv_a(sR, K, sX, lane); }
        if (V == 1) { ok = chol_b<10>(sW, sR, lane); inv_b<10>(sR, sX, lane); }
        if (V == 2) { ok = chol_c<10, 0>(sW, sR, sX, lane); }
        if (V == 3) { ok = chol_c<10, 1>(sW, sR, sX, lane); }
        if (lane == 0) sW[0] += 0.0 * sX[1];  // keep the dependence across reps
        __syncwarp();
    }
    long long t1 = clock64();
    for (int q = lane; q < 100; q += 32) out[q] = sX[q];
    if (lane == 0) { cyc[0] = (t1 - t0) / reps; cyc[1] = ok; }
}

int main() {
    const int K = 10;
    double hW[100];
    double B[100];
    for (int i = 0; i < 100; ++i) B[i] = sin(1.7 * i + 0.3) + (i % 11 == 0 ? 3.0 : 0.0);
    for (int i = 0; i < K; ++i)
        for (int j = 0; j < K; ++j) {
            double s = 0.0;
            for (int k = 0; k < K; ++k) s += B[k * K + i] * B[k * K + j];
            hW[i * K + j] = s;
        }
    double *dW, *dO;
    long long* dc;
    cudaMalloc(&dW, 800); cudaMalloc(&dO, 800 * 4); cudaMalloc(&dc, 16 * 4);
    cudaMemcpy(dW, hW, 800, cudaMemcpyHostToDevice);
    bench<0><<<1, 32>>>(dW, dO, dc, K, 50);
    bench<1><<<1, 32>>>(dW, dO + 100, dc + 2, K, 50);
    bench<2><<<1, 32>>>(dW, dO + 200, dc + 4, K, 50);
    bench<3><<<1, 32>>>(dW, dO + 300, dc + 6, K, 50);
    cudaDeviceSynchronize();
    double hO[400]; long long hc[8];
    cudaMemcpy(hO, dO, 3200, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc, dc, 64, cudaMemcpyDeviceToHost);
    double d1 = 0, d2 = 0, d3 = 0;
    for (int i = 0; i < 100; ++i) { d1 = fmax(d1, fabs(hO[i] - hO[100 + i])); d2 = fmax(d2, fabs(hO[i] - hO[200 + i])); d3 = fmax(d3, fabs(hO[i] - hO[300 + i])); }
    printf("chol+inv K=10 cycles: smem runtime-K %lld (ok %lld), smem compile-time K %lld, registers %lld, registers+rsqrt %lld; max|dX| b %.3g c %.3g d %.3g (%s)\n",
           hc[0], hc[1], hc[2], hc[4], hc[6], d1, d2, d3, cudaGetErrorString(cudaGetLastError()));
}
