// Microbenchmark: fp64 FMA vs fp64 tensor-core MMA (mma.sync m8n8k4) throughput on
// this GPU, plus a correctness check of the m8n8k4 fragment layout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cstdlib>
#include <cmath>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void k_layout(const double* A, const double* B, double* D) {
    const int l = threadIdx.x;
    double a = A[(l >> 2) * 4 + (l & 3)];        // A 8x4 row-major
    double b = B[(l & 3) * 8 + (l >> 2)];        // B 4x8 row-major, fragment = B[k][n]
    double d0 = 0, d1 = 0;
    dmma(d0, d1, a, b);
    D[(l >> 2) * 8 + 2 * (l & 3)] = d0;
    D[(l >> 2) * 8 + 2 * (l & 3) + 1] = d1;
}

__global__ void k_dfma(double* out, int iters) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-9 + i;
    const double b = 1.0000001, c = 1e-12;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.0) out[0] = s;
}

__global__ void k_dmma(double* out, int iters) {
    double d[8][2];
    for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-9;
    const double a = 1.0000001, b = 1e-3;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(d[i][0], d[i][1], a, b);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double hA[32], hB[32], hD[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = std::sin(i + 1.0); hB[i] = std::cos(2.0 * i + 0.5); }
    for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int k = 0; k < 4; ++k) s += hA[r * 4 + k] * hB[k * 8 + c];
            ref[r * 8 + c] = s;
        }
    double *dA, *dB, *dD, *dO;
    cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dD, 512); cudaMalloc(&dO, 8);
    cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
    k_layout<<<1, 32>>>(dA, dB, dD);
    cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 64; ++i) err = std::fmax(err, std::fabs(hD[i] - ref[i]));
    printf("m8n8k4 layout max err %.3e\n", err);
    int dev; cudaGetDevice(&dev);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096, blocks = sms * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(dO, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * iters * (double)blocks * threads;
        printf("DFMA  %.2f TFLOP/s\n", flops / ms / 1e9);
        cudaEventRecord(e0);
        k_dmma<<<blocks, threads>>>(dO, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
        printf("DMMA  %.2f TFLOP/s\n", flops / ms / 1e9);
    }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
