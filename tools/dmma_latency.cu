// Microbenchmark: mma.sync m8n8k4 f64 issue rate of ONE warp per SM sub-partition as a function of
// the number of independent accumulator chains, and with 1..4 warps per sub-partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_latency tools/dmma_latency.cu && tools/dmma_latency
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int CH>
__global__ void k(double* out, int iters, long long* cyc) {
    double d[CH][2];
    for (int i = 0; i < CH; ++i) d[i][0] = d[i][1] = threadIdx.x * 1e-9;
    const double a = 1.0000001, b = 1e-3;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < CH; ++i) dmma(d[i][0], d[i][1], a, b);
    const long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < CH; ++i) s += d[i][0] + d[i][1];
    if (s == 12345.0) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CH>
void run(int threads, double* dO, long long* dC) {
    const int iters = 2048;
    k<CH><<<148, threads>>>(dO, iters, dC);
    k<CH><<<148, threads>>>(dO, iters, dC);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, dC, 8, cudaMemcpyDeviceToHost);
    printf("chains %2d warps/SM %2d: %.1f cycles per DMMA per warp, %.1f cycles per DMMA per sub-partition\n", CH,
           threads / 32, (double)c / (iters * CH), (double)c / (iters * CH) / ((threads / 32 + 3) / 4));
}

int main() {
    double* dO;
    long long* dC;
    cudaMalloc(&dO, 8);
    cudaMalloc(&dC, 8);
    for (int threads : {32, 128, 256, 512}) {
        run<1>(threads, dO, dC);
        run<2>(threads, dO, dC);
        run<3>(threads, dO, dC);
        run<6>(threads, dO, dC);
        run<12>(threads, dO, dC);
        run<24>(threads, dO, dC);
    }
    return 0;
}
