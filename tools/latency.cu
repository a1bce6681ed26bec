// Memory latency / launch overhead calibration on the box (not part of the library).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_chase(const int64_t* __restrict__ p, int64_t start, int n, int64_t* out) {
    int64_t i = start;
    for (int s = 0; s < n; ++s) i = p[i];
    out[threadIdx.x + blockIdx.x * blockDim.x] = i;
}
__global__ void k_empty(int64_t* out) { if (threadIdx.x == 1023) out[0] = 1; }

int main() {
    const int64_t big = (int64_t)1 << 27;   // 1 GiB of int64
    int64_t* d; int64_t* out;
    cudaMalloc(&d, big * 8); cudaMalloc(&out, 1 << 20);
    std::vector<int64_t> h(big);
    for (int64_t span : {(int64_t)1 << 15, (int64_t)1 << 20, (int64_t)1 << 24, big}) {   // 256KB, 8MB, 128MB, 1GB
        uint64_t x = 88172645463325252ull;
        for (int64_t i = 0; i < span; ++i) h[i] = i;
        for (int64_t i = span - 1; i > 0; --i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; int64_t j = x % i; std::swap(h[i], h[j]); }
        // cycle through a random permutation, stride 64 elements (512 B) apart
        std::vector<int64_t> perm(h.begin(), h.begin() + span);
        std::vector<int64_t> nxt(span);
        const int64_t step = span >= 4096 ? 64 : 1;
        const int64_t nodes = span / step;
        for (int64_t i = 0; i < nodes; ++i) nxt[(perm[i] % nodes) * step] = (perm[(i + 1) % nodes] % nodes) * step;
        cudaMemcpy(d, nxt.data(), span * 8, cudaMemcpyHostToDevice);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        const int n = 2000;
        k_chase<<<1, 1>>>(d, 0, 100, out);
        cudaEventRecord(a); k_chase<<<1, 1>>>(d, 0, n, out); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("span %8lld KB: %.0f ns per dependent load (1 thread)\n", (long long)(span * 8 / 1024), 1e6 * ms / n);
        // loaded: 148*8 warps chasing concurrently
        cudaEventRecord(a); k_chase<<<148 * 4, 64>>>(d, 0, n / 4, out); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("span %8lld KB: %.0f ns per dependent load (592x64 threads)\n", (long long)(span * 8 / 1024), 1e6 * ms / (n / 4));
    }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a); for (int i = 0; i < 100; ++i) k_empty<<<30, 256>>>(out); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("empty kernel stream launch: %.2f us each\n", 1e3 * ms / 100);
    }
    cudaStream_t s; cudaStreamCreate(&s);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; ++i) k_empty<<<30, 256, 0, s>>>(out);
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("empty kernel in graph: %.2f us each\n", 1e3 * ms / 100);
    return 0;
}
