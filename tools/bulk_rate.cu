// Microbenchmark: per-SM rate of cp.async.bulk (global -> shared, mbarrier completion) as a function
// of the copy size, the ring depth and the CTAs per SM, against 16-byte cp.async issued by a warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulk_rate tools/bulk_rate.cu && tools/bulk_rate
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t ph) {
    uint32_t done;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(b), "r"(ph) : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// one thread per CTA streams `n` copies of `bytes` through a ring of `depth` stages; `split` copies per stage
__global__ void k_bulk(const char* src, size_t per_cta, int n, int bytes, int depth, int split) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bars[16];
    if (threadIdx.x == 0) {
        for (int i = 0; i < depth; ++i) mbar_init(s32(&bars[i]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const char* p = src + (size_t)blockIdx.x * per_cta;
    const int piece = bytes / split;
    for (int i = 0; i < n + depth; ++i) {
        const int s = i % depth;
        if (i >= depth) mbar_wait(s32(&bars[s]), ((i / depth) - 1) & 1);
        if (i < n) {
            mbar_expect(s32(&bars[s]), bytes);
            for (int q = 0; q < split; ++q)
                bulk(s32(sm) + s * bytes + q * piece, p + (size_t)i * bytes + q * piece, piece, s32(&bars[s]));
        }
    }
}

// one warp per CTA streams the same bytes with 16-byte cp.async (commit groups, depth stages)
__global__ void k_ldgsts(const char* src, size_t per_cta, int n, int bytes, int depth) {
    extern __shared__ __align__(128) unsigned char sm[];
    const char* p = src + (size_t)blockIdx.x * per_cta;
    const int lane = threadIdx.x;
    for (int i = 0; i < n + depth; ++i) {
        const int s = i % depth;
        if (i < n) {
            for (int o = lane * 16; o < bytes; o += 512) {
                const uint32_t d = s32(sm) + s * bytes + o;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(p + (size_t)i * bytes + o));
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(2) : "memory");   // depth 3
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

int main() {
    const size_t total = (size_t)3 << 30;
    char* d;
    cudaMalloc(&d, total);
    cudaMemset(d, 1, total);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    printf("kind bytes depth split ctas/SM : GB/s total, GB/s per SM, copies/us per SM\n");
    for (int per_sm : {1, 2, 4}) {
        const int ctas = 148 * per_sm;
        for (int bytes : {2048, 4096, 8192, 16384}) {
            for (int depth : {3, 6}) {
                if ((size_t)bytes * depth * per_sm > 200 * 1024) continue;
                for (int split : {1, 2}) {
                    const size_t per_cta = total / ctas / 4096 * 4096;
                    const int n = (int)std::min<size_t>(per_cta / bytes, 2048);
                    float best = 1e9f;
                    for (int rep = 0; rep < 3; ++rep) {
                        cudaEventRecord(e0);
                        k_bulk<<<ctas, 32, bytes * depth>>>(d, per_cta, n, bytes, depth, split);
                        cudaEventRecord(e1);
                        cudaEventSynchronize(e1);
                        float ms;
                        cudaEventElapsedTime(&ms, e0, e1);
                        best = ms < best ? ms : best;
                    }
                    const double gb = (double)ctas * n * bytes / 1e9;
                    printf("bulk   %6d %d %d %d : %8.1f %7.1f %7.2f\n", bytes, depth, split, per_sm, gb / (best / 1e3),
                           gb / (best / 1e3) / 148, (double)per_sm * n * split / (best * 1e3));
                }
            }
            {
                const size_t per_cta = total / ctas / 4096 * 4096;
                const int n = (int)std::min<size_t>(per_cta / bytes, 2048);
                float best = 1e9f;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(e0);
                    k_ldgsts<<<ctas, 32, bytes * 3>>>(d, per_cta, n, bytes, 3);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    best = ms < best ? ms : best;
                }
                const double gb = (double)ctas * n * bytes / 1e9;
                printf("ldgsts %6d 3 - %d : %8.1f %7.1f\n", bytes, per_sm, gb / (best / 1e3), gb / (best / 1e3) / 148);
            }
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
