// fp64 tensor-core (DMMA, mma.sync m8n8k4) versions of the block-sweep panel
// kernels: HPANEL, UPDATE, GPANEL.  Same algebra and work items as the DFMA
// kernels in ens_mf.cu; a CTA computes one 64x64 output tile with 8 warps
// (2 x 4, each 32 rows x 16 cols = 4 x 2 m8n8 tiles), operands staged in
// shared memory with a bank-conflict-free stride (LDM = 68).  fp64 MMA on B200
// runs at the fp64 FMA rate (measured: tools/fp64_peak.cu); its point here is
// operand reuse -- one m8n8k4 = 256 FMAs for two shared-memory loads per lane.
#include "ens_internal.cuh"
#include "ens_mf_common.cuh"

#define LDM 68

__device__ __forceinline__ int outside_m(int r, int a, int pw) { return r < a ? r : r + pw; }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// acc[i][j][e] += sum_k As[row][k] Bs[k][col], row = 32 wr + 8 i + g, col = 16 wc + 8 j + 2 q + e
__device__ __forceinline__ void mma_64x64(const double* __restrict__ As, const double* __restrict__ Bs, int Kpad,
                                          double acc[4][2][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wr = warp & 1, wc = warp >> 1;
    const int g = lane >> 2, q = lane & 3;
    const double* ap = As + (32 * wr + g) * LDM + q;
    const double* bp = Bs + q * LDM + 16 * wc + g;
#pragma unroll 4
    for (int k0 = 0; k0 < Kpad; k0 += 4) {
        double a[4], b[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = ap[8 * i * LDM + k0];
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = bp[k0 * LDM + 8 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
}

#define ACC_ZERO(acc)                                   \
    _Pragma("unroll") for (int i = 0; i < 4; ++i)       \
        _Pragma("unroll") for (int j = 0; j < 2; ++j) { \
            acc[i][j][0] = 0.0;                         \
            acc[i][j][1] = 0.0;                         \
        }

// UPDATE: F[Q-rows, Q-cols] -= F[Q-rows, P] F[P, Q-cols]
__global__ void __launch_bounds__(256) k_update_mma(MfDev d, int item0, double* __restrict__ F) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1], r0 = it[2], c0 = it[3];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int t = m - pw;
    const int nr = min(ENS_TILE, t - r0), nc = min(ENS_TILE, t - c0);
    const int Kpad = (pw + 3) & ~3;
    double* Cs = sm;                 // [64][LDM]  C[r][k]
    double* Hs = sm + 64 * LDM;      // [64][LDM]  H[k][c]
    double* base = F + (int64_t)mat * d.storage + d.off[f];
    for (int e = threadIdx.x; e < 64 * Kpad; e += blockDim.x) {
        const int r = e / Kpad, kk = e % Kpad;
        Cs[r * LDM + kk] = (r < nr && kk < pw) ? base[(int64_t)outside_m(r0 + r, a, pw) * m + a + kk] : 0.0;
    }
    for (int e = threadIdx.x; e < Kpad * 64; e += blockDim.x) {
        const int kk = e >> 6, cc = e & 63;
        Hs[kk * LDM + cc] = (kk < pw && cc < nc) ? base[(int64_t)(a + kk) * m + outside_m(c0 + cc, a, pw)] : 0.0;
    }
    __syncthreads();
    double acc[4][2][2];
    ACC_ZERO(acc);
    mma_64x64(Cs, Hs, Kpad, acc);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wr = warp & 1, wc = warp >> 1, g = lane >> 2, q = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = 32 * wr + 8 * i + g;
        if (r >= nr) continue;
        double* row = base + (int64_t)outside_m(r0 + r, a, pw) * m;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int cc = 16 * wc + 8 * j + 2 * q + e;
                if (cc < nc) row[outside_m(c0 + cc, a, pw)] -= acc[i][j][e];
            }
    }
}

// HPANEL: F[P, Q-tile] <- D^-1 F[P, Q-tile]   (D^-1 = -F[P,P])
__global__ void __launch_bounds__(256) k_hpanel_mma(MfDev d, int item0, double* __restrict__ F) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1], c0 = it[2];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int t = m - pw;
    const int nc = min(ENS_TILE, t - c0);
    const int Kpad = (pw + 3) & ~3;
    double* Ds = sm;                 // [64][LDM]  D^-1[r][k]
    double* Rs = sm + 64 * LDM;      // [64][LDM]  R[k][c]
    double* base = F + (int64_t)mat * d.storage + d.off[f];
    for (int e = threadIdx.x; e < 64 * Kpad; e += blockDim.x) {
        const int r = e / Kpad, kk = e % Kpad;
        Ds[r * LDM + kk] = (r < pw && kk < pw) ? -base[(int64_t)(a + r) * m + a + kk] : 0.0;
    }
    for (int e = threadIdx.x; e < Kpad * 64; e += blockDim.x) {
        const int kk = e >> 6, cc = e & 63;
        Rs[kk * LDM + cc] = (kk < pw && cc < nc) ? base[(int64_t)(a + kk) * m + outside_m(c0 + cc, a, pw)] : 0.0;
    }
    __syncthreads();
    double acc[4][2][2];
    ACC_ZERO(acc);
    mma_64x64(Ds, Rs, Kpad, acc);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wr = warp & 1, wc = warp >> 1, g = lane >> 2, q = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = 32 * wr + 8 * i + g;
        if (r >= pw) continue;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int cc = 16 * wc + 8 * j + 2 * q + e;
                if (cc < nc) base[(int64_t)(a + r) * m + outside_m(c0 + cc, a, pw)] = acc[i][j][e];
            }
    }
}

// GPANEL: F[Q-tile, P] <- F[Q-tile, P] D^-1
__global__ void __launch_bounds__(256) k_gpanel_mma(MfDev d, int item0, double* __restrict__ F) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1], r0 = it[2];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int t = m - pw;
    const int nr = min(ENS_TILE, t - r0);
    const int Kpad = (pw + 3) & ~3;
    double* Cs = sm;                 // [64][LDM]  C[r][k]
    double* Ds = sm + 64 * LDM;      // [64][LDM]  D^-1[k][c]
    double* base = F + (int64_t)mat * d.storage + d.off[f];
    for (int e = threadIdx.x; e < 64 * Kpad; e += blockDim.x) {
        const int r = e / Kpad, kk = e % Kpad;
        Cs[r * LDM + kk] = (r < nr && kk < pw) ? base[(int64_t)outside_m(r0 + r, a, pw) * m + a + kk] : 0.0;
    }
    for (int e = threadIdx.x; e < Kpad * 64; e += blockDim.x) {
        const int kk = e >> 6, cc = e & 63;
        Ds[kk * LDM + cc] = (kk < pw && cc < pw) ? -base[(int64_t)(a + kk) * m + a + cc] : 0.0;
    }
    __syncthreads();
    double acc[4][2][2];
    ACC_ZERO(acc);
    mma_64x64(Cs, Ds, Kpad, acc);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wr = warp & 1, wc = warp >> 1, g = lane >> 2, q = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = 32 * wr + 8 * i + g;
        if (r >= nr) continue;
        double* row = base + (int64_t)outside_m(r0 + r, a, pw) * m + a;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int cc = 16 * wc + 8 * j + 2 * q + e;
                if (cc < pw) row[cc] = acc[i][j][e];
            }
    }
}

static const size_t SM_MMA = sizeof(double) * 2 * 64 * LDM;

int mf_mma_setup() {
    ENS_CK(cudaFuncSetAttribute(k_update_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_MMA));
    ENS_CK(cudaFuncSetAttribute(k_hpanel_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_MMA));
    ENS_CK(cudaFuncSetAttribute(k_gpanel_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_MMA));
    return ENS_OK;
}

void launch_update_mma(const MfDev& d, int off, int n, double* F, cudaStream_t s) {
    k_update_mma<<<dim3(n, 2), 256, SM_MMA, s>>>(d, off, F);
}
void launch_hpanel_mma(const MfDev& d, int off, int n, double* F, cudaStream_t s) {
    k_hpanel_mma<<<dim3(n, 2), 256, SM_MMA, s>>>(d, off, F);
}
void launch_gpanel_mma(const MfDev& d, int off, int n, double* F, cudaStream_t s) {
    k_gpanel_mma<<<dim3(n, 2), 256, SM_MMA, s>>>(d, off, F);
}
