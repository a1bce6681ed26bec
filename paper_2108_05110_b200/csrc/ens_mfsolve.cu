// Multi-column solves with the block-sweep fronts (sm_100a, fp64).
//
// After ens_mf.cu's sweep each front holds [-F11^-1, F11^-1 F12; F21 F11^-1, S].
// Per tree level (leaves -> root) the forward pass is
//     fr_f = [b(pivots); 0] + extend-add of the children's CB vectors
//     fr_f[C] -= F[C,P] fr_f[P]
// and per level (root -> leaves) the backward pass is
//     x[P] = -[F[P,P] F[P,C]] [fr_f[P]; x[C]].
// Both products are skinny GEMMs (N = J members) computed by k_sgemm: a CTA
// owns 16 rows x 32 member columns, streams the factor rows through a
// two-stage cp.async pipeline in shared memory, and writes its rows exactly
// once (no atomics: bitwise-identical members stay identical).
#include "ens_internal.cuh"
#include "ens_mf_common.cuh"

__global__ void k_finit(MfDev d, int item0, const double* __restrict__ B, double* __restrict__ FR, int64_t N, int J,
                        int64_t nidx) {
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], r0 = it[1];
    const int mat = blockIdx.y;
    const int m = d.m[f], k = d.k[f];
    const int rows = min(ENS_VEC_ROWS, m - r0);
    const int64_t fo = d.idx_off[f];
    double* fr = FR + (int64_t)mat * nidx * J;
    const double* b = B + (int64_t)mat * N * J;
    for (int t = threadIdx.x; t < rows * J; t += blockDim.x) {
        const int i = r0 + t / J, j = t % J;
        fr[(fo + i) * J + j] = i < k ? b[(int64_t)d.idx[fo + i] * J + j] : 0.0;
    }
}

__global__ void k_fext(MfDev d, int item0, double* __restrict__ FR, int J, int64_t nidx) {
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int c = it[0], r0 = it[1];
    const int mat = blockIdx.y;
    const int p = d.parent[c];
    const int kc = d.k[c], cbn = d.m[c] - kc;
    const int rows = min(ENS_VEC_ROWS, cbn - r0);
    const int32_t* map = d.cmap + d.cmap_off[c];
    double* fr = FR + (int64_t)mat * nidx * J;
    const int64_t co = d.idx_off[c], po = d.idx_off[p];
    for (int t = threadIdx.x; t < rows * J; t += blockDim.x) {
        const int i = r0 + t / J, j = t % J;
        fr[(po + map[i]) * J + j] += fr[(co + kc + i) * J + j];
    }
}

__global__ void k_bgather(MfDev d, int item0, const double* __restrict__ X, double* __restrict__ FR, int64_t N, int J,
                          int64_t nidx) {
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], r0 = it[1];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int rows = min(ENS_VEC_ROWS, m - r0);
    const int64_t fo = d.idx_off[f];
    double* fr = FR + (int64_t)mat * nidx * J;
    const double* x = X + (int64_t)mat * N * J;
    for (int t = threadIdx.x; t < rows * J; t += blockDim.x) {
        const int i = r0 + t / J, j = t % J;
        fr[(fo + i) * J + j] = x[(int64_t)d.idx[fo + i] * J + j];
    }
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = pred ? 8 : 0;   // src-size 0 -> zero fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

#define SG_R 16     // rows per CTA
#define SG_C 32     // member columns per CTA
#define SG_K 64     // inner chunk
#define SG_T 128    // threads

// forward (bwd=0): fr[k+r0+i] -= sum_{t<k} F[k+r0+i][t] fr[t]
// backward (bwd=1): x[idx[r0+i]] = -sum_{t<m} F[r0+i][t] fr[t]
__global__ void __launch_bounds__(SG_T) k_sgemm(MfDev d, int item0, const double* __restrict__ F,
                                                double* __restrict__ FR, double* __restrict__ X, int64_t N, int J,
                                                int64_t nidx, int bwd) {
    __shared__ double As[2][SG_R][SG_K];
    __shared__ double Bs[2][SG_K][SG_C];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], r0 = it[1];
    const int mat = blockIdx.y;
    const int j0 = blockIdx.z * SG_C;
    const int jn = min(SG_C, J - j0);
    const int m = d.m[f], k = d.k[f];
    const int rbase = bwd ? r0 : k + r0;
    const int nr = min(SG_R, (bwd ? k : m) - rbase);
    const int K = bwd ? m : k;
    const double* base = F + (int64_t)mat * d.storage + d.off[f];
    double* fr = FR + (int64_t)mat * nidx * J + d.idx_off[f] * J;
    const int tid = threadIdx.x;
    const int nchunk = (K + SG_K - 1) / SG_K;

    auto load = [&](int stage, int t0) {
#pragma unroll
        for (int u = 0; u < (SG_R * SG_K) / SG_T; ++u) {
            const int e = tid + u * SG_T;
            const int r = e / SG_K, kk = e % SG_K;
            const bool ok = r < nr && t0 + kk < K;
            cp_async8(&As[stage][r][kk], ok ? base + (int64_t)(rbase + r) * m + t0 + kk : base, ok);
        }
#pragma unroll
        for (int u = 0; u < (SG_K * SG_C) / SG_T; ++u) {
            const int e = tid + u * SG_T;
            const int kk = e / SG_C, j = e % SG_C;
            const bool ok = t0 + kk < K && j < jn;
            cp_async8(&Bs[stage][kk][j], ok ? fr + (int64_t)(t0 + kk) * J + j0 + j : fr, ok);
        }
        cp_async_commit();
    };

    const int tx = tid & 15, ty = tid >> 4;   // cols tx, tx+16 ; rows ty, ty+8
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    if (nchunk > 0) load(0, 0);
    for (int c = 0; c < nchunk; ++c) {
        if (c + 1 < nchunk) {
            load((c + 1) & 1, (c + 1) * SG_K);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int st = c & 1;
#pragma unroll 8
        for (int kk = 0; kk < SG_K; ++kk) {
            const double a0 = As[st][ty][kk], a1 = As[st][ty + 8][kk];
            const double b0 = Bs[st][kk][tx], b1 = Bs[st][kk][tx + 16];
            acc[0][0] = fma(a0, b0, acc[0][0]);
            acc[0][1] = fma(a0, b1, acc[0][1]);
            acc[1][0] = fma(a1, b0, acc[1][0]);
            acc[1][1] = fma(a1, b1, acc[1][1]);
        }
        __syncthreads();
    }
    double* x = X + (int64_t)mat * N * J;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int r = ty + 8 * i;
        if (r >= nr) continue;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int j = tx + 16 * jj;
            if (j >= jn) continue;
            if (bwd)
                x[(int64_t)d.idx[d.idx_off[f] + rbase + r] * J + j0 + j] = -acc[i][jj];
            else
                fr[(int64_t)(rbase + r) * J + j0 + j] -= acc[i][jj];
        }
    }
}

int mf_solve(ens_ctx* c, cudaStream_t s, const double* r, double* z) {
    MfDev d = mfdev(c);
    const int J = c->J;
    const int64_t N = c->n_total, nidx = c->p.n_idx;
    const unsigned zc = (unsigned)((J + SG_C - 1) / SG_C);
    {
        const int rc = launch_copy_cons(c, s, r, z);
        if (rc != ENS_OK) return rc;
    }
    const int64_t nf = (int64_t)c->sched_fwd.size() / 5;
    for (int64_t i = 0; i < nf; ++i) {
        const int64_t* q = &c->sched_fwd[5 * i];
        const int op = (int)q[0], off = (int)q[2], n = (int)q[3];
        if (n == 0) continue;
        switch (op) {
            case SOP_FINIT:
                k_finit<<<dim3(n, 2), 256, 0, s>>>(d, off, r, c->frvec, N, J, nidx);
                break;
            case SOP_FEXT:
                k_fext<<<dim3(n, 2), 256, 0, s>>>(d, off, c->frvec, J, nidx);
                break;
            case SOP_FGEMM:
                k_sgemm<<<dim3(n, 2, zc), SG_T, 0, s>>>(d, off, c->fronts, c->frvec, z, N, J, nidx, 0);
                break;
            default:
                ens_set_error("bad fwd op", __FILE__, __LINE__);
                return ENS_EINVAL;
        }
        ENS_CKL();
    }
    const int64_t nb = (int64_t)c->sched_bwd.size() / 5;
    for (int64_t i = 0; i < nb; ++i) {
        const int64_t* q = &c->sched_bwd[5 * i];
        const int op = (int)q[0], off = (int)q[2], n = (int)q[3];
        if (n == 0) continue;
        switch (op) {
            case SOP_BGATHER:
                k_bgather<<<dim3(n, 2), 256, 0, s>>>(d, off, z, c->frvec, N, J, nidx);
                break;
            case SOP_BGEMM:
                k_sgemm<<<dim3(n, 2, zc), SG_T, 0, s>>>(d, off, c->fronts, c->frvec, z, N, J, nidx, 1);
                break;
            default:
                ens_set_error("bad bwd op", __FILE__, __LINE__);
                return ENS_EINVAL;
        }
        ENS_CKL();
    }
    return ENS_OK;
}
