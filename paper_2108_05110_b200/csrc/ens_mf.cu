// Multifrontal block-sweep factorisation of the two shared saddle matrices and
// the multi-column solves (sm_100a, fp64).  Symbolic structure and the launch
// schedule come from paper_2108_05110_b200/symbolic.py; this file executes it.
//
// Each front is a dense m x m row-major block whose first k rows/cols are its
// pivots.  For every panel P = [a, a+pw) of the pivots (the block-sweep /
// Gauss-Jordan step, Q = all front rows/cols outside P):
//   DIAG    F[P,P] <- -D^-1                 (D = F[P,P]; register Gauss-Jordan, in-panel pivoting)
//   HPANEL  F[P,Q] <- D^-1 F[P,Q]
//   UPDATE  F[Q,Q] <- F[Q,Q] - F[Q,P] F[P,Q]   (F[P,Q] already scaled)
//   GPANEL  F[Q,P] <- F[Q,P] D^-1
// After all panels the front holds [-F11^-1, F11^-1 F12; F21 F11^-1, S] with S
// the Schur complement (extend-added into the parent).  Solves are then one
// batched GEMM per tree level and direction:
//   forward  fr[C] -= F[C,P] fr[P]             backward  x[P] = -[F[P,P] F[P,C]] [fr[P]; x[C]]
#include <cmath>
#include <cstdlib>

#include "ens_internal.cuh"

#include "ens_mf_common.cuh"

// outside-panel index -> front row/col
__device__ __forceinline__ int outside(int r, int a, int pw) { return r < a ? r : r + pw; }

// ---------------------------------------------------------------------------
// assembly of the fronts (original entries, child contribution blocks)
// ---------------------------------------------------------------------------
__global__ void k_orig(const int64_t* __restrict__ dst, const int32_t* __restrict__ src, int64_t n0, int64_t n1,
                       const double* __restrict__ as_vals, int nnz, const double* __restrict__ bsrc,
                       double* __restrict__ F, int64_t storage) {
    const int64_t i = n0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n1) return;
    const int mat = blockIdx.y;
    const int s = src[i];
    const double v = s < nnz ? as_vals[(int64_t)mat * nnz + s] : bsrc[s - nnz];
    F[(int64_t)mat * storage + dst[i]] = v;
}

__global__ void k_extadd(MfDev d, int item0, double* __restrict__ F) {
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int c = it[0], r0 = it[1];
    const int mat = blockIdx.y;
    const int p = d.parent[c];
    const int kc = d.k[c], mc = d.m[c], mp = d.m[p];
    const int cbn = mc - kc;
    const int rows = min(ENS_EXT_ROWS, cbn - r0);
    const int32_t* map = d.cmap + d.cmap_off[c];
    const double* C = F + (int64_t)mat * d.storage + d.off[c];
    double* P = F + (int64_t)mat * d.storage + d.off[p];
    for (int t = threadIdx.x; t < rows * cbn; t += blockDim.x) {
        const int i = r0 + t / cbn, jj = t % cbn;
        P[(int64_t)map[i] * mp + map[jj]] += C[(int64_t)(kc + i) * mc + kc + jj];
    }
}

// ---------------------------------------------------------------------------
// DIAG: F[P,P] <- -D^-1.  In-place Gauss-Jordan held in registers (16x16
// threads, 4x4 elements each); partial pivoting without row swaps: the pivot
// row of column k is the unused row with the largest |a[r][k]|, and the
// inverse is recovered as A^-1[i][j] = a[piv[i]][ipiv[j]].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_diag(MfDev d, int item0, double* __restrict__ F, int32_t* __restrict__ npert) {
    __shared__ double s_col[2][ENS_PW];
    __shared__ double s_row[2][ENS_PW];
    __shared__ int s_piv[ENS_PW];
    __shared__ int s_ipiv[ENS_PW];
    __shared__ unsigned char s_used[ENS_PW];
    __shared__ double s_scale;
    __shared__ double s_out[ENS_PW][ENS_PW + 1];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a0 = it[1];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a0);
    double* Fb = F + (int64_t)mat * d.storage + d.off[f] + (int64_t)a0 * m + a0;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double a[4][4];
    double amax = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = ty + 16 * i, c = tx + 16 * j;
            double v = (r == c) ? 1.0 : 0.0;
            if (r < pw && c < pw) v = Fb[(int64_t)r * m + c];
            a[i][j] = v;
            if (r < pw && c < pw) amax = fmax(amax, fabs(v));
        }
    if (threadIdx.x < ENS_PW) s_used[threadIdx.x] = 0;
    // block max for the tiny-pivot threshold
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (threadIdx.x == 0) s_scale = 0.0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)&s_scale, (unsigned long long)__double_as_longlong(amax));
    __syncthreads();
    const double thr = 1e-14 * (s_scale > 0.0 ? s_scale : 1.0);
    for (int k = 0; k < pw; ++k) {
        const int buf = k & 1;
        // 1. column k to smem
        if (tx == (k & 15)) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int jj = k >> 4;
                double v = 0.0;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j == jj) v = a[i][j];
                s_col[buf][ty + 16 * i] = v;
            }
        }
        __syncthreads();
        // 2. pivot row: largest |a[r][k]| among unused rows r < pw
        if (threadIdx.x < 32) {
            double best = -1.0;
            int br = ENS_PW;
            for (int r = threadIdx.x; r < pw; r += 32) {
                if (s_used[r]) continue;
                const double v = fabs(s_col[buf][r]);
                if (v > best) {
                    best = v;
                    br = r;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int orr = __shfl_xor_sync(0xffffffffu, br, o);
                if (ob > best || (ob == best && orr < br)) {
                    best = ob;
                    br = orr;
                }
            }
            if (threadIdx.x == 0) {
                if (br >= pw) {        // NaN column: take the first unused row
                    for (int r = 0; r < pw; ++r)
                        if (!s_used[r]) {
                            br = r;
                            break;
                        }
                }
                if (!(best > thr)) {   // singular/tiny pivot: static perturbation, GMRES corrects it
                    s_col[buf][br] = (s_col[buf][br] < 0.0 ? -thr : thr);
                    atomicAdd(npert, 1);
                }
                s_used[br] = 1;
                s_piv[k] = br;
                s_ipiv[br] = k;
            }
        }
        __syncthreads();
        const int p = s_piv[k];
        // 3. pivot row to smem
        if (ty == (p & 15)) {
            const int ii = p >> 4;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                double v = 0.0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (i == ii) v = a[i][j];
                s_row[buf][tx + 16 * j] = v;
            }
        }
        __syncthreads();
        // 4. eliminate (pivot element of column k treated as 1, in-place inverse)
        const double inv = 1.0 / s_col[buf][p];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = tx + 16 * j;
            const double np = (c == k ? 1.0 : s_row[buf][c]) * inv;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = ty + 16 * i;
                if (r == p) {
                    a[i][j] = np;
                } else {
                    const double fr = s_col[buf][r];
                    a[i][j] = (c == k ? 0.0 : a[i][j]) - fr * np;
                }
            }
        }
    }
    // un-permute and store -D^-1
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s_out[ty + 16 * i][tx + 16 * j] = a[i][j];
    __syncthreads();
    for (int t = threadIdx.x; t < pw * pw; t += blockDim.x) {
        const int r = t / pw, c = t % pw;
        Fb[(int64_t)r * m + c] = -s_out[s_piv[r]][s_ipiv[c]];
    }
}

// ---------------------------------------------------------------------------
// register-tiled 64x64 (rows) x 64 (cols) GEMM piece from shared memory:
// acc[i][j] += sum_t A[ty+16i][t] * B[t][tx+16j]
// ---------------------------------------------------------------------------
#define LDA (ENS_TILE + 1)

__device__ __forceinline__ void tile_mma(const double* __restrict__ As, const double* __restrict__ Bs, int K,
                                         double acc[4][4], int tx, int ty) {
    // As: row-major [64][LDA] indexed As[r*LDA + t]; Bs: [K][64]
    for (int t = 0; t < K; ++t) {
        double av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[(ty + 16 * i) * LDA + t];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[t * ENS_TILE + tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
}

// HPANEL: F[P, Q-tile] <- D^-1 F[P, Q-tile]   (D^-1 = -F[P,P])
__global__ void __launch_bounds__(256) k_hpanel(MfDev d, int item0, double* __restrict__ F) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1], c0 = it[2];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int t = m - pw;
    const int nc = min(ENS_TILE, t - c0);
    double* Ds = sm;                       // [64][LDA]  (D^-1)
    double* Rs = sm + ENS_PW * LDA;        // [pw][64]
    double* base = F + (int64_t)mat * d.storage + d.off[f];
    for (int e = threadIdx.x; e < ENS_PW * ENS_PW; e += blockDim.x) {
        const int r = e / ENS_PW, cc = e % ENS_PW;
        Ds[r * LDA + cc] = (r < pw && cc < pw) ? -base[(int64_t)(a + r) * m + a + cc] : 0.0;
    }
    for (int e = threadIdx.x; e < pw * ENS_TILE; e += blockDim.x) {
        const int r = e / ENS_TILE, cc = e % ENS_TILE;
        Rs[e] = cc < nc ? base[(int64_t)(a + r) * m + outside(c0 + cc, a, pw)] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4] = {};
    tile_mma(Ds, Rs, pw, acc, tx, ty);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = ty + 16 * i;
        if (r >= pw) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int cc = tx + 16 * j;
            if (cc < nc) base[(int64_t)(a + r) * m + outside(c0 + cc, a, pw)] = acc[i][j];
        }
    }
}

// UPDATE: F[Q-rows, Q-cols] -= F[Q-rows, P] F[P, Q-cols]
__global__ void __launch_bounds__(256) k_update(MfDev d, int item0, double* __restrict__ F) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1], r0 = it[2], c0 = it[3];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int t = m - pw;
    const int nr = min(ENS_TILE, t - r0), nc = min(ENS_TILE, t - c0);
    double* Cs = sm;                       // [64][LDA]
    double* Hs = sm + ENS_TILE * LDA;      // [pw][64]
    double* base = F + (int64_t)mat * d.storage + d.off[f];
    for (int e = threadIdx.x; e < ENS_TILE * pw; e += blockDim.x) {
        const int r = e / pw, kk = e % pw;
        Cs[r * LDA + kk] = r < nr ? base[(int64_t)outside(r0 + r, a, pw) * m + a + kk] : 0.0;
    }
    for (int e = threadIdx.x; e < pw * ENS_TILE; e += blockDim.x) {
        const int kk = e / ENS_TILE, cc = e % ENS_TILE;
        Hs[e] = cc < nc ? base[(int64_t)(a + kk) * m + outside(c0 + cc, a, pw)] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4] = {};
    tile_mma(Cs, Hs, pw, acc, tx, ty);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = ty + 16 * i;
        if (r >= nr) continue;
        double* row = base + (int64_t)outside(r0 + r, a, pw) * m;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int cc = tx + 16 * j;
            if (cc < nc) {
                const int col = outside(c0 + cc, a, pw);
                row[col] -= acc[i][j];
            }
        }
    }
}

// GPANEL: F[Q-tile, P] <- F[Q-tile, P] D^-1
__global__ void __launch_bounds__(256) k_gpanel(MfDev d, int item0, double* __restrict__ F) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1], r0 = it[2];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int t = m - pw;
    const int nr = min(ENS_TILE, t - r0);
    double* Cs = sm;                       // [64][LDA]
    double* Ds = sm + ENS_TILE * LDA;      // [pw][64]  (D^-1)
    double* base = F + (int64_t)mat * d.storage + d.off[f];
    for (int e = threadIdx.x; e < ENS_TILE * pw; e += blockDim.x) {
        const int r = e / pw, kk = e % pw;
        Cs[r * LDA + kk] = r < nr ? base[(int64_t)outside(r0 + r, a, pw) * m + a + kk] : 0.0;
    }
    for (int e = threadIdx.x; e < pw * ENS_TILE; e += blockDim.x) {
        const int kk = e / ENS_TILE, cc = e % ENS_TILE;
        Ds[e] = cc < pw ? -base[(int64_t)(a + kk) * m + a + cc] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4] = {};
    tile_mma(Cs, Ds, pw, acc, tx, ty);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = ty + 16 * i;
        if (r >= nr) continue;
        double* row = base + (int64_t)outside(r0 + r, a, pw) * m + a;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int cc = tx + 16 * j;
            if (cc < pw) row[cc] = acc[i][j];
        }
    }
}

// ---------------------------------------------------------------------------
// host drivers
// ---------------------------------------------------------------------------
static const size_t SM_HP = sizeof(double) * (ENS_PW * LDA + ENS_PW * ENS_TILE);
static const size_t SM_UP = sizeof(double) * (ENS_TILE * LDA + ENS_PW * ENS_TILE);
static const size_t SM_GP = sizeof(double) * (ENS_TILE * LDA + ENS_PW * ENS_TILE);

int mf_setup(ens_ctx* c) {
    ENS_CK(cudaFuncSetAttribute(k_hpanel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_HP));
    ENS_CK(cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_UP));
    ENS_CK(cudaFuncSetAttribute(k_gpanel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_GP));
    (void)c;
    return ENS_OK;
}

static int mf_factor_launches(ens_ctx* c, cudaStream_t s, const double* as_vals, int64_t* nlaunch) {
    MfDev d = mfdev(c);
    const int64_t st = c->p.front_storage;
    int64_t cnt = 0;
    ENS_CK(cudaMemsetAsync(c->d_count, 0, sizeof(int32_t), s));
    const int64_t nrow = (int64_t)c->sched_factor.size() / 5;
    for (int64_t i = 0; i < nrow; ++i) {
        const int64_t* r = &c->sched_factor[5 * i];
        const int op = (int)r[0], L = (int)r[1], off = (int)r[2], n = (int)r[3];
        switch (op) {
            case OP_ZERO: {
                const int64_t a = c->level_storage_off[L], b = c->level_storage_off[L + 1];
                for (int mat = 0; mat < 2; ++mat)
                    ENS_CK(cudaMemsetAsync(c->fronts + mat * st + a, 0, sizeof(double) * (size_t)(b - a), s));
                continue;   // a memset, not a kernel launch
            }
            case OP_ORIG: {
                const int64_t a = c->orig_level_off[L], b = c->orig_level_off[L + 1];
                if (b <= a) continue;
                dim3 grid((unsigned)((b - a + 255) / 256), 2);
                k_orig<<<grid, 256, 0, s>>>(c->p.orig_dst, c->p.orig_src, a, b, as_vals, c->m.nnz_s,
                                            c->p.bsrc_vals, c->fronts, st);
                break;
            }
            case OP_EXTADD:
                k_extadd<<<dim3(n, 2), 256, 0, s>>>(d, off, c->fronts);
                break;
            case OP_DIAG:
                k_diag<<<dim3(n, 2), 256, 0, s>>>(d, off, c->fronts, c->d_count);
                break;
            case OP_HPANEL:
                k_hpanel<<<dim3(n, 2), 256, SM_HP, s>>>(d, off, c->fronts);
                break;
            case OP_UPDATE:
                k_update<<<dim3(n, 2), 256, SM_UP, s>>>(d, off, c->fronts);
                break;
            case OP_GPANEL:
                k_gpanel<<<dim3(n, 2), 256, SM_GP, s>>>(d, off, c->fronts);
                break;
            default:
                ens_set_error("bad factor op", __FILE__, __LINE__);
                return ENS_EINVAL;
        }
        ENS_CKL();
        ++cnt;
    }
    *nlaunch = cnt;
    return ENS_OK;
}

// The factorisation's launch sequence is fixed per mesh: capture it once into a
// CUDA graph (keyed on the value buffer) and replay it every sub-step.
int mf_factor(ens_ctx* c, cudaStream_t s, const double* as_vals, int32_t* n_pert) {
    const char* e = std::getenv("ENS_NO_GRAPH");
    const bool graphs = !(e && e[0] == '1') && s != 0;
    if (!graphs) {
        int64_t n = 0;
        const int rc = mf_factor_launches(c, s, as_vals, &n);
        if (rc != ENS_OK) return rc;
    } else {
        if (c->g_factor && c->g_factor_key != as_vals) {
            cudaGraphExecDestroy((cudaGraphExec_t)c->g_factor);
            c->g_factor = nullptr;
        }
        if (!c->g_factor) {
            cudaGraph_t g;
            ENS_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            int64_t n = 0;
            const int rc = mf_factor_launches(c, s, as_vals, &n);
            const cudaError_t ce = cudaStreamEndCapture(s, &g);
            if (rc != ENS_OK) return rc;
            ENS_CK(ce);
            ENS_CK(cudaGraphInstantiate((cudaGraphExec_t*)&c->g_factor, g, 0));
            cudaGraphDestroy(g);
            c->g_factor_key = as_vals;
            c->g_factor_kernels = n;
            g_ens_launches -= (unsigned long long)n;
        }
        ENS_CK(cudaGraphLaunch((cudaGraphExec_t)c->g_factor, s));
        g_ens_launches += (unsigned long long)c->g_factor_kernels;
    }
    if (n_pert) {
        ENS_CK(cudaMemcpyAsync(c->h_count, c->d_count, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        ENS_CK(cudaStreamSynchronize(s));
        *n_pert = c->h_count[0];
    }
    return ENS_OK;
}

