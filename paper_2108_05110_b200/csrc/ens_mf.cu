// Multifrontal LU of the two shared saddle matrices + multi-column triangular
// solves (sm_100a, fp64).  Symbolic structure and the launch schedule come from
// paper_2108_05110_b200/symbolic.py; this file executes it.
//
// Per front (dense m x m, row-major) and per panel [a, b) of its pivots:
//   DIAG    D  <- D^-1                      (Gauss-Jordan, partial pivoting in-panel)
//   HPANEL  R  <- H = -D^-1 R               (rows a..b, cols b..m)
//   UPDATE  T  <- T + C H                   (rows/cols b..m; C = cols a..b, rows b..m)
//   GPANEL  C  <- G = -C D^-1
// The trailing T of the last panel is the contribution block, extend-added into
// the parent front.  Solves use the stored (D^-1, H, G) directly:
//   forward:  fr[b:m] += G fr[a:b]           backward: x[a:b] = D^-1 fr[a:b] + H x[b:m]
// which equals forward/backward substitution with the block LU factors.
#include <cmath>

#include "ens_internal.cuh"

enum { OP_ZERO = 0, OP_ORIG, OP_EXTADD, OP_DIAG, OP_HPANEL, OP_UPDATE, OP_GPANEL };
enum { SOP_FINIT = 0, SOP_FEXT, SOP_FPANEL, SOP_BGATHER, SOP_BPANEL, SOP_BSCATTER };

struct MfDev {
    const int32_t* m;
    const int32_t* k;
    const int64_t* off;
    const int64_t* idx_off;
    const int32_t* idx;
    const int32_t* parent;
    const int64_t* cmap_off;
    const int32_t* cmap;
    const int32_t* work;
    int64_t storage;
};

static MfDev mfdev(const ens_ctx* c) {
    MfDev d;
    d.m = c->p.f_m;
    d.k = c->p.f_k;
    d.off = c->p.f_off;
    d.idx_off = c->p.f_idx_off;
    d.idx = c->p.f_idx;
    d.parent = c->p.f_parent;
    d.cmap_off = c->p.f_cmap_off;
    d.cmap = c->p.f_cmap;
    d.work = c->p.work;
    d.storage = c->p.front_storage;
    return d;
}

// ---------------------------------------------------------------------------
// factorisation kernels; grid = (items, 2 matrices)
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

// D^-1 by Gauss-Jordan with partial pivoting inside the panel (augmented [D | I])
__global__ void __launch_bounds__(256) k_diag(MfDev d, int item0, double* __restrict__ F, int32_t* __restrict__ npert) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int W = 2 * pw;
    double* A = sm;                      // pw x W
    double* fac = sm + pw * W;           // pw
    __shared__ int s_piv;
    __shared__ double s_scale;
    double* Fb = F + (int64_t)mat * d.storage + d.off[f] + (int64_t)a * m + a;
    for (int t = threadIdx.x; t < pw * W; t += blockDim.x) {
        const int r = t / W, cc = t % W;
        A[t] = cc < pw ? Fb[(int64_t)r * m + cc] : (cc - pw == r ? 1.0 : 0.0);
    }
    __syncthreads();
    if (threadIdx.x < 32) {   // block scale for the tiny-pivot threshold
        double mx = 0.0;
        for (int t = threadIdx.x; t < pw * pw; t += 32) mx = fmax(mx, fabs(A[(t / pw) * W + t % pw]));
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (threadIdx.x == 0) s_scale = mx;
    }
    __syncthreads();
    for (int col = 0; col < pw; ++col) {
        if (threadIdx.x < 32) {
            double best = -1.0;
            int br = col;
            for (int r = col + threadIdx.x; r < pw; r += 32) {
                const double v = fabs(A[r * W + col]);
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
                s_piv = br;
                const double thr = 1e-14 * (s_scale > 0.0 ? s_scale : 1.0);
                if (!(best > thr)) {   // singular / tiny pivot: static perturbation, GMRES corrects it
                    A[br * W + col] = (A[br * W + col] < 0.0 ? -thr : thr);
                    atomicAdd(npert, 1);
                }
            }
        }
        __syncthreads();
        const int pr = s_piv;
        if (pr != col) {
            for (int cc = threadIdx.x; cc < W; cc += blockDim.x) {
                const double t0 = A[col * W + cc];
                A[col * W + cc] = A[pr * W + cc];
                A[pr * W + cc] = t0;
            }
        }
        __syncthreads();
        const double inv = 1.0 / A[col * W + col];
        for (int r = threadIdx.x; r < pw; r += blockDim.x) fac[r] = A[r * W + col];
        __syncthreads();
        for (int cc = threadIdx.x; cc < W; cc += blockDim.x) A[col * W + cc] *= inv;
        __syncthreads();
        for (int t = threadIdx.x; t < pw * W; t += blockDim.x) {
            const int r = t / W, cc = t % W;
            if (r != col) A[t] -= fac[r] * A[col * W + cc];
        }
        __syncthreads();
    }
    for (int t = threadIdx.x; t < pw * pw; t += blockDim.x) {
        const int r = t / pw, cc = t % pw;
        Fb[(int64_t)r * m + cc] = A[r * W + pw + cc];
    }
}

// H = -D^-1 R for a 64-column tile of R (in place)
__global__ void __launch_bounds__(256) k_hpanel(MfDev d, int item0, double* __restrict__ F) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1], c0 = it[2];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int b = a + pw;
    const int nc = min(ENS_TILE, m - b - c0);
    double* Ds = sm;                       // pw x pw
    double* Rs = sm + ENS_PW * ENS_PW;     // pw x 64
    double* base = F + (int64_t)mat * d.storage + d.off[f];
    for (int t = threadIdx.x; t < pw * pw; t += blockDim.x) Ds[t] = base[(int64_t)(a + t / pw) * m + a + t % pw];
    for (int t = threadIdx.x; t < pw * ENS_TILE; t += blockDim.x) {
        const int r = t / ENS_TILE, cc = t % ENS_TILE;
        Rs[t] = cc < nc ? base[(int64_t)(a + r) * m + b + c0 + cc] : 0.0;
    }
    __syncthreads();
    const int cc = threadIdx.x % ENS_TILE;
    for (int i = threadIdx.x / ENS_TILE; i < pw; i += blockDim.x / ENS_TILE) {
        double acc = 0.0;
        for (int t = 0; t < pw; ++t) acc += Ds[i * pw + t] * Rs[t * ENS_TILE + cc];
        if (cc < nc) base[(int64_t)(a + i) * m + b + c0 + cc] = -acc;
    }
}

// T += C H on a 64x64 tile (K = pw)
__global__ void __launch_bounds__(256) k_update(MfDev d, int item0, double* __restrict__ F) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1], r0 = it[2], c0 = it[3];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int b = a + pw;
    const int nr = min(ENS_TILE, m - b - r0), nc = min(ENS_TILE, m - b - c0);
    const int LD = ENS_TILE + 1;
    double* Cs = sm;                     // pw x LD  (transposed C tile)
    double* Hs = sm + ENS_PW * LD;       // pw x 64
    double* base = F + (int64_t)mat * d.storage + d.off[f];
    for (int t = threadIdx.x; t < ENS_TILE * pw; t += blockDim.x) {
        const int r = t / pw, kk = t % pw;
        Cs[kk * LD + r] = r < nr ? base[(int64_t)(b + r0 + r) * m + a + kk] : 0.0;
    }
    for (int t = threadIdx.x; t < pw * ENS_TILE; t += blockDim.x) {
        const int kk = t / ENS_TILE, cc = t % ENS_TILE;
        Hs[t] = cc < nc ? base[(int64_t)(a + kk) * m + b + c0 + cc] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
    for (int kk = 0; kk < pw; ++kk) {
        double av[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) av[u] = Cs[kk * LD + ty + 16 * u];
#pragma unroll
        for (int v = 0; v < 4; ++v) bv[v] = Hs[kk * ENS_TILE + tx + 16 * v];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int r = ty + 16 * u;
        if (r >= nr) continue;
        double* row = base + (int64_t)(b + r0 + r) * m + b + c0;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int cc = tx + 16 * v;
            if (cc < nc) row[cc] += acc[u][v];
        }
    }
}

// G = -C D^-1 for a 64-row tile of C (in place)
__global__ void __launch_bounds__(256) k_gpanel(MfDev d, int item0, double* __restrict__ F) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1], r0 = it[2];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int b = a + pw;
    const int nr = min(ENS_TILE, m - b - r0);
    double* Ds = sm;                       // pw x pw
    double* Cs = sm + ENS_PW * ENS_PW;     // 64 x pw
    double* base = F + (int64_t)mat * d.storage + d.off[f];
    for (int t = threadIdx.x; t < pw * pw; t += blockDim.x) Ds[t] = base[(int64_t)(a + t / pw) * m + a + t % pw];
    for (int t = threadIdx.x; t < ENS_TILE * pw; t += blockDim.x) {
        const int r = t / pw, kk = t % pw;
        Cs[t] = r < nr ? base[(int64_t)(b + r0 + r) * m + a + kk] : 0.0;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nr * pw; t += blockDim.x) {
        const int r = t / pw, cc = t % pw;
        double acc = 0.0;
        for (int kk = 0; kk < pw; ++kk) acc += Cs[r * pw + kk] * Ds[kk * pw + cc];
        base[(int64_t)(b + r0 + r) * m + a + cc] = -acc;
    }
}

// ---------------------------------------------------------------------------
// solve kernels: grid = (items, 2 matrices, column chunks of 64)
// ---------------------------------------------------------------------------
#define SJT 64

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

// fr[b+r0 .. +64] += G[rows, a:b] fr[a:b]
__global__ void __launch_bounds__(256) k_fpanel(MfDev d, int item0, const double* __restrict__ F,
                                                double* __restrict__ FR, int J, int64_t nidx) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1], r0 = it[2];
    const int mat = blockIdx.y;
    const int j0 = blockIdx.z * SJT;
    const int jn = min(SJT, J - j0);
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int b = a + pw;
    const int nr = min(ENS_TILE, m - b - r0);
    const double* base = F + (int64_t)mat * d.storage + d.off[f];
    double* fr = FR + (int64_t)mat * nidx * J + d.idx_off[f] * J;
    double* Gs = sm;                   // 64 x pw
    double* Xs = sm + ENS_TILE * ENS_PW;   // pw x SJT
    for (int t = threadIdx.x; t < nr * pw; t += blockDim.x) {
        const int r = t / pw, kk = t % pw;
        Gs[r * pw + kk] = base[(int64_t)(b + r0 + r) * m + a + kk];
    }
    for (int t = threadIdx.x; t < pw * jn; t += blockDim.x) {
        const int kk = t / jn, j = t % jn;
        Xs[kk * SJT + j] = fr[(int64_t)(a + kk) * J + j0 + j];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nr * jn; t += blockDim.x) {
        const int r = t / jn, j = t % jn;
        double acc = 0.0;
        for (int kk = 0; kk < pw; ++kk) acc += Gs[r * pw + kk] * Xs[kk * SJT + j];
        fr[(int64_t)(b + r0 + r) * J + j0 + j] += acc;
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

// x[a:b] = [D^-1 H] fr[a:m]   (in place into fr[a:b])
__global__ void __launch_bounds__(256) k_bpanel(MfDev d, int item0, const double* __restrict__ F,
                                                double* __restrict__ FR, int J, int64_t nidx) {
    extern __shared__ double sm[];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1];
    const int mat = blockIdx.y;
    const int j0 = blockIdx.z * SJT;
    const int jn = min(SJT, J - j0);
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const double* base = F + (int64_t)mat * d.storage + d.off[f];
    double* fr = FR + (int64_t)mat * nidx * J + d.idx_off[f] * J;
    double* As = sm;                         // pw x 64 (row-chunk of [D^-1 H])
    double* Xs = sm + ENS_PW * ENS_TILE;     // 64 x SJT
    const int nout = pw * jn;
    double acc[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc[u] = 0.0;
    for (int c0 = a; c0 < m; c0 += ENS_TILE) {
        const int kc = min(ENS_TILE, m - c0);
        __syncthreads();
        for (int t = threadIdx.x; t < pw * ENS_TILE; t += blockDim.x) {
            const int r = t / ENS_TILE, kk = t % ENS_TILE;
            As[t] = kk < kc ? base[(int64_t)(a + r) * m + c0 + kk] : 0.0;
        }
        for (int t = threadIdx.x; t < ENS_TILE * SJT; t += blockDim.x) {
            const int kk = t / SJT, j = t % SJT;
            Xs[t] = (kk < kc && j < jn) ? fr[(int64_t)(c0 + kk) * J + j0 + j] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int o = threadIdx.x + u * 256;
            if (o < nout) {
                const int r = o / jn, j = o % jn;
                double s = 0.0;
                for (int kk = 0; kk < kc; ++kk) s += As[r * ENS_TILE + kk] * Xs[kk * SJT + j];
                acc[u] += s;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const int o = threadIdx.x + u * 256;
        if (o < nout) {
            const int r = o / jn, j = o % jn;
            fr[(int64_t)(a + r) * J + j0 + j] = acc[u];
        }
    }
}

__global__ void k_bscatter(MfDev d, int item0, const double* __restrict__ FR, double* __restrict__ X, int64_t N, int J,
                           int64_t nidx) {
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], r0 = it[1];
    const int mat = blockIdx.y;
    const int k = d.k[f];
    const int rows = min(ENS_VEC_ROWS, k - r0);
    const int64_t fo = d.idx_off[f];
    const double* fr = FR + (int64_t)mat * nidx * J;
    double* x = X + (int64_t)mat * N * J;
    for (int t = threadIdx.x; t < rows * J; t += blockDim.x) {
        const int i = r0 + t / J, j = t % J;
        x[(int64_t)d.idx[fo + i] * J + j] = fr[(fo + i) * J + j];
    }
}

// ---------------------------------------------------------------------------
// host drivers
// ---------------------------------------------------------------------------
static const size_t SM_DIAG = sizeof(double) * (ENS_PW * 2 * ENS_PW + ENS_PW);
static const size_t SM_HP = sizeof(double) * (ENS_PW * ENS_PW + ENS_PW * ENS_TILE);
static const size_t SM_UP = sizeof(double) * (ENS_PW * (ENS_TILE + 1) + ENS_PW * ENS_TILE);
static const size_t SM_GP = sizeof(double) * (ENS_PW * ENS_PW + ENS_TILE * ENS_PW);
static const size_t SM_FP = sizeof(double) * (ENS_TILE * ENS_PW + ENS_PW * SJT);
static const size_t SM_BP = sizeof(double) * (ENS_PW * ENS_TILE + ENS_TILE * SJT);

int mf_setup(ens_ctx* c) {
    ENS_CK(cudaFuncSetAttribute(k_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_DIAG));
    ENS_CK(cudaFuncSetAttribute(k_hpanel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_HP));
    ENS_CK(cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_UP));
    ENS_CK(cudaFuncSetAttribute(k_gpanel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_GP));
    ENS_CK(cudaFuncSetAttribute(k_fpanel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_FP));
    ENS_CK(cudaFuncSetAttribute(k_bpanel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_BP));
    (void)c;
    return ENS_OK;
}

int mf_factor(ens_ctx* c, cudaStream_t s, const double* as_vals, int32_t* n_pert) {
    MfDev d = mfdev(c);
    const int64_t st = c->p.front_storage;
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
                k_diag<<<dim3(n, 2), 256, SM_DIAG, s>>>(d, off, c->fronts, c->d_count);
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
    }
    if (n_pert) {
        ENS_CK(cudaMemcpyAsync(c->h_count, c->d_count, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        ENS_CK(cudaStreamSynchronize(s));
        *n_pert = c->h_count[0];
    }
    return ENS_OK;
}

int mf_solve(ens_ctx* c, cudaStream_t s, const double* r, double* z) {
    MfDev d = mfdev(c);
    const int J = c->J;
    const int64_t N = c->n_total, nidx = c->p.n_idx;
    const unsigned zc = (unsigned)((J + SJT - 1) / SJT);
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
            case SOP_FPANEL:
                k_fpanel<<<dim3(n, 2, zc), 256, SM_FP, s>>>(d, off, c->fronts, c->frvec, J, nidx);
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
            case SOP_BPANEL:
                k_bpanel<<<dim3(n, 2, zc), 256, SM_BP, s>>>(d, off, c->fronts, c->frvec, J, nidx);
                break;
            case SOP_BSCATTER:
                k_bscatter<<<dim3(n, 2), 256, 0, s>>>(d, off, c->frvec, z, N, J, nidx);
                break;
            default:
                ens_set_error("bad bwd op", __FILE__, __LINE__);
                return ENS_EINVAL;
        }
        ENS_CKL();
    }
    return ENS_OK;
}
