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
#include <vector>
#include <algorithm>

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
    // 2 barriers per elimination step: (A) column k+1 published by its owners right
    // after their update; (B) every warp finds the pivot row redundantly from smem
    // (no serial section), then the pivot row's owners publish it.
    __shared__ double s_col[2][ENS_PW];
    __shared__ double s_row[2][ENS_PW];
    __shared__ int s_piv[ENS_PW];
    __shared__ int s_ipiv[ENS_PW];
    __shared__ unsigned char s_used[2][ENS_PW];
    __shared__ double s_wmax[8];
    __shared__ double s_out[ENS_PW][ENS_PW + 1];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a0 = it[1];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a0);
    double* Fb = F + (int64_t)mat * d.storage + d.off[f] + (int64_t)a0 * m + a0;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) s_wmax[warp] = amax;
    if (threadIdx.x < ENS_PW) s_used[0][threadIdx.x] = s_used[1][threadIdx.x] = 0;
    // publish column 0
    if (tx == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) s_col[0][ty + 16 * i] = a[i][0];
    }
    __syncthreads();
    double scale = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) scale = fmax(scale, s_wmax[w]);
    const double thr = 1e-14 * (scale > 0.0 ? scale : 1.0);
    int pert = 0;
    for (int k = 0; k < pw; ++k) {
        const int buf = k & 1;
        // (B) pivot search, redundantly in every warp: rows lane, lane+32
        double best = -1.0;
        int br = ENS_PW;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = lane + 32 * h;
            if (r < pw && !s_used[buf][r]) {
                const double v = fabs(s_col[buf][r]);
                if (v > best) {
                    best = v;
                    br = r;
                }
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
        if (br >= pw) {   // NaN column: first unused row
            for (int r = 0; r < pw; ++r)
                if (!s_used[buf][r]) {
                    br = r;
                    break;
                }
        }
        const int p = br;
        double piv = s_col[buf][p];
        if (!(best > thr)) {   // tiny pivot: static perturbation (FGMRES corrects it)
            piv = piv < 0.0 ? -thr : thr;
            pert = 1;
        }
        if (threadIdx.x < ENS_PW) s_used[buf ^ 1][threadIdx.x] = s_used[buf][threadIdx.x] | (threadIdx.x == p);
        if (threadIdx.x == 0) {
            s_piv[k] = p;
            s_ipiv[p] = k;
        }
        if (ty == (p & 15)) {   // publish row p
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
        // update (pivot element of column k treated as 1: in-place inverse)
        const double inv = 1.0 / piv;
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
        // (A) publish column k+1 into the other buffer
        if (k + 1 < pw && tx == ((k + 1) & 15)) {
            const int jj = (k + 1) >> 4;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                double v = 0.0;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (j == jj) v = a[i][j];
                s_col[buf ^ 1][ty + 16 * i] = v;
            }
        }
        __syncthreads();
    }
    if (pert && threadIdx.x == 0) atomicAdd(npert, 1);
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

// DIAG without pivoting (default): the symbolic ordering (velocities before pressures, pressures moved
// above all their velocity neighbours) makes every leading block of a panel nonsingular, so the
// in-place Gauss-Jordan can take the diagonal pivots; a pivot below 1e-14 x max|D| is perturbed and
// counted, and the host then refactorises with the pivoting kernel (k_diag).
// Blocked: 8 x 8 blocks on the fp64 tensor cores.  Warp w keeps row block w (8 x 64) in registers in the DMMA accumulator layout
// (lane (g, q): row g, columns 8 j + 2 q + {0, 1}) through all 8 block steps.  Block step k:
//   pivot warp k : P = A[k,k]^-1 by scalar Gauss-Jordan in registers (warp shuffles; pivots below
//                  1e-14 x max|D| perturbed and counted), then its new row block
//                  R = P A[k,:] (block k of it: P itself) by DMMA, published in shared memory;
//   other warps i: A[i,j] -= A[i,k] R[j] (j != k), A[i,k] = -A[i,k] P -- one rank-8 DMMA update of
//                  the warp's registers (the A[i,k] fragment comes from the accumulator layout by
//                  shuffles).
// One CTA barrier per block step (R double-buffered): 18 us per panel instead of the 36 us of 64
// scalar steps with a barrier each (round 1).
#define DB_LD 68
__device__ __forceinline__ void up_mma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}
__device__ __forceinline__ double db_shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
// 1 / x for a pivot (|x| >= the perturbation threshold, finite): hardware seed + three Newton steps.
// The division is on the serial path of every scalar pivot step, IEEE division costs ~10x this.
__device__ __forceinline__ double db_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    r = fma(fma(-x, r, 1.0), r, r);
    r = fma(fma(-x, r, 1.0), r, r);
    r = fma(fma(-x, r, 1.0), r, r);
    return r;
}

__global__ void __launch_bounds__(256) k_diag_blk(MfDev d, int item0, double* __restrict__ F,
                                                  int32_t* __restrict__ npert) {
    __shared__ __align__(16) double s_R[2][8 * DB_LD];
    __shared__ __align__(16) double s_P[8 * 12];   // the pivot block's inverse as the A operand of R = P A[k,:]
    __shared__ double s_wmax[8];
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a0 = it[1];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a0);
    double* Fb = F + (int64_t)mat * d.storage + d.off[f] + (int64_t)a0 * m + a0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
    const int row = 8 * warp + g;
    double acc[8][2];
    double amax = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int c = 8 * j + 2 * q + e;
            double v = (row == c) ? 1.0 : 0.0;
            if (row < pw && c < pw) {
                v = Fb[(int64_t)row * m + c];
                amax = fmax(amax, fabs(v));
            }
            acc[j][e] = v;
        }
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) s_wmax[warp] = amax;
    __syncthreads();
    double scale = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) scale = fmax(scale, s_wmax[w]);
    const double thr = 1e-14 * (scale > 0.0 ? scale : 1.0);
    int pert = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        double* R = s_R[k & 1];
        if (warp == k) {
            // old row block -> shared memory (the B operand of R = P A[k,:])
#pragma unroll
            for (int j = 0; j < 8; ++j)
                *reinterpret_cast<double2*>(&R[g * DB_LD + 8 * j + 2 * q]) = make_double2(acc[j][0], acc[j][1]);
            // P = A[k,k]^-1 in registers: b0 = B[g][2q], b1 = B[g][2q+1]
            double b0 = acc[k][0], b1 = acc[k][1];
#pragma unroll
            for (int s2 = 0; s2 < 8; ++s2) {
                const int hs = s2 >> 1, od = s2 & 1;
                double piv = db_shfl(od ? b1 : b0, 4 * s2 + hs);
                if (!(fabs(piv) > thr)) {
                    piv = piv < 0.0 ? -thr : thr;
                    pert = 1;
                }
                const double inv = db_rcp(piv);
                const double r0 = db_shfl(b0, 4 * s2 + q) * inv, r1 = db_shfl(b1, 4 * s2 + q) * inv;   // row s2 / piv
                const double cs = db_shfl(od ? b1 : b0, 4 * g + hs);                                  // B[g][s2]
                const bool c0 = (2 * q == s2), c1 = (2 * q + 1 == s2);                              // my column s2?
                if (g == s2) {
                    b0 = c0 ? inv : r0;
                    b1 = c1 ? inv : r1;
                } else {
                    b0 = c0 ? -cs * inv : b0 - cs * r0;
                    b1 = c1 ? -cs * inv : b1 - cs * r1;
                }
            }
            __syncwarp();
            *reinterpret_cast<double2*>(&s_P[g * 12 + 2 * q]) = make_double2(b0, b1);
            __syncwarp();
            double nr[8][2];
#pragma unroll
            for (int j = 0; j < 8; ++j) nr[j][0] = nr[j][1] = 0.0;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const double av = s_P[g * 12 + 4 * u + q];
#pragma unroll
                for (int j = 0; j < 8; ++j) up_mma(nr[j][0], nr[j][1], av, R[(4 * u + q) * DB_LD + 8 * j + g]);
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                acc[j][0] = j == k ? b0 : nr[j][0];
                acc[j][1] = j == k ? b1 : nr[j][1];
                *reinterpret_cast<double2*>(&R[g * DB_LD + 8 * j + 2 * q]) = make_double2(acc[j][0], acc[j][1]);
            }
        }
        __syncthreads();
        if (warp != k) {
            // -A[i,k] as the A operand (row g, columns 4 u + q) from the accumulator layout
            double av[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int c = 4 * u + q, src = 4 * g + (c >> 1);
                const double x0 = db_shfl(acc[k][0], src), x1 = db_shfl(acc[k][1], src);
                av[u] = -((c & 1) ? x1 : x0);
            }
            acc[k][0] = acc[k][1] = 0.0;
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int j = 0; j < 8; ++j) up_mma(acc[j][0], acc[j][1], av[u], R[(4 * u + q) * DB_LD + 8 * j + g]);
        }
    }
    pert = __syncthreads_or(pert);
    if (pert && threadIdx.x == 0) atomicAdd(npert, 1);
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int c = 8 * j + 2 * q + e;
            if (row < pw && c < pw) Fb[(int64_t)row * m + c] = -acc[j][e];
        }
}

// UPDATE on the fp64 tensor cores with one asynchronous staging round trip:
// the output tile C (64 x 64, rows/cols outside the panel) is prefetched into the
// accumulator fragments while A = F[Q-rows, P] and B = F[P, Q-cols] stream into
// shared memory by cp.async (zero-filled past the panel width); then
// C += (-A) B with mma.sync m8n8k4 (warp w: rows 8w..8w+7, all 8 column tiles)
// and C is stored straight from the fragments.
#define UP_LD 68   // = 4 (mod 16) doubles: conflict-free m8n8k4 fragment reads
__device__ __forceinline__ void up_cp16(double* sdst, const double* g, bool pred) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void up_cp8(double* sdst, const double* g, bool pred) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(pred ? 8 : 0));
}

__global__ void __launch_bounds__(256, 3) k_update2(MfDev d, int item0, double* __restrict__ F,
                                                    const double* __restrict__ colp, int f0, int64_t prow) {
    extern __shared__ double sm[];
    double* As = sm;                    // [64 rows][UP_LD]   A[r][k]
    double* Bs = sm + 64 * UP_LD;       // [64 k][UP_LD]      B[k][c]
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], a = it[1], r0 = it[2], c0 = it[3];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int t = m - pw;
    const int nr = min(ENS_TILE, t - r0), nc = min(ENS_TILE, t - c0);
    double* base = F + (int64_t)mat * d.storage + d.off[f];
    // A = the UNSCALED column panel F[Q-rows, P], saved row by row (64 doubles, zero past the panel
    // width) by the panel kernel before it scaled the panel in place
    const double* ap0 = colp + ((int64_t)mat * prow + (d.idx_off[f] - d.idx_off[f0]) + r0) * ENS_PW;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
    // (1) operands -> shared memory (one commit group); row r = e >> 6, inner kk = e & 63
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int e = tid + 256 * i, r = e >> 5, kk = (e & 31) * 2;
        const bool ok = r < nr;
        up_cp16(&As[r * UP_LD + kk], ok ? ap0 + (int64_t)r * ENS_PW + kk : colp, ok);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int e = tid + 256 * i, kk = e >> 6, cc = e & 63;
        const bool ok = kk < pw && cc < nc;
        up_cp8(&Bs[kk * UP_LD + cc], ok ? base + (int64_t)(a + kk) * m + outside(c0 + cc, a, pw) : base, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::);
    // (2) C fragments (row 8w+g, cols 8ct + 2q + {0,1}) in flight meanwhile
    const int row = 8 * warp + g;
    const bool row_ok = row < nr;
    double* crow = base + (int64_t)outside(r0 + (row_ok ? row : 0), a, pw) * m;
    double acc[8][2];
#pragma unroll
    for (int ct = 0; ct < 8; ++ct)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int cc = 8 * ct + 2 * q + e;
            acc[ct][e] = (row_ok && cc < nc) ? crow[outside(c0 + cc, a, pw)] : 0.0;
        }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    // (3) C -= A B
    const double* ap = As + row * UP_LD + q;
    const double* bp = Bs + q * UP_LD + g;
    const int ksteps = (pw + 3) >> 2;
#pragma unroll 4
    for (int u = 0; u < ksteps; ++u) {
        const double av = -ap[4 * u];
#pragma unroll
        for (int ct = 0; ct < 8; ++ct) up_mma(acc[ct][0], acc[ct][1], av, bp[4 * u * UP_LD + 8 * ct]);
    }
    // (4) store
    if (!row_ok) return;
#pragma unroll
    for (int ct = 0; ct < 8; ++ct)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int cc = 8 * ct + 2 * q + e;
            if (cc < nc) crow[outside(c0 + cc, a, pw)] = acc[ct][e];
        }
}
static const size_t SM_UP2 = sizeof(double) * 2 * 64 * UP_LD;

// HPANEL and GPANEL in one launch (same staging + tensor-core pattern as the update; in place: the
// operand being overwritten is staged completely before any store).  Blocks [0, nH) scale a tile of
// the row panel, the rest a tile of the column panel:
//   HPANEL: F[P, Q-tile] <- (-F[P,P]) F[P, Q-tile]      (D^-1 = -F[P,P])
//   GPANEL: F[Q-tile, P] <- F[Q-tile, P] (-F[P,P])      and the UNSCALED tile is saved to colp for
//           the update, which follows (round 1 ran GPANEL as a fourth launch after the update)
__global__ void __launch_bounds__(256, 3) k_panel_hg(MfDev d, int offH, int nH, int offG, double* __restrict__ F,
                                                     double* __restrict__ colp, int f0, int64_t prow) {
    extern __shared__ double sm[];
    double* As = sm;                    // [64][UP_LD]
    double* Bs = sm + 64 * UP_LD;       // [64][UP_LD]
    const bool H = (int)blockIdx.x < nH;
    const int* it = d.work + 4LL * (H ? offH + blockIdx.x : offG + (blockIdx.x - nH));
    const int f = it[0], a = it[1], x0 = it[2];
    const int mat = blockIdx.y;
    const int m = d.m[f];
    const int pw = min(ENS_PW, d.k[f] - a);
    const int t = m - pw;
    const int nx = min(ENS_TILE, t - x0);          // HPANEL: tile columns, GPANEL: tile rows
    double* base = F + (int64_t)mat * d.storage + d.off[f];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int e = tid + 256 * i, r = e >> 6, cc = e & 63;
        // D = F[P,P] (A of HPANEL, B of GPANEL)
        const bool okd = r < pw && cc < pw;
        up_cp8(&(H ? As : Bs)[r * UP_LD + cc], okd ? base + (int64_t)(a + r) * m + a + cc : base, okd);
        if (H) {   // B = F[P, Q-tile]: rows r < pw, cols cc < nx
            const bool ok = r < pw && cc < nx;
            up_cp8(&Bs[r * UP_LD + cc], ok ? base + (int64_t)(a + r) * m + outside(x0 + cc, a, pw) : base, ok);
        } else {   // A = F[Q-tile, P]: rows r < nx, cols cc < pw
            const bool ok = r < nx && cc < pw;
            up_cp8(&As[r * UP_LD + cc], ok ? base + (int64_t)outside(x0 + r, a, pw) * m + a + cc : base, ok);
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    if (!H) {   // the unscaled tile, row by row (zero past the panel width), for the update
        double* cp = colp + ((int64_t)mat * prow + (d.idx_off[f] - d.idx_off[f0]) + x0) * ENS_PW;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e = tid + 256 * i, r = e >> 5, cc = (e & 31) * 2;
            if (r < nx)
                *reinterpret_cast<double2*>(cp + (int64_t)r * ENS_PW + cc) =
                    make_double2(As[r * UP_LD + cc], As[r * UP_LD + cc + 1]);
        }
    }
    const int row = 8 * warp + g;
    const double* ap = As + row * UP_LD + q;
    const double* bp = Bs + q * UP_LD + g;
    double acc[8][2];
#pragma unroll
    for (int ct = 0; ct < 8; ++ct) acc[ct][0] = acc[ct][1] = 0.0;
    const int ksteps = (pw + 3) >> 2;
#pragma unroll 4
    for (int u = 0; u < ksteps; ++u) {
        const double av = -ap[4 * u];   // one operand is -F[P,P]: negate A (HPANEL) ...
#pragma unroll
        for (int ct = 0; ct < 8; ++ct) {
            const double bv = bp[4 * u * UP_LD + 8 * ct];
            up_mma(acc[ct][0], acc[ct][1], H ? av : -av, H ? bv : -bv);   // ... or B (GPANEL)
        }
    }
    const int nrow = H ? pw : nx, ncol = H ? nx : pw;
    if (row >= nrow) return;
#pragma unroll
    for (int ct = 0; ct < 8; ++ct)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int cc = 8 * ct + 2 * q + e;
            if (cc >= ncol) continue;
            if (H)
                base[(int64_t)(a + row) * m + outside(x0 + cc, a, pw)] = acc[ct][e];
            else
                base[(int64_t)outside(x0 + row, a, pw) * m + a + cc] = acc[ct][e];
        }
}


// ---------------------------------------------------------------------------
// host drivers
// ---------------------------------------------------------------------------
int mf_setup(ens_ctx* c) {
    (void)c;
    ENS_CK(cudaFuncSetAttribute(k_update2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_UP2));
    ENS_CK(cudaFuncSetAttribute(k_panel_hg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_UP2));
    return ENS_OK;
}

static int mf_factor_launches(ens_ctx* c, cudaStream_t s, const double* as_vals, int64_t* nlaunch) {
    MfDev d = mfdev(c);
    const int64_t st = c->p.front_storage;
    int64_t cnt = 0;
    ENS_CK(cudaMemsetAsync(c->d_count, 0, sizeof(int32_t), s));
    const int64_t nrow = (int64_t)c->sched_factor.size() / 5;
    std::vector<char> done((size_t)nrow, 0);
    bool zeroed = false;
    for (int64_t i = 0; i < nrow; ++i) {
        const int64_t* r = &c->sched_factor[5 * i];
        const int op = (int)r[0], L = (int)r[1], off = (int)r[2], n = (int)r[3];
        switch (op) {
            case OP_ZERO: {
                // the level ranges are disjoint and only ever accumulated into after their own zeroing,
                // so the first OP_ZERO clears every level of both systems at once (one memset instead
                // of two per level when the levels tile the storage)
                if (zeroed) continue;
                zeroed = true;
                const int64_t top = c->level_storage_off.back();
                if (top == st) {
                    ENS_CK(cudaMemsetAsync(c->fronts, 0, sizeof(double) * (size_t)(2 * st), s));
                } else {
                    for (int mat = 0; mat < 2; ++mat)
                        ENS_CK(cudaMemsetAsync(c->fronts + mat * st, 0, sizeof(double) * (size_t)top, s));
                }
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
                if (c->diag_pivot)
                    k_diag<<<dim3(n, 2), 256, 0, s>>>(d, off, c->fronts, c->d_count);
                else
                    k_diag_blk<<<dim3(n, 2), 256, 0, s>>>(d, off, c->fronts, c->d_count);
                break;
            case OP_HPANEL: {
                // the panel step's GPANEL row (scheduled after the update in the plan) runs in the same
                // launch: the update reads the unscaled column panel from colp instead
                int64_t j = i + 1;
                while (j < nrow && !((int)c->sched_factor[5 * j] == OP_GPANEL && (int)c->sched_factor[5 * j + 1] == L)) ++j;
                if (j >= nrow) {
                    ens_set_error("factor schedule: HPANEL without its GPANEL", __FILE__, __LINE__);
                    return ENS_EINVAL;
                }
                const int offG = (int)c->sched_factor[5 * j + 2], nG = (int)c->sched_factor[5 * j + 3];
                done[j] = 1;
                k_panel_hg<<<dim3(n + nG, 2), 256, SM_UP2, s>>>(d, off, n, offG, c->fronts, c->colpanel,
                                                              c->level_front_off[L], c->colpanel_rows);
                break;
            }
            case OP_UPDATE:
                k_update2<<<dim3(n, 2), 256, SM_UP2, s>>>(d, off, c->fronts, c->colpanel, c->level_front_off[L],
                                                          c->colpanel_rows);
                break;
            case OP_GPANEL:
                if (done[i]) continue;   // (ran with its HPANEL)
                ens_set_error("factor schedule: GPANEL without an HPANEL before it", __FILE__, __LINE__);
                return ENS_EINVAL;
            default:
                ens_set_error("bad factor op", __FILE__, __LINE__);
                return ENS_EINVAL;
        }
        ENS_CKL();
        ++cnt;
    }
    {   // streamed solve: factor entries re-laid out per work tile (ens_mfsolve.cu)
        const int rc = mf_stream_pack(c, s);
        if (rc != ENS_OK) return rc;
        if (c->stiles) ++cnt;
    }
    *nlaunch = cnt;
    return ENS_OK;
}

// The factorisation's launch sequence is fixed per mesh: capture it once into a
// CUDA graph (keyed on the value buffer) and replay it every sub-step.
int mf_factor(ens_ctx* c, cudaStream_t s, const double* as_vals, int32_t* n_pert) {
    {
        const int rc = mf_stream_prepare(c);   // allocations happen outside any graph capture
        if (rc != ENS_OK) return rc;
    }
    if (!c->colpanel) {
        // unscaled column panels of one panel step of one level: a row of ENS_PW doubles per front row
        const int nf = (int)c->p.nfront;
        std::vector<int64_t> io((size_t)nf + 1);
        ENS_CK(cudaMemcpy(io.data(), c->p.f_idx_off, sizeof(int64_t) * (nf + 1), cudaMemcpyDeviceToHost));
        int64_t rows = 1;
        for (size_t L = 0; L + 1 < c->level_front_off.size(); ++L)
            rows = std::max(rows, io[c->level_front_off[L + 1]] - io[c->level_front_off[L]]);
        const size_t bytes = sizeof(double) * 2 * (size_t)rows * ENS_PW;
        if (cudaMalloc(&c->colpanel, bytes) != cudaSuccess) {
            cudaGetLastError();
            ens_set_error("out of device memory for the factorisation's column panels", __FILE__, __LINE__);
            return ENS_ENOMEM;
        }
        ENS_CK(cudaMemset(c->colpanel, 0, bytes));
        c->colpanel_rows = rows;
        c->ws_bytes += bytes;
    }
    const char* e = std::getenv("ENS_NO_GRAPH");
    const bool graphs = !(e && e[0] == '1') && s != 0;
    if (!graphs) {
        int64_t n = 0;
        const int rc = mf_factor_launches(c, s, as_vals, &n);
        if (rc != ENS_OK) return rc;
    } else {
        // two cached graphs: time loops that announce their steps keep two sets of assembled values
        // (one per state-buffer parity), and the graph is bound to the value buffer it was captured on
        if (c->g_factor && (c->g_factor_key != as_vals || c->g_factor_pivot != c->diag_pivot)) {
            std::swap(c->g_factor, c->g_factor_alt);
            std::swap(c->g_factor_key, c->g_factor_key_alt);
            std::swap(c->g_factor_pivot, c->g_factor_pivot_alt);
            if (c->g_factor && (c->g_factor_key != as_vals || c->g_factor_pivot != c->diag_pivot)) {
                cudaGraphExecDestroy((cudaGraphExec_t)c->g_factor);
                c->g_factor = nullptr;
            }
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
            c->g_factor_pivot = c->diag_pivot;
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

