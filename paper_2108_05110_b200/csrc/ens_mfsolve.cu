// Multi-column solves with the block-sweep fronts (sm_100a, fp64).
//
// After ens_mf.cu's sweep each front holds [-F11^-1, F11^-1 F12; F21 F11^-1, S].
// Forward, one launch per tree level (leaves -> root):
//     fr[P] = b[P] + children's contribution rows           (gathered in-kernel)
//     fr[C] = children's contribution rows - F[C,P] fr[P]
// Backward, one launch per level (root -> leaves):
//     x[P]  = -[F[P,P] F[P,C]] [fr[P]; x[C]]                (x[C] read from the iterate)
// The products are skinny GEMMs (N = J members).  A CTA owns 64 rows x 32
// member columns over an inner range of <= split_k, staged in shared memory
// with one cp.async group (shared memory sized per launch from the level's
// largest inner range, so leaf levels run many CTAs per SM).  Long inner
// dimensions are split into items that store partial products; the last CTA of
// a group to finish (atomic ticket) sums them in a fixed order -- deterministic,
// so bitwise-identical members stay identical.
//
// The whole solve is captured once into a CUDA graph; the in/out blocks are
// passed through a 2-pointer device table so the graph serves every Krylov vector.
#include <cstdlib>

#include "ens_internal.cuh"
#include "ens_mf_common.cuh"

struct SolveIO {
    const double* r;
    double* z;
};

__global__ void k_set_io(SolveIO* io, const double* r, double* z) {
    io->r = r;
    io->z = z;
}

// identity rows: z[cons] = r[cons]
__global__ void k_copy_cons_io(const int32_t* __restrict__ crow, int ncons, const SolveIO* __restrict__ io, int64_t N,
                               int J) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)ncons * J;
    if (t >= 2 * per) return;
    const int mat = (int)(t / per);
    const int64_t u = t - mat * per;
    const int64_t idx = (int64_t)mat * N * J + (int64_t)crow[u / J] * J + (u % J);
    io->z[idx] = io->r[idx];
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = pred ? 8 : 0;   // src-size 0 -> zero fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

#define SG_R 64     // rows per CTA (= symbolic.SOLVE_ROWS)
#define SG_C 32     // member columns per CTA
#define SG_KMAX 128 // max inner range per work item (>= symbolic.SPLIT_K)
#define SG_T 256    // threads
#define SG_LDB 36   // Bs row stride (= 4 mod 16)

__device__ __forceinline__ void dmma8(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// children's contribution rows mapped onto front row `row` (+ b at pivots)
__device__ __forceinline__ double gather_row(const MfDev& d, const double* __restrict__ FRm,
                                             const double* __restrict__ b, int64_t row, int J, int j, bool pivot) {
    double v = pivot ? b[(int64_t)d.idx[row] * J + j] : 0.0;
    const int32_t* g = d.gsrc + 4 * row;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int32_t src = g[s];
        if (src >= 0) v += FRm[(int64_t)src * J + j];
    }
    return v;
}

// item = (f, r0, ks, slot)
//   r0 = -1 : forward pivot-only item (front without contribution block)
//   slot<0  : whole inner range, result applied here
//   slot>=0 : inner range [ks*split_k, ...) of group s0 = slot - ks; the last
//             CTA of the group reduces partial[s0 .. s0+ns) in order
__global__ void __launch_bounds__(SG_T) k_sgemm(MfDev d, int item0, const double* __restrict__ F,
                                                double* __restrict__ FR, const SolveIO* __restrict__ io, int64_t N,
                                                int J, int64_t nidx, int bwd, int split_k, int kmax,
                                                double* __restrict__ partial, int* __restrict__ ticket,
                                                int64_t nslot) {
    extern __shared__ double sm[];
    __shared__ int s_last;
    // strides = 4 (mod 16) doubles: conflict-free m8n8k4 fragment reads
    const int lda = ((kmax + 15) & ~15) + 4;
    double* As = sm;                          // [SG_R][lda]
    double* Bs = sm + SG_R * lda;             // [kpad][SG_LDB]
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], r0 = it[1], ks = it[2], slot = it[3];
    const int mat = blockIdx.y;
    const int j0 = blockIdx.z * SG_C;
    const int jn = min(SG_C, J - j0);
    const int m = d.m[f], k = d.k[f];
    const int64_t fo = d.idx_off[f];
    const double* base = F + (int64_t)mat * d.storage + d.off[f];
    double* FRm = FR + (int64_t)mat * nidx * J;
    double* fr = FRm + fo * J;
    const double* b = io->r + (int64_t)mat * N * J;
    double* x = io->z + (int64_t)mat * N * J;
    const int tid = threadIdx.x;
    double init[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    if (!bwd && r0 < 0) {   // pivot rows [t0, t0+64) of a front without contribution block
        const int t0 = -1 - r0, t1 = min(k, t0 + SG_R);
        for (int e = tid; e < (t1 - t0) * SG_C; e += SG_T) {
            const int t = t0 + e / SG_C, j = e % SG_C;
            if (j < jn) fr[(int64_t)t * J + j0 + j] = gather_row(d, FRm, b, fo + t, J, j0 + j, true);
        }
        return;
    }
    const int rbase = bwd ? r0 : k + r0;
    const int nr = min(SG_R, (bwd ? k : m) - rbase);
    const int K = bwd ? m : k;
    const int kbeg = slot < 0 ? 0 : ks * split_k;
    const int kend = slot < 0 ? K : min(K, kbeg + split_k);
    const int kc = kend - kbeg;               // <= kmax by construction of the schedule
    // stage A rows (consecutive lanes -> consecutive inner index: coalesced, conflict-free)
    for (int e = tid; e < SG_R * kc; e += SG_T) {
        const int r = e / kc, kk = e % kc;
        const bool ok = r < nr;
        cp_async8(&As[r * lda + kk], ok ? base + (int64_t)(rbase + r) * m + kbeg + kk : base, ok);
    }
    if (bwd) {
        const int j = tid & (SG_C - 1);
        const bool jok = j < jn;
        for (int kb4 = tid / SG_C; kb4 < kc; kb4 += 4 * (SG_T / SG_C)) {
            int ix[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {   // descriptors first: 4 independent index loads in flight
                const int t = kbeg + kb4 + u * (SG_T / SG_C);
                ix[u] = (kb4 + u * (SG_T / SG_C) < kc && t >= k) ? d.idx[fo + t] : -1;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int kk = kb4 + u * (SG_T / SG_C);
                if (kk >= kc) continue;
                const int t = kbeg + kk;
                const double* src = fr;
                if (jok) src = (t < k) ? fr + (int64_t)t * J + j0 + j : x + (int64_t)ix[u] * J + j0 + j;
                cp_async8(&Bs[kk * SG_LDB + j], src, jok);
            }
        }
        cp_async_commit();
    } else {
        cp_async_commit();
        // contribution-block rows' children sums for the epilogue (non-split items):
        // issued first so these loads overlap the pivot gather below
        if (slot < 0) {
            const int tx_ = tid & 15, ty_ = tid >> 4;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = ty_ + 16 * i;
                const int4 g = (r < nr) ? *reinterpret_cast<const int4*>(d.gsrc + 4 * (fo + rbase + r))
                                        : make_int4(-1, -1, -1, -1);
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    const int j = j0 + tx_ + 16 * jj;
                    const bool jok = tx_ + 16 * jj < jn;
                    double v = 0.0;
                    if (jok && g.x >= 0) v += FRm[(int64_t)g.x * J + j];
                    if (jok && g.y >= 0) v += FRm[(int64_t)g.y * J + j];
                    if (jok && g.z >= 0) v += FRm[(int64_t)g.z * J + j];
                    if (jok && g.w >= 0) v += FRm[(int64_t)g.w * J + j];
                    init[i][jj] = v;
                }
            }
        }
        const bool store_piv = (r0 == 0);     // one row tile per front persists fr[P] for the backward pass
        // gather b + children rows; 4 rows per thread in flight (descriptors first, then values)
        const int j = tid & (SG_C - 1);
        const bool jok = j < jn;
        for (int kb4 = tid / SG_C; kb4 < kc; kb4 += 4 * (SG_T / SG_C)) {
            int4 g[4];
            int ix[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int kk = kb4 + u * (SG_T / SG_C);
                const int64_t row = fo + kbeg + kk;
                const bool ok = kk < kc;
                g[u] = ok ? *reinterpret_cast<const int4*>(d.gsrc + 4 * row) : make_int4(-1, -1, -1, -1);
                ix[u] = ok ? d.idx[row] : -1;
            }
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                v[u] = (jok && ix[u] >= 0) ? b[(int64_t)ix[u] * J + j0 + j] : 0.0;
                if (jok && g[u].x >= 0) v[u] += FRm[(int64_t)g[u].x * J + j0 + j];
                if (jok && g[u].y >= 0) v[u] += FRm[(int64_t)g[u].y * J + j0 + j];
                if (jok && g[u].z >= 0) v[u] += FRm[(int64_t)g[u].z * J + j0 + j];
                if (jok && g[u].w >= 0) v[u] += FRm[(int64_t)g[u].w * J + j0 + j];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int kk = kb4 + u * (SG_T / SG_C);
                if (kk >= kc) continue;
                Bs[kk * SG_LDB + j] = v[u];
                if (store_piv && jok) fr[(int64_t)(kbeg + kk) * J + j0 + j] = v[u];
            }
        }
    }
    // zero the K padding (kc -> multiple of 4) of both operands
    const int kpad = (kc + 3) & ~3;
    for (int e = tid; e < (kpad - kc) * SG_R; e += SG_T) As[(e % SG_R) * lda + kc + e / SG_R] = 0.0;
    for (int e = tid; e < (kpad - kc) * SG_C; e += SG_T) Bs[(kc + e / SG_C) * SG_LDB + e % SG_C] = 0.0;
    cp_async_wait_all();
    __syncthreads();
    // fp64 tensor-core MMA (m8n8k4): warp w owns rows 8w..8w+7, all 8-column tiles
    const int lane = tid & 31, warp = tid >> 5, g = lane >> 2, q = lane & 3;
    const int nct = (jn + 7) >> 3;
    double dacc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    {
        const double* ap = As + (8 * warp + g) * lda + q;
        const double* bp = Bs + q * SG_LDB + g;
        for (int k0 = 0; k0 < kpad; k0 += 4) {
            const double av = ap[k0];
#pragma unroll
            for (int ct = 0; ct < 4; ++ct)
                if (ct < nct) dmma8(dacc[ct][0], dacc[ct][1], av, bp[k0 * SG_LDB + 8 * ct]);
        }
    }
    __syncthreads();   // operands consumed: reuse As as the 64 x 32 output tile
    double* Cs = As;
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) {
        Cs[(8 * warp + g) * (SG_C + 1) + 8 * ct + 2 * q] = dacc[ct][0];
        Cs[(8 * warp + g) * (SG_C + 1) + 8 * ct + 2 * q + 1] = dacc[ct][1];
    }
    __syncthreads();
    const int tx = tid & 15, ty = tid >> 4;   // epilogue mapping: cols tx, tx+16 ; rows ty + 16 i
    double acc[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        acc[i][0] = Cs[(ty + 16 * i) * (SG_C + 1) + tx];
        acc[i][1] = Cs[(ty + 16 * i) * (SG_C + 1) + tx + 16];
    }
    if (slot < 0) {
        if (bwd) {
            int ix[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) ix[i] = (ty + 16 * i < nr) ? d.idx[fo + rbase + ty + 16 * i] : 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (ty + 16 * i >= nr) continue;
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    const int j = tx + 16 * jj;
                    if (j < jn) x[(int64_t)ix[i] * J + j0 + j] = -acc[i][jj];
                }
            }
        } else {
            // contribution-block rows: children's rows (gathered up front) minus the product
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = ty + 16 * i;
                if (r >= nr) continue;
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    const int j = tx + 16 * jj;
                    if (j < jn) FRm[(fo + rbase + r) * J + j0 + j] = init[i][jj] - acc[i][jj];
                }
            }
        }
        return;
    }
    // split: publish the partial, the last CTA of the group reduces in ks order
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = ty + 16 * i;
        if (r >= nr) continue;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int j = tx + 16 * jj;
            if (j < jn) partial[(((int64_t)mat * nslot + slot) * SG_R + r) * J + j0 + j] = acc[i][jj];
        }
    }
    __threadfence();
    __syncthreads();
    const int s0 = slot - ks;
    const int ns = (K + split_k - 1) / split_k;
    const int tk = (int)(((int64_t)mat * nslot + s0) * gridDim.z + blockIdx.z);
    if (tid == 0) s_last = (atomicAdd(ticket + tk, 1) == ns - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int e = tid; e < nr * jn; e += SG_T) {
        const int r = e / jn, j = e % jn;
        double sum = 0.0;
        for (int q = 0; q < ns; ++q) sum += __ldcg(&partial[(((int64_t)mat * nslot + s0 + q) * SG_R + r) * J + j0 + j]);
        if (bwd) {
            x[(int64_t)d.idx[fo + rbase + r] * J + j0 + j] = -sum;
        } else {
            const int64_t row = fo + rbase + r;
            FRm[row * J + j0 + j] = gather_row(d, FRm, b, row, J, j0 + j, false) - sum;
        }
    }
    if (tid == 0) ticket[tk] = 0;   // ready for the next solve / graph replay
}

static size_t sg_smem(int kmax) {
    const size_t lda = ((kmax + 15) & ~15) + 4, kpad = (kmax + 3) & ~3;
    const size_t ops = SG_R * lda + kpad * SG_LDB, out = SG_R * (SG_C + 1);   // output tile reuses the operands
    return sizeof(double) * (ops > out ? ops : out);
}

// record the launch sequence of one solve (io table fixed)
static int mf_solve_launches(ens_ctx* c, cudaStream_t s, SolveIO* io, int64_t* nlaunch) {
    MfDev d = mfdev(c);
    const int J = c->J;
    const int64_t N = c->n_total, nidx = c->p.n_idx;
    const unsigned zc = (unsigned)((J + SG_C - 1) / SG_C);
    const int sk = c->p.split_k;
    const int64_t nslot = c->p.n_slot;
    int64_t cnt = 0;
    if (c->m.ncons > 0) {
        const int64_t tot = 2LL * c->m.ncons * J;
        k_copy_cons_io<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(c->m.cons_row, c->m.ncons, io, N, J);
        ENS_CKL();
        ++cnt;
    }
    for (const std::vector<int64_t>* sched : {&c->sched_fwd, &c->sched_bwd}) {
        const int64_t nrow = (int64_t)sched->size() / 5;
        for (int64_t i = 0; i < nrow; ++i) {
            const int64_t* q = &(*sched)[5 * i];
            const int op = (int)q[0], off = (int)q[2], n = (int)q[3], kmax = (int)q[4];
            if (n == 0) continue;
            if ((op != SOP_FGEMM && op != SOP_BGEMM) || kmax > SG_KMAX || kmax < 1) {
                ens_set_error("bad solve schedule row", __FILE__, __LINE__);
                return ENS_EINVAL;
            }
            k_sgemm<<<dim3(n, 2, zc), SG_T, sg_smem(kmax), s>>>(d, off, c->fronts, c->frvec, io, N, J, nidx,
                                                               op == SOP_BGEMM, sk, kmax, c->partial, c->ticket,
                                                               nslot);
            ENS_CKL();
            ++cnt;
        }
    }
    *nlaunch = cnt;
    return ENS_OK;
}

static bool graphs_enabled() {
    const char* e = std::getenv("ENS_NO_GRAPH");
    return !(e && e[0] == '1');
}

int mf_solve(ens_ctx* c, cudaStream_t s, const double* r, double* z) {
    if (!c->solve_io) {
        if (c->p.split_k > SG_KMAX) {
            ens_set_error("plan split_k exceeds the solve kernel's inner tile", __FILE__, __LINE__);
            return ENS_EINVAL;
        }
        ENS_CK(cudaMalloc(&c->solve_io, sizeof(SolveIO)));
        ENS_CK(cudaFuncSetAttribute(k_sgemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sg_smem(SG_KMAX)));
        const int64_t ns = c->p.n_slot > 0 ? c->p.n_slot : 1;
        const size_t pbytes = sizeof(double) * 2 * (size_t)ns * SG_R * c->J;
        const size_t tbytes = sizeof(int) * 2 * (size_t)ns * ((c->J + SG_C - 1) / SG_C);
        if (cudaMalloc(&c->partial, pbytes) != cudaSuccess || cudaMalloc(&c->ticket, tbytes) != cudaSuccess) {
            ens_set_error("out of device memory for split-K partials", __FILE__, __LINE__);
            return ENS_ENOMEM;
        }
        ENS_CK(cudaMemset(c->ticket, 0, tbytes));
        c->ws_bytes += pbytes + tbytes;
    }
    SolveIO* io = (SolveIO*)c->solve_io;
    k_set_io<<<1, 1, 0, s>>>(io, r, z);
    ENS_CKL();
    if (!graphs_enabled() || s == 0) {
        int64_t n = 0;
        return mf_solve_launches(c, s, io, &n);
    }
    if (!c->g_solve) {
        cudaGraph_t g;
        ENS_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        int64_t n = 0;
        const int rc = mf_solve_launches(c, s, io, &n);
        const cudaError_t e = cudaStreamEndCapture(s, &g);
        if (rc != ENS_OK) return rc;
        ENS_CK(e);
        ENS_CK(cudaGraphInstantiate((cudaGraphExec_t*)&c->g_solve, g, 0));
        cudaGraphDestroy(g);
        c->g_solve_kernels = n;
        g_ens_launches -= (unsigned long long)n;   // counted again at every replay below
    }
    ENS_CK(cudaGraphLaunch((cudaGraphExec_t)c->g_solve, s));
    g_ens_launches += (unsigned long long)c->g_solve_kernels;
    return ENS_OK;
}
