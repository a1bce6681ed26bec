// Multi-column solves with the block-sweep fronts (sm_100a, fp64).
//
// After ens_mf.cu's sweep each front holds [-F11^-1, F11^-1 F12; F21 F11^-1, S].
// Forward, per tree level (leaves -> root):
//     FINIT  fr_f = [b(pivots); 0] + the children's contribution rows (one gather pass)
//     FGEMM  fr_f[C] -= F[C,P] fr_f[P]
// Backward, per level (root -> leaves):
//     BGEMM  x[P] = -[F[P,P] F[P,C]] [fr_f[P]; x[C]]   (x[C] read straight from the iterate)
// The products are skinny GEMMs (N = J members).  A CTA owns 64 rows x 32
// member columns over an inner range of <= split_k (128) staged in shared
// memory with one cp.async group.  Long inner
// dimensions (top of the tree) are split into independent items whose partial
// products land in scratch slots and are summed in a fixed order by *RED
// (deterministic, no atomics: bitwise-identical members stay identical).
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

__global__ void k_finit(MfDev d, int item0, const SolveIO* __restrict__ io, double* __restrict__ FR, int64_t N, int J,
                        int64_t nidx) {
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], r0 = it[1];
    const int mat = blockIdx.y;
    const int m = d.m[f], k = d.k[f];
    const int rows = min(ENS_VEC_ROWS, m - r0);
    const int64_t fo = d.idx_off[f];
    double* fr = FR + (int64_t)mat * nidx * J;
    const double* b = io->r + (int64_t)mat * N * J;
    for (int t = threadIdx.x; t < rows * J; t += blockDim.x) {
        const int i = r0 + t / J, j = t % J;
        const int64_t row = fo + i;
        double v = i < k ? b[(int64_t)d.idx[row] * J + j] : 0.0;
        const int32_t* g = d.gsrc + 4 * row;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int32_t src = g[s];
            if (src >= 0) v += fr[(int64_t)src * J + j];
        }
        fr[row * J + j] = v;
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

#define SG_R 64     // rows per CTA (= symbolic.SOLVE_ROWS)
#define SG_C 32     // member columns per CTA
#define SG_KMAX 128 // max inner range per work item (= symbolic.SPLIT_K)
#define SG_T 256    // threads
#define SG_LDA (SG_KMAX + 1)

// forward (bwd=0): fr[k+r0+i] -= sum_{t<k} F[k+r0+i][t] fr[t]
// backward (bwd=1): x[idx[r0+i]] = -sum_{t<m} F[r0+i][t] (t < k ? fr[t] : x[idx[t]])
// item = (f, r0, ks, slot): slot < 0 -> whole inner range (<= SG_KMAX), result applied here;
//                          slot >= 0 -> range [ks*split_k, ...), product stored to partial[slot]
// The whole inner range is staged at once (one cp.async group): rows are
// row-major with a +1 pad so both the async writes and the compute reads are
// bank-conflict free.
__global__ void __launch_bounds__(SG_T) k_sgemm(MfDev d, int item0, const double* __restrict__ F,
                                                double* __restrict__ FR, const SolveIO* __restrict__ io, int64_t N,
                                                int J, int64_t nidx, int bwd, int split_k,
                                                double* __restrict__ partial, int64_t nslot) {
    extern __shared__ double sm[];
    double* As = sm;                          // [SG_R][SG_LDA]
    double* Bs = sm + SG_R * SG_LDA;          // [SG_KMAX][SG_C]
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], r0 = it[1], ks = it[2], slot = it[3];
    const int mat = blockIdx.y;
    const int j0 = blockIdx.z * SG_C;
    const int jn = min(SG_C, J - j0);
    const int m = d.m[f], k = d.k[f];
    const int rbase = bwd ? r0 : k + r0;
    const int nr = min(SG_R, (bwd ? k : m) - rbase);
    const int K = bwd ? m : k;
    const int kbeg = slot < 0 ? 0 : ks * split_k;
    const int kend = slot < 0 ? K : min(K, kbeg + split_k);
    const int kc = kend - kbeg;               // <= SG_KMAX by construction of the schedule
    const double* base = F + (int64_t)mat * d.storage + d.off[f];
    const int64_t fo = d.idx_off[f];
    double* fr = FR + (int64_t)mat * nidx * J + fo * J;
    double* x = io->z + (int64_t)mat * N * J;
    const int tid = threadIdx.x;
    // stage A rows (consecutive lanes -> consecutive inner index: coalesced, conflict-free)
    for (int e = tid; e < SG_R * SG_KMAX; e += SG_T) {
        const int r = e / SG_KMAX, kk = e % SG_KMAX;
        if (kk >= kc) continue;
        const bool ok = r < nr;
        cp_async8(&As[r * SG_LDA + kk], ok ? base + (int64_t)(rbase + r) * m + kbeg + kk : base, ok);
    }
    for (int e = tid; e < SG_KMAX * SG_C; e += SG_T) {
        const int kk = e / SG_C, j = e % SG_C;
        if (kk >= kc) continue;
        const int t = kbeg + kk;
        const bool ok = j < jn;
        const double* src = fr;
        if (ok) src = (t < k) ? fr + (int64_t)t * J + j0 + j : x + (int64_t)d.idx[fo + t] * J + j0 + j;
        cp_async8(&Bs[kk * SG_C + j], src, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const int tx = tid & 15, ty = tid >> 4;   // cols tx, tx+16 ; rows ty + 16 i
    double acc[4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < kc; ++kk) {
        double a[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[(ty + 16 * i) * SG_LDA + kk];
        const double b0 = Bs[kk * SG_C + tx], b1 = Bs[kk * SG_C + tx + 16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            acc[i][0] = fma(a[i], b0, acc[i][0]);
            acc[i][1] = fma(a[i], b1, acc[i][1]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = ty + 16 * i;
        if (r >= nr) continue;
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int j = tx + 16 * jj;
            if (j >= jn) continue;
            if (slot >= 0)
                partial[(((int64_t)mat * nslot + slot) * SG_R + r) * J + j0 + j] = acc[i][jj];
            else if (bwd)
                x[(int64_t)d.idx[fo + rbase + r] * J + j0 + j] = -acc[i][jj];
            else
                fr[(int64_t)(rbase + r) * J + j0 + j] -= acc[i][jj];
        }
    }
}

static const size_t SM_SG = sizeof(double) * (SG_R * SG_LDA + SG_KMAX * SG_C);
// ordered sum of the split-K partials + the update; item = (f, r0, nsplit, slot0)
__global__ void k_sred(MfDev d, int item0, double* __restrict__ FR, const SolveIO* __restrict__ io, int64_t N, int J,
                       int64_t nidx, int bwd, const double* __restrict__ partial, int64_t nslot) {
    const int* it = d.work + 4LL * (item0 + blockIdx.x);
    const int f = it[0], r0 = it[1], ns = it[2], s0 = it[3];
    const int mat = blockIdx.y;
    const int m = d.m[f], k = d.k[f];
    const int rbase = bwd ? r0 : k + r0;
    const int nr = min(SG_R, (bwd ? k : m) - rbase);
    const int64_t fo = d.idx_off[f];
    double* fr = FR + (int64_t)mat * nidx * J + fo * J;
    double* x = io->z + (int64_t)mat * N * J;
    for (int t = threadIdx.x; t < nr * J; t += blockDim.x) {
        const int r = t / J, j = t % J;
        double s = 0.0;
        for (int q = 0; q < ns; ++q) s += partial[(((int64_t)mat * nslot + s0 + q) * SG_R + r) * J + j];
        if (bwd)
            x[(int64_t)d.idx[fo + rbase + r] * J + j] = -s;
        else
            fr[(int64_t)(rbase + r) * J + j] -= s;
    }
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
            const int op = (int)q[0], off = (int)q[2], n = (int)q[3];
            if (n == 0) continue;
            switch (op) {
                case SOP_FINIT:
                    k_finit<<<dim3(n, 2), 256, 0, s>>>(d, off, io, c->frvec, N, J, nidx);
                    break;
                case SOP_FGEMM:
                case SOP_BGEMM:
                    k_sgemm<<<dim3(n, 2, zc), SG_T, SM_SG, s>>>(d, off, c->fronts, c->frvec, io, N, J, nidx,
                                                            op == SOP_BGEMM, sk, c->partial, nslot);
                    break;
                case SOP_FRED:
                case SOP_BRED:
                    k_sred<<<dim3(n, 2), 256, 0, s>>>(d, off, c->frvec, io, N, J, nidx, op == SOP_BRED, c->partial,
                                                      nslot);
                    break;
                default:
                    ens_set_error("bad solve op", __FILE__, __LINE__);
                    return ENS_EINVAL;
            }
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
        ENS_CK(cudaMalloc(&c->solve_io, sizeof(SolveIO)));
        ENS_CK(cudaFuncSetAttribute(k_sgemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_SG));
        if (c->p.split_k > SG_KMAX) {
            ens_set_error("plan split_k exceeds the solve kernel's inner tile", __FILE__, __LINE__);
            return ENS_EINVAL;
        }
    }
    if (!c->partial && c->p.n_slot > 0) {
        const size_t bytes = sizeof(double) * 2 * (size_t)c->p.n_slot * SG_R * c->J;
        if (cudaMalloc(&c->partial, bytes) != cudaSuccess) {
            ens_set_error("out of device memory for split-K partials", __FILE__, __LINE__);
            return ENS_ENOMEM;
        }
        c->ws_bytes += bytes;
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
