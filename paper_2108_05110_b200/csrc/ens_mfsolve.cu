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
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "ens_internal.cuh"
#include "ens_mf_common.cuh"

// Programmatic dependent launch (sm_90+): a kernel launched with programmatic stream
// serialisation may start while its predecessor drains; everything before pdl_wait() must
// read only data that no in-flight kernel writes (here: factor entries, descriptors, index
// lists).  Both are no-ops for kernels launched normally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

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

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

#define SG_R 64     // rows per CTA (= symbolic.SOLVE_ROWS)
#define SG_C 32     // member columns per CTA
#ifndef SG_KMAX
#define SG_KMAX 256 // max inner range per work item (>= the plan's split lengths)
#endif
#ifndef SG_KC
#define SG_KC 32    // inner chunk of the pipelined mainloop
#endif
#define SG_LDA 36   // A stage row stride (= 4 mod 16: conflict-free fragment reads)
#define SG_T 256    // threads

__device__ __forceinline__ void dmma8(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// value at row r (>= 0) of a member-minor block, 0 for r < 0; the load itself is
// unconditional (clamped row) so the compiler can batch a whole gather's loads
// instead of serialising them behind per-source branches
__device__ __forceinline__ double gsel(const double* __restrict__ p, int r, int J) {
    const double t = p[(int64_t)max(r, 0) * J];
    return r >= 0 ? t : 0.0;
}

// Solve work item with its front's geometry, one 48-byte record so a CTA learns
// everything it addresses with a single dependent load:
//   [0] = {f, r0, ks, slot}   [1] = {m, k, has_children, -}   [2] = {off lo/hi, idx_off lo/hi}
__global__ void k_build_sitem(MfDev d, int64_t nwork, int nfront, const uint8_t* __restrict__ hasch,
                              int4* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nwork) return;
    const int4 w = reinterpret_cast<const int4*>(d.work)[i];
    const int f = (w.x >= 0 && w.x < nfront) ? w.x : 0;
    const int64_t off = d.off[f], io = d.idx_off[f];
    out[3 * i] = w;
    out[3 * i + 1] = make_int4(d.m[f], d.k[f], (int)hasch[f], 0);
    out[3 * i + 2] = make_int4((int)(off & 0xffffffff), (int)(off >> 32), (int)(io & 0xffffffff), (int)(io >> 32));
}

// Forward assembly of one tree level, before its GEMM launch: every front row
// gets the children's contribution rows mapped onto it (+ b at pivot rows):
//     fr[P] = b[P] + children rows,   fr[C] = children rows
// `rows` lists the level's rows that need it (pivot rows: value | (1 << 31));
// contribution rows of leaf fronts are not listed -- they start from zero in the
// GEMM epilogue.  Grid-stride over (row, column pair) so the launch stays small.
__global__ void __launch_bounds__(256) k_finit(const int32_t* __restrict__ rows, int64_t nrows,
                                               const int32_t* __restrict__ idx, const int32_t* __restrict__ gsrc,
                                               double* __restrict__ FR, const SolveIO* __restrict__ io, int64_t N,
                                               int J, int64_t nidx) {
    const int mat = blockIdx.y;
    pdl_wait();   // children's contribution rows come from the previous level's GEMM
    const double* b = io->r + (int64_t)mat * N * J;
    double* FRm = FR + (int64_t)mat * nidx * J;
    if ((J & 1) == 0 && nrows * (J >> 1) < (int64_t)INT32_MAX - (int64_t)gridDim.x * blockDim.x) {
        // 32-bit (row, column-pair) split: the 64-bit division by H dominated the index math
        const int H = J >> 1;
        const double2* b2 = reinterpret_cast<const double2*>(b);
        double2* F2 = reinterpret_cast<double2*>(FRm);
        const int tot = (int)(nrows * H);
        for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += gridDim.x * blockDim.x) {
            const int rq = t / H;
            const int e = rows[rq];
            const int i = t - rq * H;
            const int64_t row = e & 0x7fffffff;
            const int4 g = *reinterpret_cast<const int4*>(gsrc + 4 * row);
            const double2 bv = b2[(int64_t)max(idx[row], 0) * H + i];
            double2 v = make_double2(0.0, 0.0);
            const int src[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double2 c = F2[(int64_t)max(src[u], 0) * H + i];
                if (src[u] >= 0) {
                    v.x += c.x;
                    v.y += c.y;
                }
            }
            F2[row * H + i] = e < 0 ? make_double2(bv.x + v.x, bv.y + v.y) : v;
        }
    } else if ((J & 1) == 0) {
        const int H = J >> 1;
        const double2* b2 = reinterpret_cast<const double2*>(b);
        double2* F2 = reinterpret_cast<double2*>(FRm);
        for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nrows * H;
             t += (int64_t)gridDim.x * blockDim.x) {
            const int e = rows[t / H];
            const int i = (int)(t % H);
            const int64_t row = e & 0x7fffffff;
            const int4 g = *reinterpret_cast<const int4*>(gsrc + 4 * row);
            const double2 bv = b2[(int64_t)max(idx[row], 0) * H + i];
            double2 v = make_double2(0.0, 0.0);
            const int src[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double2 c = F2[(int64_t)max(src[u], 0) * H + i];
                if (src[u] >= 0) {
                    v.x += c.x;
                    v.y += c.y;
                }
            }
            F2[row * H + i] = e < 0 ? make_double2(bv.x + v.x, bv.y + v.y) : v;
        }
    } else {
        for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nrows * J;
             t += (int64_t)gridDim.x * blockDim.x) {
            const int e = rows[t / J];
            const int j = (int)(t % J);
            const int64_t row = e & 0x7fffffff;
            const int4 g = *reinterpret_cast<const int4*>(gsrc + 4 * row);
            const double bv = b[(int64_t)max(idx[row], 0) * J + j];
            const double* p = FRm + j;
            const double v = gsel(p, g.x, J) + gsel(p, g.y, J) + gsel(p, g.z, J) + gsel(p, g.w, J);
            FRm[row * J + j] = e < 0 ? bv + v : v;
        }
    }
    pdl_trigger();
}

__device__ __forceinline__ void cp_async_wait_n(int n) {
    if (n <= 0) asm volatile("cp.async.wait_group 0;\n" ::);
    else if (n == 1) asm volatile("cp.async.wait_group 1;\n" ::);
    else if (n == 2) asm volatile("cp.async.wait_group 2;\n" ::);
    else if (n == 3) asm volatile("cp.async.wait_group 3;\n" ::);
    else asm volatile("cp.async.wait_group 4;\n" ::);
}

// item = (f, r0, ks, slot)
//   r0 < 0  : forward pivot-only item (front without contribution block): its
//             rows were assembled by k_finit, nothing left to do
//   slot<0  : whole inner range, result applied here
//   slot>=0 : inner range [ks*split_k, ...) of group s0 = slot - ks; the last
//             CTA of the group reduces partial[s0 .. s0+ns) in order
//
// Mainloop: the inner range runs in SG_KC-wide chunks through an nstage-deep
// cp.async pipeline (A = 64 front rows, B = 32 operand rows x 32 member
// columns per stage), so loads of chunk c+nstage-1 are in flight while chunk c
// runs on the fp64 tensor cores (mma.sync m8n8k4, warp w owns rows 8w..8w+7).
//   forward : B = fr[P] rows (assembled by k_finit), C rows fr[C] -= A B
//   backward: B = [fr[P]; x[C]] rows,                x[P] = -A B
#ifndef SG_MINB
#define SG_MINB 3
#endif
// CW: member columns per CTA (32, or 64 for wide ensembles: each staged factor chunk then
// feeds twice the tensor-core work); NCT <= CW / 8 column tiles are computed.
template <int NCT, int CW = 32>
__global__ void __launch_bounds__(SG_T, CW == 64 ? 2 : SG_MINB) k_sgemm(MfDev d, const int4* __restrict__ sitem, int item0,
                                                const double* __restrict__ F, double* __restrict__ FR,
                                                const SolveIO* __restrict__ io, int64_t N, int J, int64_t nidx,
                                                int bwd, int split_k, int nstage, double* __restrict__ partial,
                                                int* __restrict__ ticket, int64_t nslot, int zbase) {
    extern __shared__ double sm[];
    __shared__ int s_last;
    __shared__ int s_idx[SG_KMAX];
    const int4* rec = sitem + 3LL * (item0 + blockIdx.x);
    const int4 w0 = rec[0], w1 = rec[1], w2 = rec[2];
    const int r0 = w0.y, ks = w0.z, slot = w0.w;
    if (r0 < 0) return;
    const int m = w1.x, k = w1.y, hasch = w1.z;
    const int64_t off = (int64_t)(unsigned)w2.x | ((int64_t)w2.y << 32);
    const int64_t fo = (int64_t)(unsigned)w2.z | ((int64_t)w2.w << 32);
    const int mat = blockIdx.y;
    const int zb = zbase + blockIdx.z;
    constexpr int LDB = CW + 4;                        // = 4 (mod 16): conflict-free fragment reads
    constexpr int STAGE = SG_R * SG_LDA + SG_KC * LDB;  // doubles per pipeline stage
    constexpr int NB = CW / 8;                         // column tiles a CTA can hold
    const int j0 = zb * CW;
    const int jn = min(CW, J - j0);
    const double* base = F + (int64_t)mat * d.storage + off;
    double* FRm = FR + (int64_t)mat * nidx * J;
    double* fr = FRm + fo * J;
    double* x = io->z + (int64_t)mat * N * J;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
    const int rbase = bwd ? r0 : k + r0;
    const int nr = min(SG_R, (bwd ? k : m) - rbase);
    const int K = bwd ? m : k;
    const int kbeg = slot < 0 ? 0 : ks * split_k;
    const int kend = slot < 0 ? K : min(K, kbeg + split_k);
    const int kc = kend - kbeg;               // <= split_k <= SG_KMAX by construction of the schedule
    const int nch = (kc + SG_KC - 1) / SG_KC;
    const int row = 8 * warp + g;
    const bool row_ok = row < nr;
    // Load issue with per-thread invariants hoisted (thread = row warp + 8 i, column lane;
    // SG_KC = 32, SG_T = 256) and the stage passed in (no runtime modulo): the leaf
    // levels were issue-bound on this address arithmetic (ncu: ~50 % of the instructions).
    static_assert(SG_KC == 32 && SG_T == 256 && (CW == 32 || CW == 64) && NCT <= CW / 8, "k_sgemm load mapping");
    const uint32_t sm_u32 = (uint32_t)__cvta_generic_to_shared(sm);
    const double* a_src = base + (int64_t)(rbase + warp) * m + kbeg + lane;
    const int64_t a_rstep = 8LL * m;
    const uint32_t a_dst = sm_u32 + 8u * (uint32_t)(warp * SG_LDA + lane);
    const uint32_t b_dst = sm_u32 + 8u * (uint32_t)(SG_R * SG_LDA + warp * LDB + lane);
    const bool jok = lane < jn;
    const double* b_fr = fr + j0 + lane;
    const double* b_x = x + j0 + lane;
    auto cpa8 = [](uint32_t s, const double* gp, bool pred) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gp), "r"(pred ? 8 : 0));
    };
    auto issue_a = [&](int c, int st) {
        const uint32_t dst = a_dst + 8u * (uint32_t)(st * STAGE);
        const bool kok = c * SG_KC + lane < kc;
        const double* src = a_src + c * SG_KC;
#pragma unroll
        for (int i = 0; i < SG_R / 8; ++i) {
            const bool ok = kok && warp + 8 * i < nr;
            cpa8(dst + 8u * (uint32_t)(8 * i * SG_LDA), ok ? src + i * a_rstep : base, ok);
        }
    };
    auto issue_b = [&](int c, int st) {
        const uint32_t dst = b_dst + 8u * (uint32_t)(st * STAGE);
#pragma unroll
        for (int h = 0; h < CW / 32; ++h) {
            const int col = lane + 32 * h;
            if (col >= 8 * NCT) break;   // member columns no column tile of this launch reads
            const bool cok = col < jn;
#pragma unroll
            for (int i = 0; i < SG_KC / 8; ++i) {
                const int kg = c * SG_KC + warp + 8 * i;
                const bool ok = cok && kg < kc;
                const int kq = min(kg, kc - 1), t = kbeg + kq;
                const double* src = (!bwd || t < k) ? b_fr + 32 * h + (int64_t)t * J
                                                    : b_x + 32 * h + (int64_t)s_idx[kq] * J;
                cpa8(dst + 8u * (uint32_t)(8 * i * LDB + 32 * h), ok ? src : base, ok);
            }
        }
    };
    // (1) first A chunk (factor entries: safe before the dependency wait), epilogue operands,
    // backward gather descriptors
    issue_a(0, 0);
    const int xrow = (bwd && row_ok) ? d.idx[fo + rbase + row] : 0;
    pdl_wait();   // front rows / the iterate come from the previous launch
    double init[NB][2];
#pragma unroll
    for (int ct = 0; ct < NB; ++ct) init[ct][0] = init[ct][1] = 0.0;
    if (!bwd && hasch && row_ok) {
        const double* pr = FRm + (fo + rbase + row) * J + j0;
#pragma unroll
        for (int ct = 0; ct < NB; ++ct)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = min(8 * ct + 2 * q + e, jn - 1);
                init[ct][e] = pr[col];
            }
    }
    if (bwd)
        for (int t = tid; t < kc; t += SG_T) s_idx[t] = (kbeg + t >= k) ? d.idx[fo + kbeg + t] : 0;
    __syncthreads();
    // (2) pipeline prologue: stages 0 .. nstage-2, one commit group each
    issue_b(0, 0);
    cp_async_commit();
    for (int c = 1; c < nstage - 1; ++c) {
        if (c < nch) {
            issue_a(c, c);
            issue_b(c, c);
        }
        cp_async_commit();
    }
    // (3) mainloop
    double dacc[NB][2];
#pragma unroll
    for (int ct = 0; ct < NB; ++ct) dacc[ct][0] = dacc[ct][1] = 0.0;
    int ust = 0;   // stage of chunk c (= c mod nstage); chunk c + nstage - 1 goes to the stage before it
    for (int c = 0; c < nch; ++c) {
        cp_async_wait_n(nstage - 2);
        __syncthreads();
        const int cn = c + nstage - 1;
        if (cn < nch) {
            const int ist = ust == 0 ? nstage - 1 : ust - 1;
            issue_a(cn, ist);
            issue_b(cn, ist);
        }
        cp_async_commit();
        const double* As = sm + ust * STAGE;
        ust = ust + 1 == nstage ? 0 : ust + 1;
        const double* ap = As + row * SG_LDA + q;
        const double* bp = As + SG_R * SG_LDA + q * LDB + g;
        const int ksteps = (min(SG_KC, kc - c * SG_KC) + 3) >> 2;
        if (8 * warp >= nr) {
            // no valid row in this warp: skip the tensor-core work (barriers above/below still hit)
        } else if (ksteps == SG_KC / 4) {
#pragma unroll
            for (int u = 0; u < SG_KC / 4; ++u) {
                const double av = ap[4 * u];
#pragma unroll
                for (int ct = 0; ct < NCT; ++ct) dmma8(dacc[ct][0], dacc[ct][1], av, bp[4 * u * LDB + 8 * ct]);
            }
        } else {
#pragma unroll 2
            for (int u = 0; u < ksteps; ++u) {
                const double av = ap[4 * u];
#pragma unroll
                for (int ct = 0; ct < NCT; ++ct) dmma8(dacc[ct][0], dacc[ct][1], av, bp[4 * u * LDB + 8 * ct]);
            }
        }
    }
    pdl_trigger();   // the next launch may start its prologue while this epilogue runs
    if (slot >= 0) {
        // split: publish the partial; the last CTA of the group sums the group's
        // partials in ks order (deterministic) and applies the epilogue
        double* pw = partial + (((int64_t)mat * nslot + slot) * SG_R + row) * J + j0;
        if (row_ok) {
#pragma unroll
            for (int ct = 0; ct < NB; ++ct)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (8 * ct + 2 * q + e < jn) pw[8 * ct + 2 * q + e] = dacc[ct][e];
        }
        __threadfence();
        __syncthreads();
        const int s0 = slot - ks;
        const int ns = (K + split_k - 1) / split_k;
        const int tk = (int)(((int64_t)mat * nslot + s0) * ((J + SG_C - 1) / SG_C) + zb);
        if (tid == 0) s_last = (atomicAdd(ticket + tk, 1) == ns - 1);
        __syncthreads();
        if (!s_last) {
            return;
        }
        __threadfence();
        if (tid == 0) ticket[tk] = 0;   // ready for the next solve / graph replay
        if (!row_ok) return;
        const double* pr = partial + (((int64_t)mat * nslot + s0) * SG_R + row) * J + j0;
        const int64_t pst = (int64_t)SG_R * J;
#pragma unroll
        for (int ct = 0; ct < NB; ++ct) dacc[ct][0] = dacc[ct][1] = 0.0;
#pragma unroll 4
        for (int qq = 0; qq < ns; ++qq) {
#pragma unroll
            for (int ct = 0; ct < NB; ++ct)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (8 * ct + 2 * q + e < jn) dacc[ct][e] += __ldcg(pr + qq * pst + 8 * ct + 2 * q + e);
        }
    }
    if (!row_ok) return;
#pragma unroll
    for (int ct = 0; ct < NB; ++ct)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int col = 8 * ct + 2 * q + e;
            if (col >= jn) continue;
            if (bwd)
                x[(int64_t)xrow * J + j0 + col] = -dacc[ct][e];
            else
                FRm[(fo + rbase + row) * J + j0 + col] = init[ct][e] - dacc[ct][e];
        }
}

#define SG_MAXST 5
static size_t sg_smem(int nstage, int cw = 32) {
    return sizeof(double) * (size_t)nstage * (SG_R * SG_LDA + SG_KC * (cw + 4));
}

// 64-member column blocks for J >= 64 (ENS_SOLVE_CW64=0 keeps 32)
static bool sg_wide(int J) {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("ENS_SOLVE_CW64");
        v = e ? std::atoi(e) : 1;
    }
    return v != 0 && J >= 64;
}

static int sg_stages(int kmax) {
    static int env = -1;
    if (env < 0) {
        const char* e = std::getenv("ENS_SOLVE_STAGES");
        env = e ? std::max(2, std::min(SG_MAXST, std::atoi(e))) : 0;
    }
    if (env > 0) return std::min(env, std::max(2, (kmax + SG_KC - 1) / SG_KC));
    return 2;   // measured: a shallow pipeline with more resident CTAs wins (stage sweep, profiles/)
}

static bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    return st != cudaStreamCaptureStatusNone;
}

static bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("ENS_PDL");
        v = e ? std::atoi(e) : 1;
    }
    return v != 0;
}

// launch with programmatic stream serialisation (overlaps this launch's prologue with the
// predecessor's tail; see pdl_wait)
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

#ifndef RET
#define RET(x)                         \
    do {                               \
        int rc_ = (x);                 \
        if (rc_ != ENS_OK) return rc_; \
    } while (0)
#endif

// ===========================================================================
// Streamed solve (default for even J): the same forward / backward products,
// restructured as a pure HBM stream.
//
//  * Work tiles of <= 32 rows (4 groups of 8) x the front's whole inner range,
//    built once per plan.  After every factorisation k_stream_pack copies each
//    tile's factor entries out of the fronts into one contiguous stream per
//    system, in the exact order the DMMA A-fragments consume them: for k-step u
//    (4 inner columns) and row group w, the 32 values A[8w+g][4u+q] in lane order
//    (g = lane/4, q = lane%4); padding is zero.  A warp's fragment load is then
//    one conflict-free 256-byte shared-memory read, and a chunk of KC inner
//    columns of a tile is one contiguous cp.async.bulk copy.
//  * Front vectors live in their own blocked layout FRS[system][column block]
//    [row][ldb] (ldb >= the block's columns, = 4 mod 16: conflict-free DMMA
//    B-fragment reads), so a chunk's B operand -- consecutive front rows -- is
//    one contiguous region: the forward pivot rows assembled by s_finit, and in
//    the backward sweep the front's rows after s_bgather has copied the
//    ancestors' solution rows x[C] next to fr[P].
//  * Persistent CTAs per level launch: one producer warp streams stages
//    (A chunk + B rows, two cp.async.bulk copies) through an mbarrier ring,
//    running several tiles ahead of the four consumer warps, which accumulate
//    with mma.sync m8n8k4 (fp64 tensor cores) and store their rows.  Units
//    (tile, system, column block) are split over the CTAs in contiguous ranges
//    of equal bytes (host side), so per-tile latency is hidden by the pipeline
//    instead of by CTA count.
//  * Every output element sums its inner range in a fixed order (k-step by
//    k-step): deterministic, identical columns stay identical.
// ===========================================================================
namespace {

struct STile {
    int a_lo, a_hi;   // offset (doubles) of the tile in its system's stream
    int fo;           // front's first index-list position (f_idx_off)
    int K;            // inner length (fwd: k, bwd: m)
    int kp;           // pivot count k of the front
    int r0;           // first row of the tile (fwd: within the C rows, bwd: within the pivots)
    int ng;           // row groups of 8 (1..4)
    int flags;        // bit0: backward, bit1: forward init rows carry children's contributions
    int src_lo, src_hi;   // front's storage offset (f_off)
    int m;            // front size
    int row0;         // first front row of the tile
    int kb, ke;       // inner range of the unit ([0, K))
    int sc_lo, sc_n;  // backward: the tile's (destination row, source row) scatter pairs in sc_ent
};
static_assert(sizeof(STile) == 64, "STile layout");

constexpr int ST_ROWS = 32;     // rows per tile
constexpr int ST_MAXST = 12;    // pipeline stages (upper bound)
constexpr int ST_THREADS = 160; // 4 consumer warps + 1 producer warp
constexpr int ST_CTAS = 4;      // resident CTAs per SM (shared memory per CTA sized for it)

__device__ __forceinline__ uint32_t st_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void st_mbar_init(uint32_t bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void st_mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void st_mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void st_mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void st_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ double st_lds(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int64_t st_i64(int lo, int hi) { return (int64_t)(unsigned)lo | ((int64_t)hi << 32); }
}  // namespace

#ifdef ST_PROBE   // diagnostic build: per-CTA timeline of consumer warp 0 (wait vs. work), launch 0 only
__device__ unsigned long long g_stp[2048][10];
__device__ __forceinline__ unsigned long long st_gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ unsigned long long g_lvl[256][2];   // per launch id: first CTA start, last CTA end
__device__ int g_probe_target;                 // launch id whose per-CTA consumer timeline is kept
extern "C" int ens_stream_probe_target(int id) { return (int)cudaMemcpyToSymbol(g_probe_target, &id, sizeof(int)); }
__device__ __forceinline__ void st_span_begin(int id) {
    if (threadIdx.x == 0 && id >= 0 && id < 256) atomicMin(&g_lvl[id][0], st_gt());
}
__device__ __forceinline__ void st_span_end(int id) {   // every thread: the last one out sets the end
    if (id >= 0 && id < 256) atomicMax(&g_lvl[id][1], st_gt());
}
extern "C" int ens_stream_probe_reset() {
    static unsigned long long h[256][2];
    for (int i = 0; i < 256; ++i) {
        h[i][0] = ~0ull;
        h[i][1] = 0;
    }
    static unsigned long long z[2048][10];
    cudaMemcpyToSymbol(g_stp, z, sizeof(z));
    return (int)cudaMemcpyToSymbol(g_lvl, h, sizeof(h));
}
extern "C" int ens_stream_probe_levels(const char* path) {
    static unsigned long long h[256][2];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, g_lvl, sizeof(h));
    FILE* f = fopen(path, "w");
    if (!f) return -1;
    for (int i = 0; i < 256; ++i) fprintf(f, "%d %llu %llu\n", i, h[i][0], h[i][1]);
    fclose(f);
    return 0;
}
extern "C" int ens_stream_probe_dump(const char* path) {
    static unsigned long long h[2048][10];
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(h, g_stp, sizeof(h));
    FILE* f = fopen(path, "w");
    if (!f) return -1;
    for (int i = 0; i < 2048; ++i)
        fprintf(f, "%d %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu\n", i, h[i][0], h[i][1], h[i][2], h[i][3],
                h[i][4], h[i][5], h[i][6], h[i][7], h[i][8], h[i][9]);
    fclose(f);
    return 0;
}
#define ST_SPAN_BEGIN(id) st_span_begin(id)
#define ST_SPAN_END(id) st_span_end(id)
// per-CTA timeline of consumer warp 0 (launch g_probe_target): slot k of row blockIdx.x
#define ST_MARK(id, k)                                                                            \
    do {                                                                                          \
        if (threadIdx.x == 0 && (id) == g_probe_target && blockIdx.x < 2048) g_stp[blockIdx.x][k] = st_gt(); \
    } while (0)
#else
#define ST_SPAN_BEGIN(id)
#define ST_SPAN_END(id)
#define ST_MARK(id, k)
#endif

// ENS_BOUNDS_CHECK builds (tools/sanitize_run.py; compute-sanitizer is not available on the GPU
// pool): device asserts on every index the streamed solve derives from the plan
#ifdef ENS_BOUNDS_CHECK
#include <cassert>
#define ST_ASSERT(c) assert(c)
#else
#define ST_ASSERT(c)
#endif

// factor entries -> fragment-ordered tile stream (one CTA per tile and system)
__global__ void __launch_bounds__(256) k_stream_pack(const STile* __restrict__ tiles, const double* __restrict__ F,
                                                     int64_t storage, double* __restrict__ S, int64_t slen) {
    const STile T = tiles[blockIdx.x];
    const int mat = blockIdx.y;
    const int Kp = (T.K + 3) & ~3;
    const int rows_total = (T.flags & 1) ? T.kp : T.m - T.kp;
    const int nr = min(ST_ROWS, rows_total - T.r0);
    const double* base = F + (int64_t)mat * storage + st_i64(T.src_lo, T.src_hi);
    double* out = S + (int64_t)mat * slen + st_i64(T.a_lo, T.a_hi);
    const int total = Kp * T.ng * 8;
    ST_ASSERT(st_i64(T.a_lo, T.a_hi) + total <= slen);
    ST_ASSERT(st_i64(T.src_lo, T.src_hi) + (int64_t)T.m * T.m <= storage);
    ST_ASSERT(T.row0 + nr <= T.m && T.K <= T.m && T.ng >= 1 && T.ng <= 4);
    // thread e writes stream entry e (coalesced); entry e = k-step u, row group w, lane (g, q)
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int lane = e & 31, grp = e >> 5;
        const int u = grp / T.ng, w = grp - u * T.ng;
        const int r = 8 * w + (lane >> 2), col = 4 * u + (lane & 3);
        out[e] = (r < nr && col < T.K) ? base[(int64_t)(T.row0 + r) * T.m + col] : 0.0;
    }
}

// Producer of a unit range: streams every chunk of units [ub, ue) through the stage ring.
// The factor stream is static during an apply, so the A copies of the first ring-full of chunks are
// issued BEFORE the dependency wait (early pass: returns how many); the pass after the wait adds
// those chunks' B copies (front rows written by the previous launch) and then streams normally.
template <int KC>
__device__ __forceinline__ int st_produce(const STile* sT, int tb, int ub, int ue, int per_tile, int ncb, int ldb,
                                          const double* __restrict__ S, int64_t slen,
                                          const double* __restrict__ FRS, int64_t nidx, int nst, uint32_t stage_bytes,
                                          uint32_t sbase, uint32_t bbase, bool early, int pre) {
    constexpr uint32_t A_BYTES = KC * ST_ROWS * 8;
    int s = 0, n = 0;
    uint32_t ph = 0;
    for (int u = ub; u < ue; ++u) {
        const STile& T = sT[u / per_tile - tb];
        const int mat = (u % per_tile) / ncb, cb = u % ncb;
        const double* Ab = S + (int64_t)mat * slen + st_i64(T.a_lo, T.a_hi);
        const double* Bb = FRS + ((int64_t)(mat * ncb + cb) * nidx + T.fo) * ldb;
        const int nch = (T.ke - T.kb + KC - 1) / KC;
        for (int c = 0; c < nch; ++c, ++n) {
            if (early && n == nst) return n;
            const int k0 = T.kb + c * KC, kr = min(KC, T.ke - k0);
            const uint32_t a_bytes = (uint32_t)((kr + 3) >> 2) * T.ng * 256u;
            const uint32_t b_bytes = (uint32_t)kr * ldb * 8u;
            ST_ASSERT(st_i64(T.a_lo, T.a_hi) + (int64_t)k0 * T.ng * 8 + a_bytes / 8 <= slen);
            ST_ASSERT(T.fo + k0 + kr <= nidx && a_bytes <= A_BYTES);
            const uint32_t full = bbase + 8 * s;
            const uint32_t st = sbase + (uint32_t)s * stage_bytes;
            if (early) {   // fresh ring: every stage is free
                st_mbar_expect_tx(full, a_bytes + b_bytes);
                st_bulk_g2s(st, Ab + (int64_t)k0 * T.ng * 8, a_bytes, full);
            } else if (n < pre) {
                st_bulk_g2s(st + A_BYTES, Bb + (int64_t)k0 * ldb, b_bytes, full);
            } else {
                st_mbar_wait(bbase + 8 * (ST_MAXST + s), ph ^ 1);
                st_mbar_expect_tx(full, a_bytes + b_bytes);
                st_bulk_g2s(st, Ab + (int64_t)k0 * T.ng * 8, a_bytes, full);
                st_bulk_g2s(st + A_BYTES, Bb + (int64_t)k0 * ldb, b_bytes, full);
            }
            s = s + 1 == nst ? 0 : s + 1;
            if (s == 0) ph ^= 1;
        }
    }
    return n;
}

// Per-row epilogue metadata of a unit (static plan data): backward, the dof the row solves for;
// forward, the <= 4 children's contribution rows mapped onto the row (else -1).
__device__ __forceinline__ int4 st_row_meta(const STile& X, int grp, int g, const int32_t* __restrict__ fidx,
                                            const int32_t* __restrict__ gsrc) {
    int4 r = make_int4(-1, -1, -1, -1);
    const int row = 8 * grp + g;
    const bool bw = X.flags & 1;
    const int nrr = min(ST_ROWS, (bw ? X.kp : X.m - X.kp) - X.r0);
    if (grp >= X.ng || row >= nrr) return r;
    const int64_t prow = X.fo + X.r0 + row + (bw ? 0 : X.kp);
    if (bw)
        r.x = __ldg(fidx + prow);
    else if (X.flags & 2)
        r = __ldg(reinterpret_cast<const int4*>(gsrc + 4 * prow));
    return r;
}

// Forward: the sum of the children's contribution rows mapped onto this thread's row (its fragment
// columns), from the row metadata.
template <int NCT>
__device__ __forceinline__ void st_child_rows(const int4 meta, const double* __restrict__ FRm, int ldb, int q,
                                              double (&init)[NCT][2]) {
    const int src[4] = {meta.x, meta.y, meta.z, meta.w};
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        if (src[v] < 0) break;
        const double* pr = FRm + (int64_t)src[v] * ldb;
#pragma unroll
        for (int ct = 0; ct < NCT; ++ct)
#pragma unroll
            for (int e = 0; e < 2; ++e) init[ct][e] += pr[min(8 * ct + 2 * q + e, ldb - 1)];
    }
}

// Epilogue of one unit, run by the four consumer warps (warp `grp` holds row group grp's sums in the
// DMMA fragment layout: lane (g, q) has row 8 grp + g, columns 8 ct + 2 q + {0, 1}).
//   forward : contribution rows  fr[C] = (children's rows) - sum        -> blocked front vectors
//   backward: solution rows      x[P]  = -sum                           -> the iterate, and into the
//             contribution rows of every descendant front that reads them (up to ~40 per row at the
//             root).  A tile's rows are consecutive pivots, so its (destination row, source row) pairs
//             are one contiguous range of sc_ent: the result tile is staged in shared memory (rt, two
//             buffers alternating per unit) and the warps walk the range together, jn/2 lanes per pair
//             with one 16-byte store each and the pair loads batched (independent).
constexpr int ST_SCU = 8;   // scatter pairs in flight per lane
__device__ __forceinline__ void st_scatter_load(int2 (&pr)[ST_SCU], const int2* __restrict__ sc_ent, int e, int e1,
                                                int stride) {
#pragma unroll
    for (int v = 0; v < ST_SCU; ++v) {
        const int ee = e + stride * v;
        pr[v] = ee < e1 ? __ldg(sc_ent + ee) : make_int2(-1, 0);
    }
}

template <int NCT>
__device__ __forceinline__ void st_epilogue(const STile& T, int& nsc, int grp, int lane, double (&sum)[NCT][2],
                                            const double (&init)[NCT][2], double* out_row, bool row_ok, int jn,
                                            double* __restrict__ FRm, int ldb, const int2* __restrict__ sc_ent,
                                            double* rtbuf, int64_t nidx, int sy = 0, int sn = 1,
                                            const int2* pre = nullptr) {
    const int g = lane >> 2, q = lane & 3;
    const bool bwd = T.flags & 1;
#pragma unroll
    for (int ct = 0; ct < NCT; ++ct)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int col = 8 * ct + 2 * q + e;
            sum[ct][e] = bwd ? -sum[ct][e] : init[ct][e] - sum[ct][e];
            if (row_ok && col < jn) out_row[col] = sum[ct][e];
        }
    if (!bwd || T.sc_n == 0) return;   // (uniform over the CTA's consumer warps)
    // (the buffer alternates per scattering unit: a warp two units ahead of the slowest cannot exist,
    // because the barrier below sits between them)
    double* rt = rtbuf + (nsc & 1) * (ST_ROWS * NCT * 8);
    ++nsc;
    if (grp < T.ng) {
        const int row = 8 * grp + g;
#pragma unroll
        for (int ct = 0; ct < NCT; ++ct)
            *reinterpret_cast<double2*>(rt + row * (NCT * 8) + 8 * ct + 2 * q) = make_double2(sum[ct][0], sum[ct][1]);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const int lpp = jn >> 1, ppw = 32 / lpp;           // lanes per pair, pairs per warp and step
    const int sub = lane / lpp, cp = lane - sub * lpp;
    const int warp = (threadIdx.x >> 5) & 3;
    const int e1 = T.sc_lo + T.sc_n;
    if (sub >= ppw) return;
    // (sy, sn): this CTA's share when several CTAs scatter one tile (k_stream_reduce)
    const int stride = 4 * sn * ppw;
    for (int e = T.sc_lo + (sy * 4 + warp) * ppw + sub; e < e1; e += ST_SCU * stride) {
        int2 pr[ST_SCU];
        if (pre && e == T.sc_lo + (sy * 4 + warp) * ppw + sub) {
#pragma unroll
            for (int v = 0; v < ST_SCU; ++v) pr[v] = pre[v];
        } else {
            st_scatter_load(pr, sc_ent, e, e1, stride);
        }
#pragma unroll
        for (int v = 0; v < ST_SCU; ++v)
            if (pr[v].x >= 0) {
                ST_ASSERT(pr[v].x < nidx && pr[v].y >= 0 && pr[v].y < ST_ROWS);
                *reinterpret_cast<double2*>(FRm + (int64_t)pr[v].x * ldb + 2 * cp) =
                    *reinterpret_cast<const double2*>(rt + pr[v].y * (NCT * 8) + 2 * cp);
            }
    }
}

// Consumers (warps 0..3) of a unit range: DMMA mainloop, then the epilogue -- or, SPLIT, the unit is
// one of `ks` pieces of a tile's inner range (one piece per CTA) and the fragment sums go to the
// partial buffer for k_stream_reduce.
template <int NCT, int KC, bool SPLIT>
__device__ __forceinline__ void st_consume(const STile* sT, int tb, int ub, int ue, int per_tile, int ncb, int cw,
                                           int ldb, double* __restrict__ FRS, const SolveIO* __restrict__ io,
                                           const int32_t* __restrict__ fidx, const int32_t* __restrict__ gsrc,
                                           const int2* __restrict__ sc_ent, int64_t N, int J, int64_t nidx,
                                           int nst, uint32_t stage_bytes, const unsigned char* smem, double* rtbuf,
                                           uint32_t bbase, double* __restrict__ part, int probe_id) {
    constexpr uint32_t A_BYTES = KC * ST_ROWS * 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    int s = 0;
    uint32_t ph = 0;
    // Row groups go to the consumer warps round-robin across the CTA's units (rot = groups handed out
    // so far): tiles with fewer than 4 groups (the 7-row tail tiles of the leaf fronts) would otherwise
    // all land on warp 0, i.e. on one SM sub-partition's tensor pipe.
    // The per-row metadata is fetched one unit ahead (mnext), so the loads that depend on it (the
    // children's rows of the forward epilogue) are issued at the top of the unit, under the mainloop.
    int rot = 0, nsc = 0;
    int4 mnext = make_int4(-1, -1, -1, -1);
    if (!SPLIT && ub < ue) mnext = st_row_meta(sT[ub / per_tile - tb], warp, g, fidx, gsrc);
    ST_MARK(probe_id, 1);
    pdl_wait();   // front rows / the iterate come from the previous launch
    ST_MARK(probe_id, 2);
    for (int u = ub; u < ue; ++u) {
        const STile T = sT[u / per_tile - tb];
        const int mat = (u % per_tile) / ncb, cb = u % ncb;
        const int j0 = cb * cw, jn = min(cw, J - j0);
        const bool bwd = T.flags & 1;
        const int nr = min(ST_ROWS, (bwd ? T.kp : T.m - T.kp) - T.r0);
        const int grp = (warp - rot) & 3;
        const int row = 8 * grp + g;
        const bool active = grp < T.ng;
        const bool row_ok = active && row < nr;
        double* FRm = FRS + (int64_t)(mat * ncb + cb) * nidx * ldb;
        double* out_row = nullptr;
        double init[NCT][2];
#pragma unroll
        for (int ct = 0; ct < NCT; ++ct) init[ct][0] = init[ct][1] = 0.0;
        if (!SPLIT) {
            const int4 meta = mnext;
            rot = (rot + T.ng) & 3;
            if (u + 1 < ue) mnext = st_row_meta(sT[(u + 1) / per_tile - tb], (warp - rot) & 3, g, fidx, gsrc);
            if (row_ok) {
                if (bwd) {
                    ST_ASSERT(meta.x >= 0 && meta.x < N);
                    out_row = io->z + (int64_t)mat * N * J + (int64_t)meta.x * J + j0;
                } else {
                    out_row = FRm + (int64_t)(T.fo + T.r0 + row + T.kp) * ldb;
                    if (T.flags & 2) st_child_rows<NCT>(meta, FRm, ldb, q, init);
                }
            }
        }
        // two accumulator sets (even / odd k-steps, summed at the end): a warp alone reaches the fp64
        // tensor pipe's issue rate with two independent chains (tools/dmma_latency.cu)
        double acc[NCT][2], acc2[NCT][2];
#pragma unroll
        for (int ct = 0; ct < NCT; ++ct) acc[ct][0] = acc[ct][1] = acc2[ct][0] = acc2[ct][1] = 0.0;
        const int nch = (T.ke - T.kb + KC - 1) / KC;
        for (int c = 0; c < nch; ++c) {
            st_mbar_wait(bbase + 8 * s, ph);
            if (u == ub && c == 0) ST_MARK(probe_id, 3);
            if (active) {
                const int kr = min(KC, T.ke - T.kb - c * KC);
                const int ksteps = (kr + 3) >> 2;
                const double* stg = reinterpret_cast<const double*>(smem + (size_t)s * stage_bytes);
                const double* ap = stg + grp * 32 + lane;
                const double* bp = stg + A_BYTES / 8 + q * ldb + g;
                const int astep = T.ng * 32, bstep = 4 * ldb;
                if (ksteps == KC / 4) {
#pragma unroll
                    for (int uu = 0; uu < KC / 4; uu += 2) {
                        const double a0 = ap[uu * astep], a1 = ap[(uu + 1) * astep];
#pragma unroll
                        for (int ct = 0; ct < NCT; ++ct) {
                            dmma8(acc[ct][0], acc[ct][1], a0, bp[uu * bstep + 8 * ct]);
                            dmma8(acc2[ct][0], acc2[ct][1], a1, bp[(uu + 1) * bstep + 8 * ct]);
                        }
                    }
                } else {
                    int uu = 0;
                    for (; uu + 1 < ksteps; uu += 2) {
                        const double a0 = ap[uu * astep], a1 = ap[(uu + 1) * astep];
#pragma unroll
                        for (int ct = 0; ct < NCT; ++ct) {
                            dmma8(acc[ct][0], acc[ct][1], a0, bp[uu * bstep + 8 * ct]);
                            dmma8(acc2[ct][0], acc2[ct][1], a1, bp[(uu + 1) * bstep + 8 * ct]);
                        }
                    }
                    if (uu < ksteps) {
                        const double a0 = ap[uu * astep];
#pragma unroll
                        for (int ct = 0; ct < NCT; ++ct) dmma8(acc[ct][0], acc[ct][1], a0, bp[uu * bstep + 8 * ct]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) st_mbar_arrive(bbase + 8 * (ST_MAXST + s));
            s = s + 1 == nst ? 0 : s + 1;
            if (s == 0) ph ^= 1;
        }
        if (u + 1 == ue) ST_MARK(probe_id, 4);
#pragma unroll
        for (int ct = 0; ct < NCT; ++ct)
#pragma unroll
            for (int e = 0; e < 2; ++e) acc[ct][e] += acc2[ct][e];
        if constexpr (SPLIT) {   // CTA index = unit * ks + piece
            if (active) {
                double* pp = part + ((int64_t)blockIdx.x * 4 + grp) * (2 * NCT * 32) + lane;
#pragma unroll
                for (int ct = 0; ct < NCT; ++ct)
#pragma unroll
                    for (int e = 0; e < 2; ++e) pp[(2 * ct + e) * 32] = acc[ct][e];
            }
        } else {
            st_epilogue<NCT>(T, nsc, grp, lane, acc, init, out_row, row_ok, jn, FRm, ldb, sc_ent, rtbuf, nidx);
        }
    }
}

// stage ring set-up
__device__ __forceinline__ void st_ring_init(unsigned char* smem, uint32_t bbase, int nst, uint32_t stage_bytes) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            st_mbar_init(bbase + 8 * s, 1);
            st_mbar_init(bbase + 8 * (ST_MAXST + s), 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // B regions start finite (rows past a tile's inner range meet zero A entries: 0 * finite = 0)
    for (uint32_t i = threadIdx.x; i < (uint32_t)nst * stage_bytes / 8; i += blockDim.x)
        reinterpret_cast<double*>(smem)[i] = 0.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// One level and direction of the streamed solve.  Units u = (tile * 2 + system) * ncb + column
// block; CTA b runs units [cta_off[b], cta_off[b+1]).  SPLIT (upper tree levels: few tiles with long
// inner ranges -- one SM pulls only ~40 GB/s from HBM, so a level has to be spread over all of
// them): ks CTAs per unit, CTA b streams piece b % ks of unit b / ks and leaves its fragment sums
// in `part`; k_stream_reduce adds the pieces in order and runs the epilogue.
template <int NCT, int KC, bool SPLIT>
__global__ void __launch_bounds__(ST_THREADS, ST_CTAS)
    k_stream_gemm(const STile* __restrict__ tiles, int tile0, const int32_t* __restrict__ cta_off, int ncb, int cw,
                  int ldb, const double* __restrict__ S, int64_t slen, double* __restrict__ FRS,
                  const SolveIO* __restrict__ io, const int32_t* __restrict__ fidx,
                  const int32_t* __restrict__ gsrc, const int2* __restrict__ sc_ent, int64_t N, int J,
                  int64_t nidx, int nst, uint32_t stage_bytes, uint32_t desc_bytes, double* __restrict__ part,
                  int ks, int probe_id) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[2 * ST_MAXST];   // full[0..nst), empty[ST_MAXST..)
    ST_SPAN_BEGIN(probe_id);
    ST_MARK(probe_id, 0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sbase = st_smem_u32(smem);
    const uint32_t bbase = st_smem_u32(bars);
    st_ring_init(smem, bbase, nst, stage_bytes);
    // this CTA's tile descriptors into shared memory (static data: before the dependency wait), so
    // neither the producer nor the consumers pay a global-load latency per unit
    const int piece = SPLIT ? (int)(blockIdx.x % (unsigned)ks) : 0;
    const int ub = SPLIT ? (int)(blockIdx.x / (unsigned)ks) : cta_off[blockIdx.x];
    const int ue = SPLIT ? ub + 1 : cta_off[blockIdx.x + 1];
    const int per_tile = 2 * ncb;
    STile* sT = reinterpret_cast<STile*>(smem + (size_t)nst * stage_bytes);
    const int tb = ub / per_tile, te = ue > ub ? (ue - 1) / per_tile + 1 : tb;
    for (int i = threadIdx.x; i < (te - tb) * (int)(sizeof(STile) / 4); i += blockDim.x) {
        int v = __ldg(reinterpret_cast<const int*>(tiles + tile0 + tb) + i);
        if (SPLIT && (i == 12 || i == 13)) {   // kb / ke: this piece's share of the tile's chunks
            const int K = __ldg(&tiles[tile0 + tb].K);
            const int nch = (K + KC - 1) / KC;
            v = min(K, (int)((unsigned)(piece + (i - 12)) * (unsigned)nch / (unsigned)ks) * KC);
        }
        reinterpret_cast<int*>(sT)[i] = v;
    }
    __syncthreads();
    pdl_trigger();
    if (warp == 4) {
        int pre = 0;
        if (lane == 0)
            pre = st_produce<KC>(sT, tb, ub, ue, per_tile, ncb, ldb, S, slen, FRS, nidx, nst, stage_bytes, sbase,
                                 bbase, true, 0);
        pdl_wait();   // front rows / the iterate come from the previous launch (consumers: in st_consume)
        if (lane == 0)
            st_produce<KC>(sT, tb, ub, ue, per_tile, ncb, ldb, S, slen, FRS, nidx, nst, stage_bytes, sbase, bbase,
                           false, pre);
        return;
    }
    double* rtbuf = reinterpret_cast<double*>(smem + (size_t)nst * stage_bytes + desc_bytes);
    st_consume<NCT, KC, SPLIT>(sT, tb, ub, ue, per_tile, ncb, cw, ldb, FRS, io, fidx, gsrc, sc_ent, N, J, nidx, nst,
                               stage_bytes, smem, rtbuf, bbase, part, probe_id);
    ST_MARK(probe_id, 5);
#ifdef ST_PROBE
    if (lane == 0) ST_SPAN_END(probe_id);
#endif
}

// Second half of a SPLIT level: four warps per unit add the unit's ks pieces in order (fixed
// summation order: deterministic) and run the epilogue; gridDim.y CTAs share a unit's scatter
// pairs (each sums the pieces itself, CTA y = 0 writes the rows' own output).
template <int NCT>
__global__ void __launch_bounds__(128) k_stream_reduce(const STile* __restrict__ tiles, int tile0, int ncb, int cw,
                                                       int ldb, double* __restrict__ FRS,
                                                       const SolveIO* __restrict__ io,
                                                       const int32_t* __restrict__ fidx,
                                                       const int32_t* __restrict__ gsrc,
                                                       const int2* __restrict__ sc_ent, int64_t N, int J,
                                                       int64_t nidx, const double* __restrict__ part, int ks,
                                                       int probe_id) {
    __shared__ __align__(16) double rt[ST_ROWS * NCT * 8];
    ST_SPAN_BEGIN(probe_id);
    const int u = blockIdx.x, per_tile = 2 * ncb;
    const int grp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    const STile T = tiles[tile0 + u / per_tile];
    const int mat = (u % per_tile) / ncb, cb = u % ncb;
    const int j0 = cb * cw, jn = min(cw, J - j0);
    const bool bwd = T.flags & 1;
    const int nr = min(ST_ROWS, (bwd ? T.kp : T.m - T.kp) - T.r0);
    const int row = 8 * grp + g;
    const bool active = grp < T.ng, row_ok = active && row < nr && blockIdx.y == 0;
    // CTAs y > 0 only share the scatter: nothing to do if the pairs do not reach their first step
    const int lpp = jn >> 1, ppw = 32 / lpp, sub = lane / lpp;
    const int e_first = T.sc_lo + ((int)blockIdx.y * 4 + grp) * ppw + sub, e1 = T.sc_lo + T.sc_n;
    if (blockIdx.y > 0 && (!bwd || T.sc_lo + (int)blockIdx.y * 4 * ppw >= e1)) return;
    pdl_trigger();
    const int4 meta = st_row_meta(T, grp, g, fidx, gsrc);
    double* FRm = FRS + (int64_t)(mat * ncb + cb) * nidx * ldb;
    int2 pre[ST_SCU];
    if (bwd && sub < ppw) st_scatter_load(pre, sc_ent, e_first, e1, 4 * (int)gridDim.y * ppw);   // (static data)
    pdl_wait();   // the pieces come from the previous launch
    double sum[NCT][2], init[NCT][2];
#pragma unroll
    for (int ct = 0; ct < NCT; ++ct) sum[ct][0] = sum[ct][1] = init[ct][0] = init[ct][1] = 0.0;
    double* out_row = nullptr;
    if (row_ok) {
        if (bwd) {
            out_row = io->z + (int64_t)mat * N * J + (int64_t)meta.x * J + j0;
        } else {
            out_row = FRm + (int64_t)(T.fo + T.r0 + row + T.kp) * ldb;
            if (T.flags & 2) st_child_rows<NCT>(meta, FRm, ldb, q, init);
        }
    }
    if (active) {
        const double* pp = part + ((int64_t)u * ks * 4 + grp) * (2 * NCT * 32) + lane;
        double v[8][NCT][2];
#pragma unroll
        for (int p = 0; p < 8; ++p)
#pragma unroll
            for (int ct = 0; ct < NCT; ++ct)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    v[p][ct][e] = p < ks ? pp[(int64_t)p * 4 * (2 * NCT * 32) + (2 * ct + e) * 32] : 0.0;
#pragma unroll
        for (int p = 0; p < 8; ++p)
#pragma unroll
            for (int ct = 0; ct < NCT; ++ct)
#pragma unroll
                for (int e = 0; e < 2; ++e) sum[ct][e] += v[p][ct][e];
    }
    int nsc = 0;
    st_epilogue<NCT>(T, nsc, grp, lane, sum, init, out_row, row_ok, jn, FRm, ldb, sc_ent, rt, nidx, (int)blockIdx.y,
                     (int)gridDim.y, bwd ? pre : nullptr);
#ifdef ST_PROBE
    if (lane == 0) ST_SPAN_END(probe_id);
#endif
}

// Forward assembly of one level's PIVOT rows into the blocked front vectors (the B operand of the
// level's GEMM): FRS[row] = b[idx[row]] + the <= 4 children's contribution rows mapped onto it.
// (Contribution rows of the level are not assembled here: the GEMM epilogue adds their children's
// rows itself.)  One thread per (row, member pair).
__global__ void __launch_bounds__(256) k_sfinit(const int32_t* __restrict__ rows, int nrows,
                                                const int32_t* __restrict__ idx, const int32_t* __restrict__ gsrc,
                                                double* __restrict__ FRS, const SolveIO* __restrict__ io, int64_t N,
                                                int J, int64_t nidx, int ncb, int cw, int ldb, int probe_id) {
    const int mat = blockIdx.y;
    ST_SPAN_BEGIN(probe_id);
    pdl_trigger();   // the level's GEMM may set up (and prefetch its factor entries) meanwhile
    const int hw = cw >> 1, per = ncb * hw;
    const double* b = io->r + (int64_t)mat * N * J;
    const int tot = nrows * per;
    // one element per thread (the grid covers tot): row map, right-hand side and the children's row
    // map are static during an apply and are fetched before the dependency wait
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const bool on = t < tot;
    const int rq = on ? t / per : 0, rem = t - rq * per, cb = rem / hw, i = rem - cb * hw;
    const int col = cb * cw + 2 * i;
    const bool live = on && col < J;
    int64_t row = 0;
    int4 g = make_int4(-1, -1, -1, -1);
    double2 v = make_double2(0.0, 0.0);
    if (live) {
        row = rows[rq];
        ST_ASSERT(row >= 0 && row < nidx && idx[row] >= 0 && idx[row] < N);
        g = *reinterpret_cast<const int4*>(gsrc + 4 * row);
        ST_ASSERT(g.x < nidx && g.y < nidx && g.z < nidx && g.w < nidx);
        v = *reinterpret_cast<const double2*>(b + (int64_t)idx[row] * J + col);
    }
    pdl_wait();   // children's contribution rows come from the previous level's GEMM
    if (live) {
        const double2* F2 = reinterpret_cast<const double2*>(FRS + (int64_t)(mat * ncb + cb) * nidx * ldb);
        const int h = ldb >> 1;
        if (g.x >= 0) {   // rows without children's contributions (all leaf rows) load nothing else
            const int src[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double2 c = F2[(int64_t)max(src[u], 0) * h + i];
                if (src[u] >= 0) {
                    v.x += c.x;
                    v.y += c.y;
                }
            }
        }
        reinterpret_cast<double2*>(FRS + (int64_t)(mat * ncb + cb) * nidx * ldb)[row * h + i] = v;
    }
#ifdef ST_PROBE
    __syncthreads();
    if (threadIdx.x == 0) ST_SPAN_END(probe_id);
#endif
}

// ---------------------------------------------------------------------------
// host side of the streamed solve
// ---------------------------------------------------------------------------
bool mf_stream_on(ens_ctx* c) {
    if (c->stream_mode < 0) {
        // streamed path for even J up to 48 (C2: 0.705 -> 0.593 ms per apply); for wider ensembles the
        // classic k_sgemm path measured equal or faster (C3 J=64: 5.50 vs 5.63 ms, C4 J=128: 3.04 vs
        // 3.05 ms).  ENS_SOLVE_STREAM=0/1 forces a path (A/B measurements, tools/apply_ab.py).
        const char* e = std::getenv("ENS_SOLVE_STREAM");
        const bool want = e ? e[0] != '0' : c->J <= 48;
        c->stream_mode = ((c->J & 1) == 0 && want) ? 1 : 0;
    }
    return c->stream_mode == 1;
}

template <int NCT>
static cudaError_t stream_attr(size_t smem) {
    const cudaError_t e =
        cudaFuncSetAttribute(k_stream_gemm<NCT, 32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_stream_gemm<NCT, 32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem);
}

// Pieces per unit of a launch with U units whose longest inner range is kmax: as many as keep every
// CTA resident at once and leave each piece at least two chunks (<= 8).  One CTA per unit cannot
// pull a sparse upper level's factor entries fast enough (~40 GB/s per SM from HBM).
// ENS_STREAM_SPLIT caps the piece count (1 = never split).
static int stream_split(int64_t U, int kmax, int KC, int sms) {
    const char* e = std::getenv("ENS_STREAM_SPLIT");   // (read per context: tests compare both paths)
    const int cmax = e ? std::max(1, std::min(8, std::atoi(e))) : 8;
    const int64_t budget = (int64_t)ST_CTAS * sms;
    const int nch = (kmax + KC - 1) / KC;
    const int64_t ks = std::min<int64_t>(std::min<int64_t>(cmax, budget / std::max<int64_t>(U, 1)), nch / 2);
    return (int)std::max<int64_t>(ks, 1);
}

// tiles, per-launch CTA partitions and the stream buffer (once per context; J-dependent only in
// the column blocking and the partition weights)
static int stream_setup(ens_ctx* c) {
    const int nf = (int)c->p.nfront;
    std::vector<int32_t> fm(nf), fk(nf), par(nf);
    std::vector<int64_t> foff(nf), fio((size_t)nf + 1);
    ENS_CK(cudaMemcpy(fm.data(), c->p.f_m, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost));
    ENS_CK(cudaMemcpy(fk.data(), c->p.f_k, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost));
    ENS_CK(cudaMemcpy(par.data(), c->p.f_parent, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost));
    ENS_CK(cudaMemcpy(foff.data(), c->p.f_off, sizeof(int64_t) * nf, cudaMemcpyDeviceToHost));
    ENS_CK(cudaMemcpy(fio.data(), c->p.f_idx_off, sizeof(int64_t) * (nf + 1), cudaMemcpyDeviceToHost));
    std::vector<uint8_t> hasch(nf, 0);
    for (int f = 0; f < nf; ++f)
        if (par[f] >= 0 && par[f] < nf) hasch[par[f]] = 1;
    const int J = c->J;
    const int ncb = (J + 63) / 64;
    int cw = (J + ncb - 1) / ncb;
    cw += cw & 1;
    const int ldb = cw + (((4 - cw) % 16) + 16) % 16;
    const int KC = 32;
    const size_t stage = ((size_t)KC * ST_ROWS * 8 + ((size_t)KC * ldb + 8) * 8 + 127) & ~(size_t)127;
    // backward epilogue: two result tiles (ST_ROWS x 8 * column tiles) + the tile's scatter range
    const size_t rtb = sizeof(double) * 2 * ST_ROWS * 8 * (size_t)((cw + 7) / 8);
    const int nst =
        (int)std::max<size_t>(2, std::min<size_t>(ST_MAXST, (216 * 1024 / ST_CTAS - 2048 - rtb) / stage));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // backward scatter pairs: for every pivot position, the contribution rows of descendant fronts
    // that hold the same dof (the backward epilogue writes the solution row straight into them),
    // as (destination row, source row within its 32-row tile), ordered by source position -- the
    // pairs of one backward tile are contiguous
    const int64_t nidx_h = c->p.n_idx;
    std::vector<int32_t> fidx_h((size_t)nidx_h);
    ENS_CK(cudaMemcpy(fidx_h.data(), c->p.f_idx, sizeof(int32_t) * nidx_h, cudaMemcpyDeviceToHost));
    std::vector<int32_t> piv_of((size_t)c->n_total, -1), piv_t((size_t)c->n_total, 0);
    for (int f = 0; f < nf; ++f)
        for (int t = 0; t < fk[f]; ++t) {
            piv_of[fidx_h[fio[f] + t]] = (int32_t)(fio[f] + t);
            piv_t[fidx_h[fio[f] + t]] = t % ST_ROWS;
        }
    std::vector<int32_t> sc_off((size_t)nidx_h + 1, 0);
    for (int f = 0; f < nf; ++f)
        for (int t = fk[f]; t < fm[f]; ++t) ++sc_off[piv_of[fidx_h[fio[f] + t]] + 1];
    for (int64_t i = 0; i < nidx_h; ++i) sc_off[i + 1] += sc_off[i];
    std::vector<int2> sc_ent((size_t)sc_off[nidx_h]);
    {
        std::vector<int32_t> fill(sc_off.begin(), sc_off.end() - 1);
        for (int f = 0; f < nf; ++f)
            for (int t = fk[f]; t < fm[f]; ++t) {
                const int32_t dof = fidx_h[fio[f] + t];
                sc_ent[fill[piv_of[dof]]++] = make_int2((int32_t)(fio[f] + t), piv_t[dof]);
            }
    }
    std::vector<STile> tiles;
    std::vector<int32_t> cta;
    c->slaunch.clear();
    int64_t aoff = 0, part_units = 0;
    auto add_tile = [&](int f, int r0, int rows, int K, int flags, int row0) {
        STile t;
        const int ng = (std::min(ST_ROWS, rows - r0) + 7) / 8;
        t.a_lo = (int)(aoff & 0xffffffff);
        t.a_hi = (int)(aoff >> 32);
        t.fo = (int)fio[f];
        t.K = K;
        t.kp = fk[f];
        t.r0 = r0;
        t.ng = ng;
        t.flags = flags;
        t.src_lo = (int)(foff[f] & 0xffffffff);
        t.src_hi = (int)(foff[f] >> 32);
        t.m = fm[f];
        t.row0 = row0;
        t.kb = 0;
        t.ke = K;
        t.sc_lo = t.sc_n = 0;
        if (flags & 1) {
            const int nr = std::min(ST_ROWS, rows - r0);
            t.sc_lo = sc_off[fio[f] + r0];
            t.sc_n = sc_off[fio[f] + r0 + nr] - t.sc_lo;
        }
        aoff += (int64_t)((K + 3) & ~3) * ng * 8;
        tiles.push_back(t);
    };
    int max_cta_tiles = 1;
    auto close_launch = [&](int dir, int L, size_t t0) {
        if (tiles.size() == t0) return;
        const int64_t nt = (int64_t)(tiles.size() - t0);
        const int64_t U = nt * 2 * ncb;
        std::vector<double> cost((size_t)U);
        double tot = 0.0;
        for (int64_t u = 0; u < U; ++u) {
            const STile& t = tiles[t0 + u / (2 * ncb)];
            const int cb = (int)(u % ncb), jn = std::min(cw, J - cb * cw);
            const int kl = t.ke - t.kb;
            cost[u] = (double)t.ng * ((kl + 3) & ~3) * 64.0 + (double)kl * jn * 8.0 + 2048.0;
            tot += cost[u];
        }
        const int64_t G = std::min<int64_t>(U, (int64_t)ST_CTAS * sms);
        const size_t base = cta.size();
        cta.push_back(0);
        double acc = 0.0;
        int64_t b = 1;
        for (int64_t u = 0; u < U && b < G; ++u) {
            acc += cost[u];
            if (acc >= tot * (double)b / (double)G) {
                cta.push_back((int32_t)(u + 1));
                ++b;
            }
        }
        while ((int64_t)(cta.size() - base) < G) cta.push_back((int32_t)U);   // degenerate tails
        cta.push_back((int32_t)U);
        for (int64_t i = 0; i < G; ++i) {   // tiles a CTA touches (descriptors staged in shared memory)
            const int64_t a = cta[base + i], b = cta[base + i + 1];
            if (b > a) max_cta_tiles = std::max<int>(max_cta_tiles, (int)((b - 1) / (2 * ncb) - a / (2 * ncb) + 1));
        }
        int kmax = 0;
        for (int64_t i = 0; i < nt; ++i) kmax = std::max(kmax, tiles[t0 + i].ke - tiles[t0 + i].kb);
        const int64_t ks = stream_split(U, kmax, KC, sms);
        if (ks > 1) part_units = std::max(part_units, U * ks);
        c->slaunch.insert(c->slaunch.end(), {dir, L, (int64_t)t0, (int64_t)base, G, ks, U});
    };
    const int nlev = (int)c->level_front_off.size() - 1;
    for (int L = 0; L < nlev; ++L) {   // forward: contribution rows of every front
        const size_t t0 = tiles.size();
        for (int f = c->level_front_off[L]; f < c->level_front_off[L + 1]; ++f) {
            const int rows = fm[f] - fk[f];
            if (rows <= 0 || fk[f] <= 0) continue;
            for (int r0 = 0; r0 < rows; r0 += ST_ROWS) add_tile(f, r0, rows, fk[f], hasch[f] ? 2 : 0, fk[f] + r0);
        }
        close_launch(0, L, t0);
    }
    for (int L = nlev - 1; L >= 0; --L) {   // backward: pivot rows over the whole front
        const size_t t0 = tiles.size();
        for (int f = c->level_front_off[L]; f < c->level_front_off[L + 1]; ++f)
            for (int r0 = 0; r0 < fk[f]; r0 += ST_ROWS) add_tile(f, r0, fk[f], fm[f], 1, r0);
        close_launch(1, L, t0);
    }
    // forward assembly rows: the pivot rows of every front, per level
    std::vector<int32_t> bg;
    c->sbg_off.assign((size_t)nlev + 1, 0);
    for (int L = 0; L < nlev; ++L) {
        c->sbg_off[L] = (int64_t)bg.size();
        for (int f = c->level_front_off[L]; f < c->level_front_off[L + 1]; ++f)
            for (int t = 0; t < fk[f]; ++t) bg.push_back((int32_t)(fio[f] + t));
    }
    c->sbg_off[nlev] = (int64_t)bg.size();
    const size_t sbytes = sizeof(double) * 2 * (size_t)std::max<int64_t>(aoff, 32);
    const size_t frbytes = sizeof(double) * 2 * (size_t)ncb * (size_t)c->p.n_idx * ldb;
    // fragment sums of the split launches: [unit * pieces + piece][row group][2 * column tiles][lane]
    const size_t pbytes = sizeof(double) * std::max<size_t>((size_t)part_units * 4 * 2 * ((cw + 7) / 8) * 32, 32);
    if (cudaMalloc(&c->sstream, sbytes) != cudaSuccess || cudaMalloc(&c->stiles, sizeof(STile) * tiles.size()) !=
                                                              cudaSuccess ||
        cudaMalloc(&c->scta, sizeof(int32_t) * cta.size()) != cudaSuccess ||
        cudaMalloc(&c->sfr, frbytes) != cudaSuccess ||
        cudaMalloc(&c->sbg_rows, sizeof(int32_t) * std::max<size_t>(bg.size(), 1)) != cudaSuccess ||
        cudaMalloc(&c->spart, pbytes) != cudaSuccess ||
        cudaMalloc(&c->ssc_ent, sizeof(int2) * std::max<size_t>(sc_ent.size(), 1)) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(c->sstream);
        cudaFree(c->stiles);
        cudaFree(c->scta);
        cudaFree(c->sfr);
        c->sstream = nullptr;
        c->stiles = nullptr;
        c->scta = nullptr;
        c->sfr = nullptr;
        ens_set_error("out of device memory for the solve stream", __FILE__, __LINE__);
        return ENS_ENOMEM;
    }
    ENS_CK(cudaMemset(c->sstream, 0, sbytes));
    ENS_CK(cudaMemset(c->sfr, 0, frbytes));   // pad columns stay zero (B stages must be finite)
    ENS_CK(cudaMemcpy(c->stiles, tiles.data(), sizeof(STile) * tiles.size(), cudaMemcpyHostToDevice));
    ENS_CK(cudaMemcpy(c->scta, cta.data(), sizeof(int32_t) * cta.size(), cudaMemcpyHostToDevice));
    if (!bg.empty())
        ENS_CK(cudaMemcpy(c->sbg_rows, bg.data(), sizeof(int32_t) * bg.size(), cudaMemcpyHostToDevice));
    if (!sc_ent.empty())
        ENS_CK(cudaMemcpy(c->ssc_ent, sc_ent.data(), sizeof(int2) * sc_ent.size(), cudaMemcpyHostToDevice));
    c->ws_bytes += sbytes + frbytes + pbytes + sizeof(STile) * tiles.size() +
                   sizeof(int32_t) * (cta.size() + bg.size() + 2 * sc_ent.size());
    // the classic front vectors are not used on this path
    c->ws_bytes -= sizeof(double) * 2 * (size_t)c->p.n_idx * c->J;
    cudaFree(c->frvec);
    c->frvec = nullptr;
    c->stream_len = std::max<int64_t>(aoff, 32);
    c->n_stiles = (int64_t)tiles.size();
    c->scw = cw;
    c->sncb = ncb;
    c->sldb = ldb;
    c->snst = nst;
    c->skc = KC;
    c->sstage = stage;
    c->sdesc = ((size_t)max_cta_tiles * sizeof(STile) + 15) & ~(size_t)15;
    c->srt = rtb;
    const size_t smem = stage * nst + c->sdesc + c->srt;
    if (smem > 220 * 1024) {
        ens_set_error("streamed solve: a CTA's tile descriptors do not fit shared memory", __FILE__, __LINE__);
        return ENS_EINVAL;
    }
    ENS_CK(stream_attr<1>(smem));
    ENS_CK(stream_attr<2>(smem));
    ENS_CK(stream_attr<3>(smem));
    ENS_CK(stream_attr<4>(smem));
    ENS_CK(stream_attr<5>(smem));
    ENS_CK(stream_attr<6>(smem));
    ENS_CK(stream_attr<7>(smem));
    ENS_CK(stream_attr<8>(smem));
    return ENS_OK;
}

int mf_stream_prepare(ens_ctx* c) {
    if (!mf_stream_on(c) || c->stiles) return ENS_OK;
    const int rc = stream_setup(c);
    if (rc != ENS_OK) c->stream_mode = 0;   // no room for the stream: the classic path
    return ENS_OK;
}

int mf_stream_pack(ens_ctx* c, cudaStream_t s) {
    if (!mf_stream_on(c) || !c->stiles || c->n_stiles == 0) return ENS_OK;
    k_stream_pack<<<dim3((unsigned)c->n_stiles, 2), 256, 0, s>>>((const STile*)c->stiles, c->fronts,
                                                                 c->p.front_storage, c->sstream, c->stream_len);
    ENS_CKL();
    return ENS_OK;
}

// launch sequence of one streamed solve (after the identity-row copy)
static int stream_launches(ens_ctx* c, cudaStream_t s, SolveIO* io, int64_t* cnt) {
    const int J = c->J;
    const int64_t N = c->n_total, nidx = c->p.n_idx;
    const int nct = (c->scw + 7) / 8;
    const int nlev = (int)c->level_front_off.size() - 1;
    std::vector<int> fwd_at(nlev, -1), bwd_at(nlev, -1);
    const size_t smem = c->sstage * c->snst + c->sdesc + c->srt;
    for (size_t i = 0; i + 7 <= c->slaunch.size(); i += 7)
        (c->slaunch[i] == 0 ? fwd_at : bwd_at)[c->slaunch[i + 1]] = (int)i;
    auto gemm = [&](int li) -> int {
        const int64_t* r = &c->slaunch[li];
        const int t0 = (int)r[2], cb = (int)r[3];
        const int ks = (int)r[5];
        const unsigned U = (unsigned)r[6], G = ks > 1 ? U * (unsigned)ks : (unsigned)r[4];
#define SGS_(NC, SPL)                                                                                              \
    ENS_CK(launch_pdl(k_stream_gemm<NC, 32, SPL>, dim3(G), dim3(ST_THREADS), smem, s, (const STile*)c->stiles, t0, \
                      (const int32_t*)(c->scta + cb), c->sncb, c->scw, c->sldb, (const double*)c->sstream,       \
                      c->stream_len, c->sfr, (const SolveIO*)io, (const int32_t*)c->p.f_idx,                    \
                      (const int32_t*)c->p.gsrc, (const int2*)c->ssc_ent, N, J, nidx, c->snst,                   \
                      (uint32_t)c->sstage, (uint32_t)c->sdesc, c->spart, ks, (int)*cnt))
#define SGS(NC)                                                                                                    \
    do {                                                                                                           \
        if (ks > 1) {                                                                                              \
            SGS_(NC, true);                                                                                        \
            ENS_CKL();                                                                                             \
            ++*cnt;                                                                                                \
            ENS_CK(launch_pdl(k_stream_reduce<NC>, dim3(U, r[0] == 1 ? 8 : 1), dim3(128), 0, s,                   \
                              (const STile*)c->stiles, t0, c->sncb,                                               \
                              c->scw, c->sldb, c->sfr, (const SolveIO*)io, (const int32_t*)c->p.f_idx,            \
                              (const int32_t*)c->p.gsrc, (const int2*)c->ssc_ent, N, J, nidx,                     \
                              (const double*)c->spart, ks, (int)*cnt));                                           \
        } else {                                                                                                   \
            SGS_(NC, false);                                                                                       \
        }                                                                                                          \
    } while (0)
        switch (nct) {
            case 1: SGS(1); break;
            case 2: SGS(2); break;
            case 3: SGS(3); break;
            case 4: SGS(4); break;
            case 5: SGS(5); break;
            case 6: SGS(6); break;
            case 7: SGS(7); break;
            default: SGS(8); break;
        }
#undef SGS
#undef SGS_
        ENS_CKL();
        ++*cnt;
        return ENS_OK;
    };
    for (int L = 0; L < nlev; ++L) {
        const int64_t a = c->sbg_off[L], nr = c->sbg_off[L + 1] - a;
        if (nr > 0) {
            const int64_t tot = nr * c->sncb * (c->scw / 2);
            ENS_CK(launch_pdl(k_sfinit, dim3((unsigned)((tot + 255) / 256), 2), dim3(256), 0, s,
                              (const int32_t*)(c->sbg_rows + a), (int)nr, (const int32_t*)c->p.f_idx,
                              (const int32_t*)c->p.gsrc, c->sfr, (const SolveIO*)io, N, J, nidx, c->sncb, c->scw,
                              c->sldb, (int)*cnt));
            ENS_CKL();
            ++*cnt;
        }
        if (fwd_at[L] >= 0) RET(gemm(fwd_at[L]));
    }
    for (int L = nlev - 1; L >= 0; --L)
        if (bwd_at[L] >= 0) RET(gemm(bwd_at[L]));
    return ENS_OK;
}

// record the launch sequence of one solve (io table fixed)
static int mf_solve_launches(ens_ctx* c, cudaStream_t s, SolveIO* io, int64_t* nlaunch) {
    MfDev d = mfdev(c);
    const int J = c->J;
    const int64_t N = c->n_total, nidx = c->p.n_idx;
    const unsigned zc = (unsigned)((J + SG_C - 1) / SG_C);
    const int64_t nslot = c->p.n_slot;
    int64_t cnt = 0;
    if (c->m.ncons > 0) {
        const int64_t tot = 2LL * c->m.ncons * J;
        k_copy_cons_io<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(c->m.cons_row, c->m.ncons, io, N, J);
        ENS_CKL();
        ++cnt;
    }
    // ENS_SOLVE_TIMING=1 (debug, uncaptured path only): per-launch event timings to stderr
    const char* tenv = std::getenv("ENS_SOLVE_TIMING");
    const bool timing = tenv && tenv[0] == '1' && !capturing(s);
    const char* renv = std::getenv("ENS_SOLVE_REPEAT");   // with timing: repeat each launch (warm timings)
    const int trep = renv ? std::max(1, std::atoi(renv)) : 1;
    std::vector<cudaEvent_t> ev;
    std::vector<std::string> lab;
    auto mark = [&](const char* tag, int a, int b2) {
        if (!timing) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev.push_back(e);
        lab.push_back(std::string(tag) + " n=" + std::to_string(a) + " kmax=" + std::to_string(b2));
    };
    mark("start", 0, 0);
    if (mf_stream_on(c) && c->stiles) {
        const int rc = stream_launches(c, s, io, &cnt);
        *nlaunch = cnt;
        return rc;
    }
    for (const std::vector<int64_t>* sched : {&c->sched_fwd, &c->sched_bwd}) {
        const int64_t nrow = (int64_t)sched->size() / 5;
        for (int64_t i = 0; i < nrow; ++i) {
            const int64_t* q = &(*sched)[5 * i];
            const int op = (int)q[0], L = (int)q[1], off = (int)q[2], n = (int)q[3], kmax = (int)q[4];
            if ((op != SOP_FGEMM && op != SOP_BGEMM) || kmax > SG_KMAX || kmax < 0 || L < 0 ||
                L >= (int)c->level_front_off.size() - 1) {
                ens_set_error("bad solve schedule row", __FILE__, __LINE__);
                return ENS_EINVAL;
            }
            if (op == SOP_FGEMM) {   // assemble the level's front rows first
                const int64_t a = c->finit_off[L], nr = c->finit_off[L + 1] - a;
                const int64_t tot = nr * ((J & 1) ? J : J / 2);
                if (nr > 0) {
                    const unsigned nb = (unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 8);
                    for (int rep = 0; rep < (timing ? trep : 1); ++rep) {
                        ENS_CK(launch_pdl(k_finit, dim3(nb, 2), dim3(256), 0, s, c->finit_rows + a, nr, c->p.f_idx,
                                          c->p.gsrc, c->frvec, io, N, J, nidx));
                        ENS_CKL();
                    }
                    ++cnt;
                    mark("finit", (int)nr, 0);
                }
            }
            if (n == 0 || kmax == 0) continue;
            const int nst = sg_stages(kmax);
            const bool wide = sg_wide(J);
            for (int rep = 0; rep < (timing ? trep : 1); ++rep) {   // launches are idempotent
                // member column blocks of CW = 32 (or 64 for wide ensembles): full blocks use all their
                // column tiles, the remainder fewer
                const int CWd = wide ? 64 : 32;
                const int zfull = J / CWd, rem = J - zfull * CWd;
#define SGL(NC, CWT, ZN, Z0)                                                                                      \
    ENS_CK(launch_pdl(k_sgemm<NC, CWT>, dim3(n, 2, ZN), dim3(SG_T), sg_smem(nst, CWT), s, d, c->sitem, off,       \
                      c->fronts, c->frvec, io, N, J, nidx, (int)(op == SOP_BGEMM), kmax, nst, c->partial,         \
                      c->ticket, nslot, (int)(Z0)))
                if (zfull > 0) {
                    if (wide) SGL(8, 64, (unsigned)zfull, 0);
                    else SGL(4, 32, (unsigned)zfull, 0);
                    ENS_CKL();
                    if (rep == 0) ++cnt;
                }
                if (rem > 0) {
                    const int nct = (rem + 7) / 8;
                    if (wide) {
                        if (nct <= 4) SGL(4, 64, 1, zfull);
                        else if (nct <= 6) SGL(6, 64, 1, zfull);
                        else SGL(8, 64, 1, zfull);
                    } else if (nct == 1) SGL(1, 32, 1, zfull);
                    else if (nct == 2) SGL(2, 32, 1, zfull);
                    else if (nct == 3) SGL(3, 32, 1, zfull);
                    else SGL(4, 32, 1, zfull);
                    ENS_CKL();
                    if (rep == 0) ++cnt;
                }
#undef SGL
            }
            mark(op == SOP_BGEMM ? "bwd" : "fwd", n, kmax);
        }
    }
    if (timing) {
        cudaEventSynchronize(ev.back());
        float tot = 0.f;
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            tot += ms;
            fprintf(stderr, "  solve launch %2zu %-22s %8.1f us\n", i, lab[i].c_str(), 1e3f * ms / trep);
        }
        fprintf(stderr, "  solve total %.1f us\n", 1e3f * tot);
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
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
        ENS_CK(cudaFuncSetAttribute(k_sgemm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sg_smem(SG_MAXST)));
        ENS_CK(cudaFuncSetAttribute(k_sgemm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sg_smem(SG_MAXST)));
        ENS_CK(cudaFuncSetAttribute(k_sgemm<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sg_smem(SG_MAXST)));
        ENS_CK(cudaFuncSetAttribute(k_sgemm<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sg_smem(SG_MAXST)));
        ENS_CK(cudaFuncSetAttribute(k_sgemm<4, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sg_smem(SG_MAXST, 64)));
        ENS_CK(cudaFuncSetAttribute(k_sgemm<6, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sg_smem(SG_MAXST, 64)));
        ENS_CK(cudaFuncSetAttribute(k_sgemm<8, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)sg_smem(SG_MAXST, 64)));
        const int64_t ns = c->p.n_slot > 0 ? c->p.n_slot : 1;
        const size_t pbytes = sizeof(double) * 2 * (size_t)ns * SG_R * c->J;
        const size_t tbytes = sizeof(int) * 2 * (size_t)ns * ((c->J + SG_C - 1) / SG_C);
        if (cudaMalloc(&c->partial, pbytes) != cudaSuccess || cudaMalloc(&c->ticket, tbytes) != cudaSuccess) {
            ens_set_error("out of device memory for split-K partials", __FILE__, __LINE__);
            return ENS_ENOMEM;
        }
        ENS_CK(cudaMemset(c->ticket, 0, tbytes));
        // front geometry on the host: children, per-row forward assembly flags
        const int nf = (int)c->p.nfront;
        std::vector<int32_t> fm(nf), fk(nf), par(nf);
        c->idx_off_h.assign((size_t)nf + 1, 0);
        ENS_CK(cudaMemcpy(fm.data(), c->p.f_m, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost));
        ENS_CK(cudaMemcpy(fk.data(), c->p.f_k, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost));
        ENS_CK(cudaMemcpy(par.data(), c->p.f_parent, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost));
        ENS_CK(cudaMemcpy(c->idx_off_h.data(), c->p.f_idx_off, sizeof(int64_t) * (nf + 1), cudaMemcpyDeviceToHost));
        std::vector<uint8_t> hasch(nf, 0);
        for (int f = 0; f < nf; ++f)
            if (par[f] >= 0 && par[f] < nf) hasch[par[f]] = 1;
        // per level: the rows k_finit assembles (pivot rows flagged in bit 31)
        const int nlev = (int)c->level_front_off.size() - 1;
        std::vector<int32_t> rows;
        c->finit_off.assign((size_t)nlev + 1, 0);
        for (int L = 0; L < nlev; ++L) {
            c->finit_off[L] = (int64_t)rows.size();
            for (int f = c->level_front_off[L]; f < c->level_front_off[L + 1]; ++f)
                for (int t = 0; t < fm[f]; ++t)
                    if (t < fk[f] || hasch[f])
                        rows.push_back((int32_t)(c->idx_off_h[f] + t) | (t < fk[f] ? (int32_t)0x80000000 : 0));
        }
        c->finit_off[nlev] = (int64_t)rows.size();
        const int64_t nidx = (int64_t)rows.size();
        uint8_t* d_hasch = nullptr;
        ENS_CK(cudaMalloc(&c->finit_rows, sizeof(int32_t) * (size_t)(nidx > 0 ? nidx : 1)));
        ENS_CK(cudaMemcpy(c->finit_rows, rows.data(), sizeof(int32_t) * (size_t)nidx, cudaMemcpyHostToDevice));
        ENS_CK(cudaMalloc(&d_hasch, (size_t)(nf > 0 ? nf : 1)));
        ENS_CK(cudaMemcpy(d_hasch, hasch.data(), (size_t)nf, cudaMemcpyHostToDevice));
        const int64_t nw = c->p.n_work;
        ENS_CK(cudaMalloc(&c->sitem, sizeof(int4) * 3 * (size_t)(nw > 0 ? nw : 1)));
        if (nw > 0) {
            k_build_sitem<<<(unsigned)((nw + 255) / 256), 256, 0, s>>>(mfdev(c), nw, nf, d_hasch, c->sitem);
            ENS_CKL();
        }
        ENS_CK(cudaStreamSynchronize(s));
        cudaFree(d_hasch);
        c->ws_bytes += pbytes + tbytes + sizeof(int4) * 3 * (size_t)nw + sizeof(int32_t) * (size_t)nidx;
    }
    {
        const int rc = mf_stream_prepare(c);
        if (rc != ENS_OK) return rc;
    }
    SolveIO* io = (SolveIO*)c->solve_io;
    k_set_io<<<1, 1, 0, s>>>(io, r, z);
    ENS_CKL();
    if (!graphs_enabled() || s == 0 || capturing(s)) {   // inside a caller's capture: become its nodes
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
