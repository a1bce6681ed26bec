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
