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
#define SG_KMAX 64 // max inner range per work item (>= symbolic.SPLIT_K); A fragments live in registers
#define SG_T 256    // threads
#define SG_LDB 36   // Bs row stride (= 4 mod 16)

#ifdef SG_PROBE   // diagnostic build: per-CTA phase timestamps of sampled CTAs to stdout
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define SG_T_(i) const unsigned long long tp##i = gtime()
#define SG_PROBE_MAX (1 << 16)
__device__ unsigned long long g_probe[SG_PROBE_MAX][8];
__device__ unsigned int g_probe_n;
extern "C" int ens_probe_dump(const char* path) {   // diagnostic build only
    static unsigned long long h[SG_PROBE_MAX][8];
    unsigned int n = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&n, g_probe_n, sizeof(n));
    n = n < SG_PROBE_MAX ? n : SG_PROBE_MAX;
    cudaMemcpyFromSymbol(h, g_probe, sizeof(unsigned long long) * 8 * n);
    FILE* f = fopen(path, "w");
    if (!f) return -1;
    for (unsigned i = 0; i < n; ++i)
        fprintf(f, "probe %llu %llu %llu %llu %llu %llu %llu %llu\n", h[i][0], h[i][1], h[i][2], h[i][3], h[i][4],
                h[i][5], h[i][6], h[i][7]);
    fclose(f);
    unsigned int z = 0;
    cudaMemcpyToSymbol(g_probe_n, &z, sizeof(z));
    return (int)n;
}
#else
#define SG_T_(i)
#endif

__device__ __forceinline__ void dmma8(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
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
//   [0] = {f, r0, ks, slot}   [1] = {m, k, -, -}   [2] = {off lo/hi, idx_off lo/hi}
__global__ void k_build_sitem(MfDev d, int64_t nwork, int nfront, int4* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nwork) return;
    const int4 w = reinterpret_cast<const int4*>(d.work)[i];
    const int f = (w.x >= 0 && w.x < nfront) ? w.x : 0;
    const int64_t off = d.off[f], io = d.idx_off[f];
    out[3 * i] = w;
    out[3 * i + 1] = make_int4(d.m[f], d.k[f], 0, 0);
    out[3 * i + 2] = make_int4((int)(off & 0xffffffff), (int)(off >> 32), (int)(io & 0xffffffff), (int)(io >> 32));
}

// item = (f, r0, ks, slot)
//   r0 < 0  : forward pivot-only item, pivot rows [t0, t0+64), t0 = -1 - r0
//             (front without contribution block)
//   slot<0  : whole inner range, result applied here
//   slot>=0 : inner range [ks*split_k, ...) of group s0 = slot - ks; the last
//             CTA of the group reduces partial[s0 .. s0+ns) in order
//
// Latency plan (every step is one dependent memory round trip, ~1 us under load):
//   1. item record
//   2. all A fragments of the inner range -> registers; descriptors (idx, gsrc)
//      of the inner range -> shared memory; epilogue descriptors -> registers
//   3. operand values (b / children rows / iterate) -> shared memory; epilogue
//      children rows -> registers
//   4. MMA, then direct stores -- or partial store + fence + ticket + reads of the
//      group's partials (three more trips, split items only)
__global__ void __launch_bounds__(SG_T, 3) k_sgemm(MfDev d, const int4* __restrict__ sitem, int item0,
                                                const double* __restrict__ F, double* __restrict__ FR,
                                                const SolveIO* __restrict__ io, int64_t N, int J, int64_t nidx,
                                                int bwd, int split_k, int kmax, double* __restrict__ partial,
                                                int* __restrict__ ticket, int64_t nslot) {
    SG_T_(0);
    extern __shared__ double sm[];
    __shared__ int s_last;
    __shared__ int4 s_gsrc[SG_KMAX];
    __shared__ int s_idx[SG_KMAX];
    double* Bs = sm;                          // [kpad][SG_LDB]: stride 4 (mod 16) doubles, conflict-free fragments
    const int4* rec = sitem + 3LL * (item0 + blockIdx.x);
    const int4 w0 = rec[0], w1 = rec[1], w2 = rec[2];
    const int r0 = w0.y, ks = w0.z, slot = w0.w;
    const int m = w1.x, k = w1.y;
    const int64_t off = (int64_t)(unsigned)w2.x | ((int64_t)w2.y << 32);
    const int64_t fo = (int64_t)(unsigned)w2.z | ((int64_t)w2.w << 32);
    const int mat = blockIdx.y;
    const int j0 = blockIdx.z * SG_C;
    const int jn = min(SG_C, J - j0);
    const double* base = F + (int64_t)mat * d.storage + off;
    double* FRm = FR + (int64_t)mat * nidx * J;
    double* fr = FRm + fo * J;
    const double* b = io->r + (int64_t)mat * N * J;
    double* x = io->z + (int64_t)mat * N * J;
    const int tid = threadIdx.x;
    const int jt = tid & (SG_C - 1), jok = jt < jn, warp = tid >> 5;
    if (!bwd && r0 < 0) {
        // pivot rows of a front without contribution block: fr[P] = b[P] + children rows
        const int t0 = -1 - r0, nt = min(k - t0, SG_R);
        int4 gq[SG_R / 8];
        int ix[SG_R / 8];
#pragma unroll
        for (int u = 0; u < SG_R / 8; ++u) {
            const int t = min((tid >> 5) + 8 * u, nt - 1);   // clamped: unconditional loads
            gq[u] = *reinterpret_cast<const int4*>(d.gsrc + 4 * (fo + t0 + t));
            ix[u] = d.idx[fo + t0 + t];
        }
        // all loads first, then the stores (fr may alias FRm: interleaving them would serialise the loads)
        double v[SG_R / 8];
#pragma unroll
        for (int u = 0; u < SG_R / 8; ++u) {
            const double* pb = FRm + j0 + (jok ? jt : 0);
            const double bv = b[(int64_t)max(ix[u], 0) * J + j0 + (jok ? jt : 0)];
            v[u] = bv + gsel(pb, gq[u].x, J) + gsel(pb, gq[u].y, J) + gsel(pb, gq[u].z, J) + gsel(pb, gq[u].w, J);
        }
#pragma unroll
        for (int u = 0; u < SG_R / 8; ++u) {
            const int t = (tid >> 5) + 8 * u;
            if (t < nt && jok) fr[(int64_t)(t0 + t) * J + j0 + jt] = v[u];
        }
        return;
    }
    const int rbase = bwd ? r0 : k + r0;
    const int nr = min(SG_R, (bwd ? k : m) - rbase);
    const int K = bwd ? m : k;
    const int kbeg = slot < 0 ? 0 : ks * split_k;
    const int kend = slot < 0 ? K : min(K, kbeg + split_k);
    const int kc = kend - kbeg;               // <= kmax <= SG_KMAX by construction of the schedule
    const int kpad = (kc + 3) & ~3;
    // (2) descriptors of the inner range -> shared memory
    for (int t = tid; t < kc; t += SG_T) {
        const int64_t r = fo + kbeg + t;
        if (bwd) {
            s_idx[t] = (kbeg + t >= k) ? d.idx[r] : -1;
        } else {
            s_idx[t] = d.idx[r];
            s_gsrc[t] = *reinterpret_cast<const int4*>(d.gsrc + 4 * r);
        }
    }
    // fp64 tensor-core MMA (m8n8k4): warp w owns rows 8w..8w+7 and every 8-column tile.
    // A fragments (lane = row g, inner q) go straight from the front into registers:
    // 8 rows x 32 contiguous bytes per warp load, the whole inner range in flight.
    const int lane = tid & 31, g = lane >> 2, q = lane & 3;
    const int row = 8 * warp + g;
    const bool row_ok = row < nr;
    const double* arow = base + (int64_t)(rbase + (row_ok ? row : 0)) * m + kbeg + q;
    double a[SG_KMAX / 4];
    if (bwd) {
#pragma unroll
        for (int u = 0; u < SG_KMAX / 4; ++u) a[u] = (row_ok && 4 * u + q < kc) ? __ldg(arow + 4 * u) : 0.0;
    }
    // epilogue descriptors (accumulator layout: row `row`, columns 8ct + 2q + {0,1})
    const int xrow = (bwd && row_ok) ? d.idx[fo + rbase + row] : 0;
    const int4 eg = (!bwd && row_ok) ? *reinterpret_cast<const int4*>(d.gsrc + 4 * (fo + rbase + row))
                                     : make_int4(-1, -1, -1, -1);
    __syncthreads();
    SG_T_(1);
    // (3) operand values -> shared memory
    if (bwd) {
        // B = [fr[P]; x[C]] rows of the inner range
        for (int kk = tid >> 5; kk < kc; kk += SG_T / SG_C) {
            const int t = kbeg + kk;
            const double* src = (t < k) ? fr + (int64_t)t * J + j0 + jt : x + (int64_t)s_idx[kk] * J + j0 + jt;
            cp_async8(&Bs[kk * SG_LDB + jt], jok ? src : fr, jok);
        }
        cp_async_commit();
    }
    // contribution-block rows' children sums for the forward epilogue
    double init[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    if (!bwd && row_ok) {
#pragma unroll
        for (int ct = 0; ct < 4; ++ct)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = 8 * ct + 2 * q + e;
                if (col >= jn) continue;
                const double* pe = FRm + j0 + col;
                init[ct][e] = gsel(pe, eg.x, J) + gsel(pe, eg.y, J) + gsel(pe, eg.z, J) + gsel(pe, eg.w, J);
            }
    }
    if (!bwd) {
        // B = b[P] + children rows; one row tile per front persists fr[P] for the backward pass
        const bool store_piv = (r0 == 0);
        // all loads first, then the stores (fr may alias FRm: interleaving them would serialise the loads)
        double v[SG_KMAX / 8];
#pragma unroll
        for (int u = 0; u < SG_KMAX / 8; ++u) {
            const int kk = warp + 8 * u;
            const int kq = min(kk, kc - 1);
            const int4 gq = s_gsrc[kq];
            const double* pb = FRm + j0 + (jok ? jt : 0);
            const double bv = b[(int64_t)s_idx[kq] * J + j0 + (jok ? jt : 0)];
            const double sv = bv + gsel(pb, gq.x, J) + gsel(pb, gq.y, J) + gsel(pb, gq.z, J) + gsel(pb, gq.w, J);
            v[u] = (kk < kc && jok) ? sv : 0.0;
        }
#pragma unroll
        for (int u = 0; u < SG_KMAX / 8; ++u) {
            const int kk = warp + 8 * u;
            if (kk < kc) {
                Bs[kk * SG_LDB + jt] = v[u];
                if (store_piv && jok) fr[(int64_t)(kbeg + kk) * J + j0 + jt] = v[u];
            }
        }
    }
    if (!bwd) {   // forward: A after the operand gather (the gather needs the registers)
#pragma unroll
        for (int u = 0; u < SG_KMAX / 4; ++u) a[u] = (row_ok && 4 * u + q < kc) ? __ldg(arow + 4 * u) : 0.0;
    }
    // zero the K padding (kc -> multiple of 4) of B (A's padding is zero-filled in registers)
    for (int e = tid; e < (kpad - kc) * SG_C; e += SG_T) Bs[(kc + e / SG_C) * SG_LDB + e % SG_C] = 0.0;
    cp_async_wait_all();
    __syncthreads();
    SG_T_(2);
    // (4) MMA
    const int nct = (jn + 7) >> 3;
    double dacc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    const double* bp = Bs + q * SG_LDB + g;
#pragma unroll
    for (int u = 0; u < SG_KMAX / 4; ++u) {
        if (4 * u < kpad) {
#pragma unroll
            for (int ct = 0; ct < 4; ++ct)
                if (ct < nct) dmma8(dacc[ct][0], dacc[ct][1], a[u], bp[4 * u * SG_LDB + 8 * ct]);
        }
    }
#ifdef SG_PROBE
    __syncthreads();
    SG_T_(3);
#define SG_END(tag)                                                                                      \
    if (tid == 0 && blockIdx.y == 0 && blockIdx.z == 0) {                                                \
        const unsigned i_ = atomicAdd(&g_probe_n, 1u);                                                   \
        if (i_ < SG_PROBE_MAX) {                                                                         \
            unsigned long long* o_ = g_probe[i_];                                                        \
            o_[0] = (unsigned long long)bwd * 1000000 + (unsigned long long)kmax * 1000 + (tag);         \
            o_[1] = blockIdx.x; o_[2] = kc; o_[3] = tp0; o_[4] = tp1 - tp0; o_[5] = tp2 - tp1;            \
            o_[6] = tp3 - tp2; o_[7] = gtime() - tp3;                                                    \
        }                                                                                                \
    }
#else
#define SG_END(tag)
#endif
    if (slot >= 0) {
        // split: publish the partial; the last CTA of the group sums the group's
        // partials in ks order (deterministic) and applies the epilogue
        double* pw = partial + (((int64_t)mat * nslot + slot) * SG_R + row) * J + j0;
        if (row_ok) {
#pragma unroll
            for (int ct = 0; ct < 4; ++ct)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (8 * ct + 2 * q + e < jn) pw[8 * ct + 2 * q + e] = dacc[ct][e];
        }
        __threadfence();
        __syncthreads();
        const int s0 = slot - ks;
        const int ns = (K + split_k - 1) / split_k;
        const int tk = (int)(((int64_t)mat * nslot + s0) * gridDim.z + blockIdx.z);
        if (tid == 0) s_last = (atomicAdd(ticket + tk, 1) == ns - 1);
        __syncthreads();
        if (!s_last) {
            SG_END(1);
            return;
        }
        __threadfence();
        if (tid == 0) ticket[tk] = 0;   // ready for the next solve / graph replay
        if (!row_ok) return;
        const double* pr = partial + (((int64_t)mat * nslot + s0) * SG_R + row) * J + j0;
        const int64_t pst = (int64_t)SG_R * J;
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) dacc[ct][0] = dacc[ct][1] = 0.0;
#pragma unroll 2
        for (int qq = 0; qq < ns; ++qq) {
#pragma unroll
            for (int ct = 0; ct < 4; ++ct)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (8 * ct + 2 * q + e < jn) dacc[ct][e] += __ldcg(pr + qq * pst + 8 * ct + 2 * q + e);
        }
    }
    if (!row_ok) return;
#pragma unroll
    for (int ct = 0; ct < 4; ++ct)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int col = 8 * ct + 2 * q + e;
            if (col >= jn) continue;
            if (bwd)
                x[(int64_t)xrow * J + j0 + col] = -dacc[ct][e];
            else
                FRm[(fo + rbase + row) * J + j0 + col] = init[ct][e] - dacc[ct][e];
        }
    SG_END(slot >= 0 ? 2 : 0);
}

static size_t sg_smem(int kmax) {
    const size_t kpad = (kmax + 3) & ~3;
    return sizeof(double) * kpad * SG_LDB;
}

static bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    return st != cudaStreamCaptureStatusNone;
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
            const int op = (int)q[0], off = (int)q[2], n = (int)q[3], kmax = (int)q[4];
            if (n == 0) continue;
            if ((op != SOP_FGEMM && op != SOP_BGEMM) || kmax > SG_KMAX || kmax < 1) {
                ens_set_error("bad solve schedule row", __FILE__, __LINE__);
                return ENS_EINVAL;
            }
            for (int rep = 0; rep < (timing ? trep : 1); ++rep) {   // launches are idempotent
                k_sgemm<<<dim3(n, 2, zc), SG_T, sg_smem(kmax), s>>>(d, c->sitem, off, c->fronts, c->frvec, io, N,
                                                                   J, nidx, op == SOP_BGEMM, sk, kmax, c->partial,
                                                                   c->ticket, nslot);
                ENS_CKL();
            }
            ++cnt;
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
        ENS_CK(cudaFuncSetAttribute(k_sgemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sg_smem(SG_KMAX)));
        const int64_t ns = c->p.n_slot > 0 ? c->p.n_slot : 1;
        const size_t pbytes = sizeof(double) * 2 * (size_t)ns * SG_R * c->J;
        const size_t tbytes = sizeof(int) * 2 * (size_t)ns * ((c->J + SG_C - 1) / SG_C);
        if (cudaMalloc(&c->partial, pbytes) != cudaSuccess || cudaMalloc(&c->ticket, tbytes) != cudaSuccess) {
            ens_set_error("out of device memory for split-K partials", __FILE__, __LINE__);
            return ENS_ENOMEM;
        }
        ENS_CK(cudaMemset(c->ticket, 0, tbytes));
        const int64_t nw = c->p.n_work;
        ENS_CK(cudaMalloc(&c->sitem, sizeof(int4) * 3 * (size_t)(nw > 0 ? nw : 1)));
        if (nw > 0) {
            k_build_sitem<<<(unsigned)((nw + 255) / 256), 256, 0, s>>>(mfdev(c), nw, (int)c->p.nfront, c->sitem);
            ENS_CKL();
        }
        c->ws_bytes += pbytes + tbytes + sizeof(int4) * 3 * (size_t)nw;
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
