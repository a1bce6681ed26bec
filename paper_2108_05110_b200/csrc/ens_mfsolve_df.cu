// Dataflow multifrontal solve (sm_100a, fp64): the whole forward (and the whole
// backward) sweep as ONE persistent launch instead of one launch per tree level.
//
// Work is a task list in topological order (children's tasks before their
// parent's).  Persistent CTAs claim tasks from a global counter; a task waits
// on per-front dependency counters filled by the tasks it depends on, so a
// front starts as soon as ITS children are done -- no level barrier, no
// per-level launch.  Deadlock-free by construction: a task only waits on tasks
// earlier in the list, which were claimed by CTAs that are already running.
//
//   forward  FINIT(f, rows)  fr[rows] = (b at pivots) + children's contribution rows
//                            waits: every row block of f's children  (c_fin[f])
//            GEMM(f, r0, ks) fr[C rows] -= F[C, P] fr[P]             (c_init[f])
//                            signals the parent's c_fin once per row block
//   backward GEMM(f, r0, ks) x[P rows] = -[F[P,P] F[P,C]] [fr[P]; x[C]]
//                            waits: every pivot row block of the parent (c_bwd)
//
// Data produced inside the launch by other CTAs is read through L2 only
// (cp.async.cg / ld.global.cg), so no SM can hold a stale L1 line of it.
// Split inner ranges keep the deterministic last-CTA reduction of k_sgemm.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ens_internal.cuh"
#include "ens_mf_common.cuh"

#define DF_R 64      // rows per GEMM task
#define DF_C 32      // member columns held in a B row (J <= 32 on this path)
#define DF_T 256     // threads
#define DF_KC 32     // inner chunk
#define DF_LDA 36    // stride = 4 (mod 16) doubles: conflict-free m8n8k4 fragments
#define DF_LDB 36
#define DF_STAGE (DF_R * DF_LDA + DF_KC * DF_LDB)
#define DF_NST 2     // pipeline stages
#define DF_KMAX 256  // max inner range of a task (>= plan split_k)
#define DF_FROWS 64  // rows per FINIT task

enum { DF_HASCH = 1, DF_FINIT = 2, DF_FRONT = 4 };   // FRONT: assembly + the front's only GEMM item

struct DfTask {
    int4 a;   // {f, r0, ks, slot}          FINIT: {f, first row, -, -}
    int4 b;   // {m, k, flags, FINIT rows}
    int4 c;   // {off lo, off hi, fo lo, fo hi}
    int4 d;   // {wait counter, wait target, signal counter, -}  (-1: none)
};

struct DfIO {
    const double* r;
    double* z;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void df_cp8(double* s, const double* g, bool pred) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void df_cp16cg(double* s, const double* g, bool pred) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void df_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void df_wait(int n) {
    if (n <= 0) asm volatile("cp.async.wait_group 0;\n" ::);
    else if (n == 1) asm volatile("cp.async.wait_group 1;\n" ::);
    else asm volatile("cp.async.wait_group 2;\n" ::);
}
__device__ __forceinline__ void df_mma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}
#ifdef DF_PROBE   // diagnostic build: per-task timestamps (claim, dependency met, done)
#define DF_PMAX (1 << 17)
__device__ unsigned long long g_dfp[DF_PMAX][4];
__device__ unsigned int g_dfp_n;
__device__ __forceinline__ unsigned long long df_gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
extern "C" int ens_df_probe_dump(const char* path) {
    static unsigned long long h[DF_PMAX][4];
    unsigned int n = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&n, g_dfp_n, sizeof(n));
    n = n < DF_PMAX ? n : DF_PMAX;
    cudaMemcpyFromSymbol(h, g_dfp, sizeof(unsigned long long) * 4 * n);
    FILE* f = fopen(path, "w");
    if (!f) return -1;
    for (unsigned i = 0; i < n; ++i) fprintf(f, "%llu %llu %llu %llu\n", h[i][0], h[i][1], h[i][2], h[i][3]);
    fclose(f);
    unsigned int z = 0;
    cudaMemcpyToSymbol(g_dfp_n, &z, sizeof(z));
    return (int)n;
}
#endif

// L2-coherent 16-byte load with a clamped (always valid) row
__device__ __forceinline__ double2 df_ldcg2(const double2* p) { return __ldcg(p); }

// rows [r0, r0 + nrows) of a front: (b at pivots) + children's contribution rows
__device__ __forceinline__ void df_finit(double* __restrict__ FRm, const double* __restrict__ b,
                                         const int32_t* __restrict__ idx, const int32_t* __restrict__ gsrc,
                                         int64_t fo, int r0, int nrows, int k, int H) {
    const double2* F2 = reinterpret_cast<const double2*>(FRm);
    const double2* b2 = reinterpret_cast<const double2*>(b);
    for (int e0 = 0; e0 < nrows * H; e0 += 4 * DF_T) {
        double2 v[4];
        int rows_[4], jp_[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + threadIdx.x + DF_T * u;
            const bool ok = e < nrows * H;
            const int rr = ok ? e / H : 0, jp = ok ? e - rr * H : 0;
            const int64_t row = fo + r0 + rr;
            const int4 gq = *reinterpret_cast<const int4*>(gsrc + 4 * row);
            const double2 bv = b2[(int64_t)max(idx[row], 0) * H + jp];
            const int src[4] = {gq.x, gq.y, gq.z, gq.w};
            double2 sm2 = make_double2(0.0, 0.0);
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const double2 cv = __ldcg(F2 + (int64_t)max(src[w], 0) * H + jp);
                if (src[w] >= 0) {
                    sm2.x += cv.x;
                    sm2.y += cv.y;
                }
            }
            if (r0 + rr < k) sm2 = make_double2(bv.x + sm2.x, bv.y + sm2.y);
            v[u] = sm2;
            rows_[u] = ok ? rr : -1;
            jp_[u] = jp;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (rows_[u] >= 0) reinterpret_cast<double2*>(FRm)[(fo + r0 + rows_[u]) * H + jp_[u]] = v[u];
    }
}

// One task = one work item for BOTH systems (V, W): halves the per-task cost
// (claim, record, dependency check, publish).  The next task is claimed and its
// record fetched while the current one runs.
template <int NCT>
#ifndef DF_MINB
#define DF_MINB 3
#endif
__global__ void __launch_bounds__(DF_T, DF_MINB)
    k_df_solve(const DfTask* __restrict__ tasks, int ntask, int* __restrict__ head, int* __restrict__ cnt,
               int* __restrict__ err, const double* __restrict__ F, int64_t storage, double* __restrict__ FR,
               const DfIO* __restrict__ iop, int64_t N, int J, int64_t nidx, const int32_t* __restrict__ idx,
               const int32_t* __restrict__ gsrc, int bwd, int split_k, double* __restrict__ partial,
               int* __restrict__ ticket, int64_t nslot) {
    extern __shared__ double sm[];
    __shared__ int s_last;
    __shared__ int s_item[2];
    __shared__ DfTask s_task[2];
    __shared__ int s_idx[DF_KMAX];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
    const int H = J >> 1;
    const DfIO io = *iop;
    if (tid == 0) {
        const int it = atomicAdd(head, 1);
        s_item[0] = it;
        if (it < ntask) s_task[0] = tasks[it];
    }
    __syncthreads();
    for (int cur = 0;; cur ^= 1) {
        const int gi = s_item[cur];
        if (gi >= ntask) return;
        const DfTask tk = s_task[cur];
#ifdef DF_PROBE
        const unsigned long long tp0 = df_gt();
#endif
        if (tid == 0) {   // claim + fetch the next task while this one runs
            const int it = atomicAdd(head, 1);
            s_item[cur ^ 1] = it;
            if (it < ntask) s_task[cur ^ 1] = tasks[it];
        }
        // ---- dependency wait (one thread spins, the barrier releases the CTA) ----
        if (tk.d.x >= 0 && tid == 0) {
            long long spins = 0;
            while (ld_acquire(cnt + tk.d.x) < tk.d.y) {
                __nanosleep(32);
                if (++spins > (1LL << 22)) {   // a broken schedule must not hang the GPU
                    atomicExch(err, 1);
                    break;
                }
            }
        }
        __syncthreads();
        __threadfence();
#ifdef DF_PROBE
        const unsigned long long tp1 = df_gt();
#endif
        const int r0 = tk.a.y, ks = tk.a.z, slot = tk.a.w;
        const int m = tk.b.x, k = tk.b.y, flags = tk.b.z;
        const int64_t off = (int64_t)(unsigned)tk.c.x | ((int64_t)tk.c.y << 32);
        const int64_t fo = (int64_t)(unsigned)tk.c.z | ((int64_t)tk.c.w << 32);
        bool signal = tk.d.z >= 0;
        if (flags & DF_FINIT) {
            const int fr0 = (flags & DF_FRONT) ? 0 : r0;
            for (int mat = 0; mat < 2; ++mat)
                df_finit(FR + (int64_t)mat * nidx * J, io.r + (int64_t)mat * N * J, idx, gsrc, fo, fr0, tk.b.w, k, H);
            if (!(flags & DF_FRONT)) goto publish;
            __threadfence();   // whole-front task: its GEMM reads the rows just assembled (through L2)
            __syncthreads();
        }
        {
            // ---- GEMM item: pipelined cp.async mainloop + fp64 tensor cores, V then W ----
            const int rbase = bwd ? r0 : k + r0;
            const int nr = min(DF_R, (bwd ? k : m) - rbase);
            const int K = bwd ? m : k;
            const int split = (flags & DF_FRONT) ? split_k : tk.b.w;   // the level's split length
            const int kbeg = slot < 0 ? 0 : ks * split;
            const int kend = slot < 0 ? K : min(K, kbeg + split);
            const int kc = kend - kbeg;
            const int nch = (kc + DF_KC - 1) / DF_KC;
            const int row = 8 * warp + g;
            const bool row_ok = row < nr;
            if (bwd)
                for (int t = tid; t < kc; t += DF_T) s_idx[t] = (kbeg + t >= k) ? idx[fo + kbeg + t] : 0;
            const int xrow = (bwd && row_ok) ? idx[fo + rbase + row] : 0;
            __syncthreads();   // s_idx
            auto store_result = [&](int mat, const double (&dacc)[4][2]) {
                if (!row_ok) return;
                double* FRm = FR + (int64_t)mat * nidx * J;
                double* x = io.z + (int64_t)mat * N * J;
                double* pc = FRm + (fo + rbase + row) * J;
#pragma unroll
                for (int ct = 0; ct < NCT; ++ct)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int col = 8 * ct + 2 * q + e;
                        if (col >= J) continue;
                        if (bwd) {
                            x[(int64_t)xrow * J + col] = -dacc[ct][e];
                        } else {
                            const double init = (flags & DF_HASCH) ? __ldcg(pc + col) : 0.0;
                            pc[col] = init - dacc[ct][e];
                        }
                    }
            };
            auto store_partial = [&](int mat, const double (&dacc)[4][2]) {
                if (!row_ok) return;
                double* pw = partial + (((int64_t)mat * nslot + slot) * DF_R + row) * J;
#pragma unroll
                for (int ct = 0; ct < NCT; ++ct)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        if (8 * ct + 2 * q + e < J) pw[8 * ct + 2 * q + e] = dacc[ct][e];
            };
            for (int mat = 0; mat < 2; ++mat) {
                const double* base = F + (int64_t)mat * storage + off;
                double* FRm = FR + (int64_t)mat * nidx * J;
                double* fr = FRm + fo * J;
                double* x = io.z + (int64_t)mat * N * J;
                auto issue = [&](int c) {
                    double* As = sm + (c % DF_NST) * DF_STAGE;
                    double* Bsb = As + DF_R * DF_LDA;
#pragma unroll
                    for (int i = 0; i < DF_R * DF_KC / DF_T; ++i) {
                        const int e = tid + DF_T * i, r = e / DF_KC, kk = e % DF_KC, kg = c * DF_KC + kk;
                        const bool ok = r < nr && kg < kc;
                        df_cp8(&As[r * DF_LDA + kk], ok ? base + (int64_t)(rbase + r) * m + kbeg + kg : base, ok);
                    }
#pragma unroll
                    for (int i = 0; i < DF_KC * (DF_C / 2) / DF_T; ++i) {
                        const int e = tid + DF_T * i, kk = e / (DF_C / 2), jp = e % (DF_C / 2), kg = c * DF_KC + kk;
                        const bool ok = jp < H && kg < kc;
                        const int kq = min(kg, kc - 1), t = kbeg + kq;
                        const double* src = (!bwd || t < k) ? fr + (int64_t)t * J + 2 * jp
                                                            : x + (int64_t)s_idx[kq] * J + 2 * jp;
                        df_cp16cg(&Bsb[kk * DF_LDB + 2 * jp], ok ? src : fr, ok);
                    }
                };
                for (int c = 0; c < DF_NST - 1; ++c) {
                    if (c < nch) issue(c);
                    df_commit();
                }
                double dacc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
                for (int c = 0; c < nch; ++c) {
                    df_wait(DF_NST - 2);
                    __syncthreads();
                    if (c + DF_NST - 1 < nch) issue(c + DF_NST - 1);
                    df_commit();
                    const double* As = sm + (c % DF_NST) * DF_STAGE;
                    const double* ap = As + row * DF_LDA + q;
                    const double* bp = As + DF_R * DF_LDA + q * DF_LDB + g;
                    const int ksteps = (min(DF_KC, kc - c * DF_KC) + 3) >> 2;
                    if (ksteps == DF_KC / 4) {
#pragma unroll
                        for (int u = 0; u < DF_KC / 4; ++u) {
                            const double av = ap[4 * u];
#pragma unroll
                            for (int ct = 0; ct < NCT; ++ct)
                                df_mma(dacc[ct][0], dacc[ct][1], av, bp[4 * u * DF_LDB + 8 * ct]);
                        }
                    } else {
#pragma unroll 2
                        for (int u = 0; u < ksteps; ++u) {
                            const double av = ap[4 * u];
#pragma unroll
                            for (int ct = 0; ct < NCT; ++ct)
                                df_mma(dacc[ct][0], dacc[ct][1], av, bp[4 * u * DF_LDB + 8 * ct]);
                        }
                    }
                }
                df_wait(0);
                __syncthreads();   // stage buffers free for the next pass
                if (slot >= 0)
                    store_partial(mat, dacc);
                else
                    store_result(mat, dacc);
            }
            if (slot >= 0) {
                // split inner range: the group's last CTA sums the partials in order (both systems)
                __threadfence();
                __syncthreads();
                const int s0 = slot - ks;
                const int ns = (K + split - 1) / split;
                if (tid == 0) s_last = (atomicAdd(ticket + s0, 1) == ns - 1);
                __syncthreads();
                signal = signal && s_last;
                if (s_last) {
                    __threadfence();
                    if (tid == 0) ticket[s0] = 0;
                    const int64_t pst = (int64_t)DF_R * J;
                    for (int mat = 0; mat < 2; ++mat) {
                        const double* pr = partial + (((int64_t)mat * nslot + s0) * DF_R + row) * J;
                        double dacc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
                        if (row_ok) {
#pragma unroll 4
                            for (int qq = 0; qq < ns; ++qq) {
#pragma unroll
                                for (int ct = 0; ct < NCT; ++ct)
#pragma unroll
                                    for (int e = 0; e < 2; ++e)
                                        if (8 * ct + 2 * q + e < J)
                                            dacc[ct][e] += __ldcg(pr + qq * pst + 8 * ct + 2 * q + e);
                            }
                        }
                        store_result(mat, dacc);
                    }
                }
            }
        }
    publish:
        // ---- publish: results visible device-wide before the counter moves ----
        __threadfence();
        __syncthreads();
        if (signal && tid == 0) atomicAdd(cnt + tk.d.z, 1);
#ifdef DF_PROBE
        if (tid == 0) {
            const unsigned i_ = atomicAdd(&g_dfp_n, 1u);
            if (i_ < DF_PMAX) {
                g_dfp[i_][0] = (unsigned long long)bwd << 62 | (unsigned long long)blockIdx.x << 40 | (unsigned)gi;
                g_dfp[i_][1] = tp0;
                g_dfp[i_][2] = tp1;
                g_dfp[i_][3] = df_gt();
            }
        }
#endif
    }
}

// ---------------------------------------------------------------------------
// host: task lists (once per plan), launches
// ---------------------------------------------------------------------------
struct DfPlan {
    DfTask* fwd = nullptr;
    DfTask* bwd = nullptr;
    int nfwd = 0, nbwd = 0, ncnt = 0;
    int* ctl = nullptr;   // [head fwd, head bwd, err, pad] + counters[ncnt]
    int grid = 0;
    DfIO* io = nullptr;
};

bool df_enabled(const ens_ctx* c) {
    // opt-in (ENS_SOLVE_DF=1): measured slower than the per-level launches at C2
    const char* e = std::getenv("ENS_SOLVE_DF");
    if (!(e && e[0] == '1')) return false;
    return (c->J & 1) == 0 && c->J <= DF_C && c->p.split_k <= DF_KMAX;
}

int df_build(ens_ctx* c, cudaStream_t s) {
    const int nf = (int)c->p.nfront;
    std::vector<int32_t> fm(nf), fk(nf), par(nf);
    std::vector<int64_t> foff(nf), fio(nf + 1);
    ENS_CK(cudaMemcpy(fm.data(), c->p.f_m, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost));
    ENS_CK(cudaMemcpy(fk.data(), c->p.f_k, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost));
    ENS_CK(cudaMemcpy(par.data(), c->p.f_parent, sizeof(int32_t) * nf, cudaMemcpyDeviceToHost));
    ENS_CK(cudaMemcpy(foff.data(), c->p.f_off, sizeof(int64_t) * nf, cudaMemcpyDeviceToHost));
    ENS_CK(cudaMemcpy(fio.data(), c->p.f_idx_off, sizeof(int64_t) * (nf + 1), cudaMemcpyDeviceToHost));
    std::vector<int32_t> work((size_t)c->p.n_work * 4);
    if (c->p.n_work > 0)
        ENS_CK(cudaMemcpy(work.data(), c->p.work, sizeof(int32_t) * work.size(), cudaMemcpyDeviceToHost));
    std::vector<uint8_t> hasch(nf, 0);
    for (int f = 0; f < nf; ++f)
        if (par[f] >= 0) hasch[par[f]] = 1;
    // dependency counters: c_fin [0, nf), c_init [nf, 2nf), c_bwd [2nf, 3nf)
    auto rb = [](int n) { return (n + DF_R - 1) / DF_R; };
    std::vector<int> target_fin(nf, 0), nfin(nf, 0);
    for (int f = 0; f < nf; ++f)
        if (par[f] >= 0) target_fin[par[f]] += rb(fm[f] - fk[f]);
    auto mk = [&](int f, int a1, int a2, int a3, int flags, int rows, int wi, int wt, int si) {
        DfTask t;
        t.a = make_int4(f, a1, a2, a3);
        t.b = make_int4(fm[f], fk[f], flags | (hasch[f] ? DF_HASCH : 0), rows);
        t.c = make_int4((int)(foff[f] & 0xffffffff), (int)(foff[f] >> 32), (int)(fio[f] & 0xffffffff),
                        (int)(fio[f] >> 32));
        t.d = make_int4(wi, wt, si, 0);
        return t;
    };
    const int nlev = (int)c->level_front_off.size() - 1;
    std::vector<std::vector<int64_t>> fitems(nlev), bitems(nlev);
    std::vector<int> fsplit(nlev, 1), bsplit(nlev, 1);
    for (size_t i = 0; i + 5 <= c->sched_fwd.size(); i += 5) {
        for (int u = 0; u < (int)c->sched_fwd[i + 3]; ++u) fitems[c->sched_fwd[i + 1]].push_back(c->sched_fwd[i + 2] + u);
        fsplit[c->sched_fwd[i + 1]] = std::max(1, (int)c->sched_fwd[i + 4]);
    }
    for (size_t i = 0; i + 5 <= c->sched_bwd.size(); i += 5) {
        for (int u = 0; u < (int)c->sched_bwd[i + 3]; ++u) bitems[c->sched_bwd[i + 1]].push_back(c->sched_bwd[i + 2] + u);
        bsplit[c->sched_bwd[i + 1]] = std::max(1, (int)c->sched_bwd[i + 4]);
    }
    std::vector<DfTask> fwd, bwd;
    for (int L = 0; L < nlev; ++L) {
        // whole-front tasks where the front has exactly one unsplit GEMM item
        std::vector<int> nitem(nf, 0);
        for (int64_t it : fitems[L])
            if (work[4 * it + 1] >= 0) ++nitem[work[4 * it]];
        std::vector<uint8_t> whole(nf, 0);
        for (int64_t it : fitems[L]) {
            const int* w = &work[4 * it];
            if (w[1] >= 0 && nitem[w[0]] == 1 && w[3] < 0) whole[w[0]] = 1;
        }
        for (int f = c->level_front_off[L]; f < c->level_front_off[L + 1]; ++f) {
            const int rows = hasch[f] ? fm[f] : fk[f];
            const int wi = target_fin[f] > 0 ? f : -1;
            if (whole[f]) {
                fwd.push_back(mk(f, 0, 0, -1, DF_FINIT | DF_FRONT, rows, wi, target_fin[f], par[f]));
                continue;
            }
            for (int r = 0; r < rows; r += DF_FROWS) {
                fwd.push_back(mk(f, r, 0, 0, DF_FINIT, std::min(DF_FROWS, rows - r), wi, target_fin[f], nf + f));
                ++nfin[f];
            }
        }
        for (int64_t it : fitems[L]) {
            const int* w = &work[4 * it];
            if (w[1] < 0 || whole[w[0]]) continue;   // pivot-only rows: FINIT; whole fronts: above
            const int f = w[0];
            fwd.push_back(mk(f, w[1], w[2], w[3], 0, fsplit[L], nf + f, nfin[f], par[f]));
        }
    }
    for (int L = nlev - 1; L >= 0; --L) {
        for (int64_t it : bitems[L]) {
            const int* w = &work[4 * it];
            const int f = w[0], p = par[f];
            bwd.push_back(mk(f, w[1], w[2], w[3], 0, bsplit[L], p >= 0 ? 2 * nf + p : -1, p >= 0 ? rb(fk[p]) : 0,
                             2 * nf + f));
        }
    }
    DfPlan* P = new DfPlan;
    P->nfwd = (int)fwd.size();
    P->nbwd = (int)bwd.size();
    P->ncnt = 3 * nf;
    ENS_CK(cudaMalloc(&P->fwd, sizeof(DfTask) * std::max<size_t>(1, fwd.size())));
    ENS_CK(cudaMalloc(&P->bwd, sizeof(DfTask) * std::max<size_t>(1, bwd.size())));
    ENS_CK(cudaMemcpy(P->fwd, fwd.data(), sizeof(DfTask) * fwd.size(), cudaMemcpyHostToDevice));
    ENS_CK(cudaMemcpy(P->bwd, bwd.data(), sizeof(DfTask) * bwd.size(), cudaMemcpyHostToDevice));
    ENS_CK(cudaMalloc(&P->ctl, sizeof(int) * (4 + (size_t)P->ncnt)));
    ENS_CK(cudaMemset(P->ctl, 0, sizeof(int) * (4 + (size_t)P->ncnt)));
    const size_t smem = sizeof(double) * DF_NST * DF_STAGE;
    const int nct = (c->J + 7) / 8;
    int occ = 0;
#define DFA(NC)                                                                                        \
    {                                                                                                  \
        ENS_CK(cudaFuncSetAttribute(k_df_solve<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        ENS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_df_solve<NC>, DF_T, smem));       \
    }
    if (nct == 1) DFA(1) else if (nct == 2) DFA(2) else if (nct == 3) DFA(3) else DFA(4)
#undef DFA
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    P->grid = std::max(1, occ) * sms;
    c->df = P;
    c->ws_bytes += sizeof(DfTask) * (fwd.size() + bwd.size()) + sizeof(int) * (4 + (size_t)P->ncnt);
    (void)s;
    return ENS_OK;
}

void df_free(ens_ctx* c) {
    DfPlan* P = (DfPlan*)c->df;
    if (!P) return;
    cudaFree(P->fwd);
    cudaFree(P->bwd);
    cudaFree(P->ctl);
    delete P;
    c->df = nullptr;
}

// forward + backward sweeps; `io` is the solve's {r, z} device pointer table
int df_solve_launches(ens_ctx* c, cudaStream_t s, const void* io, int64_t* nlaunch) {
    if (!c->df) {
        const int rc = df_build(c, s);
        if (rc != ENS_OK) return rc;
    }
    DfPlan* P = (DfPlan*)c->df;
    const int J = c->J, nct = (J + 7) / 8;
    const size_t smem = sizeof(double) * DF_NST * DF_STAGE;
    ENS_CK(cudaMemsetAsync(P->ctl, 0, sizeof(int) * (4 + (size_t)P->ncnt), s));
    for (int dir = 0; dir < 2; ++dir) {
        const DfTask* tasks = dir ? P->bwd : P->fwd;
        const int nt = dir ? P->nbwd : P->nfwd;
        if (nt == 0) continue;
        const unsigned grid = (unsigned)std::min(P->grid, nt);
#define DFL(NC)                                                                                                 \
    k_df_solve<NC><<<grid, DF_T, smem, s>>>(tasks, nt, P->ctl + dir, P->ctl + 4, P->ctl + 2, c->fronts,           \
                                            c->p.front_storage, c->frvec, (const DfIO*)io, c->n_total, J,          \
                                            c->p.n_idx, c->p.f_idx, c->p.gsrc, dir, c->p.split_k, c->partial,       \
                                            c->ticket, c->p.n_slot)
        if (nct == 1) DFL(1);
        else if (nct == 2) DFL(2);
        else if (nct == 3) DFL(3);
        else DFL(4);
#undef DFL
        ENS_CKL();
        ++*nlaunch;
    }
    return ENS_OK;
}

// device error flag of the last solve (a dependency wait that timed out)
int df_error(ens_ctx* c) {
    DfPlan* P = (DfPlan*)c->df;
    if (!P) return 0;
    int e = 0;
    cudaMemcpy(&e, P->ctl + 2, sizeof(int), cudaMemcpyDeviceToHost);
    return e;
}
