// Saddle-operator SpMM for both sub-step systems (the Krylov core), fp64, sm_100a.
//
//   y = K x   (mode 0)   or   y = b - K x   (mode 1), per system m in {V, W}:
//   velocity node i, comp c:  sum_k A_m[k] x[2 col_k + c]  -  sum_t (bx|by)_t x[p_t]
//   pressure row p:           sum_t bx_t x[2 n_t] + by_t x[2 n_t + 1]
//   identity rows (cflag):    x            (Dirichlet rows / pin, stepper.py:214-215)
// which is exactly the reference's assembled matrix (stepper.py:208-215) applied
// to all J member columns at once (linalg.py:111-118 uses the same product).
//
// Layout: member-minor blocks, so one node's (x, y) values for all members are
// 2J contiguous doubles -> each nonzero gathers one coalesced segment that
// serves every member and both components.  A segment of S lanes owns a row;
// the row's column indices and values are fetched lane-parallel once and
// broadcast with shuffles, so the x gathers of 4 consecutive nonzeros are
// independent and in flight together (memory-level parallelism instead of an
// index->gather dependency chain per nonzero).  Summation order is fixed per
// row, identical for every member column (deterministic).
#include "ens_internal.cuh"

#define FULL 0xffffffffu

static inline int next_pow2_h(int x) {
    int s = 1;
    while (s < x) s <<= 1;
    return s;
}

__device__ __forceinline__ int warp_max(int v) {
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

template <int OPL>
__global__ void __launch_bounds__(256) k_spmm_vel(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                  const double* __restrict__ A, int nnz,
                                                  const int32_t* __restrict__ btp, const int32_t* __restrict__ btc,
                                                  const double* __restrict__ btv, const uint8_t* __restrict__ cflag,
                                                  const double* __restrict__ X, const double* __restrict__ Bv,
                                                  double* __restrict__ Y, int ns, int64_t N, int J, int S, int mode) {
    const int lane = threadIdx.x & 31;
    const int seg = lane / S, sl = lane % S;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw * (32 / S) >= ns) return;                 // warp-uniform exit
    const int64_t node = gw * (32 / S) + seg;
    const bool live = node < ns;
    const int mat = blockIdx.y;
    const double* Am = A + (int64_t)mat * nnz;
    const double* Xm = X + (int64_t)mat * N * J;
    double* Ym = Y + (int64_t)mat * N * J;
    const int W2 = 2 * J;
    const int64_t nvel = 2LL * ns;
    double acc[OPL];
#pragma unroll
    for (int o = 0; o < OPL; ++o) acc[o] = 0.0;

    // ---- A_s part: both components share the row ----
    int k0 = 0, n = 0;
    if (live) {
        k0 = rp[node];
        n = rp[node + 1] - k0;
    }
    const int nmax = warp_max(n);
    for (int kb = 0; kb < nmax; kb += S) {
        int myc = 0;
        double mya = 0.0;
        if (kb + sl < n) {
            myc = col[k0 + kb + sl];
            mya = Am[k0 + kb + sl];
        }
        const int cnt = min(S, nmax - kb);
        for (int t = 0; t < cnt; t += 4) {
            int cc[4];
            double aa[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int src = (t + u) & (S - 1);
                cc[u] = __shfl_sync(FULL, myc, src, S);
                aa[u] = __shfl_sync(FULL, mya, src, S);
                if (t + u >= cnt) aa[u] = 0.0;
            }
            double xv[4][OPL];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int o = 0; o < OPL; ++o) {
                    const int l = sl + o * S;
                    xv[u][o] = l < W2 ? __ldg(Xm + 2LL * cc[u] * J + l) : 0.0;
                }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int o = 0; o < OPL; ++o) acc[o] = fma(aa[u], xv[u][o], acc[o]);
        }
    }
    // ---- -B^T part: pressure neighbours ----
    int t0 = 0, nt = 0;
    if (live) {
        t0 = btp[node];
        nt = btp[node + 1] - t0;
    }
    const int ntmax = warp_max(nt);
    for (int kb = 0; kb < ntmax; kb += S) {
        int myp = 0;
        double mbx = 0.0, mby = 0.0;
        if (kb + sl < nt) {
            myp = btc[t0 + kb + sl];
            mbx = btv[2 * (t0 + kb + sl)];
            mby = btv[2 * (t0 + kb + sl) + 1];
        }
        const int cnt = min(S, ntmax - kb);
        for (int t = 0; t < cnt; t += 4) {
            int pp[4];
            double bx[4], by[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int src = (t + u) & (S - 1);
                pp[u] = __shfl_sync(FULL, myp, src, S);
                bx[u] = __shfl_sync(FULL, mbx, src, S);
                by[u] = __shfl_sync(FULL, mby, src, S);
                if (t + u >= cnt) bx[u] = by[u] = 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int o = 0; o < OPL; ++o) {
                    const int l = sl + o * S;
                    if (l < W2) {
                        const int c2 = l >= J ? 1 : 0;
                        const double xp = __ldg(Xm + (nvel + pp[u]) * J + (l - c2 * J));
                        acc[o] = fma(-(c2 ? by[u] : bx[u]), xp, acc[o]);
                    }
                }
        }
    }
    if (!live) return;
    const double* xs = Xm + 2 * node * J;
#pragma unroll
    for (int o = 0; o < OPL; ++o) {
        const int l = sl + o * S;
        if (l >= W2) continue;
        const int c2 = l >= J ? 1 : 0;
        const int64_t idx = 2 * node * J + l;
        double val = cflag[2 * node + c2] ? xs[l] : acc[o];
        if (mode == 1) val = Bv[(int64_t)mat * N * J + idx] - val;
        Ym[idx] = val;
    }
}

template <int OPL>
__global__ void __launch_bounds__(256) k_spmm_pres(const int32_t* __restrict__ bp, const int32_t* __restrict__ bc,
                                                   const double* __restrict__ bv, const uint8_t* __restrict__ cflag,
                                                   const double* __restrict__ X, const double* __restrict__ Bv,
                                                   double* __restrict__ Y, int npres, int64_t nvel, int64_t N, int J,
                                                   int S, int mode) {
    const int lane = threadIdx.x & 31;
    const int seg = lane / S, sl = lane % S;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw * (32 / S) >= npres) return;
    const int64_t p = gw * (32 / S) + seg;
    const bool live = p < npres;
    const int mat = blockIdx.y;
    const double* Xm = X + (int64_t)mat * N * J;
    double* Ym = Y + (int64_t)mat * N * J;
    double acc[OPL];
#pragma unroll
    for (int o = 0; o < OPL; ++o) acc[o] = 0.0;
    int t0 = 0, n = 0;
    if (live) {
        t0 = bp[p];
        n = bp[p + 1] - t0;
    }
    const int nmax = warp_max(n);
    for (int kb = 0; kb < nmax; kb += S) {
        int myn = 0;
        double mbx = 0.0, mby = 0.0;
        if (kb + sl < n) {
            myn = bc[t0 + kb + sl];
            mbx = bv[2 * (t0 + kb + sl)];
            mby = bv[2 * (t0 + kb + sl) + 1];
        }
        const int cnt = min(S, nmax - kb);
        for (int t = 0; t < cnt; t += 4) {
            int nn[4];
            double bx[4], by[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int src = (t + u) & (S - 1);
                nn[u] = __shfl_sync(FULL, myn, src, S);
                bx[u] = __shfl_sync(FULL, mbx, src, S);
                by[u] = __shfl_sync(FULL, mby, src, S);
                if (t + u >= cnt) bx[u] = by[u] = 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int o = 0; o < OPL; ++o) {
                    const int l = sl + o * S;
                    if (l < J) {
                        const double* xr = Xm + 2LL * nn[u] * J;
                        acc[o] = fma(bx[u], __ldg(xr + l), acc[o]);
                        acc[o] = fma(by[u], __ldg(xr + J + l), acc[o]);
                    }
                }
        }
    }
    if (!live) return;
    const int64_t row = nvel + p;
#pragma unroll
    for (int o = 0; o < OPL; ++o) {
        const int l = sl + o * S;
        if (l >= J) continue;
        const int64_t idx = row * J + l;
        double val = cflag[row] ? Xm[idx] : acc[o];
        if (mode == 1) val = Bv[(int64_t)mat * N * J + idx] - val;
        Ym[idx] = val;
    }
}

int launch_spmm(ens_ctx* c, cudaStream_t s, const double* as_vals, const double* x, const double* b, double* y,
                int mode) {
    const int J = c->J, W2 = 2 * J;
    {
        const int S = W2 >= 32 ? 32 : next_pow2_h(W2);
        const int opl = (W2 + S - 1) / S;
        const int64_t warps = ((int64_t)c->m.ns + (32 / S) - 1) / (32 / S);
        dim3 grid((unsigned)((warps * 32 + 255) / 256), 2);
#define SPV(V)                                                                                                    \
    k_spmm_vel<V><<<grid, 256, 0, s>>>(c->m.s_rowptr, c->m.s_col, as_vals, c->m.nnz_s, c->m.bt_rowptr, c->m.bt_col, \
                                       c->m.bt_val, c->m.cflag, x, b, y, c->m.ns, c->n_total, J, S, mode)
        if (opl <= 1) SPV(1);
        else if (opl <= 2) SPV(2);
        else if (opl <= 4) SPV(4);
        else if (opl <= 8) SPV(8);
        else if (opl <= 16) SPV(16);
        else {
            ens_set_error("J too large for spmm", __FILE__, __LINE__);
            return ENS_EINVAL;
        }
#undef SPV
        ENS_CKL();
    }
    {
        const int S = J >= 32 ? 32 : next_pow2_h(J);
        const int opl = (J + S - 1) / S;
        const int64_t warps = ((int64_t)c->m.n_pres + (32 / S) - 1) / (32 / S);
        dim3 grid((unsigned)((warps * 32 + 255) / 256), 2);
#define SPP(V)                                                                                                  \
    k_spmm_pres<V><<<grid, 256, 0, s>>>(c->m.b_rowptr, c->m.b_col, c->m.b_val, c->m.cflag, x, b, y, c->m.n_pres, \
                                        c->n_vel, c->n_total, J, S, mode)
        if (opl <= 1) SPP(1);
        else if (opl <= 2) SPP(2);
        else if (opl <= 4) SPP(4);
        else if (opl <= 8) SPP(8);
        else {
            ens_set_error("J too large for spmm", __FILE__, __LINE__);
            return ENS_EINVAL;
        }
#undef SPP
        ENS_CKL();
    }
    return ENS_OK;
}
