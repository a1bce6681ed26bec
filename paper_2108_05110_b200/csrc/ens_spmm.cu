// Saddle-operator SpMM for both sub-step systems (the Krylov core), fp64, sm_100a.
//
// Applies exactly the reference's assembled saddle matrix (stepper.py:208-215)
// to all J member columns at once (the product behind linalg.py:111-118).
// Layout: member-minor blocks, so one node's (x, y) values for all members are
// 2J contiguous doubles -> each nonzero gathers one coalesced segment that
// serves every member and both components.  A segment of S lanes owns a row;
// summation order is fixed per row and identical for every member column.
// (A variant that preloads the row's indices lane-parallel and broadcasts them
// with shuffles measured slower at C2: 0.24 ms vs 0.17 ms per launch pair.)
#include "ens_internal.cuh"

static inline int next_pow2(int x) {
    int s = 1;
    while (s < x) s <<= 1;
    return s;
}

// ---------------------------------------------------------------------------
// saddle SpMM, both systems: y = K x or y = b - K x
//   velocity node i, comp c: sum_k A[k] x[2 col_k + c] - sum_t Bc^T[t] x[p_t]
//   pressure row p:          sum_t bx x[2 n_t] + by x[2 n_t + 1]
//   identity rows (cflag):   x
// Each node row gathers the 2J contiguous doubles of its neighbours (member-
// minor layout => one coalesced segment per nonzero, shared by x and y).
// ---------------------------------------------------------------------------
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
    const int64_t node = gw * (32 / S) + seg;
    if (node >= ns) return;
    const int mat = blockIdx.y;
    const double* Am = A + (int64_t)mat * nnz;
    const double* Xm = X + (int64_t)mat * N * J;
    double* Ym = Y + (int64_t)mat * N * J;
    const int W2 = 2 * J;
    const int64_t nvel = 2LL * ns;
    double acc[OPL];
#pragma unroll
    for (int o = 0; o < OPL; ++o) acc[o] = 0.0;
    const int k0 = rp[node], k1 = rp[node + 1];
    for (int k = k0; k < k1; ++k) {
        const double a = Am[k];
        const double* xr = Xm + 2LL * col[k] * J;
#pragma unroll
        for (int o = 0; o < OPL; ++o) {
            const int l = sl + o * S;
            if (l < W2) acc[o] += a * xr[l];
        }
    }
    const int t0 = btp[node], t1 = btp[node + 1];
    for (int t = t0; t < t1; ++t) {
        const double bxv = btv[2 * t], byv = btv[2 * t + 1];
        const double* xp = Xm + (nvel + btc[t]) * J;
#pragma unroll
        for (int o = 0; o < OPL; ++o) {
            const int l = sl + o * S;
            if (l < W2) {
                const int cc = l >= J ? 1 : 0;
                acc[o] -= (cc ? byv : bxv) * xp[l - cc * J];
            }
        }
    }
    const double* xs = Xm + 2 * node * J;
#pragma unroll
    for (int o = 0; o < OPL; ++o) {
        const int l = sl + o * S;
        if (l >= W2) continue;
        const int cc = l >= J ? 1 : 0;
        const int64_t idx = 2 * node * J + l;
        double val = cflag[2 * node + cc] ? xs[l] : acc[o];
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
    const int64_t p = gw * (32 / S) + seg;
    if (p >= npres) return;
    const int mat = blockIdx.y;
    const double* Xm = X + (int64_t)mat * N * J;
    double* Ym = Y + (int64_t)mat * N * J;
    double acc[OPL];
#pragma unroll
    for (int o = 0; o < OPL; ++o) acc[o] = 0.0;
    const int t0 = bp[p], t1 = bp[p + 1];
    for (int t = t0; t < t1; ++t) {
        const double bxv = bv[2 * t], byv = bv[2 * t + 1];
        const double* xr = Xm + 2LL * bc[t] * J;
#pragma unroll
        for (int o = 0; o < OPL; ++o) {
            const int l = sl + o * S;
            if (l < J) acc[o] += bxv * xr[l] + byv * xr[J + l];
        }
    }
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
        const int S = W2 >= 32 ? 32 : next_pow2(W2);
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
        else { ens_set_error("J too large for spmm", __FILE__, __LINE__); return ENS_EINVAL; }
#undef SPV
        ENS_CKL();
    }
    {
        const int S = J >= 32 ? 32 : next_pow2(J);
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
        else { ens_set_error("J too large for spmm", __FILE__, __LINE__); return ENS_EINVAL; }
#undef SPP
        ENS_CKL();
    }
    return ENS_OK;
}
