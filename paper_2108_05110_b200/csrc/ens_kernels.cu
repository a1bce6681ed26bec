#include <algorithm>
// Element, member, right-hand-side, SpMM and reduction kernels (sm_100a, fp64).
//
// Layout (see include/ensmhd_b200.h): a field block has n_total rows in the
// internal order (velocity row 2*node+comp, then pressures) and J contiguous
// member columns; the V and W systems are two such blocks back to back.  The
// velocity part of the V block is the state v, of the W block the state w.
#include <cmath>
#include <cstdio>

#include "ens_internal.cuh"

__constant__ double c_qw[ENS_NQ];
__constant__ double c_phi[ENS_NQ][6];
__constant__ double c_dphi[ENS_NQ][6][3];

// ---------------------------------------------------------------------------
// reference-element tables (fem.py:33-86): same formulas, same point order
// ---------------------------------------------------------------------------
int ens_upload_tables() {
    double pts[ENS_NQ][3], w[ENS_NQ];
    const double r15 = std::sqrt(15.0);
    pts[0][0] = pts[0][1] = pts[0][2] = 1.0 / 3.0;
    w[0] = 9.0 / 40.0;
    const double as[2] = {(6.0 + r15) / 21.0, (6.0 - r15) / 21.0};
    const double ws[2] = {(155.0 + r15) / 1200.0, (155.0 - r15) / 1200.0};
    int q = 1;
    for (int s = 0; s < 2; ++s) {
        const double a = as[s], b = 1.0 - 2.0 * a;
        const double tri[3][3] = {{b, a, a}, {a, b, a}, {a, a, b}};
        for (int t = 0; t < 3; ++t, ++q) {
            for (int i = 0; i < 3; ++i) pts[q][i] = tri[t][i];
            w[q] = ws[s];
        }
    }
    double phi[ENS_NQ][6], dphi[ENS_NQ][6][3];
    for (int q2 = 0; q2 < ENS_NQ; ++q2) {
        const double l0 = pts[q2][0], l1 = pts[q2][1], l2 = pts[q2][2];
        phi[q2][0] = l0 * (2 * l0 - 1);
        phi[q2][1] = l1 * (2 * l1 - 1);
        phi[q2][2] = l2 * (2 * l2 - 1);
        phi[q2][3] = 4 * l0 * l1;
        phi[q2][4] = 4 * l1 * l2;
        phi[q2][5] = 4 * l2 * l0;
        for (int a = 0; a < 6; ++a)
            for (int i = 0; i < 3; ++i) dphi[q2][a][i] = 0.0;
        dphi[q2][0][0] = 4 * l0 - 1;
        dphi[q2][1][1] = 4 * l1 - 1;
        dphi[q2][2][2] = 4 * l2 - 1;
        dphi[q2][3][0] = 4 * l1;
        dphi[q2][3][1] = 4 * l0;
        dphi[q2][4][1] = 4 * l2;
        dphi[q2][4][2] = 4 * l1;
        dphi[q2][5][2] = 4 * l0;
        dphi[q2][5][0] = 4 * l2;
    }
    ENS_CK(cudaMemcpyToSymbol(c_qw, w, sizeof(w)));
    ENS_CK(cudaMemcpyToSymbol(c_phi, phi, sizeof(phi)));
    ENS_CK(cudaMemcpyToSymbol(c_dphi, dphi, sizeof(dphi)));
    return ENS_OK;
}

// physical gradient of local shape function a at quadrature point q
__device__ __forceinline__ void grad_phi(const double* gl, int q, int a, double& gx, double& gy) {
    const double d0 = c_dphi[q][a][0], d1 = c_dphi[q][a][1], d2 = c_dphi[q][a][2];
    gx = d0 * gl[0] + d1 * gl[2] + d2 * gl[4];
    gy = d0 * gl[1] + d1 * gl[3] + d2 * gl[5];
}

static bool red_vec_ok(int J, const void* a, const void* b) {
    return (J & 1) == 0 && J <= 512 && (reinterpret_cast<uintptr_t>(a) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(b) & 15) == 0;
}

static inline int next_pow2(int x) {
    int s = 1;
    while (s < x) s <<= 1;
    return s;
}

// ---------------------------------------------------------------------------
// member sums (ensemble.py:222-223 mean numerator), both families
// ---------------------------------------------------------------------------
__global__ void k_member_sums(const double* __restrict__ X, double* __restrict__ sums, int nvel, int64_t N, int J,
                              int S) {
    const int lane = threadIdx.x & 31;
    const int seg = lane / S, sl = lane % S;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t r = gw * (32 / S) + seg;     // row in [0, 2*nvel)
    if (r >= 2 * (int64_t)nvel) return;
    const int mat = (int)(r / nvel);
    const int64_t row = r - (int64_t)mat * nvel;
    const double* xr = X + (int64_t)mat * N * J + row * J;
    double acc = 0.0;
    for (int j = sl; j < J; j += S) acc += xr[j];
    for (int o = S / 2; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o, S);
    if (sl == 0) sums[r] = acc;
}

__global__ void __launch_bounds__(256) k_lincomb2(double a, const double2* __restrict__ x, double b,
                                                  double2* __restrict__ y, int64_t n2) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n2; t += (int64_t)gridDim.x * blockDim.x) {
        const double2 u = x[t];
        double2 v = y[t];
        v.x = a * u.x + b * v.x;
        v.y = a * u.y + b * v.y;
        y[t] = v;
    }
}

__global__ void __launch_bounds__(256) k_lincomb(double a, const double* __restrict__ x, double b,
                                                 double* __restrict__ y, int64_t n) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        y[t] = a * x[t] + b * y[t];
}

int launch_lincomb(ens_ctx* c, cudaStream_t s, double a, const double* x, double b, double* y) {
    const int64_t n = 2LL * c->n_total * c->J;
    if ((n & 1) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0) {
        const int64_t n2 = n / 2;
        const unsigned nb = (unsigned)std::min<int64_t>((n2 + 255) / 256, 148 * 16);
        k_lincomb2<<<nb, 256, 0, s>>>(a, reinterpret_cast<const double2*>(x), b, reinterpret_cast<double2*>(y), n2);
    } else {
        const unsigned nb = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
        k_lincomb<<<nb, 256, 0, s>>>(a, x, b, y, n);
    }
    ENS_CKL();
    return ENS_OK;
}

// thread per row (even J): H 16-byte loads, fixed sequential member order
__global__ void __launch_bounds__(256) k_member_sums2(const double* __restrict__ X, double* __restrict__ sums,
                                                      int nvel, int64_t N, int J) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= 2 * (int64_t)nvel) return;
    const int mat = (int)(r / nvel);
    const int64_t row = r - (int64_t)mat * nvel;
    const double2* xr = reinterpret_cast<const double2*>(X + (int64_t)mat * N * J + row * J);
    double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
    for (int i = 0; i < (J >> 1); ++i) {
        const double2 v = xr[i];
        a0 += v.x;
        a1 += v.y;
    }
    sums[r] = a0 + a1;
}

int launch_member_sums(ens_ctx* c, cudaStream_t s, const double* x, double* sums) {
    if ((c->J & 1) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        const int64_t rows = 2LL * c->n_vel;
        k_member_sums2<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(x, sums, c->n_vel, c->n_total, c->J);
        ENS_CKL();
        return ENS_OK;
    }
    const int S = c->J >= 32 ? 32 : next_pow2(c->J);
    const int64_t rows = 2LL * c->n_vel;
    const int64_t warps = (rows + (32 / S) - 1) / (32 / S);
    const int64_t blocks = (warps * 32 + 255) / 256;
    k_member_sums<<<(unsigned)blocks, 256, 0, s>>>(x, sums, c->n_vel, c->n_total, c->J, S);
    ENS_CKL();
    return ENS_OK;
}

// means[r] = sums[r] * inv_members (the ensemble means of ensemble.py:216-224 from the -- in sharded runs
// all-reduced -- member sums); the same IEEE product as the host expression sums * (1 / J)
__global__ void __launch_bounds__(256) k_means(const double* __restrict__ sums, double inv_members,
                                               double* __restrict__ means, int64_t n) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) means[r] = sums[r] * inv_members;
}

int launch_means(ens_ctx* c, cudaStream_t s, const double* sums, double inv_members, double* means) {
    const int64_t n = 2LL * c->n_vel;
    k_means<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sums, inv_members, means, n);
    ENS_CKL();
    return ENS_OK;
}

// ---------------------------------------------------------------------------
// right-hand sides, velocity rows (stepper.py:235-247) for both sub-steps
// ---------------------------------------------------------------------------
template <int OPL>
__global__ void k_rhs(const int32_t* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ mass,
                      const double* __restrict__ stiff, const double* __restrict__ X, const double* __restrict__ coef,
                      double inv_dt, int K, const double* __restrict__ lbasis, const double* __restrict__ lcoef,
                      const double* __restrict__ ldense, double* __restrict__ rhs, int ns, int64_t N, int J, int S) {
    const int lane = threadIdx.x & 31;
    const int seg = lane / S, sl = lane % S;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t node = gw * (32 / S) + seg;
    if (node >= ns) return;
    const int W2 = 2 * J;
    const double* Xv = X;
    const double* Xw = X + N * J;
    double mv[OPL], kv[OPL], mw[OPL], kw[OPL];
#pragma unroll
    for (int o = 0; o < OPL; ++o) mv[o] = kv[o] = mw[o] = kw[o] = 0.0;
    const int k0 = rp[node], k1 = rp[node + 1];
    for (int k = k0; k < k1; ++k) {
        const int64_t q = col[k];
        const double a = mass[k], b = stiff[k];
        const double* xv = Xv + 2 * q * J;
        const double* xw = Xw + 2 * q * J;
#pragma unroll
        for (int o = 0; o < OPL; ++o) {
            const int l = sl + o * S;
            if (l < W2) {
                const double v = xv[l], w = xw[l];
                mv[o] += a * v;
                kv[o] += b * v;
                mw[o] += a * w;
                kw[o] += b * w;
            }
        }
    }
    const int64_t nvel = 2LL * ns;
#pragma unroll
    for (int o = 0; o < OPL; ++o) {
        const int l = sl + o * S;
        if (l >= W2) continue;
        const int cc = l >= J ? 1 : 0;
        const int j = l - cc * J;
        const int64_t row = 2 * node + cc;
        const double ls = coef[j], lc = coef[J + j];
        double lv = 0.0, lw = 0.0;
        for (int kk = 0; kk < K; ++kk) {
            const double bval = lbasis[(int64_t)kk * nvel + row];
            lv += lcoef[(int64_t)kk * J + j] * bval;
            lw += lcoef[(int64_t)(K + kk) * J + j] * bval;
        }
        if (ldense) {
            lv += ldense[row * J + j];
            lw += ldense[nvel * J + row * J + j];
        }
        rhs[row * J + j] = (mv[o] * inv_dt - ls * kv[o] - lc * kw[o]) + lv;
        rhs[N * J + row * J + j] = (mw[o] * inv_dt - ls * kw[o] - lc * kv[o]) + lw;
    }
}

// even J: a velocity row's 2J values over L lanes x V2 double2, 32/L rows per warp
// (as k_spmm_vel_v); mass and stiffness products of both families in one pass
template <int V2>
__global__ void __launch_bounds__(256) k_rhs_v(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                               const double* __restrict__ mass, const double* __restrict__ stiff,
                                               const double* __restrict__ X, const double* __restrict__ coef,
                                               double inv_dt, int K, const double* __restrict__ lbasis,
                                               const double* __restrict__ lcoef, const double* __restrict__ ldense,
                                               double* __restrict__ rhs, int ns, int64_t N, int J, int L) {
    const int lane = threadIdx.x & 31;
    const int R = 32 / L;
    const int r = lane / L, part = lane - r * L;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t node = gw * R + r;
    if (r >= R || node >= ns) return;
    const int H = J >> 1;
    const double2* Xv = reinterpret_cast<const double2*>(X);
    const double2* Xw = reinterpret_cast<const double2*>(X + N * J);
    double2 mv[V2], kv[V2], mw[V2], kw[V2];
#pragma unroll
    for (int v = 0; v < V2; ++v) mv[v] = kv[v] = mw[v] = kw[v] = make_double2(0.0, 0.0);
    const int k0 = rp[node], k1 = rp[node + 1];
    int k = k0;
    for (; k + 2 <= k1; k += 2) {
        const int64_t q0 = col[k], q1 = col[k + 1];
        const double a0 = mass[k], b0 = stiff[k], a1 = mass[k + 1], b1 = stiff[k + 1];
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int i = V2 * part + v;
            if (i < J) {
                const double2 x0 = Xv[q0 * J + i], w0 = Xw[q0 * J + i], x1 = Xv[q1 * J + i], w1 = Xw[q1 * J + i];
                mv[v].x += a0 * x0.x; mv[v].y += a0 * x0.y; kv[v].x += b0 * x0.x; kv[v].y += b0 * x0.y;
                mw[v].x += a0 * w0.x; mw[v].y += a0 * w0.y; kw[v].x += b0 * w0.x; kw[v].y += b0 * w0.y;
                mv[v].x += a1 * x1.x; mv[v].y += a1 * x1.y; kv[v].x += b1 * x1.x; kv[v].y += b1 * x1.y;
                mw[v].x += a1 * w1.x; mw[v].y += a1 * w1.y; kw[v].x += b1 * w1.x; kw[v].y += b1 * w1.y;
            }
        }
    }
    for (; k < k1; ++k) {
        const int64_t q0 = col[k];
        const double a0 = mass[k], b0 = stiff[k];
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int i = V2 * part + v;
            if (i < J) {
                const double2 x0 = Xv[q0 * J + i], w0 = Xw[q0 * J + i];
                mv[v].x += a0 * x0.x; mv[v].y += a0 * x0.y; kv[v].x += b0 * x0.x; kv[v].y += b0 * x0.y;
                mw[v].x += a0 * w0.x; mw[v].y += a0 * w0.y; kw[v].x += b0 * w0.x; kw[v].y += b0 * w0.y;
            }
        }
    }
    const int64_t nvel = 2LL * ns;
#pragma unroll
    for (int v = 0; v < V2; ++v) {
        const int i = V2 * part + v;
        if (i >= J) continue;
        const int cc = i >= H ? 1 : 0;
        const int64_t row = 2 * node + cc;
        double ov[2], ow[2];
        const double mvv[2] = {mv[v].x, mv[v].y}, kvv[2] = {kv[v].x, kv[v].y};
        const double mww[2] = {mw[v].x, mw[v].y}, kww[2] = {kw[v].x, kw[v].y};
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int j = 2 * (i - cc * H) + e;
            const double ls = coef[j], lc = coef[J + j];
            double lv = 0.0, lw = 0.0;
            for (int kk = 0; kk < K; ++kk) {
                const double bval = lbasis[(int64_t)kk * nvel + row];
                lv += lcoef[(int64_t)kk * J + j] * bval;
                lw += lcoef[(int64_t)(K + kk) * J + j] * bval;
            }
            if (ldense) {
                lv += ldense[row * J + j];
                lw += ldense[nvel * J + row * J + j];
            }
            ov[e] = (mvv[e] * inv_dt - ls * kvv[e] - lc * kww[e]) + lv;
            ow[e] = (mww[e] * inv_dt - ls * kww[e] - lc * kvv[e]) + lw;
        }
        reinterpret_cast<double2*>(rhs)[node * J + i] = make_double2(ov[0], ov[1]);
        reinterpret_cast<double2*>(rhs + N * J)[node * J + i] = make_double2(ow[0], ow[1]);
    }
}

int launch_rhs(ens_ctx* c, cudaStream_t s, const double* x, const double* coef, double inv_dt,
               const ens_data_desc* loads, double* rhs) {
    if ((c->J & 1) == 0 && c->J <= 512 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(rhs) & 15) == 0) {
        const int J = c->J;
        const int64_t N = c->n_total;
        for (int mat = 0; mat < 2; ++mat)
            ENS_CK(cudaMemsetAsync(rhs + mat * N * J + (int64_t)c->n_vel * J, 0,
                                   sizeof(double) * (size_t)c->m.n_pres * J, s));
        const int V2 = J <= 64 ? 2 : (J <= 128 ? 4 : 8);
        const int L = (J + V2 - 1) / V2, R = 32 / L;
        const int64_t warps = ((int64_t)c->m.ns + R - 1) / R;
        const unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
        const int K = loads ? loads->K : 0;
        const double* lb = loads ? loads->basis : nullptr;
        const double* lc = loads ? loads->coef : nullptr;
        const double* ld = loads ? loads->dense : nullptr;
#define RHV(V)                                                                                                    \
    k_rhs_v<V><<<blocks, 256, 0, s>>>(c->m.s_rowptr, c->m.s_col, c->m.s_mass, c->m.s_stiff, x, coef, inv_dt, K, lb, \
                                      lc, ld, rhs, c->m.ns, N, J, L)
        if (V2 == 2) RHV(2);
        else if (V2 == 4) RHV(4);
        else RHV(8);
#undef RHV
        ENS_CKL();
        return ENS_OK;
    }
    const int J = c->J, W2 = 2 * J;
    const int S = W2 >= 32 ? 32 : next_pow2(W2);
    const int opl = (W2 + S - 1) / S;
    const int64_t warps = ((int64_t)c->m.ns + (32 / S) - 1) / (32 / S);
    const unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
    const int K = loads ? loads->K : 0;
    const double* lb = loads ? loads->basis : nullptr;
    const double* lc = loads ? loads->coef : nullptr;
    const double* ld = loads ? loads->dense : nullptr;
    const int64_t N = c->n_total;
    // pressure rows of the right-hand side are zero (stepper.py:245-246)
    for (int mat = 0; mat < 2; ++mat)
        ENS_CK(cudaMemsetAsync(rhs + mat * N * J + (int64_t)c->n_vel * J, 0,
                               sizeof(double) * (size_t)c->m.n_pres * J, s));
#define RHS_CASE(V)                                                                                               \
    case V:                                                                                                       \
        k_rhs<V><<<blocks, 256, 0, s>>>(c->m.s_rowptr, c->m.s_col, c->m.s_mass, c->m.s_stiff, x, coef, inv_dt, K, \
                                        lb, lc, ld, rhs, c->m.ns, N, J, S);                                       \
        break;
    switch (opl) {
        RHS_CASE(1)
        RHS_CASE(2)
        RHS_CASE(3)
        RHS_CASE(4)
        RHS_CASE(8)
        default:
            if (opl <= 8) {
                k_rhs<8><<<blocks, 256, 0, s>>>(c->m.s_rowptr, c->m.s_col, c->m.s_mass, c->m.s_stiff, x, coef, inv_dt,
                                                K, lb, lc, ld, rhs, c->m.ns, N, J, S);
            } else {
                k_rhs<16><<<blocks, 256, 0, s>>>(c->m.s_rowptr, c->m.s_col, c->m.s_mass, c->m.s_stiff, x, coef,
                                                 inv_dt, K, lb, lc, ld, rhs, c->m.ns, N, J, S);
            }
    }
#undef RHS_CASE
    ENS_CKL();
    return ENS_OK;
}

// ---------------------------------------------------------------------------
// member pass: fluctuation transport on both RHS + max_j |z'_j|^2 per qp
//   (fem.py:411-420, ensemble.py:227-238); one thread per (element, member),
//   elements of one colour touch disjoint dofs -> plain read-modify-write.
// ---------------------------------------------------------------------------
// FULL (ens_rhs_fused): the element buffer receives the whole element right-hand side of
// both sub-steps, M same/dt - N(z') same - K(ls same + lc other) (stepper.py:235-247 with
// fem.py:411-420), evaluated at the 7 quadrature points that assemble M and K exactly;
// k_member_gather<true> then sums it per row and adds the loads -- no CSR pass.
template <bool FULL>
__global__ void k_member_pass(const int32_t* __restrict__ enodes, const double* __restrict__ egeo, int e0, int ne,
                              const double* __restrict__ X, const double* __restrict__ means, double* __restrict__ rhs,
                              unsigned long long* __restrict__ maxsq, int nt, int nvel, int64_t N, int J, int JB,
                              double* __restrict__ ec, const double* __restrict__ mcoef, double inv_dt) {
    extern __shared__ double sh_sq[];   // [EPB][2][7][JB], then the elements' nodal means [EPB][2][6][2]
    const int EPB = blockDim.x / JB;
    const int el = threadIdx.x / JB, jj = threadIdx.x % JB;
    const int e = e0 + blockIdx.x * EPB + el;
    const int j = blockIdx.y * JB + jj;
    const bool live = (el < EPB) && (e < e0 + ne) && (j < J);
    double* sq = sh_sq + (size_t)el * 2 * ENS_NQ * JB;
    // the ensemble means at the element's nodes are member-independent: staged once per
    // element in shared memory instead of 24 per-thread registers (occupancy)
    double* smn = sh_sq + (size_t)EPB * 2 * ENS_NQ * JB + (size_t)el * 24;
    // physical shape-function gradients at the quadrature points, member-independent too:
    // computed once per element into shared memory ([EPB][7][6][2]) instead of per thread
    double* sgr = sh_sq + (size_t)EPB * 2 * ENS_NQ * JB + (size_t)EPB * 24 + (size_t)el * ENS_NQ * 12;
    if (el < EPB && e < e0 + ne) {
        for (int t = jj; t < 24; t += JB) {
            const int fam = t / 12, a = (t % 12) >> 1, cc = t & 1;
            smn[t] = means[(int64_t)fam * nvel + 2LL * enodes[(int64_t)e * 6 + a] + cc];
        }
        double gle[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) gle[i] = egeo[(int64_t)e * 8 + 1 + i];
        for (int t = jj; t < ENS_NQ * 6; t += JB) {
            const int q = t / 6, a = t % 6;
            grad_phi(gle, q, a, sgr[2 * t], sgr[2 * t + 1]);
        }
    }
    __syncthreads();
    if (live) {
        const double* Xv = X;
        const double* Xw = X + N * J;
        int nd[6];
#pragma unroll
        for (int a = 0; a < 6; ++a) nd[a] = enodes[(int64_t)e * 6 + a];
        const double area = egeo[(int64_t)e * 8];
        double v[6][2], w[6][2];
#pragma unroll
        for (int a = 0; a < 6; ++a) {
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int64_t row = 2LL * nd[a] + cc;
                v[a][cc] = Xv[row * J + j];
                w[a][cc] = Xw[row * J + j];
            }
        }
        double rv[6][2], rw[6][2];
#pragma unroll
        for (int a = 0; a < 6; ++a) rv[a][0] = rv[a][1] = rw[a][0] = rw[a][1] = 0.0;
        const double ls = FULL ? mcoef[j] : 0.0, lc = FULL ? mcoef[J + j] : 0.0;
#pragma unroll 1
        for (int q = 0; q < ENS_NQ; ++q) {
            double fvq0 = 0, fvq1 = 0, fwq0 = 0, fwq1 = 0;
            double vq0 = 0, vq1 = 0, wq0 = 0, wq1 = 0;
            double gv00 = 0, gv01 = 0, gv10 = 0, gv11 = 0, gw00 = 0, gw01 = 0, gw10 = 0, gw11 = 0;
#pragma unroll
            for (int a = 0; a < 6; ++a) {
                const double ph = c_phi[q][a];
                const double gx = sgr[(q * 6 + a) * 2], gy = sgr[(q * 6 + a) * 2 + 1];
                fvq0 += (v[a][0] - smn[2 * a]) * ph;
                fvq1 += (v[a][1] - smn[2 * a + 1]) * ph;
                fwq0 += (w[a][0] - smn[12 + 2 * a]) * ph;
                fwq1 += (w[a][1] - smn[12 + 2 * a + 1]) * ph;
                if (FULL) {
                    vq0 += v[a][0] * ph;
                    vq1 += v[a][1] * ph;
                    wq0 += w[a][0] * ph;
                    wq1 += w[a][1] * ph;
                }
                gv00 += v[a][0] * gx;
                gv01 += v[a][0] * gy;
                gv10 += v[a][1] * gx;
                gv11 += v[a][1] * gy;
                gw00 += w[a][0] * gx;
                gw01 += w[a][0] * gy;
                gw10 += w[a][1] * gx;
                gw11 += w[a][1] * gy;
            }
            sq[(0 * ENS_NQ + q) * JB + jj] = fwq0 * fwq0 + fwq1 * fwq1;   // V-step matrix: w'
            sq[(1 * ENS_NQ + q) * JB + jj] = fvq0 * fvq0 + fvq1 * fvq1;   // W-step matrix: v'
            const double wd = area * c_qw[q];
            // V-step: (w' . grad) v ; W-step: (v' . grad) w
            const double cv0 = wd * (fwq0 * gv00 + fwq1 * gv01);
            const double cv1 = wd * (fwq0 * gv10 + fwq1 * gv11);
            const double cw0 = wd * (fvq0 * gw00 + fvq1 * gw01);
            const double cw1 = wd * (fvq0 * gw10 + fvq1 * gw11);
            if (FULL) {
                // value part (M same/dt - convection) and gradient part (K terms) of both systems
                const double wdt = wd * inv_dt;
                const double tv0 = wdt * vq0 - cv0, tv1 = wdt * vq1 - cv1;
                const double tw0 = wdt * wq0 - cw0, tw1 = wdt * wq1 - cw1;
                const double hv0x = wd * (ls * gv00 + lc * gw00), hv0y = wd * (ls * gv01 + lc * gw01);
                const double hv1x = wd * (ls * gv10 + lc * gw10), hv1y = wd * (ls * gv11 + lc * gw11);
                const double hw0x = wd * (ls * gw00 + lc * gv00), hw0y = wd * (ls * gw01 + lc * gv01);
                const double hw1x = wd * (ls * gw10 + lc * gv10), hw1y = wd * (ls * gw11 + lc * gv11);
#pragma unroll
                for (int a = 0; a < 6; ++a) {
                    const double ph = c_phi[q][a];
                    const double gx = sgr[(q * 6 + a) * 2], gy = sgr[(q * 6 + a) * 2 + 1];
                    rv[a][0] += ph * tv0 - (gx * hv0x + gy * hv0y);
                    rv[a][1] += ph * tv1 - (gx * hv1x + gy * hv1y);
                    rw[a][0] += ph * tw0 - (gx * hw0x + gy * hw0y);
                    rw[a][1] += ph * tw1 - (gx * hw1x + gy * hw1y);
                }
            } else {
#pragma unroll
                for (int a = 0; a < 6; ++a) {
                    const double ph = c_phi[q][a];
                    rv[a][0] += cv0 * ph;
                    rv[a][1] += cv1 * ph;
                    rw[a][0] += cw0 * ph;
                    rw[a][1] += cw1 * ph;
                }
            }
        }
        if (ec) {   // element buffer [mat][e][a][cc][j], gathered per row by k_member_gather
            const int64_t eb = (int64_t)e * 12 * J + j, ms = (int64_t)nt * 12 * J;
#pragma unroll
            for (int a = 0; a < 6; ++a)
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    ec[eb + (2 * a + cc) * J] = rv[a][cc];
                    ec[ms + eb + (2 * a + cc) * J] = rw[a][cc];
                }
        } else {
#pragma unroll
            for (int a = 0; a < 6; ++a) {
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    const int64_t row = 2LL * nd[a] + cc;
                    rhs[row * J + j] -= rv[a][cc];
                    rhs[N * J + row * J + j] -= rw[a][cc];
                }
            }
        }
    } else if (el < EPB) {
        for (int q = 0; q < 2 * ENS_NQ; ++q) sq[q * JB + jj] = 0.0;
    }
    __syncthreads();
    // reduce max over members of this block for each (element, family, q)
    const int nred = EPB * 2 * ENS_NQ;
    for (int t = threadIdx.x; t < nred; t += blockDim.x) {
        const int le = t / (2 * ENS_NQ), fq = t % (2 * ENS_NQ);
        const int ee = e0 + blockIdx.x * EPB + le;
        if (ee >= e0 + ne) continue;
        const double* p = sh_sq + ((size_t)le * 2 * ENS_NQ + fq) * JB;
        double mx = 0.0;
        const int jmax = min(JB, J - (int)blockIdx.y * JB);
        for (int k = 0; k < jmax; ++k) mx = fmax(mx, p[k]);
        const int fam = fq / ENS_NQ, q = fq % ENS_NQ;
        // non-negative doubles order like their bit patterns
        atomicMax(maxsq + ((int64_t)fam * nt + ee) * ENS_NQ + q, (unsigned long long)__double_as_longlong(mx));
    }
}

// rhs[mat][row][j] -= sum over the node's element entries (fixed order) -- even J, 16-byte lanes
// FULL: rhs[mat][row][j] = sum of the entries + loads (basis x coefficients and/or dense)
template <bool FULL>
__global__ void __launch_bounds__(256) k_member_gather(const int32_t* __restrict__ n2e_ptr,
                                                       const int32_t* __restrict__ n2e, const double* __restrict__ ec,
                                                       double* __restrict__ rhs, int ns, int nt, int64_t N, int J,
                                                       int K, const double* __restrict__ lbasis,
                                                       const double* __restrict__ lcoef,
                                                       const double* __restrict__ ldense) {
    const int H = J >> 1;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2LL * ns * H) return;
    const int mat = blockIdx.y;
    const int64_t row = t / H;                   // velocity row 2*node + cc
    const int jp = (int)(t - row * H);
    const int node = (int)(row >> 1), cc = (int)(row & 1);
    const double2* e2 = reinterpret_cast<const double2*>(ec + (int64_t)mat * nt * 12 * J);
    double2 acc = make_double2(0.0, 0.0);
    const int k0 = n2e_ptr[node], k1 = n2e_ptr[node + 1];
    for (int k = k0; k < k1; ++k) {
        const int ea = n2e[k];                   // e*6 + a
        const double2 v = e2[((int64_t)ea * 2 + cc) * H + jp];
        acc.x += v.x;
        acc.y += v.y;
    }
    double2* r2 = reinterpret_cast<double2*>(rhs + (int64_t)mat * N * J);
    if (FULL) {
        const int64_t nvel = 2LL * ns;
        const int j = 2 * jp;
        for (int kk = 0; kk < K; ++kk) {
            const double bval = lbasis[(int64_t)kk * nvel + row];
            const double* cf = lcoef + ((int64_t)mat * K + kk) * J + j;
            acc.x += cf[0] * bval;
            acc.y += cf[1] * bval;
        }
        if (ldense) {
            const double2 dd = reinterpret_cast<const double2*>(ldense + (int64_t)mat * nvel * J)[row * H + jp];
            acc.x += dd.x;
            acc.y += dd.y;
        }
        r2[row * H + jp] = acc;
        return;
    }
    double2 r = r2[row * H + jp];
    r.x -= acc.x;
    r.y -= acc.y;
    r2[row * H + jp] = r;
}

// the member pass stages per-element tables in dynamic shared memory (small J => many elements
// per block => more than the default 48 KB)
static int member_pass_smem_setup() {
    static bool done = false;
    if (!done) {
        ENS_CK(cudaFuncSetAttribute(k_member_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        ENS_CK(cudaFuncSetAttribute(k_member_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        done = true;
    }
    return ENS_OK;
}

int launch_member_pass(ens_ctx* c, cudaStream_t s, const double* x, const double* means, double* rhs,
                       double* maxsq) {
    {
        const int rc = member_pass_smem_setup();
        if (rc != ENS_OK) return rc;
    }
    if (c->m.n2e && (c->J & 1) == 0) {
        // all elements in one launch into an element buffer, then one ordered gather per row
        const int J = c->J;
        const int JB = J < 128 ? J : 128;
        const int EPB = 128 / JB > 0 ? 128 / JB : 1;
        const int threads = EPB * JB;
        const size_t shm = sizeof(double) * ((size_t)EPB * 2 * ENS_NQ * JB + (size_t)EPB * 24 + (size_t)EPB * ENS_NQ * 12);
        const size_t ecb = sizeof(double) * 2 * (size_t)c->m.nt * 12 * J;
        if (!c->ec) {
            ENS_CK(cudaMalloc(&c->ec, ecb));
            c->ws_bytes += ecb;
        }
        ENS_CK(cudaMemsetAsync(maxsq, 0, sizeof(double) * 2 * (size_t)c->m.nt * ENS_NQ, s));
        dim3 grid((c->m.nt + EPB - 1) / EPB, (J + JB - 1) / JB);
        k_member_pass<false><<<grid, threads, shm, s>>>(c->m.e_nodes, c->m.e_geo, 0, c->m.nt, x, means, rhs,
                                                         reinterpret_cast<unsigned long long*>(maxsq), c->m.nt,
                                                         c->n_vel, c->n_total, J, JB, c->ec, nullptr, 0.0);
        ENS_CKL();
        const int64_t tot = 2LL * c->m.ns * (J / 2);
        k_member_gather<false><<<dim3((unsigned)((tot + 255) / 256), 2), 256, 0, s>>>(
            c->m.n2e_ptr, c->m.n2e, c->ec, rhs, c->m.ns, c->m.nt, c->n_total, J, 0, nullptr, nullptr, nullptr);
        ENS_CKL();
        return ENS_OK;
    }
    const int J = c->J;
    const int JB = J < 128 ? J : 128;
    const int EPB = 128 / JB > 0 ? 128 / JB : 1;
    const int threads = EPB * JB;
    const size_t shm = sizeof(double) * ((size_t)EPB * 2 * ENS_NQ * JB + (size_t)EPB * 24 + (size_t)EPB * ENS_NQ * 12);
    ENS_CK(cudaMemsetAsync(maxsq, 0, sizeof(double) * 2 * (size_t)c->m.nt * ENS_NQ, s));
    for (int col = 0; col < c->m.ncolor; ++col) {
        const int e0 = c->color_off[col], ne = c->color_off[col + 1] - e0;
        if (ne == 0) continue;
        dim3 grid((ne + EPB - 1) / EPB, (J + JB - 1) / JB);
        k_member_pass<false><<<grid, threads, shm, s>>>(c->m.e_nodes, c->m.e_geo, e0, ne, x, means, rhs,
                                                         reinterpret_cast<unsigned long long*>(maxsq), c->m.nt,
                                                         c->n_vel, c->n_total, J, JB, nullptr, nullptr, 0.0);
        ENS_CKL();
    }
    return ENS_OK;
}

// whole velocity right-hand side of both sub-steps and the eddy-viscosity maxima in one element
// pass + one ordered row gather (replaces launch_rhs + launch_member_pass for even J)
int launch_rhs_fused(ens_ctx* c, cudaStream_t s, const double* x, const double* means, const double* coef,
                     double inv_dt, const ens_data_desc* loads, double* rhs, double* maxsq) {
    const int J = c->J;
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(rhs) |
                           (loads && loads->dense ? reinterpret_cast<uintptr_t>(loads->dense) : 0)) & 15) == 0;
    if (!c->m.n2e || (J & 1) || !aligned) {
        const int rc = launch_rhs(c, s, x, coef, inv_dt, loads, rhs);
        if (rc != ENS_OK) return rc;
        return launch_member_pass(c, s, x, means, rhs, maxsq);
    }
    const int64_t N = c->n_total;
    {
        const int rc = member_pass_smem_setup();
        if (rc != ENS_OK) return rc;
    }
    for (int mat = 0; mat < 2; ++mat)   // pressure rows of the right-hand side are zero (stepper.py:245-246)
        ENS_CK(cudaMemsetAsync(rhs + mat * N * J + (int64_t)c->n_vel * J, 0,
                               sizeof(double) * (size_t)c->m.n_pres * J, s));
    const int JB = J < 128 ? J : 128;
    const int EPB = 128 / JB > 0 ? 128 / JB : 1;
    const int threads = EPB * JB;
    const size_t shm = sizeof(double) * ((size_t)EPB * 2 * ENS_NQ * JB + (size_t)EPB * 24 + (size_t)EPB * ENS_NQ * 12);
    const size_t ecb = sizeof(double) * 2 * (size_t)c->m.nt * 12 * J;
    if (!c->ec) {
        ENS_CK(cudaMalloc(&c->ec, ecb));
        c->ws_bytes += ecb;
    }
    ENS_CK(cudaMemsetAsync(maxsq, 0, sizeof(double) * 2 * (size_t)c->m.nt * ENS_NQ, s));
    dim3 grid((c->m.nt + EPB - 1) / EPB, (J + JB - 1) / JB);
    k_member_pass<true><<<grid, threads, shm, s>>>(c->m.e_nodes, c->m.e_geo, 0, c->m.nt, x, means, rhs,
                                                    reinterpret_cast<unsigned long long*>(maxsq), c->m.nt, c->n_vel,
                                                    N, J, JB, c->ec, coef, inv_dt);
    ENS_CKL();
    const int64_t tot = 2LL * c->m.ns * (J / 2);
    k_member_gather<true><<<dim3((unsigned)((tot + 255) / 256), 2), 256, 0, s>>>(
        c->m.n2e_ptr, c->m.n2e, c->ec, rhs, c->m.ns, c->m.nt, N, J, loads ? loads->K : 0,
        loads ? loads->basis : nullptr, loads ? loads->coef : nullptr, loads ? loads->dense : nullptr);
    ENS_CKL();
    return ENS_OK;
}

// ---------------------------------------------------------------------------
// identity rows: Dirichlet data / pin (stepper.py:250-251)
// ---------------------------------------------------------------------------
__global__ void k_apply_bc(const int32_t* __restrict__ crow, const int32_t* __restrict__ cbidx, int ncons, int K,
                           const double* __restrict__ basis, int64_t brows, const double* __restrict__ coef,
                           const double* __restrict__ dense, double* __restrict__ rhs, int64_t N, int J) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)ncons * J;
    if (t >= 2 * per) return;
    const int mat = (int)(t / per);
    const int64_t u = t - mat * per;
    const int ci = (int)(u / J), j = (int)(u % J);
    const int b = cbidx[ci];
    double val = 0.0;
    if (b >= 0) {
        for (int k = 0; k < K; ++k) val += coef[((int64_t)mat * K + k) * J + j] * basis[(int64_t)k * brows + b];
        if (dense) val += dense[((int64_t)mat * brows + b) * J + j];
    }
    rhs[(int64_t)mat * N * J + (int64_t)crow[ci] * J + j] = val;
}

int launch_apply_bc(ens_ctx* c, cudaStream_t s, const ens_data_desc* bv, double* rhs) {
    if (c->m.ncons == 0) return ENS_OK;
    const int64_t tot = 2LL * c->m.ncons * c->J;
    const int64_t brows = bv ? bv->rows : 0;
    k_apply_bc<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(c->m.cons_row, c->m.cons_bidx, c->m.ncons,
                                                             bv ? bv->K : 0, bv ? bv->basis : nullptr, brows,
                                                             bv ? bv->coef : nullptr, bv ? bv->dense : nullptr, rhs,
                                                             c->n_total, c->J);
    ENS_CKL();
    return ENS_OK;
}

__global__ void k_copy_cons(const int32_t* __restrict__ crow, int ncons, const double* __restrict__ src,
                            double* __restrict__ dst, int64_t N, int J) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)ncons * J;
    if (t >= 2 * per) return;
    const int mat = (int)(t / per);
    const int64_t u = t - mat * per;
    const int64_t idx = (int64_t)mat * N * J + (int64_t)crow[u / J] * J + (u % J);
    dst[idx] = src[idx];
}

int launch_copy_cons(ens_ctx* c, cudaStream_t s, const double* src, double* dst) {
    if (c->m.ncons == 0) return ENS_OK;
    const int64_t tot = 2LL * c->m.ncons * c->J;
    k_copy_cons<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(c->m.cons_row, c->m.ncons, src, dst, c->n_total, c->J);
    ENS_CKL();
    return ENS_OK;
}

// ---------------------------------------------------------------------------
// shared velocity-block values (stepper.py:195-206): one thread per element,
// colours make the 36 slot writes conflict-free; V uses <w>, W uses <v>.
// ---------------------------------------------------------------------------
__global__ void k_assemble(const int32_t* __restrict__ enodes, const double* __restrict__ egeo,
                           const int32_t* __restrict__ eslots, int e0, int ne, const double* __restrict__ means,
                           const double* __restrict__ maxsq, double two_mu_dt, double* __restrict__ vals, int nt,
                           int nvel, int nnz, double* __restrict__ el) {
    const int e = e0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e0 + ne) return;
    const int mat = blockIdx.y;
    const double* mean = means + (mat == 0 ? nvel : 0);
    const double* msq = maxsq + ((int64_t)mat * nt + e) * ENS_NQ;
    double* out = vals + (int64_t)mat * nnz;
    double gl[6];
    const double area = egeo[(int64_t)e * 8];
#pragma unroll
    for (int i = 0; i < 6; ++i) gl[i] = egeo[(int64_t)e * 8 + 1 + i];
    double bx[6], by[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) {
        const int64_t nd = enodes[(int64_t)e * 6 + a];
        bx[a] = mean[2 * nd];
        by[a] = mean[2 * nd + 1];
    }
    double loc[6][6];
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int b = 0; b < 6; ++b) loc[a][b] = 0.0;
#pragma unroll 1
    for (int q = 0; q < ENS_NQ; ++q) {
        double gx[6], gy[6];
        double bqx = 0.0, bqy = 0.0;
#pragma unroll
        for (int a = 0; a < 6; ++a) {
            grad_phi(gl, q, a, gx[a], gy[a]);
            bqx += bx[a] * c_phi[q][a];
            bqy += by[a] * c_phi[q][a];
        }
        const double wd = area * c_qw[q];
        const double cq = wd * two_mu_dt * msq[q];
#pragma unroll
        for (int b = 0; b < 6; ++b) {
            const double tb = wd * (bqx * gx[b] + bqy * gy[b]);
#pragma unroll
            for (int a = 0; a < 6; ++a) loc[a][b] += tb * c_phi[q][a] + cq * (gx[a] * gx[b] + gy[a] * gy[b]);
        }
    }
    if (el) {   // element-local buffer [mat][ab][e], gathered per CSR slot by k_assemble_gather
        double* o = el + (int64_t)mat * 36 * nt + e;
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
            for (int b = 0; b < 6; ++b) o[(int64_t)(a * 6 + b) * nt] = loc[a][b];
        return;
    }
    const int32_t* sl = eslots + (int64_t)e * 36;
#pragma unroll
    for (int a = 0; a < 6; ++a)
#pragma unroll
        for (int b = 0; b < 6; ++b) out[sl[a * 6 + b]] += loc[a][b];
}

// vals[mat][slot] = base[slot] + sum of the slot's element-local entries (fixed order)
__global__ void __launch_bounds__(256) k_assemble_gather(const int32_t* __restrict__ s2e_ptr,
                                                         const int32_t* __restrict__ s2e,
                                                         const double* __restrict__ el,
                                                         const double* __restrict__ base, double* __restrict__ vals,
                                                         int nnz, int nt) {
    const int sidx = blockIdx.x * blockDim.x + threadIdx.x;
    if (sidx >= nnz) return;
    const int mat = blockIdx.y;
    const double* elm = el + (int64_t)mat * 36 * nt;
    double acc = base[sidx];
    const int k0 = s2e_ptr[sidx], k1 = s2e_ptr[sidx + 1];
    for (int k = k0; k < k1; ++k) acc += elm[s2e[k]];
    vals[(int64_t)mat * nnz + sidx] = acc;
}

int launch_assemble(ens_ctx* c, cudaStream_t s, const double* base, const double* means, const double* maxsq,
                    double two_mu_dt, double* as_vals) {
    if (c->m.s2e) {
        const size_t elb = sizeof(double) * 2 * 36 * (size_t)c->m.nt;
        if (!c->el) {
            ENS_CK(cudaMalloc(&c->el, elb));
            c->ws_bytes += elb;
        }
        dim3 grid((c->m.nt + 127) / 128, 2);
        k_assemble<<<grid, 128, 0, s>>>(c->m.e_nodes, c->m.e_geo, c->m.e_slots, 0, c->m.nt, means, maxsq, two_mu_dt,
                                       as_vals, c->m.nt, c->n_vel, c->m.nnz_s, c->el);
        ENS_CKL();
        k_assemble_gather<<<dim3((unsigned)((c->m.nnz_s + 255) / 256), 2), 256, 0, s>>>(
            c->m.s2e_ptr, c->m.s2e, c->el, base, as_vals, c->m.nnz_s, c->m.nt);
        ENS_CKL();
        return ENS_OK;
    }
    const size_t nb = sizeof(double) * (size_t)c->m.nnz_s;
    ENS_CK(cudaMemcpyAsync(as_vals, base, nb, cudaMemcpyDeviceToDevice, s));
    ENS_CK(cudaMemcpyAsync(as_vals + c->m.nnz_s, base, nb, cudaMemcpyDeviceToDevice, s));
    for (int col = 0; col < c->m.ncolor; ++col) {
        const int e0 = c->color_off[col], ne = c->color_off[col + 1] - e0;
        if (ne == 0) continue;
        dim3 grid((ne + 127) / 128, 2);
        k_assemble<<<grid, 128, 0, s>>>(c->m.e_nodes, c->m.e_geo, c->m.e_slots, e0, ne, means, maxsq, two_mu_dt,
                                       as_vals, c->m.nt, c->n_vel, c->m.nnz_s, nullptr);
        ENS_CKL();
    }
    return ENS_OK;
}

// ---------------------------------------------------------------------------
// deterministic column reductions: out[mat][l][j] = sum_r A_l[mat][r][j] B[mat][r][j]
// fixed grid of ENS_RED_BLOCKS row blocks -> partials -> ordered finalize
// ---------------------------------------------------------------------------
__global__ void k_coldot_part(const double* __restrict__ A, int64_t lstride, const double* __restrict__ B,
                              int64_t rows, int64_t matstride, int J, int L, double* __restrict__ part) {
    // grid: (RB, L, 2); block 256; thread -> (row offset, column)
    __shared__ double red[256];
    const int l = blockIdx.y, mat = blockIdx.z;
    const double* a = A + (int64_t)l * lstride + (int64_t)mat * matstride;
    const double* b = B + (int64_t)mat * matstride;
    const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per;
    const int64_t r1 = min(rows, r0 + per);
    for (int jc = 0; jc < J; jc += 256) {
        const int JB = min(256, J - jc);
        const int RPB = 256 / JB;
        const int jj = threadIdx.x % JB, ro = threadIdx.x / JB;
        double acc = 0.0;
        if (ro < RPB) {
            for (int64_t r = r0 + ro; r < r1; r += RPB) {
                const int64_t idx = r * J + jc + jj;
                acc += a[idx] * b[idx];
            }
        }
        red[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < JB) {
            double s = 0.0;
            for (int k = 0; k < RPB; ++k) s += red[k * JB + threadIdx.x];
            part[(((int64_t)blockIdx.x * 2 + mat) * L + l) * J + jc + threadIdx.x] = s;
        }
        __syncthreads();
    }
}

__global__ void k_coldot_fin(const double* __restrict__ part, int RB, int L, int J, double* __restrict__ out);

// W -= sum_l V_l h[mat][l][j] and per-block partial sums of the new W^2 per column
__global__ void k_axpy_norm_part(double* __restrict__ W, const double* __restrict__ V, int64_t lstride, int L,
                                 const double* __restrict__ h, int64_t rows, int64_t matstride, int J,
                                 double* __restrict__ part) {
    __shared__ double red[256];
    const int mat = blockIdx.z;
    const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per;
    const int64_t r1 = min(rows, r0 + per);
    for (int jc = 0; jc < J; jc += 256) {
        const int JB = min(256, J - jc);
        const int RPB = 256 / JB;
        const int jj = threadIdx.x % JB, ro = threadIdx.x / JB;
        const int j = jc + jj;
        double hl[ENS_MAX_RESTART + 1];
        for (int l = 0; l < L; ++l) hl[l] = h[((int64_t)mat * L + l) * J + j];
        double acc = 0.0;
        if (ro < RPB) {
            for (int64_t r = r0 + ro; r < r1; r += RPB) {
                const int64_t idx = (int64_t)mat * matstride + r * J + j;
                double s = 0.0;
                for (int l = 0; l < L; ++l) s += V[(int64_t)l * lstride + idx] * hl[l];
                const double w = W[idx] - s;
                W[idx] = w;
                acc += w * w;
            }
        }
        red[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < JB) {
            double s2 = 0.0;
            for (int k = 0; k < RPB; ++k) s2 += red[k * JB + threadIdx.x];
            part[((int64_t)blockIdx.x * 2 + mat) * J + j] = s2;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_axpy_norm_part2(double* __restrict__ W, const double* __restrict__ V,
                                                         int64_t lstride, int L, const double* __restrict__ h,
                                                         int64_t rows, int64_t matstride, int J,
                                                         double* __restrict__ part) {
    __shared__ double2 red[256];
    const int mat = blockIdx.z;
    const int H = J >> 1;
    const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per;
    const int64_t r1 = min(rows, r0 + per);
    const int RPB = 256 / H;
    const int jp = threadIdx.x % H, ro = threadIdx.x / H;
    double2 hl[ENS_MAX_RESTART + 1];
    for (int l = 0; l < L; ++l)
        hl[l] = ro < RPB ? reinterpret_cast<const double2*>(h + ((int64_t)mat * L + l) * J)[jp] : make_double2(0, 0);
    double2* w2 = reinterpret_cast<double2*>(W + (int64_t)mat * matstride);
    const double2* v2 = reinterpret_cast<const double2*>(V + (int64_t)mat * matstride);
    double2 acc[2] = {{0.0, 0.0}, {0.0, 0.0}};
    if (ro < RPB) {
        int64_t r = r0 + ro;
        for (int u = 0; r < r1; r += RPB, u ^= 1) {
            const int64_t i = r * H + jp;
            double2 sum = make_double2(0.0, 0.0);
            for (int l = 0; l < L; ++l) {
                const double2 v = v2[(int64_t)l * (lstride >> 1) + i];
                sum.x += v.x * hl[l].x;
                sum.y += v.y * hl[l].y;
            }
            double2 w = w2[i];
            w.x -= sum.x;
            w.y -= sum.y;
            w2[i] = w;
            acc[u].x += w.x * w.x;
            acc[u].y += w.y * w.y;
        }
    }
    red[threadIdx.x] = make_double2(acc[0].x + acc[1].x, acc[0].y + acc[1].y);
    __syncthreads();
    if (threadIdx.x < H) {
        double2 sum = make_double2(0.0, 0.0);
        for (int k = 0; k < RPB; ++k) {
            sum.x += red[k * H + threadIdx.x].x;
            sum.y += red[k * H + threadIdx.x].y;
        }
        double* o = part + ((int64_t)blockIdx.x * 2 + mat) * J + 2 * threadIdx.x;
        o[0] = sum.x;
        o[1] = sum.y;
    }
}

int launch_axpy_norm(ens_ctx* c, cudaStream_t s, double* W, const double* V, int64_t lstride, int L,
                     const double* h, int64_t rows, double* out) {
    const int RB = ENS_RED_BLOCKS;
    if (L > ENS_MAX_RESTART + 1) return ENS_EINVAL;
    if (red_vec_ok(c->J, W, V) && (lstride & 1) == 0)
        k_axpy_norm_part2<<<dim3(RB, 1, 2), 256, 0, s>>>(W, V, lstride, L, h, rows, (int64_t)c->n_total * c->J, c->J,
                                                        c->red_part);
    else
        k_axpy_norm_part<<<dim3(RB, 1, 2), 256, 0, s>>>(W, V, lstride, L, h, rows, (int64_t)c->n_total * c->J, c->J,
                                                       c->red_part);
    ENS_CKL();
    const int tot = 2 * c->J;
    k_coldot_fin<<<(tot * 32 + 255) / 256, 256, 0, s>>>(c->red_part, RB, 1, c->J, out);
    ENS_CKL();
    return ENS_OK;
}

// one warp per output: lanes sum a fixed strided subset of the partials, then a
// fixed butterfly -- same order for every output, so identical columns agree bitwise
__global__ void k_coldot_fin(const double* __restrict__ part, int RB, int L, int J, double* __restrict__ out) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int tot = 2 * L * J;
    if (t >= tot) return;
    double s = 0.0;
    for (int b = lane; b < RB; b += 32) s += part[(int64_t)b * tot + t];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[t] = s;
}

// even J: 16-byte lanes (member pairs), 4 independent row streams per thread.
// Fixed row partition and summation order => deterministic, identical columns agree.
__global__ void __launch_bounds__(256) k_coldot_part2(const double* __restrict__ A, int64_t lstride,
                                                      const double* __restrict__ B, int64_t rows, int64_t matstride,
                                                      int J, int L, double* __restrict__ part) {
    __shared__ double2 red[256];
    const int l = blockIdx.y, mat = blockIdx.z;
    const int H = J >> 1;
    const double2* a = reinterpret_cast<const double2*>(A + (int64_t)l * lstride + (int64_t)mat * matstride);
    const double2* b = reinterpret_cast<const double2*>(B + (int64_t)mat * matstride);
    const int64_t per = (rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per;
    const int64_t r1 = min(rows, r0 + per);
    const int RPB = 256 / H;
    const int jp = threadIdx.x % H, ro = threadIdx.x / H;
    double2 acc[4] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    if (ro < RPB) {
        int64_t r = r0 + ro;
        for (; r + 3 * RPB < r1; r += 4 * RPB) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t i = (r + u * RPB) * H + jp;
                const double2 x = a[i], y = b[i];
                acc[u].x += x.x * y.x;
                acc[u].y += x.y * y.y;
            }
        }
        for (int u = 0; r < r1; r += RPB, ++u) {
            const int64_t i = r * H + jp;
            const double2 x = a[i], y = b[i];
            acc[u].x += x.x * y.x;
            acc[u].y += x.y * y.y;
        }
    }
    red[threadIdx.x] = make_double2((acc[0].x + acc[1].x) + (acc[2].x + acc[3].x),
                                    (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y));
    __syncthreads();
    if (threadIdx.x < H) {
        double2 sum = make_double2(0.0, 0.0);
        for (int k = 0; k < RPB; ++k) {
            sum.x += red[k * H + threadIdx.x].x;
            sum.y += red[k * H + threadIdx.x].y;
        }
        double* o = part + (((int64_t)blockIdx.x * 2 + mat) * L + l) * J + 2 * threadIdx.x;
        o[0] = sum.x;
        o[1] = sum.y;
    }
}

int launch_coldot(ens_ctx* c, cudaStream_t s, const double* A, int64_t lstride, int L, const double* B,
                  int64_t rows, double* out) {
    const int RB = ENS_RED_BLOCKS;
    dim3 grid(RB, L, 2);
    if (red_vec_ok(c->J, A, B) && (lstride & 1) == 0)
        k_coldot_part2<<<grid, 256, 0, s>>>(A, lstride, B, rows, (int64_t)c->n_total * c->J, c->J, L, c->red_part);
    else
        k_coldot_part<<<grid, 256, 0, s>>>(A, lstride, B, rows, (int64_t)c->n_total * c->J, c->J, L, c->red_part);
    ENS_CKL();
    const int tot = 2 * L * c->J;
    k_coldot_fin<<<(tot * 32 + 255) / 256, 256, 0, s>>>(c->red_part, RB, L, c->J, out);
    ENS_CKL();
    return ENS_OK;
}

// ---------------------------------------------------------------------------
// pressure epilogue (stepper.py:119-123): p -= (p . int rho) / area per member
// ---------------------------------------------------------------------------
__global__ void k_pres_dot(const double* __restrict__ X, const double* __restrict__ w, int64_t nvel, int npres,
                           int64_t N, int J, double* __restrict__ part) {
    __shared__ double red[256];
    const int mat = blockIdx.z;
    const double* x = X + (int64_t)mat * N * J + nvel * J;
    const int64_t per = ((int64_t)npres + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min((int64_t)npres, r0 + per);
    for (int jc = 0; jc < J; jc += 256) {
        const int JB = min(256, J - jc);
        const int RPB = 256 / JB;
        const int jj = threadIdx.x % JB, ro = threadIdx.x / JB;
        double acc = 0.0;
        if (ro < RPB)
            for (int64_t r = r0 + ro; r < r1; r += RPB) acc += x[r * J + jc + jj] * w[r];
        red[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < JB) {
            double s2 = 0.0;
            for (int k = 0; k < RPB; ++k) s2 += red[k * JB + threadIdx.x];
            part[((int64_t)blockIdx.x * 2 + mat) * J + jc + threadIdx.x] = s2;
        }
        __syncthreads();
    }
}

// means[mat][j] = sum of the RB partials (fixed order, warp per output) / area
__global__ void k_pres_fin(const double* __restrict__ part, int RB, int J, double inv_area, double* __restrict__ mean) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= 2 * J) return;
    const int mat = t / J, j = t % J;
    double s = 0.0;
    for (int b = lane; b < RB; b += 32) s += part[((int64_t)b * 2 + mat) * J + j];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) mean[t] = s * inv_area;
}

__global__ void k_pres_sub(const double* __restrict__ X, const double* __restrict__ mean, int64_t nvel, int npres,
                           int64_t N, int J, double* __restrict__ P) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)npres * J;
    if (t >= 2 * per) return;
    const int mat = (int)(t / per);
    const int64_t u = t - mat * per;
    const int j = (int)(u % J);
    P[t] = X[(int64_t)mat * N * J + nvel * J + u] - (mean ? mean[mat * J + j] : 0.0);
}

int launch_epilogue(ens_ctx* c, cudaStream_t s, const double* x, double* p_out) {
    const int RB = 148;
    double* mean = nullptr;
    if (c->m.mean_zero) {
        dim3 grid(RB, 1, 2);
        k_pres_dot<<<grid, 256, 0, s>>>(x, c->m.pres_int, c->n_vel, c->m.n_pres, c->n_total, c->J, c->red_part);
        ENS_CKL();
        // 2J doubles past the Krylov scalars [bn2|rn2|h1|h2|hn2|scale|y] of the small-output area
        mean = c->red_out + 2 * (size_t)c->J * (4 + 3 * (ENS_MAX_RESTART + 1));
        k_pres_fin<<<(2 * c->J * 32 + 255) / 256, 256, 0, s>>>(c->red_part, RB, c->J, 1.0 / c->m.area, mean);
        ENS_CKL();
    }
    const int64_t tot = 2LL * c->m.n_pres * c->J;
    k_pres_sub<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(x, mean, c->n_vel, c->m.n_pres, c->n_total, c->J, p_out);
    ENS_CKL();
    return ENS_OK;
}

// ---------------------------------------------------------------------------
// diagnostics (stepper.py:397-439, fem.py:508-514)
// ---------------------------------------------------------------------------
// energy of the means: mean^T M mean for v and w (single block per family, ordered)
// grid (RBm, 2): block b of family fam sums a fixed node range -> part[fam][b]; k_diag_fin adds the
// partials in order
__global__ void k_mean_energy(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const double* __restrict__ mass, const double* __restrict__ means, int ns,
                              double* __restrict__ part) {
    __shared__ double red[256];
    const int fam = blockIdx.y;
    const double* m = means + (int64_t)fam * 2 * ns;
    const int64_t per = ((int64_t)ns + gridDim.x - 1) / gridDim.x;
    const int64_t n0 = (int64_t)blockIdx.x * per, n1 = min((int64_t)ns, n0 + per);
    double acc = 0.0;
    for (int64_t i = n0 + threadIdx.x; i < n1; i += blockDim.x) {
        for (int cc = 0; cc < 2; ++cc) {
            double s = 0.0;
            for (int k = rp[i]; k < rp[i + 1]; ++k) s += mass[k] * m[2LL * col[k] + cc];
            acc += m[2 * i + cc] * s;
        }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int k = 0; k < (int)blockDim.x; ++k) s += red[k];
        part[(int64_t)fam * gridDim.x + blockIdx.x] = s;
    }
}

// Error of the ensemble means against a separable exact field, in the mass and stiffness forms
// (the squared H1 norm of the mean error, experiments.py:59-73 / fem.py:502-505):
//   d = <z> - sum_k coef[fam][k] basis[k]   (internal order, both components interleaved)
//   part[(fam*2 + 0)][blk] = d^T M d,  part[(fam*2 + 1)][blk] = d^T K d   (M, K per component)
// Fixed row partition and block order: deterministic.
__global__ void k_mean_error(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const double* __restrict__ mass, const double* __restrict__ stiff,
                             const double* __restrict__ means, int ns, const double* __restrict__ basis,
                             const double* __restrict__ coef, int K, double* __restrict__ part) {
    __shared__ double red[2][256];
    const int fam = blockIdx.y;
    const int64_t nv = 2LL * ns;
    const double* m = means + (int64_t)fam * nv;
    const double* cf = coef + (int64_t)fam * K;
    auto d = [&](int64_t r) {
        double v = m[r];
        for (int k = 0; k < K; ++k) v -= cf[k] * basis[(int64_t)k * nv + r];
        return v;
    };
    const int64_t per = ((int64_t)ns + gridDim.x - 1) / gridDim.x;
    const int64_t n0 = (int64_t)blockIdx.x * per, n1 = min((int64_t)ns, n0 + per);
    double am = 0.0, ak = 0.0;
    for (int64_t i = n0 + threadIdx.x; i < n1; i += blockDim.x) {
        for (int cc = 0; cc < 2; ++cc) {
            double sm = 0.0, sk = 0.0;
            for (int k = rp[i]; k < rp[i + 1]; ++k) {
                const double dj = d(2LL * col[k] + cc);
                sm += mass[k] * dj;
                sk += stiff[k] * dj;
            }
            const double di = d(2 * i + cc);
            am += di * sm;
            ak += di * sk;
        }
    }
    red[0][threadIdx.x] = am;
    red[1][threadIdx.x] = ak;
    __syncthreads();
    if (threadIdx.x < 2) {
        double t = 0.0;
        for (int k = 0; k < (int)blockDim.x; ++k) t += red[threadIdx.x][k];
        part[(int64_t)(fam * 2 + threadIdx.x) * gridDim.x + blockIdx.x] = t;
    }
}

__global__ void k_mean_error_fin(const double* __restrict__ part, int nblk, double* __restrict__ out) {
    const int t = threadIdx.x;
    if (t >= 4) return;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(int64_t)t * nblk + b];
    out[t] = s;
}

int launch_mean_error(ens_ctx* c, cudaStream_t s, const double* means, const ens_data_desc* exact, double* out) {
    const int RB = 148 * 2;
    const size_t need = (size_t)RB * 4;
    if (c->diag_part_n < need) {
        cudaFree(c->diag_part);
        c->diag_part = nullptr;
        ENS_CK(cudaMalloc(&c->diag_part, sizeof(double) * need));
        c->diag_part_n = need;
    }
    k_mean_error<<<dim3(RB, 2), 256, 0, s>>>(c->m.s_rowptr, c->m.s_col, c->m.s_mass, c->m.s_stiff, means, c->m.ns,
                                            exact->basis, exact->coef, exact->K, c->diag_part);
    ENS_CKL();
    k_mean_error_fin<<<1, 32, 0, s>>>(c->diag_part, RB, out);
    ENS_CKL();
    return ENS_OK;
}

// Per-member quadratic forms by element quadrature, thread per (element, member), per-block
// partials part[blk][6][J]: v.Mv, w.Mw, v.Kv, w.Kw (K applied per component), ||div v||^2, ||div w||^2.
// The 7-point rule integrates the P2 mass (degree 4) and stiffness (degree 2) integrands exactly,
// so these equal the assembled-matrix forms (stepper.py:113-114, 397-439; fem.py:508-514) up to
// rounding.
__global__ void k_member_quad(const int32_t* __restrict__ enodes, const double* __restrict__ egeo, int nt,
                              const double* __restrict__ X, int64_t N, int J, int JB, double* __restrict__ part) {
    extern __shared__ double red6[];   // [6][blockDim]
    const int EPB = blockDim.x / JB;
    const int el = threadIdx.x / JB, jj = threadIdx.x % JB;
    const int j = blockIdx.y * JB + jj;
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (el < EPB && j < J) {
        for (int e = blockIdx.x * EPB + el; e < nt; e += gridDim.x * EPB) {
            double gl[6];
            const double area = egeo[(int64_t)e * 8];
#pragma unroll
            for (int i = 0; i < 6; ++i) gl[i] = egeo[(int64_t)e * 8 + 1 + i];
            double z[2][6][2];   // [field v/w][node][comp]
#pragma unroll
            for (int a = 0; a < 6; ++a) {
                const int64_t nd = enodes[(int64_t)e * 6 + a];
#pragma unroll
                for (int f = 0; f < 2; ++f)
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) z[f][a][cc] = X[(int64_t)f * N * J + (2 * nd + cc) * J + j];
            }
            for (int q = 0; q < ENS_NQ; ++q) {
                double val[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, grd[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}},
                                                                           {{0.0, 0.0}, {0.0, 0.0}}};
#pragma unroll
                for (int a = 0; a < 6; ++a) {
                    const double ph = c_phi[q][a];
                    double gx, gy;
                    grad_phi(gl, q, a, gx, gy);
#pragma unroll
                    for (int f = 0; f < 2; ++f)
#pragma unroll
                        for (int cc = 0; cc < 2; ++cc) {
                            val[f][cc] += z[f][a][cc] * ph;
                            grd[f][cc][0] += z[f][a][cc] * gx;
                            grd[f][cc][1] += z[f][a][cc] * gy;
                        }
                }
                const double wd = area * c_qw[q];
#pragma unroll
                for (int f = 0; f < 2; ++f) {
                    acc[f] += wd * (val[f][0] * val[f][0] + val[f][1] * val[f][1]);
                    acc[2 + f] += wd * (grd[f][0][0] * grd[f][0][0] + grd[f][0][1] * grd[f][0][1] +
                                        grd[f][1][0] * grd[f][1][0] + grd[f][1][1] * grd[f][1][1]);
                    const double dv = grd[f][0][0] + grd[f][1][1];
                    acc[4 + f] += wd * dv * dv;
                }
            }
        }
    }
#pragma unroll
    for (int f = 0; f < 6; ++f) red6[f * blockDim.x + threadIdx.x] = acc[f];
    __syncthreads();
    if (threadIdx.x < JB && j < J) {
        for (int f = 0; f < 6; ++f) {
            double a = 0.0;
            for (int k = 0; k < EPB; ++k) a += red6[f * blockDim.x + k * JB + threadIdx.x];
            part[((int64_t)blockIdx.x * 6 + f) * J + j] = a;
        }
    }
}

__global__ void k_diag_fin(const double* __restrict__ pd, int RBd, int J, const double* __restrict__ pm, int RBm,
                           double* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 6 * J + 2) return;
    if (t >= 6 * J) {   // mean energies <v> M <v>, <w> M <w>
        const int fam = t - 6 * J;
        double s = 0.0;
        for (int b = 0; b < RBm; ++b) s += pm[(int64_t)fam * RBm + b];
        out[fam] = s;
        return;
    }
    const int f = t / J, j = t % J;
    double s = 0.0;
    for (int b = 0; b < RBd; ++b) s += pd[((int64_t)b * 6 + f) * J + j];
    // out layout: vMv, wMw, vKv, wKw, div_v^2, div_w^2
    out[2 + (int64_t)f * J + j] = s;
}

int launch_diagnostics(ens_ctx* c, cudaStream_t s, const double* x, const double* means, double* out) {
    // fixed grids (deterministic partial orders) sized to fill the GPU: these run every step of
    // run() (`_record`, stepper.py:432-439)
    const int J = c->J;
    const int RBd = 148 * 8, RBm = 148 * 2;
    const size_t need = (size_t)RBd * 6 * J + (size_t)RBm * 2;
    if (c->diag_part_n < need) {
        cudaFree(c->diag_part);
        c->diag_part = nullptr;
        ENS_CK(cudaMalloc(&c->diag_part, sizeof(double) * need));
        c->diag_part_n = need;
    }
    double* pd = c->diag_part;
    double* pm = pd + (size_t)RBd * 6 * J;
    const int JB = J < 128 ? J : 128;
    const int EPB = 128 / JB > 0 ? 128 / JB : 1;
    dim3 grid(RBd, (J + JB - 1) / JB);
    // the y-dimension splits members; partial index uses blockIdx.x only (members disjoint per y)
    k_member_quad<<<grid, EPB * JB, sizeof(double) * 6 * EPB * JB, s>>>(c->m.e_nodes, c->m.e_geo, c->m.nt, x,
                                                                       c->n_total, J, JB, pd);
    ENS_CKL();
    k_mean_energy<<<dim3(RBm, 2), 256, 0, s>>>(c->m.s_rowptr, c->m.s_col, c->m.s_mass, means, c->m.ns, pm);
    ENS_CKL();
    k_diag_fin<<<(6 * J + 2 + 255) / 256, 256, 0, s>>>(pd, RBd, J, pm, RBm, out);
    ENS_CKL();
    return ENS_OK;
}

// ---------------------------------------------------------------------------
// state layout: reference order (member-major (J, n) blocks, reference dof numbering -- the
// EnsembleState arrays of ensemble.py:183-190) <-> the internal member-minor blocks in
// nested-dissection dof order.  One tile of LT_C reference dofs x LT_J members per CTA through
// shared memory: the reference side is read / written in 512-byte runs along the dofs, the
// internal side in whole member rows.  row[c] = internal row of reference dof c.
// ---------------------------------------------------------------------------
constexpr int LT_C = 64, LT_J = 64;

template <bool IMPORT>
__global__ void __launch_bounds__(256) k_layout(double* __restrict__ ref, int64_t ld, int64_t ref_ms, int64_t n,
                                                const int64_t* __restrict__ row, double* __restrict__ x,
                                                int64_t x_ms, int J) {
    __shared__ double tile[LT_C][LT_J + 1];
    __shared__ int64_t srow[LT_C];
    const int64_t c0 = (int64_t)blockIdx.x * LT_C;
    const int j0 = blockIdx.y * LT_J;
    const int nc = (int)min((int64_t)LT_C, n - c0), nj = min(LT_J, J - j0);
    double* R = ref + (int64_t)blockIdx.z * ref_ms;
    double* X = x + (int64_t)blockIdx.z * x_ms;
    if (threadIdx.x < nc) srow[threadIdx.x] = row[c0 + threadIdx.x];
    if (IMPORT) {
        for (int e = threadIdx.x; e < LT_C * nj; e += 256) {
            const int cl = e % LT_C, jj = e / LT_C;
            if (cl < nc) tile[cl][jj] = R[(int64_t)(j0 + jj) * ld + c0 + cl];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < nc * nj; e += 256) {
            const int cl = e / nj, jj = e - cl * nj;
            X[srow[cl] * J + j0 + jj] = tile[cl][jj];
        }
    } else {
        __syncthreads();
        for (int e = threadIdx.x; e < nc * nj; e += 256) {
            const int cl = e / nj, jj = e - cl * nj;
            tile[cl][jj] = X[srow[cl] * J + j0 + jj];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < LT_C * nj; e += 256) {
            const int cl = e % LT_C, jj = e / LT_C;
            if (cl < nc) R[(int64_t)(j0 + jj) * ld + c0 + cl] = tile[cl][jj];
        }
    }
}

int launch_layout(ens_ctx* c, cudaStream_t s, bool import, double* ref, int64_t ld, int64_t ref_ms, int64_t n,
                  const int64_t* row, double* x, int64_t x_ms, int nsys) {
    if (n <= 0) return ENS_OK;
    dim3 grid((unsigned)((n + LT_C - 1) / LT_C), (unsigned)((c->J + LT_J - 1) / LT_J), (unsigned)nsys);
    if (import)
        k_layout<true><<<grid, 256, 0, s>>>(ref, ld, ref_ms, n, row, x, x_ms, c->J);
    else
        k_layout<false><<<grid, 256, 0, s>>>(ref, ld, ref_ms, n, row, x, x_ms, c->J);
    ENS_CKL();
    return ENS_OK;
}
