// Saddle-operator SpMM for both sub-step systems (the Krylov core), fp64, sm_100a.
//
// Applies exactly the reference's assembled saddle matrix (stepper.py:208-215)
// to all J member columns at once (the product behind linalg.py:111-118).
// Layout: member-minor blocks, so one node's (x, y) values for all members are
// 2J contiguous doubles -> each nonzero gathers one coalesced segment that
// serves every member and both components.  A segment of S lanes owns a row;
// summation order is fixed per row and identical for every member column.
// (A variant that preloads the row's indices lane-parallel and broadcasts them
// with shuffles measured slower at C2: 0.24 ms vs 0.17 ms per launch pair.
// Later in round 1, also measured no faster (warm, both kernels, C2, J = 20,
// baseline 105-115 us): indices/values preloaded per warp into shared memory
// with 2- or 4-nonzero gather batches (121 / 127 us), evict-first hints on the
// streamed operands and output (120 us), register caps for 5 CTAs/SM (121-123
// us, spills), a 64-register cap (107-111 us); the tile-staged kernel
// (ens_spmm_tiles.cu) reached 123 us at best.)
#include <cstdlib>

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
    int k = k0;
    // 4 nonzeros per iteration: indices first, then 4 independent row gathers in flight
    for (; k + 4 <= k1; k += 4) {
        const int64_t c0 = col[k], c1 = col[k + 1], c2 = col[k + 2], c3 = col[k + 3];
        const double a0 = Am[k], a1 = Am[k + 1], a2 = Am[k + 2], a3 = Am[k + 3];
        const double* x0 = Xm + 2 * c0 * J;
        const double* x1 = Xm + 2 * c1 * J;
        const double* x2 = Xm + 2 * c2 * J;
        const double* x3 = Xm + 2 * c3 * J;
#pragma unroll
        for (int o = 0; o < OPL; ++o) {
            const int l = sl + o * S;
            if (l < W2) {
                const double v0 = x0[l], v1 = x1[l], v2 = x2[l], v3 = x3[l];
                acc[o] = fma(a0, v0, acc[o]);
                acc[o] = fma(a1, v1, acc[o]);
                acc[o] = fma(a2, v2, acc[o]);
                acc[o] = fma(a3, v3, acc[o]);
            }
        }
    }
    for (; k < k1; ++k) {
        const double a = Am[k];
        const double* xr = Xm + 2LL * col[k] * J;
#pragma unroll
        for (int o = 0; o < OPL; ++o) {
            const int l = sl + o * S;
            if (l < W2) acc[o] = fma(a, xr[l], acc[o]);
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

// ---------------------------------------------------------------------------
// Vectorised variant (even J): a row's 2J (velocity) or J (pressure) values are
// split over L lanes holding V2 double2 each, and 32/L rows share a warp.  Per
// nonzero a lane issues V2 16-byte loads and 2*V2 FMAs -- about a third of the
// scalar kernel's instructions per row at J = 20 (10 lanes x 3 rows per warp).
// Summation order per output is unchanged (CSR order, then B^T in order).
// ---------------------------------------------------------------------------
// fixed-order reduction of per-lane member-pair squares: row groups of the warp
// (lanes part + L*rr), then the block's warps; one partial row per block
__device__ __forceinline__ void nrm_block_reduce(double2 (&sq)[2][2], int lane, int part, int L, int R, int J,
                                                 double* __restrict__ nrm, int bid) {
    __shared__ double2 red[8][2][2][32];
    const int warp = threadIdx.x >> 5;
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int br = 0; br < 2; ++br) {
            double2 t = make_double2(0.0, 0.0);
            for (int rr = 0; rr < R; ++rr) {
                const double x = __shfl_sync(0xffffffffu, sq[m][br].x, part + L * rr);
                const double y = __shfl_sync(0xffffffffu, sq[m][br].y, part + L * rr);
                t.x += x;
                t.y += y;
            }
            if (lane < L) red[warp][m][br][lane] = t;
        }
    __syncthreads();
    const int nw = blockDim.x >> 5;
    for (int e = threadIdx.x; e < 2 * 2 * L; e += blockDim.x) {
        const int m = e / (2 * L), br = (e / L) & 1, p = e % L;
        double2 t = make_double2(0.0, 0.0);
        for (int w = 0; w < nw; ++w) {
            t.x += red[w][m][br][p].x;
            t.y += red[w][m][br][p].y;
        }
        double* o = nrm + (((int64_t)bid * 2 + m) * 2 + br) * J + 2 * p;
        o[0] = t.x;
        o[1] = t.y;
    }
}

// NRM (mode 1, V2 == 2, L == J/2): also the per-column squares of b and b - K x,
// reduced in fixed order (row groups of the warp, warps of the block) to one
// partial per block: nrm[blk][mat][{b, r}][J]
template <int V2, bool NRM>
__device__ __forceinline__ void spmm_vel_body(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                    const double* __restrict__ A, int nnz,
                                                    const int32_t* __restrict__ btp, const int32_t* __restrict__ btc,
                                                    const double* __restrict__ btv, const uint8_t* __restrict__ cflag,
                                                    const double* __restrict__ X, const double* __restrict__ Bv,
                                                    double* __restrict__ Y, int ns, int64_t N, int J, int L, int mode,
                                                    double* __restrict__ nrm, int bid) {
    // both systems per thread: one index stream feeds two independent gathers
    const int lane = threadIdx.x & 31;
    const int R = 32 / L;
    const int r = lane / L, part = lane - r * L;
    const int64_t gw = ((int64_t)bid * blockDim.x + threadIdx.x) >> 5;
    const int64_t node = gw * R + r;
    double2 sq[2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};   // [mat][b, r]
    if (!NRM && (r >= R || node >= ns)) return;
    if (r < R && node < ns) {
    const int H = J >> 1;                       // double2 per component
    const int64_t MS = N * H;                   // double2 per system block
    const double2* X2 = reinterpret_cast<const double2*>(X);
    double2* Y2 = reinterpret_cast<double2*>(Y);
    const double2* B2 = reinterpret_cast<const double2*>(Bv);
    const int64_t nvel = 2LL * ns;
    double2 acc[2][V2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int v = 0; v < V2; ++v) acc[m][v] = make_double2(0.0, 0.0);
    const int k0 = rp[node], k1 = rp[node + 1];
    int k = k0;
    for (; k + 2 <= k1; k += 2) {
        const int64_t c0 = col[k], c1 = col[k + 1];
        const double a00 = A[k], a01 = A[k + 1], a10 = A[nnz + k], a11 = A[nnz + k + 1];
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int i = part + L * v;   // lane-contiguous per v: fewer L1 lines per load
            if (i < J) {
                const double2 x00 = X2[c0 * J + i], x01 = X2[c1 * J + i];
                const double2 x10 = X2[MS + c0 * J + i], x11 = X2[MS + c1 * J + i];
                acc[0][v].x = fma(a00, x00.x, acc[0][v].x);
                acc[0][v].y = fma(a00, x00.y, acc[0][v].y);
                acc[1][v].x = fma(a10, x10.x, acc[1][v].x);
                acc[1][v].y = fma(a10, x10.y, acc[1][v].y);
                acc[0][v].x = fma(a01, x01.x, acc[0][v].x);
                acc[0][v].y = fma(a01, x01.y, acc[0][v].y);
                acc[1][v].x = fma(a11, x11.x, acc[1][v].x);
                acc[1][v].y = fma(a11, x11.y, acc[1][v].y);
            }
        }
    }
    for (; k < k1; ++k) {
        const int64_t c0 = col[k];
        const double a00 = A[k], a10 = A[nnz + k];
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int i = part + L * v;   // lane-contiguous per v: fewer L1 lines per load
            if (i < J) {
                const double2 x00 = X2[c0 * J + i], x10 = X2[MS + c0 * J + i];
                acc[0][v].x = fma(a00, x00.x, acc[0][v].x);
                acc[0][v].y = fma(a00, x00.y, acc[0][v].y);
                acc[1][v].x = fma(a10, x10.x, acc[1][v].x);
                acc[1][v].y = fma(a10, x10.y, acc[1][v].y);
            }
        }
    }
    // pressure couplings (same B^T for both systems): pressure rows are J wide at row nvel + p
    const int t0 = btp[node], t1 = btp[node + 1];
    const double2* P2 = X2 + nvel * H;
    for (int t = t0; t < t1; ++t) {
        const double2 b0 = reinterpret_cast<const double2*>(btv)[t];
        const int64_t p0 = btc[t];
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int i = part + L * v;   // lane-contiguous per v: fewer L1 lines per load
            if (i < J) {
                const bool ycomp = i >= H;
                const int64_t o = p0 * H + (ycomp ? i - H : i);
                const double2 x0 = P2[o], x1 = P2[MS + o];
                const double f0 = ycomp ? b0.y : b0.x;
                acc[0][v].x -= f0 * x0.x;
                acc[0][v].y -= f0 * x0.y;
                acc[1][v].x -= f0 * x1.x;
                acc[1][v].y -= f0 * x1.y;
            }
        }
    }
#pragma unroll
    for (int v = 0; v < V2; ++v) {
        const int i = part + L * v;   // lane-contiguous per v: fewer L1 lines per load
        if (i >= J) continue;
        const int64_t o = node * J + i;
        const bool ident = cflag[2 * node + (i >= H ? 1 : 0)] != 0;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            double2 val = ident ? X2[m * MS + o] : acc[m][v];
            if (mode == 1) {
                const double2 bb = B2[m * MS + o];
                val = make_double2(bb.x - val.x, bb.y - val.y);
                if (NRM) {
                    sq[m][0].x += bb.x * bb.x;
                    sq[m][0].y += bb.y * bb.y;
                    sq[m][1].x += val.x * val.x;
                    sq[m][1].y += val.y * val.y;
                }
            }
            Y2[m * MS + o] = val;
        }
    }
    }   // live row
    if (NRM) nrm_block_reduce(sq, lane, part, L, R, J, nrm, bid);
}

template <int V2, bool NRM>
__global__ void __launch_bounds__(256) k_spmm_vel_v(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                    const double* __restrict__ A, int nnz,
                                                    const int32_t* __restrict__ btp, const int32_t* __restrict__ btc,
                                                    const double* __restrict__ btv, const uint8_t* __restrict__ cflag,
                                                    const double* __restrict__ X, const double* __restrict__ Bv,
                                                    double* __restrict__ Y, int ns, int64_t N, int J, int L, int mode,
                                                    double* __restrict__ nrm) {
    spmm_vel_body<V2, NRM>(rp, col, A, nnz, btp, btc, btv, cflag, X, Bv, Y, ns, N, J, L, mode, nrm, blockIdx.x);
}

// NRM: as k_spmm_vel_v; a lane holds member pairs 2*part + v (v = 0, 1)
template <int V2, bool NRM>
__device__ __forceinline__ void spmm_pres_body(const int32_t* __restrict__ bp, const int32_t* __restrict__ bc,
                                                     const double* __restrict__ bv, const uint8_t* __restrict__ cflag,
                                                     const double* __restrict__ X, const double* __restrict__ Bv,
                                                     double* __restrict__ Y, int npres, int64_t nvel, int64_t N, int J,
                                                     int L, int mode, double* __restrict__ nrm, int bid) {
    const int lane = threadIdx.x & 31;
    const int R = 32 / L;
    const int r = lane / L, part = lane - r * L;
    const int64_t gw = ((int64_t)bid * blockDim.x + threadIdx.x) >> 5;
    const int64_t p = gw * R + r;
    double2 sq[2][2][2] = {};   // [v][mat][b, r]
    if (!NRM && (r >= R || p >= npres)) return;
    if (r < R && p < npres) {
    const int H = J >> 1;
    const int64_t MS = N * H;
    const double2* X2 = reinterpret_cast<const double2*>(X);
    double2* Y2 = reinterpret_cast<double2*>(Y);
    const double2* B2 = reinterpret_cast<const double2*>(Bv);
    const int64_t row = nvel + p;
    double2 acc[2][V2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int v = 0; v < V2; ++v) acc[m][v] = make_double2(0.0, 0.0);
    const int t0 = bp[p], t1 = bp[p + 1];
    for (int t = t0; t < t1; ++t) {
        const double2 b0 = reinterpret_cast<const double2*>(bv)[t];
        const int64_t n0 = bc[t];
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int i = V2 * part + v;
            if (i < H) {
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    const double2 u0 = X2[m * MS + n0 * J + i], w0 = X2[m * MS + n0 * J + H + i];
                    acc[m][v].x += b0.x * u0.x + b0.y * w0.x;
                    acc[m][v].y += b0.x * u0.y + b0.y * w0.y;
                }
            }
        }
    }
    const bool ident = cflag[row] != 0;
#pragma unroll
    for (int v = 0; v < V2; ++v) {
        const int i = V2 * part + v;
        if (i >= H) continue;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            const int64_t o = m * MS + row * H + i;
            double2 val = ident ? X2[o] : acc[m][v];
            if (mode == 1) {
                const double2 bb = B2[o];
                val = make_double2(bb.x - val.x, bb.y - val.y);
                if (NRM && v < 2) {
                    sq[v][m][0].x += bb.x * bb.x;
                    sq[v][m][0].y += bb.y * bb.y;
                    sq[v][m][1].x += val.x * val.x;
                    sq[v][m][1].y += val.y * val.y;
                }
            }
            Y2[o] = val;
        }
    }
    }   // live row
    if (NRM) {
        // pairs 2*part + v: reduce each v as its own "part" stream, interleaved into one row
        __shared__ double2 redp[8][2][2][2][32];
        const int warp = threadIdx.x >> 5;
#pragma unroll
        for (int v = 0; v < 2; ++v)
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int br = 0; br < 2; ++br) {
                    double2 t = make_double2(0.0, 0.0);
                    for (int rr = 0; rr < R; ++rr) {
                        t.x += __shfl_sync(0xffffffffu, sq[v][m][br].x, part + L * rr);
                        t.y += __shfl_sync(0xffffffffu, sq[v][m][br].y, part + L * rr);
                    }
                    if (lane < L) redp[warp][v][m][br][lane] = t;
                }
        __syncthreads();
        const int nw = blockDim.x >> 5;
        const int H2 = J >> 1;
        for (int e = threadIdx.x; e < 2 * 2 * H2; e += blockDim.x) {
            const int m = e / (2 * H2), br = (e / H2) & 1, pr = e % H2;   // member pair pr = 2*part + v
            const int pp = pr >> 1, v = pr & 1;
            double2 t = make_double2(0.0, 0.0);
            for (int w = 0; w < nw; ++w) {
                t.x += redp[w][v][m][br][pp].x;
                t.y += redp[w][v][m][br][pp].y;
            }
            double* o = nrm + (((int64_t)bid * 2 + m) * 2 + br) * J + 2 * pr;
            o[0] = t.x;
            o[1] = t.y;
        }
    }
}

template <int V2, bool NRM>
__global__ void __launch_bounds__(256) k_spmm_pres_v(const int32_t* __restrict__ bp, const int32_t* __restrict__ bc,
                                                     const double* __restrict__ bv, const uint8_t* __restrict__ cflag,
                                                     const double* __restrict__ X, const double* __restrict__ Bv,
                                                     double* __restrict__ Y, int npres, int64_t nvel, int64_t N, int J,
                                                     int L, int mode, double* __restrict__ nrm) {
    spmm_pres_body<V2, NRM>(bp, bc, bv, cflag, X, Bv, Y, npres, nvel, N, J, L, mode, nrm, blockIdx.x);
}

// velocity and pressure rows in one launch: blocks [0, nbv) take velocity rows, the rest pressure
// rows (the pressure blocks fill the velocity kernel's last wave; one launch instead of two)
template <int V2>
__global__ void __launch_bounds__(256) k_spmm_both_v(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                     const double* __restrict__ A, int nnz,
                                                     const int32_t* __restrict__ btp, const int32_t* __restrict__ btc,
                                                     const double* __restrict__ btv,
                                                     const int32_t* __restrict__ bp, const int32_t* __restrict__ bc,
                                                     const double* __restrict__ bv, const uint8_t* __restrict__ cflag,
                                                     const double* __restrict__ X, const double* __restrict__ Bv,
                                                     double* __restrict__ Y, int ns, int npres, int64_t N, int J,
                                                     int Lv, int Lp, int nbv, int mode) {
    if ((int)blockIdx.x < nbv)
        spmm_vel_body<V2, false>(rp, col, A, nnz, btp, btc, btv, cflag, X, Bv, Y, ns, N, J, Lv, mode, nullptr,
                                 blockIdx.x);
    else
        spmm_pres_body<V2, false>(bp, bc, bv, cflag, X, Bv, Y, npres, 2LL * ns, N, J, Lp, mode, nullptr,
                                  blockIdx.x - nbv);
}

// ---------------------------------------------------------------------------
// Row-pair variant (velocity rows 2p, 2p+1 together): the pair's column lists are
// merged (host, once per mesh) into one sorted union with each row's CSR slot or -1,
// so a neighbour segment both rows touch is gathered once for both (P2 meshes in
// nested-dissection order: 27 % fewer gathers, 31 % fewer for the B^T pairs).  Each
// row accumulates exactly its own entries in CSR order (absent entries are skipped,
// not multiplied by zero): results are bitwise identical to the one-row kernels.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void spmm_pair_body(const int32_t* __restrict__ pp, const int32_t* __restrict__ pc,
                                               const int2* __restrict__ ps, const double* __restrict__ A, int nnz,
                                               const int32_t* __restrict__ tp, const int32_t* __restrict__ tc,
                                               const int2* __restrict__ ts, const double* __restrict__ btv,
                                               const uint8_t* __restrict__ cflag, const double* __restrict__ X,
                                               const double* __restrict__ Bv, double* __restrict__ Y, int ns,
                                               int64_t N, int J, int L, int mode, int bid) {
    constexpr int V2 = 2;
    const int lane = threadIdx.x & 31;
    const int R = 32 / L;
    const int r = lane / L, part = lane - r * L;
    const int64_t gw = ((int64_t)bid * blockDim.x + threadIdx.x) >> 5;
    const int64_t pr = gw * R + r;
    const int64_t npair = ((int64_t)ns + 1) >> 1;
    if (r >= R || pr >= npair) return;
    const int H = J >> 1;
    const int64_t MS = N * H;
    const double2* X2 = reinterpret_cast<const double2*>(X);
    double2* Y2 = reinterpret_cast<double2*>(Y);
    const double2* B2 = reinterpret_cast<const double2*>(Bv);
    const int64_t nvel = 2LL * ns;
    double2 acc[2][2][V2];   // [row of the pair][system][v]
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int v = 0; v < V2; ++v) acc[h][m][v] = make_double2(0.0, 0.0);
    const int k0 = pp[pr], k1 = pp[pr + 1];
    for (int k = k0; k < k1; ++k) {
        const int64_t c0 = pc[k];
        const int2 sl = ps[k];
        const bool h0 = sl.x >= 0, h1 = sl.y >= 0;
        const double a00 = h0 ? A[sl.x] : 0.0, a01 = h0 ? A[nnz + sl.x] : 0.0;   // row 0: systems 0, 1
        const double a10 = h1 ? A[sl.y] : 0.0, a11 = h1 ? A[nnz + sl.y] : 0.0;   // row 1
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int i = part + L * v;
            if (i < J) {
                const double2 x0 = X2[c0 * J + i], x1 = X2[MS + c0 * J + i];
                if (h0) {
                    acc[0][0][v].x = fma(a00, x0.x, acc[0][0][v].x);
                    acc[0][0][v].y = fma(a00, x0.y, acc[0][0][v].y);
                    acc[0][1][v].x = fma(a01, x1.x, acc[0][1][v].x);
                    acc[0][1][v].y = fma(a01, x1.y, acc[0][1][v].y);
                }
                if (h1) {
                    acc[1][0][v].x = fma(a10, x0.x, acc[1][0][v].x);
                    acc[1][0][v].y = fma(a10, x0.y, acc[1][0][v].y);
                    acc[1][1][v].x = fma(a11, x1.x, acc[1][1][v].x);
                    acc[1][1][v].y = fma(a11, x1.y, acc[1][1][v].y);
                }
            }
        }
    }
    // pressure couplings of both rows (same B^T for both systems)
    const double2* P2 = X2 + nvel * H;
    const double2* bt2 = reinterpret_cast<const double2*>(btv);
    const int t0 = tp[pr], t1 = tp[pr + 1];
    for (int t = t0; t < t1; ++t) {
        const int64_t p0 = tc[t];
        const int2 sl = ts[t];
        const bool h0 = sl.x >= 0, h1 = sl.y >= 0;
        const double2 b0 = h0 ? bt2[sl.x] : make_double2(0.0, 0.0);
        const double2 b1 = h1 ? bt2[sl.y] : make_double2(0.0, 0.0);
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int i = part + L * v;
            if (i < J) {
                const bool ycomp = i >= H;
                const int64_t o = p0 * H + (ycomp ? i - H : i);
                const double2 x0 = P2[o], x1 = P2[MS + o];
                if (h0) {
                    const double f0 = ycomp ? b0.y : b0.x;
                    acc[0][0][v].x -= f0 * x0.x;
                    acc[0][0][v].y -= f0 * x0.y;
                    acc[0][1][v].x -= f0 * x1.x;
                    acc[0][1][v].y -= f0 * x1.y;
                }
                if (h1) {
                    const double f1 = ycomp ? b1.y : b1.x;
                    acc[1][0][v].x -= f1 * x0.x;
                    acc[1][0][v].y -= f1 * x0.y;
                    acc[1][1][v].x -= f1 * x1.x;
                    acc[1][1][v].y -= f1 * x1.y;
                }
            }
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int64_t node = 2 * pr + h;
        if (node >= ns) break;
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int i = part + L * v;
            if (i >= J) continue;
            const int64_t o = node * J + i;
            const bool ident = cflag[2 * node + (i >= H ? 1 : 0)] != 0;
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                double2 val = ident ? X2[m * MS + o] : acc[h][m][v];
                if (mode == 1) {
                    const double2 bb = B2[m * MS + o];
                    val = make_double2(bb.x - val.x, bb.y - val.y);
                }
                Y2[m * MS + o] = val;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Wide-member variants (J >= 64: one row per warp, lanes over member pairs).
// The row's CSR entries are loaded lane-parallel once (one coalesced load per
// stream instead of a dependent index load per nonzero) and broadcast with
// shuffles, so U nonzeros' gathers (U x 2 systems x V2 16-byte loads per
// lane) are in flight together.  Per-output summation order is the CSR order
// of the kernels above.
// ---------------------------------------------------------------------------
template <int V2, int U>
__global__ void __launch_bounds__(256) k_spmm_vel_w(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                    const double* __restrict__ A, int nnz,
                                                    const int32_t* __restrict__ btp, const int32_t* __restrict__ btc,
                                                    const double* __restrict__ btv, const uint8_t* __restrict__ cflag,
                                                    const double* __restrict__ X, const double* __restrict__ Bv,
                                                    double* __restrict__ Y, int ns, int64_t N, int J, int mode) {
    const int lane = threadIdx.x & 31;
    const int64_t node = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (node >= ns) return;
    const int H = J >> 1;
    const int64_t MS = N * H;
    const double2* X2 = reinterpret_cast<const double2*>(X);
    double2* Y2 = reinterpret_cast<double2*>(Y);
    const double2* B2 = reinterpret_cast<const double2*>(Bv);
    const int64_t nvel = 2LL * ns;
    const int k0 = rp[node], n = rp[node + 1] - k0;
    const int t0 = btp[node], np = btp[node + 1] - t0;
    int myc = (int)node, myp = 0;
    double mya0 = 0.0, mya1 = 0.0;
    double2 myb = make_double2(0.0, 0.0);
    if (lane < n) {
        myc = col[k0 + lane];
        mya0 = A[k0 + lane];
        mya1 = A[nnz + k0 + lane];
    }
    if (lane < np) {
        myp = btc[t0 + lane];
        myb = reinterpret_cast<const double2*>(btv)[t0 + lane];
    }
    double2 acc[2][V2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int v = 0; v < V2; ++v) acc[m][v] = make_double2(0.0, 0.0);
    const int nc = min(n, 32);
    for (int k = 0; k < nc; k += U) {
        int64_t c[U];
        double a0[U], a1[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int src = (k + u) & 31;
            c[u] = __shfl_sync(0xffffffffu, myc, src);
            a0[u] = __shfl_sync(0xffffffffu, mya0, src);
            a1[u] = __shfl_sync(0xffffffffu, mya1, src);
            ok[u] = k + u < nc;
            if (!ok[u]) c[u] = node;   // in-bounds dummy gather, not accumulated
        }
        double2 x0[U][V2], x1[U][V2];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int v = 0; v < V2; ++v) {
                const int64_t o = c[u] * J + lane + 32 * v;
                x0[u][v] = X2[o];
                x1[u][v] = X2[MS + o];
            }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
#pragma unroll
            for (int v = 0; v < V2; ++v) {
                acc[0][v].x = fma(a0[u], x0[u][v].x, acc[0][v].x);
                acc[0][v].y = fma(a0[u], x0[u][v].y, acc[0][v].y);
                acc[1][v].x = fma(a1[u], x1[u][v].x, acc[1][v].x);
                acc[1][v].y = fma(a1[u], x1[u][v].y, acc[1][v].y);
            }
        }
    }
    for (int k = 32; k < n; ++k) {   // rows longer than a warp (not produced by P2 meshes)
        const int64_t c0 = col[k0 + k];
        const double a00 = A[k0 + k], a10 = A[nnz + k0 + k];
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int64_t o = c0 * J + lane + 32 * v;
            const double2 x00 = X2[o], x10 = X2[MS + o];
            acc[0][v].x = fma(a00, x00.x, acc[0][v].x);
            acc[0][v].y = fma(a00, x00.y, acc[0][v].y);
            acc[1][v].x = fma(a10, x10.x, acc[1][v].x);
            acc[1][v].y = fma(a10, x10.y, acc[1][v].y);
        }
    }
    // pressure couplings: member pair i = lane + 32 v of component (i >= H) reads pressure pair i mod H
    const double2* P2 = X2 + nvel * H;
    const int npc = min(np, 32);
    for (int t = 0; t < npc; ++t) {
        const int64_t p0 = __shfl_sync(0xffffffffu, myp, t);
        const double bx = __shfl_sync(0xffffffffu, myb.x, t), by = __shfl_sync(0xffffffffu, myb.y, t);
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int i = lane + 32 * v;
            const bool ycomp = i >= H;
            const int64_t o = p0 * H + (ycomp ? i - H : i);
            const double2 x0 = P2[o], x1 = P2[MS + o];
            const double f0 = ycomp ? by : bx;
            acc[0][v].x -= f0 * x0.x;
            acc[0][v].y -= f0 * x0.y;
            acc[1][v].x -= f0 * x1.x;
            acc[1][v].y -= f0 * x1.y;
        }
    }
    for (int t = 32; t < np; ++t) {
        const double2 b0 = reinterpret_cast<const double2*>(btv)[t0 + t];
        const int64_t p0 = btc[t0 + t];
#pragma unroll
        for (int v = 0; v < V2; ++v) {
            const int i = lane + 32 * v;
            const bool ycomp = i >= H;
            const int64_t o = p0 * H + (ycomp ? i - H : i);
            const double2 x0 = P2[o], x1 = P2[MS + o];
            const double f0 = ycomp ? b0.y : b0.x;
            acc[0][v].x -= f0 * x0.x;
            acc[0][v].y -= f0 * x0.y;
            acc[1][v].x -= f0 * x1.x;
            acc[1][v].y -= f0 * x1.y;
        }
    }
#pragma unroll
    for (int v = 0; v < V2; ++v) {
        const int i = lane + 32 * v;
        const int64_t o = node * J + i;
        const bool ident = cflag[2 * node + (i >= H ? 1 : 0)] != 0;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            double2 val = ident ? X2[m * MS + o] : acc[m][v];
            if (mode == 1) {
                const double2 bb = B2[m * MS + o];
                val = make_double2(bb.x - val.x, bb.y - val.y);
            }
            Y2[m * MS + o] = val;
        }
    }
}

// pressure rows, J >= 64: one row per warp, lane pairs i = lane + 32 v of each component
template <int V2, int U>
__global__ void __launch_bounds__(256) k_spmm_pres_w(const int32_t* __restrict__ bp, const int32_t* __restrict__ bc,
                                                     const double* __restrict__ bv, const uint8_t* __restrict__ cflag,
                                                     const double* __restrict__ X, const double* __restrict__ Bv,
                                                     double* __restrict__ Y, int npres, int64_t nvel, int64_t N,
                                                     int J, int mode) {
    const int lane = threadIdx.x & 31;
    const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (p >= npres) return;
    const int H = J >> 1;
    const int64_t MS = N * H;
    const double2* X2 = reinterpret_cast<const double2*>(X);
    double2* Y2 = reinterpret_cast<double2*>(Y);
    const double2* B2 = reinterpret_cast<const double2*>(Bv);
    const int t0 = bp[p], n = bp[p + 1] - t0;
    int myc = 0;
    double2 myb = make_double2(0.0, 0.0);
    if (lane < n) {
        myc = bc[t0 + lane];
        myb = reinterpret_cast<const double2*>(bv)[t0 + lane];
    }
    double2 acc[2][V2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int v = 0; v < V2; ++v) acc[m][v] = make_double2(0.0, 0.0);
    const int nc = min(n, 32);
    for (int k = 0; k < nc; k += U) {
        int64_t c[U];
        double bx[U], by[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int src = (k + u) & 31;
            c[u] = __shfl_sync(0xffffffffu, myc, src);
            bx[u] = __shfl_sync(0xffffffffu, myb.x, src);
            by[u] = __shfl_sync(0xffffffffu, myb.y, src);
            ok[u] = k + u < nc;
            if (!ok[u]) c[u] = 0;
        }
        double2 uu[U][2][V2], ww[U][2][V2];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int v = 0; v < V2; ++v) {
                    const int i = lane + 32 * v;
                    const int64_t o = m * MS + c[u] * J + (i < H ? i : 0);
                    uu[u][m][v] = X2[o];
                    ww[u][m][v] = X2[o + H];
                }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int v = 0; v < V2; ++v) {
                    acc[m][v].x += bx[u] * uu[u][m][v].x + by[u] * ww[u][m][v].x;
                    acc[m][v].y += bx[u] * uu[u][m][v].y + by[u] * ww[u][m][v].y;
                }
        }
    }
    for (int k = 32; k < n; ++k) {
        const double2 b0 = reinterpret_cast<const double2*>(bv)[t0 + k];
        const int64_t n0 = bc[t0 + k];
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int v = 0; v < V2; ++v) {
                const int i = lane + 32 * v;
                if (i < H) {
                    const double2 u0 = X2[m * MS + n0 * J + i], w0 = X2[m * MS + n0 * J + H + i];
                    acc[m][v].x += b0.x * u0.x + b0.y * w0.x;
                    acc[m][v].y += b0.x * u0.y + b0.y * w0.y;
                }
            }
    }
    const int64_t row = nvel + p;
    const bool ident = cflag[row] != 0;
#pragma unroll
    for (int v = 0; v < V2; ++v) {
        const int i = lane + 32 * v;
        if (i >= H) continue;
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            const int64_t o = m * MS + row * H + i;
            double2 val = ident ? X2[o] : acc[m][v];
            if (mode == 1) {
                const double2 bb = B2[o];
                val = make_double2(bb.x - val.x, bb.y - val.y);
            }
            Y2[o] = val;
        }
    }
}

// ENS_SPMM_WIDE (read once per context): 1 (default) on, 0 off (the direct kernels)
static int spmm_wide_variant(ens_ctx* c) {
    if (c->spmm_wide < 0) {
        const char* e = std::getenv("ENS_SPMM_WIDE");
        c->spmm_wide = e ? std::atoi(e) : 1;
    }
    return c->spmm_wide;
}

// J in {64, 128, 192, 256} (multiples of 64): one row per warp; returns false when not applicable
static bool launch_spmm_wide(ens_ctx* c, cudaStream_t s, const double* as_vals, const double* x, const double* b,
                             double* y, int mode) {
    const int J = c->J;
    const int wv = spmm_wide_variant(c);
    if (wv == 0 || J % 64 != 0 || J > 256) return false;
    const int V2 = J / 32;   // double2 per lane per system (velocity rows: 2J doubles = J double2)
    const dim3 gv((unsigned)(((int64_t)c->m.ns * 32 + 255) / 256));
    const dim3 gp((unsigned)(((int64_t)c->m.n_pres * 32 + 255) / 256));
#define WV(V, UU)                                                                                                  \
    k_spmm_vel_w<V, UU><<<gv, 256, 0, s>>>(c->m.s_rowptr, c->m.s_col, as_vals, c->m.nnz_s, c->m.bt_rowptr,          \
                                           c->m.bt_col, c->m.bt_val, c->m.cflag, x, b ? b : x, y, c->m.ns,          \
                                           c->n_total, J, mode)
#define WP(V, UU)                                                                                                  \
    k_spmm_pres_w<V, UU><<<gp, 256, 0, s>>>(c->m.b_rowptr, c->m.b_col, c->m.b_val, c->m.cflag, x, b ? b : x, y,     \
                                            c->m.n_pres, c->n_vel, c->n_total, J, mode)
    // measured at C2 (warm, both kernels): J = 64 direct 228 us -> 203 us (U = 2; U = 4 275 us),
    // J = 128 direct 451 us -> 416 us (velocity U = 2, pressure U = 4)
    if (V2 == 2) WV(2, 2);
    else if (V2 == 4) WV(4, 2);
    else if (V2 == 6) WV(6, 1);
    else WV(8, 1);
    ENS_CKL();
    // pressure rows: H = J/2 pairs per component -> V2p = ceil(H / 32) pairs per lane
    const int V2p = (J / 2 + 31) / 32;
    if (V2p == 1) WP(1, 2);
    else if (V2p == 2) WP(2, 4);
    else if (V2p == 3) WP(3, 2);
    else WP(4, 2);
#undef WV
#undef WP
    ENS_CKL();
    return true;
}

static bool spmm_merge() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("ENS_SPMM_MERGE");
        v = e ? std::atoi(e) : 1;
    }
    return v != 0;
}

static int launch_spmm_vec(ens_ctx* c, cudaStream_t s, const double* as_vals, const double* x, const double* b,
                           double* y, int mode, double* nrm, int* nblk) {
    const int J = c->J;
    int blocks_total = 0;
    if (!nrm && J <= 64 && J / 2 <= 64 && spmm_merge()) {
        const int Lv = (J + 1) / 2, Rv = 32 / Lv;
        const int H = J / 2, Lp = (H + 1) / 2, Rp = 32 / Lp;
        const int nbv = (int)(((((int64_t)c->m.ns + Rv - 1) / Rv) * 32 + 255) / 256);
        const int nbp = (int)(((((int64_t)c->m.n_pres + Rp - 1) / Rp) * 32 + 255) / 256);
        k_spmm_both_v<2><<<nbv + nbp, 256, 0, s>>>(c->m.s_rowptr, c->m.s_col, as_vals, c->m.nnz_s, c->m.bt_rowptr,
                                                   c->m.bt_col, c->m.bt_val, c->m.b_rowptr, c->m.b_col, c->m.b_val,
                                                   c->m.cflag, x, b ? b : x, y, c->m.ns, c->m.n_pres, c->n_total, J,
                                                   Lv, Lp, nbv, mode);
        ENS_CKL();
        if (nblk) *nblk = nbv + nbp;
        return ENS_OK;
    }
    {
        const int V2 = J <= 64 ? 2 : (J <= 128 ? 4 : 8);
        const int L = (J + V2 - 1) / V2, R = 32 / L;
        const int64_t warps = ((int64_t)c->m.ns + R - 1) / R;
        dim3 grid((unsigned)((warps * 32 + 255) / 256), 1);
#define SPV(V, NR)                                                                                                 \
    k_spmm_vel_v<V, NR><<<grid, 256, 0, s>>>(c->m.s_rowptr, c->m.s_col, as_vals, c->m.nnz_s, c->m.bt_rowptr,        \
                                             c->m.bt_col, c->m.bt_val, c->m.cflag, x, b ? b : x, y, c->m.ns,        \
                                             c->n_total, J, L, mode, nrm)
        if (nrm) SPV(2, true);
        else if (V2 == 2) SPV(2, false);
        else if (V2 == 4) SPV(4, false);
        else SPV(8, false);
#undef SPV
        ENS_CKL();
        blocks_total += (int)grid.x;
    }
    {
        const int H = J / 2;
        const int V2 = H <= 64 ? 2 : (H <= 128 ? 4 : 8);
        const int L = (H + V2 - 1) / V2, R = 32 / L;
        const int64_t warps = ((int64_t)c->m.n_pres + R - 1) / R;
        dim3 grid((unsigned)((warps * 32 + 255) / 256), 1);
        double* nrm_p = nrm ? nrm + (int64_t)blocks_total * 4 * J : nullptr;
#define SPP(V, NR)                                                                                                 \
    k_spmm_pres_v<V, NR><<<grid, 256, 0, s>>>(c->m.b_rowptr, c->m.b_col, c->m.b_val, c->m.cflag, x, b ? b : x, y,   \
                                              c->m.n_pres, c->n_vel, c->n_total, J, L, mode, nrm_p)
        if (nrm) SPP(2, true);
        else if (V2 == 2) SPP(2, false);
        else if (V2 == 4) SPP(4, false);
        else SPP(8, false);
#undef SPP
        ENS_CKL();
        blocks_total += (int)grid.x;
    }
    if (nblk) *nblk = blocks_total;
    return ENS_OK;
}

// out[k][mat][j] (k = 0: ||b||^2, 1: ||b - K x||^2) from the per-block partials, fixed order
__global__ void k_nrm_fin(const double* __restrict__ part, int nblk, int J, double* __restrict__ bn2,
                          double* __restrict__ rn2) {
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= 4 * J) return;
    const int br = t / (2 * J), mj = t % (2 * J), mat = mj / J, j = mj % J;
    double acc = 0.0;
    for (int b = lane; b < nblk; b += 32) acc += part[(((int64_t)b * 2 + mat) * 2 + br) * J + j];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) (br ? rn2 : bn2)[mj] = acc;
}

bool spmm_resnorm_ok(const ens_ctx* c) {
    // opt-in (ENS_FUSED_NORM=1): measured slower at C2 (block reductions + finalise
    // cost more than the two 24 MB column-dot passes they replace)
    const char* e = std::getenv("ENS_FUSED_NORM");
    if (!(e && e[0] == '1')) return false;
    return (c->J & 1) == 0 && c->J >= 2 && c->J <= 64;
}

// y = b - K x plus the per-column squares of b and y (bn2, rn2: [mat][J])
int launch_spmm_resnorm(ens_ctx* c, cudaStream_t s, const double* as_vals, const double* x, const double* b,
                        double* y, double* bn2, double* rn2) {
    if (!c->nrm_part) {
        const int J = c->J;
        const int64_t bv = ((((int64_t)c->m.ns + (32 / (J / 2)) - 1) / (32 / (J / 2))) * 32 + 255) / 256;
        const int Lp = (J / 2 + 1) / 2;
        const int64_t bp = ((((int64_t)c->m.n_pres + (32 / Lp) - 1) / (32 / Lp)) * 32 + 255) / 256;
        const size_t bytes = sizeof(double) * 4 * (size_t)J * (size_t)(bv + bp);
        ENS_CK(cudaMalloc(&c->nrm_part, bytes));
        c->ws_bytes += bytes;
    }
    int nblk = 0;
    const int rc = launch_spmm_vec(c, s, as_vals, x, b, y, 1, c->nrm_part, &nblk);
    if (rc != ENS_OK) return rc;
    k_nrm_fin<<<(4 * c->J * 32 + 255) / 256, 256, 0, s>>>(c->nrm_part, nblk, c->J, bn2, rn2);
    ENS_CKL();
    return ENS_OK;
}

int launch_spmm(ens_ctx* c, cudaStream_t s, const double* as_vals, const double* x, const double* b, double* y,
                int mode) {
    const int J = c->J, W2 = 2 * J;
    if ((J & 1) == 0 && J <= 512 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(y) & 15) == 0 && (!b || (reinterpret_cast<uintptr_t>(b) & 15) == 0))
    {
        if (launch_spmm_wide(c, s, as_vals, x, b, y, mode)) return ENS_OK;
        return launch_spmm_vec(c, s, as_vals, x, b, y, mode, nullptr, nullptr);
    }
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
