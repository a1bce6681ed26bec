#include <algorithm>
// Column-batched right-preconditioned FGMRES over both saddle systems.
//
// Every ensemble member is an independent column (no block Krylov mixing, so
// identical members stay bitwise identical, tests/test_stepper.py:213-229 of
// the reference); all columns share each SpMM and each preconditioner sweep.
// Per-column Krylov scalars (Hessenberg, Givens, residual estimate) live on the
// device; the host only reads one counter per iteration to stop early.
// Replaces Factorization.solve_block + relative_residual (linalg.py:62-76, 111-118).
#include <cmath>
#include <cstdlib>
#include <string>

#include "ens_internal.cuh"

struct GmresCol {
    double H[(ENS_MAX_RESTART + 1) * ENS_MAX_RESTART];
    double cs[ENS_MAX_RESTART], sn[ENS_MAX_RESTART], g[ENS_MAX_RESTART + 1];
    double bnorm, tol;
    int active, kused;
};

size_t gmres_col_bytes() { return sizeof(GmresCol); }

// Krylov blocks for `restart` vectors; when device memory is short (large
// meshes x many members) the cycle is shortened instead of failing -- the
// lagged-preconditioner FGMRES needs 1-3 vectors per cycle and restarts keep
// the same true-residual stopping test.  Returns the usable cycle length in
// c->kry_restart.
int gmres_alloc(ens_ctx* c, int restart) {
    if (restart < 1 || restart > ENS_MAX_RESTART) {
        ens_set_error("restart out of range", __FILE__, __LINE__);
        return ENS_EINVAL;
    }
    if (c->kry && c->kry_restart >= restart) return ENS_OK;
    if (c->kry && c->kry_short) return ENS_OK;   // already shortened for memory: keep it
    if (c->kry) {
        cudaFree(c->kry);
        c->ws_bytes -= c->kry_bytes;
        c->kry = nullptr;
    }
    const size_t blk = 2ull * (size_t)c->n_total * c->J;
    // leave room for the solve's lazily allocated workspace (split-K partials, graphs)
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = total_b = 0;
    const size_t reserve = std::max<size_t>(size_t(4) << 30, total_b / 20);
    for (int r = restart; r >= 2; --r) {
        const size_t nblk = 2 * (size_t)r + 3;   // V[0..R], Z[0..R-1], R, W
        if (r > 2 && free_b && sizeof(double) * blk * nblk + reserve > free_b) continue;
        if (cudaMalloc(&c->kry, sizeof(double) * blk * nblk) == cudaSuccess) {
            c->kry_bytes = sizeof(double) * blk * nblk;
            c->ws_bytes += c->kry_bytes;
            c->kry_restart = r;
            c->kry_short = r < restart ? 1 : 0;
            return ENS_OK;
        }
        cudaGetLastError();   // clear the allocation failure
        c->kry = nullptr;
    }
    ens_set_error("out of device memory for Krylov blocks", __FILE__, __LINE__);
    return ENS_ENOMEM;
}

// scalar buffers inside red_out:  [bn2 | rn2 | h1 | h2 | hn2 | scale | y]
struct KBuf {
    double *bn2, *rn2, *h1, *h2, *hn2, *scale, *y;
};

static KBuf kbuf(ens_ctx* c) {
    const size_t J2 = 2 * (size_t)c->J;
    const size_t L = ENS_MAX_RESTART + 1;
    KBuf b;
    b.bn2 = c->red_out;
    b.rn2 = b.bn2 + J2;
    b.h1 = b.rn2 + J2;
    b.h2 = b.h1 + J2 * L;
    b.hn2 = b.h2 + J2 * L;
    b.scale = b.hn2 + J2;
    b.y = b.scale + J2;
    return b;
}

__global__ void k_gm_init(GmresCol* cols, const double* bn2, const double* rn2, double rtol, double* scale,
                          int32_t* count, int n) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    GmresCol& g = cols[c];
    const double bn = sqrt(bn2[c]);
    const double beta = sqrt(rn2[c]);
    g.bnorm = bn;
    g.tol = rtol * fmax(bn, 2.2250738585072014e-308);
    g.active = beta > g.tol ? 1 : 0;
    g.kused = 0;
    for (int i = 0; i <= ENS_MAX_RESTART; ++i) g.g[i] = 0.0;
    g.g[0] = beta;
    scale[c] = g.active ? 1.0 / beta : 0.0;
    if (g.active) atomicAdd(count, 1);
    if (c == 0) count[2] += 1;   // sequence number of the round trip (ens_solve_finish polls it in pinned memory)
}

// Host side of a begun solve's round trip: spin on the sequence word the D2H copy of the counters
// carries (pinned memory); the stream is only queried now and then to notice a failed launch.
static int wait_round_trip(ens_ctx* c, cudaStream_t s) {
    volatile int32_t* hc = c->h_count;
    for (unsigned long spins = 1;; ++spins) {
        if (hc[2] != c->gm_seq) break;
        if ((spins & 0xfff) == 0) {
            const cudaError_t q = cudaStreamQuery(s);
            if (q == cudaSuccess) {
                if (hc[2] != c->gm_seq) break;
                ens_set_error("solve finish: no begun solve on this stream", __FILE__, __LINE__);
                return ENS_EINVAL;
            }
            if (q != cudaErrorNotReady) ENS_CK(q);
        }
    }
    __sync_synchronize();
    c->gm_seq = hc[2];
    return ENS_OK;
}

// dst = src * scale[col]
__global__ void k_scale_cols(double* __restrict__ dst, const double* __restrict__ src,
                             const double* __restrict__ scale, int64_t N, int J) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = N * J;
    if (t >= 2 * per) return;
    const int mat = (int)(t / per);
    const int j = (int)((t - mat * per) % J);
    dst[t] = src[t] * scale[mat * J + j];
}

// even J: 16-byte lanes over (mat, member pair); 32-bit index math, grid-stride
__global__ void __launch_bounds__(256) k_scale_cols2(double* __restrict__ dst, const double* __restrict__ src,
                                                     const double* __restrict__ scale, int per2, int H) {
    const int mat = blockIdx.y;
    const double2* s2 = reinterpret_cast<const double2*>(src) + (int64_t)mat * per2;
    double2* d2 = reinterpret_cast<double2*>(dst) + (int64_t)mat * per2;
    const double2* sc = reinterpret_cast<const double2*>(scale + (int64_t)mat * 2 * H);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < per2; t += gridDim.x * blockDim.x) {
        const double2 a = s2[t], f = sc[t % H];
        d2[t] = make_double2(a.x * f.x, a.y * f.y);
    }
}

__global__ void __launch_bounds__(256) k_axpy_multi2(double* __restrict__ W, const double* __restrict__ V,
                                                     int64_t lstride, int L, const double* __restrict__ h, double sign,
                                                     int per2, int H) {
    const int mat = blockIdx.y;
    double2* w2 = reinterpret_cast<double2*>(W) + (int64_t)mat * per2;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < per2; t += gridDim.x * blockDim.x) {
        const int jp = t % H;
        double2 acc = make_double2(0.0, 0.0);
        for (int l = 0; l < L; ++l) {
            const double2 v = reinterpret_cast<const double2*>(V + (int64_t)l * lstride)[(int64_t)mat * per2 + t];
            const double2 y = reinterpret_cast<const double2*>(h + ((int64_t)mat * L + l) * 2 * H)[jp];
            acc.x += v.x * y.x;
            acc.y += v.y * y.y;
        }
        double2 w = w2[t];
        w.x += sign * acc.x;
        w.y += sign * acc.y;
        w2[t] = w;
    }
}

// x += z over both systems (the Richardson correction of the first cycle)
__global__ void __launch_bounds__(256) k_add2(double2* __restrict__ x, const double2* __restrict__ z, int64_t n2) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n2; t += (int64_t)gridDim.x * blockDim.x) {
        const double2 a = x[t], b = z[t];
        x[t] = make_double2(a.x + b.x, a.y + b.y);
    }
}
__global__ void k_add1(double* __restrict__ x, const double* __restrict__ z, int64_t n) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) x[t] += z[t];
}

static unsigned vec_blocks(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16); }

static bool vec_ok(int J, int64_t N, const void* a, const void* b) {
    return (J & 1) == 0 && N * J / 2 < (1LL << 31) && (reinterpret_cast<uintptr_t>(a) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(b) & 15) == 0;
}

static void scale_cols(cudaStream_t s, double* dst, const double* src, const double* scale, int64_t N, int J) {
    if (vec_ok(J, N, dst, src)) {
        const int per2 = (int)(N * J / 2);
        k_scale_cols2<<<dim3(vec_blocks(per2), 2), 256, 0, s>>>(dst, src, scale, per2, J / 2);
    } else {
        k_scale_cols<<<(unsigned)((2 * N * J + 255) / 256), 256, 0, s>>>(dst, src, scale, N, J);
    }
}

// W -= sum_l V_l h[mat][l][j]  (sign = -1) or X += sum_l Z_l y (sign = +1)
__global__ void k_axpy_multi(double* __restrict__ W, const double* __restrict__ V, int64_t lstride, int L,
                             const double* __restrict__ h, double sign, int64_t N, int J) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = N * J;
    if (t >= 2 * per) return;
    const int mat = (int)(t / per);
    const int j = (int)((t - mat * per) % J);
    double acc = 0.0;
    for (int l = 0; l < L; ++l) acc += V[(int64_t)l * lstride + t] * h[((int64_t)mat * L + l) * J + j];
    W[t] += sign * acc;
}

// store Hessenberg column i (h1 + h2), apply Givens, update residual estimate
__global__ void k_gm_givens(GmresCol* cols, const double* h1, const double* h2, const double* hn2, int i,
                            double* scale, int32_t* count, int n, int J) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    GmresCol& g = cols[c];
    const int R = ENS_MAX_RESTART;
    const int mat = c / J, j = c % J;
    const int L = i + 1;
    if (!g.active) {
        scale[c] = 0.0;
        return;
    }
    double col[ENS_MAX_RESTART + 1];
    for (int l = 0; l <= i; ++l) {
        const int64_t idx = ((int64_t)mat * L + l) * J + j;
        col[l] = h2 ? h1[idx] + h2[idx] : h1[idx];
    }
    const double hn = sqrt(hn2[c]);
    col[i + 1] = hn;
    for (int l = 0; l < i; ++l) {   // previous rotations
        const double t0 = g.cs[l] * col[l] + g.sn[l] * col[l + 1];
        col[l + 1] = -g.sn[l] * col[l] + g.cs[l] * col[l + 1];
        col[l] = t0;
    }
    const double a = col[i], b = col[i + 1];
    const double r = hypot(a, b);
    double cs = 1.0, sn = 0.0;
    if (r > 0.0) {
        cs = a / r;
        sn = b / r;
    }
    g.cs[i] = cs;
    g.sn[i] = sn;
    col[i] = r;
    col[i + 1] = 0.0;
    for (int l = 0; l <= i; ++l) g.H[l * R + i] = col[l];
    g.g[i + 1] = -sn * g.g[i];
    g.g[i] = cs * g.g[i];
    g.kused = i + 1;
    const double res = fabs(g.g[i + 1]);
    const bool breakdown = !(hn > 1e-300 * fmax(g.bnorm, 1e-300)) || r == 0.0;
    if (res <= g.tol || breakdown) {
        g.active = 0;
        scale[c] = 0.0;
    } else {
        scale[c] = 1.0 / hn;
        atomicAdd(count, 1);
    }
}

// y = H^-1 g (per column), layout y[mat][l][j] with L = Lmax rows
__global__ void k_gm_solve_y(GmresCol* cols, double* y, int Lmax, int n, int J) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    GmresCol& g = cols[c];
    const int R = ENS_MAX_RESTART;
    const int mat = c / J, j = c % J;
    double yy[ENS_MAX_RESTART];
    const int k = g.kused;
    for (int l = k - 1; l >= 0; --l) {
        double s = g.g[l];
        for (int t = l + 1; t < k; ++t) s -= g.H[l * R + t] * yy[t];
        yy[l] = g.H[l * R + l] != 0.0 ? s / g.H[l * R + l] : 0.0;
    }
    for (int l = 0; l < Lmax; ++l) y[((int64_t)mat * Lmax + l) * J + j] = l < k ? yy[l] : 0.0;
}

static int read_count(ens_ctx* c, cudaStream_t s, int* out) {
    ENS_CK(cudaMemcpyAsync(c->h_count, c->d_count, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    ENS_CK(cudaStreamSynchronize(s));
    *out = c->h_count[0];
    return ENS_OK;
}

#define RET(x)                        \
    do {                              \
        int rc_ = (x);                \
        if (rc_ != ENS_OK) return rc_; \
    } while (0)

// phase 0: the whole solve.  phase 1 (BEGIN, stream-capturable, needs *iters = predict > 0):
// the blind first cycle and the next cycle's true residual, whose active-column
// count and norms are copied to pinned host memory -- no host synchronisation.
// phase 2 (FINISH): synchronise, then continue exactly where phase 0 would.
int gmres_solve(ens_ctx* c, cudaStream_t s, const double* as_vals, const double* rhs, double* x, double rtol,
                int restart, int max_restarts, int32_t* iters, double* relres, int phase) {
    RET(gmres_alloc(c, restart));
    restart = std::min(restart, c->kry_restart);
    const int J = c->J;
    const int n = 2 * J;
    const int64_t N = c->n_total;
    const int64_t blk = 2LL * N * J;
    double* V = c->kry;                          // restart+1 blocks
    double* Z = V + blk * (restart + 1);         // restart blocks
    double* Rb = Z + blk * restart;
    double* Wb = Rb + blk;
    KBuf kb = kbuf(c);
    const unsigned eb = (unsigned)((blk + 255) / 256);
    const unsigned cb = (unsigned)((n + 127) / 128);
    const bool fused = spmm_resnorm_ok(c);   // residual SpMM also yields ||b||^2 and ||r||^2
    // predicted iteration count: the first cycle runs that many iterations without
    // host round trips; the true residual of the restart then decides (as always)
    const int predict = phase == 2 ? c->gm_predict : std::max(0, std::min(*iters, restart));
    if (phase == 1 && predict < 1) {
        ens_set_error("solve begin needs a predicted iteration count >= 1", __FILE__, __LINE__);
        return ENS_EINVAL;
    }
    // (a begin captured into a graph runs without this host code: its host-side
    // results -- total_it, predict -- are set at capture and are replay-invariant)
    bool resume = phase == 2;
    int total_it = resume ? c->gm_total_it : 0;
    if (!resume) {
        // identity rows of the iterate carry the data exactly (stepper.py:214-215, 250-251)
        RET(launch_copy_cons(c, s, rhs, x));
        if (!fused) RET(launch_coldot(c, s, rhs, 0, 1, rhs, N, kb.bn2));
    }
    // first cycle as one Richardson step x += P^-1 (b - K x) when a single iteration is
    // predicted (default; ENS_KRYLOV_FIRST=fgmres keeps a one-vector FGMRES cycle): the
    // true residual then decides exactly as after an FGMRES cycle, and FGMRES continues
    // from that iterate if needed.  Saves the cycle's K z product and its Gram-Schmidt /
    // Givens / scaling passes (C2 1.72 -> 1.61 ms/step, C4 19.7 -> 18.6, C3 45.5 -> 43.8).
    if (c->krylov_first < 0) {
        const char* e = std::getenv("ENS_KRYLOV_FIRST");
        c->krylov_first = (e && std::string(e) == "fgmres") ? 0 : 1;
    }
    const bool rich = c->krylov_first == 1 && predict == 1;
    for (int cyc = resume ? 1 : 0; cyc <= max_restarts; ++cyc) {
        const bool blind = !resume && cyc == 0 && predict > 0;
        if (blind && rich) {
            RET(launch_spmm(c, s, as_vals, x, rhs, Rb, 1));
            RET(mf_solve(c, s, Rb, Z));
            if (vec_ok(J, N, x, Z)) {
                k_add2<<<vec_blocks(blk / 2), 256, 0, s>>>(reinterpret_cast<double2*>(x),
                                                          reinterpret_cast<const double2*>(Z), blk / 2);
            } else {
                k_add1<<<eb, 256, 0, s>>>(x, Z, blk);
            }
            ENS_CKL();
            ++total_it;
            continue;
        }
        int active = 1;
        if (resume) {
            // the begin phase left the norms and the count on their way to pinned memory: wait for the
            // count's sequence word, not for the stream -- the caller may already have enqueued the
            // next step's pre-solve work behind this solve
            RET(wait_round_trip(c, s));
            active = *c->h_count;
            resume = false;
        } else {
            if (fused) {
                RET(launch_spmm_resnorm(c, s, as_vals, x, rhs, Rb, kb.bn2, kb.rn2));
            } else {
                RET(launch_spmm(c, s, as_vals, x, rhs, Rb, 1));
                RET(launch_coldot(c, s, Rb, 0, 1, Rb, N, kb.rn2));
            }
            ENS_CK(cudaMemsetAsync(c->d_count, 0, sizeof(int32_t), s));
            k_gm_init<<<cb, 128, 0, s>>>(c->cols, kb.bn2, kb.rn2, rtol, kb.scale, c->d_count, n);
            ENS_CKL();
            if (!blind) {
                // one round trip: active-column count and the residual norms
                // (the norms first: the count's sequence word tells the host that both have landed)
                ENS_CK(cudaMemcpyAsync(c->h_small, kb.bn2, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, s));
                ENS_CK(cudaMemcpyAsync(c->h_count, c->d_count, 3 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
                if (phase == 1) {
                    c->gm_total_it = total_it;
                    c->gm_predict = predict;
                    return ENS_OK;
                }
                ENS_CK(cudaStreamSynchronize(s));
                c->gm_seq = c->h_count[2];
                active = *c->h_count;
            }
        }
        if (!blind && (active == 0 || cyc == max_restarts)) {
            // true relative residual per matrix (linalg.py:111-118)
            for (int mat = 0; mat < 2; ++mat) {
                double worst = 0.0;
                for (int j = 0; j < J; ++j) {
                    const double bn = std::sqrt(c->h_small[mat * J + j]);
                    const double rn = std::sqrt(c->h_small[n + mat * J + j]);
                    worst = std::fmax(worst, rn / std::fmax(bn, 2.2250738585072014e-308));
                }
                relres[mat] = worst;
            }
            *iters = total_it;
            return active == 0 ? ENS_OK : ENS_ENOCONV;
        }
        scale_cols(s, V, Rb, kb.scale, N, J);
        ENS_CKL();
        int used = 0;
        for (int i = 0; i < restart; ++i) {
            double* Vi = V + blk * i;
            double* Zi = Z + blk * i;
            RET(mf_solve(c, s, Vi, Zi));
            RET(launch_spmm(c, s, as_vals, Zi, nullptr, Wb, 0));
            // classical Gram-Schmidt against V[0..i] (one pass: with the LU
            // preconditioner FGMRES needs 1-3 vectors, and every restart re-checks
            // the true residual); the update is fused with the norm of the result
            RET(launch_coldot(c, s, V, blk, i + 1, Wb, N, kb.h1));
            RET(launch_axpy_norm(c, s, Wb, V, blk, i + 1, kb.h1, N, kb.hn2));
            ENS_CK(cudaMemsetAsync(c->d_count, 0, sizeof(int32_t), s));
            k_gm_givens<<<cb, 128, 0, s>>>(c->cols, kb.h1, nullptr, kb.hn2, i, kb.scale, c->d_count, n, J);
            ENS_CKL();
            scale_cols(s, V + blk * (i + 1), Wb, kb.scale, N, J);
            ENS_CKL();
            used = i + 1;
            ++total_it;
            if (blind) {
                if (used == predict) break;
                continue;
            }
            RET(read_count(c, s, &active));
            if (active == 0) break;
        }
        k_gm_solve_y<<<cb, 128, 0, s>>>(c->cols, kb.y, used, n, J);
        ENS_CKL();
        if (vec_ok(J, N, x, Z) && (blk & 1) == 0) {
            const int per2 = (int)(N * J / 2);
            k_axpy_multi2<<<dim3(vec_blocks(per2), 2), 256, 0, s>>>(x, Z, blk, used, kb.y, 1.0, per2, J / 2);
        } else {
            k_axpy_multi<<<eb, 256, 0, s>>>(x, Z, blk, used, kb.y, 1.0, N, J);
        }
        ENS_CKL();
    }
    return ENS_ENOCONV;
}
