// Tile-staged saddle SpMM (both sub-step systems), fp64, sm_100a.
//
// Same operator and per-output summation order as the direct gather kernels in
// ens_spmm.cu (the reference's assembled saddle matrix, stepper.py:208-215,
// applied to every member column as in linalg.py:111-118), restructured so the
// neighbour-row gathers never wait on HBM/L2 latency in registers:
//
//  * rows are cut (host side, once per mesh: spmm_tiles.py) into tiles of
//    consecutive velocity nodes or pressure rows; a tile's stage holds every
//    neighbour segment its rows touch (member-minor rows: one node = 2J
//    contiguous doubles per system) plus its slices of the CSR streams
//    (row pointers, tile-local column slots, both systems' values, B^T pairs);
//  * one producer warp per CTA moves a tile with cp.async.bulk copies (a
//    precomputed list of (source, destination, bytes) records; consecutive
//    neighbour ids are merged into one copy) that complete on the stage's
//    mbarrier, NSTAGE tiles ahead of the consumers (persistent CTAs, tiles
//    strided by the grid so concurrently processed rows stay close in L2);
//  * consumer warps compute rows exactly as the direct kernels do (row groups
//    of L lanes, 16-byte member pairs, both systems per thread), reading the
//    staged operands from shared memory, and release the stage.
#include <cstdint>

#include "ens_internal.cuh"

namespace {

struct TileDesc {
    int kind, row0, row1, rec_off, n_rec, total, segsys, o_pres;
    int o_rp, o_col, o_a0, o_a1, o_btp, o_btl, o_btv, pad;
};
struct CopyRec {
    long long src;
    int dst;
    int bk;   // bytes | kind << 24
};

constexpr int MAXSTAGE = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
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
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ int lds_s32(uint32_t a) {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}

struct TileSrc {
    const char* base[10];   // record kinds: X, A, s_rowptr, lcol_a, bt_rowptr, lcol_bt, bt_val, b_rowptr, lcol_b, b_val
};

template <int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    k_spmm_tiles(const TileDesc* __restrict__ tiles, int ntiles, const CopyRec* __restrict__ recs, TileSrc srcs,
                 const uint8_t* __restrict__ cflag, const double* __restrict__ X, const double* __restrict__ Bv,
                 double* __restrict__ Y, int64_t N, int J, int nvel, int mode, int stage_bytes, int nstage) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[2 * MAXSTAGE];   // full[0..S), empty[S..2S)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bbase = smem_u32(bars);
    if (threadIdx.x == 0) {
        for (int s = 0; s < nstage; ++s) {
            mbar_init(bbase + 8 * s, 1);
            mbar_init(bbase + 8 * (MAXSTAGE + s), NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW) {
        // producer: stream tile stages ahead of the consumers
        int s = 0;
        uint32_t ph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            mbar_wait(bbase + 8 * (MAXSTAGE + s), ph ^ 1);
            const int rec_off = __ldg(&tiles[t].rec_off), n_rec = __ldg(&tiles[t].n_rec);
            const uint32_t full = bbase + 8 * s;
            if (lane == 0) mbar_expect_tx(full, (uint32_t)__ldg(&tiles[t].total));
            __syncwarp();
            const uint32_t dst0 = sbase + (uint32_t)(s * stage_bytes);
            for (int r = lane; r < n_rec; r += 32) {
                const CopyRec cr = recs[rec_off + r];
                const int kind = cr.bk >> 24, bytes = cr.bk & 0xffffff;
                const char* src = kind == 0 ? reinterpret_cast<const char*>(X) + cr.src : srcs.base[kind] + cr.src;
                bulk_g2s(dst0 + (uint32_t)cr.dst, src, (uint32_t)bytes, full);
            }
            if (++s == nstage) {
                s = 0;
                ph ^= 1;
            }
        }
        return;
    }

    // consumers
    const int H = J >> 1;                     // double2 per component
    const int64_t MS = N * H;                 // double2 per system block
    const double2* X2 = reinterpret_cast<const double2*>(X);
    double2* Y2 = reinterpret_cast<double2*>(Y);
    const double2* B2 = reinterpret_cast<const double2*>(Bv);
    const int Lv = H, Rv = 32 / Lv;           // velocity rows: J double2 per system over H lanes x 2
    const int Lp = (H + 1) >> 1, Rp = 32 / Lp; // pressure rows: H double2 pairs over Lp lanes x 2
    const uint32_t rowb_v = (uint32_t)(J * 16), rowb_p = (uint32_t)(H * 16);
    int s = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileDesc d = tiles[t];
        mbar_wait(bbase + 8 * s, ph);
        const uint32_t st = sbase + (uint32_t)(s * stage_bytes);
        const uint32_t seg1 = (uint32_t)d.segsys;
        if (d.kind == 0) {
            const int r = lane / Lv, part = lane - r * Lv;
            if (r < Rv) {
                for (int node = d.row0 + warp * Rv + r; node < d.row1; node += NCW * Rv) {
                    double2 acc[2][2];
#pragma unroll
                    for (int m = 0; m < 2; ++m)
#pragma unroll
                        for (int v = 0; v < 2; ++v) acc[m][v] = make_double2(0.0, 0.0);
                    const int k0 = lds_s32(st + (uint32_t)(d.o_rp + 4 * node));
                    const int k1 = lds_s32(st + (uint32_t)(d.o_rp + 4 * node + 4));
                    int k = k0;
                    for (; k + 2 <= k1; k += 2) {
                        const uint32_t l0 = (uint32_t)lds_s32(st + (uint32_t)(d.o_col + 4 * k));
                        const uint32_t l1 = (uint32_t)lds_s32(st + (uint32_t)(d.o_col + 4 * k + 4));
                        const double a00 = lds_f64(st + (uint32_t)(d.o_a0 + 8 * k));
                        const double a01 = lds_f64(st + (uint32_t)(d.o_a0 + 8 * k + 8));
                        const double a10 = lds_f64(st + (uint32_t)(d.o_a1 + 8 * k));
                        const double a11 = lds_f64(st + (uint32_t)(d.o_a1 + 8 * k + 8));
#pragma unroll
                        for (int v = 0; v < 2; ++v) {
                            const int i = part + Lv * v;
                            const uint32_t o = 16u * (uint32_t)i;
                            const double2 x00 = lds_f64x2(st + l0 * rowb_v + o);
                            const double2 x01 = lds_f64x2(st + l1 * rowb_v + o);
                            const double2 x10 = lds_f64x2(st + seg1 + l0 * rowb_v + o);
                            const double2 x11 = lds_f64x2(st + seg1 + l1 * rowb_v + o);
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
                    for (; k < k1; ++k) {
                        const uint32_t l0 = (uint32_t)lds_s32(st + (uint32_t)(d.o_col + 4 * k));
                        const double a00 = lds_f64(st + (uint32_t)(d.o_a0 + 8 * k));
                        const double a10 = lds_f64(st + (uint32_t)(d.o_a1 + 8 * k));
#pragma unroll
                        for (int v = 0; v < 2; ++v) {
                            const uint32_t o = 16u * (uint32_t)(part + Lv * v);
                            const double2 x00 = lds_f64x2(st + l0 * rowb_v + o);
                            const double2 x10 = lds_f64x2(st + seg1 + l0 * rowb_v + o);
                            acc[0][v].x = fma(a00, x00.x, acc[0][v].x);
                            acc[0][v].y = fma(a00, x00.y, acc[0][v].y);
                            acc[1][v].x = fma(a10, x10.x, acc[1][v].x);
                            acc[1][v].y = fma(a10, x10.y, acc[1][v].y);
                        }
                    }
                    // pressure couplings: staged pressure rows (H double2 per component slot)
                    const int t0 = lds_s32(st + (uint32_t)(d.o_btp + 4 * node));
                    const int t1 = lds_s32(st + (uint32_t)(d.o_btp + 4 * node + 4));
                    for (int q = t0; q < t1; ++q) {
                        const uint32_t lq = (uint32_t)lds_s32(st + (uint32_t)(d.o_btl + 4 * q));
                        const double2 b0 = lds_f64x2(st + (uint32_t)(d.o_btv + 16 * q));
#pragma unroll
                        for (int v = 0; v < 2; ++v) {
                            // v = 0: x component (member pair part), v = 1: y component
                            const uint32_t o = (uint32_t)d.o_pres + lq * rowb_p + 16u * (uint32_t)part;
                            const double2 x0 = lds_f64x2(st + o), x1 = lds_f64x2(st + seg1 + o);
                            const double f0 = v ? b0.y : b0.x;
                            acc[0][v].x -= f0 * x0.x;
                            acc[0][v].y -= f0 * x0.y;
                            acc[1][v].x -= f0 * x1.x;
                            acc[1][v].y -= f0 * x1.y;
                        }
                    }
#pragma unroll
                    for (int v = 0; v < 2; ++v) {
                        const int i = part + Lv * v;
                        const int64_t o = (int64_t)node * J + i;
                        const bool ident = cflag[2 * node + v] != 0;
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
            }
        } else {
            const int r = lane / Lp, part = lane - r * Lp;
            if (r < Rp) {
                for (int p = d.row0 + warp * Rp + r; p < d.row1; p += NCW * Rp) {
                    double2 acc[2][2];
#pragma unroll
                    for (int m = 0; m < 2; ++m)
#pragma unroll
                        for (int v = 0; v < 2; ++v) acc[m][v] = make_double2(0.0, 0.0);
                    const int t0 = lds_s32(st + (uint32_t)(d.o_rp + 4 * p));
                    const int t1 = lds_s32(st + (uint32_t)(d.o_rp + 4 * p + 4));
                    for (int q = t0; q < t1; ++q) {
                        const uint32_t l0 = (uint32_t)lds_s32(st + (uint32_t)(d.o_col + 4 * q));
                        const double2 b0 = lds_f64x2(st + (uint32_t)(d.o_a0 + 16 * q));
#pragma unroll
                        for (int v = 0; v < 2; ++v) {
                            const int i = 2 * part + v;
                            if (i < H) {
#pragma unroll
                                for (int m = 0; m < 2; ++m) {
                                    const uint32_t o = st + m * seg1 + l0 * rowb_v + 16u * (uint32_t)i;
                                    const double2 u0 = lds_f64x2(o), w0 = lds_f64x2(o + rowb_p);
                                    acc[m][v].x += b0.x * u0.x + b0.y * w0.x;
                                    acc[m][v].y += b0.x * u0.y + b0.y * w0.y;
                                }
                            }
                        }
                    }
                    const int64_t row = (int64_t)nvel + p;
                    const bool ident = cflag[row] != 0;
#pragma unroll
                    for (int v = 0; v < 2; ++v) {
                        const int i = 2 * part + v;
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
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bbase + 8 * (MAXSTAGE + s));
        if (++s == nstage) {
            s = 0;
            ph ^= 1;
        }
    }
}

constexpr int NCW_DEFAULT = 8;

}  // namespace

int spmm_tiles_setup(ens_ctx* c) {
    const int bytes = c->tiles.stage_bytes * c->tiles.nstage;
    ENS_CK(cudaFuncSetAttribute(k_spmm_tiles<NCW_DEFAULT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    return ENS_OK;
}

bool spmm_tiles_usable(const ens_ctx* c, const double* x, const double* b, const double* y) {
    if (!c->use_tiles) return false;
    const uintptr_t m = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                        (b ? reinterpret_cast<uintptr_t>(b) : 0);
    return (m & 15) == 0;
}

int launch_spmm_tiles(ens_ctx* c, cudaStream_t s, const double* as_vals, const double* x, const double* b, double* y,
                      int mode) {
    const ens_spmm_tiles& T = c->tiles;
    TileSrc srcs;
    srcs.base[0] = nullptr;
    srcs.base[1] = reinterpret_cast<const char*>(as_vals);
    srcs.base[2] = reinterpret_cast<const char*>(c->m.s_rowptr);
    srcs.base[3] = reinterpret_cast<const char*>(T.lcol_a);
    srcs.base[4] = reinterpret_cast<const char*>(c->m.bt_rowptr);
    srcs.base[5] = reinterpret_cast<const char*>(T.lcol_bt);
    srcs.base[6] = reinterpret_cast<const char*>(c->m.bt_val);
    srcs.base[7] = reinterpret_cast<const char*>(c->m.b_rowptr);
    srcs.base[8] = reinterpret_cast<const char*>(T.lcol_b);
    srcs.base[9] = reinterpret_cast<const char*>(c->m.b_val);
    const int grid = T.ntiles < T.grid ? T.ntiles : T.grid;
    k_spmm_tiles<NCW_DEFAULT><<<grid, (NCW_DEFAULT + 1) * 32, (size_t)T.stage_bytes * T.nstage, s>>>(
        reinterpret_cast<const TileDesc*>(T.tiles), T.ntiles, reinterpret_cast<const CopyRec*>(T.recs), srcs,
        c->m.cflag, x, b ? b : x, y, c->n_total, c->J, (int)c->n_vel, mode, T.stage_bytes, T.nstage);
    ENS_CKL();
    return ENS_OK;
}
