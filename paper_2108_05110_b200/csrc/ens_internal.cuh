// Internal declarations shared by the B200 kernels and the C-ABI layer.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/ensmhd_b200.h"

#define ENS_NQ 7
#define ENS_PW 64
#define ENS_TILE 64
#define ENS_EXT_ROWS 8
#define ENS_VEC_ROWS 64
#define ENS_RED_BLOCKS 296   // 2 x 148 SMs: fixed grid => deterministic two-stage reductions
#define ENS_MAX_RESTART 16

void ens_set_error(const char* msg, const char* file, int line);

#define ENS_CK(x)                                                             \
    do {                                                                      \
        cudaError_t e_ = (x);                                                 \
        if (e_ != cudaSuccess) {                                              \
            ens_set_error(cudaGetErrorString(e_), __FILE__, __LINE__);       \
            return ENS_ECUDA;                                                 \
        }                                                                     \
    } while (0)

// every kernel launch site ends with ENS_CKL(): it also counts the launch
extern unsigned long long g_ens_launches;
#define ENS_CKL()                  \
    do {                           \
        ++g_ens_launches;          \
        ENS_CK(cudaGetLastError()); \
    } while (0)

struct GmresCol;   // per-column Krylov scalars (device)

struct ens_ctx {
    int device = 0;
    ens_mesh_desc m{};
    ens_plan_desc p{};
    int32_t n_vel = 0, n_total = 0, J = 0;
    std::vector<int32_t> color_off;
    std::vector<int64_t> orig_level_off, level_storage_off;
    std::vector<int32_t> level_front_off;
    std::vector<int64_t> sched_factor, sched_fwd, sched_bwd;
    // workspace (owned)
    double* fronts = nullptr;      // nmat * front_storage
    double* frvec = nullptr;       // nmat * n_idx * J
    double* kry = nullptr;         // Krylov blocks
    int32_t kry_restart = 0;
    int32_t kry_short = 0;         // cycle shortened for lack of device memory
    int32_t gm_total_it = 0;       // iterations of a begun solve (ens_solve_begin / _finish)
    int32_t gm_predict = 0;
    int32_t gm_seq = 0;            // last round-trip sequence number seen in h_count[2]
    int32_t krylov_first = -1;     // 1 (default): Richardson first cycle; 0: FGMRES (ENS_KRYLOV_FIRST)
    size_t kry_bytes = 0;
    double* red_part = nullptr;    // reduction partials
    double* red_out = nullptr;     // small outputs
    GmresCol* cols = nullptr;      // nmat*J
    int32_t* d_count = nullptr;    // device counters
    double* colpanel = nullptr;    // factorisation: unscaled column panels of the current panel step (per level)
    int64_t colpanel_rows = 0;
    int32_t* h_count = nullptr;    // pinned
    double* h_small = nullptr;     // pinned
    size_t ws_bytes = 0;
    // CUDA graphs of the fixed launch sequences
    void* solve_io = nullptr;      // device {r, z} pointer table of the solve graph
    double* partial = nullptr;     // split-K partial products of the solve GEMMs
    int* ticket = nullptr;         // split-K arrival counters (last CTA reduces)
    int4* sitem = nullptr;         // solve work items with their front's geometry (3 x int4 per item)
    // streamed solve (ens_mfsolve.cu, "stream" path): factor entries re-laid out per work tile in
    // DMMA fragment order after each factorisation, read by bulk copies in a producer/consumer pipeline
    int stream_mode = -1;          // -1 undecided, 0 classic k_sgemm path, 1 streamed
    double* sstream = nullptr;     // [2][stream_len] packed factor tiles
    int64_t stream_len = 0;        // doubles per system
    void* stiles = nullptr;        // STile[n]
    int64_t n_stiles = 0;
    int32_t* scta = nullptr;       // per launch: CTA unit offsets
    std::vector<int64_t> slaunch;  // per launch: (dir, level, first tile, cta_off index, grid, pieces per unit, units)
    double* sfr = nullptr;         // blocked front vectors [2][ncb][n_idx][ldb]
    int32_t* sbg_rows = nullptr;   // per level: pivot rows the forward assembly fills
    std::vector<int64_t> sbg_off;  // level offsets into sbg_rows
    void* ssc_ent = nullptr;       // backward scatter pairs (int2: descendant's contribution row, source row in its tile)
    double* spart = nullptr;       // fragment sums of the split launches' pieces
    int scw = 0, sncb = 0, sldb = 0, snst = 0, skc = 0;
    size_t sstage = 0;
    size_t sdesc = 0;              // shared-memory bytes for a CTA's tile descriptors
    size_t srt = 0;                // ... for the backward epilogue's result tiles
    double* nrm_part = nullptr;    // fused residual-norm partials of the SpMM
    double* diag_part = nullptr;   // per-block partials of the diagnostics (launch_diagnostics)
    size_t diag_part_n = 0;
    double* ec = nullptr;          // member-pass element buffer [2][nt][6][2][J]
    double* el = nullptr;          // assembly element buffer [2][36][nt]
    int32_t* finit_rows = nullptr; // per level: front rows k_finit assembles (bit 31: pivot row)
    std::vector<int64_t> finit_off;   // level offsets into finit_rows
    std::vector<int64_t> idx_off_h;   // host copy of the plan's f_idx_off
    void* g_solve = nullptr;       // cudaGraphExec_t
    int64_t g_solve_kernels = 0;
    void* g_factor = nullptr;      // cudaGraphExec_t
    const double* g_factor_key = nullptr;
    void* g_factor_alt = nullptr;  // the graph of the other value buffer (announced steps: one per parity)
    const double* g_factor_key_alt = nullptr;
    int g_factor_pivot_alt = 0;
    int diag_pivot = 0;            // 1: in-panel partial pivoting in DIAG (k_diag), 0: k_diag_np
    int spmm_wide = -1;            // wide-member SpMM variant (ENS_SPMM_WIDE, read on first use)
    int g_factor_pivot = 0;
    int64_t g_factor_kernels = 0;
};

// ---- kernels launchers (ens_kernels.cu) ----
int launch_member_sums(ens_ctx* c, cudaStream_t s, const double* x, double* sums);
int launch_lincomb(ens_ctx* c, cudaStream_t s, double a, const double* x, double b, double* y);
int launch_rhs(ens_ctx* c, cudaStream_t s, const double* x, const double* coef, double inv_dt,
               const ens_data_desc* loads, double* rhs);
int launch_member_pass(ens_ctx* c, cudaStream_t s, const double* x, const double* means, double* rhs, double* maxsq);
int launch_rhs_fused(ens_ctx* c, cudaStream_t s, const double* x, const double* means, const double* coef,
                     double inv_dt, const ens_data_desc* loads, double* rhs, double* maxsq);
int launch_apply_bc(ens_ctx* c, cudaStream_t s, const ens_data_desc* bv, double* rhs);
int launch_assemble(ens_ctx* c, cudaStream_t s, const double* base, const double* means, const double* maxsq,
                    double two_mu_dt, double* as_vals);
int launch_spmm(ens_ctx* c, cudaStream_t s, const double* as_vals, const double* x, const double* b, double* y,
                int mode);
bool spmm_resnorm_ok(const ens_ctx* c);
int launch_spmm_resnorm(ens_ctx* c, cudaStream_t s, const double* as_vals, const double* x, const double* b,
                        double* y, double* bn2, double* rn2);
int launch_epilogue(ens_ctx* c, cudaStream_t s, const double* x, double* p_out);
int launch_diagnostics(ens_ctx* c, cudaStream_t s, const double* x, const double* means, double* out);
int launch_mean_error(ens_ctx* c, cudaStream_t s, const double* means, const ens_data_desc* exact, double* out);
int launch_copy_cons(ens_ctx* c, cudaStream_t s, const double* src, double* dst);
int launch_means(ens_ctx* c, cudaStream_t s, const double* sums, double inv_members, double* means);
// reference-order (J, n) blocks <-> internal member-minor blocks (import: ref -> x)
int launch_layout(ens_ctx* c, cudaStream_t s, bool import, double* ref, int64_t ld, int64_t ref_ms, int64_t n,
                  const int64_t* row, double* x, int64_t x_ms, int nsys);
// column reductions: out[mat][l][j] = sum_r A_l[mat][r][j] * B[mat][r][j]; A_l = A + l*lstride
int launch_coldot(ens_ctx* c, cudaStream_t s, const double* A, int64_t lstride, int L, const double* B,
                  int64_t rows, double* out);
// W -= sum_l V_l h_l (per column) and out[mat][j] = ||W_j||^2
int launch_axpy_norm(ens_ctx* c, cudaStream_t s, double* W, const double* V, int64_t lstride, int L,
                     const double* h, int64_t rows, double* out);

// ---- multifrontal (ens_mf.cu) ----
int mf_factor(ens_ctx* c, cudaStream_t s, const double* as_vals, int32_t* n_pert);
int mf_solve(ens_ctx* c, cudaStream_t s, const double* r, double* z);
int mf_setup(ens_ctx* c);
int mf_stream_pack(ens_ctx* c, cudaStream_t s);   // after a factorisation (no-op on the classic path)
int mf_stream_prepare(ens_ctx* c);                 // tiles + stream buffer, before any capture
bool mf_stream_on(ens_ctx* c);

// ---- Krylov (ens_krylov.cu) ----
int gmres_solve(ens_ctx* c, cudaStream_t s, const double* as_vals, const double* rhs, double* x, double rtol,
                int restart, int max_restarts, int32_t* iters, double* relres, int phase = 0);
int gmres_alloc(ens_ctx* c, int restart);
