/*
 * ensmhd_b200.h -- C ABI of the B200-native ensemble-MHD time-step hot path.
 *
 * The reference (`arxiv/paper_2108_05110`, package `ensmhd`) is pure Python;
 * its hot path is `stepper.advance` (pkg/src/ensmhd/stepper.py:360-394) and the
 * `run` loop (stepper.py:442-502).  That Python API is kept verbatim by
 * `paper_2108_05110_b200/stepper.py`, which drives the entry points below in
 * this order every time-step (one process per GPU, members = columns):
 *
 *   ens_member_sums      <- ensemble_stats means        (ensemble.py:216-224)
 *   [allreduce SUM of the member sums across ranks]
 *   ens_rhs + ens_member_pass + ens_apply_bc
 *                        <- _rhs_block                  (stepper.py:223-252)
 *                           eddy_viscosity_at_quadrature (ensemble.py:227-238)
 *   [allreduce MAX of the per-quadrature-point maxima]
 *   ens_assemble         <- assemble_shared_lhs values  (stepper.py:181-213)
 *   ens_factor           <- factorize                   (linalg.py:79-108)
 *   ens_solve            <- Factorization.solve_block   (linalg.py:62-76)
 *                           + relative_residual          (linalg.py:111-118)
 *   ens_epilogue         <- mean_zero_pressure          (stepper.py:119-123, 389-390)
 *   ens_diagnostics      <- _record / energy            (stepper.py:397-439)
 *
 * Conventions: every pointer is a DEVICE pointer unless named *_host.  Fields
 * are fp64, laid out member-minor: a block X has n_total rows (internal dof
 * order: velocity rows 2*node+comp, then pressures) and J contiguous columns,
 * one per local ensemble member; the V- and W-systems are two such blocks
 * back to back (nmat = 2).  State and right-hand-side buffers belong to the
 * caller; factorisation and Krylov workspace belong to the context.  Calls are
 * stream-ordered on `stream`; a context is bound to one device and is not
 * thread-safe.  Status codes map to Python exceptions in the host layer
 * (ENS_EINVAL -> ValueError, ENS_ENOMEM -> MemoryError,
 *  ENS_ENOCONV / ENS_ECUDA -> StepFailure, stepper.py:40-46).
 */
#ifndef ENSMHD_B200_H
#define ENSMHD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ENS_OK 0
#define ENS_EINVAL 1
#define ENS_ENOMEM 2
#define ENS_ENOCONV 3
#define ENS_ECUDA 4

#define ENS_ABI_VERSION 1

typedef struct ens_ctx ens_ctx;

/* Mesh, dof maps and constant operators (stepper.py:64-83, fem.py:112-176). */
typedef struct {
    int32_t ns;        /* P2 scalar nodes                                   */
    int32_t n_pres;    /* pressure dofs                                      */
    int32_t nt;        /* triangles                                          */
    int32_t nnz_s;     /* nnz of the scalar P2 pattern                       */
    int32_t J;         /* local ensemble members (columns)                   */
    int32_t ncolor;    /* element colours                                    */
    int32_t ncons;     /* identity rows (Dirichlet dofs + pin)               */
    int32_t pad0;
    /* scalar CSR pattern over internal nodes + constant values in it */
    const int32_t* s_rowptr;   /* ns+1 */
    const int32_t* s_col;      /* nnz_s */
    const double*  s_mass;     /* nnz_s, mass_scalar     (fem.py:254-259) */
    const double*  s_stiff;    /* nnz_s, stiffness_scalar (fem.py:262-273) */
    /* B^T rows by velocity node: (pressure index, bx, by) */
    const int32_t* bt_rowptr;  /* ns+1 */
    const int32_t* bt_col;     /* pairs */
    const double*  bt_val;     /* 2*pairs (bx, by) */
    /* B rows by pressure dof: (node, bx, by)  (fem.py:330-344) */
    const int32_t* b_rowptr;   /* n_pres+1 */
    const int32_t* b_col;
    const double*  b_val;
    const uint8_t* cflag;      /* n_total: 1 -> identity row (stepper.py:214-215) */
    /* elements, sorted by colour */
    const int32_t* e_nodes;    /* nt*6 internal node ids                */
    const double*  e_geo;      /* nt*8: area, grad lambda (3x2), pad    */
    const int32_t* e_slots;    /* nt*36 positions in the scalar pattern */
    const int32_t* color_off_host; /* ncolor+1 (HOST)                   */
    /* identity rows and where their values come from */
    const int32_t* cons_row;   /* ncons internal rows                   */
    const int32_t* cons_bidx;  /* ncons: boundary-value index, -1 -> 0  */
    const double*  pres_int;   /* n_pres: int rho_p (stepper.py:71-72)  */
    double area;               /* domain area                           */
    int32_t mean_zero;         /* subtract the pressure mean after solve */
    int32_t pad1;
    /* deterministic scatter-free assembly (element buffers gathered per row / slot) */
    const int32_t* n2e_ptr;    /* ns+1: velocity node -> element-local entries  */
    const int32_t* n2e;        /* nt*6: entries e*6 + a, element order per node */
    const int32_t* s2e_ptr;    /* nnz_s+1: CSR slot -> element-local entries     */
    const int32_t* s2e;        /* nt*36: entries ab*nt + e                        */
} ens_mesh_desc;

/* Multifrontal plan produced once per mesh by symbolic.py. */
typedef struct {
    int32_t nfront, nlevels, pw, tile;
    int64_t front_storage;      /* doubles per matrix                       */
    int64_t n_orig;
    int64_t n_cmap, n_idx, n_work;
    const int32_t* f_m;         /* device, nfront */
    const int32_t* f_k;
    const int64_t* f_off;
    const int64_t* f_idx_off;   /* nfront+1 */
    const int32_t* f_idx;
    const int32_t* f_parent;
    const int64_t* f_cmap_off;  /* nfront+1 */
    const int32_t* f_cmap;
    const int64_t* orig_dst;
    const int32_t* orig_src;
    const double*  bsrc_vals;   /* signed B / -B^T values                   */
    const int32_t* work;        /* n_work x 4 */
    const int32_t* gsrc;        /* n_idx x 4: child contribution rows gathered per front row (-1 none) */
    /* HOST arrays */
    const int64_t* orig_level_off_host;    /* nlevels+1 */
    const int64_t* level_storage_off_host; /* nlevels+1 */
    const int32_t* level_front_off_host;   /* nlevels+1 */
    const int64_t* sched_factor_host; int64_t n_sched_factor;  /* rows of 5 */
    const int64_t* sched_fwd_host;    int64_t n_sched_fwd;
    const int64_t* sched_bwd_host;    int64_t n_sched_bwd;
    int32_t max_m;
    int32_t split_k;            /* inner-dimension length of one solve-GEMM work item */
    int64_t n_slot;             /* split-K partial slots (64 rows x J each)          */
} ens_plan_desc;

/* Problem data: value_j = sum_k coef[k*J + j] * basis[k*rows + row] (+ dense). */
typedef struct {
    int32_t K;                  /* number of basis vectors (0 allowed)   */
    int32_t pad;
    int64_t rows;               /* basis row count: n_vel for loads, #boundary dofs for Dirichlet data */
    const double* basis;        /* K x rows */
    const double* coef;         /* nmat x K x J */
    const double* dense;        /* optional nmat x rows x J, or NULL     */
} ens_data_desc;

int  ens_abi_version(void);
const char* ens_last_error(void);
/* Process-wide count of kernels this library has launched (bench evidence). */
int64_t ens_kernel_launches(void);

int  ens_create(const ens_mesh_desc* mesh, const ens_plan_desc* plan, int device, ens_ctx** out);
void ens_destroy(ens_ctx* ctx);
int  ens_workspace_bytes(const ens_ctx* ctx, int64_t* bytes);
/* Panel inverses with in-panel partial pivoting (1) or diagonal pivots (0, default;
 * the symbolic ordering guarantees nonsingular leading blocks in exact arithmetic). */
int  ens_set_pivoting(ens_ctx* ctx, int on);
/* Diagnostics: how many tree-level launches of the streamed preconditioner apply run as split-K
 * pieces + reduction (0 before the first factorisation or on the classic path). */
int  ens_stream_split_launches(const ens_ctx* ctx);

/* y = a x + b y over one iterate block set (2 x n_total x J); used for the
 * extrapolated FGMRES initial iterate 2 x^n - x^{n-1}. */
int  ens_lincomb(ens_ctx* ctx, void* stream, double a, const double* x, double b, double* y);

/* Member sums over the J local columns: sum_v[r] = sum_j Xv[r][j] (r < n_vel), same for w. */
int  ens_member_sums(ens_ctx* ctx, void* stream, const double* x, double* sums);

/* means[2 * n_vel] = sums * inv_members: the ensemble means <v>, <w> (ensemble.py:216-224) from the
 * member sums -- after the allreduce SUM when members are sharded (inv_members = 1 / J_total). */
int  ens_means(ens_ctx* ctx, void* stream, const double* sums, double inv_members, double* means);

/* RHS velocity rows (stepper.py:235-247): for both sub-steps
 *   rhs_V = (M/dt - ls_j K) v_j - lc_j K w_j + load_V      (same = v, other = w)
 *   rhs_W = (M/dt - ls_j K) w_j - lc_j K v_j + load_W
 * member_coef = [ls(J) | lc(J)]; loads over n_vel rows. */
int  ens_rhs(ens_ctx* ctx, void* stream, const double* x, const double* member_coef, double inv_dt,
             const ens_data_desc* loads, double* rhs);

/* Member pass (element-parallel x member-parallel): subtract the explicit
 * fluctuation transport N(z'_j) same_j from both right-hand sides
 * (fem.py:411-420) and write max_j |z'_j(x_q)|^2 for both families into
 * maxsq (nmat x nt x 7; matrix V uses w', W uses v') (ensemble.py:227-238). */
int  ens_member_pass(ens_ctx* ctx, void* stream, const double* x, const double* means, double* rhs, double* maxsq);

/* ens_rhs + ens_member_pass in one element pass (even J): every element's whole
 * right-hand side of both sub-steps, M same/dt - N(z') same - K(ls same + lc other),
 * at the 7 quadrature points that assemble M and K exactly, summed per row in a
 * fixed order with the loads added; maxsq as ens_member_pass (stepper.py:223-252). */
int  ens_rhs_fused(ens_ctx* ctx, void* stream, const double* x, const double* means, const double* member_coef,
                   double inv_dt, const ens_data_desc* loads, double* rhs, double* maxsq);

/* Identity-row values: rhs[cons] = Dirichlet data (stepper.py:250) or 0 (pin, stepper.py:251). */
int  ens_apply_bc(ens_ctx* ctx, void* stream, const ens_data_desc* bvals, double* rhs);

/* Shared velocity-block values for both sub-steps (stepper.py:195-206):
 *   A_m = base + N(mean_m) + K(2 mu dt maxsq_m), base = M/dt + (nu_bar+nu_m_bar)/2 K. */
int  ens_assemble(ens_ctx* ctx, void* stream, const double* base, const double* means, const double* maxsq,
                  double two_mu_dt, double* as_vals);

/* Multifrontal LU of both saddle matrices (preconditioner, built per sub-step). */
int  ens_factor(ens_ctx* ctx, void* stream, const double* as_vals, int32_t* n_perturbed_host);

/* Column-batched right-preconditioned FGMRES on both systems.  x holds the
 * initial guess (identity rows are overwritten from rhs) and returns the
 * solution; relres_host[m] = max_j ||b_j - K x_j|| / max(||b_j||, tiny).
 * iters_host: in = predicted iteration count p >= 0 (the first cycle runs p
 * iterations without host round trips, then the true residual decides; 0 =
 * check after every iteration), out = iterations performed. */
int  ens_solve(ens_ctx* ctx, void* stream, const double* as_vals, const double* rhs, double* x,
               double rtol, int32_t restart, int32_t max_restarts, int32_t* iters_host, double* relres_host);
/* ens_solve split at its one host round trip, so a whole time step can be
 * captured into a CUDA graph: ens_solve_begin enqueues the first cycle
 * (`predict` >= 1 iterations) and the next true residual, whose active-column
 * count and norms go to pinned host memory, with no synchronisation (stream-
 * capturable); ens_solve_finish synchronises the stream and continues exactly
 * as ens_solve would (further cycles only if some member is above rtol). */
int  ens_solve_begin(ens_ctx* ctx, void* stream, const double* as_vals, const double* rhs, double* x,
                     double rtol, int32_t restart, int32_t predict);
int  ens_solve_finish(ens_ctx* ctx, void* stream, const double* as_vals, const double* rhs, double* x,
                      double rtol, int32_t restart, int32_t max_restarts, int32_t* iters_host, double* relres_host);

/* y = K x (mode 0) or y = b - K x (mode 1), both matrices. */
int  ens_spmm(ens_ctx* ctx, void* stream, const double* as_vals, const double* x, const double* b, double* y, int mode);

/* z = P^-1 r with the current factorisation (identity rows copied). */
int  ens_precond_apply(ens_ctx* ctx, void* stream, const double* r, double* z);

/* Pressure epilogue: p_out[m] = x_m pressure rows minus their discrete mean. */
int  ens_epilogue(ens_ctx* ctx, void* stream, const double* x, double* p_out);

/* Diagnostics of _record (stepper.py:432-439) on device:
 *   out[0] = <v>^T M <v>, out[1] = <w>^T M <w>  (from the global means)
 *   out[2 + 0*J + j] = v_j^T M v_j, [2+J..] = w_j^T M w_j, [2+2J..] = v_j^T K v_j,
 *   [2+3J..] = w_j^T K w_j, [2+4J..] = ||div v_j||^2, [2+5J..] = ||div w_j||^2 */
int  ens_diagnostics(ens_ctx* ctx, void* stream, const double* x, const double* means, double* out);

/* Squared errors of the ensemble means against a separable exact field (device):
 * out = [d_v^T M d_v, d_v^T K d_v, d_w^T M d_w, d_w^T K d_w], d = <z> - sum_k coef[fam][k] basis[k]
 * (exact->rows = n_vel internal rows, exact->coef = 2 x K): the summands of the discrete
 * L2(0,T;H1) error norm of experiments.error_norm_21 (experiments.py:59-73, fem.py:502-505). */
int  ens_mean_error(ens_ctx* ctx, void* stream, const double* means, const ens_data_desc* exact, double* out);

/* State layout conversion on the device (the EnsembleState arrays of ensemble.py:183-190 cross
 * PCIe in the reference's own layout; this replaces the reference's host-side array views):
 *   ref: nsys blocks (stride ref_stride doubles) of J member rows of length ld, reference dof
 *        order (the (J, n) arrays v, w or q, r), in device memory;
 *   x:   nsys internal member-minor blocks (stride x_stride doubles), x[row[c] * J + j];
 *   row[c] (device, int64): internal row of reference dof c, c in [0, n).
 * import: x[s][row[c]][j] = ref[s][j][c];  export: ref[s][j][c] = x[s][row[c]][j]. */
int  ens_layout_import(ens_ctx* ctx, void* stream, const double* ref, int64_t ld, int64_t ref_stride, int64_t n,
                       const int64_t* row, double* x, int64_t x_stride, int32_t nsys);
/* The upload half of a host-array step in one call: the (J, n) host arrays v, w (pinned: asynchronous
 * DMA) -> staging[2][J][n] on the device -> ens_layout_import into x (two systems, stride x_stride). */
int  ens_state_upload(ens_ctx* ctx, void* stream, const double* host_v, const double* host_w, int64_t n,
                      double* staging, const int64_t* row, double* x, int64_t x_stride);
int  ens_layout_export(ens_ctx* ctx, void* stream, const double* x, int64_t x_stride, int64_t n, const int64_t* row,
                       double* ref, int64_t ld, int64_t ref_stride, int32_t nsys);

#ifdef __cplusplus
}
#endif
#endif
