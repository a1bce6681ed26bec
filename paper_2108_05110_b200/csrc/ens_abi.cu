// extern "C" entry points of include/ensmhd_b200.h: context lifetime and the
// per-step calls the Python host layer (stepper.py) makes.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "ens_internal.cuh"

int ens_upload_tables();
size_t gmres_col_bytes();

static thread_local std::string g_err;
unsigned long long g_ens_launches = 0;

void ens_set_error(const char* msg, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "%s (%s:%d)", msg, file, line);
    g_err = buf;
}

#define RET(x)                         \
    do {                               \
        int rc_ = (x);                 \
        if (rc_ != ENS_OK) return rc_; \
    } while (0)

extern "C" {

int ens_abi_version(void) { return ENS_ABI_VERSION; }

const char* ens_last_error(void) { return g_err.c_str(); }

int64_t ens_kernel_launches(void) { return (int64_t)g_ens_launches; }

int ens_create(const ens_mesh_desc* mesh, const ens_plan_desc* plan, int device, ens_ctx** out) {
    if (!mesh || !plan || !out) {
        ens_set_error("null argument", __FILE__, __LINE__);
        return ENS_EINVAL;
    }
    if (mesh->J < 1 || mesh->ns < 1 || mesh->nt < 1 || plan->pw != ENS_PW || plan->tile != ENS_TILE) {
        ens_set_error("invalid mesh/plan description", __FILE__, __LINE__);
        return ENS_EINVAL;
    }
    ENS_CK(cudaSetDevice(device));
    ens_ctx* c = new ens_ctx();
    c->device = device;
    c->m = *mesh;
    c->p = *plan;
    c->n_vel = 2 * mesh->ns;
    c->n_total = c->n_vel + mesh->n_pres;
    c->J = mesh->J;
    c->color_off.assign(mesh->color_off_host, mesh->color_off_host + mesh->ncolor + 1);
    c->orig_level_off.assign(plan->orig_level_off_host, plan->orig_level_off_host + plan->nlevels + 1);
    c->level_storage_off.assign(plan->level_storage_off_host, plan->level_storage_off_host + plan->nlevels + 1);
    c->level_front_off.assign(plan->level_front_off_host, plan->level_front_off_host + plan->nlevels + 1);
    c->sched_factor.assign(plan->sched_factor_host, plan->sched_factor_host + 5 * plan->n_sched_factor);
    c->sched_fwd.assign(plan->sched_fwd_host, plan->sched_fwd_host + 5 * plan->n_sched_fwd);
    c->sched_bwd.assign(plan->sched_bwd_host, plan->sched_bwd_host + 5 * plan->n_sched_bwd);
    c->m.color_off_host = nullptr;
    // workspace
    const size_t J = (size_t)c->J;
    const size_t L = ENS_MAX_RESTART + 1;
    const size_t want[4] = {
        sizeof(double) * 2 * (size_t)plan->front_storage,
        sizeof(double) * 2 * (size_t)plan->n_idx * J,
        sizeof(double) * (size_t)ENS_RED_BLOCKS * 2 * L * J,
        sizeof(double) * 2 * J * (6 + 3 * L),
    };
    void* ptrs[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int i = 0; i < 4; ++i) {
        if (cudaMalloc(&ptrs[i], want[i]) != cudaSuccess) {
            for (int k = 0; k < i; ++k) cudaFree(ptrs[k]);
            delete c;
            ens_set_error("out of device memory for factorisation workspace", __FILE__, __LINE__);
            return ENS_ENOMEM;
        }
        c->ws_bytes += want[i];
    }
    c->fronts = (double*)ptrs[0];
    c->frvec = (double*)ptrs[1];
    c->red_part = (double*)ptrs[2];
    c->red_out = (double*)ptrs[3];
    const size_t colb = gmres_col_bytes() * 2 * J;
    if (cudaMalloc((void**)&c->cols, colb) != cudaSuccess || cudaMalloc(&c->d_count, 16) != cudaSuccess) {
        ens_set_error("out of device memory", __FILE__, __LINE__);
        ens_destroy(c);
        return ENS_ENOMEM;
    }
    c->ws_bytes += colb;
    if (cudaMallocHost(&c->h_count, 16) != cudaSuccess ||
        cudaMallocHost(&c->h_small, sizeof(double) * 4 * J + 64) != cudaSuccess) {
        ens_set_error("pinned allocation failed", __FILE__, __LINE__);
        ens_destroy(c);
        return ENS_ENOMEM;
    }
    cudaMemset(c->d_count, 0, 16);   // [0] active columns / pivot count, [2] solve round-trip sequence number
    c->h_count[0] = c->h_count[1] = c->h_count[2] = c->h_count[3] = 0;
    int rc = ens_upload_tables();
    if (rc == ENS_OK) rc = mf_setup(c);
    if (rc != ENS_OK) {
        ens_destroy(c);
        return rc;
    }
    *out = c;
    return ENS_OK;
}

void ens_destroy(ens_ctx* c) {
    if (!c) return;
    cudaFree(c->fronts);
    cudaFree(c->frvec);
    cudaFree(c->kry);
    cudaFree(c->red_part);
    cudaFree(c->red_out);
    cudaFree(c->cols);
    cudaFree(c->d_count);
    cudaFree(c->colpanel);
    if (c->h_count) cudaFreeHost(c->h_count);
    if (c->h_small) cudaFreeHost(c->h_small);
    if (c->g_solve) cudaGraphExecDestroy((cudaGraphExec_t)c->g_solve);
    if (c->g_factor) cudaGraphExecDestroy((cudaGraphExec_t)c->g_factor);
    if (c->g_factor_alt) cudaGraphExecDestroy((cudaGraphExec_t)c->g_factor_alt);
    cudaFree(c->solve_io);
    cudaFree(c->partial);
    cudaFree(c->ticket);
    cudaFree(c->sitem);
    cudaFree(c->sstream);
    cudaFree(c->stiles);
    cudaFree(c->scta);
    cudaFree(c->sfr);
    cudaFree(c->sbg_rows);
    cudaFree(c->ssc_ent);
    cudaFree(c->spart);
    cudaFree(c->finit_rows);
    cudaFree(c->ec);
    cudaFree(c->nrm_part);
    cudaFree(c->diag_part);
    cudaFree(c->el);
    delete c;
}

int ens_set_pivoting(ens_ctx* c, int on) {
    if (!c) return ENS_EINVAL;
    c->diag_pivot = on ? 1 : 0;
    return ENS_OK;
}

int ens_stream_split_launches(const ens_ctx* c) {
    if (!c) return -1;
    int n = 0;
    for (size_t i = 0; i + 7 <= c->slaunch.size(); i += 7) n += c->slaunch[i + 5] > 1 ? 1 : 0;
    return n;
}

int ens_workspace_bytes(const ens_ctx* c, int64_t* bytes) {
    if (!c || !bytes) return ENS_EINVAL;
    *bytes = (int64_t)c->ws_bytes;
    return ENS_OK;
}

int ens_lincomb(ens_ctx* c, void* stream, double a, const double* x, double b, double* y) {
    if (!c || !x || !y) return ENS_EINVAL;
    return launch_lincomb(c, (cudaStream_t)stream, a, x, b, y);
}

int ens_member_sums(ens_ctx* c, void* stream, const double* x, double* sums) {
    if (!c || !x || !sums) return ENS_EINVAL;
    return launch_member_sums(c, (cudaStream_t)stream, x, sums);
}

int ens_means(ens_ctx* c, void* stream, const double* sums, double inv_members, double* means) {
    if (!c || !sums || !means || !(inv_members > 0.0)) return ENS_EINVAL;
    return launch_means(c, (cudaStream_t)stream, sums, inv_members, means);
}

int ens_rhs(ens_ctx* c, void* stream, const double* x, const double* member_coef, double inv_dt,
            const ens_data_desc* loads, double* rhs) {
    if (!c || !x || !member_coef || !rhs) return ENS_EINVAL;
    return launch_rhs(c, (cudaStream_t)stream, x, member_coef, inv_dt, loads, rhs);
}

int ens_member_pass(ens_ctx* c, void* stream, const double* x, const double* means, double* rhs, double* maxsq) {
    if (!c || !x || !means || !rhs || !maxsq) return ENS_EINVAL;
    return launch_member_pass(c, (cudaStream_t)stream, x, means, rhs, maxsq);
}

int ens_rhs_fused(ens_ctx* c, void* stream, const double* x, const double* means, const double* member_coef,
                  double inv_dt, const ens_data_desc* loads, double* rhs, double* maxsq) {
    if (!c || !x || !means || !member_coef || !rhs || !maxsq) return ENS_EINVAL;
    return launch_rhs_fused(c, (cudaStream_t)stream, x, means, member_coef, inv_dt, loads, rhs, maxsq);
}

int ens_apply_bc(ens_ctx* c, void* stream, const ens_data_desc* bvals, double* rhs) {
    if (!c || !rhs) return ENS_EINVAL;
    return launch_apply_bc(c, (cudaStream_t)stream, bvals, rhs);
}

int ens_assemble(ens_ctx* c, void* stream, const double* base, const double* means, const double* maxsq,
                 double two_mu_dt, double* as_vals) {
    if (!c || !base || !means || !maxsq || !as_vals) return ENS_EINVAL;
    return launch_assemble(c, (cudaStream_t)stream, base, means, maxsq, two_mu_dt, as_vals);
}

int ens_factor(ens_ctx* c, void* stream, const double* as_vals, int32_t* n_perturbed_host) {
    if (!c || !as_vals) return ENS_EINVAL;
    return mf_factor(c, (cudaStream_t)stream, as_vals, n_perturbed_host);
}

int ens_solve(ens_ctx* c, void* stream, const double* as_vals, const double* rhs, double* x, double rtol,
              int32_t restart, int32_t max_restarts, int32_t* iters_host, double* relres_host) {
    if (!c || !as_vals || !rhs || !x || !iters_host || !relres_host || !(rtol > 0.0)) return ENS_EINVAL;
    return gmres_solve(c, (cudaStream_t)stream, as_vals, rhs, x, rtol, restart, max_restarts, iters_host,
                       relres_host);
}

int ens_solve_begin(ens_ctx* c, void* stream, const double* as_vals, const double* rhs, double* x, double rtol,
                    int32_t restart, int32_t predict) {
    if (!c || !as_vals || !rhs || !x || !(rtol > 0.0) || predict < 1) return ENS_EINVAL;
    int32_t it = predict;
    double rel[2] = {0.0, 0.0};
    return gmres_solve(c, (cudaStream_t)stream, as_vals, rhs, x, rtol, restart, 1, &it, rel, 1);
}

int ens_solve_finish(ens_ctx* c, void* stream, const double* as_vals, const double* rhs, double* x, double rtol,
                     int32_t restart, int32_t max_restarts, int32_t* iters_host, double* relres_host) {
    if (!c || !as_vals || !rhs || !x || !iters_host || !relres_host || !(rtol > 0.0)) return ENS_EINVAL;
    return gmres_solve(c, (cudaStream_t)stream, as_vals, rhs, x, rtol, restart, max_restarts, iters_host,
                       relres_host, 2);
}

int ens_spmm(ens_ctx* c, void* stream, const double* as_vals, const double* x, const double* b, double* y, int mode) {
    if (!c || !as_vals || !x || !y || (mode == 1 && !b)) return ENS_EINVAL;
    return launch_spmm(c, (cudaStream_t)stream, as_vals, x, b, y, mode);
}

int ens_precond_apply(ens_ctx* c, void* stream, const double* r, double* z) {
    if (!c || !r || !z) return ENS_EINVAL;
    return mf_solve(c, (cudaStream_t)stream, r, z);
}

int ens_epilogue(ens_ctx* c, void* stream, const double* x, double* p_out) {
    if (!c || !x || !p_out) return ENS_EINVAL;
    return launch_epilogue(c, (cudaStream_t)stream, x, p_out);
}

int ens_mean_error(ens_ctx* c, void* stream, const double* means, const ens_data_desc* exact, double* out) {
    if (!c || !means || !exact || !out || exact->K < 1 || !exact->basis || !exact->coef ||
        exact->rows != (int64_t)c->n_vel)
        return ENS_EINVAL;
    return launch_mean_error(c, (cudaStream_t)stream, means, exact, out);
}

int ens_diagnostics(ens_ctx* c, void* stream, const double* x, const double* means, double* out) {
    if (!c || !x || !means || !out) return ENS_EINVAL;
    return launch_diagnostics(c, (cudaStream_t)stream, x, means, out);
}

int ens_layout_import(ens_ctx* c, void* stream, const double* ref, int64_t ld, int64_t ref_stride, int64_t n,
                      const int64_t* row, double* x, int64_t x_stride, int32_t nsys) {
    if (!c || !ref || !row || !x || n < 0 || ld < n || nsys < 1) return ENS_EINVAL;
    return launch_layout(c, (cudaStream_t)stream, true, const_cast<double*>(ref), ld, ref_stride, n, row, x, x_stride,
                         nsys);
}

int ens_state_upload(ens_ctx* c, void* stream, const double* host_v, const double* host_w, int64_t n,
                     double* staging, const int64_t* row, double* x, int64_t x_stride) {
    if (!c || !host_v || !host_w || !staging || !row || !x || n < 0) return ENS_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = sizeof(double) * (size_t)c->J * (size_t)n;
    ENS_CK(cudaMemcpyAsync(staging, host_v, bytes, cudaMemcpyHostToDevice, s));
    ENS_CK(cudaMemcpyAsync(staging + (int64_t)c->J * n, host_w, bytes, cudaMemcpyHostToDevice, s));
    return launch_layout(c, s, true, staging, n, (int64_t)c->J * n, n, row, x, x_stride, 2);
}

int ens_layout_export(ens_ctx* c, void* stream, const double* x, int64_t x_stride, int64_t n, const int64_t* row,
                      double* ref, int64_t ld, int64_t ref_stride, int32_t nsys) {
    if (!c || !ref || !row || !x || n < 0 || ld < n || nsys < 1) return ENS_EINVAL;
    return launch_layout(c, (cudaStream_t)stream, false, ref, ld, ref_stride, n, row, const_cast<double*>(x), x_stride,
                         nsys);
}

}  // extern "C"
