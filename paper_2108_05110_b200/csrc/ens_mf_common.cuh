// Shared device-side view of the multifrontal plan (ens_mf.cu / ens_mfsolve.cu).
#pragma once
#include "ens_internal.cuh"

enum { OP_ZERO = 0, OP_ORIG, OP_EXTADD, OP_DIAG, OP_HPANEL, OP_UPDATE, OP_GPANEL };
enum { SOP_FINIT = 0, SOP_FEXT, SOP_FGEMM, SOP_BGATHER, SOP_BGEMM, SOP_FRED, SOP_BRED };

struct MfDev {
    const int32_t* m;
    const int32_t* k;
    const int64_t* off;
    const int64_t* idx_off;
    const int32_t* idx;
    const int32_t* parent;
    const int64_t* cmap_off;
    const int32_t* cmap;
    const int32_t* work;
    const int32_t* gsrc;
    int64_t storage;
};

static inline MfDev mfdev(const ens_ctx* c) {
    MfDev d;
    d.m = c->p.f_m;
    d.k = c->p.f_k;
    d.off = c->p.f_off;
    d.idx_off = c->p.f_idx_off;
    d.idx = c->p.f_idx;
    d.parent = c->p.f_parent;
    d.cmap_off = c->p.f_cmap_off;
    d.cmap = c->p.f_cmap;
    d.work = c->p.work;
    d.gsrc = c->p.gsrc;
    d.storage = c->p.front_storage;
    return d;
}

