"""Numpy emulation of the device multifrontal sweep factorisation / solve (test helper).

Executes the exact launch schedule of `symbolic.build_schedule` with dense
numpy ops, so the plan (ordering, maps, panels, block-sweep algebra) is
verified on CPU against a direct solve before any GPU run.
"""

import numpy as np

from paper_2108_05110_b200 import symbolic as S


def _outside(idx, a, pw):
    """Map outside-panel indices r' to front rows: r' < a ? r' : r' + pw."""
    idx = np.asarray(idx)
    return np.where(idx < a, idx, idx + pw)


def factor(plan, as_vals, pw=S.PW):
    """Return the per-matrix front storage after the sweep (flat float64)."""
    st = np.zeros(plan.front_storage)
    src = np.concatenate([as_vals, plan.bsrc_vals])
    work = plan.schedule["work"]
    fm, fk, off = plan.f_m, plan.f_k, plan.f_off

    def front(f):
        m = int(fm[f])
        return st[off[f]:off[f] + m * m].reshape(m, m)

    for op, L, io, n, arg in plan.schedule["factor"]:
        items = work[io:io + n]
        if op == S.OP_ZERO:
            st[plan.level_storage_off[L]:plan.level_storage_off[L + 1]] = 0.0
        elif op == S.OP_ORIG:
            a, b = plan.orig_level_off[L], plan.orig_level_off[L + 1]
            st[plan.orig_dst[a:b]] = src[plan.orig_src[a:b]]
        elif op == S.OP_EXTADD:
            for c, r0, _, _ in items:
                p = plan.f_parent[c]
                kc = fk[c]
                mp = plan.f_cmap[plan.f_cmap_off[c]:plan.f_cmap_off[c + 1]]
                rows = np.arange(r0, min(r0 + S.EXT_ROWS, len(mp)))
                F, P = front(c), front(p)
                P[np.ix_(mp[rows], mp)] += F[kc + rows][:, kc:]
        else:
            for f, a, x0, y0 in items:
                F = front(f)
                pwf = min(pw, fk[f] - a)
                P = slice(a, a + pwf)
                t = fm[f] - pwf
                if op == S.OP_DIAG:
                    F[P, P] = -np.linalg.inv(F[P, P])
                elif op == S.OP_HPANEL:
                    cols = _outside(np.arange(x0, min(x0 + S.TILE, t)), a, pwf)
                    F[P, cols] = -F[P, P] @ F[P, cols]
                elif op == S.OP_UPDATE:
                    rows = _outside(np.arange(x0, min(x0 + S.TILE, t)), a, pwf)
                    cols = _outside(np.arange(y0, min(y0 + S.TILE, t)), a, pwf)
                    F[np.ix_(rows, cols)] -= F[rows, P] @ F[P, cols]
                elif op == S.OP_GPANEL:
                    rows = _outside(np.arange(x0, min(x0 + S.TILE, t)), a, pwf)
                    F[rows, P] = -F[rows, P] @ F[P, P]
    return st


def solve(plan, st, rhs):
    """Apply the factorisation to rhs (n_total_internal, J); returns x (free rows)."""
    work = plan.schedule["work"]
    gsrc = plan.schedule["gsrc"]
    fm, fk, off, io_ = plan.f_m, plan.f_k, plan.f_off, plan.f_idx_off
    J = rhs.shape[1]
    fr = np.zeros((int(io_[-1]), J))
    x = np.zeros_like(rhs)
    partial = {}

    def front(f):
        m = int(fm[f])
        return st[off[f]:off[f] + m * m].reshape(m, m)

    for op, L, io, n, arg in plan.schedule["fwd"]:
        for it in work[io:io + n]:
            f, r0 = it[0], it[1]
            base = io_[f]
            if op == S.SOP_FINIT:
                rows = np.arange(r0, min(r0 + S.VEC_ROWS, fm[f]))
                val = np.where((rows < fk[f])[:, None], rhs[plan.f_idx[base + rows]], 0.0)
                for s_ in range(S.MAX_GSRC):
                    src = gsrc[base + rows, s_]
                    val = val + np.where((src >= 0)[:, None], fr[np.maximum(src, 0)], 0.0)
                fr[base + rows] = val
            elif op in (S.SOP_FGEMM, S.SOP_FRED):
                k = fk[f]
                rows = np.arange(k + r0, min(k + r0 + S.SOLVE_ROWS, fm[f]))
                if op == S.SOP_FGEMM:
                    ks, slot = it[2], it[3]
                    kr = slice(ks * plan.schedule["split_k"], min(k, (ks + 1) * plan.schedule["split_k"]))
                    prod = front(f)[rows, kr] @ fr[base + kr.start:base + kr.stop]
                    if slot < 0:
                        fr[base + rows] -= prod
                    else:
                        partial[slot] = prod
                else:
                    fr[base + rows] -= sum(partial[it[3] + s_] for s_ in range(it[2]))
    for op, L, io, n, arg in plan.schedule["bwd"]:
        for it in work[io:io + n]:
            f, r0 = it[0], it[1]
            base = io_[f]
            k, m = fk[f], fm[f]
            rows = np.arange(r0, min(r0 + S.SOLVE_ROWS, k))
            if op == S.SOP_BGEMM:
                ks, slot = it[2], it[3]
                bop = np.vstack([fr[base:base + k], x[plan.f_idx[base + k:base + m]]])
                kr = slice(ks * plan.schedule["split_k"], min(m, (ks + 1) * plan.schedule["split_k"]))
                prod = front(f)[rows, kr] @ bop[kr]
                if slot < 0:
                    x[plan.f_idx[base + rows]] = -prod
                else:
                    partial[slot] = prod
            elif op == S.SOP_BRED:
                x[plan.f_idx[base + rows]] = -sum(partial[it[3] + s_] for s_ in range(it[2]))
    return x
