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
    fm, fk, off = plan.f_m, plan.f_k, plan.f_off
    J = rhs.shape[1]
    fr = [np.zeros((int(fm[f]), J)) for f in range(plan.nfront)]
    x = np.zeros_like(rhs)

    def front(f):
        m = int(fm[f])
        return st[off[f]:off[f] + m * m].reshape(m, m)

    def idx(f):
        return plan.f_idx[plan.f_idx_off[f]:plan.f_idx_off[f + 1]]

    for op, L, io, n, arg in plan.schedule["fwd"]:
        for it in work[io:io + n]:
            f, r0 = it[0], it[1]
            if op == S.SOP_FINIT:
                rows = np.arange(r0, min(r0 + S.VEC_ROWS, fm[f]))
                fr[f][rows] = np.where((rows < fk[f])[:, None], rhs[idx(f)[rows]], 0.0)
            elif op == S.SOP_FEXT:
                c = f
                p = plan.f_parent[c]
                mp = plan.f_cmap[plan.f_cmap_off[c]:plan.f_cmap_off[c + 1]]
                rows = np.arange(r0, min(r0 + S.VEC_ROWS, len(mp)))
                fr[p][mp[rows]] += fr[c][fk[c] + rows]
            elif op == S.SOP_FGEMM:
                k = fk[f]
                rows = slice(k + r0, min(k + r0 + S.SOLVE_ROWS, fm[f]))
                fr[f][rows] -= front(f)[rows, :k] @ fr[f][:k]
    for op, L, io, n, arg in plan.schedule["bwd"]:
        for it in work[io:io + n]:
            f, r0 = it[0], it[1]
            if op == S.SOP_BGATHER:
                rows = np.arange(r0, min(r0 + S.VEC_ROWS, fm[f]))
                fr[f][rows] = x[idx(f)[rows]]
            elif op == S.SOP_BGEMM:
                rows = np.arange(r0, min(r0 + S.SOLVE_ROWS, fk[f]))
                x[idx(f)[rows]] = -front(f)[rows, :] @ fr[f]
    return x
