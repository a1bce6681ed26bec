"""Numpy emulation of the device multifrontal factorisation / solve (test helper).

Executes the exact launch schedule of `symbolic.build_schedule` with dense
numpy ops, so the plan (ordering, maps, panels, explicit-inverse algebra) is
verified on CPU against a direct solve before any GPU run.
"""

import numpy as np

from paper_2108_05110_b200 import symbolic as S


def factor(plan, as_vals, pw=S.PW):
    """Return the per-matrix front storage after factorisation (flat float64)."""
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
        elif op == S.OP_DIAG:
            for f, a, _, _ in items:
                F = front(f)
                b = min(a + pw, fk[f])
                F[a:b, a:b] = np.linalg.inv(F[a:b, a:b])
        elif op == S.OP_HPANEL:
            for f, a, c0, _ in items:
                F = front(f)
                b = min(a + pw, fk[f])
                cols = slice(b + c0, min(b + c0 + S.TILE, fm[f]))
                F[a:b, cols] = -F[a:b, a:b] @ F[a:b, cols]
        elif op == S.OP_UPDATE:
            for f, a, r0, c0 in items:
                F = front(f)
                b = min(a + pw, fk[f])
                rows = slice(b + r0, min(b + r0 + S.TILE, fm[f]))
                cols = slice(b + c0, min(b + c0 + S.TILE, fm[f]))
                F[rows, cols] += F[rows, a:b] @ F[a:b, cols]
        elif op == S.OP_GPANEL:
            for f, a, r0, _ in items:
                F = front(f)
                b = min(a + pw, fk[f])
                rows = slice(b + r0, min(b + r0 + S.TILE, fm[f]))
                F[rows, a:b] = -F[rows, a:b] @ F[a:b, a:b]
    return st


def solve(plan, st, rhs, pw=S.PW):
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
            f = it[0]
            if op == S.SOP_FINIT:
                r0 = it[1]
                rows = np.arange(r0, min(r0 + S.VEC_ROWS, fm[f]))
                ii = idx(f)
                fr[f][rows] = np.where((rows < fk[f])[:, None], rhs[ii[rows]], 0.0)
            elif op == S.SOP_FEXT:
                c, r0 = it[0], it[1]
                p = plan.f_parent[c]
                mp = plan.f_cmap[plan.f_cmap_off[c]:plan.f_cmap_off[c + 1]]
                rows = np.arange(r0, min(r0 + S.VEC_ROWS, len(mp)))
                fr[p][mp[rows]] += fr[c][fk[c] + rows]
            elif op == S.SOP_FPANEL:
                a, r0 = it[1], it[2]
                b = min(a + pw, fk[f])
                rows = slice(b + r0, min(b + r0 + S.TILE, fm[f]))
                fr[f][rows] += front(f)[rows, a:b] @ fr[f][a:b]
    for op, L, io, n, arg in plan.schedule["bwd"]:
        for it in work[io:io + n]:
            f = it[0]
            if op == S.SOP_BGATHER:
                r0 = it[1]
                rows = np.arange(r0, min(r0 + S.VEC_ROWS, fm[f]))
                fr[f][rows] = x[idx(f)[rows]]
            elif op == S.SOP_BPANEL:
                a = it[1]
                b = min(a + pw, fk[f])
                F = front(f)
                fr[f][a:b] = F[a:b, a:b] @ fr[f][a:b] + F[a:b, b:] @ fr[f][b:]
            elif op == S.SOP_BSCATTER:
                r0 = it[1]
                rows = np.arange(r0, min(r0 + S.VEC_ROWS, fk[f]))
                x[idx(f)[rows]] = fr[f][rows]
    return x
