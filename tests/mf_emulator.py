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
    R = plan.schedule["solve_rows"]
    fm, fk, off, io_ = plan.f_m, plan.f_k, plan.f_off, plan.f_idx_off
    J = rhs.shape[1]
    fr = np.zeros((int(io_[-1]), J))
    x = np.zeros_like(rhs)

    def front(f):
        m = int(fm[f])
        return st[off[f]:off[f] + m * m].reshape(m, m)

    def gathered(rows_abs, pivot_mask):
        val = np.where(pivot_mask[:, None], rhs[plan.f_idx[rows_abs]], 0.0)
        for s_ in range(S.MAX_GSRC):
            src = gsrc[rows_abs, s_]
            val = val + np.where((src >= 0)[:, None], fr[np.maximum(src, 0)], 0.0)
        return val

    for op, L, io, n, kmax in plan.schedule["fwd"]:
        assert op == S.SOP_FGEMM
        groups = {}
        for it in work[io:io + n]:
            f, r0, ks, slot = it
            base, k, m = io_[f], fk[f], fm[f]
            if r0 < 0:                            # pivot-only chunk [t0, t0 + R)
                t0 = -1 - r0
                t1 = min(k, t0 + R)
                fr[base + t0:base + t1] = gathered(base + np.arange(t0, t1), np.ones(t1 - t0, dtype=bool))
                continue
            kb = 0 if slot < 0 else ks * kmax          # split items: kmax is the level's split
            ke = k if slot < 0 else min(k, kb + kmax)
            assert ke - kb <= kmax
            piv = gathered(base + np.arange(kb, ke), np.ones(ke - kb, dtype=bool))
            if r0 == 0:
                fr[base + kb:base + ke] = piv
            rows = np.arange(k + r0, min(k + r0 + R, m))
            prod = front(f)[rows, kb:ke] @ piv
            if slot < 0:
                fr[base + rows] = gathered(base + rows, np.zeros(len(rows), dtype=bool)) - prod
            else:
                groups.setdefault((f, r0), []).append((ks, prod))
        for (f, r0), parts in groups.items():
            base, k, m = io_[f], fk[f], fm[f]
            rows = np.arange(k + r0, min(k + r0 + R, m))
            tot = sum(p_ for _, p_ in sorted(parts, key=lambda t: t[0]))
            fr[base + rows] = gathered(base + rows, np.zeros(len(rows), dtype=bool)) - tot
    for op, L, io, n, kmax in plan.schedule["bwd"]:
        assert op == S.SOP_BGEMM
        groups = {}
        for it in work[io:io + n]:
            f, r0, ks, slot = it
            base, k, m = io_[f], fk[f], fm[f]
            rows = np.arange(r0, min(r0 + R, k))
            bop = np.vstack([fr[base:base + k], x[plan.f_idx[base + k:base + m]]])
            kb = 0 if slot < 0 else ks * kmax
            ke = m if slot < 0 else min(m, kb + kmax)
            assert ke - kb <= kmax
            prod = front(f)[rows, kb:ke] @ bop[kb:ke]
            if slot < 0:
                x[plan.f_idx[base + rows]] = -prod
            else:
                groups.setdefault((f, r0), []).append((ks, prod))
        for (f, r0), parts in groups.items():
            base, k = io_[f], fk[f]
            rows = np.arange(r0, min(r0 + R, k))
            x[plan.f_idx[base + rows]] = -sum(p_ for _, p_ in sorted(parts, key=lambda t: t[0]))
    return x
