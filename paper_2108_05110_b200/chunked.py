"""Member-column chunking: a rank whose ensemble shard does not fit its GPU at once.

Columns are independent within a sub-step (`linalg.py:62-76`), so the J-dependent
work of a step runs chunk by chunk through one C-ABI context whose column count is
the chunk width Jc, while everything J-independent -- the two shared matrices, their
factorisation, the means and the eddy-viscosity maxima -- is computed once per step
from all chunks:

  1. member sums of every chunk, summed in chunk order   -> [allreduce SUM] -> means
  2. every chunk's element pass, eddy maxima max-combined -> [allreduce MAX]
  3. one assembly and (when the renewal rule asks) one factorisation
  4. per chunk: right-hand sides (element pass again), Dirichlet values, extrapolated
     initial iterate, column-batched Krylov solve, pressure epilogue.

The state is stored chunk-major: chunk c of a buffer set is its own (2, n_total, Jc)
member-minor block, so every kernel runs unchanged with J = Jc.  Step graphs are not
used (a chunked step is hundreds of milliseconds); results equal the unchunked engine
up to the J-dependent tiling of the kernels (tests/test_gpu_chunked.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from . import exchange as XC
from .engine import DeviceState, Engine, _dptr
from .ensemble import viscosity_stats


def per_column_bytes(hm, restart=2):
    """Device bytes one member column costs: both state buffer sets (iterate + pressures), and the
    chunk workspace (right-hand side, Krylov blocks for ``restart`` vectors, element buffer, front
    vectors, staging)."""
    ntot, npres, nt = hm.ntot, hm.npres, len(hm.e_nodes)
    n_idx = int(hm.plan.f_idx_off[-1])
    state = 8 * (2 * 2 * ntot + 2 * 2 * npres)
    work = 8 * (2 * ntot * (1 + 2 * restart + 3) + 2 * nt * 12 + 2 * n_idx)
    staging = 8 * (2 * hm.nvel + 2 * npres + 2 * ntot)     # reference-layout blocks + the import block
    return state, work + staging


def largest_divisor_at_most(n, cap):
    cap = max(1, min(n, cap))
    for d in range(cap, 0, -1):
        if n % d == 0:
            return d
    return 1


def plan_chunk(hm, J, device, restart=2, reserve_frac=0.12):
    """Chunk width for J local columns on ``device``: J when everything fits, else the largest
    divisor of J whose chunk workspace fits next to the full state and both systems' fronts."""
    free, total = torch.cuda.mem_get_info(device)
    budget = free - int(reserve_frac * total)
    fronts = 8 * 2 * hm.plan.front_storage
    state_col, work_col = per_column_bytes(hm, restart)
    if fronts + J * (state_col + work_col) <= budget:
        return J
    room = budget - fronts - J * state_col
    if room <= work_col:
        raise MemoryError(f"{J} member columns do not fit the device even one at a time "
                          f"(state {J * state_col / 1e9:.1f} GB + fronts {fronts / 1e9:.1f} GB)")
    return largest_divisor_at_most(J, room // work_col)


class ChunkedEngine(Engine):
    """Engine for J local members processed in chunks of Jc columns (see module docstring)."""

    supports_ahead = False   # (no step(then=...): a chunked step is many passes over the chunks)
    step_fetch = False       # (no step(fetch=True): states are downloaded chunk by chunk on demand)

    def __init__(self, disc, config, j0=0, J=None, chunk=None, device=None, comm=None, **opts):
        J = config.num_members if J is None else J
        if chunk is None or chunk < 1 or J % chunk:
            raise ValueError(f"chunk width {chunk} must divide the {J} local members")
        opts = dict(opts)
        opts["restart"] = min(opts.get("restart", 8), 2)   # lagged-preconditioner FGMRES needs 1-3 vectors
        super().__init__(disc, config, j0=j0, J=chunk, device=device, comm=comm, **opts)
        self.step_graphs = False
        self.Jc, self.J_local, self.nchunk = chunk, J, J // chunk
        from .engine import cost_model
        cm = cost_model(self.hm, chunk)
        self.rho = cm["t_factor"] / (self.nchunk * cm["t_iter"])   # an iteration runs once per chunk
        d = self.dev
        f64 = dict(dtype=torch.float64, device=d)
        st = viscosity_stats(config)
        lag_same = 0.5 * (st.nu_fluct + st.nu_m_fluct)
        lag_cross = 0.5 * (config.nu - config.nu_m)
        self.coef_c = []
        for c in range(self.nchunk):
            sl = slice(j0 + c * chunk, j0 + (c + 1) * chunk)
            self.coef_c.append(torch.as_tensor(np.concatenate([lag_same[sl], lag_cross[sl]])).to(d))
        ntot, npres = self.ntot, self.npres
        # chunk-major buffer sets; chunk 0 lives in the base engine's blocks
        self.Xc = [[self.X[b]] + [torch.zeros(2, ntot, chunk, **f64) for _ in range(self.nchunk - 1)]
                   for b in range(2)]
        self.Pqc = [[self.Pq[b]] + [torch.zeros(2, npres, chunk, **f64) for _ in range(self.nchunk - 1)]
                    for b in range(2)]
        self.maxsq_acc = torch.zeros_like(self.maxsq_ext)
        self.sums_part = torch.zeros_like(self.sums)
        self._cdata = {}

    # ------------------------------------------------------------------
    # state transfer (chunk by chunk, chunk-sized staging)
    # ------------------------------------------------------------------
    def load_state(self, v, w, q, r):
        g = self._staging()
        s = self.stream
        nv, Jc = self.nvel, self.Jc
        from .problems import RankOneMembers, member_rows
        v, w = (a if isinstance(a, RankOneMembers) else np.asarray(a, dtype=float) for a in (v, w))
        has_p = q is not None and np.asarray(q).size > 0
        cur = self.cur
        self._retire(cur)
        for c in range(self.nchunk):
            sl = slice(c * Jc, (c + 1) * Jc)
            with torch.cuda.stream(s):
                Xs = g["x_in"]
                nt, npr = self.ntot, self.npres
                for m, a in enumerate((v, w)):
                    self._copy_members(g["d_vel"][m], member_rows(a, c * Jc, Jc))   # lazy stays lazy
                N.check(self.lib.ens_layout_import(self.ctx, self.sptr, _dptr(g["d_vel"]), nv, Jc * nv, nv,
                                                   _dptr(g["row_v"]), _dptr(Xs), nt * Jc, 2), "ens_layout_import")
                if has_p:
                    for m, a in enumerate((q, r)):
                        g["d_pres"][m].copy_(self._host_tensor(np.asarray(a, float)[sl]))
                    N.check(self.lib.ens_layout_import(self.ctx, self.sptr, _dptr(g["d_pres"]), npr, Jc * npr, npr,
                                                       _dptr(g["row_p"]), _dptr(Xs[0, nv:]), nt * Jc, 2),
                            "ens_layout_import")
                else:
                    Xs[:, nv:] = 0.0
                self.Xc[cur][c].copy_(Xs)
                self.Pqc[cur][c].copy_(Xs[:, nv:])
            s.synchronize()
        self.gen[cur] += 1
        self.means_valid = False
        self.prev_valid = False

    def fields_to_host(self, buf):
        g = self._staging()
        s = self.stream
        Jc, nv, npr = self.Jc, self.nvel, self.npres
        out = {k: np.empty((self.J_local, nv if k in "vw" else npr)) for k in "vwqr"}
        for c in range(self.nchunk):
            sl = slice(c * Jc, (c + 1) * Jc)
            with torch.cuda.stream(s):
                nt = self.ntot
                N.check(self.lib.ens_layout_export(self.ctx, self.sptr, _dptr(self.Xc[buf][c]), nt * Jc, nv,
                                                   _dptr(g["row_v"]), _dptr(g["d_vel"]), nv, Jc * nv, 2),
                        "ens_layout_export")
                N.check(self.lib.ens_layout_export(self.ctx, self.sptr, _dptr(self.Pqc[buf][c]), npr * Jc, npr,
                                                   _dptr(g["row_p"]), _dptr(g["d_pres"]), npr, Jc * npr, 2),
                        "ens_layout_export")
            s.synchronize()
            out["v"][sl], out["w"][sl] = g["d_vel"][0].cpu().numpy(), g["d_vel"][1].cpu().numpy()
            out["q"][sl], out["r"][sl] = g["d_pres"][0].cpu().numpy(), g["d_pres"][1].cpu().numpy()
        return out

    def release(self):
        super().release()
        self.Xc = self.Pqc = None

    def state_handle(self):
        import weakref
        h = DeviceState(self, self.cur, self.gen[self.cur], self.J_local)
        self.live[self.cur] = weakref.ref(h)
        return h

    # ------------------------------------------------------------------
    # problem data per chunk
    # ------------------------------------------------------------------
    def _chunk_data(self, obj, kind, t, c):
        """ens_data_desc of chunk c (members j0 + c Jc ...) for loads / Dirichlet values at t."""
        hm, Jc = self.hm, self.Jc
        sl = slice(self.j0 + c * Jc, self.j0 + (c + 1) * Jc)
        dd = N.DataDesc()
        dd.rows = self.nvel if kind == "loads" else hm.nbdofs
        keep = []
        if hasattr(obj, "separable"):
            key = (kind, id(obj))
            if key not in self._cdata:
                sep = obj.separable(self.disc, self.config)
                basis = np.asarray(sep.basis, dtype=float).reshape(len(sep.basis), -1)
                if kind == "loads":
                    basis = basis[:, hm.ref_of_int[:self.nvel]]
                self._cdata[key] = (sep, torch.as_tensor(np.ascontiguousarray(basis)).to(self.dev), obj)
            sep, basis_t, _ = self._cdata[key]
            cv, cw = sep.coef(t)
            coef = np.stack([np.asarray(cv, float)[:, sl], np.asarray(cw, float)[:, sl]])
            coef_t = torch.as_tensor(np.ascontiguousarray(coef)).to(self.dev)
            dd.K, dd.basis, dd.coef, dd.dense = basis_t.shape[0], _dptr(basis_t), _dptr(coef_t), None
            keep += [basis_t, coef_t]
            return dd, keep
        if kind == "loads":
            lv, lw = obj.loads(t, self.disc, self.config)
            if lv is None and lw is None:
                return None, keep
            z = np.zeros((self.J_total, self.nvel))
            lv = z if lv is None else np.asarray(lv)
            lw = z if lw is None else np.asarray(lw)
            dense = np.stack([hm.vel_to_internal(lv[sl]), hm.vel_to_internal(lw[sl])])
        else:
            bv, bw = obj.values(t, self.disc, self.config)
            dense = np.stack([np.asarray(bv, float)[sl].T, np.asarray(bw, float)[sl].T])
        dense_t = torch.as_tensor(np.ascontiguousarray(dense)).to(self.dev)
        dd.K, dd.basis, dd.coef, dd.dense = 0, None, None, _dptr(dense_t)
        keep.append(dense_t)
        return dd, keep

    # ------------------------------------------------------------------
    # the chunked step
    # ------------------------------------------------------------------
    def _compute_means(self):
        lib, ctx, s = self.lib, self.ctx, self.sptr
        X = self.Xc[self.cur]
        for c in range(self.nchunk):
            dst = self.sums if c == 0 else self.sums_part
            N.check(lib.ens_member_sums(ctx, s, _dptr(X[c]), _dptr(dst)), "ens_member_sums")
            if c:
                self.sums.add_(self.sums_part)
        XC.allreduce_member_sums(self.sums, self.comm)
        N.check(lib.ens_means(ctx, s, _dptr(self.sums), 1.0 / self.J_total, _dptr(self.means)), "ens_means")
        self.means_valid = True

    def _element_pass(self, X, c, loads):
        N.check(self.lib.ens_rhs_fused(self.ctx, self.sptr, _dptr(X), _dptr(self.means), _dptr(self.coef_c[c]),
                                       1.0 / self.config.dt, C.byref(loads) if loads is not None else None,
                                       _dptr(self.rhs), _dptr(self.maxsq)), "ens_rhs_fused")

    def step(self, t_next, forcing, boundary):
        with self.on_stream():
            return self._step_chunked(t_next, forcing, boundary)

    def _step_chunked(self, t_next, forcing, boundary):
        lib, ctx, s = self.lib, self.ctx, self.sptr
        cur, nxt = self.cur, 1 - self.cur
        Xs, Xn = self.Xc[cur], self.Xc[nxt]
        self.flush_global()
        self._cost_begin()
        if not self.means_valid:
            self._compute_means()
        keep = []
        loads, bcs = [], []
        for c in range(self.nchunk):
            lo, k1 = self._chunk_data(forcing, "loads", t_next, c)
            bc, k2 = self._chunk_data(boundary, "bc", t_next, c)
            loads.append(lo)
            bcs.append(bc)
            keep += k1 + k2
        # eddy maxima over every chunk (the right-hand sides of this pass are recomputed per chunk below)
        nq = 2 * self.nt * 7
        for c in range(self.nchunk):
            self._element_pass(Xs[c], c, loads[c])
            if c == 0:
                self.maxsq_acc[:nq].copy_(self.maxsq_ext[:nq])
            else:
                torch.maximum(self.maxsq_acc[:nq], self.maxsq_ext[:nq], out=self.maxsq_acc[:nq])
        XC.allreduce_eddy_max(self.maxsq_acc[:nq], self.comm)
        self.maxsq_ext[:nq].copy_(self.maxsq_acc[:nq])
        N.check(lib.ens_assemble(ctx, s, _dptr(self.base), _dptr(self.means), _dptr(self.maxsq), self.two_mu_dt,
                                 _dptr(self.as_vals)), "ens_assemble")
        need = self._need_factor()
        if need:
            self._factor_timed()
        else:
            self.since_factor += 1
        self._retire(nxt)
        iters_max, rel_max = 0, [0.0, 0.0]
        for c in range(self.nchunk):
            self._element_pass(Xs[c], c, loads[c])
            N.check(lib.ens_apply_bc(ctx, s, C.byref(bcs[c]), _dptr(self.rhs)), "ens_apply_bc")
            if self.guess == "extrapolate" and self.prev_valid:
                N.check(lib.ens_lincomb(ctx, s, 2.0, _dptr(Xs[c]), -1.0, _dptr(Xn[c])), "ens_lincomb")
            else:
                Xn[c].copy_(Xs[c])
            code, iters, rel = self._solve(Xn[c])
            if code == N.ENS_ENOCONV and not need:      # stale preconditioner: rebuild, redo this chunk
                self._factor_timed()
                need = True
                Xn[c].copy_(Xs[c])
                code, iters2, rel = self._solve(Xn[c])
                iters += iters2
            self.last_relres = rel
            N.check(code, "ens_solve")
            N.check(lib.ens_epilogue(ctx, s, _dptr(Xn[c]), _dptr(self.Pqc[nxt][c])), "ens_epilogue")
            iters_max = max(iters_max, iters)
            rel_max = [max(rel_max[0], rel[0]), max(rel_max[1], rel[1])]
        del keep
        self.last_iters, self.last_relres = iters_max, tuple(rel_max)
        self.gen[nxt] += 1
        self.cur = nxt
        self.means_valid = False
        self.prev_valid = True
        renew = self._step_done(iters_max)
        self._nstep += 1
        if self.comm is None:
            self._renew = renew
            return max(self.last_relres)
        res, it, rn = XC.allreduce_max_values([max(self.last_relres), float(self.last_iters), float(bool(renew))],
                                              self.comm, self.dev)
        self._agreed(it)
        if self.refactor == "timed":
            self._renew = rn > 0.0
        return res

    def _diagnostics(self):
        if not self.means_valid:
            self._compute_means()
        Jc = self.Jc
        series = np.empty((6, self.J_local))
        energy = 0.0
        for c in range(self.nchunk):
            N.check(self.lib.ens_diagnostics(self.ctx, self.sptr, _dptr(self.Xc[self.cur][c]), _dptr(self.means),
                                             _dptr(self.diag_out)), "ens_diagnostics")
            out = self.diag_out.cpu().numpy()
            energy = 0.5 * (out[0] + out[1])
            series[:, c * Jc:(c + 1) * Jc] = out[2:].reshape(6, Jc)
        return dict(energy=energy, l2v=series[0], l2w=series[1], gradv=series[2], gradw=series[3],
                    div_v=np.sqrt(np.maximum(series[4], 0.0)), div_w=np.sqrt(np.maximum(series[5], 0.0)))
