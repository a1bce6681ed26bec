"""Device engine: uploads one mesh once, then runs time-steps through the C ABI.

One engine per (Discretization, local member count, device).  All per-step
data stays in HBM; the host only uploads tiny per-step coefficient tables
(problem data in separable form) and reads a handful of scalars.

Per time-step (reference `stepper.advance`, `stepper.py:360-394`):
  1. ens_member_sums            -> [allreduce SUM]   -> means  (ensemble.py:216-224)
  2. ens_rhs, ens_member_pass   -> [allreduce MAX of max_j |z'_j|^2]  (stepper.py:223-252,
                                                                       ensemble.py:227-238)
  3. ens_apply_bc               (stepper.py:250-251)
  4. ens_assemble               both shared velocity blocks (stepper.py:195-206)
  5. ens_factor                 multifrontal LU of both saddle matrices (linalg.py:79-108)
  6. ens_solve                  column-batched FGMRES, true residual (linalg.py:62-76, 111-118)
  7. ens_epilogue               mean-zero pressures (stepper.py:389-390)
The V and W sub-steps share every launch (2 matrices per grid), since they
depend on level-n data only (`stepper.py:363-366`).
"""

from __future__ import annotations

import ctypes as C
import os
import weakref
from collections import OrderedDict

import numpy as np
import scipy.sparse as sp
import torch

from . import _native as N
from . import exchange as XC
from . import fe
from . import symbolic as S
from .ensemble import viscosity_stats


_RENEW_DEBUG = os.environ.get("ENS_RENEW_DEBUG", "0") == "1"
MAX_PROBLEM_OBJECTS = 8   # forcing / boundary / exact objects whose device data and step graphs an engine keeps
RENEW_WINDOW = int(os.environ.get("ENS_RENEW_WINDOW", "6"))   # lifetimes a per-position cost stays usable
RENEW_STALE = int(os.environ.get("ENS_RENEW_STALE", str(4 * RENEW_WINDOW)))


# Cost model of the renewal rule, fitted to the round-2 kernels on B200: a
# factorisation costs a fixed latency per tree level plus its flops at an effective DMMA rate; an
# apply costs a latency per level and direction plus the larger of its bytes and flops terms.  The
# constants are fixed, so the rule built on them is a deterministic function of the plan, J and the
# iteration counts (fit: C2 6.84 / 0.47 ms, C3 36.6 / 4.9 ms, C4 7.65 / 2.7 ms factor / apply).
FACTOR_LEVEL_S = 0.257e-3      # per tree level (panel, update and extend-add launches)
RATE_FACTOR_FLOPS = 9.87e12    # sweep factorisation, fp64 DMMA
APPLY_LEVEL_S = 10e-6          # per tree level and sweep direction
RATE_APPLY_BYTES = 4.1e12      # preconditioner apply, algorithmic bytes
RATE_APPLY_FLOPS = 13.7e12     # preconditioner apply at large J (fp64 DMMA)
RATE_SPMM_BYTES = 1.39e12      # saddle SpMM, algorithmic bytes


def spmm_bytes(hm, J):
    """Algorithmic HBM bytes of one ens_spmm launch (both systems)."""
    ns, npres, ntot, nnz = hm.ns, hm.npres, hm.ntot, hm.nnz_s
    npairs = len(hm.b_col)
    per_mat = (12 * nnz + 4 * (ns + 1)            # A_s values + column indices + row pointers
               + 20 * npairs + 4 * (ns + 1)       # B^T (p, bx, by) by node
               + 20 * npairs + 4 * (npres + 1)    # B (node, bx, by) by pressure row
               + ntot                             # identity-row flags
               + 16 * ntot * J)                   # X read once, Y written once
    return 2 * per_mat


def apply_bytes(hm, J):
    """Algorithmic bytes of one preconditioner apply (both systems): factor entries read once per
    sweep direction pair, right-hand side / iterate traffic of the forward and backward sweeps."""
    nnz_lu = hm.plan.stats["nnz_lu"]
    return 2 * 8 * nnz_lu + 2 * 2 * 8 * hm.ntot * J * 2


def apply_flops(hm, J):
    return 2.0 * 2 * hm.plan.stats["nnz_lu"] * J


def cost_model(hm, J):
    """Modelled seconds of a factorisation and of one Krylov iteration (apply + SpMM), both systems."""
    nlev = hm.plan.nlevels
    t_f = nlev * FACTOR_LEVEL_S + 2 * hm.plan.stats["factor_flops"] / RATE_FACTOR_FLOPS
    t_apply = 2 * nlev * APPLY_LEVEL_S + max(apply_bytes(hm, J) / RATE_APPLY_BYTES,
                                             apply_flops(hm, J) / RATE_APPLY_FLOPS)
    t_it = t_apply + spmm_bytes(hm, J) / RATE_SPMM_BYTES
    return dict(t_factor=t_f, t_iter=t_it, rho=t_f / t_it)


def _dptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _color_elements(cell_dofs: np.ndarray, ns: int) -> np.ndarray:
    """Greedy element colouring: elements sharing a P2 node get different colours."""
    node_mask = np.zeros(ns, dtype=np.int64)
    colors = np.empty(len(cell_dofs), dtype=np.int64)
    cd = cell_dofs.tolist()
    nm = node_mask.tolist()
    for e, nodes in enumerate(cd):
        used = 0
        for n in nodes:
            used |= nm[n]
        c = 0
        while used >> c & 1:
            c += 1
        colors[e] = c
        bit = 1 << c
        for n in nodes:
            nm[n] |= bit
    return colors


class HostMesh:
    """All host-side arrays of one mesh in the engine's internal numbering (built once)."""

    def __init__(self, disc):
        self.disc = disc
        vel, pres = disc.velocity, disc.pressure
        ns, npres, nvel = disc.n_scalar, disc.n_pres, disc.n_vel
        self.ns, self.npres, self.nvel, self.ntot = ns, npres, nvel, nvel + npres
        plan = S.analyse(disc)
        self.plan = plan
        nperm, pperm = plan.node_perm, plan.pres_perm
        # internal row of every reference dof, and the inverse
        int_id = np.empty(self.ntot, dtype=np.int64)
        int_id[:ns] = 2 * nperm
        int_id[ns:nvel] = 2 * nperm + 1
        int_id[nvel:] = nvel + pperm
        self.int_id = int_id
        self.ref_of_int = np.empty_like(int_id)
        self.ref_of_int[int_id] = np.arange(self.ntot)
        # scalar operators in internal node order
        P = sp.csr_matrix((np.ones(ns), (nperm, np.arange(ns))), shape=(ns, ns))
        pat = fe.scalar_pattern(vel)
        ipat = (P @ pat @ P.T).tocsr()
        ipat.sort_indices()
        self.s_rowptr = ipat.indptr.astype(np.int32)
        self.s_col = ipat.indices.astype(np.int32)
        self.nnz_s = ipat.nnz

        def aligned(mat):
            m2 = (P @ mat @ P.T).tocsr()
            m2.sort_indices()
            out = np.zeros(self.nnz_s)
            # map values by (row, col) -> slot
            rows = np.repeat(np.arange(ns), np.diff(m2.indptr))
            slot = self._slot(rows, m2.indices)
            out[slot] = m2.data
            return out

        self.s_mass = aligned(disc.mass_s)
        self.s_stiff = aligned(disc.stiff_s)
        # the plan indexes A_s values in the reference pattern order; the device
        # stores them in internal order -> remap those source indices once
        ref_rows = np.repeat(np.arange(ns), np.diff(pat.indptr))
        ref_to_int_slot = self._slot(nperm[ref_rows], nperm[pat.indices])
        src = plan.orig_src.astype(np.int64)
        is_a = src < self.nnz_s
        src[is_a] = ref_to_int_slot[src[is_a]]
        self.orig_src = src.astype(np.int32)
        # B by pressure row and B^T by node, (bx, by) pairs on one pattern
        bip, bcol, bx, by = fe.divergence_pair(vel, pres)
        brow = np.repeat(np.arange(npres), np.diff(bip))
        r_int, c_int = pperm[brow], nperm[bcol]
        o = S.host_argsort(r_int * (ns + 1) + c_int)         # == lexsort((c_int, r_int))
        self.b_rowptr = np.concatenate([[0], np.cumsum(np.bincount(r_int, minlength=npres))]).astype(np.int32)
        self.b_col = c_int[o].astype(np.int32)
        self.b_val = np.stack([bx[o], by[o]], axis=1).ravel()
        o2 = S.host_argsort(c_int * (npres + 1) + r_int)     # == lexsort((r_int, c_int))
        self.bt_rowptr = np.concatenate([[0], np.cumsum(np.bincount(c_int, minlength=ns))]).astype(np.int32)
        self.bt_col = r_int[o2].astype(np.int32)
        self.bt_val = np.stack([bx[o2], by[o2]], axis=1).ravel()
        # identity rows
        cons_ref = disc.constrained_rows
        self.cflag = np.zeros(self.ntot, dtype=np.uint8)
        self.cflag[int_id[cons_ref]] = 1
        nb = disc.bdofs.size
        self.cons_row = int_id[cons_ref].astype(np.int32)
        self.cons_bidx = np.concatenate([np.arange(nb), -np.ones(len(cons_ref) - nb)]).astype(np.int32)
        self.nbdofs = nb
        # elements, coloured
        colors = _color_elements(vel.cell_dofs, ns)
        inodes = nperm[vel.cell_dofs]
        eorder = np.lexsort((inodes.min(axis=1), colors))
        self.ncolor = int(colors.max()) + 1
        self.color_off = np.searchsorted(colors[eorder], np.arange(self.ncolor + 1)).astype(np.int32)
        self.e_nodes = inodes[eorder].astype(np.int32)
        geo = np.zeros((len(eorder), 8))
        geo[:, 0] = vel.areas[eorder]
        geo[:, 1:7] = vel.grad_lam[eorder].reshape(-1, 6)
        self.e_geo = geo.ravel()
        a_idx = np.repeat(self.e_nodes, 6, axis=1)
        b_idx = np.tile(self.e_nodes, (1, 6))
        self.e_slots = self._slot(a_idx.ravel(), b_idx.ravel()).astype(np.int32)
        self.eorder = eorder
        # gather lists for the scatter-free member pass / assembly (fixed element order)
        nt = len(self.e_nodes)
        en = self.e_nodes.ravel()
        o = S.host_argsort(en)                                          # stable
        self.n2e = o.astype(np.int32)                                   # e*6 + a
        self.n2e_ptr = np.concatenate([[0], np.cumsum(np.bincount(en, minlength=ns))]).astype(np.int32)
        o = S.host_argsort(self.e_slots)
        self.s2e = ((o % 36) * nt + o // 36).astype(np.int32)          # ab*nt + e
        self.s2e_ptr = np.concatenate([[0], np.cumsum(np.bincount(self.e_slots, minlength=self.nnz_s))]).astype(np.int32)
        self.pres_int = np.empty(npres)
        self.pres_int[pperm] = disc.pressure_integrals
        self._allkey = None                                             # slot-lookup keys: setup only

    def _slot(self, rows, cols):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        key = rows * (self.ns + 1) + cols
        if getattr(self, "_allkey", None) is None:
            allrows = np.repeat(np.arange(self.ns, dtype=np.int64), np.diff(self.s_rowptr))
            self._allkey = allrows * (self.ns + 1) + self.s_col
        allkey = self._allkey
        pos = S.host_searchsorted(allkey, key)
        assert np.all(allkey[np.minimum(pos, allkey.size - 1)] == key), "slot lookup failed"
        return pos

    # host <-> internal conversions (numpy)
    def vel_to_internal(self, arr_ref):
        """(J, n_vel) reference order -> (n_vel, J) internal order."""
        return np.ascontiguousarray(np.asarray(arr_ref, dtype=float).T[self.ref_of_int[:self.nvel]])

    def pres_to_internal(self, arr_ref):
        return np.ascontiguousarray(np.asarray(arr_ref, dtype=float).T[self.ref_of_int[self.nvel:] - self.nvel])


def host_mesh(disc) -> HostMesh:
    """The mesh's HostMesh, built once per Discretization (large meshes: through the on-disk
    setup cache, setup_cache.py)."""
    key = "b200-hostmesh"
    if key not in disc._cache:
        from . import setup_cache
        disc._cache[key] = setup_cache.host_mesh(disc)
    return disc._cache[key]


class DeviceState:
    """Handle on one engine buffer set; materialises numpy on demand."""

    def __init__(self, engine, buf, gen, num_members):
        self.engine = engine
        self.buf = buf
        self.gen = gen
        self.num_members = num_members
        self._host = {}
        self._pending = None      # (pinned tensors, event): a download enqueued by the step itself

    @property
    def valid(self):
        return self.engine is not None and self.engine.gen[self.buf] == self.gen

    def materialize(self):
        for name in "vwqr":
            self.to_host(name)
        self.engine = None

    def to_host(self, name):
        if name in self._host:
            return self._host[name]
        if self._pending is None and not self.valid:
            raise RuntimeError("device state was overwritten before it was read")
        if self._pending is None and not getattr(self.engine, "step_fetch", False):
            fields = self.engine.fields_to_host(self.buf)     # (chunked engine: chunk by chunk)
        else:
            if self._pending is not None:
                # enqueued behind the step that produced this state: it holds the state's values even if
                # the device buffers have been overwritten since
                (tens, ev), self._pending = self._pending, None
            else:
                tens, ev = self.engine._enqueue_fetch(self.buf)   # all four fields, one wait
            fields = {k: t.numpy() for k, t in tens.items()}      # (views: built while the copies are in flight)
            for a in fields.values():
                a.setflags(write=False)
            ev.synchronize()
            if self.engine is not None:
                # (load_state recognises these arrays if the caller passes them straight back in)
                self.engine._handed = ((self.buf, self.gen), tens)
        for a in fields.values():
            # an EnsembleState is immutable (`ensemble.py:183-190`): a caller editing a returned field in
            # place would otherwise be silently ignored by a device-resident next step
            a.setflags(write=False)
        self._host.update(fields)
        return self._host[name]


class Engine:
    """Device-resident ensemble on one GPU (member columns [j0, j0+J) of J_total)."""

    step_fetch = True      # step(fetch=True) is supported (the chunked engine downloads on demand)
    _fetched = None        # (pinned tensors, event, (buffer, generation)) of the last step(fetch=True)
    _handed = None         # ((buffer, generation), pinned tensors) last handed out as write-protected arrays
    n_own_uploads = 0      # load_state calls that recognised their own handed-out arrays (no comparison, no sync)

    def __init__(self, disc, config, j0=0, J=None, device=None, comm=None, restart=8, max_restarts=20, rtol=1e-12,
                 refactor="adaptive", lag_max_iters=8, lag_max_steps=500, guess="extrapolate"):
        """``refactor``: "always" rebuilds the LU preconditioner every step (the
        reference refactorises every sub-step, `stepper.py:216`); "adaptive"
        keeps the last factorisation until the deterministic renewal rule
        (``_renewal``: iteration counts against the modelled factorisation cost)
        fires, FGMRES needs more than ``lag_max_iters`` iterations, or
        ``lag_max_steps`` steps have passed; "timed" is "adaptive" with the rule fed
        by measured device times (``_cost_end``; not reproducible run to run).
        Whatever the policy every solve is converged to the same true residual
        ``rtol`` on the *current* matrix.

        ``guess``: FGMRES initial iterate -- "extrapolate" (2 x^n - x^{n-1} when
        the previous level is resident, an O(dt^2) guess that usually saves one
        preconditioned iteration) or "previous" (x^n)."""
        if refactor not in ("always", "adaptive", "timed"):
            raise ValueError("refactor must be 'always', 'adaptive' or 'timed'")
        if guess not in ("extrapolate", "previous"):
            raise ValueError("guess must be 'extrapolate' or 'previous'")
        self.guess = guess
        self.prev_valid = False   # buffer 1-cur holds level n-1 of the current trajectory
        self.refactor, self.lag_max_iters, self.lag_max_steps = refactor, lag_max_iters, lag_max_steps
        self.factored = False
        self.since_factor = 0
        self.n_factor = 0
        self._renew = False        # renewal rule fired (adaptive policy), agreed over ranks
        self._ev = None            # step / factorisation CUDA events of the renewal rule
        self._cyc = None           # [factorisation ms, step ms since, steps since]
        self._prof = []            # [step ms, lifetime] by position within a factorisation's lifetime
        self._life = 0             # factorisations so far
        self._lk = None            # iteration counts of the current factorisation's lifetime
        self._pending = None       # sharded: renewal waiting for the agreed iteration count
        self._fac_this = False
        self.pivoting = False
        if not torch.cuda.is_available():
            raise RuntimeError("the B200 time-step engine needs a CUDA device (no CPU fallback)")
        self.lib = N.load()
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.hm = hm = host_mesh(disc)
        self.disc = disc
        self.J_total = config.num_members
        self.j0 = j0
        self.J = J = self.J_total if J is None else J
        self.rho = cost_model(hm, J)["rho"]
        self.comm = comm
        self.restart, self.max_restarts, self.rtol = restart, max_restarts, rtol
        self.ntot, self.nvel, self.npres = hm.ntot, hm.nvel, hm.npres
        d = self.dev
        f64 = dict(dtype=torch.float64, device=d)

        def up(a, dtype):
            return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(d)

        i32, i64 = torch.int32, torch.int64
        self._keep = []
        mesh_t = dict(
            s_rowptr=up(hm.s_rowptr, i32), s_col=up(hm.s_col, i32), s_mass=up(hm.s_mass, torch.float64),
            s_stiff=up(hm.s_stiff, torch.float64), bt_rowptr=up(hm.bt_rowptr, i32), bt_col=up(hm.bt_col, i32),
            bt_val=up(hm.bt_val, torch.float64), b_rowptr=up(hm.b_rowptr, i32), b_col=up(hm.b_col, i32),
            b_val=up(hm.b_val, torch.float64), cflag=up(hm.cflag, torch.uint8), e_nodes=up(hm.e_nodes, i32),
            e_geo=up(hm.e_geo, torch.float64), e_slots=up(hm.e_slots, i32),
            cons_row=up(hm.cons_row if len(hm.cons_row) else np.zeros(1, np.int32), i32),
            cons_bidx=up(hm.cons_bidx if len(hm.cons_bidx) else np.zeros(1, np.int32), i32),
            pres_int=up(hm.pres_int, torch.float64), n2e_ptr=up(hm.n2e_ptr, i32), n2e=up(hm.n2e, i32),
            s2e_ptr=up(hm.s2e_ptr, i32), s2e=up(hm.s2e, i32))
        self.mesh_t = mesh_t
        self._color_off = np.ascontiguousarray(hm.color_off, dtype=np.int32)
        md = N.MeshDesc()
        md.ns, md.n_pres, md.nt, md.nnz_s, md.J = hm.ns, hm.npres, len(hm.e_nodes), hm.nnz_s, J
        md.ncolor, md.ncons = hm.ncolor, len(hm.cons_row)
        for k, t in mesh_t.items():
            setattr(md, k, _dptr(t))
        md.color_off_host = self._color_off.ctypes.data
        md.area = float(disc.area)
        md.mean_zero = 1 if disc.pin_pressure else 0
        self.nt = md.nt
        p = hm.plan
        plan_t = dict(
            f_m=up(p.f_m, i32), f_k=up(p.f_k, i32), f_off=up(p.f_off, i64), f_idx_off=up(p.f_idx_off, i64),
            f_idx=up(p.f_idx, i32), f_parent=up(p.f_parent, i32), f_cmap_off=up(p.f_cmap_off, i64),
            f_cmap=up(p.f_cmap if len(p.f_cmap) else np.zeros(1, np.int32), i32), orig_dst=up(p.orig_dst, i64),
            orig_src=up(hm.orig_src, i32), bsrc_vals=up(p.bsrc_vals, torch.float64),
            work=up(p.schedule["work"].ravel() if p.schedule["work"].size else np.zeros(4, np.int32), i32),
            gsrc=up(p.schedule["gsrc"].ravel(), i32))
        self.plan_t = plan_t
        self._host_keep = dict(
            orig_level_off=np.ascontiguousarray(p.orig_level_off, dtype=np.int64),
            level_storage_off=np.ascontiguousarray(p.level_storage_off, dtype=np.int64),
            level_front_off=np.ascontiguousarray(p.level_front_off, dtype=np.int32),
            factor=np.ascontiguousarray(p.schedule["factor"], dtype=np.int64),
            fwd=np.ascontiguousarray(p.schedule["fwd"], dtype=np.int64),
            bwd=np.ascontiguousarray(p.schedule["bwd"], dtype=np.int64))
        pd = N.PlanDesc()
        pd.nfront, pd.nlevels, pd.pw, pd.tile = p.nfront, p.nlevels, S.PW, S.TILE
        pd.front_storage, pd.n_orig = p.front_storage, len(p.orig_dst)
        pd.n_cmap, pd.n_idx, pd.n_work = len(p.f_cmap), int(p.f_idx_off[-1]), len(p.schedule["work"])
        for k, t in plan_t.items():
            setattr(pd, k, _dptr(t))
        hk = self._host_keep
        pd.orig_level_off_host = hk["orig_level_off"].ctypes.data
        pd.level_storage_off_host = hk["level_storage_off"].ctypes.data
        pd.level_front_off_host = hk["level_front_off"].ctypes.data
        pd.sched_factor_host, pd.n_sched_factor = hk["factor"].ctypes.data, len(hk["factor"])
        pd.sched_fwd_host, pd.n_sched_fwd = hk["fwd"].ctypes.data, len(hk["fwd"])
        pd.sched_bwd_host, pd.n_sched_bwd = hk["bwd"].ctypes.data, len(hk["bwd"])
        pd.max_m = int(p.f_m.max())
        pd.split_k = int(p.schedule.get("split_k", S.SPLIT_K))
        pd.n_slot = int(p.schedule["nslot"])
        self._md, self._pd = md, pd
        ctx = C.c_void_p()
        with torch.cuda.device(self.dev):
            N.check(self.lib.ens_create(C.byref(md), C.byref(pd), self.dev.index, C.byref(ctx)), "ens_create")
        self.ctx = ctx
        # per-run constants
        st = viscosity_stats(config)
        self.config = config
        base = hm.s_mass / config.dt + 0.5 * (st.nu_bar + st.nu_m_bar) * hm.s_stiff
        self.base = up(base, torch.float64)
        lag_same = 0.5 * (st.nu_fluct + st.nu_m_fluct)
        lag_cross = 0.5 * (config.nu - config.nu_m)
        sl = slice(j0, j0 + J)
        self.member_coef = up(np.concatenate([lag_same[sl], lag_cross[sl]]), torch.float64)
        self.two_mu_dt = 2.0 * config.mu * config.dt
        if not (config.mu > 0.0):
            raise ValueError("mu and dt must be positive")
        # buffers
        ntot, nvel = self.ntot, self.nvel
        self.X = [torch.zeros(2, ntot, J, **f64), torch.zeros(2, ntot, J, **f64)]
        self.Pq = [torch.zeros(2, self.npres, J, **f64), torch.zeros(2, self.npres, J, **f64)]
        self.gen = [0, 0]
        self.live = [None, None]
        self.cur = 0
        # per-step work buffers (right-hand sides, member sums / means, eddy maxima, assembled A_s
        # values): one set, or -- once a time loop announces its steps (step(then=...)) -- one per
        # state-buffer parity, so that the next step's pre-solve graph can be enqueued while this
        # step's solve may still need its own right-hand sides and matrix values (_enable_ahead)
        self._f64 = f64
        self._wb = [self._work_set(), None]
        self.means_valid = False
        # (eddy maxima of both families, plus a 3-double tail on which the sharded step sends the
        # previous step's (residual, iterations, renewal flag) through the same MAX exchange)
        self._tail = self._wb[0]["maxsq_ext"][2 * self.nt * 7:]
        self._tail_in = torch.zeros(3, dtype=torch.float64, pin_memory=True)
        self._tail_out = torch.zeros(3, dtype=torch.float64, pin_memory=True)
        self._tail_ev = torch.cuda.Event()
        self._prev_local = None        # (residual, iterations, renew) of the last step, this rank
        self._nstep = 0
        self.global_residuals = {}     # engine step index -> residual max over ranks (sharded runs)
        self.diag_out = torch.zeros(2 + 6 * J, **f64)
        # a dedicated (non-default) stream: the factorisation and solve sequences
        # are captured once into CUDA graphs, which needs a capturable stream
        self.stream = torch.cuda.Stream(self.dev)
        torch.cuda.synchronize(self.dev)
        self._data_cache = {}
        self.last_iters = 0
        self.last_pert = 0
        self.last_relres = (0.0, 0.0)
        # whole-step CUDA graphs (ENS_STEP_GRAPH=0 disables): per buffer parity and problem,
        # the pre-solve sequence and the solve's first cycle + epilogue, replayed every step
        self.step_graphs = os.environ.get("ENS_STEP_GRAPH", "1") != "0"
        self.rhs_fused = os.environ.get("ENS_RHS_FUSED", "1") != "0"
        self._graphs = {}
        self._gdata_cache = {}
        self._lru = OrderedDict()        # problem-data objects with cached device data, least recent first
        self._gspec = {}
        self._spec = None              # pre-solve graph of the announced next step already enqueued (step(then=))
        self._ones = 0                 # consecutive steps whose solve converged in its first cycle
        self.graph_launch_credit = 0   # kernels replayed by step graphs minus kernels captured

    def _work_set(self):
        f64, J = self._f64, self.J
        return dict(rhs=torch.zeros(2, self.ntot, J, **f64), sums=torch.zeros(2 * self.nvel, **f64),
                    means=torch.zeros(2 * self.nvel, **f64), maxsq_ext=torch.zeros(2 * self.nt * 7 + 3, **f64),
                    as_vals=torch.zeros(2, self.hm.nnz_s, **f64))

    def _wset(self):
        w = self._wb[self.cur]
        return w if w is not None else self._wb[0]

    rhs = property(lambda self: self._wset()["rhs"])
    sums = property(lambda self: self._wset()["sums"])
    means = property(lambda self: self._wset()["means"])
    maxsq_ext = property(lambda self: self._wset()["maxsq_ext"])
    as_vals = property(lambda self: self._wset()["as_vals"])
    maxsq = property(lambda self: self._wset()["maxsq_ext"][:2 * self.nt * 7].view(2, self.nt, 7))

    def _enable_ahead(self):
        """Second work-buffer set (and per-parity data blocks / step graphs) for announced steps."""
        torch.cuda.synchronize(self.dev)
        self._wb[1] = self._work_set()
        for k, v in self._wb[0].items():
            self._wb[1][k].copy_(v)
        self._graphs.clear()
        self._gdata_cache.clear()
        self._gspec.clear()

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                self.lib.ens_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    @property
    def sptr(self):
        return C.c_void_p(self.stream.cuda_stream)

    # ------------------------------------------------------------------
    # state upload / download
    # ------------------------------------------------------------------
    def _staging(self):
        """Pinned host + device staging (reference layout) and the permutations, allocated once."""
        if getattr(self, "_stg", None) is None:
            hm, J, d = self.hm, self.J, self.dev
            self._stg = dict(
                d_vel=torch.empty(2, J, self.nvel, dtype=torch.float64, device=d),
                d_pres=torch.empty(2, J, self.npres, dtype=torch.float64, device=d),
                x_in=torch.empty(2, self.ntot, J, dtype=torch.float64, device=d),
                # row maps of the layout kernels (ens_layout_import / _export): internal row of each reference dof
                row_v=torch.as_tensor(hm.int_id[:self.nvel].astype(np.int64)).to(d),
                row_p=torch.as_tensor((hm.int_id[self.nvel:] - self.nvel).astype(np.int64)).to(d))
        return self._stg

    @staticmethod
    def _host_tensor(a):
        """torch view of a (J, n) float64 host array (no copy when already contiguous float64; read
        only -- states a step returns are write-protected host views)."""
        arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
        if not arr.flags.writeable:
            import warnings
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", UserWarning)
                return torch.from_numpy(arr)
        return torch.from_numpy(arr)

    def _copy_members(self, dst, a):
        """dst (J, n) on the device <- a (J, n) member array.  A RankOneMembers (amp x base) is
        expanded on the device -- the same IEEE products as np.outer -- so only amp and base cross
        PCIe; anything else is copied from host memory.  Returns the host tensor to keep alive
        until the copy completes (None for the device expansion)."""
        from .problems import RankOneMembers
        if isinstance(a, RankOneMembers):
            amp = torch.from_numpy(np.ascontiguousarray(a.amp)).to(dst.device)
            base = torch.from_numpy(np.ascontiguousarray(a.base)).to(dst.device)
            torch.mul(amp[:, None], base[None, :], out=dst)
            return None
        h = self._host_tensor(a)
        dst.copy_(h, non_blocking=h.is_pinned())
        return h

    def load_state(self, v, w, q, r):
        """Upload a host state (reference layout, this rank's members) into the current buffer set.

        H2D copies of the (J, n) arrays -- straight from the caller's buffers
        when they are pinned (e.g. the arrays a previous step returned), else
        from pageable memory -- then the member-minor transpose and the internal
        dof permutation on the device.  When the uploaded velocities equal the
        ones already resident in the current buffer set (a caller passing a
        step's output straight back in), the resident trajectory is kept, so the
        extrapolated initial iterate stays available, and q, r are not uploaded:
        the reference's step reads only v and w (`stepper.py:360-394`); the
        pressures enter here only as part of the initial iterate.
        """
        spec, self._spec = self._spec, None
        g = self._staging()
        s = self.stream
        nv = self.nvel
        own = self._own_arrays(v, w)
        if own is not None:
            if spec is not None:
                s.synchronize()     # (an announced step's graph is still enqueued: as for any dropped announcement)
            # the caller passes back, unmodified (write-protected views of our pinned buffers), the very
            # arrays this buffer set was downloaded into: same values by construction.  They are
            # uploaded and become the resident velocities like any caller's arrays, but nothing has to
            # be compared, so no host synchronisation: the step's graphs queue up behind the copies.
            self.n_own_uploads += 1
            # (one C call: two asynchronous copies from the pinned buffers + the layout kernel, on the engine stream)
            N.check(self.lib.ens_state_upload(self.ctx, self.sptr, own["v"].data_ptr(), own["w"].data_ptr(), nv,
                                              _dptr(g["d_vel"]), _dptr(g["row_v"]), _dptr(self.X[self.cur]),
                                              self.ntot * self.J), "ens_state_upload")
            return
        has_p = q is not None and np.asarray(q).size > 0
        with torch.cuda.stream(s):
            hv = self._copy_members(g["d_vel"][0], v)
            hw = self._copy_members(g["d_vel"][1], w)
            Xs = g["x_in"]
            J, nt = self.J, self.ntot
            N.check(self.lib.ens_layout_import(self.ctx, self.sptr, _dptr(g["d_vel"]), nv, J * nv, nv,
                                               _dptr(g["row_v"]), _dptr(Xs), nt * J, 2), "ens_layout_import")
            cur = self.cur
            same = self.gen[cur] > 0 and torch.equal(Xs[:, :nv], self.X[cur][:, :nv])
        keep = (hv, hw)
        if same:
            # the velocities are the resident level: the step needs nothing else from the host
            # (pressures enter a step only through the initial iterate, stepper.py:223-252), so
            # the resident trajectory -- pressures included -- is kept and q, r are not uploaded
            s.synchronize()      # caller buffers may be reused once we return
            del keep
            return
        with torch.cuda.stream(s):
            if has_p:
                hq, hr = self._host_tensor(q), self._host_tensor(r)
                keep = keep + (hq, hr)
                g["d_pres"][0].copy_(hq, non_blocking=hq.is_pinned())
                g["d_pres"][1].copy_(hr, non_blocking=hr.is_pinned())
                npr = self.npres
                N.check(self.lib.ens_layout_import(self.ctx, self.sptr, _dptr(g["d_pres"]), npr, J * npr, npr,
                                                   _dptr(g["row_p"]), _dptr(Xs[0, nv:]), nt * J, 2),
                        "ens_layout_import")
            else:
                Xs[:, nv:] = 0.0
        self._retire(cur)
        with torch.cuda.stream(s):
            self.X[cur].copy_(Xs)
            self.Pq[cur].copy_(Xs[:, nv:])
        s.synchronize()
        del keep
        self.gen[cur] += 1
        self.means_valid = False
        self.prev_valid = False

    def _enqueue_fetch(self, buf):
        """Enqueue the download of buffer set ``buf``: two layout kernels (internal member-minor
        blocks -> reference-order (J, n) staging), then four D2H copies straight into freshly
        allocated pinned buffers.  Returns ({v, w, q, r} pinned tensors, event after the last copy)."""
        g = self._staging()
        J, nv, npr, nt = self.J, self.nvel, self.npres, self.ntot
        out = {}
        with torch.cuda.stream(self.stream):
            N.check(self.lib.ens_layout_export(self.ctx, self.sptr, _dptr(self.X[buf]), nt * J, nv, _dptr(g["row_v"]),
                                               _dptr(g["d_vel"]), nv, J * nv, 2), "ens_layout_export")
            N.check(self.lib.ens_layout_export(self.ctx, self.sptr, _dptr(self.Pq[buf]), npr * J, npr,
                                               _dptr(g["row_p"]), _dptr(g["d_pres"]), npr, J * npr, 2),
                    "ens_layout_export")
            for m, name in ((0, "v"), (1, "w")):
                h = torch.empty(J, nv, dtype=torch.float64, pin_memory=True)
                h.copy_(g["d_vel"][m], non_blocking=True)
                out[name] = h
            for m, name in ((0, "q"), (1, "r")):
                h = torch.empty(J, npr, dtype=torch.float64, pin_memory=True)
                h.copy_(g["d_pres"][m], non_blocking=True)
                out[name] = h
            ev = torch.cuda.Event()
            ev.record(self.stream)
        return out, ev

    def _own_arrays(self, v, w):
        """The pinned tensors behind (v, w) when these are exactly the write-protected arrays handed out
        for the current buffer set and generation (``DeviceState.to_host``); else None."""
        h = self._handed
        if h is None or h[0] != (self.cur, self.gen[self.cur]):
            return None
        tens = h[1]
        for a, t in ((v, tens["v"]), (w, tens["w"])):
            if not (isinstance(a, np.ndarray) and not a.flags.writeable and a.dtype == np.float64
                    and a.shape == tuple(t.shape) and a.flags.c_contiguous
                    and a.__array_interface__["data"][0] == t.data_ptr()):
                return None
        return tens

    def fields_to_host(self, buf):
        """{v, w, q, r}: (J, n) reference-layout numpy arrays of buffer set ``buf``.

        One layout kernel per field pair (hand-written transpose + dof permutation), D2H straight
        into freshly allocated pinned buffers (the returned arrays are views of them -- no host
        copy, and a later upload of the same arrays is a direct DMA), one wait.
        """
        out, ev = self._enqueue_fetch(buf)
        ev.synchronize()
        return {k: t.numpy() for k, t in out.items()}

    def field_to_host(self, buf, name):
        """(J, n) reference-layout numpy copy of one field of buffer set ``buf``."""
        return self.fields_to_host(buf)[name]

    def state_handle(self):
        h = DeviceState(self, self.cur, self.gen[self.cur], self.J)
        self.live[self.cur] = weakref.ref(h)
        pre, self._fetched = getattr(self, "_fetched", None), None
        if pre is not None and pre[2] == (self.cur, self.gen[self.cur]):
            h._pending = pre[:2]          # this state's download is already on its way (step(fetch=True))
        return h

    def _retire(self, buf):
        ref = self.live[buf]
        if ref is not None:
            h = ref()
            if h is not None and h.engine is self and h.gen == self.gen[buf]:
                h.materialize()
        self.live[buf] = None

    # ------------------------------------------------------------------
    # problem data
    # ------------------------------------------------------------------
    def _data(self, obj, kind, t):
        """ens_data_desc for loads ('loads') or Dirichlet values ('bc') at time t."""
        hm, J, sl = self.hm, self.J, slice(self.j0, self.j0 + self.J)
        rows = self.nvel if kind == "loads" else hm.nbdofs
        sep = None
        if hasattr(obj, "separable"):
            # keyed by id(obj); the entry keeps obj alive, so the id cannot be reused by another object
            self._touch(obj)
            key = (kind, id(obj))
            if key not in self._data_cache:
                s = obj.separable(self.disc, self.config)
                basis = np.asarray(s.basis, dtype=float).reshape(len(s.basis), -1)
                if kind == "loads":
                    basis = basis[:, hm.ref_of_int[:self.nvel]]
                self._data_cache[key] = (s, torch.as_tensor(np.ascontiguousarray(basis)).to(self.dev), obj)
            sep = self._data_cache[key][:2]
        dd = N.DataDesc()
        dd.rows = rows
        keep = []
        if sep is not None:
            s, basis_t = sep
            cv, cw = s.coef(t)
            coef = np.stack([np.asarray(cv, float)[:, sl], np.asarray(cw, float)[:, sl]])
            coef_t = torch.as_tensor(np.ascontiguousarray(coef)).to(self.dev, non_blocking=True)
            dd.K, dd.basis, dd.coef, dd.dense = basis_t.shape[0], _dptr(basis_t), _dptr(coef_t), None
            keep += [basis_t, coef_t]
        else:
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
    # the time-step
    # ------------------------------------------------------------------
    class _OnStream:
        """Run on the engine stream, ordered after / before the caller's stream."""

        def __init__(self, eng):
            self.eng = eng

        def __enter__(self):
            caller = torch.cuda.current_stream(self.eng.dev)
            self.caller = caller
            self.eng.stream.wait_stream(caller)
            self.ctx = torch.cuda.stream(self.eng.stream)
            self.ctx.__enter__()

        def __exit__(self, *exc):
            self.ctx.__exit__(*exc)
            self.caller.wait_stream(self.eng.stream)
            return False

    def on_stream(self):
        return Engine._OnStream(self)

    def compute_means(self):
        with self.on_stream():
            self._compute_means()

    supports_ahead = True   # step(then=...): see below

    def step(self, t_next, forcing, boundary, then=None, fetch=False):
        """One time-step of all local members; returns the max relative residual.

        ``then = (t, forcing, boundary)`` announces the call that follows (a time loop knows it): the
        pre-solve graph of that step (member sums, right-hand sides, assembly -- it only reads the new
        state and writes work buffers) is enqueued before this call returns, so the host's
        bookkeeping between two steps (~80 us of Python at C2) no longer leaves the GPU idle.  A next
        call that differs from the announcement simply redoes the pre-solve work.

        ``fetch=True`` (a caller that reads the new state on the host, `advance()` with host arrays
        in): the download of the new state -- layout kernels and D2H copies into pinned buffers -- is
        enqueued by the step itself, right behind the solve when the recent solves converged in their
        first cycle (redone if this one does not), instead of when the first field is read."""
        with self.on_stream():
            if self._graph_ok(forcing, boundary, t_next):
                failed = None
                try:
                    fresh = self._ensure_graphs(forcing, boundary)
                except (RuntimeError, N.NativeError) as exc:   # capture unsupported here: eager steps
                    failed, fresh = exc, True
                if fresh and self.comm is not None:
                    # every rank must take the same (graphed or eager) path: the two paths issue
                    # different collectives, so a capture failure on one rank disables graphs on all
                    bad = XC.allreduce_max_values([1.0 if failed is not None else 0.0], self.comm, self.dev)[0]
                    if bad > 0.0 and failed is None:
                        failed = RuntimeError("step-graph capture failed on another rank")
                if failed is not None:
                    import logging
                    logging.getLogger(__name__).warning("step graphs disabled (%s)", failed)
                    self.step_graphs = False
                    self._graphs.clear()
                    torch.cuda.synchronize(self.dev)
                    return self._eager(t_next, forcing, boundary, fetch)
                return self._step_graphed(t_next, forcing, boundary, then, fetch)
            return self._eager(t_next, forcing, boundary, fetch)

    def _eager(self, t_next, forcing, boundary, fetch):
        res = self._step(t_next, forcing, boundary)
        if fetch:      # (right behind the finished step; the graphed path enqueues it behind the solve)
            self._fetched = self._enqueue_fetch(self.cur) + ((self.cur, self.gen[self.cur]),)
        return res

    def _ensure_graphs(self, forcing, boundary):
        """Capture this parity's step graphs; returns True when they were captured now.  No state
        is modified."""
        lo = self._gdata(forcing, "loads") if hasattr(forcing, "separable") else None
        bc = self._gdata(boundary, "bc")
        n = len(self._graphs)
        self._step_graphs(lo, bc)
        return len(self._graphs) != n

    # ------------------------------------------------------------------
    # whole-step CUDA graphs
    # ------------------------------------------------------------------
    def _graph_ok(self, forcing, boundary, t_next):
        """Graph replay needs the extrapolated initial iterate (level n-1 resident) and separable data
        (or no body force at all)."""
        if not (self.step_graphs and self.prev_valid and self.guess == "extrapolate"
                and hasattr(boundary, "separable")):
            return False
        return hasattr(forcing, "separable") or self._no_loads(forcing, t_next)

    def _no_loads(self, forcing, t):
        lv, lw = forcing.loads(t, self.disc, self.config)
        return lv is None and lw is None

    def _gdata(self, obj, kind, parity=None):
        """(coefficient function, pinned host and device coefficient blocks, fixed DataDesc) of one data kind."""
        self._touch(obj)
        par = self.cur if (parity is None and self._wb[1] is not None) else (parity or 0)
        key = (kind, id(obj), par)       # (pinned / device coefficient blocks per parity once steps run ahead)
        ent = self._gdata_cache.get(key)
        if ent is None:
            self._data(obj, kind, 0.0)                   # builds the device basis once
            sep, basis_t = self._data_cache[(kind, id(obj))][:2]
            K = basis_t.shape[0]
            pin = torch.zeros(2, K, self.J, dtype=torch.float64, pin_memory=True)
            dev = torch.zeros(2, K, self.J, dtype=torch.float64, device=self.dev)
            dd = N.DataDesc()
            dd.rows = self.nvel if kind == "loads" else self.hm.nbdofs
            dd.K, dd.basis, dd.coef, dd.dense = K, _dptr(basis_t), _dptr(dev), None
            ent = (sep, pin, dev, dd)
            self._gdata_cache[key] = ent
        return ent

    def _touch(self, obj):
        """LRU bookkeeping of problem-data objects: beyond MAX_PROBLEM_OBJECTS the least recently used
        object's device data, coefficient blocks and step graphs are released."""
        oid = id(obj)
        if oid in self._lru:
            self._lru.move_to_end(oid)
            return
        self._lru[oid] = True
        while len(self._lru) > MAX_PROBLEM_OBJECTS:
            old, _ = self._lru.popitem(last=False)
            gone = set()
            for k in [k for k in self._gdata_cache if k[1] == old]:
                ent = self._gdata_cache.pop(k)
                gone.add(id(ent))
                self._gspec.pop(id(ent), None)
            for k in [k for k in self._data_cache if k[1] == old]:
                del self._data_cache[k]
            for k in [k for k in self._graphs if k[1] in gone or k[2] in gone]:
                del self._graphs[k]

    def release(self):
        """Free the device context and buffers (live states are copied to the host first)."""
        for b in (0, 1):
            self._retire(b)
        self._graphs.clear()
        self._gdata_cache.clear()
        self._data_cache.clear()
        if getattr(self, "ctx", None):
            torch.cuda.synchronize(self.dev)
            self.lib.ens_destroy(self.ctx)
            self.ctx = None
        for name in ("X", "Pq", "mesh_t", "plan_t", "_stg"):
            if hasattr(self, name):
                setattr(self, name, None)
        self._wb = [None, None]

    def _gcoef(self, ent, t):
        sep = ent[0]
        cv, cw = sep.coef(t)
        sl = slice(self.j0, self.j0 + self.J)
        return np.stack([np.asarray(cv, dtype=float)[:, sl], np.asarray(cw, dtype=float)[:, sl]])

    def _gfill(self, ent, t):
        """Coefficients at t into the pinned block the captured H2D copy reads (prefetched when t was predicted)."""
        spec = self._gspec.get(id(ent))
        h = ent[1].numpy()
        if spec is not None and spec[0] == t:
            h[...] = spec[1]
        else:
            h[...] = self._gcoef(ent, t)

    def _gprefetch(self, ent, t):
        """Evaluate the next step's coefficients while the GPU runs this step (callers advance t by dt)."""
        self._gspec[id(ent)] = (t, self._gcoef(ent, t))

    def _capture(self, fn):
        """Capture fn() on the engine stream into a CUDA graph; returns (graph, kernels in it)."""
        l0 = self.lib.ens_kernel_launches()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream, capture_error_mode="thread_local"):
            fn()
        n = int(self.lib.ens_kernel_launches() - l0)
        self.graph_launch_credit -= n
        return g, n

    def _step_graphs(self, lo, bc, cached_for=None):
        """Graph segments for the current buffer parity: split at the collectives when members are sharded.
        ``cached_for``: only look up the segments of that parity (None when not captured yet)."""
        lib, ctx, s = self.lib, self.ctx, self.sptr
        if cached_for is not None:
            return self._graphs.get((cached_for, id(lo), id(bc)))
        cur, nxt = self.cur, 1 - self.cur
        key = (cur, id(lo), id(bc))
        segs = self._graphs.get(key)
        if segs is not None:
            return segs
        X, Xn = self.X[cur], self.X[nxt]

        def sums():
            N.check(lib.ens_member_sums(ctx, s, _dptr(X), _dptr(self.sums)), "ens_member_sums")

        def rhs():
            N.check(lib.ens_means(ctx, s, _dptr(self.sums), 1.0 / self.J_total, _dptr(self.means)), "ens_means")
            if lo is not None:
                lo[2].copy_(lo[1], non_blocking=True)
            self._rhs_and_member_pass(X, C.byref(lo[3]) if lo is not None else None)

        def assemble():
            bc[2].copy_(bc[1], non_blocking=True)
            N.check(lib.ens_apply_bc(ctx, s, C.byref(bc[3]), _dptr(self.rhs)), "ens_apply_bc")
            N.check(lib.ens_assemble(ctx, s, _dptr(self.base), _dptr(self.means), _dptr(self.maxsq),
                                     self.two_mu_dt, _dptr(self.as_vals)), "ens_assemble")

        def solve():
            N.check(lib.ens_lincomb(ctx, s, 2.0, _dptr(X), -1.0, _dptr(Xn)), "ens_lincomb")   # 2 x^n - x^{n-1}
            N.check(lib.ens_solve_begin(ctx, s, _dptr(self.as_vals), _dptr(self.rhs), _dptr(Xn), self.rtol,
                                        self.restart, 1), "ens_solve_begin")
            N.check(lib.ens_epilogue(ctx, s, _dptr(Xn), _dptr(self.Pq[nxt])), "ens_epilogue")

        if self.comm is None:
            def pre():
                sums()
                rhs()
                assemble()
            parts = [("pre", pre), ("solve", solve)]
        else:
            parts = [("sums", sums), ("rhs", rhs), ("assemble", assemble), ("solve", solve)]
        segs = {name: self._capture(fn) for name, fn in parts}
        self._graphs[key] = segs
        return segs

    def _replay(self, seg):
        g, n = seg
        g.replay()
        self.graph_launch_credit += n

    def _step_graphed(self, t_next, forcing, boundary, then=None, fetch=False):
        lib, ctx, s = self.lib, self.ctx, self.sptr
        if then is not None and self.comm is None and self.refactor != "timed" and self._wb[1] is None:
            self._enable_ahead()         # first announced step: work buffers and data blocks per parity
        cur, nxt = self.cur, 1 - self.cur
        X, Xn = self.X[cur], self.X[nxt]
        spec, self._spec = self._spec, None
        ahead = spec is not None and spec == (t_next, id(forcing), id(boundary), cur, self._nstep)
        if spec is not None and not ahead:
            self.stream.synchronize()    # the enqueued graph's H2D copies still read the pinned coefficient blocks
        lo = self._gdata(forcing, "loads") if hasattr(forcing, "separable") else None   # None: no body force
        bc = self._gdata(boundary, "bc")
        if not ahead:
            if lo is not None:
                self._gfill(lo, t_next)
            self._gfill(bc, t_next)
        segs = self._step_graphs(lo, bc)
        self._retire(nxt)          # (a caller's copy of the state about to be overwritten: not step cost)
        self._cost_begin()
        if self.comm is None:
            need = self._need_factor()
            if not ahead:
                self._replay(segs["pre"])
        else:
            self._replay(segs["sums"])
            XC.allreduce_member_sums(self.sums, self.comm)
            self._replay(segs["rhs"])
            # the previous step's (residual, iterations, renewal flag) ride on the MAX exchange:
            # no separate scalar collective and no extra synchronisation per step
            prev = self._prev_local if self._prev_local is not None else (0.0, 0.0, 0.0)
            self._tail_in.numpy()[:] = prev
            self._tail.copy_(self._tail_in, non_blocking=True)
            XC.allreduce_eddy_max(self.maxsq_ext, self.comm)
            self._tail_out.copy_(self._tail, non_blocking=True)
            self._tail_ev.record(self.stream)
            self._replay(segs["assemble"])
            self._tail_ev.synchronize()            # the assembly keeps the GPU busy meanwhile
            g = self._tail_out.numpy().copy()
            if self._prev_local is not None:
                self.global_residuals[self._nstep - 1] = float(g[0])
                self._agreed(g[1])
                if self.refactor == "timed":
                    self._renew = g[2] > 0.0
                self._prev_local = None
            need = self._need_factor()
        if need:
            self._factor_timed()
        else:
            self.since_factor += 1
        self._replay(segs["solve"])
        if then is None:
            t_pred = t_next + self.config.dt              # host work overlapped with the solve
            if lo is not None:
                self._gprefetch(lo, t_pred)
            self._gprefetch(bc, t_pred)
        ahead_segs, early = None, False
        if then is not None and self.comm is None and self.refactor != "timed":
            ahead_segs = self._prepare_ahead(nxt, *then)
            if ahead_segs is not None and self._ones >= 4 and self._wb[1] is not None:
                # the last four solves converged in their first cycle: expect the same and enqueue the announced
                # step's pre-solve graph behind this solve right away (it works on the other parity's
                # buffers; if this solve does need more cycles, that work is simply redone)
                nsegs, nlo, nbc = ahead_segs
                if nlo is not None:
                    self._gfill(nlo, then[0])
                self._gfill(nbc, then[0])
                self._replay(nsegs["pre"])
                early = True
        pre = self._enqueue_fetch(nxt) if fetch and self._ones >= 4 else None   # (speculative, as above)
        iters = N.I32(0)
        rel = (N.F64 * 2)()
        code = lib.ens_solve_finish(ctx, s, _dptr(self.as_vals), _dptr(self.rhs), _dptr(Xn), self.rtol,
                                    self.restart, self.max_restarts, C.byref(iters), rel)
        iters, rel = int(iters.value), (rel[0], rel[1])
        redo = iters > 1                                  # more cycles ran after the captured epilogue
        if code == N.ENS_ENOCONV and not need:            # stale preconditioner: rebuild and retry once
            self._factor_timed()
            Xn.copy_(X)
            code, iters2, rel = self._solve(Xn, predict=1)
            iters += iters2
            redo = True
        self.last_iters, self.last_relres = iters, rel
        self._ones = self._ones + 1 if iters == 1 else 0
        N.check(code, "ens_solve_finish")
        if redo:
            N.check(lib.ens_epilogue(ctx, s, _dptr(Xn), _dptr(self.Pq[nxt])), "ens_epilogue")
        self.gen[nxt] += 1
        self.cur = nxt
        self.means_valid = False
        self.prev_valid = True
        if fetch:
            if pre is None or redo:
                pre = self._enqueue_fetch(nxt)
            self._fetched = pre + ((nxt, self.gen[nxt]),)
        if early:
            # (this solve needed more cycles after all: the work enqueued ahead read an unfinished
            # state and is redone -- after a stream synchronisation, as for any stale announcement)
            self._spec = (then[0], id(then[1]), id(then[2]), self.cur, self._nstep + 1) if not redo else ("stale",)
        elif then is not None and self.comm is None and self.refactor != "timed":
            # first thing after the solve: the GPU has only the pressure epilogue left to run
            if ahead_segs is not None:
                nsegs, nlo, nbc = ahead_segs
                if nlo is not None:
                    self._gfill(nlo, then[0])
                self._gfill(nbc, then[0])
                self._replay(nsegs["pre"])
                self._spec = (then[0], id(then[1]), id(then[2]), self.cur, self._nstep + 1)
            else:
                self._enqueue_ahead(*then)
        renew = self._step_done(iters)
        self._nstep += 1
        if self.comm is None:
            self._renew = renew
            return max(self.last_relres)
        # sharded: this rank's values travel with the next step's MAX exchange (or flush_global)
        self._prev_local = (max(self.last_relres), float(self.last_iters), float(bool(renew)))
        return max(self.last_relres)

    def _prepare_ahead(self, parity, t, forcing, boundary):
        """While this step's solve runs: the announced next step's graph segments (buffer parity
        ``parity``) and data entries; None when its graphs are not captured yet."""
        if not self._graph_ok(forcing, boundary, t):
            return None
        lo = self._gdata(forcing, "loads", parity) if hasattr(forcing, "separable") else None
        bc = self._gdata(boundary, "bc", parity)
        segs = self._step_graphs(lo, bc, cached_for=parity)
        if segs is None:
            return None
        # (the pinned coefficient blocks are filled after the solve's host round trip: this step's
        # own pre-solve graph, enqueued but possibly not executed yet, still reads them)
        return segs, lo, bc

    def _enqueue_ahead(self, t, forcing, boundary):
        """Enqueue the announced next step's pre-solve graph now (see ``step``)."""
        if not self._graph_ok(forcing, boundary, t):
            return
        try:
            lo = self._gdata(forcing, "loads") if hasattr(forcing, "separable") else None
            bc = self._gdata(boundary, "bc")
            segs = self._step_graphs(lo, bc)     # (this parity's graphs: captured on its first use)
        except (RuntimeError, N.NativeError):
            return
        if lo is not None:
            self._gfill(lo, t)
        self._gfill(bc, t)
        self._replay(segs["pre"])
        self._spec = (t, id(forcing), id(boundary), self.cur, self._nstep + 1)   # (the step count once this step is booked)

    def flush_global(self):
        """Sharded runs: agree on the last step's (residual, iterations, renewal) now instead of in
        the next step's exchange; returns the residual max over ranks."""
        if self.comm is None or self._prev_local is None:
            return None
        res, it, rn = XC.allreduce_max_values(list(self._prev_local), self.comm, self.dev)
        self.global_residuals[self._nstep - 1] = res
        self._agreed(it)
        if self.refactor == "timed":
            self._renew = rn > 0.0
        self._prev_local = None
        return res

    def diagnostics(self):
        """Device-side _record (stepper.py:432-439) of the current state."""
        with self.on_stream():
            return self._diagnostics()

    def mean_error(self, exact, t):
        """Squared H1 errors (||d_v||^2, ||d_w||^2) of the current ensemble means against a separable
        exact field (``exact.mean_separable(disc, config)``), computed on the device
        (ens_mean_error; the summands of experiments.error_norm_21, `experiments.py:59-73`)."""
        self._touch(exact)
        key = ("mean-exact", id(exact))
        ent = self._data_cache.get(key)
        if ent is None:
            sep = exact.mean_separable(self.disc, self.config)
            basis = np.asarray(sep.basis, dtype=float).reshape(len(sep.basis), -1)[:, self.hm.ref_of_int[:self.nvel]]
            ent = (sep, torch.as_tensor(np.ascontiguousarray(basis)).to(self.dev), exact,
                   torch.zeros(4, dtype=torch.float64, device=self.dev))
            self._data_cache[key] = ent
        sep, basis_t, _, out = ent
        cv, cw = sep.coef(t)
        coef_t = torch.as_tensor(np.stack([np.asarray(cv, float).reshape(-1), np.asarray(cw, float).reshape(-1)]))
        with self.on_stream():
            if not self.means_valid:
                self._compute_means()
            coef_d = coef_t.to(self.dev, non_blocking=False)
            dd = N.DataDesc()
            dd.rows, dd.K, dd.basis, dd.coef, dd.dense = self.nvel, basis_t.shape[0], _dptr(basis_t), _dptr(coef_d), None
            N.check(self.lib.ens_mean_error(self.ctx, self.sptr, _dptr(self.means), C.byref(dd), _dptr(out)),
                    "ens_mean_error")
            r = out.cpu().numpy()
        return float(r[0] + r[1]), float(r[2] + r[3])

    def _compute_means(self):
        lib, ctx, s = self.lib, self.ctx, self.sptr
        X = self.X[self.cur]
        N.check(lib.ens_member_sums(ctx, s, _dptr(X), _dptr(self.sums)), "ens_member_sums")
        XC.allreduce_member_sums(self.sums, self.comm)
        N.check(lib.ens_means(ctx, s, _dptr(self.sums), 1.0 / self.J_total, _dptr(self.means)), "ens_means")
        self.means_valid = True

    def _step(self, t_next, forcing, boundary):
        lib, ctx, s = self.lib, self.ctx, self.sptr
        self._spec = None
        cur, nxt = self.cur, 1 - self.cur
        X = self.X[cur]
        self.flush_global()        # sharded: agree on the previous graphed step's values first
        self._retire(1 - cur)
        self._cost_begin()
        if not self.means_valid:
            self._compute_means()
        loads, keep1 = self._data(forcing, "loads", t_next)
        self._rhs_and_member_pass(X, C.byref(loads) if loads is not None else None)
        XC.allreduce_eddy_max(self.maxsq, self.comm)
        bvals, keep2 = self._data(boundary, "bc", t_next)
        N.check(lib.ens_apply_bc(ctx, s, C.byref(bvals), _dptr(self.rhs)), "ens_apply_bc")
        N.check(lib.ens_assemble(ctx, s, _dptr(self.base), _dptr(self.means), _dptr(self.maxsq), self.two_mu_dt,
                                 _dptr(self.as_vals)), "ens_assemble")
        need = self._need_factor()
        if need:
            self._factor_timed()
        else:
            self.since_factor += 1
        self._retire(nxt)
        Xn = self.X[nxt]
        if self.guess == "extrapolate" and self.prev_valid:
            N.check(lib.ens_lincomb(ctx, s, 2.0, _dptr(X), -1.0, _dptr(Xn)), "ens_lincomb")   # 2 x^n - x^{n-1}
        else:
            Xn.copy_(X)                               # warm start from level n
        code, iters, rel = self._solve(Xn)
        if code == N.ENS_ENOCONV and not need:        # stale preconditioner: rebuild and retry once
            self._factor_timed()
            Xn.copy_(X)
            code, iters2, rel = self._solve(Xn, predict=1)
            iters += iters2
        self.last_iters, self.last_relres = iters, rel
        N.check(code, "ens_solve")
        N.check(lib.ens_epilogue(ctx, s, _dptr(Xn), _dptr(self.Pq[nxt])), "ens_epilogue")
        del keep1, keep2
        self.gen[nxt] += 1
        self.cur = nxt
        self.means_valid = False
        self.prev_valid = True
        # residual max, iteration count and the renewal decision over ranks: every rank then
        # takes the same refactorisation decision next step (identical shared matrices, lockstep timing)
        renew = self._step_done(iters)
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

    # ------------------------------------------------------------------
    # preconditioner renewal
    # ------------------------------------------------------------------
    def _need_factor(self):
        return (self.refactor == "always" or not self.factored or self.since_factor >= self.lag_max_steps
                or self.last_iters > self.lag_max_iters or self._renew)

    def _cost_begin(self):
        self._fac_this = False
        if self.refactor != "timed":
            return
        if self._ev is None:
            self._ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        self._ev[0].record(self.stream)

    def _factor_timed(self):
        if self.refactor == "timed":
            self._ev[1].record(self.stream)
        self._factor()
        if self.refactor == "timed":
            self._ev[2].record(self.stream)
        self._fac_this = True

    def _step_done(self, iters):
        """End of a step: the renewal decision for the next step.

        "adaptive" (default) decides from the step's Krylov iteration count only
        (agreed over ranks first when members are sharded, see ``_renewal``), so a
        run is a deterministic function of its inputs.  "timed" keeps the
        measured-device-time rule (``_cost_end``).  Returns the renewal flag this
        rank proposes, or None when the decision waits for the agreed count."""
        fac = self._fac_this
        if self.refactor == "timed":
            return self._cost_end()
        if self.comm is not None:
            self._pending = fac      # decided once the iteration count is agreed over ranks
            return None
        return self._renewal(iters, fac)

    def _agreed(self, iters):
        """Sharded runs: the step's iteration count maxed over ranks has arrived."""
        self.last_iters = int(iters)
        if self.refactor != "timed" and self._pending is not None:
            self._renew = self._renewal(int(iters), self._pending)
            self._pending = None

    def _renewal(self, k, fac):
        """Deterministic renewal rule (the optimal stopping rule of a renewal process).

        A factorisation costs F, a step whose solve needs k preconditioned Krylov
        iterations costs c0 + k c_it (``cost_model``).  With k_1..k_L the counts of
        the current factorisation's lifetime, rebuilding before step L+1 lowers the
        average cost per step iff  c0 + k_{L+1} c_it > (F + sum_i (c0 + k_i c_it)) / L,
        i.e. iff  sum_i (k_{L+1} - k_i) > rho = F / c_it  (c0 cancels).  k_{L+1} is
        predicted from the count at the same lifetime position in recent lifetimes
        (exponentially averaged), else from k_L.  Only iteration counts enter, which
        every rank agrees on, so two runs on the same inputs rebuild at the same
        steps and are bitwise identical."""
        if fac:
            self._life += 1
            self._lk = [k]
        elif self._lk is None:
            return False
        else:
            self._lk.append(k)
        pos = len(self._lk)
        fresh = max(2, self._life - RENEW_WINDOW)
        if len(self._prof) < pos:
            self._prof.append([float(k), self._life])
        else:
            old = self._prof[pos - 1]
            self._prof[pos - 1] = [0.5 * (old[0] + k) if old[1] >= fresh else float(k), self._life]
        if self.refactor != "adaptive":
            return False
        nxt = float(k)
        if pos < len(self._prof) and self._prof[pos][1] >= max(2, self._life - RENEW_STALE):
            nxt = self._prof[pos][0]
        excess = sum(nxt - ki for ki in self._lk)
        if _RENEW_DEBUG:
            print(f"renew: pos {pos} k {k} pred {nxt:.2f} excess {excess:.2f} rho {self.rho:.2f}", flush=True)
        return excess > self.rho

    def _cost_end(self):
        """Timed renewal rule (refactor="timed", opt-in): with F the last factorisation's device
        time and A_1..A_L the device times of the steps since (factorisation excluded), rebuild
        before the next step when the next step would cost more than the lifetime's average cost
        per step, A_{L+1} > (F + sum A) / L.  The next step's cost is predicted from the cost at
        the same position of earlier lifetimes when known, else from this step.  Decisions depend
        on measured times, so runs are reproducible only up to the solver tolerance."""
        ev = self._ev
        ev[3].record(self.stream)
        ev[3].synchronize()
        step_ms = ev[0].elapsed_time(ev[3])
        if self._fac_this:
            f = ev[1].elapsed_time(ev[2])
            self._cyc = [f, step_ms - f, 1]
            self._life += 1
            a = step_ms - f
        elif self._cyc is not None:
            self._cyc[1] += step_ms
            self._cyc[2] += 1
            a = step_ms
        else:
            return False
        steps = self._cyc[2]
        fresh = max(2, self._life - RENEW_WINDOW)
        if len(self._prof) < steps:
            self._prof.append([a, self._life])
        else:
            old = self._prof[steps - 1]
            self._prof[steps - 1] = [0.5 * (old[0] + a) if old[1] >= fresh else a, self._life]
        nxt = a
        if steps < len(self._prof) and self._prof[steps][1] >= max(2, self._life - RENEW_STALE):
            nxt = self._prof[steps][0]
        return nxt > (self._cyc[0] + self._cyc[1]) / steps

    def _rhs_and_member_pass(self, X, loads_ref):
        """Right-hand sides of both sub-steps + eddy-viscosity maxima (one element pass by default;
        ENS_RHS_FUSED=0: the CSR mass/stiffness pass followed by the fluctuation-transport pass)."""
        lib, ctx, s = self.lib, self.ctx, self.sptr
        if self.rhs_fused:
            N.check(lib.ens_rhs_fused(ctx, s, _dptr(X), _dptr(self.means), _dptr(self.member_coef),
                                      1.0 / self.config.dt, loads_ref, _dptr(self.rhs), _dptr(self.maxsq)),
                    "ens_rhs_fused")
            return
        N.check(lib.ens_rhs(ctx, s, _dptr(X), _dptr(self.member_coef), 1.0 / self.config.dt, loads_ref,
                            _dptr(self.rhs)), "ens_rhs")
        N.check(lib.ens_member_pass(ctx, s, _dptr(X), _dptr(self.means), _dptr(self.rhs), _dptr(self.maxsq)),
                "ens_member_pass")

    def _factor(self):
        npert = N.I32(0)
        N.check(self.lib.ens_factor(self.ctx, self.sptr, _dptr(self.as_vals), C.byref(npert)), "ens_factor")
        if npert.value > 0 and not self.pivoting:
            # a diagonal pivot was tiny: switch this engine to in-panel pivoting for good
            self.pivoting = True
            N.check(self.lib.ens_set_pivoting(self.ctx, 1), "ens_set_pivoting")
            N.check(self.lib.ens_factor(self.ctx, self.sptr, _dptr(self.as_vals), C.byref(npert)), "ens_factor")
        self.last_pert = int(npert.value)
        self.factored = True
        self.since_factor = 0
        self.n_factor += 1

    def _solve(self, Xn, predict=1):
        # first FGMRES cycle: `predict` iterations without host round trips, then the
        # true residual decides (one iteration is the steady state with the
        # extrapolated guess; otherwise the next cycles check every iteration)
        iters = N.I32(predict)
        rel = (N.F64 * 2)()
        code = self.lib.ens_solve(self.ctx, self.sptr, _dptr(self.as_vals), _dptr(self.rhs), _dptr(Xn), self.rtol,
                                  self.restart, self.max_restarts, C.byref(iters), rel)
        return code, int(iters.value), (rel[0], rel[1])

    def _diagnostics(self):
        if not self.means_valid:
            self._compute_means()
        N.check(self.lib.ens_diagnostics(self.ctx, self.sptr, _dptr(self.X[self.cur]), _dptr(self.means),
                                         _dptr(self.diag_out)), "ens_diagnostics")
        out = self.diag_out.cpu().numpy()
        J = self.J
        series = out[2:].reshape(6, J)
        return dict(energy=0.5 * (out[0] + out[1]), l2v=series[0], l2w=series[1], gradv=series[2], gradw=series[3],
                    div_v=np.sqrt(np.maximum(series[4], 0.0)), div_w=np.sqrt(np.maximum(series[5], 0.0)))

    # ------------------------------------------------------------------
    # lower seams of the reference API: stepper.assemble_shared_lhs / assemble_member_rhs and
    # linalg.factorize (`stepper.py:181-278`, `linalg.py:46-108`).  Same kernels as the step.
    # ------------------------------------------------------------------
    def block_to_internal(self, blk_ref):
        """(n_total, J) reference-order rows -> (n_total, J) internal rows (numpy)."""
        out = np.empty_like(np.asarray(blk_ref, dtype=float))
        out[self.hm.int_id] = blk_ref
        return out

    def block_to_ref(self, blk_int):
        return np.asarray(blk_int)[self.hm.int_id]

    def _seam_state(self, v, w):
        self.load_state(v, w, None, None)
        self.prev_valid = False

    def shared_block_values(self, system, mean_adv, flucts):
        """A_s values (internal slot order) of one sub-step matrix: system 0 = V (advected by the
        given mean, eddy viscosity of the given fluctuations), 1 = W; `stepper.py:195-206`."""
        hm, J = self.hm, self.J
        flucts = np.asarray(flucts, dtype=float)
        if flucts.shape != (J, self.nvel):
            raise ValueError(f"fluctuations shape {flucts.shape} != ({J}, {self.nvel})")
        fields = np.asarray(mean_adv, dtype=float)[None, :] + flucts
        self._seam_state(fields, fields)
        mean_int = hm.vel_to_internal(np.asarray(mean_adv, dtype=float)[None, :])[:, 0]
        lib, ctx, s = self.lib, self.ctx, self.sptr
        with self.on_stream():
            m = torch.as_tensor(mean_int).to(self.dev)
            self.means[:self.nvel].copy_(m)
            self.means[self.nvel:].copy_(m)
            self._rhs_and_member_pass(self.X[self.cur], None)
            N.check(lib.ens_assemble(ctx, s, _dptr(self.base), _dptr(self.means), _dptr(self.maxsq),
                                     self.two_mu_dt, _dptr(self.as_vals)), "ens_assemble")
            out = self.as_vals[system].cpu().numpy()
        self.means_valid = False
        return out

    def member_rhs_block(self, system, v, w, loads, bvals):
        """(n_total, J) right-hand sides of one sub-step in reference order (`stepper.py:223-252`):
        ``loads`` (J, n_vel) or None and ``bvals`` (J, nb) of that sub-step."""
        hm, J = self.hm, self.J
        self._seam_state(v, w)
        lib, ctx, s = self.lib, self.ctx, self.sptr
        with self.on_stream():
            self._compute_means()
            keep = []
            lref = None
            if loads is not None:
                dense = np.zeros((2, self.nvel, J))
                dense[system] = hm.vel_to_internal(np.asarray(loads, dtype=float))
                lt = torch.as_tensor(dense).to(self.dev)
                keep.append(lt)
                ld = N.DataDesc()
                ld.rows, ld.K, ld.basis, ld.coef, ld.dense = self.nvel, 0, None, None, _dptr(lt)
                lref = C.byref(ld)
            self._rhs_and_member_pass(self.X[self.cur], lref)
            dense = np.zeros((2, hm.nbdofs, J))
            dense[system] = np.asarray(bvals, dtype=float).reshape(J, hm.nbdofs).T
            bt = torch.as_tensor(dense).to(self.dev)
            bd = N.DataDesc()
            bd.rows, bd.K, bd.basis, bd.coef, bd.dense = hm.nbdofs, 0, None, None, _dptr(bt)
            N.check(lib.ens_apply_bc(ctx, s, C.byref(bd), _dptr(self.rhs)), "ens_apply_bc")
            out = self.rhs[system].cpu().numpy()
            del keep, bt
        self.means_valid = False
        return self.block_to_ref(out)

    def solve_values(self, a_vals, rhs_ref, factor=True):
        """Solve the saddle system with A_s = ``a_vals`` (internal slots) for the (n_total, J) block
        ``rhs_ref`` (reference order): the same factorisation-preconditioned column-batched Krylov
        as the step, converged to ``rtol`` per column.  Returns (x_ref, relres)."""
        J = self.J
        self._spec = None
        rhs_int = self.block_to_internal(np.asarray(rhs_ref, dtype=float).reshape(self.ntot, J))
        lib, ctx, s = self.lib, self.ctx, self.sptr
        with self.on_stream():
            a = torch.as_tensor(np.asarray(a_vals, dtype=float)).to(self.dev)
            self.as_vals[0].copy_(a)
            self.as_vals[1].copy_(a)
            if factor:
                self._factor()
            self.rhs.zero_()
            self.rhs[0].copy_(torch.as_tensor(rhs_int))
            x = torch.zeros_like(self.rhs)
            code, iters, rel = self._solve(x, predict=0)
            N.check(code, "ens_solve")
            out = x[0].cpu().numpy()
        self.last_relres = rel
        return self.block_to_ref(out), rel[0]

    # raw access for tests
    def spmm(self, x, b=None, mode=0, out=None):
        self._spec = None
        out = torch.empty_like(x) if out is None else out
        with self.on_stream():
            N.check(self.lib.ens_spmm(self.ctx, self.sptr, _dptr(self.as_vals), _dptr(x),
                                      _dptr(b) if b is not None else None, _dptr(out), mode), "ens_spmm")
        return out

    def factor(self):
        self._spec = None
        with self.on_stream():
            self._factor()
        return self.last_pert

    def precond(self, r, out=None):
        self._spec = None
        out = torch.zeros_like(r) if out is None else out
        with self.on_stream():
            N.check(self.lib.ens_precond_apply(self.ctx, self.sptr, _dptr(r), _dptr(out)), "ens_precond_apply")
        return out
