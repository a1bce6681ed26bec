"""CPU ORACLE -- test infrastructure only, never the product path.

Restates, in numpy/scipy, the reference's time-step hot path
(`/root/reference/pkg/src/ensmhd/stepper.py` + the per-step pieces of
`fem.py` / `ensemble.py` / `linalg.py`), so the GPU engine can be checked on
the same seeded inputs.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline leg may import this module.

Pinning: ``tests/golden/make_golden.py`` runs the *real* reference (importable
in the build container from /root/reference) on small cases and stores its
outputs as ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this
restatement against those fixtures (bitwise-level tolerances for assembly,
1e-12 for solves), so parity is pinned to the reference itself.

Mesh / dof-map / constant-operator setup is taken from the package's host
setup modules (pure numpy, also pinned against the golden fixtures); every
per-step quantity below is recomputed here independently of the GPU code.
The linear solve is SciPy SuperLU, i.e. the backend the reference itself
falls back to when cvxopt/UMFPACK is absent (`linalg.py:99-108`).
"""

from __future__ import annotations

import time as _time
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from paper_2108_05110_b200 import fe
from paper_2108_05110_b200.ensemble import viscosity_stats


# ----------------------------------------------------------------------
# element-level per-step kernels (reference fem.py / ensemble.py)
# ----------------------------------------------------------------------


def _scatter_scalar(vel, local):
    ns = vel.num_scalar_dofs
    r = np.broadcast_to(vel.cell_dofs[:, :, None], local.shape).ravel()
    c = np.broadcast_to(vel.cell_dofs[:, None, :], local.shape).ravel()
    a = sp.coo_matrix((local.ravel(), (r, c)), shape=(ns, ns)).tocsr()
    a.sort_indices()
    return a


def convection_scalar(vel, beta):
    """N_ab = sum_q w_q (beta_q . grad phi_b) phi_a, non-skew (`fem.py:309-317`)."""
    bq = fe.eval_at_quadrature(vel, beta)                      # (nt,7,2)
    bg = np.einsum("eqd,eqjd->eqj", bq, vel.basis_grad)        # (nt,7,6)
    local = np.einsum("eq,eqj,qi->eij", vel.wdet, bg, fe.PHI)
    return _scatter_scalar(vel, local)


def stiffness_coeff(vel, coeff):
    """K(c)_ab = sum_q w_q c_q grad phi_a . grad phi_b; rejects c < 0 (`fem.py:268-282`)."""
    c = np.asarray(coeff, dtype=float)
    if np.any(c < 0.0):
        raise ValueError("diffusion coefficient is negative at a quadrature point")
    local = np.einsum("eq,eqid,eqjd->eij", vel.wdet * c, vel.basis_grad, vel.basis_grad)
    return _scatter_scalar(vel, local)


def eddy_viscosity(vel, fluct, mu, dt):
    """mu dt max_j |z'_j(x_q)|^2 at quadrature points, (nt, 7) (`ensemble.py:227-238`)."""
    if mu <= 0.0 or dt <= 0.0:
        raise ValueError("mu and dt must be positive")
    vals = fe.eval_at_quadrature(vel, fluct)                   # (J,nt,7,2)
    sq = np.einsum("jeqd,jeqd->jeq", vals, vals)
    return mu * dt * sq.max(axis=0)


def convection_apply(vel, beta, field):
    """r_a = int (beta . grad field) . phi_a, batched over members (`fem.py:411-420`)."""
    bq = fe.eval_at_quadrature(vel, beta)
    gq = fe.eval_gradient_at_quadrature(vel, field)
    conv = np.einsum("...eqd,...eqcd->...eqc", bq, gq)
    return fe.load_vector(vel, conv)


def divergence_l2(vel, coeffs):
    """||div z||_L2 by quadrature, batched (`fem.py:508-514`)."""
    g = fe.eval_gradient_at_quadrature(vel, coeffs)
    div = g[..., 0, 0] + g[..., 1, 1]
    return np.sqrt(np.einsum("eq,...eq->...", vel.wdet, div * div))


def replace_rows_with_identity(a, rows):
    """Zero the rows, put 1 on their diagonal (`fem.py:446-460`)."""
    a = a.tocsr(copy=True)
    rows = np.asarray(rows, dtype=np.int64)
    if rows.size:
        for r in rows:
            a.data[a.indptr[r]:a.indptr[r + 1]] = 0.0
        a = (a + sp.csr_matrix((np.ones(rows.size), (rows, rows)), shape=a.shape)).tocsr()
    a.sort_indices()
    return a


# ----------------------------------------------------------------------
# shared matrix, member right-hand sides, one step (reference stepper.py)
# ----------------------------------------------------------------------


def velocity_block(mean_adv, fluct, config, disc):
    """a_s = M/dt + N(mean) + (nu_bar+nu_m_bar)/2 K + K(2 nu_T) (`stepper.py:195-206`)."""
    st = viscosity_stats(config)
    vel = disc.velocity
    nu_t = eddy_viscosity(vel, fluct, config.mu, config.dt)
    return (disc.mass_s / config.dt + convection_scalar(vel, mean_adv)
            + 0.5 * (st.nu_bar + st.nu_m_bar) * disc.stiff_s + stiffness_coeff(vel, 2.0 * nu_t))


def saddle_matrix(a_s, disc):
    """[[A,0,-Bx^T],[0,A,-By^T],[Bx,By,0]] with identity rows (`stepper.py:208-215`)."""
    ns = disc.n_scalar
    bx, by = disc.divergence[:, :ns], disc.divergence[:, ns:]
    full = sp.bmat([[a_s, None, -bx.T], [None, a_s, -by.T], [bx, by, None]], format="csr")
    full = replace_rows_with_identity(full, disc.bdofs)
    if disc.pin_pressure:
        full = replace_rows_with_identity(full, np.array([disc.pin_row]))
    return full


def shared_matrix(kind, v, w, config, disc):
    """Shared sub-step matrix: V uses <w>, w'; W uses <v>, v' (`stepper.py:181-220`)."""
    if kind == "v":
        mean, fl = w.mean(axis=0), w - w.mean(axis=0)
    else:
        mean, fl = v.mean(axis=0), v - v.mean(axis=0)
    return saddle_matrix(velocity_block(mean, fl, config, disc), disc)


def rhs_block(kind, v, w, loads, bvals, config, disc):
    """(n_total, J) right-hand sides of one sub-step (`stepper.py:223-252`)."""
    if kind == "v":
        same, other, fl = v, w, w - w.mean(axis=0)
    else:
        same, other, fl = w, v, v - v.mean(axis=0)
    st = viscosity_stats(config)
    lag_cross = 0.5 * (config.nu - config.nu_m)
    lag_same = 0.5 * (st.nu_fluct + st.nu_m_fluct)
    r = disc.apply_mass(same) / config.dt
    r -= convection_apply(disc.velocity, fl, same)
    r -= lag_cross[:, None] * disc.apply_stiffness(other)
    r -= lag_same[:, None] * disc.apply_stiffness(same)
    if loads is not None:
        r = r + loads
    rhs = np.zeros((disc.n_total, config.num_members))
    rhs[:disc.n_vel] = r.T
    rhs[disc.bdofs] = np.asarray(bvals).T
    if disc.pin_pressure:
        rhs[disc.pin_row] = 0.0
    return rhs


def solve_block(matrix, rhs):
    """SuperLU factor once, solve all columns (`linalg.py:62-108`)."""
    lu = spla.splu(matrix.tocsc())
    return lu.solve(rhs)


def relative_residual(matrix, x, b):
    """max_j ||A x_j - b_j|| / max(||b_j||, tiny) (`linalg.py:111-118`)."""
    r = matrix @ x - b
    denom = np.maximum(np.linalg.norm(b, axis=0), np.finfo(float).tiny)
    return float(np.max(np.linalg.norm(r, axis=0) / denom))


@dataclass
class OracleState:
    v: np.ndarray
    w: np.ndarray
    q: np.ndarray
    r: np.ndarray
    step: int = 0
    time: float = 0.0


def advance(state: OracleState, config, disc, forcing, boundary):
    """One full time-step, both sub-steps from level-n data (`stepper.py:360-394`)."""
    t_next = state.time + config.dt
    lv, lw = forcing.loads(t_next, disc, config)
    bv, bw = boundary.values(t_next, disc, config)
    out = {}
    res = 0.0
    for kind, loads, bvals in (("v", lv, bv), ("w", lw, bw)):
        mat = shared_matrix(kind, state.v, state.w, config, disc)
        rhs = rhs_block(kind, state.v, state.w, loads, bvals, config, disc)
        sol = solve_block(mat, rhs)
        res = max(res, relative_residual(mat, sol, rhs))
        out[kind] = sol
    nv = disc.n_vel
    new = OracleState(
        v=np.ascontiguousarray(out["v"][:nv].T), w=np.ascontiguousarray(out["w"][:nv].T),
        q=disc.mean_zero_pressure(out["v"][nv:].T), r=disc.mean_zero_pressure(out["w"][nv:].T),
        step=state.step + 1, time=t_next)
    return new, res


def energy(v, w, disc):
    """E = 1/2 (<v>^T M <v> + <w>^T M <w>) (`stepper.py:397-401`)."""
    mv, mw = v.mean(axis=0), w.mean(axis=0)
    return 0.5 * float(mv @ disc.apply_mass(mv) + mw @ disc.apply_mass(mw))


def record(state, disc):
    """Per-level diagnostics of `_record` (`stepper.py:432-439`)."""
    return dict(
        energy=energy(state.v, state.w, disc),
        div_v=float(np.max(divergence_l2(disc.velocity, state.v))),
        div_w=float(np.max(divergence_l2(disc.velocity, state.w))),
        l2v=np.einsum("ji,ji->j", state.v, disc.apply_mass(state.v)),
        l2w=np.einsum("ji,ji->j", state.w, disc.apply_mass(state.w)),
        gradv=np.einsum("ji,ji->j", state.v, disc.apply_stiffness(state.v)),
        gradw=np.einsum("ji,ji->j", state.w, disc.apply_stiffness(state.w)),
    )


def run(config, disc, v0, w0, forcing, boundary, steps=None, with_record=True):
    """M-step loop (`stepper.py:442-502`); returns (final state, records, per-step seconds)."""
    m = int(round(config.t_end / config.dt)) if steps is None else int(steps)
    j = config.num_members
    st = OracleState(np.array(v0, float), np.array(w0, float), np.zeros((j, disc.n_pres)), np.zeros((j, disc.n_pres)))
    recs = [record(st, disc)] if with_record else []
    wall, resid = [], []
    for _ in range(m):
        t0 = _time.perf_counter()
        st, res = advance(st, config, disc, forcing, boundary)
        wall.append(_time.perf_counter() - t0)
        resid.append(res)
        if with_record:
            recs.append(record(st, disc))
    return st, recs, np.array(wall), np.array(resid)
