"""Generate golden fixtures by running the REAL reference (`/root/reference`).

Run in the build container only (the reference does not exist on the GPU
box):   python tests/golden/make_golden.py

Every fixture is produced by the unmodified reference package `ensmhd`
(SuperLU backend, since cvxopt/UMFPACK is absent here).  Taylor-Hood cases
use the two-line pressure-space shim of SURVEY.md Appendix B, which changes
only the pressure dof map; all arithmetic is the reference's own.  BASELINE
problem data is expressed through the reference's own
forcing/boundary protocol (`stepper.py:286-341`) with `fem.assemble_load`.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from ensmhd import fem, mms  # noqa: E402
from ensmhd import mesh as rmesh  # noqa: E402
from ensmhd.ensemble import (EnsembleConfig, EnsembleState, MemberParams,  # noqa: E402
                             eddy_viscosity_at_quadrature, sample_viscosities)
from ensmhd.fem import FeKind, FeSpace  # noqa: E402
from ensmhd.stepper import (Discretization, Problem, StepKind, _rhs_block, advance,  # noqa: E402
                            assemble_shared_lhs, run)


def th_disc(mesh):
    vel = FeSpace(FeKind.VECTOR_P2, mesh)
    pres = FeSpace(FeKind.SCALAR_P1_DISC, mesh)
    pres.cell_dofs = mesh.triangles.copy()
    pres.num_scalar_dofs = mesh.num_vertices
    pres.dof_coords = mesh.vertices
    return Discretization(mesh, vel, pres, fem.mass_scalar(vel), fem.stiffness_scalar(vel),
                          fem.assemble_divergence(vel, pres),
                          fem.assemble_load(pres, np.ones_like(pres.wdet)), mesh.total_area, vel.boundary_dofs())


class BaselineForcing:
    """SURVEY.md §8.0 forcing, assembled per member the reference's way."""

    def loads(self, t, disc, config):
        q = disc.velocity.quad_coords
        x, y = q[..., 0][None], q[..., 1][None]
        nu, nm = config.nu[:, None, None], config.nu_m[:, None, None]
        e = config.nu[:, None, None] / 0.01 - 1.0
        a1 = (1 + e) * (0.02 + (nu + nm) * (1 + 0.01 * t))
        a2 = (nu - nm) * (1 + e) * (1 + 0.01 * t)
        cp = (1 + t) * np.cos(x + y)
        f1 = np.stack([a1 * np.cos(y) + cp, a1 * np.sin(x) + cp], axis=-1)
        f2 = np.stack([a2 * np.cos(y) + cp, a2 * np.sin(x) + cp], axis=-1)
        return fem.assemble_load(disc.velocity, f1), fem.assemble_load(disc.velocity, f2)


class BaselineBoundary:
    def values(self, t, disc, config):
        e = config.nu / 0.01 - 1.0
        base = fem.interpolate(lambda x, y, tt: (np.cos(y), np.sin(x)), t, disc.velocity)[disc.bdofs]
        return np.outer(2 * (1 + e) * (1 + 0.01 * t), base), np.zeros((config.num_members, disc.bdofs.size))


def baseline_initial(disc, config):
    e = config.nu / 0.01 - 1.0
    base = fem.interpolate(lambda x, y, tt: (np.cos(y), np.sin(x)), 0.0, disc.velocity)
    return np.outer(2 * (1 + e), base), np.zeros((config.num_members, disc.n_vel))


def series(report):
    return dict(energy=report.energy, div_v=report.div_v, div_w=report.div_w, residuals=report.residuals,
                l2v=report.member_l2v_sq, l2w=report.member_l2w_sq, gradv=report.member_gradv_sq,
                gradw=report.member_gradw_sq)


def setup_pins(prefix, disc):
    out = {}
    out[prefix + "cell_dofs"] = disc.velocity.cell_dofs
    out[prefix + "pres_cell_dofs"] = disc.pressure.cell_dofs
    out[prefix + "bdofs"] = disc.bdofs
    out[prefix + "mass_dense"] = disc.mass_s.toarray()
    out[prefix + "stiff_dense"] = disc.stiff_s.toarray()
    out[prefix + "div_dense"] = disc.divergence.toarray()
    out[prefix + "pintg"] = disc.pressure_integrals
    return out


def main():
    out = {}
    rng = np.random.default_rng(1234)

    # ---- A: reference-native Scott-Vogelius, paper MMS, 2 steps --------------
    mesh = rmesh.barycentric_refine(rmesh.build_structured_square(2))
    disc = Discretization.from_mesh(mesh)
    out.update(setup_pins("sv2_", disc))
    members = (MemberParams(0.01, 0.1), MemberParams(0.012, 0.09), MemberParams(0.009, 0.11))
    cfg = EnsembleConfig(members=members, coupling=1.0, mu=1.0, dt=0.05, t_end=0.1, perturbation=0.01)
    v0, w0 = mms.mms_initial_fields(disc, cfg)
    st = EnsembleState(v=v0, w=w0, q=np.zeros((3, disc.n_pres)), r=np.zeros((3, disc.n_pres)), step=0, time=0.0)
    # shared matrices and rhs at level 0 with perturbed fields (so the eddy term is nonzero)
    vp = v0 + 0.3 * rng.standard_normal(v0.shape)
    wp = w0 + 0.3 * rng.standard_normal(w0.shape)
    stp = EnsembleState(v=vp, w=wp, q=np.zeros((3, disc.n_pres)), r=np.zeros((3, disc.n_pres)), step=0, time=0.0)
    out["sv2_pert_v"], out["sv2_pert_w"] = vp, wp
    for kind, name in ((StepKind.V_STEP, "V"), (StepKind.W_STEP, "W")):
        adv, fl = (stp.mean_w, stp.fluct_w) if kind is StepKind.V_STEP else (stp.mean_v, stp.fluct_v)
        sysm = assemble_shared_lhs(kind, adv, fl, cfg, disc)
        out[f"sv2_mat{name}"] = sysm.matrix.toarray()
        lv, lw = mms.MmsForcing().loads(cfg.dt, disc, cfg)
        bv, bw = mms.MmsBoundary().values(cfg.dt, disc, cfg)
        out[f"sv2_rhs{name}"] = _rhs_block(kind, stp, lv if name == "V" else lw, bv if name == "V" else bw, cfg, disc)
    out["sv2_nut_w"] = eddy_viscosity_at_quadrature(disc.velocity, stp.fluct_w, cfg.mu, cfg.dt)
    out["sv2_loads_v"], out["sv2_loads_w"] = mms.MmsForcing().loads(0.05, disc, cfg)
    out["sv2_bvals_v"], out["sv2_bvals_w"] = mms.MmsBoundary().values(0.05, disc, cfg)
    s1, res1 = advance(stp, cfg, disc, mms.MmsForcing(), mms.MmsBoundary())
    out["sv2_step1_v"], out["sv2_step1_w"], out["sv2_step1_q"], out["sv2_step1_r"] = s1.v, s1.w, s1.q, s1.r
    out["sv2_step1_res"] = np.array(res1)
    rep, fin, _ = run(cfg, Problem(disc, v0, w0, mms.MmsForcing(), mms.MmsBoundary()))
    for k, v in series(rep).items():
        out["sv2_run_" + k] = v
    out["sv2_run_v"], out["sv2_run_w"], out["sv2_run_q"], out["sv2_run_r"] = fin.v, fin.w, fin.q, fin.r

    # ---- B: Taylor-Hood shim, n = 4, BASELINE MMS, J = 3, 3 steps ------------
    mesh4 = rmesh.build_structured_square(4)
    d4 = th_disc(mesh4)
    out.update(setup_pins("th4_", d4))
    mem = sample_viscosities((0.009, 0.011), (0.009, 0.011), 3, 0)
    cfg4 = EnsembleConfig(members=mem, coupling=1.0, mu=1.0, dt=0.01, t_end=0.03, seed=0)
    v0, w0 = baseline_initial(d4, cfg4)
    rep, fin, _ = run(cfg4, Problem(d4, v0, w0, BaselineForcing(), BaselineBoundary()))
    for k, v in series(rep).items():
        out["th4_run_" + k] = v
    out["th4_run_v"], out["th4_run_w"], out["th4_run_q"], out["th4_run_r"] = fin.v, fin.w, fin.q, fin.r
    out["th4_loads_v"], out["th4_loads_w"] = BaselineForcing().loads(0.01, d4, cfg4)

    # ---- C: BASELINE config C1 (TH 16x16, J=3, dt=0.01, 10 steps) -------------
    mesh16 = rmesh.build_structured_square(16)
    d16 = th_disc(mesh16)
    mem = sample_viscosities((0.009, 0.011), (0.009, 0.011), 3, 0)
    cfg16 = EnsembleConfig(members=mem, coupling=1.0, mu=1.0, dt=0.01, t_end=0.1, seed=0)
    v0, w0 = baseline_initial(d16, cfg16)
    rep, fin, _ = run(cfg16, Problem(d16, v0, w0, BaselineForcing(), BaselineBoundary()))
    for k, v in series(rep).items():
        out["c1_run_" + k] = v
    out["c1_run_v"], out["c1_run_w"], out["c1_run_q"], out["c1_run_r"] = fin.v, fin.w, fin.q, fin.r

    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
