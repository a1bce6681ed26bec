"""Golden fixtures at the BASELINE sizes, produced by the REAL reference.

Build container only (the reference does not exist on the GPU box):

    OMP_NUM_THREADS=1 python tests/golden/make_golden_large.py C2        # 100 steps, ~75 min
    OMP_NUM_THREADS=1 python tests/golden/make_golden_large.py C3s1      # 2 steps, ~30 min, ~19 GB
    ... C3s0.1, C3s0.01, C4d0.01, C4d0.1

Each case runs the unmodified reference package `ensmhd` (SuperLU backend)
on the BASELINE configuration as stated, with the
Taylor-Hood pressure-space shim of SURVEY.md Appendix B.  C4's do-nothing
outflow cannot be expressed by the reference (`stepper.py:82` makes every
boundary dof Dirichlet, `stepper.py:215` pins a pressure, `stepper.py:389-390`
mean-zeroes it), so its variant is applied *around* the reference code:
the Dirichlet set is WALL+INLET, the pin call of `assemble_shared_lhs` is a
no-op and `mean_zero_pressure` is the identity.  Everything else is the
reference's own arithmetic.

A full (J, n) field block at these sizes is 20-300 MB, so each fixture keeps
(1) the whole per-step RunReport series (energies, member L2/H1 norms,
divergences, residuals -- quadratic forms of the *full* fields), (2) every
member field and the ensemble means at a fixed uniform subsample of dofs,
and (3) four seeded Gaussian projections of every full member field
(`projection_matrix`).  tests/test_gpu_large_parity.py recomputes the same
summaries from the GPU run.
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

PROJ_SEED = 20260
NPROJ = 4


def projection_matrix(n: int) -> np.ndarray:
    """(NPROJ, n) seeded Gaussian projection vectors (shared with the tests)."""
    return np.random.default_rng(PROJ_SEED + n).standard_normal((NPROJ, n))


def strides(n: int, J: int):
    """Subsample strides: ~4k dofs of the means, ~16k values over all members of a field."""
    return max(1, n // 4096), max(1, (n * J) // 16384)


def summarize(prefix: str, v, w, q, r, members: bool = True) -> dict:
    """Subsampled fields + full-field projections of one ensemble state (arrays (J, n)).

    Means of all four fields at ~4k dofs, four Gaussian projections of every full member field,
    and (``members``) every member's v and w at a common subsample (~16k values per field)."""
    out = {}
    for name, a in (("v", v), ("w", w), ("q", q), ("r", r)):
        a = np.asarray(a, dtype=float)
        sm, sj = strides(a.shape[1], a.shape[0])
        out[f"{prefix}{name}_mean_sub"] = a.mean(axis=0)[::sm]
        if members and name in "vw":
            out[f"{prefix}{name}_sub"] = a[:, ::sj]
        out[f"{prefix}{name}_proj"] = projection_matrix(a.shape[1]) @ a.T
    return out


CASES = {
    "C2": dict(kind="mms", n=128, J=20, dt=0.005, steps=100, snaps=(10,)),
    "C3s1": dict(kind="cavity", n=256, J=64, dt=0.01, steps=2, coupling=1.0, snaps=(1,)),
    "C3s0.1": dict(kind="cavity", n=256, J=64, dt=0.01, steps=2, coupling=0.1, snaps=(1,)),
    "C3s0.01": dict(kind="cavity", n=256, J=64, dt=0.01, steps=2, coupling=0.01, snaps=(1,)),
    "C4d0.01": dict(kind="channel", k=8, J=128, dt=0.02, steps=3, delta=0.01, snaps=(1,)),
    "C4d0.1": dict(kind="channel", k=8, J=128, dt=0.02, steps=3, delta=0.1, snaps=(1,)),
    # small twins of C3 / C4 (seconds; used by the CPU check of this script's problem set-up)
    "C3tiny": dict(kind="cavity", n=6, J=4, dt=0.01, steps=2, coupling=0.1, snaps=(1,)),
    "C4tiny": dict(kind="channel", k=1, J=3, dt=0.02, steps=2, delta=0.1, snaps=(1,), length=8.0),
}


def fixture_path(case: str) -> str:
    return os.path.join(HERE, f"large_{case}.npz")


def main(case: str):
    sys.path.insert(0, "/root/reference/pkg/src")
    from ensmhd import fem, stepper  # noqa: F401
    from ensmhd import mesh as rmesh
    from ensmhd.ensemble import EnsembleConfig, MemberParams, elsasser_from_primitive, sample_viscosities
    from ensmhd.fem import FeKind, FeSpace
    from ensmhd.stepper import Discretization, Problem, run

    spec = CASES[case]
    J, dt, steps = spec["J"], spec["dt"], spec["steps"]
    t_end = dt * steps

    def th_disc(mesh, bdofs=None, cls=Discretization):
        vel = FeSpace(FeKind.VECTOR_P2, mesh)
        pres = FeSpace(FeKind.SCALAR_P1_DISC, mesh)
        pres.cell_dofs = mesh.triangles.copy()
        pres.num_scalar_dofs = mesh.num_vertices
        pres.dof_coords = mesh.vertices
        return cls(mesh, vel, pres, fem.mass_scalar(vel), fem.stiffness_scalar(vel),
                   fem.assemble_divergence(vel, pres), fem.assemble_load(pres, np.ones_like(pres.wdet)),
                   mesh.total_area, vel.boundary_dofs() if bdofs is None else bdofs(vel))

    t0 = time.time()
    if spec["kind"] == "mms":
        mesh = rmesh.build_structured_square(spec["n"])
        disc = th_disc(mesh)
        mem = sample_viscosities((0.009, 0.011), (0.009, 0.011), J, 0)
        cfg = EnsembleConfig(members=mem, coupling=1.0, mu=1.0, dt=dt, t_end=t_end, seed=0)
        e = cfg.nu / 0.01 - 1.0

        class Forcing:
            def loads(self, t, disc, config):
                qc = disc.velocity.quad_coords
                x, y = qc[..., 0][None], qc[..., 1][None]
                nu, nm = config.nu[:, None, None], config.nu_m[:, None, None]
                ee = e[:, None, None]
                a1 = (1 + ee) * (0.02 + (nu + nm) * (1 + 0.01 * t))
                a2 = (nu - nm) * (1 + ee) * (1 + 0.01 * t)
                cp = (1 + t) * np.cos(x + y)
                f1 = np.stack([a1 * np.cos(y) + cp, a1 * np.sin(x) + cp], axis=-1)
                f2 = np.stack([a2 * np.cos(y) + cp, a2 * np.sin(x) + cp], axis=-1)
                return fem.assemble_load(disc.velocity, f1), fem.assemble_load(disc.velocity, f2)

        class Boundary:
            def values(self, t, disc, config):
                base = fem.interpolate(lambda x, y, tt: (np.cos(y), np.sin(x)), t, disc.velocity)[disc.bdofs]
                return np.outer(2 * (1 + e) * (1 + 0.01 * t), base), np.zeros((J, disc.bdofs.size))

        base = fem.interpolate(lambda x, y, tt: (np.cos(y), np.sin(x)), 0.0, disc.velocity)
        v0, w0 = np.outer(2 * (1 + e), base), np.zeros((J, disc.n_vel))
        problem = Problem(disc, v0, w0, Forcing(), Boundary())
    elif spec["kind"] == "cavity":
        s = spec["coupling"]
        mesh = rmesh.build_structured_square(spec["n"], per_side_markers=True)
        disc = th_disc(mesh)
        rng = np.random.default_rng(0)
        eps = rng.uniform(-0.05, 0.05, size=J)
        eta = rng.uniform(-0.01, 0.01, size=J)
        nu = (1.0 / 15000.0) * (1.0 + eps)
        cfg = EnsembleConfig(members=tuple(MemberParams(float(a), float(a)) for a in nu), coupling=s, mu=1.0,
                             dt=dt, t_end=t_end, seed=0)
        vel = disc.velocity
        sc = vel.boundary_scalar_dofs()
        lid = np.isin(sc, vel.boundary_scalar_dofs(markers=rmesh.Marker.LID))
        ux = np.concatenate([lid.astype(float), np.zeros(sc.size)])
        bb = np.concatenate([np.ones(sc.size), np.zeros(sc.size)])
        rs = math.sqrt(s)
        bv = np.outer(1.0 + eta, ux) + rs * bb[None, :]
        bw = np.outer(1.0 + eta, ux) - rs * bb[None, :]

        class Boundary:
            def values(self, t, disc, config):
                return bv, bw

        class NoForcing:
            def loads(self, t, disc, config):
                return None, None

        ns = disc.n_scalar
        v0b, w0b = elsasser_from_primitive(np.zeros(disc.n_vel), np.concatenate([np.ones(ns), np.zeros(ns)]), s)
        problem = Problem(disc, np.tile(v0b, (J, 1)), np.tile(w0b, (J, 1)), NoForcing(), Boundary())
    else:
        # C4: the 30-long channel (a variant of `mesh.py:184-234`, which is 40 long) in the reference's Mesh
        sys.path.insert(0, ROOT)
        from paper_2108_05110_b200.mesh import build_step_channel
        m = build_step_channel(length=spec.get("length", 30.0), height=spec.get("height", 10.0),
                               cells_per_unit=spec["k"])
        mesh = rmesh.Mesh(np.array(m.vertices), np.array(m.triangles), np.array(m.boundary_edges),
                          np.array(m.boundary_markers))
        height = spec.get("height", 10.0)

        class DoNothingDisc(Discretization):
            def mean_zero_pressure(self, p):          # outflow fixes the pressure level
                return np.asarray(p, dtype=float)

        disc = th_disc(mesh, bdofs=lambda vel: vel.boundary_dofs(markers=(rmesh.Marker.WALL, rmesh.Marker.INLET)),
                       cls=DoNothingDisc)
        pin = disc.pin_row
        orig = fem.replace_rows_with_identity

        def no_pin(matrix, rows):                     # the pin call (`stepper.py:215`) becomes a no-op
            rows = np.asarray(rows)
            if rows.size == 1 and int(rows[0]) == pin:
                return matrix.tocsr()
            return orig(matrix, rows)

        fem.replace_rows_with_identity = no_pin
        delta = spec["delta"]
        rng = np.random.default_rng(0)
        eps = rng.uniform(-delta, delta, size=J)
        nu = (1.0 / 600.0) * (1.0 + eps)
        s = 0.01
        cfg = EnsembleConfig(members=tuple(MemberParams(float(a), float(a)) for a in nu), coupling=s, mu=1.0,
                             dt=dt, t_end=t_end, perturbation=delta, seed=0)
        vel = disc.velocity
        sc = vel.boundary_scalar_dofs((rmesh.Marker.WALL, rmesh.Marker.INLET))
        inlet = np.isin(sc, vel.boundary_scalar_dofs(markers=rmesh.Marker.INLET))
        yc = vel.dof_coords[sc, 1]
        ub = np.concatenate([np.where(inlet, yc * (height - yc) / 25.0, 0.0), np.zeros(sc.size)])
        bb = np.concatenate([np.zeros(sc.size), np.ones(sc.size)])
        rs = math.sqrt(s)
        fac = 1.0 + eps
        bv = np.outer(fac, ub) + rs * bb[None, :]
        bw = np.outer(fac, ub) - rs * bb[None, :]

        class Boundary:
            def values(self, t, disc, config):
                return bv, bw

        class NoForcing:
            def loads(self, t, disc, config):
                return None, None

        prof = fem.interpolate(lambda x, y, t: (y * (height - y) / 25.0, np.zeros_like(x)), 0.0, vel)
        v0 = np.outer(fac, prof)
        problem = Problem(disc, v0, v0.copy(), NoForcing(), Boundary())
    print(f"[{case}] setup {time.time() - t0:.1f} s, n_total={disc.n_total}, J={J}", flush=True)

    tick = [time.time()]

    def observer(step, t, state):
        now = time.time()
        print(f"[{case}] step {step} t={t:.4f} ({now - tick[0]:.1f} s)", flush=True)
        tick[0] = now

    rep, fin, snaps = run(cfg, problem, observer=observer, snapshot_steps=tuple(spec["snaps"]))
    out = dict(energy=rep.energy, div_v=rep.div_v, div_w=rep.div_w, residuals=rep.residuals,
               l2v=rep.member_l2v_sq, l2w=rep.member_l2w_sq, gradv=rep.member_gradv_sq, gradw=rep.member_gradw_sq,
               wall_clock=rep.wall_clock, steps=np.array(steps), snaps=np.array(spec["snaps"]))
    for k, st in snaps.items():
        out.update(summarize(f"s{k}_", st.v, st.w, st.q, st.r, members=False))
    out.update(summarize(f"s{steps}_", fin.v, fin.w, fin.q, fin.r))
    # full final state kept outside the repo, so the summaries can be re-cut without re-running
    np.savez(f"/tmp/large_{case}_final.npz", v=fin.v, w=fin.w, q=fin.q, r=fin.r)
    np.savez_compressed(fixture_path(case), **out)
    print(f"[{case}] wrote {fixture_path(case)} ({os.path.getsize(fixture_path(case))} bytes) "
          f"in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:]:
        main(c)
