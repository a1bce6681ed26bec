"""Problem data: initial fields, forcing loads and Dirichlet values.

Protocol (reference `stepper.py:286-341`):
  * ``forcing.loads(t, disc, config) -> (loads_v, loads_w)``, each (J, n_vel) or None;
  * ``boundary.values(t, disc, config) -> (bv, bw)``, each (J, nb).

GPU fast path: an object may also expose
``separable(disc, config)`` returning a :class:`Separable` whose data is
``sum_k coef_k,j(t) * basis_k`` -- constant basis vectors uploaded once and a
tiny (K, J) coefficient table per step, so the host never materialises
(J, n_vel) blocks.  Objects without it go through the generic path (host
arrays uploaded each step), so any reference-style Problem still works.

Problems here: the reference's own (zero data, scaled profiles, the paper's
manufactured solution of `mms.py`) and the five BASELINE.json configurations
(C1/C2/C5 manufactured solution with u = B, C3 unit-square cavity, C4 30-long
step channel with a do-nothing outflow), following SURVEY.md §8.0.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import fe
from .discretization import Discretization
from .ensemble import (EnsembleConfig, MemberParams, elsasser_from_primitive, perturbation_factors,
                       sample_viscosities)
from .mesh import Marker, build_step_channel, build_structured_square


@dataclass
class Separable:
    """data_j(t) = sum_k coef[k, j](t) * basis[k] for both Elsasser families."""

    basis: np.ndarray          # (K, n) constant
    coef: object               # callable t -> (cv (K, J), cw (K, J))
    key: str = ""              # cache key for the uploaded basis


class RankOneMembers:
    """Member fields amp[j] * base as a lazy (J, n) array.

    The BASELINE MMS initial fields are rank one; at C5 (J=1024, n_vel=2.1M) the dense
    np.outer would be a 17 GB host array built only to be sliced per member chunk.  Row
    slices (``x[a:b]``) build just those rows; ``np.asarray(x)`` materialises the whole array
    (the reference's (J, n_vel) interface, identical values)."""

    def __init__(self, amp, base):
        self.amp = np.asarray(amp, dtype=float)
        self.base = np.asarray(base, dtype=float)
        self.shape = (self.amp.size, self.base.size)
        self.dtype = np.dtype(float)
        self.ndim = 2

    def __len__(self):
        return self.shape[0]

    def __getitem__(self, idx):
        if isinstance(idx, slice):
            return np.outer(self.amp[idx], self.base)
        return np.asarray(self)[idx]

    def __array__(self, dtype=None, copy=None):
        out = np.outer(self.amp, self.base)
        return out if dtype is None else out.astype(dtype, copy=False)


def member_rows(arr, j0, jl):
    """Rows j0 .. j0+jl of a (J, n) member array: a float64 ndarray, or a RankOneMembers of those
    rows (still lazy: the engines expand it on the device)."""
    if isinstance(arr, RankOneMembers):
        return RankOneMembers(arr.amp[j0:j0 + jl], arr.base)
    return np.asarray(arr[j0:j0 + jl], dtype=float)


class ZeroForcing:
    """No body forces (`stepper.py:286-290`)."""

    def loads(self, t, disc, config):
        return None, None


class ZeroBoundary:
    """Homogeneous Dirichlet data (`stepper.py:293-299`)."""

    def values(self, t, disc, config):
        z = np.zeros((config.num_members, disc.bdofs.size))
        return z, z

    def separable(self, disc, config):
        j = config.num_members
        basis = np.zeros((1, disc.bdofs.size))
        return Separable(basis, lambda t: (np.zeros((1, j)), np.zeros((1, j))), "zero-bc")


class ScaledProfileBoundary:
    """factors[j] * profile(x, y, t) on the Dirichlet dofs (`stepper.py:302-318`)."""

    def __init__(self, v_profile, w_profile, factors):
        self.v_profile, self.w_profile = v_profile, w_profile
        self.factors = np.asarray(factors, dtype=float)

    def values(self, t, disc, config):
        bv = fe.interpolate(self.v_profile, t, disc.velocity)[disc.bdofs]
        bw = fe.interpolate(self.w_profile, t, disc.velocity)[disc.bdofs]
        return np.outer(self.factors, bv), np.outer(self.factors, bw)


class ConstantBoundary:
    """Time-independent member-scaled data: bv_j = factors_j * base_v."""

    def __init__(self, base_v, base_w, factors):
        self.base_v = np.asarray(base_v, dtype=float)
        self.base_w = np.asarray(base_w, dtype=float)
        self.factors = np.asarray(factors, dtype=float)

    def values(self, t, disc, config):
        return np.outer(self.factors, self.base_v), np.outer(self.factors, self.base_w)

    def separable(self, disc, config):
        f = self.factors[None, :]
        z = np.zeros_like(f)
        basis = np.stack([self.base_v, self.base_w])
        return Separable(basis, lambda t: (np.vstack([f, z]), np.vstack([z, f])), f"const-bc-{id(self)}")


# ----------------------------------------------------------------------
# the paper's manufactured solution (reference `mms.py`)
# ----------------------------------------------------------------------


def paper_v(x, y, t):
    g = 1.0 + np.exp(t)
    return np.cos(y) + g * np.sin(y), np.sin(x) + g * np.cos(x)


def paper_w(x, y, t):
    g = 1.0 + np.exp(t)
    return np.cos(y) - g * np.sin(y), np.sin(x) - g * np.cos(x)


def paper_forcing_values(x, y, t, c, nu, nu_m):
    """Elsasser forcing of the paper MMS (`mms.py:79-108`): Delta v = -v, Delta w = -w."""
    g, et = 1.0 + np.exp(t), np.exp(t)
    sx, cx, sy, cy = np.sin(x), np.cos(x), np.sin(y), np.cos(y)
    v1, v2 = cy + g * sy, sx + g * cx
    w1, w2 = cy - g * sy, sx - g * cx
    gq = g * np.cos(x + y)
    a, b = 0.5 * (nu + nu_m) * c, 0.5 * (nu - nu_m) * c
    f1 = (c * et * sy + c * c * w2 * (g * cy - sy) + a * v1 + b * w1 + gq,
          c * et * cx + c * c * w1 * (cx - g * sx) + a * v2 + b * w2 + gq)
    f2 = (-c * et * sy + c * c * v2 * (-sy - g * cy) + a * w1 + b * v1 + gq,
          -c * et * cx + c * c * v1 * (cx + g * sx) + a * w2 + b * v2 + gq)
    return f1, f2


class PaperMmsForcing:
    """Assembled paper-MMS loads for all members (`mms.py:125-137`)."""

    def loads(self, t, disc, config):
        q = disc.velocity.quad_coords
        x, y = q[..., 0], q[..., 1]
        c = perturbation_factors(config.num_members, config.perturbation)[:, None, None]
        f1, f2 = paper_forcing_values(x, y, t, c, config.nu[:, None, None], config.nu_m[:, None, None])
        return (fe.load_vector(disc.velocity, np.stack(f1, axis=-1)),
                fe.load_vector(disc.velocity, np.stack(f2, axis=-1)))


class PaperMmsBoundary:
    """Exact paper-MMS member fields on the Dirichlet dofs (`mms.py:140-147`)."""

    def values(self, t, disc, config):
        f = perturbation_factors(config.num_members, config.perturbation)
        bv = fe.interpolate(paper_v, t, disc.velocity)[disc.bdofs]
        bw = fe.interpolate(paper_w, t, disc.velocity)[disc.bdofs]
        return np.outer(f, bv), np.outer(f, bw)

    def separable(self, disc, config):
        # base_v(t) = (cos y, sin x) + g(t) (sin y, cos x), base_w = (cos y, sin x) - g(t) (sin y, cos x)
        f = perturbation_factors(config.num_members, config.perturbation)[None, :]
        e1 = fe.interpolate(lambda x, y, t: (np.cos(y), np.sin(x)), 0.0, disc.velocity)[disc.bdofs]
        e2 = fe.interpolate(lambda x, y, t: (np.sin(y), np.cos(x)), 0.0, disc.velocity)[disc.bdofs]

        def coef(t):
            g = 1.0 + math.exp(t)
            return np.vstack([f, g * f]), np.vstack([f, -g * f])

        return Separable(np.stack([e1, e2]), coef, "paper-mms-bc")


def paper_mms_initial_fields(disc, config):
    f = perturbation_factors(config.num_members, config.perturbation)
    return (np.outer(f, fe.interpolate(paper_v, 0.0, disc.velocity)),
            np.outer(f, fe.interpolate(paper_w, 0.0, disc.velocity)))


# ----------------------------------------------------------------------
# BASELINE configs C1 / C2 / C5: u_j = B_j = (1+eps_j)(1+0.01 t)(cos y, sin x)
# ----------------------------------------------------------------------


def _cs(x, y, t):
    return np.cos(y), np.sin(x)


class BaselineMms:
    """Manufactured problem of BASELINE.json configs C1, C2, C5.

    With s = 1: v_j = 2 u_j, w_j = 0, q_j = r_j = (1+t) sin(x+y) and
      f1_j = (1+e_j)[0.02 + (nu_j+nu_mj)(1+0.01t)] (cos y, sin x) + (1+t) cos(x+y) (1,1)
      f2_j = (nu_j-nu_mj)(1+e_j)(1+0.01t) (cos y, sin x)        + (1+t) cos(x+y) (1,1)
    where e_j = nu_j/nu_bar0 - 1 (nu_bar0 = 0.01).  Loads are separable:
    load_j(t) = a_j(t) L_c + b(t) L_p with L_c, L_p assembled once.
    """

    def __init__(self, nu0: float = 0.01):
        self.nu0 = nu0

    def eps(self, config):
        return config.nu / self.nu0 - 1.0

    def _check(self, config):
        if abs(config.coupling - 1.0) > 1e-15:
            raise ValueError("BaselineMms is derived for coupling s = 1")

    def _basis(self, disc):
        key = ("baseline-mms-loads", id(disc))
        if key not in disc._cache:
            q = disc.velocity.quad_coords
            x, y = q[..., 0], q[..., 1]
            lc = fe.load_vector(disc.velocity, np.stack([np.cos(y), np.sin(x)], axis=-1))
            cp = np.cos(x + y)
            lp = fe.load_vector(disc.velocity, np.stack([cp, cp], axis=-1))
            disc._cache[key] = np.stack([lc, lp])
        return disc._cache[key]

    def _coef(self, t, config):
        e = self.eps(config)
        nu, nm = config.nu, config.nu_m
        a1 = (1.0 + e) * (0.02 + (nu + nm) * (1.0 + 0.01 * t))
        a2 = (nu - nm) * (1.0 + e) * (1.0 + 0.01 * t)
        b = np.full_like(a1, 1.0 + t)
        return np.stack([a1, b]), np.stack([a2, b])

    # forcing protocol
    def loads(self, t, disc, config):
        self._check(config)
        basis = self._basis(disc)
        cv, cw = self._coef(t, config)
        return cv.T @ basis, cw.T @ basis

    # boundary protocol
    def values(self, t, disc, config):
        self._check(config)
        base = fe.interpolate(_cs, t, disc.velocity)[disc.bdofs]
        amp = 2.0 * (1.0 + self.eps(config)) * (1.0 + 0.01 * t)
        return np.outer(amp, base), np.zeros((config.num_members, disc.bdofs.size))

    def forcing_separable(self, disc, config):
        self._check(config)
        return Separable(self._basis(disc), lambda t: self._coef(t, config), f"baseline-mms-loads-{id(disc)}")

    def boundary_separable(self, disc, config):
        self._check(config)
        base = fe.interpolate(_cs, 0.0, disc.velocity)[disc.bdofs][None, :]
        e = self.eps(config)

        def coef(t):
            amp = (2.0 * (1.0 + e) * (1.0 + 0.01 * t))[None, :]
            return amp, np.zeros_like(amp)

        return Separable(base, coef, f"baseline-mms-bc-{id(disc)}")

    def initial_fields(self, disc, config):
        base = fe.interpolate(_cs, 0.0, disc.velocity)
        amp = 2.0 * (1.0 + self.eps(config))
        # <w>(0) = 0: a zero rank-one product (0 * +0 = +0, bitwise np.zeros)
        return RankOneMembers(amp, base), RankOneMembers(np.zeros(config.num_members), np.zeros(disc.n_vel))

    def exact_v(self, t, disc, config):
        base = fe.interpolate(_cs, t, disc.velocity)
        return np.outer(2.0 * (1.0 + self.eps(config)) * (1.0 + 0.01 * t), base)


class BaselineMmsExact:
    """Exact ensemble means of the BASELINE MMS for run(..., exact=...): <v>(t) = 2(1+<e>)(1+0.01t)
    (cos y, sin x), <w> = 0 (nodal interpolants, `experiments.py:59-73`)."""

    def __init__(self, nu0: float = 0.01):
        self.nu0 = nu0

    def mean_separable(self, disc, config):
        base = fe.interpolate(_cs, 0.0, disc.velocity)[None, :]
        e = float(np.mean(config.nu / self.nu0 - 1.0))
        return Separable(base, lambda t: (np.array([2.0 * (1.0 + e) * (1.0 + 0.01 * t)]), np.zeros(1)),
                         "baseline-mms-exact")

    def mean_v(self, x, y, t, config):
        a = 2.0 * (1.0 + float(np.mean(config.nu / self.nu0 - 1.0))) * (1.0 + 0.01 * t)
        return a * np.cos(y), a * np.sin(x)


class PaperMmsExact:
    """The reference's convergence targets for the paper MMS: base_v, base_w (`experiments.py:146-147`,
    `mms.py:26-37`): (cos y, sin x) +- g(t) (sin y, cos x), g = 1 + e^t."""

    def mean_separable(self, disc, config):
        e1 = fe.interpolate(lambda x, y, t: (np.cos(y), np.sin(x)), 0.0, disc.velocity)
        e2 = fe.interpolate(lambda x, y, t: (np.sin(y), np.cos(x)), 0.0, disc.velocity)

        def coef(t):
            g = 1.0 + math.exp(t)
            return np.array([1.0, g]), np.array([1.0, -g])

        return Separable(np.stack([e1, e2]), coef, "paper-mms-exact")


class _ForcingView:
    def __init__(self, owner):
        self.owner = owner

    def loads(self, t, disc, config):
        return self.owner.loads(t, disc, config)

    def separable(self, disc, config):
        return self.owner.forcing_separable(disc, config)


class _BoundaryView:
    def __init__(self, owner):
        self.owner = owner

    def values(self, t, disc, config):
        return self.owner.values(t, disc, config)

    def separable(self, disc, config):
        return self.owner.boundary_separable(disc, config)


# ----------------------------------------------------------------------
# config builders (BASELINE.json configs[0..4])
# ----------------------------------------------------------------------

CONFIGS = {
    "C1": dict(kind="mms", n=16, J=3, dt=0.01, steps=10),
    "C2": dict(kind="mms", n=128, J=20, dt=0.005, steps=100),
    "C3": dict(kind="cavity", n=256, J=64, dt=0.01, steps=500, coupling=1.0),
    "C4": dict(kind="channel", k=8, J=128, dt=0.02, steps=1000, delta=0.1),
    "C5": dict(kind="mms", n=512, J=1024, dt=0.002, steps=50),
}


def build_case(name: str, seed: int = 0, mu: float = 1.0, pressure: str = "th", **over):
    """Return (disc, config, problem) for a BASELINE configuration.

    ``over`` overrides n / J / dt / steps / coupling / delta / k (parity tests
    shrink the big configs).  Members are seeded draws (ν draws then ν_m draws,
    `ensemble.py:139-141`).
    """
    from .stepper import Problem  # local import: stepper pulls in the GPU engine

    spec = dict(CONFIGS[name])
    spec.update(over)
    kind, J, dt, steps = spec["kind"], int(spec["J"]), float(spec["dt"]), int(spec["steps"])
    t_end = dt * steps
    if kind == "mms":
        mesh = build_structured_square(int(spec["n"]))
        disc = Discretization.from_mesh(mesh, pressure=pressure)
        members = sample_viscosities((0.009, 0.011), (0.009, 0.011), J, seed)
        config = EnsembleConfig(members, coupling=1.0, mu=mu, dt=dt, t_end=t_end, seed=seed)
        mms = BaselineMms()
        v0, w0 = mms.initial_fields(disc, config)
        return disc, config, Problem(disc, v0, w0, _ForcingView(mms), _BoundaryView(mms))
    if kind == "cavity":
        s = float(spec.get("coupling", 1.0))
        mesh = build_structured_square(int(spec["n"]), per_side_markers=True)
        disc = Discretization.from_mesh(mesh, pressure=pressure)
        rng = np.random.default_rng(seed)
        eps = rng.uniform(-0.05, 0.05, size=J)
        eta = rng.uniform(-0.01, 0.01, size=J)
        nu = (1.0 / 15000.0) * (1.0 + eps)
        members = tuple(MemberParams(float(a), float(a)) for a in nu)
        config = EnsembleConfig(members, coupling=s, mu=mu, dt=dt, t_end=t_end, seed=seed)
        vel = disc.velocity
        sc = vel.boundary_scalar_dofs()
        lid = np.isin(sc, vel.boundary_scalar_dofs(markers=Marker.LID))
        nsb = sc.size
        # u = (1+eta_j)(1,0) on the lid (endpoints included, `experiments.py:293-298`), 0 elsewhere; B = (1,0)
        ub = np.concatenate([lid.astype(float), np.zeros(nsb)])
        bb = np.concatenate([np.ones(nsb), np.zeros(nsb)])
        rs = math.sqrt(s)
        basis = np.stack([ub, bb])               # v = (1+eta) ub + rs bb ; w = (1+eta) ub - rs bb
        fac = 1.0 + eta

        class CavityBoundary:
            def values(self, t, disc_, config_):
                return np.outer(fac, ub) + rs * bb[None, :], np.outer(fac, ub) - rs * bb[None, :]

            def separable(self, disc_, config_):
                one = np.ones((1, J))
                return Separable(basis, lambda t: (np.vstack([fac[None, :], rs * one]),
                                                   np.vstack([fac[None, :], -rs * one])), f"cavity-bc-{id(self)}")

        ns = disc.n_scalar
        u0 = np.zeros(disc.n_vel)
        b0 = np.concatenate([np.ones(ns), np.zeros(ns)])
        v0b, w0b = elsasser_from_primitive(u0, b0, s)
        v0, w0 = np.tile(v0b, (J, 1)), np.tile(w0b, (J, 1))
        return disc, config, Problem(disc, v0, w0, ZeroForcing(), CavityBoundary())
    if kind == "channel":
        s = float(spec.get("coupling", 0.01))
        delta = float(spec.get("delta", 0.1))
        k = int(spec.get("k", 8))
        mesh = build_step_channel(length=float(spec.get("length", 30.0)), cells_per_unit=k)
        disc = Discretization.from_mesh(mesh, pressure=pressure,
                                        dirichlet_markers=(Marker.WALL, Marker.INLET), pin_pressure=False)
        rng = np.random.default_rng(seed)
        eps = rng.uniform(-delta, delta, size=J) if delta > 0 else np.zeros(J)
        nu = (1.0 / 600.0) * (1.0 + eps)
        members = tuple(MemberParams(float(a), float(a)) for a in nu)
        config = EnsembleConfig(members, coupling=s, mu=mu, dt=dt, t_end=t_end, perturbation=delta, seed=seed)
        vel = disc.velocity
        sc = vel.boundary_scalar_dofs((Marker.WALL, Marker.INLET))
        inlet = np.isin(sc, vel.boundary_scalar_dofs(markers=Marker.INLET))
        yc = vel.dof_coords[sc, 1]
        ux = np.where(inlet, yc * (10.0 - yc) / 25.0, 0.0)
        ub = np.concatenate([ux, np.zeros(sc.size)])
        bb = np.concatenate([np.zeros(sc.size), np.ones(sc.size)])
        rs = math.sqrt(s)
        fac = 1.0 + eps
        basis = np.stack([ub, bb])

        class ChannelBoundary:
            def values(self, t, disc_, config_):
                return np.outer(fac, ub) + rs * bb[None, :], np.outer(fac, ub) - rs * bb[None, :]

            def separable(self, disc_, config_):
                one = np.ones((1, J))
                return Separable(basis, lambda t: (np.vstack([fac[None, :], rs * one]),
                                                   np.vstack([fac[None, :], -rs * one])), f"channel-bc-{id(self)}")

        prof = fe.interpolate(lambda x, y, t: (y * (10.0 - y) / 25.0, np.zeros_like(x)), 0.0, vel)
        v0 = np.outer(fac, prof)
        return disc, config, Problem(disc, v0, v0.copy(), ZeroForcing(), ChannelBoundary())
    raise ValueError(f"unknown config kind {kind}")
