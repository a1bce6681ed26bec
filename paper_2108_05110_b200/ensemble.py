"""Ensemble parameters, statistics bookkeeping and the ensemble state.

Host-side mirror of the reference's `pkg/src/ensmhd/ensemble.py` API
(`MemberParams`, `EnsembleConfig`, `viscosity_stats`, `sample_viscosities`,
Elsasser transforms, perturbation factors, `EnsembleState`).  The per-step
statistics that the reference computes in numpy (`ensemble_stats`,
`ensemble.py:216-224`; `eddy_viscosity_at_quadrature`, `ensemble.py:227-238`)
are computed on the GPU by ``csrc/member.cu``; ``EnsembleState`` here can hold
either host numpy arrays or a device-resident state produced by the GPU
engine, materialising numpy arrays only when a caller reads them.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


class DegenerateCouplingError(ValueError):
    """Magnetic field recovery is impossible at zero coupling."""


@dataclass(frozen=True)
class MemberParams:
    """(nu, nu_m) of one member (`ensemble.py:25-34`)."""

    nu: float
    nu_m: float

    def __post_init__(self):
        if self.nu <= 0.0 or self.nu_m <= 0.0:
            raise ValueError(f"viscosities must be positive, got ({self.nu}, {self.nu_m})")


@dataclass(frozen=True)
class EnsembleConfig:
    """Run parameters shared by all members (`ensemble.py:37-85`)."""

    members: tuple
    coupling: float
    mu: float
    dt: float
    t_end: float
    perturbation: float = 0.0
    seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "members", tuple(self.members))
        if len(self.members) < 1:
            raise ValueError("ensemble needs at least one member")
        if self.coupling < 0.0:
            raise ValueError("coupling must be >= 0")
        if self.dt <= 0.0 or self.t_end <= 0.0:
            raise ValueError("dt and t_end must be positive")
        if self.perturbation < 0.0:
            raise ValueError("perturbation must be >= 0")

    @property
    def num_members(self) -> int:
        return len(self.members)

    @property
    def nu(self) -> np.ndarray:
        return np.array([m.nu for m in self.members])

    @property
    def nu_m(self) -> np.ndarray:
        return np.array([m.nu_m for m in self.members])


@dataclass(frozen=True)
class ViscosityStats:
    nu_bar: float
    nu_m_bar: float
    nu_fluct: np.ndarray
    nu_m_fluct: np.ndarray
    alpha: np.ndarray

    @property
    def nonpositive_alpha(self) -> np.ndarray:
        return np.nonzero(self.alpha <= 0.0)[0]


def viscosity_stats(config: EnsembleConfig) -> ViscosityStats:
    """Means, fluctuations and alpha_j (`ensemble.py:104-115`)."""
    nu, nu_m = config.nu, config.nu_m
    nb, nmb = float(nu.mean()), float(nu_m.mean())
    nf, nmf = nu - nb, nu_m - nmb
    alpha = nb + nmb - np.abs(nu - nu_m) - np.abs(nf + nmf)
    return ViscosityStats(nb, nmb, nf, nmf, alpha)


def sample_viscosities(nu_range, nu_m_range, count: int, seed=None, deterministic_grid: bool = False):
    """Seeded uniform (or midpoint-grid) viscosity pairs (`ensemble.py:118-142`).

    Draw order matters for reproducibility: all nu first, then all nu_m.
    """
    lo, hi = float(nu_range[0]), float(nu_range[1])
    lo_m, hi_m = float(nu_m_range[0]), float(nu_m_range[1])
    if not (0.0 < lo <= hi and 0.0 < lo_m <= hi_m):
        raise ValueError("viscosity ranges must be nonempty with positive bounds")
    if count < 1:
        raise ValueError("member count must be >= 1")
    if deterministic_grid:
        offs = (np.arange(count) + 0.5) / count
        nu, nu_m = lo + offs * (hi - lo), lo_m + offs * (hi_m - lo_m)
    else:
        rng = np.random.default_rng(seed)
        nu = rng.uniform(lo, hi, size=count)
        nu_m = rng.uniform(lo_m, hi_m, size=count)
    return tuple(MemberParams(float(a), float(b)) for a, b in zip(nu, nu_m))


def elsasser_from_primitive(u, b, coupling: float):
    """(u, B) -> (u + sqrt(s) B, u - sqrt(s) B) (`ensemble.py:150-159`)."""
    if coupling < 0.0:
        raise ValueError("coupling must be >= 0")
    u, b = np.asarray(u, dtype=float), np.asarray(b, dtype=float)
    if u.shape != b.shape:
        raise ValueError(f"mismatched field shapes {u.shape} vs {b.shape}")
    rs = math.sqrt(coupling)
    return u + rs * b, u - rs * b


def primitive_from_elsasser(v, w, coupling: float):
    """(v, w) -> ((v + w)/2, (v - w)/(2 sqrt(s))) (`ensemble.py:162-175`)."""
    v, w = np.asarray(v, dtype=float), np.asarray(w, dtype=float)
    if v.shape != w.shape:
        raise ValueError(f"mismatched field shapes {v.shape} vs {w.shape}")
    u = 0.5 * (v + w)
    if coupling == 0.0:
        if not np.array_equal(v, w):
            raise DegenerateCouplingError("cannot recover B from v != w at zero coupling")
        return u, np.zeros_like(u)
    if coupling < 0.0:
        raise ValueError("coupling must be >= 0")
    return u, (v - w) / (2.0 * math.sqrt(coupling))


def perturbation_factor(j: int, eps: float) -> float:
    """1 + (-1)^(j+1) ceil(j/2) eps / 5, j 1-based (`ensemble.py:246-255`)."""
    if j < 1:
        raise ValueError("member index is 1-based")
    return 1.0 + ((-1) ** (j + 1)) * math.ceil(j / 2) * eps / 5.0


def perturbation_factors(count: int, eps: float) -> np.ndarray:
    return np.array([perturbation_factor(j, eps) for j in range(1, count + 1)])


def perturbed_member_field(base, j: int, eps: float) -> np.ndarray:
    return perturbation_factor(j, eps) * np.asarray(base, dtype=float)


# ----------------------------------------------------------------------
# ensemble state
# ----------------------------------------------------------------------


class EnsembleState:
    """Member fields at one time level (`ensemble.py:183-213`).

    ``v``/``w`` are (J, n_vel), ``q``/``r`` (J, n_pres) in the reference's dof
    order.  A state produced by the GPU engine keeps its fields in HBM (the
    engine's member-minor internal layout) and converts to numpy lazily, so a
    ``run`` never copies fields to the host unless the caller looks at them.
    The object is treated as immutable, like the reference's frozen dataclass.
    """

    __slots__ = ("_v", "_w", "_q", "_r", "step", "time", "_dev", "_mean_v", "_mean_w")

    def __init__(self, v=None, w=None, q=None, r=None, step: int = 0, time: float = 0.0, *, device=None):
        self._v = None if v is None else np.asarray(v, dtype=float)
        self._w = None if w is None else np.asarray(w, dtype=float)
        self._q = None if q is None else np.asarray(q, dtype=float)
        self._r = None if r is None else np.asarray(r, dtype=float)
        self.step = int(step)
        self.time = float(time)
        self._dev = device
        self._mean_v = None
        self._mean_w = None
        if device is None:
            if self._v is None or self._w is None:
                raise ValueError("EnsembleState needs v and w")
            if self._v.shape != self._w.shape or self._v.ndim != 2:
                raise ValueError(f"v/w must be matching (J, n_vel) arrays, got {self._v.shape}, {self._w.shape}")
            j = self._v.shape[0]
            if self._q is None:
                self._q = np.zeros((j, 0))
            if self._r is None:
                self._r = np.zeros_like(self._q)

    # -- host views ---------------------------------------------------
    def _pull(self, name):
        arr = getattr(self, "_" + name)
        if arr is None:
            arr = self._dev.to_host(name)
            setattr(self, "_" + name, arr)
        return arr

    @property
    def v(self) -> np.ndarray:
        return self._pull("v")

    @property
    def w(self) -> np.ndarray:
        return self._pull("w")

    @property
    def q(self) -> np.ndarray:
        return self._pull("q")

    @property
    def r(self) -> np.ndarray:
        return self._pull("r")

    @property
    def mean_v(self) -> np.ndarray:
        if self._mean_v is None:
            self._mean_v = self.v.mean(axis=0)
        return self._mean_v

    @property
    def mean_w(self) -> np.ndarray:
        if self._mean_w is None:
            self._mean_w = self.w.mean(axis=0)
        return self._mean_w

    @property
    def fluct_v(self) -> np.ndarray:
        return self.v - self.mean_v

    @property
    def fluct_w(self) -> np.ndarray:
        return self.w - self.mean_w

    @property
    def num_members(self) -> int:
        if self._dev is not None:
            return self._dev.num_members
        return self._v.shape[0]

    @property
    def on_device(self) -> bool:
        return self._dev is not None

    @property
    def device_state(self):
        return self._dev

    def __repr__(self):
        where = "device" if self._dev is not None else "host"
        return f"EnsembleState(J={self.num_members}, step={self.step}, time={self.time:.6g}, {where})"


def ensemble_stats(state) -> tuple:
    """(mean_v, mean_w, fluct_v, fluct_w) (`ensemble.py:216-224`)."""
    mv, mw = state.v.mean(axis=0), state.w.mean(axis=0)
    return mv, mw, state.v - mv, state.w - mw
