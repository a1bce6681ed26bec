"""``Discretization``: mesh, spaces and constant operators of one domain.

Mirror of the reference's `stepper.Discretization` (`stepper.py:49-123`):
same fields, same properties (`n_scalar`, `n_vel`, `n_pres`, `n_total`,
`pin_row`), same helpers (`apply_componentwise`, `apply_mass`,
`apply_stiffness`, `mean_zero_pressure`).  Host-side setup only: the GPU
engine uploads these operators once per mesh.

Additions, each needed by a BASELINE.json config and defaulting to the
reference's behaviour:
  * ``pressure="disc"`` (reference Scott-Vogelius pair, `stepper.py:66-67`) or
    ``"th"`` (Taylor-Hood, configs C1-C5);
  * ``dirichlet_markers``: restrict the Dirichlet set (C4's do-nothing outflow;
    the reference always takes the whole boundary, `stepper.py:82`);
  * ``pin_pressure``: pin the first pressure dof and mean-zero after the solve
    (reference behaviour, `stepper.py:214-215`, `stepper.py:389-390`), or
    neither (C4, where the outflow fixes the pressure level).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import fe
from .mesh import Marker


@dataclass
class Discretization:
    mesh: object
    velocity: fe.VelocitySpace
    pressure: fe.PressureSpace
    mass_s: sp.csr_matrix
    stiff_s: sp.csr_matrix
    divergence: sp.csr_matrix
    pressure_integrals: np.ndarray
    area: float
    bdofs: np.ndarray
    pin_pressure: bool = True
    saddle_symbolic: object = None
    _cache: dict = field(default_factory=dict, repr=False)

    @classmethod
    def from_mesh(cls, mesh, pressure: str = "disc", dirichlet_markers=None, pin_pressure: bool = True):
        vel = fe.VelocitySpace(mesh)
        pres = fe.PressureSpace(mesh, pressure)
        return cls(
            mesh=mesh,
            velocity=vel,
            pressure=pres,
            mass_s=fe.mass_scalar(vel),
            stiff_s=fe.stiffness_scalar(vel),
            divergence=fe.divergence(vel, pres),
            pressure_integrals=fe.pressure_integrals(pres),
            area=mesh.total_area,
            bdofs=vel.boundary_dofs(dirichlet_markers),
            pin_pressure=pin_pressure,
        )

    @property
    def n_scalar(self) -> int:
        return self.velocity.num_scalar_dofs

    @property
    def n_vel(self) -> int:
        return 2 * self.n_scalar

    @property
    def n_pres(self) -> int:
        return self.pressure.num_scalar_dofs

    @property
    def n_total(self) -> int:
        return self.n_vel + self.n_pres

    @property
    def pin_row(self) -> int:
        """Global row of the pinned pressure dof (first pressure dof, `stepper.py:101-104`)."""
        return self.n_vel

    @property
    def constrained_rows(self) -> np.ndarray:
        """Rows replaced by identity rows: Dirichlet dofs, then the pin."""
        if self.pin_pressure:
            return np.concatenate([self.bdofs, [self.pin_row]]).astype(np.int64)
        return self.bdofs.astype(np.int64)

    def apply_componentwise(self, scalar_mat, fields) -> np.ndarray:
        x = np.asarray(fields, dtype=float)
        comp = x.reshape(-1, 2, self.n_scalar)
        out = (scalar_mat @ comp.reshape(-1, self.n_scalar).T).T
        return out.reshape(x.shape)

    def apply_mass(self, fields) -> np.ndarray:
        return self.apply_componentwise(self.mass_s, fields)

    def apply_stiffness(self, fields) -> np.ndarray:
        return self.apply_componentwise(self.stiff_s, fields)

    def mean_zero_pressure(self, p) -> np.ndarray:
        """Subtract the discrete mean (`stepper.py:119-123`); identity when unpinned."""
        p = np.asarray(p, dtype=float)
        if not self.pin_pressure:
            return p.copy()
        means = (p @ self.pressure_integrals) / self.area
        return p - means[..., None]


__all__ = ["Discretization", "Marker"]
