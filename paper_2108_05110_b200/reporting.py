"""Error norms, rate tables and output formats.

The reference computes the paper's convergence tables from the ensemble means
of a run (`experiments.py:59-115`) and writes CSV tables and legacy-VTK field
snapshots (`reporting.py:33-110`; CSV schema `SPEC.md:567`).  Here:

* `error_norm_21` is the discrete L2(0,T;H1) norm of the ensemble-average error
  sqrt(dt sum_{n>=1} ||<z>^n - I_h z(t^n)||_H1^2).  `run(..., exact=...)`
  accumulates its summands ON THE DEVICE every step (`ens_mean_error`: the mean
  error against a separable exact field in the mass and stiffness forms), so a
  convergence study never copies the means to the host; the host function here
  takes host means (the reference's own interface) and pins the device series.
* `compute_rate`, `RateRow`, `RateTable.from_errors` restate the reference's rate
  bookkeeping; `write_rate_csv` / `write_energy_csv` / `write_distance_csv` /
  `write_vtk` write the reference's formats byte for byte (same headers, number
  formats and VTK layout), `vertex_fields` samples the ensemble-average fields at
  the vertices as the reference exports them.  Figures (matplotlib) are out of scope.
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import fe


def ensure_dir(path) -> Path:
    out = Path(path)
    out.mkdir(parents=True, exist_ok=True)
    return out


# ----------------------------------------------------------------------
# error norms and rates (`experiments.py:59-115`)
# ----------------------------------------------------------------------


def h1_norm_sq(disc, coeffs) -> float:
    """x^T M x + x^T K x per component (the reference's `fem.norm_h1` squared, `fem.py:502-505`)."""
    x = np.asarray(coeffs, dtype=float)
    return float(x @ disc.apply_mass(x) + x @ disc.apply_stiffness(x))


def error_norm_21(means, times, exact, disc) -> float:
    """sqrt(dt sum_{n=1..M} ||means[n] - I_h exact(t^n)||_H1^2) (`experiments.py:59-73`).

    ``means``: (M+1, n_vel) ensemble means per level (reference order); ``exact``: f(x, y, t) ->
    (fx, fy); ``disc``: the Discretization (its velocity space interpolates ``exact``)."""
    times = np.asarray(times, dtype=float)
    dt = float(times[1] - times[0])
    total = 0.0
    for n in range(1, len(times)):
        diff = np.asarray(means[n], dtype=float) - fe.interpolate(exact, float(times[n]), disc.velocity)
        total += h1_norm_sq(disc, diff)
    return math.sqrt(dt * total)


def error_norm_21_from_series(err_sq, dt) -> float:
    """The same norm from per-level squared H1 errors (entry 0, the initial level, is excluded)."""
    return math.sqrt(dt * float(np.sum(np.asarray(err_sq, dtype=float)[1:])))


def compute_rate(e1: float, e2: float, s1: float, s2: float) -> float:
    """Observed order log(e1/e2) / log(s1/s2) (`experiments.py:76-82`)."""
    if e1 <= 0.0 or e2 <= 0.0 or s1 <= 0.0 or s2 <= 0.0:
        raise ValueError("errors and step sizes must be positive")
    if s1 == s2:
        raise ValueError("step sizes must differ")
    return math.log(e1 / e2) / math.log(s1 / s2)


@dataclass(frozen=True)
class RateRow:
    step: float
    err_v: float
    rate_v: float | None
    err_w: float
    rate_w: float | None


@dataclass(frozen=True)
class RateTable:
    """Rows of (h or dt, error, observed rate) for both Elsasser fields (`experiments.py:85-115`)."""

    label: str
    variable: str  # "h" or "dt"
    rows: tuple

    @classmethod
    def from_errors(cls, label, variable, steps, errs_v, errs_w) -> "RateTable":
        rows = []
        for i, (s, ev, ew) in enumerate(zip(steps, errs_v, errs_w)):
            if i == 0:
                rows.append(RateRow(s, ev, None, ew, None))
            else:
                rows.append(RateRow(s, ev, compute_rate(errs_v[i - 1], ev, steps[i - 1], s), ew,
                                    compute_rate(errs_w[i - 1], ew, steps[i - 1], s)))
        return cls(label, variable, tuple(rows))


# ----------------------------------------------------------------------
# CSV (`reporting.py:33-78`)
# ----------------------------------------------------------------------


def write_rate_csv(path, table) -> Path:
    """Schema h_or_dt, err_v, rate_v, err_w, rate_w; rates blank on the first row (`SPEC.md:567`)."""
    path = Path(path)
    with path.open("w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["h_or_dt", "err_v", "rate_v", "err_w", "rate_w"])
        for row in table.rows:
            w.writerow([f"{row.step:.10g}", f"{row.err_v:.6e}", "" if row.rate_v is None else f"{row.rate_v:.2f}",
                        f"{row.err_w:.6e}", "" if row.rate_w is None else f"{row.rate_w:.2f}"])
    return path


def write_energy_csv(path, times, energies) -> Path:
    path = Path(path)
    with path.open("w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["step", "time", "energy"])
        for n, (t, e) in enumerate(zip(times, energies)):
            w.writerow([n, f"{t:.10g}", f"{e:.12e}"])
    return path


def write_distance_csv(path, rows) -> Path:
    """Channel comparison table: eps, l2_distance_to_single_run."""
    path = Path(path)
    with path.open("w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["eps", "l2_distance"])
        for eps, dist in rows:
            w.writerow([f"{eps:.10g}", f"{dist:.6e}"])
    return path


# ----------------------------------------------------------------------
# legacy VTK (`reporting.py:84-110`)
# ----------------------------------------------------------------------


def write_vtk(path, mesh, point_data=None, title="ensmhd fields") -> Path:
    """Legacy ASCII VTK unstructured grid with optional vertex data ((nv,) scalars or (nv, 2) vectors)."""
    path = Path(path)
    nv, nt = mesh.num_vertices, mesh.num_triangles
    lines = ["# vtk DataFile Version 2.0", title, "ASCII", "DATASET UNSTRUCTURED_GRID", f"POINTS {nv} double"]
    lines += [f"{x:.12g} {y:.12g} 0.0" for x, y in np.asarray(mesh.vertices)]
    lines.append(f"CELLS {nt} {4 * nt}")
    lines += [f"3 {a} {b} {c}" for a, b, c in np.asarray(mesh.triangles)]
    lines.append(f"CELL_TYPES {nt}")
    lines += ["5"] * nt
    if point_data:
        lines.append(f"POINT_DATA {nv}")
        for name, values in point_data.items():
            values = np.asarray(values)
            if values.ndim == 1:
                lines += [f"SCALARS {name} double", "LOOKUP_TABLE default"]
                lines += [f"{v:.12g}" for v in values]
            else:
                lines.append(f"VECTORS {name} double")
                lines += [f"{vx:.12g} {vy:.12g} 0.0" for vx, vy in values]
    path.write_text("\n".join(lines) + "\n")
    return path


def vertex_fields(state, disc, coupling: float) -> dict:
    """Vertex-sampled ensemble-average fields for export (`experiments.py:507-522`): velocity and
    speed, plus the magnetic field and |B| when the coupling is positive."""
    from .ensemble import primitive_from_elsasser
    nv, ns = disc.mesh.num_vertices, disc.n_scalar

    def at_vertices(coeffs):
        return np.column_stack([coeffs[:ns][:nv], coeffs[ns:][:nv]])

    mv, mw = np.asarray(state.mean_v, dtype=float), np.asarray(state.mean_w, dtype=float)
    u = at_vertices(0.5 * (mv + mw))
    fields = {"velocity": u, "speed": np.linalg.norm(u, axis=1)}
    if coupling > 0.0:
        b = at_vertices(primitive_from_elsasser(mv, mw, coupling)[1])
        fields["magnetic"] = b
        fields["bmag"] = np.linalg.norm(b, axis=1)
    return fields
