"""Finite-element spaces and time-independent operators (host-side setup).

Builds the dof maps and constant operators the time-step consumes, with the
reference's exact numbering and conventions (`pkg/src/ensmhd/fem.py`):

  * 7-point degree-5 quadrature, points ordered centre / a+ triple / a- triple
    (`fem.py:33-57`);
  * P2 local dofs [v0, v1, v2, m01, m12, m20]; global scalar numbering is all
    vertices, then the lexicographically sorted unique edges (`fem.py:140-160`);
  * vector fields are component-blocked [x(ns) | y(ns)] (`fem.py:9-12`);
  * pressure spaces: ``"disc"`` is the reference's P1-discontinuous space with
    dof 3e+k (`fem.py:162-176`, Scott-Vogelius on barycentric meshes); ``"th"``
    is continuous P1 on the vertices (Taylor-Hood), which BASELINE.json's
    configs use.  ``"th"`` reproduces exactly the shim of SURVEY.md Appendix B
    (pressure cell_dofs = triangles, dof coords = vertices).

Only setup lives here; every per-step quantity is computed on the GPU by the
kernels in ``csrc/``.  These routines also feed the CPU oracle in ``oracle/``.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

# ----------------------------------------------------------------------
# quadrature and reference-element tables
# ----------------------------------------------------------------------


def quadrature_deg5():
    """(points (7,3) barycentric, weights (7,)) -- weights sum to 1 (`fem.py:46-57`)."""
    r15 = np.sqrt(15.0)
    pts = [(1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0)]
    wts = [9.0 / 40.0]
    for a, w in (((6.0 + r15) / 21.0, (155.0 + r15) / 1200.0), ((6.0 - r15) / 21.0, (155.0 - r15) / 1200.0)):
        b = 1.0 - 2.0 * a
        pts += [(b, a, a), (a, b, a), (a, a, b)]
        wts += [w, w, w]
    return np.array(pts), np.array(wts)


QPTS, QWTS = quadrature_deg5()
NQ = 7


def p2_values(lam: np.ndarray) -> np.ndarray:
    """P2 shape functions at barycentric points, (nq, 6) (`fem.py:60-71`)."""
    l0, l1, l2 = lam[:, 0], lam[:, 1], lam[:, 2]
    return np.stack([l0 * (2 * l0 - 1), l1 * (2 * l1 - 1), l2 * (2 * l2 - 1),
                     4 * l0 * l1, 4 * l1 * l2, 4 * l2 * l0], axis=1)


def p2_dlambda(lam: np.ndarray) -> np.ndarray:
    """d(phi_k)/d(lambda_i), (nq, 6, 3) (`fem.py:74-86`)."""
    l0, l1, l2 = lam[:, 0], lam[:, 1], lam[:, 2]
    z = np.zeros_like(l0)
    rows = [
        (4 * l0 - 1, z, z),
        (z, 4 * l1 - 1, z),
        (z, z, 4 * l2 - 1),
        (4 * l1, 4 * l0, z),
        (z, 4 * l2, 4 * l1),
        (4 * l2, z, 4 * l0),
    ]
    return np.stack([np.stack(r, axis=1) for r in rows], axis=1)


PHI = p2_values(QPTS)          # (7, 6)
DPHI = p2_dlambda(QPTS)        # (7, 6, 3)


def grad_lambda(corners: np.ndarray, areas: np.ndarray) -> np.ndarray:
    """Barycentric gradients per element (nt, 3, 2) (`fem.py:89-97`)."""
    x, y = corners[:, :, 0], corners[:, :, 1]
    g = np.empty((corners.shape[0], 3, 2))
    for i in range(3):
        j, k = (i + 1) % 3, (i + 2) % 3
        g[:, i, 0] = y[:, j] - y[:, k]
        g[:, i, 1] = x[:, k] - x[:, j]
    return g / (2.0 * areas)[:, None, None]


# ----------------------------------------------------------------------
# spaces
# ----------------------------------------------------------------------


class VelocitySpace:
    """Vector P2 space with the reference dof numbering."""

    components = 2

    def __init__(self, mesh):
        self.mesh = mesh
        t = mesh.triangles
        nv = mesh.num_vertices
        pairs = np.sort(np.vstack([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]]), axis=1)
        # == np.unique(pairs, axis=0, return_inverse=True): lexicographic pairs order as one int64 key
        ukey, inv = np.unique(pairs[:, 0].astype(np.int64) * nv + pairs[:, 1], return_inverse=True)
        self.edges = np.stack([ukey // nv, ukey % nv], axis=1).astype(pairs.dtype)
        inv = inv.reshape(-1)
        nt = mesh.num_triangles
        cell_edges = np.stack([inv[:nt], inv[nt:2 * nt], inv[2 * nt:]], axis=1)
        self.cell_dofs = np.ascontiguousarray(np.hstack([t, nv + cell_edges]))
        self.num_scalar_dofs = nv + len(self.edges)
        mids = 0.5 * (mesh.vertices[self.edges[:, 0]] + mesh.vertices[self.edges[:, 1]])
        self.dof_coords = np.vstack([mesh.vertices, mids])
        corners = mesh.corners()
        self.areas = mesh.areas()
        self.wdet = self.areas[:, None] * QWTS[None, :]
        self.quad_coords = np.einsum("qi,eid->eqd", QPTS, corners)
        self.grad_lam = grad_lambda(corners, self.areas)
        self._basis_grad = None
        self._edge_key = self.edges[:, 0] * (self.num_scalar_dofs + 1) + self.edges[:, 1]

    @property
    def dof_count(self) -> int:
        return 2 * self.num_scalar_dofs

    @property
    def basis_grad(self) -> np.ndarray:
        """(nt, 7, 6, 2) physical gradients of the P2 shape functions."""
        if self._basis_grad is None:
            self._basis_grad = np.einsum("qki,eid->eqkd", DPHI, self.grad_lam)
        return self._basis_grad

    def edge_ids(self, vertex_pairs) -> np.ndarray:
        p = np.sort(np.asarray(vertex_pairs, dtype=np.int64), axis=1)
        key = p[:, 0] * (self.num_scalar_dofs + 1) + p[:, 1]
        pos = np.searchsorted(self._edge_key, key)
        if np.any(pos >= len(self._edge_key)) or np.any(self._edge_key[np.minimum(pos, len(self._edge_key) - 1)] != key):
            raise ValueError("vertex pair is not a mesh edge")
        return pos

    def boundary_scalar_dofs(self, markers=None) -> np.ndarray:
        """Sorted scalar dofs on the selected boundary segments (`fem.py:191-200`)."""
        m = self.mesh
        edges = m.boundary_edges[m.edge_mask(markers)]
        mids = m.num_vertices + self.edge_ids(edges)
        return np.unique(np.concatenate([np.unique(edges), mids]))

    def boundary_dofs(self, markers=None) -> np.ndarray:
        """Vector-expanded boundary dofs: x block then y block (`fem.py:202-207`)."""
        sc = self.boundary_scalar_dofs(markers)
        return np.concatenate([sc, self.num_scalar_dofs + sc])

    def interior_scalar_dofs(self) -> np.ndarray:
        mask = np.ones(self.num_scalar_dofs, dtype=bool)
        mask[self.boundary_scalar_dofs()] = False
        return np.nonzero(mask)[0]


class PressureSpace:
    """Linear pressures: ``kind='th'`` continuous vertex P1, ``'disc'`` P1-discontinuous."""

    components = 1

    def __init__(self, mesh, kind: str = "th"):
        if kind not in ("th", "disc"):
            raise ValueError(f"unknown pressure space kind {kind!r}")
        self.mesh = mesh
        self.kind = kind
        nt = mesh.num_triangles
        if kind == "th":
            self.cell_dofs = np.ascontiguousarray(mesh.triangles.astype(np.int64))
            self.num_scalar_dofs = mesh.num_vertices
            self.dof_coords = mesh.vertices
        else:
            self.cell_dofs = np.arange(3 * nt, dtype=np.int64).reshape(nt, 3)
            self.num_scalar_dofs = 3 * nt
            self.dof_coords = mesh.corners().reshape(-1, 2)
        self.areas = mesh.areas()
        self.wdet = self.areas[:, None] * QWTS[None, :]

    @property
    def dof_count(self) -> int:
        return self.num_scalar_dofs

    def node_of_dof(self, vel: VelocitySpace) -> np.ndarray:
        """P2 node (== mesh vertex) each pressure dof sits on."""
        out = np.empty(self.num_scalar_dofs, dtype=np.int64)
        out[self.cell_dofs.ravel()] = self.mesh.triangles.ravel()
        return out


# ----------------------------------------------------------------------
# assembly of constant operators
# ----------------------------------------------------------------------


def _scatter(rows_dofs, cols_dofs, local, shape) -> sp.csr_matrix:
    r = np.broadcast_to(rows_dofs[:, :, None], local.shape).ravel()
    c = np.broadcast_to(cols_dofs[:, None, :], local.shape).ravel()
    a = sp.coo_matrix((local.ravel(), (r, c)), shape=shape).tocsr()
    a.sort_indices()
    return a


def scalar_pattern(vel: VelocitySpace) -> sp.csr_matrix:
    """Element-connectivity pattern of the scalar P2 operators (values = 1); built once per space
    (callers must not modify it)."""
    cached = getattr(vel, "_pattern", None)
    if cached is not None:
        return cached
    nt = vel.mesh.num_triangles
    ns = vel.num_scalar_dofs
    a = _scatter(vel.cell_dofs, vel.cell_dofs, np.ones((nt, 6, 6)), (ns, ns))
    a.data[:] = 1.0
    vel._pattern = a
    return a


def mass_scalar(vel: VelocitySpace) -> sp.csr_matrix:
    """M_ab = int phi_a phi_b (`fem.py:254-259`)."""
    ref = np.einsum("q,qi,qj->ij", QWTS, PHI, PHI)
    ns = vel.num_scalar_dofs
    return _scatter(vel.cell_dofs, vel.cell_dofs, vel.areas[:, None, None] * ref[None], (ns, ns))


def stiffness_scalar(vel: VelocitySpace, coeff=None) -> sp.csr_matrix:
    """K_ab = int c grad phi_a . grad phi_b (`fem.py:262-282`); c per (nt, 7) or None."""
    w = vel.wdet if coeff is None else vel.wdet * np.asarray(coeff, dtype=float)
    bg = vel.basis_grad
    local = np.einsum("eq,eqid,eqjd->eij", w, bg, bg)
    ns = vel.num_scalar_dofs
    return _scatter(vel.cell_dofs, vel.cell_dofs, local, (ns, ns))


def divergence(vel: VelocitySpace, pres: PressureSpace) -> sp.csr_matrix:
    """B_pa = int rho_p div phi_a, shape (n_p, 2 ns) (`fem.py:330-344`)."""
    n_p, ns = pres.num_scalar_dofs, vel.num_scalar_dofs
    blocks = []
    for d in range(2):
        local = np.einsum("eq,qp,eqa->epa", vel.wdet, QPTS, vel.basis_grad[..., d])
        blocks.append(_scatter(pres.cell_dofs, vel.cell_dofs, local, (n_p, ns)))
    out = sp.hstack(blocks, format="csr")
    out.sort_indices()
    return out


def divergence_pair(vel: VelocitySpace, pres: PressureSpace):
    """Bx, By (each n_p x ns) on one shared CSR pattern: (indptr, indices, bx, by).

    Same element integrals and COO->CSR scatter as :func:`divergence`, so the
    values equal the reference's B blocks (`fem.py:330-344`); the common
    pattern lets the GPU store (bx, by) pairs.
    """
    n_p, ns = pres.num_scalar_dofs, vel.num_scalar_dofs
    out = []
    for d in range(2):
        local = np.einsum("eq,qp,eqa->epa", vel.wdet, QPTS, vel.basis_grad[..., d])
        r = np.broadcast_to(pres.cell_dofs[:, :, None], local.shape).ravel()
        c = np.broadcast_to(vel.cell_dofs[:, None, :], local.shape).ravel()
        coo = sp.coo_matrix((local.ravel(), (r, c)), shape=(n_p, ns))
        coo.sum_duplicates()               # canonical (row, col) order, explicit zeros kept
        out.append(coo)
    bx, by = out
    assert np.array_equal(bx.row, by.row) and np.array_equal(bx.col, by.col)
    indptr = np.concatenate([[0], np.cumsum(np.bincount(bx.row, minlength=n_p))])
    return indptr, bx.col.astype(np.int64), bx.data.copy(), by.data.copy()


def load_vector(space, values: np.ndarray) -> np.ndarray:
    """Load vector(s) from quadrature-point values (`fem.py:347-375`).

    ``values``: (..., nt, 7) for a pressure space or (..., nt, 7, 2) for the
    velocity space; leading axes are batched.
    """
    values = np.asarray(values, dtype=float)
    if isinstance(space, PressureSpace):
        basis, n, comps = QPTS, space.num_scalar_dofs, None
    else:
        basis, n, comps = PHI, space.num_scalar_dofs, 2

    def one(vals):
        local = np.einsum("...eq,qi->...ei", space.wdet * vals, basis)
        lead = local.shape[:-2]
        flat = local.reshape(-1, local.shape[-2] * local.shape[-1])
        idx = space.cell_dofs.ravel()
        out = np.stack([np.bincount(idx, weights=f, minlength=n) for f in flat])
        return out.reshape(*lead, n)

    if comps is None:
        return one(values)
    return np.concatenate([one(values[..., 0]), one(values[..., 1])], axis=-1)


def pressure_integrals(pres: PressureSpace) -> np.ndarray:
    """int rho_p over the domain (`stepper.py:71-72`)."""
    return load_vector(pres, np.ones_like(pres.wdet))


def interpolate(f, t: float, vel: VelocitySpace) -> np.ndarray:
    """Nodal interpolant of f(x, y, t) -> (fx, fy), component-blocked (`fem.py:423-438`)."""
    x, y = vel.dof_coords[:, 0], vel.dof_coords[:, 1]
    fx, fy = f(x, y, t)
    fx = np.broadcast_to(np.asarray(fx, dtype=float), x.shape)
    fy = np.broadcast_to(np.asarray(fy, dtype=float), x.shape)
    return np.concatenate([fx, fy])


def eval_at_quadrature(vel: VelocitySpace, coeffs: np.ndarray) -> np.ndarray:
    """Values of vector P2 fields at quadrature points: (..., nt, 7, 2) (`fem.py:394-398`)."""
    c = np.asarray(coeffs, dtype=float)
    ns = vel.num_scalar_dofs
    comp = c.reshape(*c.shape[:-1], 2, ns)
    loc = np.moveaxis(comp[..., :, vel.cell_dofs], -3, -1)   # (..., nt, 6, 2)
    return np.einsum("qi,...eic->...eqc", PHI, loc)


def eval_gradient_at_quadrature(vel: VelocitySpace, coeffs: np.ndarray) -> np.ndarray:
    """Gradients (..., nt, 7, 2[comp], 2[deriv]) (`fem.py:401-408`)."""
    c = np.asarray(coeffs, dtype=float)
    ns = vel.num_scalar_dofs
    comp = c.reshape(*c.shape[:-1], 2, ns)
    loc = np.moveaxis(comp[..., :, vel.cell_dofs], -3, -1)
    return np.einsum("eqid,...eic->...eqcd", vel.basis_grad, loc)
