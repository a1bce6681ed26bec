"""Factor-once / solve-many interface of the reference (`linalg.py:1-118`), backed by the B200 engine.

`factorize(matrix, symbolic)` builds the GPU multifrontal factorisation of one
sub-step saddle matrix of a `Discretization` (the only matrices the time-step
path factorises, `stepper.py:216`); `Factorization.solve` / `solve_block`
solve with the same column-batched Krylov iteration the step uses, converged
per column to a true relative residual of ``rtol`` (default 1e-12), so they
meet the reference's own bar (dense-LU agreement at 1e-10,
`tests/test_linalg.py:28-35`).  Columns are independent: a block solve equals
stacked single solves.  There is no CPU fallback: a matrix that is not a
saddle matrix of a known discretisation is rejected with ValueError.

`symbolic` is the discretisation's `SaddleSymbolic` (the nested-dissection
plan, reused across factorisations exactly as the reference reuses UMFPACK's
symbolic analysis, `stepper.py:216-218`).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


class SingularMatrixError(RuntimeError):
    """Raised when a factorisation meets an exactly singular matrix (`linalg.py:31-36`)."""


class SaddleSymbolic:
    """Reusable analysis of a Discretization's saddle pattern (the engine's host mesh + plan)."""

    def __init__(self, disc):
        from .engine import host_mesh
        self.disc = disc
        self.hm = host_mesh(disc)

    def velocity_values(self, matrix) -> np.ndarray:
        """A_s values (internal slot order) read off a saddle matrix [[A,0,-Bx^T],[0,A,-By^T],[Bx,By,0]]
        whose constrained rows are identity rows: each scalar row comes from the first component
        whose row is not constrained (constrained rows never enter the factorisation)."""
        disc, hm = self.disc, self.hm
        n, ns = disc.n_total, disc.n_scalar
        m = sp.csr_matrix(matrix)
        if m.shape != (n, n):
            raise ValueError(f"matrix shape {m.shape} is not the saddle size ({n}, {n}) of this discretisation")
        cons = np.zeros(n, dtype=bool)
        cons[disc.constrained_rows] = True
        xblk = m[:ns, :ns].tocoo()
        yblk = m[ns:2 * ns, ns:2 * ns].tocoo()
        take_x = ~cons[xblk.row]
        take_y = ~cons[ns + yblk.row] & cons[yblk.row]
        rows = np.concatenate([xblk.row[take_x], yblk.row[take_y]])
        cols = np.concatenate([xblk.col[take_x], yblk.col[take_y]])
        vals = np.concatenate([xblk.data[take_x], yblk.data[take_y]])
        perm = hm.plan.node_perm
        out = np.zeros(hm.nnz_s)
        if rows.size:
            out[hm._slot(perm[rows], perm[cols])] = vals
        return out


def saddle_matrix(disc, a_int) -> sp.csr_matrix:
    """CSR view (reference dof order) of the saddle matrix with velocity block A_s = ``a_int``
    (internal slot order): [[A,0,-Bx^T],[0,A,-By^T],[Bx,By,0]], Dirichlet rows and the pin replaced
    by identity rows (`stepper.py:208-215`, `fem.py:446-460`)."""
    from .engine import host_mesh
    hm = host_mesh(disc)
    ns = disc.n_scalar
    inv = np.empty(ns, dtype=np.int64)
    inv[hm.plan.node_perm] = np.arange(ns)
    rows = np.repeat(np.arange(ns), np.diff(hm.s_rowptr))
    a_s = sp.csr_matrix((np.asarray(a_int, dtype=float), (inv[rows], inv[hm.s_col])), shape=(ns, ns))
    bx, by = disc.divergence[:, :ns], disc.divergence[:, ns:]
    full = sp.bmat([[a_s, None, -bx.T], [None, a_s, -by.T], [bx, by, None]], format="csr")
    cons = np.asarray(disc.constrained_rows, dtype=np.int64)
    if cons.size:
        full = full.tolil()
        for r in cons:
            full.rows[r] = [int(r)]
            full.data[r] = [1.0]
        full = full.tocsr()
    full.eliminate_zeros()
    full.sort_indices()
    return full


class Factorization:
    """Reusable factorisation of one saddle matrix (`linalg.py:46-76`); immutable, safe to share."""

    def __init__(self, shape, backend, handle, symbolic=None):
        self.shape = shape
        self.backend = backend
        self._handle = handle          # (disc, A_s values in internal slot order)
        self.symbolic = symbolic
        self._engines = {}

    def _engine(self, ncols):
        eng = self._engines.get(ncols)
        if eng is None:
            from .engine import Engine
            from .ensemble import EnsembleConfig, MemberParams
            disc = self._handle[0]
            cfg = EnsembleConfig(members=tuple(MemberParams(1.0, 1.0) for _ in range(ncols)), coupling=1.0, mu=1.0,
                                 dt=1.0, t_end=1.0)
            from .stepper import get_solver_options
            opts = get_solver_options()
            eng = Engine(disc, cfg, rtol=opts["rtol"], restart=opts["restart"], max_restarts=opts["max_restarts"])
            self._engines[ncols] = eng
            eng.solve_values(self._handle[1], np.zeros((self.shape[0], ncols)), factor=True)
        return eng

    def solve(self, b: np.ndarray) -> np.ndarray:
        """Solve A x = b for one right-hand side."""
        b = np.asarray(b, dtype=float)
        if b.shape != (self.shape[0],):
            raise ValueError(f"rhs shape {b.shape} does not match matrix size {self.shape[0]}")
        return self.solve_block(b[:, None])[:, 0]

    def solve_block(self, rhs_block: np.ndarray) -> np.ndarray:
        """Solve A X = B for B of shape (n, ncols); columns are independent."""
        rhs = np.asarray(rhs_block, dtype=float)
        if rhs.ndim != 2 or rhs.shape[0] != self.shape[0]:
            raise ValueError(f"rhs block shape {rhs.shape} does not match matrix size {self.shape[0]}")
        if rhs.shape[1] == 0:
            return np.zeros_like(rhs)
        x, _ = self._engine(rhs.shape[1]).solve_values(self._handle[1], rhs, factor=False)
        return x


def factorize(matrix, symbolic=None) -> Factorization:
    """GPU factorisation of a saddle matrix of a Discretization (`linalg.py:79-108`).

    ``symbolic``: the discretisation's `SaddleSymbolic` (``disc.saddle_symbolic`` after the first
    `assemble_shared_lhs`).  The input matrix is not modified."""
    if matrix.shape[0] != matrix.shape[1]:
        raise ValueError(f"matrix is not square: {matrix.shape}")
    if not isinstance(symbolic, SaddleSymbolic):
        raise ValueError("the B200 factorisation needs the saddle symbolic analysis of a Discretization "
                         "(symbolic=SaddleSymbolic(disc), cached as disc.saddle_symbolic)")
    vals = symbolic.velocity_values(matrix)
    if not np.all(np.isfinite(vals)):
        raise SingularMatrixError("matrix has non-finite entries")
    return Factorization(matrix.shape, "b200", (symbolic.disc, vals), symbolic)


def relative_residual(matrix, x: np.ndarray, b: np.ndarray) -> float:
    """max over columns of ||A x - b|| / ||b|| (`linalg.py:111-118`)."""
    r = matrix @ x - b
    if r.ndim == 1:
        denom = max(np.linalg.norm(b), np.finfo(float).tiny)
        return float(np.linalg.norm(r) / denom)
    denom = np.maximum(np.linalg.norm(b, axis=0), np.finfo(float).tiny)
    return float(np.max(np.linalg.norm(r, axis=0) / denom))
