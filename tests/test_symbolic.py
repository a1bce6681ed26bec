"""CPU checks of the host-side symbolic analysis and schedule (no GPU).

The numpy emulator executes exactly the device launch schedule; solving the
oracle-assembled saddle matrix through it proves ordering, maps, panels and
the block-sweep algebra before any kernel runs.
"""

import numpy as np
import pytest

from oracle import ensmhd_oracle as O
import mf_emulator as E
from paper_2108_05110_b200 import fe
from paper_2108_05110_b200 import symbolic as S
from paper_2108_05110_b200.discretization import Discretization
from paper_2108_05110_b200.ensemble import EnsembleConfig, MemberParams
from paper_2108_05110_b200.mesh import Marker, barycentric_refine, build_step_channel, build_structured_square


def internal_ids(disc, plan):
    ns, nv = disc.n_scalar, disc.n_vel
    iid = np.empty(disc.n_total, dtype=np.int64)
    iid[:ns] = 2 * plan.node_perm
    iid[ns:nv] = 2 * plan.node_perm + 1
    iid[nv:] = nv + plan.pres_perm
    return iid


@pytest.mark.parametrize("case", ["th8", "sv2", "sv4", "channel"])
def test_plan_solves_saddle_system(case, rng):
    if case == "th8":
        disc = Discretization.from_mesh(build_structured_square(8), pressure="th")
    elif case == "sv2":
        disc = Discretization.from_mesh(barycentric_refine(build_structured_square(2)))
    elif case == "sv4":
        disc = Discretization.from_mesh(barycentric_refine(build_structured_square(4)))
    else:
        disc = Discretization.from_mesh(build_step_channel(length=8.0, cells_per_unit=1), pressure="th",
                                        dirichlet_markers=(Marker.WALL, Marker.INLET), pin_pressure=False)
    plan = S.analyse(disc)
    cfg = EnsembleConfig((MemberParams(0.01, 0.011), MemberParams(0.009, 0.01)), 1.0, 1.0, 0.01, 0.1)
    v = rng.standard_normal((2, disc.n_vel))
    w = rng.standard_normal((2, disc.n_vel))
    a_s = O.velocity_block(w.mean(0), w - w.mean(0), cfg, disc)
    pat = fe.scalar_pattern(disc.velocity)
    a_s = (a_s + 0.0 * pat).tocsr()
    a_s.sort_indices()
    if a_s.nnz != pat.nnz:        # exact zeros dropped by scipy: realign to the pattern
        full = pat.copy()
        full.data[:] = 0.0
        full = full.tolil()
        coo = a_s.tocoo()
        full[coo.row, coo.col] = coo.data
        a_s = full.tocsr()
        a_s.sort_indices()
    K = O.saddle_matrix(a_s, disc)
    st = E.factor(plan, a_s.data)
    iid = internal_ids(disc, plan)
    b = rng.standard_normal((disc.n_total, 3))
    b[disc.constrained_rows] = 0.0
    bi = np.zeros_like(b)
    bi[iid] = b
    x = E.solve(plan, st, bi)[iid]
    res = np.linalg.norm(K @ x - b, axis=0) / np.linalg.norm(b, axis=0)
    assert res.max() < 1e-11, res


def test_plan_invariants():
    disc = Discretization.from_mesh(build_structured_square(16), pressure="th")
    plan = S.analyse(disc)
    # every free dof is a pivot of exactly one front
    piv = np.concatenate([plan.f_idx[plan.f_idx_off[f]:plan.f_idx_off[f] + plan.f_k[f]] for f in range(plan.nfront)])
    assert len(np.unique(piv)) == len(piv) == disc.n_total - len(disc.constrained_rows)
    # parents are processed after children, and the root has no contribution block
    for f in range(plan.nfront):
        p = plan.f_parent[f]
        if p >= 0:
            assert plan.f_level[p] > plan.f_level[f]
        else:
            assert plan.f_m[f] == plan.f_k[f]
    # each original free-free entry has a unique slot
    assert len(np.unique(plan.orig_dst)) == len(plan.orig_dst)
    sched = plan.schedule
    assert sched["work"].shape[1] == 4
    assert set(np.unique(sched["factor"][:, 0])) <= set(range(7))


@pytest.mark.parametrize("heights", [(), (1,), (1, 2), (1, 3), (2, 4)])
def test_amalgamated_trees_solve(heights, rng, monkeypatch):
    """Merging tree levels into their parents (symbolic._amalgamate) keeps the plan a valid
    factorisation: every free dof is still eliminated exactly once, children precede parents, and
    the emulated factor + solve reproduces the saddle solution; each merged height removes a level."""
    disc = Discretization.from_mesh(build_structured_square(12), pressure="th")
    monkeypatch.setattr(S, "AMALGAMATE", ())
    base = S.analyse(disc, leaf=6)
    monkeypatch.setattr(S, "AMALGAMATE", heights)
    plan = S.analyse(disc, leaf=6)
    assert plan.nlevels == base.nlevels - len(heights)
    piv = np.concatenate([plan.f_idx[plan.f_idx_off[f]:plan.f_idx_off[f] + plan.f_k[f]] for f in range(plan.nfront)])
    assert len(np.unique(piv)) == len(piv) == disc.n_total - len(disc.constrained_rows)
    for f in range(plan.nfront):
        p = plan.f_parent[f]
        if p >= 0:
            assert plan.f_level[p] > plan.f_level[f]
    cfg = EnsembleConfig((MemberParams(0.01, 0.011), MemberParams(0.009, 0.01)), 1.0, 1.0, 0.01, 0.1)
    w = rng.standard_normal((2, disc.n_vel))
    pat = fe.scalar_pattern(disc.velocity)
    a_s = (O.velocity_block(w.mean(0), w - w.mean(0), cfg, disc) + 0.0 * pat).tocsr()
    a_s.sort_indices()
    assert a_s.nnz == pat.nnz
    K = O.saddle_matrix(a_s, disc)
    st = E.factor(plan, a_s.data)
    iid = internal_ids(disc, plan)
    b = rng.standard_normal((disc.n_total, 2))
    b[disc.constrained_rows] = 0.0
    bi = np.zeros_like(b)
    bi[iid] = b
    x = E.solve(plan, st, bi)[iid]
    res = np.linalg.norm(K @ x - b, axis=0) / np.linalg.norm(b, axis=0)
    assert res.max() < 1e-11, res


def test_split_k_schedule(rng, monkeypatch):
    """Force tiny split-K so the partial/reduce path of the solve schedule is exercised."""
    monkeypatch.setattr(S, "SPLIT_K", 16)
    disc = Discretization.from_mesh(build_structured_square(8), pressure="th")
    plan = S.analyse(disc)
    assert plan.schedule["nslot"] > 0 and plan.schedule["split_k"] == 16
    cfg = EnsembleConfig((MemberParams(0.01, 0.011), MemberParams(0.009, 0.01)), 1.0, 1.0, 0.01, 0.1)
    w = rng.standard_normal((2, disc.n_vel))
    pat = fe.scalar_pattern(disc.velocity)
    a_s = O.velocity_block(w.mean(0), w - w.mean(0), cfg, disc)
    vals = np.zeros(pat.nnz)
    coo = a_s.tocoo()
    rows = np.repeat(np.arange(pat.shape[0]), np.diff(pat.indptr))
    key = rows * pat.shape[0] + pat.indices
    vals[np.searchsorted(key, coo.row * pat.shape[0] + coo.col)] = coo.data
    a_s = pat.copy()
    a_s.data = vals
    K = O.saddle_matrix(a_s, disc)
    st = E.factor(plan, vals)
    iid = internal_ids(disc, plan)
    b = rng.standard_normal((disc.n_total, 2))
    b[disc.constrained_rows] = 0.0
    bi = np.zeros_like(b)
    bi[iid] = b
    x = E.solve(plan, st, bi)[iid]
    res = np.linalg.norm(K @ x - b, axis=0) / np.linalg.norm(b, axis=0)
    assert res.max() < 1e-11, res


@pytest.mark.parametrize("n", [4, 16, 40])
def test_host_nested_dissection_matches_python_spec(n):
    """csrc/host_symbolic.cpp's nested dissection = symbolic._nested_dissection_py (node sets, tree
    shape, numbering), on the P2 node graph of an n x n square."""
    from paper_2108_05110_b200 import fe
    from paper_2108_05110_b200 import symbolic as S
    disc = Discretization.from_mesh(build_structured_square(n), pressure="th")
    g = fe.scalar_pattern(disc.velocity).copy()
    g.setdiag(0)
    g.eliminate_zeros()
    g.sort_indices()
    a = S._nested_dissection(disc.velocity.dof_coords, g.indptr, g.indices, 24)
    b = S._nested_dissection_py(disc.velocity.dof_coords, g.indptr, g.indices, 24)
    assert len(a[0]) == len(b[0]) and a[1] == b[1]
    for x, y in zip(a[0], b[0]):
        assert np.array_equal(np.sort(x), np.sort(y)) and np.array_equal(x, y)
