"""Pin the CPU oracle (and the host setup it shares) to the real reference.

Fixtures in tests/golden/reference_golden.npz were produced by the unmodified
reference (tests/golden/make_golden.py).  These tests run on CPU only.
"""

import os
import sys

import numpy as np
import pytest

from oracle import ensmhd_oracle as O
from paper_2108_05110_b200 import fe
from paper_2108_05110_b200.discretization import Discretization
from paper_2108_05110_b200.ensemble import EnsembleConfig, MemberParams, sample_viscosities
from paper_2108_05110_b200.mesh import barycentric_refine, build_structured_square
from paper_2108_05110_b200.problems import (BaselineMms, PaperMmsBoundary, PaperMmsForcing, _BoundaryView,
                                            _ForcingView, paper_mms_initial_fields)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def sv2():
    return Discretization.from_mesh(barycentric_refine(build_structured_square(2)))


@pytest.fixture(scope="module")
def th4():
    return Discretization.from_mesh(build_structured_square(4), pressure="th")


def sv_config():
    members = (MemberParams(0.01, 0.1), MemberParams(0.012, 0.09), MemberParams(0.009, 0.11))
    return EnsembleConfig(members=members, coupling=1.0, mu=1.0, dt=0.05, t_end=0.1, perturbation=0.01)


@pytest.mark.parametrize("prefix,fixture", [("sv2_", "sv2"), ("th4_", "th4")])
def test_setup_matches_reference(golden, prefix, fixture, request):
    d = request.getfixturevalue(fixture)
    assert np.array_equal(d.velocity.cell_dofs, golden[prefix + "cell_dofs"])
    assert np.array_equal(d.pressure.cell_dofs, golden[prefix + "pres_cell_dofs"])
    assert np.array_equal(d.bdofs, golden[prefix + "bdofs"])
    for name, mat in (("mass_dense", d.mass_s), ("stiff_dense", d.stiff_s), ("div_dense", d.divergence)):
        ref = golden[prefix + name]
        assert np.max(np.abs(mat.toarray() - ref)) <= 1e-15 * np.abs(ref).max()
    assert np.allclose(d.pressure_integrals, golden[prefix + "pintg"], rtol=0, atol=1e-16)


def test_shared_matrices_and_rhs(golden, sv2):
    cfg = sv_config()
    v, w = golden["sv2_pert_v"], golden["sv2_pert_w"]
    nut = O.eddy_viscosity(sv2.velocity, w - w.mean(axis=0), cfg.mu, cfg.dt)
    assert np.max(np.abs(nut - golden["sv2_nut_w"])) <= 1e-15 * golden["sv2_nut_w"].max()
    lv, lw = PaperMmsForcing().loads(cfg.dt, sv2, cfg)
    assert rel(lv, golden["sv2_loads_v"]) < 1e-14 and rel(lw, golden["sv2_loads_w"]) < 1e-14
    bv, bw = PaperMmsBoundary().values(cfg.dt, sv2, cfg)
    assert np.array_equal(bv, golden["sv2_bvals_v"]) and np.array_equal(bw, golden["sv2_bvals_w"])
    for kind, name, loads, bvals in (("v", "V", lv, bv), ("w", "W", lw, bw)):
        mat = O.shared_matrix(kind, v, w, cfg, sv2).toarray()
        ref = golden[f"sv2_mat{name}"]
        assert np.max(np.abs(mat - ref)) <= 1e-13 * np.abs(ref).max()
        rhs = O.rhs_block(kind, v, w, loads, bvals, cfg, sv2)
        ref = golden[f"sv2_rhs{name}"]
        assert np.max(np.abs(rhs - ref)) <= 1e-12 * np.abs(ref).max()


def test_one_step_sv(golden, sv2):
    cfg = sv_config()
    j = cfg.num_members
    st = O.OracleState(golden["sv2_pert_v"], golden["sv2_pert_w"], np.zeros((j, sv2.n_pres)), np.zeros((j, sv2.n_pres)))
    new, res = O.advance(st, cfg, sv2, PaperMmsForcing(), PaperMmsBoundary())
    for f in "vwqr":
        assert rel(getattr(new, f), golden["sv2_step1_" + f]) < 1e-10
    assert res < 1e-12


def test_run_sv_paper_mms(golden, sv2):
    cfg = sv_config()
    v0, w0 = paper_mms_initial_fields(sv2, cfg)
    st, recs, _, res = O.run(cfg, sv2, v0, w0, PaperMmsForcing(), PaperMmsBoundary())
    for f in "vw":
        assert rel(getattr(st, f), golden["sv2_run_" + f]) < 1e-10
    e = np.array([r["energy"] for r in recs])
    assert rel(e, golden["sv2_run_energy"]) < 1e-12
    assert rel(np.array([r["l2v"] for r in recs]), golden["sv2_run_l2v"]) < 1e-12
    assert rel(np.array([r["gradw"] for r in recs]), golden["sv2_run_gradw"]) < 1e-12
    assert rel(np.array([r["div_v"] for r in recs]), golden["sv2_run_div_v"]) < 1e-6


@pytest.mark.parametrize("prefix,n,steps", [("th4_", 4, 3), ("c1_", 16, 10)])
def test_run_th_baseline(golden, prefix, n, steps):
    disc = Discretization.from_mesh(build_structured_square(n), pressure="th")
    members = sample_viscosities((0.009, 0.011), (0.009, 0.011), 3, 0)
    cfg = EnsembleConfig(members=members, coupling=1.0, mu=1.0, dt=0.01, t_end=0.01 * steps, seed=0)
    mms = BaselineMms()
    v0, w0 = mms.initial_fields(disc, cfg)
    if prefix == "th4_":
        lv, lw = mms.loads(0.01, disc, cfg)
        assert rel(lv, golden["th4_loads_v"]) < 1e-14 and rel(lw, golden["th4_loads_w"]) < 1e-14
    st, recs, _, res = O.run(cfg, disc, v0, w0, _ForcingView(mms), _BoundaryView(mms))
    for f in "vw":
        assert rel(getattr(st, f), golden[prefix + "run_" + f]) < 1e-11
    for f in "qr":
        assert rel(getattr(st, f), golden[prefix + "run_" + f]) < 1e-9
    e = np.array([r["energy"] for r in recs])
    assert rel(e, golden[prefix + "run_energy"]) < 1e-12
    assert np.all(res < 1e-12)


# ----------------------------------------------------------------------
# the BASELINE problem set-ups (C3 cavity, C4 do-nothing channel) against the
# real reference: tiny twins of tests/golden/make_golden_large.py's cases
# ----------------------------------------------------------------------


@pytest.mark.parametrize("case,name,over", [
    ("C3tiny", "C3", dict(n=6, J=4, dt=0.01, steps=2, coupling=0.1)),
    ("C4tiny", "C4", dict(k=1, J=3, dt=0.02, steps=2, delta=0.1, length=8.0)),
])
def test_case_setup_matches_reference_variant(case, name, over):
    """build_case's C3/C4 problems run through the oracle reproduce the reference run of the same
    configuration (C4: the reference with the do-nothing outflow variant wrapped around it -- no pin,
    no mean-zeroing, Dirichlet on WALL+INLET) to round-off."""
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import make_golden_large as G
    from paper_2108_05110_b200.problems import build_case
    fx = np.load(G.fixture_path(case))
    disc, cfg, prob = build_case(name, **over)
    st, recs, _, res = O.run(cfg, disc, prob.initial_v, prob.initial_w, prob.forcing, prob.boundary)
    got = G.summarize("s2_", st.v, st.w, st.q, st.r)
    assert set(got) == {k for k in fx.files if k.startswith("s2_")}
    for k, v in got.items():
        assert np.linalg.norm(v - fx[k]) <= 1e-12 * max(np.linalg.norm(fx[k]), 1e-300), k
    assert np.allclose([r["energy"] for r in recs], fx["energy"], rtol=1e-13, atol=0)


def test_do_nothing_channel_step_matches_dense_solve():
    """The no-pin / do-nothing branch of the oracle (`oracle/ensmhd_oracle.py` saddle_matrix with
    pin_pressure=False): the saddle system is nonsingular (the outflow fixes the pressure level) and
    SuperLU's block solve equals a dense LU solve, per member."""
    from paper_2108_05110_b200.problems import build_case
    disc, cfg, prob = build_case("C4", k=1, J=3, dt=0.02, steps=1, delta=0.1, length=8.0)
    assert not disc.pin_pressure
    v, w = np.asarray(prob.initial_v), np.asarray(prob.initial_w)
    bv, bw = prob.boundary.values(cfg.dt, disc, cfg)
    for kind, bvals in (("v", bv), ("w", bw)):
        mat = O.shared_matrix(kind, v, w, cfg, disc)
        rhs = O.rhs_block(kind, v, w, None, bvals, cfg, disc)
        dense = mat.toarray()
        assert np.linalg.cond(dense) < 1e12
        x_dense = np.linalg.solve(dense, rhs)
        x = O.solve_block(mat, rhs)
        assert np.linalg.norm(x - x_dense) <= 1e-11 * np.linalg.norm(x_dense)
        assert O.relative_residual(mat, x, rhs) < 1e-13
