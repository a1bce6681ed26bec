"""Pin the CPU oracle (and the host setup it shares) to the real reference.

Fixtures in tests/golden/reference_golden.npz were produced by the unmodified
reference (tests/golden/make_golden.py).  These tests run on CPU only.
"""

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
