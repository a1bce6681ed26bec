"""Error norms, rate tables and output formats (§8(f) row 4) against the real reference's outputs
(tests/golden/reporting_golden.json, made by tests/golden/make_golden_reporting.py)."""

import json
import os

import numpy as np
import pytest

from oracle import ensmhd_oracle as O
import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import reporting as R
from paper_2108_05110_b200.problems import PaperMmsBoundary, PaperMmsForcing, paper_mms_initial_fields, paper_v, paper_w

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reporting_golden.json")))


def test_rate_table_matches_reference():
    steps = [0.25, 0.125, 0.0625]
    t = R.RateTable.from_errors("spatial", "h", steps, [3.1e-2, 8.2e-3, 2.05e-3], [1.7e-2, 4.1e-3, 1.1e-3])
    for row, ref in zip(t.rows, GOLD["rates"]):
        got = [row.step, row.err_v, row.rate_v, row.err_w, row.rate_w]
        for a, b in zip(got, ref):
            assert (a is None and b is None) or a == b
    with pytest.raises(ValueError):
        R.compute_rate(1.0, 0.0, 0.5, 0.25)
    with pytest.raises(ValueError):
        R.compute_rate(1.0, 0.5, 0.5, 0.5)


def test_writers_are_byte_identical(tmp_path):
    t = R.RateTable.from_errors("spatial", "h", [0.25, 0.125, 0.0625], [3.1e-2, 8.2e-3, 2.05e-3],
                                [1.7e-2, 4.1e-3, 1.1e-3])
    R.write_rate_csv(tmp_path / "r.csv", t)
    R.write_energy_csv(tmp_path / "e.csv", np.array([0.0, 0.05, 0.1]), np.array([1.5, 1.25, 1.125]))
    R.write_distance_csv(tmp_path / "d.csv", [(0.01, 1.5e-3), (0.1, 2.5e-2)])
    mesh = P.barycentric_refine(P.build_structured_square(1))
    R.write_vtk(tmp_path / "f.vtk", mesh, {"velocity": np.array(GOLD["vtk_vel"]), "speed": np.array(GOLD["vtk_speed"])},
                title="golden")
    for k in ("r.csv", "e.csv", "d.csv", "f.vtk"):
        assert (tmp_path / k).read_text() == GOLD["file_" + k], k


def test_error_norm_21_matches_reference_run():
    """The reference's run_mms_case(n=2, dt=0.05, T=0.1, eps=0.01) errors, recomputed from the oracle
    run's means with this package's host error_norm_21 (`experiments.py:59-73`)."""
    disc = P.Discretization.from_mesh(P.barycentric_refine(P.build_structured_square(2)))
    members = (P.MemberParams(0.01, 0.1), P.MemberParams(0.012, 0.09), P.MemberParams(0.009, 0.11))
    cfg = P.EnsembleConfig(members=members, coupling=1.0, mu=1.0, dt=0.05, t_end=0.1, perturbation=0.01)
    v0, w0 = paper_mms_initial_fields(disc, cfg)
    st = O.OracleState(v0, w0, np.zeros((3, disc.n_pres)), np.zeros((3, disc.n_pres)))
    mv, mw = [v0.mean(0)], [w0.mean(0)]
    for _ in range(2):
        st, _ = O.advance(st, cfg, disc, PaperMmsForcing(), PaperMmsBoundary())
        mv.append(st.v.mean(0))
        mw.append(st.w.mean(0))
    times = np.array([0.0, 0.05, 0.1])
    assert R.error_norm_21(np.array(mv), times, paper_v, disc) == pytest.approx(GOLD["mms_err_v"], rel=1e-9)
    assert R.error_norm_21(np.array(mw), times, paper_w, disc) == pytest.approx(GOLD["mms_err_w"], rel=1e-9)
