"""Device-side error norms (run(..., exact=...), ens_mean_error) against the reference's
error_norm_21 (tests/golden/reporting_golden.json) and the host restatement."""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2108_05110_b200 as P  # noqa: E402
from paper_2108_05110_b200 import reporting as R  # noqa: E402
from paper_2108_05110_b200.problems import (BaselineMmsExact, PaperMmsBoundary, PaperMmsExact,  # noqa: E402
                                            PaperMmsForcing, paper_mms_initial_fields)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reporting_golden.json")))


def test_device_error_norm_matches_reference_run_mms_case():
    disc = P.Discretization.from_mesh(P.barycentric_refine(P.build_structured_square(2)))
    members = (P.MemberParams(0.01, 0.1), P.MemberParams(0.012, 0.09), P.MemberParams(0.009, 0.11))
    cfg = P.EnsembleConfig(members=members, coupling=1.0, mu=1.0, dt=0.05, t_end=0.1, perturbation=0.01)
    v0, w0 = paper_mms_initial_fields(disc, cfg)
    rep, _, _ = P.run(cfg, P.Problem(disc, v0, w0, PaperMmsForcing(), PaperMmsBoundary()), exact=PaperMmsExact())
    ev, ew = rep.error_norm_21()
    assert ev == pytest.approx(GOLD["mms_err_v"], rel=1e-9)
    assert ew == pytest.approx(GOLD["mms_err_w"], rel=1e-9)


def test_device_error_series_matches_host_on_c1():
    disc, cfg, prob = P.build_case("C1")
    means = []
    rep, _, _ = P.run(cfg, prob, exact=BaselineMmsExact(),
                      observer=lambda n, t, st: means.append((np.array(st.mean_v), np.array(st.mean_w))))
    ex = BaselineMmsExact()
    for n, (mv, mw) in enumerate(means):
        t = rep.times[n]
        iv = P.fe.interpolate(lambda x, y, tt: ex.mean_v(x, y, tt, cfg), t, disc.velocity)
        assert rep.err_v_h1_sq[n] == pytest.approx(R.h1_norm_sq(disc, mv - iv), rel=1e-9, abs=1e-28)
        assert rep.err_w_h1_sq[n] == pytest.approx(R.h1_norm_sq(disc, mw), rel=1e-9, abs=1e-28)
    ev, _ = rep.error_norm_21()
    assert 0.0 < ev < 1e-3        # discretisation error of the P2 interpolant-level scheme
