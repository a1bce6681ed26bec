"""Member-column chunking (paper_2108_05110_b200/chunked.py) against the unchunked engine.

A chunked engine solves the same columns chunk by chunk through a context of Jc columns; the
J-independent work (means, eddy maxima, shared matrices, factorisation) is done once per step
from all chunks, so the run reproduces the unchunked run up to the kernels' J-dependent tiling.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2108_05110_b200 as P  # noqa: E402
from paper_2108_05110_b200 import stepper as ST  # noqa: E402
from paper_2108_05110_b200.chunked import ChunkedEngine, largest_divisor_at_most  # noqa: E402


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("case,over,chunk", [("C2", dict(J=20, steps=8), 5), ("C3", dict(n=16, J=6, steps=6), 2),
                                             ("C4", dict(k=2, J=9, steps=6), 3)])
def test_chunked_run_matches_unchunked(case, over, chunk):
    disc, cfg, prob = P.build_case(case, **over)
    rep0, fin0, _ = P.run(cfg, prob)
    ST.set_member_chunk(chunk)
    try:
        disc2, cfg2, prob2 = P.build_case(case, **over)
        rep1, fin1, snaps = P.run(cfg2, prob2, snapshot_steps=(2,))
        eng = ST.get_engine(disc2, cfg2)
    finally:
        ST.set_member_chunk(None)
    assert isinstance(eng, ChunkedEngine) and eng.nchunk == over["J"] // chunk
    # both runs converge every solve to the 1e-12 true residual; the chunked engine's shorter Krylov
    # cycle (restart <= 2) takes a different iteration path, so they agree at the solver tolerance
    scale = np.linalg.norm(fin0.v)
    assert np.linalg.norm(fin1.v - fin0.v) <= 1e-10 * scale
    assert np.linalg.norm(fin1.w - fin0.w) <= 1e-10 * max(np.linalg.norm(fin0.w), scale)
    assert rel(fin1.q, fin0.q) <= 1e-8
    assert np.allclose(rep1.energy, rep0.energy, rtol=1e-10, atol=0)
    assert np.allclose(rep1.member_l2v_sq, rep0.member_l2v_sq, rtol=1e-10, atol=0)
    assert np.all(rep1.residuals[1:] <= 1e-11)
    assert snaps[2].v.shape == fin0.v.shape


def test_chunked_advance_roundtrip():
    """advance() through a chunked engine with host state in and out, two steps."""
    disc, cfg, prob = P.build_case("C1", J=6, steps=2)
    st = P.Problem(disc, prob.initial_v, prob.initial_w, prob.forcing, prob.boundary).initial_state(cfg)
    a1, _ = P.advance(st, cfg, disc, prob.forcing, prob.boundary)
    a2, _ = P.advance(a1, cfg, disc, prob.forcing, prob.boundary)
    ref = np.array(a2.v)
    ST.set_member_chunk(3)
    try:
        disc2, cfg2, prob2 = P.build_case("C1", J=6, steps=2)
        st = P.Problem(disc2, prob2.initial_v, prob2.initial_w, prob2.forcing, prob2.boundary).initial_state(cfg2)
        b1, _ = P.advance(st, cfg2, disc2, prob2.forcing, prob2.boundary)
        host = P.EnsembleState(v=np.array(b1.v), w=np.array(b1.w), q=np.array(b1.q), r=np.array(b1.r), step=1,
                               time=b1.time)
        b2, res = P.advance(host, cfg2, disc2, prob2.forcing, prob2.boundary)
    finally:
        ST.set_member_chunk(None)
    assert np.linalg.norm(b2.v - ref) <= 1e-12 * np.linalg.norm(ref) and res <= 1e-11


def test_largest_divisor():
    assert largest_divisor_at_most(1024, 100) == 64
    assert largest_divisor_at_most(20, 7) == 5
    assert largest_divisor_at_most(13, 5) == 1
