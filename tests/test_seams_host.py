"""Host-side pieces of the lower seams (CPU): the CSR read-back of a sub-step matrix and the A_s
extraction `factorize` performs are inverse to each other on oracle-assembled saddle matrices."""

import numpy as np
import pytest

from oracle import ensmhd_oracle as O
import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import linalg as LA


@pytest.mark.parametrize("case,over", [("C1", dict(n=4, J=3)), ("C4", dict(k=1, J=3, length=8.0))])
def test_saddle_readback_roundtrip(case, over, rng):
    disc, cfg, prob = P.build_case(case, **over)
    v = np.asarray(prob.initial_v) + 0.1 * rng.standard_normal((3, disc.n_vel))
    w = np.asarray(prob.initial_w) + 0.1 * rng.standard_normal((3, disc.n_vel))
    ref = O.shared_matrix("v", v, w, cfg, disc)
    sym = LA.SaddleSymbolic(disc)
    vals = sym.velocity_values(ref)
    back = LA.saddle_matrix(disc, vals)
    assert np.array_equal(back.toarray(), ref.toarray())


def test_factorize_needs_saddle_symbolic():
    disc, cfg, prob = P.build_case("C1", n=2, J=1)
    m = O.shared_matrix("v", np.asarray(prob.initial_v), np.asarray(prob.initial_w), cfg, disc)
    with pytest.raises(ValueError):
        P.factorize(m)
    f = P.factorize(m, symbolic=LA.SaddleSymbolic(disc))
    assert f.backend == "b200" and f.shape == m.shape
