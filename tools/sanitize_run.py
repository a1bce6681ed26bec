"""Small workloads that touch every default-path kernel, for compute-sanitizer (memcheck / racecheck /
synccheck):  classic solve path (odd J), streamed solve path (even J), chunked engine, lower seams,
device error norms.  profiles/r02_sanitizer.md records the runs.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("ENS_STEP_GRAPH", "0")
import numpy as np

import paper_2108_05110_b200 as P
from paper_2108_05110_b200 import stepper as ST
from paper_2108_05110_b200.problems import BaselineMmsExact

for J in (3, 4):                                   # J=3: classic k_sgemm solve; J=4: streamed solve
    disc, cfg, prob = P.build_case("C1", n=6, J=J, steps=3)
    rep, fin, _ = P.run(cfg, prob, exact=BaselineMmsExact())
    assert np.all(np.isfinite(fin.v)) and rep.residuals[1:].max() < 1e-10, rep.residuals
ST.set_member_chunk(2)                             # chunked engine
disc, cfg, prob = P.build_case("C1", n=6, J=4, steps=2)
rep, fin, _ = P.run(cfg, prob)
ST.set_member_chunk(None)
assert np.all(np.isfinite(fin.v))
disc, cfg, prob = P.build_case("C4", k=1, J=2, steps=2, length=8.0)   # no pin, do-nothing outflow
rep, fin, _ = P.run(cfg, prob)
st = P.EnsembleState(v=np.asarray(prob.initial_v), w=np.asarray(prob.initial_w), q=np.zeros((2, disc.n_pres)),
                     r=np.zeros((2, disc.n_pres)))
sysm = P.assemble_shared_lhs(P.StepKind.V_STEP, st.mean_w, st.w - st.mean_w, cfg, disc)
x = sysm.factorization.solve_block(np.ones((disc.n_total, 2)))
assert np.all(np.isfinite(x))
print("sanitize workload done")
