"""Member-sharded runs of the engine with two ranks against the unsharded run (SURVEY.md §8(c),(e)).

C5 has no CPU oracle; its parity is inherited from single-GPU parity plus this self-consistency:
two ranks, each holding half the members and exchanging the member sums (allreduce SUM) and the
eddy-viscosity maxima (allreduce MAX) every step, reproduce the one-rank run.  Both ranks run on
cuda:0 over gloo (the driver's GPU box has one GPU); the exchange logic is the same as over NCCL.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2108_05110_b200 as P  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case,over", [("C2", dict(J=20, steps=10)), ("C3", dict(n=32, J=6, steps=6)),
                                       ("C4", dict(k=2, J=5, steps=6))])
def test_two_rank_run_matches_single_rank(tmp_path, case, over):
    import json
    out = str(tmp_path / "run")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(HERE, "workers", "sharded_run.py"),
           out, case, json.dumps(over)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=dict(os.environ, OMP_NUM_THREADS="2"))
    assert r.returncode == 0, r.stderr[-4000:]
    parts = [np.load(f"{out}.rank{k}.npz") for k in range(2)]
    disc, cfg, prob = P.build_case(case, **over)
    rep, fin, _ = P.run(cfg, prob)
    v = np.concatenate([p["v"] for p in parts])
    w = np.concatenate([p["w"] for p in parts])
    q = np.concatenate([p["q"] for p in parts])
    scale_v = np.linalg.norm(fin.v)
    assert np.linalg.norm(v - fin.v) <= 1e-14 * scale_v
    assert np.linalg.norm(w - fin.w) <= 1e-14 * max(np.linalg.norm(fin.w), scale_v)
    # pressures: same bits up to the kernels' J-dependent tiling (rank shards have half the columns)
    assert np.linalg.norm(q - fin.q) <= 1e-10 * np.linalg.norm(fin.q)
    for p in parts:   # every rank reports the whole ensemble's diagnostics
        assert np.allclose(p["energy"], rep.energy, rtol=1e-14, atol=0)
        assert np.allclose(p["l2v"], rep.member_l2v_sq, rtol=1e-13, atol=0)
        # (the initial interpolant is divergence-free to round-off: compare against the series scale)
        assert np.allclose(p["div_v"], rep.div_v, rtol=1e-12, atol=1e-9 * rep.div_v.max()), (p["div_v"], rep.div_v)
        assert np.all(p["residuals"][1:] <= 1e-11)
