"""Golden outputs of the reference's error norms, rate tables and writers (build container only).

    python tests/golden/make_golden_reporting.py

Runs the REAL reference (`experiments.run_mms_case`, `error_norm_21`, `RateTable`,
`reporting.write_*`) on small inputs; `matplotlib` (imported at module level by
`reporting.py:13-18`, absent here) is stubbed -- no figure function is called.
Writes tests/golden/reporting_golden.json.
"""

import json
import os
import sys
import tempfile
import types

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
for name in ("matplotlib", "matplotlib.pyplot", "matplotlib.tri"):
    m = types.ModuleType(name)
    m.use = lambda *a, **k: None
    sys.modules[name] = m
sys.modules["matplotlib"].pyplot = sys.modules["matplotlib.pyplot"]
sys.modules["matplotlib"].tri = sys.modules["matplotlib.tri"]

import numpy as np  # noqa: E402

from ensmhd import experiments as X  # noqa: E402
from ensmhd import reporting as R  # noqa: E402
from ensmhd.ensemble import MemberParams  # noqa: E402
from ensmhd.mesh import barycentric_refine, build_structured_square  # noqa: E402


def main():
    out = {}
    members = (MemberParams(0.01, 0.1), MemberParams(0.012, 0.09), MemberParams(0.009, 0.11))
    res = X.run_mms_case(2, 0.05, 0.1, 0.01, members)
    out["mms_err_v"], out["mms_err_w"] = res.err_v, res.err_w
    steps = [0.25, 0.125, 0.0625]
    ev, ew = [3.1e-2, 8.2e-3, 2.05e-3], [1.7e-2, 4.1e-3, 1.1e-3]
    table = X.RateTable.from_errors("spatial", "h", steps, ev, ew)
    out["rates"] = [[r.step, r.err_v, r.rate_v, r.err_w, r.rate_w] for r in table.rows]
    mesh = barycentric_refine(build_structured_square(1))
    rng = np.random.default_rng(3)
    vel = rng.standard_normal((mesh.num_vertices, 2))
    sc = rng.standard_normal(mesh.num_vertices)
    with tempfile.TemporaryDirectory() as d:
        R.write_rate_csv(os.path.join(d, "r.csv"), table)
        R.write_energy_csv(os.path.join(d, "e.csv"), np.array([0.0, 0.05, 0.1]), np.array([1.5, 1.25, 1.125]))
        R.write_distance_csv(os.path.join(d, "d.csv"), [(0.01, 1.5e-3), (0.1, 2.5e-2)])
        R.write_vtk(os.path.join(d, "f.vtk"), mesh, {"velocity": vel, "speed": sc}, title="golden")
        for k in ("r.csv", "e.csv", "d.csv", "f.vtk"):
            out["file_" + k] = open(os.path.join(d, k)).read()
    out["vtk_vel"], out["vtk_speed"] = vel.tolist(), sc.tolist()
    path = os.path.join(HERE, "reporting_golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
