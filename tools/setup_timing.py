"""Setup-time breakdown at one BASELINE configuration.

python tools/setup_timing.py C5 [--steps 2]  -> one JSON line: build_case, analyse (plan),
HostMesh (rest), engine (device buffers, factor/apply plans), first step (factorisation +
graph capture), next steps; plus the host core count."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", nargs="?", default="C5")
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    import torch
    import paper_2108_05110_b200 as P
    from paper_2108_05110_b200 import engine as E, stepper as ST, symbolic as S
    out = dict(case=args.case, cores=os.cpu_count())
    t = time.perf_counter()
    disc, cfg, prob = P.build_case(args.case, steps=args.steps)
    out["build_case_s"] = time.perf_counter() - t
    t = time.perf_counter()
    plan = S.analyse(disc)
    out["analyse_s"] = time.perf_counter() - t
    orig = S.analyse
    S.analyse = lambda d, *a, **k: plan
    t = time.perf_counter()
    E.host_mesh(disc)
    out["hostmesh_rest_s"] = time.perf_counter() - t
    S.analyse = orig
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    torch.cuda.synchronize()
    t = time.perf_counter()
    eng = ST.get_engine(disc, cfg)
    torch.cuda.synchronize()
    out["engine_s"] = time.perf_counter() - t
    t = time.perf_counter()
    J = cfg.num_members
    eng.load_state(P.member_rows(prob.initial_v, 0, J), P.member_rows(prob.initial_w, 0, J), None, None)
    torch.cuda.synchronize()
    out["load_state_s"] = time.perf_counter() - t
    steps = []
    tt = 0.0
    for _ in range(args.steps):
        tt += cfg.dt
        t = time.perf_counter()
        eng.step(tt, prob.forcing, prob.boundary)
        torch.cuda.synchronize()
        steps.append(time.perf_counter() - t)
    out["step_s"] = steps
    out["setup_total_s"] = sum(out[k] for k in ("build_case_s", "analyse_s", "hostmesh_rest_s", "engine_s", "load_state_s"))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
