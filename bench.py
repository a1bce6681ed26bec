#!/usr/bin/env python
"""Benchmark: ensemble member-timesteps/s of the B200 time-step path (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[1] = "C2": manufactured MHD problem on the
unit square, 128x128 cells (2 triangles each), Taylor-Hood P2/P1, fp64, J=20
members, dt=0.005.  A bench *step* is one full time-step
(both Elsasser sub-steps, all members): member sums, right-hand sides, eddy
viscosity, shared-matrix assembly, multifrontal LU of both saddle matrices,
column-batched FGMRES to a true relative residual of 1e-12 per member, and
the pressure epilogue.  For N>1 (torchrun, one rank per GPU) the workload is
BASELINE configs[4] = "C5" (512x512, J = 1024 members in total, strong
scaling: 1024/N per GPU, chunked when a shard does not fit at once) and every
step does the two real exchanges of the scheme over NCCL: allreduce SUM of the
member sums and allreduce MAX of the eddy-viscosity maxima.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line on rank 0.  See DESIGN.md §6 for every field.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ensemble member-timesteps/sec at fixed mesh"
UNIT = "member-steps/s"
CASE = "C2"
CASE_MULTI = "C5"
J_PER_GPU = 20
# BASELINE configurations (bench.py --case): (members, scaling, workload text).  "weak": members per
# GPU; "strong": members in total, sharded over the GPUs.
CASES = {
    "C2": (20, "weak", "C2: unit square 128x128, TH P2/P1, J=20/GPU, dt=0.005"),
    "C3": (64, "weak", "C3: lid-driven cavity, unit square 256x256, TH P2/P1, J=64/GPU, s=1, dt=0.01"),
    "C4": (128, "weak", "C4: channel past a step [0,30]x[0,10], h=1/8, TH P2/P1, J=128/GPU, delta=0.1, dt=0.02"),
    "C5": (1024, "strong", "C5: unit square 512x512, TH P2/P1, J=1024 sharded over the GPUs, dt=0.002"),
    "C5shard": (128, "weak", "C5 shard: unit square 512x512, TH P2/P1, J=128/GPU (the 8-GPU shard of J=1024), "
                             "dt=0.002"),
}


def single_thread():
    """Pin this process to one core and one BLAS thread: the reference path is serial (SuperLU,
    sparsetools and einsum; SURVEY.md §8(d) measured 8 BLAS threads slower)."""
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except (AttributeError, OSError):
        pass
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


REF_NOTE = ("reference solve backend: SciPy SuperLU -- the reference's fallback (linalg.py:86-108); its default, "
            "UMFPACK via cvxopt, is not installable here (no cvxopt wheel)")


def fp64_peak():
    """Measured fp64 tensor-core (DMMA) rate, TFLOP/s (profiles/r01_fp64_peak.json, tools/fp64_peak.cu)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as f:
            return float(json.load(f)["dmma_m8n8k4_tflops"]), "measured"
    except Exception:
        return 37.0, "fallback"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region.

    In-process NVML (nvidia_ml_py) from a sampling thread every few milliseconds, so that a timed
    region of ~20 ms holds several samples; `nvidia-smi -lms` in a subprocess when NVML cannot be
    loaded (its 100 ms period then only brackets the region)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index, period_s=0.004):
        self.index = index
        self.period = period_s
        self.proc = None
        self.thread = None
        self.samples = []          # (sm MHz, reasons bitmask)
        self.max_mhz = None
        self._stop = False
        self.kind = os.environ.get("BENCH_SAMPLER", "nvml")

    def _nvml_loop(self, nv, h):
        while not self._stop:
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.kind == "nvml":
            try:
                import threading
                import pynvml as nv
                nv.nvmlInit()
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[self.index].isdigit() else self.index
                h = nv.nvmlDeviceGetHandleByIndex(idx)
                self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
                self._nv = nv
                self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
                self.thread.start()
                return
            except Exception:
                self.thread = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def ready(self):
        """True once the sampler has delivered (nvml) or had time to deliver (nvidia-smi) a first sample."""
        return len(self.samples) > 0 if self.thread is not None else False

    def stop(self):
        if self.thread is not None:
            time.sleep(3 * self.period)
            self._stop = True
            self.thread.join(timeout=2)
            nv = self._nv
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            reasons = sorted(n for n, b in bits.items() if any(r & b for _, r in self.samples))
            sm = [c for c, _ in self.samples]
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(sm), "sampler": "nvml in-process, every 4 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=5)
        sm, mx, reasons = [], [], set()
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "sampler": "nvidia-smi -lms 100"}


def cpu_baseline(disc, cfg, prob, steps=1):
    """The oracle (numpy/SciPy port of the reference path) on this host: bounded sample."""
    from oracle import ensmhd_oracle as O
    J = cfg.num_members
    st = O.OracleState(np.array(prob.initial_v, float), np.array(prob.initial_w, float),
                       np.zeros((J, disc.n_pres)), np.zeros((J, disc.n_pres)))
    t0 = time.perf_counter()
    for _ in range(steps):
        st, _ = O.advance(st, cfg, disc, prob.forcing, prob.boundary)
    dt = time.perf_counter() - t0
    return J * steps / dt, dt


def run_reference(args):
    """--impl reference: the reference path's CPU restatement (oracle port, pinned to the reference's
    own outputs) on one host core, same config / metric as the b200 arm, bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    single_thread()
    import paper_2108_05110_b200 as P
    case = args.case or (CASE if args.gpus == 1 else CASE_MULTI)
    jn, scaling, workload = CASES[case]
    J = jn * args.gpus if scaling == "weak" else jn
    sample = dict(J=J)
    note = ""
    if case in ("C5", "C5shard") or J > 64:
        # SuperLU on the 512x512 saddle system (N = 2.36M) does not finish in a bounded sample: time
        # the reference algorithm on C2's mesh with the config's member count, per member-step
        sample = dict(J=J)
        case_run, note = "C2", f" on the C2 mesh (the {case} mesh is infeasible for SuperLU on one core)"
    else:
        case_run = case
    disc, cfg, prob = P.build_case(case_run, **sample)
    steps = 1
    value, secs = cpu_baseline(disc, cfg, prob, steps)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": steps,
        "warmup": 0, "ms_per_step": 1e3 * secs / steps, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded manufactured solution, SURVEY.md §8.0)",
        "config": {"workload": workload, "case": case, "members_total": J},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"{steps} full time-step of {case_run} with {J} members{note}, 1 thread pinned "
                                   f"to one core of {os.cpu_count()}; {REF_NOTE}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spmm_traffic(name="r01_spmm_traffic.json"):
    """DRAM bytes per launch from a committed ncu capture (profiles/), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name)
    try:
        with open(path) as fh:
            return int(json.load(fh)["traffic_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        return None


def cusparse_spmm_ms(eng, disc, reps=20):
    """The library bar: cuSPARSE SpMM (torch.sparse.mm on CSR, fp64)
    of the same saddle matrices (reference order, identity rows included) times the same member
    block, both systems; CUDA events, warm."""
    import torch
    from paper_2108_05110_b200 import linalg as LA
    mats, xs = [], []
    for m in range(2):
        a = LA.saddle_matrix(disc, eng.as_vals[m].cpu().numpy())
        mats.append(torch.sparse_csr_tensor(torch.as_tensor(a.indptr.astype(np.int32)),
                                            torch.as_tensor(a.indices.astype(np.int32)),
                                            torch.as_tensor(a.data), size=a.shape).cuda())
        xs.append(torch.randn(a.shape[0], eng.J, dtype=torch.float64, device="cuda"))
    for m in range(2):
        torch.sparse.mm(mats[m], xs[m])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for m in range(2):
            torch.sparse.mm(mats[m], xs[m])
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--always-steps", type=int, default=5)
    ap.add_argument("--full-run", type=int, default=-1,
                    help="also time run() over this many steps (-1: the config's own step count at N=1 for C2)")
    ap.add_argument("--case", default=None, choices=sorted(CASES),
                    help="default: C2 at N=1, C5 (strong scaling, J=1024 in total) at N>1")
    args = ap.parse_args()
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.case is None:
        args.case = CASE if max(world_env, args.gpus) == 1 else CASE_MULTI
    case = args.case
    jn, scaling, workload = CASES[case]
    if case != CASE:
        args.no_cpu_baseline = True   # the SciPy oracle needs minutes to hours per step beyond C2
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = world_env
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    _stdout_fd = None
    # BENCH_FORCE_DIST=1 (testing only): take the sharded code path even on one rank
    if world > 1 or os.environ.get("BENCH_FORCE_DIST") == "1":
        # library banners printed to the process's stdout (NCCL / c10d communicator set-up) are sent
        # to stderr until the result line, so rank 0's stdout is exactly one JSON line
        sys.stdout.flush()
        _stdout_fd = os.dup(1)
        os.dup2(2, 1)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = dist.group.WORLD
    import paper_2108_05110_b200 as P
    from paper_2108_05110_b200 import stepper as ST
    from paper_2108_05110_b200.engine import _dptr, apply_bytes, apply_flops, spmm_bytes
    from paper_2108_05110_b200 import _native as N

    J_total = jn * world if scaling == "weak" else jn
    spec_case = "C5" if case == "C5shard" else case
    # setup, cold: the on-disk setup cache points at a fresh directory
    import tempfile
    from paper_2108_05110_b200 import setup_cache as SC
    from paper_2108_05110_b200.engine import host_mesh
    cache_tmp = tempfile.mkdtemp(prefix="bench_setup_cache_")
    os.environ["ENS_SETUP_CACHE"] = cache_tmp
    setup = {}
    tq = time.perf_counter()
    disc, cfg, prob = P.build_case(spec_case, J=J_total, steps=max(args.steps + args.warmup, 1))
    setup["build_case_s"] = time.perf_counter() - tq
    tq = time.perf_counter()
    host_mesh(disc)
    setup["host_mesh_cold_s"] = time.perf_counter() - tq
    setup["cache"] = dict(SC.last)
    j0, jl = ST.member_slice(J_total, rank, world)
    torch.cuda.synchronize()
    tq = time.perf_counter()
    eng = ST.get_engine(disc, cfg, j0=j0, J=jl, comm=comm)
    eng.load_state(P.member_rows(prob.initial_v, j0, jl), P.member_rows(prob.initial_w, j0, jl), None, None)
    torch.cuda.synchronize()
    setup["engine_and_state_s"] = time.perf_counter() - tq
    # warm: a second Discretization of the same mesh finds the entry the cold pass wrote
    tq = time.perf_counter()
    disc_w, _, _ = P.build_case(spec_case, J=J_total, steps=1)
    tb = time.perf_counter()
    host_mesh(disc_w)
    setup["host_mesh_warm_s"] = time.perf_counter() - tb
    setup["warm_hit"] = bool(SC.last.get("hit"))
    del disc_w
    import shutil
    shutil.rmtree(cache_tmp, ignore_errors=True)
    setup["cold_s"] = setup["build_case_s"] + setup["host_mesh_cold_s"] + setup["engine_and_state_s"]
    setup["warm_s"] = setup["build_case_s"] + setup["host_mesh_warm_s"] + setup["engine_and_state_s"]
    setup["note"] = ("wall clock, host + device: build_case (mesh, spaces, constant operators), HostMesh "
                     "(multifrontal plan + operator maps; cold = built, warm = loaded from the on-disk "
                     "setup cache written by the cold pass), engine creation + initial state upload; "
                     "the first step's factorisation and graph capture are not included")
    t = 0.0
    ahead = getattr(eng, "supports_ahead", False)
    for _ in range(args.warmup):
        t += cfg.dt
        if ahead:   # (announced like the timed steps: the first announcement sets up per-parity buffers and graphs)
            eng.step(t, prob.forcing, prob.boundary, then=(t + cfg.dt, prob.forcing, prob.boundary))
        else:
            eng.step(t, prob.forcing, prob.boundary)
    torch.cuda.synchronize()
    if comm is not None:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    # the sampler needs a moment to deliver its first sample: the GPU keeps stepping meanwhile (untimed,
    # announced like the timed steps), so the timed region starts on a busy GPU, not after an idle gap
    t_wait = time.perf_counter()
    busy = os.environ.get("BENCH_IDLE", "busy") == "busy"
    extra_warm = 0

    def keep_waiting():
        if comm is not None:
            # every rank must run the same number of steps (a step holds collectives): a fixed count
            return extra_warm < 2
        return time.perf_counter() - t_wait < 0.3 and not (busy and sampler.ready() and
                                                           time.perf_counter() - t_wait > 0.02)

    while keep_waiting():
        if busy or comm is not None:
            t += cfg.dt
            extra_warm += 1
            if ahead:
                eng.step(t, prob.forcing, prob.boundary, then=(t + cfg.dt, prob.forcing, prob.boundary))
            else:
                eng.step(t, prob.forcing, prob.boundary)
        else:
            time.sleep(0.01)
    s = eng.stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if comm is not None:
        dist.barrier()
    w0 = time.perf_counter()
    l0 = eng.lib.ens_kernel_launches()
    c0 = eng.graph_launch_credit
    nf0 = eng.n_factor
    ev0.record(s)
    iters = []
    for i in range(args.steps):
        t += cfg.dt
        # as run() does: every step but the last announces the next call, whose pre-solve graph the
        # engine then enqueues before returning (the time loop's host work overlaps GPU work)
        if ahead and i + 1 < args.steps:
            eng.step(t, prob.forcing, prob.boundary, then=(t + cfg.dt, prob.forcing, prob.boundary))
        else:
            eng.step(t, prob.forcing, prob.boundary)
        iters.append(eng.last_iters)
    ev1.record(s)
    torch.cuda.synchronize()
    launches = int(eng.lib.ens_kernel_launches() - l0) + (eng.graph_launch_credit - c0)   # + step-graph replays
    n_factor = eng.n_factor - nf0
    wall = time.perf_counter() - w0
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    tmax = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if comm is not None:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms = float(tmax.item())
    value = J_total * args.steps / (ms / 1e3)
    Jc = getattr(eng, "Jc", jl)          # columns per device pass (chunked engines)

    # ---- end-to-end through the public reference-facing API with host buffers ----
    # (this leg continues the timed steps' trajectory, so it runs right after them)
    e2e = None
    if world == 1 and args.e2e_steps > 0:
        from paper_2108_05110_b200.ensemble import EnsembleState
        # the trajectory of the timed steps continues, now through host arrays (a restart from the initial
        # state would re-enter the start-up transient with the factorisation of a later time: two-cycle solves)
        st = EnsembleState(step=args.warmup + extra_warm + args.steps, time=t, device=eng.state_handle())
        host = EnsembleState(v=st.v, w=st.w, q=st.q, r=st.r, step=st.step, time=st.time)
        for _ in range(max(10, args.warmup)):   # warm: engine, graphs, pinned host-buffer cache, one-cycle solves
            st, _ = P.advance(host, cfg, disc, prob.forcing, prob.boundary)
            host = EnsembleState(v=st.v, w=st.w, q=st.q, r=st.r, step=st.step, time=st.time)
        del st                                   # only the live state keeps pinned buffers
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        marks = []
        for _ in range(args.e2e_steps):
            new, _ = P.advance(host, cfg, disc, prob.forcing, prob.boundary)
            host = EnsembleState(v=new.v, w=new.w, q=new.q, r=new.r, step=new.step, time=new.time)
            marks.append(time.perf_counter())
        e2e_s = time.perf_counter() - t0
        step_ms = [round(1e3 * (b - a), 3) for a, b in zip([t0] + marks[:-1], marks)]
        per_v = 8 * J_total * 2 * disc.n_vel                   # v, w
        per = per_v + 8 * J_total * 2 * disc.n_pres           # v, w, q, r
        # H2D: v, w every step (q, r only when the velocities are not the resident level, never
        # here) + the problem-data coefficients; D2H: the full new state + the residual
        e2e = {"value": J_total * args.e2e_steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": per_v + 8 * 2 * 2 * 3 * J_total,
               "d2h_bytes_per_step": per + 16, "steps": args.e2e_steps, "step_ms": step_ms,
               "api": "paper_2108_05110_b200.advance(state, config, disc, forcing, boundary), numpy state in/out"}
        # the transfer floor the e2e step runs against: pinned host<->device copy bandwidth measured here
        # (CUDA events, best of 5, one buffer of the per-step state size), plus the device-timed step
        hb = torch.empty(per // 8, dtype=torch.float64, pin_memory=True)
        db = torch.empty(per // 8, dtype=torch.float64, device="cuda")
        pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        bw = {}
        for name, dst, src in (("h2d", db, hb), ("d2h", hb, db)):
            best = None
            for _ in range(5):
                pe0.record()
                dst.copy_(src, non_blocking=True)
                pe1.record()
                pe1.synchronize()
                tt = pe0.elapsed_time(pe1)
                best = tt if best is None else min(best, tt)
            bw[name] = per / (best * 1e-3) / 1e9
        del hb, db
        ms_step = ms / args.steps
        floor = ms_step + 1e3 * (e2e["h2d_bytes_per_step"] / (bw["h2d"] * 1e9) + e2e["d2h_bytes_per_step"] / (bw["d2h"] * 1e9))
        e2e["transfer_floor"] = {"h2d_gbs": bw["h2d"], "d2h_gbs": bw["d2h"], "device_step_ms": ms_step,
                                 "floor_ms": floor, "frac": floor / float(np.median(step_ms))}

    # ---- per-phase device timing (same stream, CUDA events), for the roofline ----
    def time_call(fn, reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        a.record(s)
        for _ in range(reps):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    X = eng.X[eng.cur]
    Y = eng.rhs            # scratch between steps (no extra device memory at the largest configs)
    spmm_ms = time_call(lambda: N.check(eng.lib.ens_spmm(eng.ctx, eng.sptr, _dptr(eng.as_vals), _dptr(X), None,
                                                         _dptr(Y), 0), "spmm"), 50)
    factor_ms = time_call(lambda: eng.factor(), 3 if case.startswith("C5") else 5)
    Z = eng.rhs
    solve_ms = time_call(lambda: eng.precond(X, out=Z), 10)
    bytes_spmm = spmm_bytes(eng.hm, Jc)
    hbm, peak_kind = peaks()
    spmm_gbs = bytes_spmm / (spmm_ms * 1e-3) / 1e9
    plan = eng.hm.plan
    solve_bytes = apply_bytes(eng.hm, Jc)
    solve_gbs = solve_bytes / (solve_ms * 1e-3) / 1e9
    solve_flops = apply_flops(eng.hm, Jc)
    solve_tflops = solve_flops / (solve_ms * 1e-3) / 1e12
    f64_peak, f64_kind = fp64_peak()
    factor_tflops = 2 * plan.stats["factor_flops"] / (factor_ms * 1e-3) / 1e12
    cus_ms = None
    if rank == 0 and world == 1:
        try:
            cus_ms = cusparse_spmm_ms(eng, disc)
        except Exception as exc:   # library timing leg only
            print(f"cusparse leg skipped: {exc}", file=sys.stderr)

    # ---- same workload with the LU preconditioner rebuilt every step (reference cadence) ----
    always = None
    from paper_2108_05110_b200.chunked import ChunkedEngine
    # (a member-chunked engine fills the device: a second engine for this leg does not fit)
    if args.always_steps > 0 and world == 1 and not isinstance(eng, ChunkedEngine):
        saved = ST.get_solver_options()
        ST.set_solver_options(refactor="always")
        eng2 = ST.get_engine(disc, cfg, j0=j0, J=jl, comm=comm)
        ST.set_solver_options(**saved)
        eng2.load_state(P.member_rows(prob.initial_v, j0, jl), P.member_rows(prob.initial_w, j0, jl), None, None)
        t2 = 0.0
        for _ in range(2):
            t2 += cfg.dt
            eng2.step(t2, prob.forcing, prob.boundary)
        torch.cuda.synchronize()
        a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a2.record(eng2.stream)
        for _ in range(args.always_steps):
            t2 += cfg.dt
            eng2.step(t2, prob.forcing, prob.boundary)
        b2.record(eng2.stream)
        torch.cuda.synchronize()
        ms2 = a2.elapsed_time(b2)
        always = {"value": J_total * args.always_steps / (ms2 / 1e3), "unit": UNIT,
                  "steps": args.always_steps, "ms_per_step": ms2 / args.always_steps}
        del eng2

    # ---- the whole run() of the configuration: start-up steps and rebuilds included ----
    full = None
    nfull = args.full_run if args.full_run >= 0 else (P.problems.CONFIGS[case]["steps"] if case == CASE and
                                                      world == 1 else 0)
    if nfull > 0 and world == 1:
        dfull, cfull, pfull = P.build_case(spec_case, J=J_total, steps=nfull)
        P.run(cfull, pfull, record=False)                  # engine, graphs, pinned buffers warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep, _, _ = P.run(cfull, pfull, record=False)
        tot = time.perf_counter() - t0
        step_s = float(np.sum(rep.wall_clock[1:]))
        efull = ST.get_engine(dfull, cfull)
        full = {"value": J_total * nfull / step_s, "unit": UNIT, "steps": nfull,
                "ms_per_step": 1e3 * step_s / nfull, "factorizations": int(efull.n_factor),
                "wall_s_incl_host": tot,
                "api": "paper_2108_05110_b200.run(config, problem) over the configuration's full step count "
                       "(RunReport.wall_clock, the reference's own timing; per-step diagnostics off)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        single_thread()
        v, secs = cpu_baseline(disc, cfg, prob, 1)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"1 full time-step of {CASE} with all {J_total} members by the numpy/SciPy oracle "
                         f"(1 thread pinned to one core), {secs:.1f} s; {REF_NOTE}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded manufactured solution, SURVEY.md §8.0)",
            "config": {"workload": workload,
                       "case": case, "members_total": J_total, "members_per_pass": Jc, "n_total_dofs": int(eng.ntot),
                       "l2": "per-step working set (2 x %.2f GB fronts) exceeds the 126 MB L2" %
                             (plan.front_storage * 8 / 1e9),
                       "rtol": eng.rtol, "parallelism": f"members sharded dp{world}",
                       "warmup_extra_steps": extra_warm,
                       "warmup_note": "untimed steps run while the clock sampler delivers its first sample "
                                      "(the timed region starts on a busy GPU), on top of --warmup"},
            "wall_s": wall, "setup": setup,
            "krylov_iters_per_step": float(np.mean(iters)) if iters else None,
            "preconditioner": {"policy": eng.refactor, "factorizations_in_timed_steps": n_factor,
                               "lag_max_iters": eng.lag_max_iters, "lag_max_steps": eng.lag_max_steps,
                               "renewal_rho": eng.rho,
                               "note": "every sub-step solve converged to the same 1e-12 true residual; "
                                       "renewal decided from iteration counts (deterministic)"},
            "value_full_run": full,
            "value_refactor_every_step": always,
            # dominant kernel of a timed step: the preconditioner apply (k_sgemm + k_finit sweep),
            # against the nearer of its two roofs (HBM for small J, fp64 tensor cores for large J)
            "roofline": (
                {"bound": "hbm", "kernel": "ens_precond_apply (multifrontal forward+backward sweep, "
                                           "both systems; streamed k_stream_gemm dominant)",
                 "achieved": solve_gbs, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                 "frac": solve_gbs / hbm,
                 "traffic": spmm_traffic("r02_apply_traffic.json") if case == CASE else None,
                 "bytes_per_launch": solve_bytes, "ms_per_launch": solve_ms,
                 "other_roof": {"bound": "tensor (fp64 DMMA)", "achieved": solve_tflops, "peak": f64_peak,
                                "peak_kind": f64_kind, "unit": "TFLOP/s", "frac": solve_tflops / f64_peak}}
                if solve_gbs / hbm >= solve_tflops / f64_peak else
                {"bound": "tensor", "kernel": "ens_precond_apply (multifrontal forward+backward sweep, both "
                                              "systems; k_sgemm on fp64 tensor cores, mma.sync m8n8k4)",
                 "achieved": solve_tflops, "peak": f64_peak, "peak_kind": f64_kind, "unit": "TFLOP/s",
                 "frac": solve_tflops / f64_peak, "traffic": None, "flops_per_launch": solve_flops,
                 "ms_per_launch": solve_ms,
                 "other_roof": {"bound": "hbm", "achieved": solve_gbs, "peak": hbm, "unit": "GB/s",
                                "frac": solve_gbs / hbm, "bytes_per_launch": solve_bytes}}),
            "roofline_spmm": {"bound": "hbm", "kernel": "ens_spmm (saddle SpMM, both systems; the Krylov core)",
                              "achieved": spmm_gbs, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                              "frac": spmm_gbs / hbm,
                              "traffic": spmm_traffic("r02_spmm_traffic.json") if case == CASE else None,
                              "bytes_per_launch": bytes_spmm, "ms_per_launch": spmm_ms,
                              "cusparse": None if cus_ms is None else {
                                  "ms_per_launch": cus_ms, "achieved": bytes_spmm / (cus_ms * 1e-3) / 1e9,
                                  "speedup_of_ens_spmm": cus_ms / spmm_ms,
                                  "how": "torch.sparse.mm(CSR fp64 saddle matrix, dense N x J) = cusparseSpMM, "
                                         "both systems, warm, CUDA events"}},
            "phases_ms": {"spmm": spmm_ms, "factor": factor_ms, "lu_solve": solve_ms,
                          "factor_tflops_fp64": factor_tflops, "lu_solve_gbs": solve_gbs},
            "clocks": clocks,
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if _stdout_fd is not None:
            sys.stdout.flush()
            os.dup2(_stdout_fd, 1)
        print(json.dumps(line), flush=True)
    if comm is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
