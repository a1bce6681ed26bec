"""World-size-2 gloo tests of the member-sharded step decomposition (CPU only).

Each rank owns a contiguous member shard and computes, with the CPU oracle,
exactly what its GPU kernels produce locally (member sums, per-quadrature
eddy maxima, its right-hand-side columns); the two exchanges of
`paper_2108_05110_b200.exchange` then must reproduce the single-process
ensemble quantities, and the shard's right-hand sides built from the
exchanged means must equal the corresponding columns of the full ensemble.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import ensmhd_oracle as O
        import paper_2108_05110_b200 as P
        from paper_2108_05110_b200 import exchange as XC
        from paper_2108_05110_b200 import fe

        disc, cfg, prob = P.build_case("C1", J=5, n=4)
        rng = np.random.default_rng(7)
        v = np.asarray(prob.initial_v) + 0.1 * rng.standard_normal((5, disc.n_vel))
        w = np.asarray(prob.initial_w) + 0.1 * rng.standard_normal((5, disc.n_vel))
        j0, jl = XC.member_slice(cfg.num_members, rank, world)
        vl, wl = v[j0:j0 + jl], w[j0:j0 + jl]
        # exchange 1: member sums -> global means
        sums = torch.from_numpy(np.concatenate([vl.sum(0), wl.sum(0)]).copy())
        XC.allreduce_member_sums(sums, dist.group.WORLD)
        means = sums.numpy() / cfg.num_members
        mv, mw = means[:disc.n_vel], means[disc.n_vel:]
        # exchange 2: local eddy maxima with the GLOBAL means -> global max
        def local_max(z, mean):
            vals = fe.eval_at_quadrature(disc.velocity, z - mean)
            return np.einsum("jeqd,jeqd->jeq", vals, vals).max(axis=0)
        msq = torch.from_numpy(np.stack([local_max(wl, mw), local_max(vl, mv)]).copy())
        XC.allreduce_eddy_max(msq, dist.group.WORLD)
        # shard RHS columns built from the exchanged means
        t = cfg.dt
        lv, lw = prob.forcing.loads(t, disc, cfg)
        bv, bw = prob.boundary.values(t, disc, cfg)
        from paper_2108_05110_b200.ensemble import viscosity_stats
        st = viscosity_stats(cfg)
        sl = slice(j0, j0 + jl)
        lag_cross = 0.5 * (cfg.nu - cfg.nu_m)[sl]
        lag_same = 0.5 * (st.nu_fluct + st.nu_m_fluct)[sl]
        r = disc.apply_mass(vl) / cfg.dt - O.convection_apply(disc.velocity, wl - mw, vl)
        r -= lag_cross[:, None] * disc.apply_stiffness(wl) + lag_same[:, None] * disc.apply_stiffness(vl)
        r += lv[sl]
        res = XC.allreduce_max_scalar(float(rank), dist.group.WORLD)
        out_q.put((rank, j0, jl, means, msq.numpy(), r, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_exchanges_reproduce_ensemble(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort()
    from oracle import ensmhd_oracle as O
    import paper_2108_05110_b200 as P
    from paper_2108_05110_b200 import fe
    disc, cfg, prob = P.build_case("C1", J=5, n=4)
    rng = np.random.default_rng(7)
    v = np.asarray(prob.initial_v) + 0.1 * rng.standard_normal((5, disc.n_vel))
    w = np.asarray(prob.initial_w) + 0.1 * rng.standard_normal((5, disc.n_vel))
    full_means = np.concatenate([v.mean(0), w.mean(0)])
    nut_w = O.eddy_viscosity(disc.velocity, w - w.mean(0), 1.0, 1.0)
    nut_v = O.eddy_viscosity(disc.velocity, v - v.mean(0), 1.0, 1.0)
    t = cfg.dt
    lv, lw = prob.forcing.loads(t, disc, cfg)
    bv, bw = prob.boundary.values(t, disc, cfg)
    rhs_full = O.rhs_block("v", v, w, lv, bv, cfg, disc)
    covered = []
    for rank, j0, jl, means, msq, r, res in outs:
        covered += list(range(j0, j0 + jl))
        assert np.allclose(means, full_means, rtol=1e-14, atol=1e-15)
        # means differ from numpy's pairwise mean only by summation order
        assert np.allclose(msq[0], nut_w, rtol=1e-12, atol=0) and np.allclose(msq[1], nut_v, rtol=1e-12, atol=0)
        ref = rhs_full[:disc.n_vel, j0:j0 + jl].T.copy()
        free = np.ones(disc.n_vel, dtype=bool)
        free[disc.bdofs] = False
        assert np.max(np.abs(r[:, free] - ref[:, free])) <= 1e-12 * np.abs(ref).max()
        assert res == world - 1
    assert covered == list(range(cfg.num_members))


def _gather_worker(rank, world, port, J, steps, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2108_05110_b200 import stepper as ST
        j0, jl = ST.member_slice(J, rank, world)
        # member diagnostics this rank would record per level: value = 1000*level + 10*member + key
        local = [np.array([[1000.0 * n + 10.0 * (j0 + j) + k for j in range(jl)] for k in range(6)])
                 for n in range(steps + 1)]
        rep = ST.RunReport(times=np.zeros(steps + 1), energy=np.zeros(steps + 1), div_v=np.zeros(steps + 1),
                           div_w=np.zeros(steps + 1), residuals=np.zeros(steps + 1), wall_clock=np.zeros(steps + 1),
                           alpha=np.zeros(J), mu=1.0, dt=1.0, member_l2v_sq=np.zeros((steps + 1, J)),
                           member_l2w_sq=np.zeros((steps + 1, J)), member_gradv_sq=np.zeros((steps + 1, J)),
                           member_gradw_sq=np.zeros((steps + 1, J)))
        ST._gather_records(rep, local, dist.group.WORLD, J)
        out_q.put((rank, rep.member_l2v_sq, rep.member_gradw_sq, rep.div_v, rep.div_w))
    finally:
        dist.destroy_process_group()


def test_run_records_gathered_once_uneven_shards():
    """Sharded run(): per-member diagnostics stay rank-local during the run and are gathered once at
    the end (padded all_gather), in member order, with uneven shards (J = 7 over 2 ranks)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    J, steps, world = 7, 3, 2
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, J, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = np.arange(steps + 1)[:, None]
    j = np.arange(J)[None, :]
    for _, l2v, gradw, div_v, div_w in outs:
        assert np.array_equal(l2v, 1000.0 * n + 10.0 * j + 0)
        assert np.array_equal(gradw, 1000.0 * n + 10.0 * j + 3)
        assert np.array_equal(div_v, 1000.0 * n[:, 0] + 10.0 * (J - 1) + 4)
        assert np.array_equal(div_w, 1000.0 * n[:, 0] + 10.0 * (J - 1) + 5)
