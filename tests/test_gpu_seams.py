"""The reference's lower seams on the GPU engine, tested the way the reference tests them.

Mirrors the classes of the reference's `tests/test_stepper.py` (TestSharedMatrix,
TestMemberRhs, TestRun, the stability bound) and `tests/test_linalg.py` (block solve
equals stacked single solves, agreement with a dense LU), against this package's
`assemble_shared_lhs`, `assemble_member_rhs` (`stepper.py:181-278`) and
`factorize(...).solve/solve_block` (`linalg.py:46-108`).  Dense references come
from the REAL reference (`tests/golden/reference_golden.npz`, made by
`tests/golden/make_golden.py`: the reference's own assemble_shared_lhs/_rhs_block
on the barycentric 2x2 square with a perturbed 3-member state).
"""

import numpy as np
import pytest
import scipy.sparse as sp

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2108_05110_b200 as P  # noqa: E402
from paper_2108_05110_b200 import linalg as LA  # noqa: E402
from paper_2108_05110_b200.discretization import Discretization  # noqa: E402
from paper_2108_05110_b200.ensemble import EnsembleConfig, EnsembleState, MemberParams  # noqa: E402
from paper_2108_05110_b200.mesh import barycentric_refine, build_structured_square  # noqa: E402
from paper_2108_05110_b200.problems import ZeroBoundary, ZeroForcing, paper_mms_initial_fields  # noqa: E402
from paper_2108_05110_b200.stepper import StepKind  # noqa: E402


def simple_config(members=None, dt=0.05, t_end=0.25, eps=0.0, mu=1.0):
    members = (MemberParams(0.01, 0.1),) if members is None else members
    return EnsembleConfig(members=members, coupling=1.0, mu=mu, dt=dt, t_end=t_end, perturbation=eps)


@pytest.fixture(scope="module")
def tiny_disc():
    return Discretization.from_mesh(barycentric_refine(build_structured_square(2)))


def sv2_config():
    members = (MemberParams(0.01, 0.1), MemberParams(0.012, 0.09), MemberParams(0.009, 0.11))
    return EnsembleConfig(members=members, coupling=1.0, mu=1.0, dt=0.05, t_end=0.1, perturbation=0.01)


def zero_state(config, disc):
    j = config.num_members
    return EnsembleState(v=np.zeros((j, disc.n_vel)), w=np.zeros((j, disc.n_vel)), q=np.zeros((j, disc.n_pres)),
                         r=np.zeros((j, disc.n_pres)))


# ----------------------------------------------------------------------------------------------
# shared matrix
# ----------------------------------------------------------------------------------------------

def test_shared_matrix_member_independence_bitwise(tiny_disc, rng):
    config = simple_config(members=tuple(MemberParams(0.01 + 0.001 * j, 0.1) for j in range(4)))
    mean_adv = rng.standard_normal(tiny_disc.n_vel)
    flucts = rng.standard_normal((4, tiny_disc.n_vel))
    systems = [P.assemble_shared_lhs(StepKind.V_STEP, mean_adv, flucts, config, tiny_disc) for _ in range(4)]
    ref = systems[0].matrix
    for s in systems[1:]:
        assert np.array_equal(ref.data, s.matrix.data)
        assert np.array_equal(ref.indices, s.matrix.indices) and np.array_equal(ref.indptr, s.matrix.indptr)


def test_shared_matrix_term_dropout_with_zero_fields(tiny_disc):
    config = simple_config()
    system = P.assemble_shared_lhs(StepKind.V_STEP, np.zeros(tiny_disc.n_vel), np.zeros((1, tiny_disc.n_vel)),
                                   config, tiny_disc)
    a_s = tiny_disc.mass_s / config.dt + 0.5 * (0.01 + 0.1) * tiny_disc.stiff_s
    ns = tiny_disc.n_scalar
    bx, by = tiny_disc.divergence[:, :ns], tiny_disc.divergence[:, ns:]
    expected = sp.bmat([[a_s, None, -bx.T], [None, a_s, -by.T], [bx, by, None]], format="lil")
    for r in tiny_disc.constrained_rows:
        expected.rows[r], expected.data[r] = [int(r)], [1.0]
    got, exp = system.matrix.toarray(), expected.toarray()
    assert np.max(np.abs(got - exp)) <= 1e-15 * np.abs(exp).max()


@pytest.mark.parametrize("kind,name,field", [(StepKind.V_STEP, "V", "w"), (StepKind.W_STEP, "W", "v")])
def test_shared_matrix_matches_reference(golden, kind, name, field):
    disc = Discretization.from_mesh(barycentric_refine(build_structured_square(2)))
    z = golden["sv2_pert_" + field]
    mean = z.mean(axis=0)
    system = P.assemble_shared_lhs(kind, mean, z - mean, sv2_config(), disc)
    ref = golden["sv2_mat" + name]
    assert np.max(np.abs(system.matrix.toarray() - ref)) <= 1e-13 * np.abs(ref).max()
    assert system.step_kind is kind and system.rhs.shape == (disc.n_total, 3)


# ----------------------------------------------------------------------------------------------
# member right-hand sides
# ----------------------------------------------------------------------------------------------

def test_member_rhs_zero_everything_gives_zero(tiny_disc):
    config = simple_config()
    rhs = P.assemble_member_rhs(StepKind.V_STEP, 0, zero_state(config, tiny_disc), None,
                                np.zeros(tiny_disc.bdofs.size), config, tiny_disc)
    assert np.all(rhs == 0.0)


def test_member_rhs_single_member_fluctuation_term_vanishes(tiny_disc, rng):
    config = simple_config()
    v = rng.standard_normal((1, tiny_disc.n_vel))
    w = rng.standard_normal((1, tiny_disc.n_vel))
    state = EnsembleState(v=v, w=w, q=np.zeros((1, tiny_disc.n_pres)), r=np.zeros((1, tiny_disc.n_pres)))
    rhs = P.assemble_member_rhs(StepKind.V_STEP, 0, state, None, np.zeros(tiny_disc.bdofs.size), config,
                                tiny_disc)
    expected = np.zeros(tiny_disc.n_total)
    expected[:tiny_disc.n_vel] = (tiny_disc.apply_mass(v[0]) / config.dt
                                  - 0.5 * (0.01 - 0.1) * tiny_disc.apply_stiffness(w[0]))
    expected[tiny_disc.bdofs] = 0.0
    expected[tiny_disc.pin_row] = 0.0
    assert np.allclose(rhs, expected, atol=1e-13)


@pytest.mark.parametrize("kind,name,fam", [(StepKind.V_STEP, "V", "v"), (StepKind.W_STEP, "W", "w")])
def test_member_rhs_matches_reference(golden, kind, name, fam):
    disc = Discretization.from_mesh(barycentric_refine(build_structured_square(2)))
    cfg = sv2_config()
    state = EnsembleState(v=golden["sv2_pert_v"], w=golden["sv2_pert_w"], q=np.zeros((3, disc.n_pres)),
                          r=np.zeros((3, disc.n_pres)))
    ref = golden["sv2_rhs" + name]
    loads, bvals = golden["sv2_loads_" + fam], golden["sv2_bvals_" + fam]
    # the seam tiles ONE member's load / boundary values over the ensemble (`stepper.py:272-277`); the
    # fluctuation term uses the whole state, so each member's column matches the reference block
    for j in range(3):
        col = P.assemble_member_rhs(kind, j, state, loads[j], bvals[j], cfg, disc)
        assert np.max(np.abs(col - ref[:, j])) <= 1e-12 * np.abs(ref).max()


def test_member_rhs_rejects_bad_load_shape(tiny_disc):
    config = simple_config()
    with pytest.raises(ValueError):
        P.assemble_member_rhs(StepKind.V_STEP, 0, zero_state(config, tiny_disc), np.zeros(3),
                              np.zeros(tiny_disc.bdofs.size), config, tiny_disc)


# ----------------------------------------------------------------------------------------------
# factorize / solve / solve_block
# ----------------------------------------------------------------------------------------------

def test_factorization_matches_dense_lu_and_block_equals_singles(golden, rng):
    disc = Discretization.from_mesh(barycentric_refine(build_structured_square(2)))
    z = golden["sv2_pert_w"]
    system = P.assemble_shared_lhs(StepKind.V_STEP, z.mean(0), z - z.mean(0), sv2_config(), disc)
    fact = system.factorization
    assert fact.shape == system.matrix.shape and fact.symbolic is disc.saddle_symbolic
    b = rng.standard_normal((disc.n_total, 4))
    x = fact.solve_block(b)
    dense = np.linalg.solve(system.matrix.toarray(), b)
    assert np.max(np.abs(x - dense)) <= 1e-10 * np.abs(dense).max()
    assert LA.relative_residual(system.matrix, x, b) <= 1e-11
    singles = np.stack([fact.solve(b[:, k]) for k in range(4)], axis=1)
    assert np.max(np.abs(singles - x)) <= 1e-13 * np.abs(x).max()
    # refactorising the same matrix through the public factorize() gives the same solution
    f2 = P.factorize(system.matrix, symbolic=disc.saddle_symbolic)
    x2 = f2.solve_block(b)
    assert np.max(np.abs(x2 - x)) <= 1e-12 * np.abs(x).max()


def test_factorization_argument_errors(golden, rng):
    disc = Discretization.from_mesh(barycentric_refine(build_structured_square(2)))
    z = golden["sv2_pert_w"]
    system = P.assemble_shared_lhs(StepKind.V_STEP, z.mean(0), z - z.mean(0), sv2_config(), disc)
    with pytest.raises(ValueError):
        system.factorization.solve(np.zeros(disc.n_total + 1))
    with pytest.raises(ValueError):
        system.factorization.solve_block(np.zeros((disc.n_total + 1, 2)))
    with pytest.raises(ValueError):
        P.factorize(sp.identity(5, format="csr"), symbolic=disc.saddle_symbolic)
    with pytest.raises(ValueError):
        P.factorize(system.matrix[:, :-1])


# ----------------------------------------------------------------------------------------------
# run() and the stability bound
# ----------------------------------------------------------------------------------------------

def test_run_single_step_when_t_end_equals_dt(tiny_disc):
    config = simple_config(dt=0.05, t_end=0.05)
    prob = P.Problem(tiny_disc, np.zeros((1, tiny_disc.n_vel)), np.zeros((1, tiny_disc.n_vel)), ZeroForcing(),
                     ZeroBoundary())
    report, state, _ = P.run(config, prob)
    assert report.num_steps == 1 and state.step == 1


def test_run_bad_step_ratio_rejected(tiny_disc):
    config = simple_config(dt=0.2, t_end=0.05)
    prob = P.Problem(tiny_disc, np.zeros((1, tiny_disc.n_vel)), np.zeros((1, tiny_disc.n_vel)), ZeroForcing(),
                     ZeroBoundary())
    with pytest.raises(ValueError):
        P.run(config, prob)


def test_decay_run_properties_and_stability_bound(tiny_disc):
    config = EnsembleConfig(members=tuple(MemberParams(0.01 + 0.0002 * (j - 10) / 10, 0.1) for j in range(20)),
                            coupling=1.0, mu=1.0, dt=0.05, t_end=0.25, perturbation=0.01)
    v0, w0 = paper_mms_initial_fields(tiny_disc, config)
    seen = []
    report, state, snaps = P.run(config, P.Problem(tiny_disc, v0, w0, ZeroForcing(), ZeroBoundary()),
                                 observer=lambda n, t, st: seen.append(n), snapshot_steps=(0, 3))
    assert set(snaps) == {0, 3} and snaps[3].step == 3
    e = report.energy
    assert np.all(e[1:] <= e[:-1] + 1e-12 * e[0])
    assert report.div_v[1:].max() <= 1e-10 and report.div_w[1:].max() <= 1e-10
    assert len(report.times) == len(report.residuals) == len(report.wall_clock) == 6
    assert seen == list(range(6))
    assert P.verify_stability_bound(report, config, tiny_disc).holds


def test_returned_state_is_write_protected(tiny_disc):
    """Advance's host views are read-only (`ensemble.py:183-190`: states are immutable), so an
    in-place edit cannot be silently ignored by the next device-resident step."""
    config = simple_config(dt=0.05, t_end=0.1)
    st = zero_state(config, tiny_disc)
    new, _ = P.advance(st, config, tiny_disc, ZeroForcing(), ZeroBoundary())
    for f in (new.v, new.w, new.q, new.r):
        assert not f.flags.writeable
        with pytest.raises(ValueError):
            f[0, 0] = 1.0
    edited = EnsembleState(v=np.array(new.v) + 1.0, w=np.array(new.w), q=np.array(new.q), r=np.array(new.r), step=1,
                           time=new.time)
    nxt, _ = P.advance(edited, config, tiny_disc, ZeroForcing(), ZeroBoundary())
    assert np.abs(nxt.v).max() > 0.0     # the edited (host) state was uploaded, not the resident one


def test_engine_caches_are_bounded():
    """Fresh problem objects on one engine: device data and step graphs of the least recently used
    objects are released (engine.MAX_PROBLEM_OBJECTS), engines per discretisation are bounded."""
    from paper_2108_05110_b200 import engine as EN
    from paper_2108_05110_b200 import stepper as ST
    from paper_2108_05110_b200.problems import BaselineMms, _BoundaryView, _ForcingView
    disc, cfg, prob = P.build_case("C1", J=4, steps=3)
    for k in range(EN.MAX_PROBLEM_OBJECTS + 4):
        mms = BaselineMms(nu0=0.01 + 1e-4 * k)
        P.run(cfg, P.Problem(disc, prob.initial_v, prob.initial_w, _ForcingView(mms), _BoundaryView(mms)))
    eng = ST.get_engine(disc, cfg)
    assert len(eng._lru) <= EN.MAX_PROBLEM_OBJECTS
    assert len(eng._gdata_cache) <= 2 * EN.MAX_PROBLEM_OBJECTS
    assert len(eng._graphs) <= 2 * EN.MAX_PROBLEM_OBJECTS
    for k in range(ST.MAX_ENGINES + 2):
        c2 = P.EnsembleConfig(members=cfg.members, coupling=1.0, mu=1.0, dt=cfg.dt * (1 + 0.1 * k), t_end=cfg.dt * 2)
        P.run(c2, prob)
    assert sum(1 for key in disc._cache if isinstance(key, tuple) and key[0] == "b200-engine") <= ST.MAX_ENGINES
