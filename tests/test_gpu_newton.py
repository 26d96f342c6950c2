"""Device tests of the Newton-level entry points the golden runs do not
reach on their own: the public ``newton_like_step`` (irkg_newton_step), the
simplified-Newton ``jacobian_refresh="frozen"`` branch, and the Arnoldi
breakdown error path -- each against the CPU oracle restatement of the
reference and the reference's own tests for them.
"""

import numpy as np
import pytest

import paper_2101_01776_b200 as pk
from oracle import irk
from oracle import tableau as otab
from oracle.problems import build_problem
from paper_2101_01776_b200.problems import GridProblem, fourier_u0

pytestmark = pytest.mark.gpu


def _oracle(prob):
    pd = build_problem(prob.kind, prob.shape, **prob.oracle_params())
    return pd, irk.OdeSystem(pd.dim, pd.rhs, pd.linearize_csr)


def _cfgs(**kw):
    inner = kw.pop("inner", 4)
    return (pk.SolverConfig(precond=pk.PrecondSpec(inner=inner), **kw),
            irk.Config(inner=inner, **kw))


@pytest.mark.parametrize("family,s", [("gauss", 3), ("radau_iia", 2)])
def test_newton_like_step_public_entry_matches_oracle(family, s):
    """newton_like_step (src/nonlinear.py:186-236) through irkg_newton_step:
    same stage vectors (1e-10), same Newton count, Krylov count within +/-1,
    per-block lists within +/-1, and the reference's value semantics (st.k
    rebound to a new array, the caller's array untouched)."""
    prob = GridProblem("burgers", (64, 64), nu=1e-2)
    u0 = fourier_u0(prob.shape, 1, 6, 0.5, seed=4)
    prep = pk.prepare_stages(pk.make_tableau(family, s))
    cfg, ocfg = _cfgs(krylov_maxit=2000)
    k_in = np.zeros((s, prob.dim))
    st = pk.StageState(k=k_in, u=u0, t=0.0, dt=2e-3)
    st2, stats = pk.newton_like_step(prob, st, prep, cfg)
    assert st2 is st and st.k is not k_in and not k_in.any()
    _, osys = _oracle(prob)
    ko, ostats = irk.newton_like_step(osys, u0, np.zeros((s, prob.dim)), 0.0, 2e-3,
                                      otab.prepare(family, s), ocfg)
    assert np.linalg.norm(st.k - ko) <= 1e-10 * np.linalg.norm(ko)
    assert stats.newton_iterations == ostats.newton_iterations
    assert abs(stats.krylov_iterations - ostats.krylov_iterations) <= 1
    assert stats.jacobian_assemblies == ostats.jacobian_assemblies
    for off, its in ostats.block_iterations.items():
        got = stats.block_iterations[off]
        assert len(got) == len(its) and all(abs(a - b) <= 1 for a, b in zip(got, its))
    np.testing.assert_allclose(stats.residual_history, ostats.residual_history, rtol=1e-6,
                               atol=1e-9 * ostats.residual_history[0])


def test_newton_like_step_continues_from_given_stages():
    """A warm start: K from a first Newton iteration fed back in converges
    to the same stages as the cold start (the loop is a fixed-point map)."""
    prob = GridProblem("nldiff", (48, 48))
    u0 = fourier_u0(prob.shape, 1, 4, 0.1, seed=1)
    prep = pk.prepare_stages(pk.make_tableau("gauss", 2))
    cfg = pk.SolverConfig(newton_rtol=1e-11, krylov_rtol=1e-11, krylov_maxit=4000,
                          precond=pk.PrecondSpec(inner=4))
    st, full = pk.newton_like_step(prob, pk.StageState(np.zeros((2, prob.dim)), u0, 0.0, 1e-3),
                                   prep, cfg)
    one = pk.SolverConfig(newton_rtol=1e-11, krylov_rtol=1e-11, krylov_maxit=4000,
                          newton_maxit=1, precond=pk.PrecondSpec(inner=4))
    st1 = pk.StageState(np.zeros((2, prob.dim)), u0, 0.0, 1e-3)
    with pytest.raises(pk.StepFailureError) as err:
        pk.newton_like_step(prob, st1, prep, one)
    assert err.value.stats.newton_iterations == 1
    k1 = pk.stage_residual(prob, st1, prep.tableau)  # residual evaluable at the rebound k
    assert np.isfinite(k1).all()
    _, osys = _oracle(prob)
    ko1, _ = irk.newton_like_step(osys, u0, np.zeros((2, prob.dim)), 0.0, 1e-3,
                                  otab.prepare("gauss", 2),
                                  irk.Config(newton_rtol=1e-11, krylov_rtol=1e-11,
                                             krylov_maxit=4000, inner=4, newton_maxit=30))
    assert np.linalg.norm(st.k - ko1) <= 1e-10 * np.linalg.norm(ko1)


def test_frozen_equals_refreshed_on_linear_problem():
    """Mirrors pkg/tests/test_nonlinear.py:377-384 of the reference: on a
    linear problem the frozen (simplified-Newton) Jacobian is the refreshed
    one, so both give the same step to 1e-12."""
    prob = GridProblem("rad", (40,), nu=0.01, c=1.0)
    u0 = fourier_u0(prob.shape, 1, 3, 0.3, seed=2)
    tab = pk.make_tableau("gauss", 2)
    kw = dict(newton_rtol=1e-12, krylov_rtol=1e-13, krylov_maxit=2000)
    u_every, st_e = pk.step(prob, u0, 0.0, 0.05, tab, pk.SolverConfig(
        precond=pk.PrecondSpec(inner=4), **kw))
    u_frozen, st_f = pk.step(prob, u0, 0.0, 0.05, tab, pk.SolverConfig(
        precond=pk.PrecondSpec(inner=4), jacobian_refresh="frozen", **kw))
    assert np.max(np.abs(u_every - u_frozen)) <= 1e-12
    assert st_f.jacobian_assemblies == tab.s  # assembled once


@pytest.mark.parametrize("shape", [(64,), (48, 48)])
def test_frozen_saves_assemblies_on_burgers_and_matches_oracle(shape):
    """Mirrors pkg/tests/test_nonlinear.py:386-395 (fewer assemblies, same
    fixed point as the refreshed iteration) and pins the frozen branch
    (src/nonlinear.py:204-209) against the oracle: same stage solution, same
    Newton count, Krylov within +/-1."""
    prob = GridProblem("burgers", shape, nu=0.02)
    u0 = fourier_u0(prob.shape, 1, 4, 0.5, seed=6)
    tab = pk.make_tableau("radau_iia", 2)
    dt = 0.02 if len(shape) == 1 else 5e-3  # (at 0.1 the frozen iteration stalls, oracle too)
    kw = dict(newton_rtol=1e-9, krylov_rtol=1e-6, newton_maxit=60, krylov_maxit=4000)
    cfg_e, _ = _cfgs(**kw)
    cfg_f, ocfg_f = _cfgs(jacobian_refresh="frozen", **kw)
    u1, st1 = pk.step(prob, u0, 0.0, dt, tab, cfg_e)
    u2, st2 = pk.step(prob, u0, 0.0, dt, tab, cfg_f)
    assert st2.jacobian_assemblies < st1.jacobian_assemblies
    assert st2.jacobian_assemblies == tab.s
    assert np.max(np.abs(u1 - u2)) <= 1e-7
    _, osys = _oracle(prob)
    uo, sto = irk.step(osys, u0, 0.0, dt, otab.prepare("radau_iia", 2), ocfg_f)
    assert np.linalg.norm(u2 - uo) <= 1e-10 * np.linalg.norm(uo)
    assert st2.newton_iterations == sto.newton_iterations
    assert abs(st2.krylov_iterations - sto.krylov_iterations) <= 1
    assert st2.jacobian_assemblies == sto.jacobian_assemblies


def test_krylov_breakdown_raises_like_the_reference():
    """The breakdown path (src/sparsela.py:229-233, 268-271): a pointwise
    operator (rad kind, nu = c = 0) makes the Jacobi-preconditioned
    operator a multiple of the identity, so the Krylov space is invariant
    after one step (h_{1,0} at rounding level -> breakdown).  With rtol
    below the rounding-level true residual the reference raises
    KrylovBreakdownError; so must the device, with the same message form.
    With a reachable rtol the same solve converges in one iteration."""
    prob = GridProblem("rad", (64, 48), nu=0.0, c=0.0, lam=-0.5, mu=0.7)
    pd, _ = _oracle(prob)
    rng = np.random.default_rng(9)
    U = rng.standard_normal((1, pd.dim))
    f = pk.OperatorField.linearize(prob, U)
    lmat = pd.linearize_csr(U[0], 0.0)
    rhs = rng.standard_normal(pd.dim)
    eta, dt = 2.0, 0.1
    solver = irk.ShiftedSolver(eta, lmat, dt, 4)
    apply_op = (lambda v: eta * v - dt * (lmat @ v))
    with pytest.raises(irk.KrylovBreakdownError):
        irk.gmres(apply_op, rhs, pd.dim, solver.solve, 1, 1e-17, 50, 20)
    with pytest.raises(pk.KrylovBreakdownError) as err:
        pk.block_gmres((eta, f, dt), rhs, pk.PrecondSpec(inner=4), 1e-17, 50, 20)
    assert "breakdown" in str(err.value)
    x, rep = pk.block_gmres((eta, f, dt), rhs, pk.PrecondSpec(inner=4), 1e-10, 50, 20)
    xo, repo = irk.gmres(apply_op, rhs, pd.dim, solver.solve, 1, 1e-10, 50, 20)
    assert rep.converged and rep.iterations == repo.iterations == 1
    assert np.linalg.norm(x - xo) <= 1e-12 * np.linalg.norm(xo)


def test_block_gmres_ring_slot_reuse_after_tail_tile():
    """a 2x2 block with 2N = 2,000,000 rows (not a multiple of
    any CGS tile height) is more than G * NST * TR rows, so every CTA
    reuses its ring slots -- including after the zero-padded tail tile,
    whose generic-proxy writes must be fenced before the slot's next TMA
    refill.  Same counts (+/-1) and solution as the oracle's GMRES."""
    prob = GridProblem("burgers", (1000, 1000), nu=1e-2)
    pd, _ = _oracle(prob)
    rng = np.random.default_rng(12)
    U = 0.5 * rng.standard_normal((2, pd.dim))
    f1 = pk.OperatorField.linearize(prob, U[:1])
    f2 = pk.OperatorField.linearize(prob, U[1:])
    l1 = pd.linearize_csr(U[0], 0.0)
    l2 = pd.linearize_csr(U[1], 0.0)
    eta, beta, phi, dt = 3.677815, 3.508762, -10.983731, 5e-4
    rhs = rng.standard_normal(2 * pd.dim)
    sysb = pk.Block2x2System(eta, beta, phi, None, f1, f2, dt)
    x, rep = pk.block_gmres(sysb, rhs, pk.PrecondSpec(inner=4), 1e-8, 200, 12)
    pre = irk.block2x2_precond(eta, beta, phi, l1, l2, dt, "star", 4)
    xo, repo = irk.gmres(lambda v: irk.block2x2_apply(eta, beta, phi, l1, l2, dt, v), rhs,
                         2 * pd.dim, pre, 2, 1e-8, 200, 12)
    assert rep.converged and repo.converged
    assert abs(rep.iterations - repo.iterations) <= 1, (rep.iterations, repo.iterations)
    assert np.linalg.norm(x - xo) <= 1e-7 * np.linalg.norm(xo)


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_linear_problem_takes_one_newton_iteration_and_variants_agree(variant):
    """Mirrors pkg/tests/test_nonlinear.py:138-157 of the reference: on a linear
    problem every linearization variant is the exact Jacobian -- one Newton
    iteration, and the same step for all variants (to the Krylov tolerance)."""
    prob = GridProblem("rad", (40, 24), nu=0.02, c=0.3, lam=-0.7, mu=0.0)
    u0 = pk.fourier_u0(prob.shape, 1, 3, 0.3, 5)
    tab = pk.make_tableau("gauss", 3)

    def run(v):
        cfg = pk.SolverConfig(variant=v, newton_rtol=1e-9, krylov_rtol=1e-12, krylov_maxit=2000,
                              precond=pk.PrecondSpec(inner=4))
        return pk.step(prob, u0, 0.0, 1e-2, tab, cfg)

    u, st = run(variant)
    u3, _ = run(3)
    assert st.newton_iterations == 1
    assert np.linalg.norm(u - u3) <= 1e-11 * np.linalg.norm(u3)


def test_dahlquist_closed_forms():
    """Mirrors pkg/tests/test_nonlinear.py:221-267: u' = lam u (rad kind with
    nu = c = mu = 0, every grid point an independent scalar problem).  Backward
    Euler (Radau IIA, s = 1) multiplies by 1 / (1 - dt lam), the implicit midpoint
    rule (Gauss, s = 1) by (1 + dt lam / 2) / (1 - dt lam / 2); ten steps give the
    tenth power; Gauss(2) is the (2, 2) Pade approximant of exp."""
    lam, dt = -1.0, 0.1
    prob = GridProblem("rad", (32,), nu=0.0, c=0.0, lam=lam, mu=0.0)
    u0 = np.linspace(0.5, 1.5, 32)
    cfg = pk.SolverConfig(newton_rtol=1e-12, krylov_rtol=1e-12, precond=pk.PrecondSpec(inner=1))
    z = dt * lam
    for family, s, per in [("radau_iia", 1, 1.0 / (1.0 - z)),
                           ("gauss", 1, (1.0 + z / 2) / (1.0 - z / 2)),
                           ("gauss", 2, (1 + z / 2 + z * z / 12) / (1 - z / 2 + z * z / 12))]:
        tab = pk.make_tableau(family, s)
        u1, st = pk.step(prob, u0, 0.0, dt, tab, cfg)
        assert np.max(np.abs(u1 - per * u0)) <= 1e-11, (family, s)
        res = pk.integrate(prob, u0, 0.0, 10 * dt, dt, tab, cfg)
        assert np.max(np.abs(res.u_final - per ** 10 * u0)) <= 1e-10, (family, s)
        assert len(res.step_stats) == 10
