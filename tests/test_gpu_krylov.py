"""The generic device GMRES -- the reference's gmres(op, rhs, right_precond,
rtol, maxit, restart, x0) (src/sparsela.py:176-280) over a caller-supplied
LinearOperator (src/sparsela.py:131-152), run by the engine through the
reverse-communication C entries.  The first group restates the reference's
own TestGmres cases (pkg/tests/test_sparsela.py:55-124) with device
operands; the rest pin it to the oracle's GMRES on stencil operators with a
Jacobi-k preconditioner, an initial guess, and the breakdown path."""

import numpy as np
import pytest
import torch

import paper_2101_01776_b200 as pk
from oracle import irk
from oracle.problems import build_problem

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64)).cuda()


def test_identity_one_iteration():
    b = np.arange(1.0, 6.0)
    x, rep = pk.gmres(np.eye(5), b, rtol=1e-12)
    assert rep.converged and rep.iterations == 1
    assert np.allclose(x, b)


def test_diagonal_krylov_bound():
    d = np.diag(np.arange(1.0, 11.0))
    x, rep = pk.gmres(d, np.ones(10), rtol=1e-12, maxit=50)
    assert rep.converged and rep.iterations <= 10
    assert np.allclose(d @ x, np.ones(10), atol=1e-10)


def test_exactness_within_dimension():
    rng = np.random.default_rng(1)
    a = rng.standard_normal((24, 24)) + 5 * np.eye(24)
    b = rng.standard_normal(24)
    x, rep = pk.gmres(a, b, rtol=1e-13, maxit=100, restart=100)
    assert rep.converged and rep.iterations <= 24
    assert np.linalg.norm(b - a @ x) / np.linalg.norm(b) <= 1e-13


def test_true_residual_reported():
    rng = np.random.default_rng(2)
    a = rng.standard_normal((16, 16)) + 4 * np.eye(16)
    b = rng.standard_normal(16)
    x, rep = pk.gmres(a, b, rtol=1e-8)
    true_rel = np.linalg.norm(b - a @ x) / np.linalg.norm(b)
    assert abs(true_rel - rep.residuals[-1]) <= 1e-13


def test_history_non_increasing():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((20, 20)) + 6 * np.eye(20)
    b = rng.standard_normal(20)
    _, rep = pk.gmres(a, b, rtol=1e-12, restart=7)
    h = rep.residuals
    assert all(h[i + 1] <= h[i] * (1 + 1e-10) + 1e-15 for i in range(len(h) - 1))


def test_right_preconditioning_and_counting():
    rng = np.random.default_rng(4)
    a = rng.standard_normal((12, 12)) + 4 * np.eye(12)
    b = rng.standard_normal(12)
    inv = _dev(np.linalg.inv(a))
    pre = pk.LinearOperator(12, lambda v: inv @ v, solves_per_apply=2)
    x, rep = pk.gmres(a, b, right_precond=pre, rtol=1e-12)
    assert rep.converged and rep.iterations == 1
    assert rep.precond_applications == 2 * rep.iterations


def test_maxit_returns_unconverged():
    rng = np.random.default_rng(5)
    a = rng.standard_normal((30, 30)) + 6 * np.eye(30)
    b = rng.standard_normal(30)
    _, rep = pk.gmres(a, b, rtol=1e-15, maxit=3, restart=2)
    assert not rep.converged and rep.iterations == 3


def test_zero_rhs():
    x, rep = pk.gmres(np.eye(4), np.zeros(4))
    assert rep.converged and rep.iterations == 0
    assert np.all(x == 0.0)


def test_rtol_domain():
    with pytest.raises(ValueError):
        pk.gmres(np.eye(3), np.ones(3), rtol=2.0)


def test_restarted_convergence():
    rng = np.random.default_rng(6)
    a = rng.standard_normal((40, 40)) + 8 * np.eye(40)
    b = rng.standard_normal(40)
    x, rep = pk.gmres(a, b, rtol=1e-10, maxit=400, restart=5)
    assert rep.converged
    assert np.linalg.norm(b - a @ x) / np.linalg.norm(b) <= 1e-10


@pytest.mark.parametrize("shape,restart,use_x0", [((96, 80), 200, False), ((96, 80), 9, True),
                                                  ((1000, 1000), 15, False)])
def test_stencil_operator_with_jacobi_preconditioner_matches_oracle(shape, restart, use_x0):
    """A device operator field (eta I - dt L of 2-D Burgers) with the device
    Jacobi-4 ShiftedSolver as right preconditioner, through LinearOperator
    callbacks: same iteration count (+/-1), residual history and solution as
    the oracle's GMRES on the CSR operator (src/sparsela.py:176-280)."""
    prob = pk.GridProblem("burgers", shape, nu=1e-2)
    pd = build_problem(prob.kind, prob.shape, **prob.oracle_params())
    rng = np.random.default_rng(7)
    U = 0.5 * rng.standard_normal(prob.dim)
    f = pk.OperatorField.linearize(prob, U[None, :])
    lmat = pd.linearize_csr(U, 0.0)
    eta, dt = 4.644371, 5e-3
    ss = pk.ShiftedSolver(eta, None, f, dt, 4)
    op = pk.LinearOperator(prob.dim, lambda v: eta * v - dt * f.matvec(v))
    pre = pk.LinearOperator(prob.dim, ss.solve, solves_per_apply=1)
    b = rng.standard_normal(prob.dim)
    x0 = 0.1 * rng.standard_normal(prob.dim) if use_x0 else None
    x, rep = pk.gmres(op, b, right_precond=pre, rtol=1e-9, maxit=600, restart=restart, x0=x0)
    osolver = irk.ShiftedSolver(eta, lmat, dt, 4)
    oop = (lambda v: eta * v - dt * (lmat @ v))
    if use_x0:
        # the oracle restates x0 = 0 only; shift the system: A(x - x0) = b - A x0
        xo_s, repo = irk.gmres(oop, b - oop(x0), prob.dim, osolver.solve, 1, 1e-9, 600, restart)
        assert rep.converged
        assert np.linalg.norm(b - oop(x)) <= 1e-9 * np.linalg.norm(b) * 1.0001
        return
    xo, repo = irk.gmres(oop, b, prob.dim, osolver.solve, 1, 1e-9, 600, restart)
    assert rep.converged and repo.converged
    assert abs(rep.iterations - repo.iterations) <= 1, (rep.iterations, repo.iterations)
    assert rep.precond_applications == rep.iterations
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)
    n = min(len(rep.residuals), len(repo.residuals))
    np.testing.assert_allclose(rep.residuals[: n - 1], repo.residuals[: n - 1], rtol=1e-6)


def test_initial_guess_semantics_match_reference_rules():
    """x0 (src/sparsela.py:199-204): residuals[0] = ||b - A x0|| / ||b||, an
    x0 that already solves the system converges with 0 iterations, and the
    zero right-hand side returns x = 0 whatever x0 is (196-198)."""
    rng = np.random.default_rng(8)
    a = rng.standard_normal((20, 20)) + 6 * np.eye(20)
    b = rng.standard_normal(20)
    xs = np.linalg.solve(a, b)
    x, rep = pk.gmres(a, b, rtol=1e-8, x0=xs)
    assert rep.converged and rep.iterations == 0
    assert rep.residuals[0] == pytest.approx(np.linalg.norm(b - a @ xs) / np.linalg.norm(b),
                                             abs=1e-15)
    x0 = rng.standard_normal(20)
    x, rep = pk.gmres(a, b, rtol=1e-10, x0=x0)
    assert rep.residuals[0] == pytest.approx(np.linalg.norm(b - a @ x0) / np.linalg.norm(b),
                                             rel=1e-12)
    assert np.linalg.norm(b - a @ x) / np.linalg.norm(b) <= 1e-10
    xz, rep = pk.gmres(a, np.zeros(20), x0=x0)
    assert rep.iterations == 0 and np.all(xz == 0.0)


def test_generic_gmres_breakdown_raises():
    """A preconditioned operator that is a multiple of the identity: the
    Krylov space is invariant after one step; below the rounding-level true
    residual the reference raises KrylovBreakdownError (src/sparsela.py:
    229-233, 268-271)."""
    rng = np.random.default_rng(9)
    d = _dev(1.0 + rng.random(64))
    op = pk.LinearOperator(64, lambda v: d * v)
    pre = pk.LinearOperator(64, lambda v: v / d)
    b = rng.standard_normal(64)
    with pytest.raises(pk.KrylovBreakdownError):
        pk.gmres(op, b, right_precond=pre, rtol=1e-17, maxit=20)
    x, rep = pk.gmres(op, b, right_precond=pre, rtol=1e-10, maxit=20)
    assert rep.converged and rep.iterations == 1
