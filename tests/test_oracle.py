"""Pin the CPU oracle against the reference: golden fixtures produced by the
real irkit (tests/golden/make_golden.py) and the reference's own
known-answer tests (restated from pkg/tests/test_irk_core.py,
test_nonlinear.py, test_sparsela.py)."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import irk
from oracle import tableau as otab
from oracle.problems import build_problem

from _golden import (case_names, grid_problem, is_survey_size, load_case, load_transformed,
                     oracle_config)

FAST_CASES = [c for c in case_names()
              if not c.startswith("cfg2_radau") and not is_survey_size(c)]


def run_oracle(meta):
    prob = grid_problem(meta)
    pd = build_problem(prob.kind, prob.shape, **prob.oracle_params())
    sysr = irk.OdeSystem(pd.dim, pd.rhs, pd.linearize_csr)
    cfg = oracle_config(meta["solver"])
    if meta["family"].startswith("sdirk"):  # the reference's _dirk_step route
        tab = otab.dirk_tableau(meta["family"])
        u = np.array(meta["u0"], dtype=float)
        states, stats = [u.copy()], []
        for j in range(meta["nsteps"]):
            u, _, st = irk.dirk_step(sysr, u, j * meta["dt"], meta["dt"], tab, cfg)
            states.append(u.copy())
            stats.append(st)
        return states, stats
    prep = otab.prepare(meta["family"], meta["s"])
    return irk.integrate(sysr, meta["u0"], 0.0, meta["nsteps"] * meta["dt"], meta["dt"], prep, cfg)


@pytest.mark.parametrize("name", FAST_CASES)
def test_oracle_matches_reference_run(name):
    meta = load_case(name)
    states, stats = run_oracle(meta)
    ref = meta["u_final"]
    rel = np.linalg.norm(states[-1] - ref) / np.linalg.norm(ref)
    assert rel <= 1e-13, rel
    for got, want in zip(stats, meta["steps"]):
        assert got.newton_iterations == want["newton_iterations"]
        assert got.krylov_iterations == want["krylov_iterations"]
        assert got.precond_applications == want["precond_applications"]
        assert got.jacobian_assemblies == want["jacobian_assemblies"]
        assert got.block_iterations == want["block_iterations"]
        hist = want["residual_history"]
        np.testing.assert_allclose(got.residual_history, hist, rtol=1e-9,
                                   atol=1e-11 * max(hist))


def test_oracle_transformed_matches_reference():
    prob_lin = build_problem("rad", (24,), nu=0.01, c=1.0, lengths=(1.0,))
    lmat = prob_lin.linearize_csr(np.zeros(24), 0.0)
    for case in load_transformed():
        prep = otab.prepare(case["family"], case["s"])
        rng = np.random.default_rng(case["seed"])
        rhs = rng.standard_normal((case["s"], 24))
        vj = irk.build_variant_jacobian(prep, [lmat] * case["s"], case["variant"])
        k, stats = irk.solve_transformed(prep, vj, case["dt"], rhs, "star", case["inner"],
                                         1e-12, 400, 200)
        assert [[o, r.iterations] for o, r in stats.reports] == case["reports"]
        assert np.max(np.abs(k - case["k"])) <= 1e-12


# ----------------------------------------- reference known-answer tests


def _scalar(v):
    return sp.csr_matrix(np.array([[v]]))


def test_block2x2_unit_vector_action():
    # pkg/tests/test_irk_core.py:52-55
    y = irk.block2x2_apply(3.0, np.sqrt(3.0), 1.0, _scalar(0.0), _scalar(0.0), 1.0,
                           np.array([1.0, 0.0]))
    assert np.allclose(y, [3.0, -3.0])


def test_block2x2_scalar_action():
    # pkg/tests/test_irk_core.py:57-60
    y = irk.block2x2_apply(3.0, np.sqrt(3.0), 1.0, _scalar(-1.0), _scalar(-2.0), 1.0,
                           np.array([1.0, 1.0]))
    assert np.allclose(y, [5.0, 2.0])


def test_precond_scalar_oracle():
    # pkg/tests/test_irk_core.py:71-73 (exact inner solves)
    pre = irk.block2x2_precond(3.0, np.sqrt(3.0), 1.0, _scalar(0.0), _scalar(0.0), 1.0,
                               "star", "exact")
    assert np.allclose(pre(np.array([1.0, 0.0])), [1.0 / 3.0, 0.25])


def test_backward_euler_single_solve():
    # pkg/tests/test_irk_core.py:130-139
    prep = otab.prepare("radau_iia", 1)
    lmat = _scalar(-2.0)
    vj = irk.build_variant_jacobian(prep, [lmat], 0)
    k, stats = irk.solve_transformed(prep, vj, 0.1, np.array([[1.0]]), "star", "exact", 1e-13)
    assert k[0, 0] == pytest.approx(1.0 / 1.2, abs=1e-12)
    assert stats.krylov_iterations == 1


def test_gmres_identity_and_counting():
    # pkg/tests/test_sparsela.py:56-60, 92-99
    b = np.arange(1.0, 6.0)
    x, rep = irk.gmres(lambda v: v, b, 5, rtol=1e-12)
    assert rep.converged and rep.iterations == 1 and np.allclose(x, b)
    rng = np.random.default_rng(4)
    a = rng.standard_normal((12, 12)) + 4 * np.eye(12)
    inv = np.linalg.inv(a)
    x, rep = irk.gmres(lambda v: a @ v, rng.standard_normal(12), 12, lambda v: inv @ v, 2,
                       rtol=1e-12)
    assert rep.converged and rep.iterations == 1 and rep.precond_applications == 2


def test_gmres_maxit_and_zero_rhs():
    # pkg/tests/test_sparsela.py:101-111
    rng = np.random.default_rng(5)
    a = rng.standard_normal((30, 30)) + 6 * np.eye(30)
    _, rep = irk.gmres(lambda v: a @ v, rng.standard_normal(30), 30, rtol=1e-15, maxit=3,
                       restart=2)
    assert not rep.converged and rep.iterations == 3
    x, rep = irk.gmres(lambda v: v, np.zeros(4), 4)
    assert rep.converged and rep.iterations == 0 and np.all(x == 0.0)
    with pytest.raises(ValueError):
        irk.gmres(lambda v: v, np.ones(3), 3, rtol=2.0)


def test_stage_residual_hand_arithmetic():
    # pkg/tests/test_nonlinear.py:67-78
    prep = otab.prepare("gauss", 2)
    mat = _scalar(-2.0)
    sysr = irk.OdeSystem(1, lambda u, t: mat @ u, lambda u, t: mat)
    res = irk.stage_residual(sysr, np.array([1.0]), np.ones((2, 1)), 0.0, 0.5, prep.tableau)
    r3 = np.sqrt(3.0)
    assert res[0, 0] == pytest.approx(-3.5 + r3 / 6.0, abs=1e-14)
    assert res[1, 0] == pytest.approx(-3.5 - r3 / 6.0, abs=1e-14)


def test_variant3_keys_and_lumping():
    # pkg/tests/test_nonlinear.py:101-135
    prep = otab.prepare("gauss", 4)
    dw, ow = irk.variant_weights(prep, 3)
    for i in range(4):
        for j in range(i + 1, 4):
            assert (i, j) in ow
    for blk in prep.blocks:
        if blk.size == 2:
            assert (blk.offset + 1, blk.offset) in ow
    picked = sorted(int(np.argmax(np.abs(prep.d[i, i]))) for i in range(4))
    assert picked == [0, 1, 2, 3]


# --------------------------------------------------------------- DAE path

from _golden import load_dae_case  # noqa: E402


@pytest.mark.parametrize("name", [c for c in case_names(dae=True)
                                  if "n128" not in c and not is_survey_size(c)])
def test_oracle_dae_matches_reference_run(name):
    from oracle import dae as odae
    from oracle.problems import DaeProblemDef

    meta = load_dae_case(name)
    pd = DaeProblemDef(tuple(meta["shape"]), meta["nu"])
    sysr = odae.DaeSystem(pd.dim, pd.dim, pd.rhs, pd.constraint, pd.blocks_csr)
    prep = otab.prepare(meta["family"], meta["s"])
    us, ws, sts = odae.dae_integrate(sysr, meta["u0"], meta["w0"], 0.0,
                                     meta["nsteps"] * meta["dt"], meta["dt"], prep,
                                     oracle_config(meta["solver"]))
    assert np.linalg.norm(us[-1] - meta["u_final"]) <= 1e-13 * np.linalg.norm(meta["u_final"])
    assert np.linalg.norm(ws[-1] - meta["w_final"]) <= 1e-12 * np.linalg.norm(meta["w_final"])
    for got, want in zip(sts, meta["steps"]):
        assert got.newton_iterations == want["newton_iterations"]
        assert got.krylov_iterations == want["krylov_iterations"]
        assert got.differential_solves == want["differential_solves"]
        assert got.constraint_solves == want["constraint_solves"]
        assert got.block_iterations == want["block_iterations"]
        assert got.constraint_residual <= 1e-12


def test_vorticity_initial_state_is_consistent():
    from oracle.problems import DaeProblemDef
    from paper_2101_01776_b200.problems import VorticityProblem, vorticity_initial_state

    for n in (16, 128, 256):
        prob = VorticityProblem((n, n))
        w0, p0 = vorticity_initial_state(prob)
        g = DaeProblemDef(prob.shape, prob.nu).constraint(w0, p0, 0.0)
        assert np.linalg.norm(g) <= 1e-10 and p0[0] == 0.0


def test_arakawa_matrix_matches_direct_form():
    from oracle.problems import arakawa_jacobian, arakawa_jacobian_matrix

    rng = np.random.default_rng(0)
    nx, ny = 9, 7
    psi, w = rng.standard_normal(nx * ny), rng.standard_normal(nx * ny)
    m = arakawa_jacobian_matrix(psi, nx, ny, 1 / nx, 1 / ny)
    np.testing.assert_allclose(m @ w, arakawa_jacobian(psi, w, nx, ny, 1 / nx, 1 / ny),
                               atol=1e-10)
    # Arakawa's form conserves energy and enstrophy: sum psi J = sum w J = 0
    j = arakawa_jacobian(psi, w, nx, ny, 1 / nx, 1 / ny)
    assert abs(np.dot(psi, j)) < 1e-9 * np.abs(j).sum() and abs(np.dot(w, j)) < 1e-9 * np.abs(j).sum()


def test_oracle_breakdown_path_matches_reference():
    """The Arnoldi-breakdown error (src/sparsela.py:229-233, 268-271): a
    pointwise operator makes the Jacobi-preconditioned operator a multiple
    of the identity; below the rounding-level true residual both the oracle
    and (when importable) irkit itself raise KrylovBreakdownError, and at a
    reachable rtol both converge in one iteration to the same x."""
    import os
    import sys

    pd = build_problem("rad", (64, 48), nu=0.0, c=0.0, lam=-0.5, mu=0.7,
                       lengths=(1.0, 1.0))
    rng = np.random.default_rng(9)
    U = rng.standard_normal(pd.dim)
    lmat = pd.linearize_csr(U, 0.0)
    rhs = rng.standard_normal(pd.dim)
    eta, dt = 2.0, 0.1
    solver = irk.ShiftedSolver(eta, lmat, dt, 4)
    op = (lambda v: eta * v - dt * (lmat @ v))
    with pytest.raises(irk.KrylovBreakdownError):
        irk.gmres(op, rhs, pd.dim, solver.solve, 1, 1e-17, 50, 20)
    x, rep = irk.gmres(op, rhs, pd.dim, solver.solve, 1, 1e-10, 50, 20)
    assert rep.converged and rep.iterations == 1
    for path in ("/root/reference/pkg/src",
                 os.path.join(os.path.dirname(os.path.dirname(__file__)), "baseline", "_ref")):
        if os.path.isdir(path) and path not in sys.path:
            sys.path.append(path)
    irkit = pytest.importorskip("irkit")
    from irkit.errors import KrylovBreakdownError
    from irkit.irk_core import ShiftedSolver, shifted_matrix
    from irkit.sparsela import LinearOperator, SparseMatrix, gmres

    L = SparseMatrix(lmat, bandwidth=64)
    pre = LinearOperator(pd.dim, ShiftedSolver(eta, None, L, dt, 4).solve, 1)
    A = LinearOperator(pd.dim, shifted_matrix(eta, None, L, dt).matvec)
    with pytest.raises(KrylovBreakdownError):
        gmres(A, rhs, right_precond=pre, rtol=1e-17, maxit=50, restart=20)
    xr, repr_ = gmres(A, rhs, right_precond=pre, rtol=1e-10, maxit=50, restart=20)
    assert repr_.iterations == 1 and np.max(np.abs(xr - x)) <= 1e-14 * np.max(np.abs(x))
    assert irkit is not None
