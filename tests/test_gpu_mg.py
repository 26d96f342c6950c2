"""PrecondSpec(inner="mg") on the device (csrc/mg.cu)
against its oracle restatement (oracle/mg.py): the V-cycle map to rounding,
the block preconditioner, and whole steps that reach the Jacobi-4 solution."""

import numpy as np
import pytest

import paper_2101_01776_b200 as pk
from paper_2101_01776_b200.problems import GridProblem, fourier_u0
from oracle.mg import VCycle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,shape,kw", [("nldiff", (64, 64), {}),
                                           ("burgers", (128, 64), dict(nu=1e-2)),
                                           ("rad", (64, 96), dict(nu=1e-2, c=0.5, lam=-1.0))])
def test_vcycle_matches_oracle(kind, shape, kw):
    prob = GridProblem(kind, shape, **kw)
    U = fourier_u0(shape, 1, 8, 0.5, 3)
    f = pk.OperatorField.linearize(prob, U[None, :])
    a = f.a.cpu().numpy()
    r = np.random.default_rng(7).standard_normal(prob.dim)
    for alpha, dt in ((3.0, 1e-3), (4.5, 5e-2)):
        x = pk.ShiftedSolver(alpha, None, f, dt, inner="mg").solve(r)
        ref = VCycle(kind, shape, (1.0, 1.0), a, f.sigma, alpha, dt, nu=kw.get("nu", 0.0),
                     c=kw.get("c", 0.0)).solve(r)
        assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref), (kind, alpha, dt)


def test_block_gmres_with_mg_converges_fast():
    """The 2x2 block of configs[2] stiffness on 256^2: a handful of MG-
    preconditioned iterations where Jacobi-4 needs hundreds."""
    n = 256
    prob = GridProblem("nldiff", (n, n))
    U = fourier_u0((n, n), 1, 16, 0.1, 0)
    f = pk.OperatorField.linearize(prob, U[None, :])
    sysb = pk.Block2x2System(3.0, 1.7320508075688772, 0.4641016151377546, None, f, f, 0.05)
    rhs = np.random.default_rng(0).standard_normal(2 * n * n)
    _, rep_mg = pk.block_gmres(sysb, rhs, pk.PrecondSpec(inner="mg"), rtol=1e-8, maxit=5000)
    _, rep_j = pk.block_gmres(sysb, rhs, pk.PrecondSpec(inner=4), rtol=1e-8, maxit=5000)
    assert rep_mg.converged and rep_j.converged
    assert rep_mg.iterations * 8 <= rep_j.iterations, (rep_mg.iterations, rep_j.iterations)


def test_integrate_with_mg_reaches_the_jacobi_solution():
    """configs[2]-type nonlinear diffusion, Gauss(2): the MG inner mode
    converges Newton to the same stage solution (1e-8 relative) with far
    fewer Krylov iterations."""
    spec = pk.baseline_config(2, n=128, nsteps=2)
    tab = pk.make_tableau("gauss", 2)
    sv = spec.solver

    def run(inner):
        cfg = pk.SolverConfig(variant=3, krylov_maxit=sv["krylov_maxit"], restart=200,
                              newton_rtol=1e-10, krylov_rtol=1e-8,
                              precond=pk.PrecondSpec(inner=inner))
        return pk.integrate(spec.problem, spec.u0(), 0.0, 2 * spec.dt, spec.dt, tab, cfg)

    rm, rj = run("mg"), run(4)
    rel = np.linalg.norm(rm.u_final - rj.u_final) / np.linalg.norm(rj.u_final)
    assert rel <= 1e-8, rel
    assert rm.total("krylov_iterations") * 2 <= rj.total("krylov_iterations")
