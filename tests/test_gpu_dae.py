"""GPU parity of the index-1 DAE path (BASELINE configs[4], vorticity /
streamfunction, reordered mode) against golden runs of the reference's
``dae_integrate`` (src/dae.py:520-564) and the CPU oracle restatement."""

import numpy as np
import pytest

import paper_2101_01776_b200 as pk
from oracle import dae as odae
from oracle import irk
from oracle import tableau as otab
from oracle.problems import DaeProblemDef

from _golden import assert_counts_within_one, case_names, load_dae_case

pytestmark = pytest.mark.gpu


def _cfg(sv):
    return pk.SolverConfig(variant=sv.get("variant", 3), krylov_maxit=sv.get("krylov_maxit", 200),
                           restart=sv.get("restart", 200),
                           precond=pk.PrecondSpec(inner=sv.get("inner", 4)))


@pytest.mark.parametrize("name", case_names(dae=True))
def test_dae_integrate_matches_reference_golden(name):
    meta = load_dae_case(name)
    prob = pk.VorticityProblem(tuple(meta["shape"]), nu=meta["nu"])
    res = pk.dae_integrate(prob, meta["u0"], meta["w0"], 0.0, meta["nsteps"] * meta["dt"],
                           meta["dt"], pk.make_tableau(meta["family"], meta["s"]),
                           _cfg(meta["solver"]))
    ru = np.linalg.norm(res.u_final - meta["u_final"]) / np.linalg.norm(meta["u_final"])
    rw = np.linalg.norm(res.w_final - meta["w_final"]) / np.linalg.norm(meta["w_final"])
    assert ru <= 1e-10 and rw <= 1e-10, (ru, rw)
    assert_counts_within_one(res.step_stats, meta["steps"])
    for got, want in zip(res.step_stats, meta["steps"]):
        assert got.constraint_solves == want["constraint_solves"]
        assert got.differential_solves == 2 * got.krylov_iterations
        assert got.constraint_residual <= 1e-11


def test_dae_stage_residual_and_step_match_oracle():
    n = 40
    prob = pk.VorticityProblem((n, n), nu=1e-3)
    w0, p0 = pk.vorticity_initial_state(prob, seed=3)
    pd = DaeProblemDef(prob.shape, prob.nu)
    osys = odae.DaeSystem(pd.dim, pd.dim, pd.rhs, pd.constraint, pd.blocks_csr)
    tab = pk.make_tableau("gauss", 2)
    cfg = pk.SolverConfig(newton_rtol=1e-11, krylov_rtol=1e-10, krylov_maxit=2000,
                          precond=pk.PrecondSpec(inner=4))
    u1, w1, st = pk.dae_step(prob, w0, p0, 0.0, 2e-3, tab, cfg)
    ocfg = irk.Config(newton_rtol=1e-11, krylov_rtol=1e-10, krylov_maxit=2000, inner=4)
    ou, ow, ost = odae.dae_step(osys, w0, p0, 0.0, 2e-3, otab.prepare("gauss", 2), ocfg)
    assert np.linalg.norm(u1 - ou) <= 1e-11 * np.linalg.norm(ou)
    assert np.linalg.norm(w1 - ow) <= 1e-11 * np.linalg.norm(ow)
    assert st.newton_iterations == ost.newton_iterations
    assert abs(st.krylov_iterations - ost.krylov_iterations) <= 1


def test_dae_inconsistent_initial_state_is_rejected():
    prob = pk.VorticityProblem((16, 16))
    w0, p0 = pk.vorticity_initial_state(prob)
    with pytest.raises(pk.ConfigurationError):
        pk.dae_integrate(prob, w0, p0 + 1e-3, 0.0, 1e-3, 1e-3, pk.make_tableau("gauss", 2),
                         pk.SolverConfig(precond=pk.PrecondSpec(inner=4)))


def test_dae_coupled_mode_and_real_eigenvalue_blocks_are_configuration_errors():
    prob = pk.VorticityProblem((16, 16))
    w0, p0 = pk.vorticity_initial_state(prob)
    cfg = pk.SolverConfig(precond=pk.PrecondSpec(inner=4))
    with pytest.raises(pk.ConfigurationError):
        pk.dae_step(prob, w0, p0, 0.0, 1e-3, pk.make_tableau("gauss", 2), cfg, mode="coupled")
    with pytest.raises(pk.ConfigurationError):
        pk.dae_step(prob, w0, p0, 0.0, 1e-3, pk.make_tableau("radau_iia", 3), cfg)


def test_dae_full_size_first_step_properties():
    """configs[4] at 2048^2: one step converges, keeps the constraint to
    rounding (the h^2-scaled pinned Poisson rows) and conserves mean vorticity
    (Arakawa J and Lap are in divergence form)."""
    spec = pk.baseline_config(4, nsteps=1)
    prob = spec.problem
    w0, p0 = pk.vorticity_initial_state(prob)
    tab = pk.make_tableau("gauss", 2)
    cfg = pk.SolverConfig(krylov_maxit=5000, precond=pk.PrecondSpec(inner=4))
    u1, w1, st = pk.dae_step(prob, w0, p0, 0.0, spec.dt, tab, cfg)
    assert st.converged and st.residual_history[-1] <= 1e-9 * st.residual_history[0]
    assert st.constraint_residual <= 1e-10
    assert abs(u1.mean() - w0.mean()) <= 1e-12 * np.abs(w0).max()
    assert st.constraint_solves == 2 * st.newton_iterations


@pytest.mark.parametrize("shape", [(64, 40), (300, 70), (24, 16), (258, 33), (65, 30), (301, 41)])
@pytest.mark.parametrize("inner", [1, 2, 4, 6])
def test_fused_arakawa_jacobi_chain_matches_oracle(shape, inner):
    """The temporally blocked inner solve of the DAE's differential operator
    (csrc/arachain.cu, all k sweeps in one pass: warp strips of column pairs
    for even nx >= 64, 256-column CTA strips otherwise) equals k separate
    damped-Jacobi sweeps of the reference (src/irk_core.py:117-123) on
    L_u = -J(psi, .) + nu Lap; strips narrower and wider than the grid,
    ragged bands, odd extents."""
    prob = pk.VorticityProblem(shape, nu=2e-3)
    pd = DaeProblemDef(prob.shape, prob.nu)
    rng = np.random.default_rng(20 + inner)
    u = rng.standard_normal(pd.dim)
    psi = rng.standard_normal(pd.dim)
    lu = pd.blocks_csr(u, psi, 0.0)[0]
    field = pk.OperatorField(prob, psi, 1.0)
    r = rng.standard_normal(pd.dim)
    got = pk.ShiftedSolver(2.7, None, field, 3e-3, inner).solve(r)
    want = irk.ShiftedSolver(2.7, lu, 3e-3, inner).solve(r)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))
