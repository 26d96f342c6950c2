"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle and
the reference-generated golden fixtures.

Bar (BASELINE.json north star): final u within 1e-10 relative L2, per-step
Newton and Krylov counts within +/-1; operator-level results to rounding.
"""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2101_01776_b200 as pk
from oracle import irk
from oracle import tableau as otab
from oracle.problems import build_problem
from paper_2101_01776_b200.problems import GridProblem

from _golden import assert_counts_within_one, case_names, grid_problem, load_case, load_transformed

pytestmark = pytest.mark.gpu

RTOL_U = 1e-10


def _solver(sv):
    return pk.SolverConfig(
        variant=sv.get("variant", 3),
        newton_rtol=sv.get("newton_rtol", 1e-9),
        newton_maxit=sv.get("newton_maxit", 30),
        krylov_rtol=sv.get("krylov_rtol", 1e-5),
        krylov_maxit=sv.get("krylov_maxit", 200),
        restart=sv.get("restart", 200),
        precond=pk.PrecondSpec(inner=sv.get("inner", 4)),
        jacobian_refresh=sv.get("jacobian_refresh", "every"),
    )


JACOBI_CASES = [c for c in case_names() if not c.endswith("_exact")]


@pytest.mark.parametrize("name", JACOBI_CASES)
def test_integrate_matches_reference_golden(name):
    meta = load_case(name)
    prob = grid_problem(meta)
    tab = pk.make_tableau(meta["family"], meta["s"])
    res = pk.integrate(prob, meta["u0"], 0.0, meta["nsteps"] * meta["dt"], meta["dt"], tab,
                       _solver(meta["solver"]))
    ref = meta["u_final"]
    rel = np.linalg.norm(res.u_final - ref) / np.linalg.norm(ref)
    assert rel <= RTOL_U, rel
    # per-step Newton and Krylov counts within +/-1, per-block lists within +/-1
    assert_counts_within_one(res.step_stats, meta["steps"])
    for got in res.step_stats:
        assert got.precond_applications >= got.krylov_iterations
        assert got.converged


def test_config0_exact_inner_mode_matches_reference_golden():
    """configs[0] in the reference's DEFAULT inner mode, PrecondSpec(inner=
    "exact") (banded LU + SMW, src/sparsela.py:283-359) on the device
    (csrc/banded.cu): per-block Krylov counts equal the reference's exactly,
    final u within 1e-10."""
    meta = load_case("cfg0_full_exact")
    prob = grid_problem(meta)
    tab = pk.make_tableau("gauss", 2)
    sv = dict(meta["solver"], inner="exact")
    cfg = pk.SolverConfig(variant=sv["variant"], newton_rtol=sv["newton_rtol"],
                          newton_maxit=sv["newton_maxit"], krylov_rtol=sv["krylov_rtol"],
                          krylov_maxit=sv["krylov_maxit"], restart=sv["restart"],
                          precond=pk.PrecondSpec(inner="exact"))
    res = pk.integrate(prob, meta["u0"], 0.0, meta["nsteps"] * meta["dt"], meta["dt"], tab, cfg)
    rel = np.linalg.norm(res.u_final - meta["u_final"]) / np.linalg.norm(meta["u_final"])
    assert rel <= RTOL_U, rel
    assert len(res.step_stats) == len(meta["steps"])
    for got, want in zip(res.step_stats, meta["steps"]):
        assert got.newton_iterations == want["newton_iterations"]
        assert got.block_iterations == want["block_iterations"]


def test_exact_shifted_solve_is_exact():
    """ShiftedSolver(inner="exact") on 1-D and 2-D periodic operators (with
    the out-of-band wrap through SMW): residual at rounding level, against a
    dense solve of the same operator assembled by the oracle."""
    from oracle.problems import build_problem

    for kind, shape, kw in (("burgers", (40, 24), dict(nu=1e-2)), ("nldiff", (32, 32), {}),
                            ("rad", (50,), dict(nu=1e-2, c=0.7, lam=-1.0))):
        prob = GridProblem(kind, shape, **kw)
        rng = np.random.default_rng(3)
        U = rng.standard_normal(prob.dim)
        f = pk.OperatorField.linearize(prob, U[None, :])
        r = rng.standard_normal(prob.dim)
        x = pk.ShiftedSolver(1.7, None, f, 0.05, inner="exact").solve(r)
        pd = build_problem(prob.kind, prob.shape, **prob.oracle_params())
        A = 1.7 * np.eye(prob.dim) - 0.05 * pd.linearize_csr(U, 0.0).toarray()
        xd = np.linalg.solve(A, r)
        assert np.linalg.norm(x - xd) <= 1e-12 * np.linalg.norm(xd), kind


def test_exact_inner_mode_limits_are_configuration_errors():
    prob = GridProblem("nldiff", (8, 8, 8))
    f = pk.OperatorField.linearize(prob, np.ones((1, 512)))
    with pytest.raises(pk.ConfigurationError):
        pk.ShiftedSolver(2.0, None, f, 1e-2, inner="exact").solve(np.ones(512))


def test_config0_counts_exact_per_block():
    meta = load_case("cfg0_full")
    prob = grid_problem(meta)
    tab = pk.make_tableau("gauss", 2)
    res = pk.integrate(prob, meta["u0"], 0.0, 10e-3, 1e-3, tab, _solver(meta["solver"]))
    assert len(res.step_stats) == len(meta["steps"])
    for got, want in zip(res.step_stats, meta["steps"]):
        assert got.newton_iterations == want["newton_iterations"]
        for off, its in want["block_iterations"].items():
            g = got.block_iterations[off]
            assert len(g) == len(its)
            assert all(abs(a - b) <= 1 for a, b in zip(g, its)), (g, its)
        assert got.jacobian_assemblies == want["jacobian_assemblies"]
        np.testing.assert_allclose(got.residual_history, want["residual_history"], rtol=1e-6,
                                   atol=1e-9 * want["residual_history"][0])


# ------------------------------------------------------ operator level


def _field(prob, vals, sigma=1.0):
    return pk.OperatorField(prob, np.asarray(vals, dtype=float), sigma)


def test_block2x2_known_answers():
    # pkg/tests/test_irk_core.py:52-60 with N = 1 ("rad" kind: L x = a x)
    prob = GridProblem("rad", (1,))
    z = _field(prob, [0.0])
    sysb = pk.Block2x2System(3.0, np.sqrt(3.0), 1.0, None, z, z, 1.0)
    np.testing.assert_allclose(pk.apply_block2x2(sysb, np.array([1.0, 0.0])), [3.0, -3.0],
                               atol=1e-15)
    sysb = pk.Block2x2System(3.0, np.sqrt(3.0), 1.0, None, _field(prob, [-1.0]),
                             _field(prob, [-2.0]), 1.0)
    np.testing.assert_allclose(pk.apply_block2x2(sysb, np.array([1.0, 1.0])), [5.0, 2.0],
                               atol=1e-14)
    sysb = pk.Block2x2System(2.0, 0.0, 1.0, None, _field(prob, [-1.0]), _field(prob, [-2.0]), 1.0)
    assert pk.apply_block2x2(sysb, np.array([1.0, 0.0]))[1] == 0.0
    with pytest.raises(ValueError):
        pk.apply_block2x2(sysb, np.zeros(3))


def test_precond_scalar_known_answer_with_jacobi():
    # test_irk_core.py:71-73 is exact mode; with N = 1 the Jacobi iteration on a
    # scalar converges geometrically: compare with the oracle's Jacobi-k.
    prob = GridProblem("rad", (1,))
    z = _field(prob, [0.0])
    sysb = pk.Block2x2System(3.0, np.sqrt(3.0), 1.0, None, z, z, 1.0)
    for k in (1, 2, 4, 7):
        got = pk.precond_block2x2(sysb, pk.PrecondSpec(inner=k), np.array([1.0, 0.0]))
        pre = irk.block2x2_precond(3.0, np.sqrt(3.0), 1.0, sp.csr_matrix([[0.0]]),
                                   sp.csr_matrix([[0.0]]), 1.0, "star", k)
        np.testing.assert_allclose(got, pre(np.array([1.0, 0.0])), rtol=1e-15, atol=1e-16)
    got = pk.precond_block2x2(sysb, pk.PrecondSpec(inner=60), np.array([1.0, 0.0]))
    np.testing.assert_allclose(got, [1.0 / 3.0, 0.25], rtol=1e-12)


KIND_CASES = [
    ("nldiff", (16, 12), {}),
    ("nldiff", (8, 6, 5), {}),
    ("nldiff", (40,), {}),
    ("burgers", (20, 18), {"nu": 0.02}),
    ("burgers", (6, 5, 4), {"nu": 0.05}),
    ("rad", (30,), {"nu": 0.01, "c": 0.5, "lam": -0.2, "mu": 0.3}),
    ("rad", (9, 7), {"nu": 0.03, "c": -0.4, "lam": 0.1, "mu": -0.5}),
]


def _oracle_sys(prob):
    pd = build_problem(prob.kind, prob.shape, **prob.oracle_params())
    return pd, irk.OdeSystem(pd.dim, pd.rhs, pd.linearize_csr)


@pytest.mark.parametrize("kind,shape,params", KIND_CASES)
def test_stage_residual_matches_oracle(kind, shape, params):
    prob = GridProblem(kind, shape, **params)
    pd, sysr = _oracle_sys(prob)
    tab = pk.make_tableau("gauss", 3)
    rng = np.random.default_rng(7)
    u = rng.standard_normal(pd.dim)
    k = rng.standard_normal((3, pd.dim))
    got = pk.stage_residual(prob, pk.StageState(k=k, u=u, t=0.0, dt=0.01), tab)
    want = irk.stage_residual(sysr, u, k, 0.0, 0.01, otab.prepare("gauss", 3).tableau)
    scale = np.max(np.abs(want))
    assert np.max(np.abs(got - want)) <= 1e-13 * scale


@pytest.mark.parametrize("kind,shape,params", KIND_CASES)
def test_operator_fields_match_weighted_csr_sum(kind, shape, params):
    # combine(w, [L(U_k)]) @ x  ==  L_eff(a, sigma) x  (via the 1x1 block operator)
    prob = GridProblem(kind, shape, **params)
    pd, _ = _oracle_sys(prob)
    rng = np.random.default_rng(3)
    U = rng.standard_normal((3, pd.dim))
    w = np.array([0.7, 0.0, -0.4])
    field = pk.OperatorField.linearize(prob, U, w)
    csr = irk.combine(w, [pd.linearize_csr(U[i], 0.0) for i in range(3)])
    x = rng.standard_normal(pd.dim)
    # block operator with beta = 0, phi = 1: top = eta x1 - dt L1 x1 + x2
    sysb = pk.Block2x2System(0.0, 0.0, 1.0, None, field, field, 1.0)
    y = pk.apply_block2x2(sysb, np.concatenate([x, np.zeros(pd.dim)]))
    want = -(csr @ x)
    assert np.max(np.abs(y[: pd.dim] - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))


@pytest.mark.parametrize("kind,shape,params", KIND_CASES[:4])
def test_shifted_jacobi_matches_oracle(kind, shape, params):
    prob = GridProblem(kind, shape, **params)
    pd, _ = _oracle_sys(prob)
    rng = np.random.default_rng(11)
    U = rng.standard_normal((1, pd.dim))
    field = pk.OperatorField.linearize(prob, U)
    lmat = pd.linearize_csr(U[0], 0.0)
    r = rng.standard_normal(pd.dim)
    for inner in (1, 4):
        got = pk.ShiftedSolver(2.5, None, field, 1e-3, inner).solve(r)
        want = irk.ShiftedSolver(2.5, lmat, 1e-3, inner).solve(r)
        assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))


FUSED_CASES = [
    ("nldiff", (32, 12), {}),
    ("nldiff", (50, 40), {}),
    ("burgers", (128, 64), {"nu": 0.01}),
    ("burgers", (37, 15), {"nu": 0.05}),
    ("rad", (64, 33), {"nu": 0.02, "c": 0.3, "lam": -0.4, "mu": 0.2}),
]


@pytest.mark.parametrize("kind,shape,params", FUSED_CASES)
@pytest.mark.parametrize("inner", [1, 2, 4, 6])
def test_fused_jacobi_chain_matches_oracle(kind, shape, params, inner):
    """The temporally blocked 2-D inner solve (csrc/jacobi.cu) equals k
    separate damped-Jacobi sweeps of the reference (src/irk_core.py:117-123)."""
    prob = GridProblem(kind, shape, **params)
    pd, _ = _oracle_sys(prob)
    rng = np.random.default_rng(inner)
    U = rng.standard_normal((1, pd.dim))
    field = pk.OperatorField.linearize(prob, U)
    lmat = pd.linearize_csr(U[0], 0.0)
    r = rng.standard_normal(pd.dim)
    got = pk.ShiftedSolver(3.1, None, field, 2e-3, inner).solve(r)
    want = irk.ShiftedSolver(3.1, lmat, 2e-3, inner).solve(r)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))


FUSED3D_CASES = [
    ("nldiff", (32, 32, 10), {}),
    ("nldiff", (58, 40, 13), {}),       # ragged last tiles in x and y, ragged z bands
    ("burgers", (34, 32, 9), {"nu": 0.02}),
    ("rad", (32, 36, 12), {"nu": 0.02, "c": 0.3, "lam": -0.4, "mu": 0.2}),
]


@pytest.mark.parametrize("kind,shape,params", FUSED3D_CASES)
@pytest.mark.parametrize("inner", [1, 2, 4, 6])
def test_fused_jacobi_chain_3d_matches_oracle(kind, shape, params, inner):
    """The 3.5-D blocked inner solve (csrc/jacobi3d.cu: 32x32 in-plane tiles
    sliding along z, all k sweeps in one pass) equals k separate damped-Jacobi
    sweeps of the reference (src/irk_core.py:117-123)."""
    prob = GridProblem(kind, shape, **params)
    pd, _ = _oracle_sys(prob)
    rng = np.random.default_rng(10 + inner)
    U = rng.standard_normal((1, pd.dim))
    field = pk.OperatorField.linearize(prob, U)
    lmat = pd.linearize_csr(U[0], 0.0)
    r = rng.standard_normal(pd.dim)
    got = pk.ShiftedSolver(3.1, None, field, 2e-3, inner).solve(r)
    want = irk.ShiftedSolver(3.1, lmat, 2e-3, inner).solve(r)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))


def test_fused_block_precond_3d_matches_oracle():
    """Block lower-triangular 2x2 preconditioner on a 3-D grid: both fused
    chains (the second with the coupling field) against the oracle."""
    prob = GridProblem("nldiff", (40, 32, 11))
    pd, _ = _oracle_sys(prob)
    rng = np.random.default_rng(5)
    U = rng.standard_normal((2, pd.dim))
    f1 = pk.OperatorField.linearize(prob, U[:1])
    f2 = pk.OperatorField.linearize(prob, U[1:])
    l1, l2 = pd.linearize_csr(U[0], 0.0), pd.linearize_csr(U[1], 0.0)
    eta, beta, phi, dt = 2.681083, 3.050430, -1.104613, 1e-3
    r = rng.standard_normal(2 * pd.dim)
    sysb = pk.Block2x2System(eta, beta, phi, None, f1, f2, dt)
    got = pk.precond_block2x2(sysb, pk.PrecondSpec(inner=4), r)
    want = irk.block2x2_precond(eta, beta, phi, l1, l2, dt, "star", 4)(r)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))


@pytest.mark.parametrize("kind,shape,params", FUSED_CASES[:3])
def test_fused_block_precond_matches_oracle(kind, shape, params):
    prob = GridProblem(kind, shape, **params)
    pd, _ = _oracle_sys(prob)
    rng = np.random.default_rng(2)
    U = rng.standard_normal((2, pd.dim))
    f1 = pk.OperatorField.linearize(prob, U[:1])
    f2 = pk.OperatorField.linearize(prob, U[1:])
    l1, l2 = pd.linearize_csr(U[0], 0.0), pd.linearize_csr(U[1], 0.0)
    eta, beta, phi, dt = 2.681083, 3.050430, -1.104613, 1e-3
    r = rng.standard_normal(2 * pd.dim)
    sysb = pk.Block2x2System(eta, beta, phi, None, f1, f2, dt)
    got = pk.precond_block2x2(sysb, pk.PrecondSpec(inner=4), r)
    want = irk.block2x2_precond(eta, beta, phi, l1, l2, dt, "star", 4)(r)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))


@pytest.mark.parametrize("size", [1, 2])
def test_block_gmres_counts_match_oracle(size):
    prob = GridProblem("burgers", (32, 32), nu=1e-2)
    pd, _ = _oracle_sys(prob)
    rng = np.random.default_rng(5)
    U = 0.5 * rng.standard_normal((2, pd.dim))
    f1 = pk.OperatorField.linearize(prob, U[:1])
    f2 = pk.OperatorField.linearize(prob, U[1:])
    l1 = pd.linearize_csr(U[0], 0.0)
    l2 = pd.linearize_csr(U[1], 0.0)
    dt = 5e-3
    eta, beta, phi = 3.677815, 3.508762, -10.983731
    rhs = rng.standard_normal(size * pd.dim)
    for restart in (200, 7):
        if size == 2:
            sysb = pk.Block2x2System(eta, beta, phi, None, f1, f2, dt)
            x, rep = pk.block_gmres(sysb, rhs, pk.PrecondSpec(inner=4), 1e-10, 500, restart)
            pre = irk.block2x2_precond(eta, beta, phi, l1, l2, dt, "star", 4)
            xo, repo = irk.gmres(lambda v: irk.block2x2_apply(eta, beta, phi, l1, l2, dt, v), rhs,
                                 2 * pd.dim, pre, 2, 1e-10, 500, restart)
        else:
            x, rep = pk.block_gmres((eta, f1, dt), rhs, pk.PrecondSpec(inner=4), 1e-10, 500,
                                    restart)
            solver = irk.ShiftedSolver(eta, l1, dt, 4)
            xo, repo = irk.gmres(lambda v: eta * v - dt * (l1 @ v), rhs, pd.dim, solver.solve, 1,
                                 1e-10, 500, restart)
        assert rep.converged and repo.converged
        assert abs(rep.iterations - repo.iterations) <= 1, (rep.iterations, repo.iterations)
        assert rep.precond_applications == size * rep.iterations
        assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)
        n = min(len(rep.residuals), len(repo.residuals))
        np.testing.assert_allclose(rep.residuals[: n - 1], repo.residuals[: n - 1], rtol=1e-6)


@pytest.mark.parametrize("shape,size", [((36, 28), 1), ((66, 50), 2), ((130, 96), 2)])
def test_block_gmres_ragged_tiles_all_cgs_forms(shape, size):
    """Block sizes that leave a partial last CGS tile (n % 1024 != 0), with
    restarts that put the basis in every row-owner bucket of the update
    sweeps (L <= 4, 8, 16) and past it (L up to 24: slot-owner tile work):
    counts within +/-1 of the oracle's GMRES (src/sparsela.py:176-280) and
    the same solution."""
    prob = GridProblem("burgers", shape, nu=1e-2)
    pd, _ = _oracle_sys(prob)
    rng = np.random.default_rng(11)
    U = 0.5 * rng.standard_normal((2, pd.dim))
    f1 = pk.OperatorField.linearize(prob, U[:1])
    f2 = pk.OperatorField.linearize(prob, U[1:])
    l1 = pd.linearize_csr(U[0], 0.0)
    l2 = pd.linearize_csr(U[1], 0.0)
    dt = 5e-3
    eta, beta, phi = 3.677815, 3.508762, -10.983731
    rhs = rng.standard_normal(size * pd.dim)
    for restart in (4, 8, 16, 24):
        if size == 2:
            sysb = pk.Block2x2System(eta, beta, phi, None, f1, f2, dt)
            x, rep = pk.block_gmres(sysb, rhs, pk.PrecondSpec(inner=4), 1e-10, 500, restart)
            pre = irk.block2x2_precond(eta, beta, phi, l1, l2, dt, "star", 4)
            xo, repo = irk.gmres(lambda v: irk.block2x2_apply(eta, beta, phi, l1, l2, dt, v), rhs,
                                 2 * pd.dim, pre, 2, 1e-10, 500, restart)
        else:
            x, rep = pk.block_gmres((eta, f1, dt), rhs, pk.PrecondSpec(inner=4), 1e-10, 500,
                                    restart)
            solver = irk.ShiftedSolver(eta, l1, dt, 4)
            xo, repo = irk.gmres(lambda v: eta * v - dt * (l1 @ v), rhs, pd.dim, solver.solve, 1,
                                 1e-10, 500, restart)
        assert rep.converged and repo.converged
        assert abs(rep.iterations - repo.iterations) <= 1, (restart, rep.iterations,
                                                            repo.iterations)
        assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)


def test_block_gmres_maxit_and_zero_rhs():
    prob = GridProblem("nldiff", (16, 16))
    f = pk.OperatorField.linearize(prob, np.ones((1, 256)))
    x, rep = pk.block_gmres((2.0, f, 1e-2), np.zeros(256))
    assert rep.converged and rep.iterations == 0 and np.all(x == 0.0)
    rng = np.random.default_rng(0)
    _, rep = pk.block_gmres((2.0, f, 1e-2), rng.standard_normal(256), pk.PrecondSpec(inner=1),
                            rtol=1e-14, maxit=3, restart=2)
    assert not rep.converged and rep.iterations == 3
    with pytest.raises(ValueError):
        pk.block_gmres((2.0, f, 1e-2), np.ones(256), rtol=2.0)


@pytest.mark.parametrize("route", ["stage_linearization", "stage_ops", "variant_jacobian"])
def test_transformed_solve_matches_reference_all_variants(route):
    """solve_transformed_system (src/irk_core.py:225-338) against the
    reference's own runs on every variant, with the operators passed each way
    the reference accepts them: stage values (the device forms the fields),
    a list of s stage operators + variant (the reference's
    ``[lmat] * s`` call, tests/test_irk_core.py:152-167), or a prebuilt
    VariantJacobian (``variant_jacobian=``, src/irk_core.py:225-237)."""
    prob = GridProblem("rad", (24,), nu=0.01, c=1.0)
    lop = pk.OperatorField.linearize(prob, np.zeros((1, 24)))
    for case in load_transformed():
        s = case["s"]
        tab = pk.make_tableau(case["family"], s)
        prep = pk.prepare_stages(tab)
        rng = np.random.default_rng(case["seed"])
        rhs = rng.standard_normal((s, 24))
        kw = dict(precond=pk.PrecondSpec(inner=case["inner"]), krylov_rtol=1e-12,
                  krylov_maxit=400)
        if route == "stage_linearization":
            lin = pk.StageLinearization(prob, np.zeros(24), np.zeros((s, 24)), 0.05)
            k, stats = pk.solve_transformed_system(prep, lin, case["variant"], case["dt"], rhs,
                                                   **kw)
        elif route == "stage_ops":
            k, stats = pk.solve_transformed_system(prep, [lop] * s, case["variant"], case["dt"],
                                                   rhs, **kw)
        else:
            vj = pk.build_variant_jacobian(prep, [lop] * s, case["variant"])
            k, stats = pk.solve_transformed_system(prep, dt=case["dt"], rhs_stages=rhs,
                                                   variant_jacobian=vj, **kw)
        got = [[o, r.iterations] for o, r in stats.reports]
        assert [g[0] for g in got] == [w[0] for w in case["reports"]]
        for g, w in zip(got, case["reports"]):
            assert abs(g[1] - w[1]) <= 1, (case["family"], s, case["variant"], got, case["reports"])
        assert np.max(np.abs(k - case["k"])) <= 1e-9


# -------------------------------------------------------- error paths


def test_stage_solve_error_carries_block_and_report():
    # pattern of pkg/tests/test_irk_core.py:200-209
    meta = load_case("cfg0_full")
    prob = grid_problem(meta)
    cfg = pk.SolverConfig(krylov_rtol=1e-13, krylov_maxit=2, newton_rtol=1e-10,
                          precond=pk.PrecondSpec(inner=4))
    with pytest.raises(pk.StageSolveError) as err:
        pk.step(prob, meta["u0"], 0.0, 1e-3, pk.make_tableau("gauss", 2), cfg)
    assert err.value.block_offset == 0
    assert err.value.report is not None and err.value.report.iterations == 2
    assert not err.value.report.converged
    assert len(err.value.report.residuals) == 3


def test_step_failure_error_carries_stats_and_partial():
    meta = load_case("cfg0_full")
    prob = grid_problem(meta)
    cfg = pk.SolverConfig(newton_maxit=1, newton_rtol=1e-12, krylov_rtol=1e-3,
                          precond=pk.PrecondSpec(inner=4))
    with pytest.raises(pk.StepFailureError) as err:
        pk.integrate(prob, meta["u0"], 0.0, 3e-3, 1e-3, pk.make_tableau("gauss", 2), cfg)
    assert err.value.stats is not None and err.value.stats.newton_iterations == 1
    assert err.value.partial is not None and len(err.value.partial.states) == 1


SDIRK_CASES = [c for c in case_names() if c.startswith("sdirk_")]


@pytest.mark.parametrize("name", SDIRK_CASES)
def test_sdirk_per_stage_counts_match_reference(name):
    """The SDIRK baseline (src/nonlinear.py:239-296) on the device: Newton
    counts per stage equal, Krylov counts per stage solve within +/-1."""
    meta = load_case(name)
    prob = grid_problem(meta)
    tab = pk.make_tableau(meta["family"])
    u = meta["u0"]
    for j, want in enumerate(meta["steps"]):
        u, got = pk.step(prob, u, j * meta["dt"], meta["dt"], tab, _solver(meta["solver"]))
        assert got.newton_iterations == want["newton_iterations"]
        assert got.jacobian_assemblies == want["jacobian_assemblies"]
        assert sorted(got.block_iterations) == sorted(want["block_iterations"])
        for stage, its in want["block_iterations"].items():
            g = got.block_iterations[stage]
            assert len(g) == len(its)
            assert all(abs(a - b) <= 1 for a, b in zip(g, its)), (stage, g, its)
        np.testing.assert_allclose(got.residual_history, want["residual_history"], rtol=1e-6,
                                   atol=1e-9 * max(want["residual_history"]))
    rel = np.linalg.norm(u - meta["u_final"]) / np.linalg.norm(meta["u_final"])
    assert rel <= RTOL_U, rel


# ------------------------------------------------- full-size properties


def test_config1_full_size_first_step_properties():
    """configs[1] at its full 1024^2 size: one step converges, the Newton
    residual drops below tolerance, and the u-update is the stage
    combination (u_next - u = dt b^T K, checked through a second route)."""
    spec = pk.baseline_config(1, nsteps=1)
    prob = spec.problem
    u0 = spec.u0()
    tab = pk.make_tableau("gauss", 3)
    cfg = _solver(spec.solver)
    u0_before = u0.copy()
    u1, stats = pk.step(prob, u0, 0.0, spec.dt, tab, cfg)
    # value semantics of the reference's step(): a new array, u untouched
    assert u1 is not u0 and np.array_equal(u0, u0_before)
    assert stats.converged
    assert stats.residual_history[-1] <= 1e-9 * stats.residual_history[0]
    assert 3 <= stats.newton_iterations <= 10
    # same step through the device-tensor path is bit-identical (deterministic reductions)
    import torch

    u1d, stats2 = pk.step(prob, torch.from_numpy(u0).cuda(), 0.0, spec.dt, tab, cfg)
    assert np.array_equal(u1d.cpu().numpy(), u1)
    assert stats2.krylov_iterations == stats.krylov_iterations
    # conservation: every kind here is in divergence form -> mean(u) preserved
    assert abs(u1.mean() - u0.mean()) <= 1e-12 * np.abs(u0).max()
