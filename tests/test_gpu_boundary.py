"""The reference-side binding INTEGRATION.md documents
(``include/irkg_ctypes.py``), executed as written against the built
``libirkg.so``: its step equals the package's ``step`` bit for bit and the
reference golden's first step (counts, 1e-10)."""

import importlib.util
import os
import sys

import numpy as np
import pytest

import paper_2101_01776_b200 as pk
from paper_2101_01776_b200 import _lib

from _golden import grid_problem, load_case

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub():
    spec = importlib.util.spec_from_file_location(
        "irkg_ctypes", os.path.join(ROOT, "include", "irkg_ctypes.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _irkit_or_mirror():
    """irkit's own StagePrep / SolverConfig when the reference is installed
    (baseline/_ref), else the package's duck-typed mirrors."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.append(ref)
    try:
        import irkit
        from irkit.irk_core import PrecondSpec
        from irkit.nonlinear import SolverConfig
        return irkit.prepare_stages, irkit.make_tableau, SolverConfig, PrecondSpec
    except ImportError:
        return pk.prepare_stages, pk.make_tableau, pk.SolverConfig, pk.PrecondSpec


def test_ctypes_stub_step_matches_package_and_golden():
    G = _stub()
    lib = G.load(_lib.LIB_PATH)
    meta = load_case("cfg1_n64")
    prob = grid_problem(meta)
    prepare, make_tab, SolverConfig, PrecondSpec = _irkit_or_mirror()
    prep = prepare(make_tab("gauss", 3))
    cfg = SolverConfig(krylov_maxit=5000, restart=200, precond=PrecondSpec(inner=4))
    u0 = np.array(meta["u0"])
    u_before = u0.copy()
    un, stats = G.step_on_gpu(lib, "burgers", prob.shape, {"nu": prob.nu}, u0, 0.0, meta["dt"],
                              prep, cfg)
    assert np.array_equal(u0, u_before)          # value semantics: u untouched
    want = meta["steps"][0]
    assert stats.newton_iterations == want["newton_iterations"]
    assert abs(stats.krylov_iterations - want["krylov_iterations"]) <= 1
    u_pk, st_pk = pk.step(prob, u0, 0.0, meta["dt"], pk.make_tableau("gauss", 3),
                          pk.SolverConfig(krylov_maxit=5000, precond=pk.PrecondSpec(inner=4)))
    assert np.array_equal(un, u_pk)              # same engine, same arithmetic
    assert stats.krylov_iterations == st_pk.krylov_iterations


def test_ctypes_stub_surfaces_step_failure():
    G = _stub()
    lib = G.load(_lib.LIB_PATH)
    prepare, make_tab, SolverConfig, PrecondSpec = _irkit_or_mirror()
    prob = pk.GridProblem("burgers", (64, 64), nu=1e-2)
    u0 = pk.fourier_u0(prob.shape, 1, 8, 0.5, seed=0)
    cfg = SolverConfig(newton_maxit=1, newton_rtol=1e-12, precond=PrecondSpec(inner=4))
    with pytest.raises(RuntimeError, match="StepFailureError"):
        G.step_on_gpu(lib, "burgers", prob.shape, {"nu": 1e-2}, u0, 0.0, 5e-4,
                      prepare(make_tab("gauss", 3)), cfg)


@pytest.mark.parametrize("kind,shape,params", [
    ("burgers", (40, 24), {"nu": 1e-2}),
    ("nldiff", (32, 32), {}),
    ("rad", (50,), {"nu": 1e-2, "c": 0.7, "lam": -1.0, "mu": 0.3}),
    ("nldiff", (12, 10, 8), {}),
])
def test_grid_problem_is_an_ode_system(kind, shape, params):
    """The problem descriptor satisfies irkit's OdeSystem protocol
    (src/nonlinear.py:35-48): dim, rhs(u, t), linearize(u, t), mass, name --
    with rhs and the Jacobian's matvec evaluated on the device and equal to
    the reference-side (oracle) CSR definitions."""
    from oracle.problems import build_problem

    prob = pk.GridProblem(kind, shape, **params)
    pd = build_problem(prob.kind, prob.shape, **prob.oracle_params())
    rng = np.random.default_rng(2)
    u = rng.standard_normal(prob.dim)
    x = rng.standard_normal(prob.dim)
    assert prob.dim == pd.dim and prob.mass is None and prob.name
    f = prob.rhs(u, 0.0)
    want = pd.rhs(u, 0.0)
    assert isinstance(f, np.ndarray) and f.shape == (prob.dim,)
    assert np.max(np.abs(f - want)) <= 1e-12 * np.max(np.abs(want))
    jac = prob.linearize(u, 0.0)
    y = jac @ x
    want = pd.linearize_csr(u, 0.0) @ x
    assert np.max(np.abs(y - want)) <= 1e-12 * np.max(np.abs(want))


def test_combine_and_variant_weights_match_reference_rules():
    """combine (src/sparsela.py:106-128) of device operator fields is the
    weighted sum of the operators (zero weights skipped; all-zero -> None)."""
    from oracle import irk
    from oracle.problems import build_problem

    prob = pk.GridProblem("burgers", (32, 16), nu=1e-2)
    pd = build_problem(prob.kind, prob.shape, **prob.oracle_params())
    rng = np.random.default_rng(4)
    U = rng.standard_normal((3, prob.dim))
    fields = [pk.OperatorField.linearize(prob, U[i]) for i in range(3)]
    mats = [pd.linearize_csr(U[i], 0.0) for i in range(3)]
    w = [0.25, 0.0, -1.5]
    x = rng.standard_normal(prob.dim)
    got = pk.combine(w, fields) @ x
    want = irk.combine(w, mats) @ x
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
    assert pk.combine([0.0, 0.0, 0.0], fields) is None
