"""The multigrid inner-solve restatement (oracle/mg.py):
a fixed linear map, and a far stronger (gamma I - dt L) preconditioner than
the Jacobi-k mode at BASELINE stiffness."""

import numpy as np
import pytest

from oracle import irk
from oracle.mg import VCycle, operator, prolong, restrict


def _field(shape, seed, kind):
    rng = np.random.default_rng(seed)
    U = rng.standard_normal(shape[0] * shape[1])
    return 1.0 + U * U if kind == "nldiff" else U


def test_restrict_prolong_shapes_and_constants():
    f = np.arange(64.0)
    assert restrict(f, 8, 8).shape == (16,)
    np.testing.assert_allclose(prolong(np.ones(16), 4, 4), np.ones(64))
    np.testing.assert_allclose(restrict(np.ones(64), 8, 8), np.ones(16))


@pytest.mark.parametrize("kind,kw", [("nldiff", {}), ("burgers", dict(nu=1e-2)),
                                     ("rad", dict(nu=1e-2, c=0.5))])
def test_vcycle_is_linear(kind, kw):
    shape = (64, 64)
    mg = VCycle(kind, shape, (1.0, 1.0), _field(shape, 1, kind), 1.0, 3.0, 2e-4, **kw)
    rng = np.random.default_rng(2)
    x, y = rng.standard_normal(4096), rng.standard_normal(4096)
    lhs = mg.solve(2.0 * x - 0.5 * y)
    rhs = 2.0 * mg.solve(x) - 0.5 * mg.solve(y)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)


def test_vcycle_beats_jacobi4_on_stiff_nldiff():
    """configs[2] stiffness (dt/h^2 ~ 3300, the 4096^2 value) on a 128^2
    grid with the seeded Fourier field a = 1 + u0^2: one V-cycle per inner
    solve keeps GMRES at ~15 iterations, Jacobi-4 needs hundreds."""
    from paper_2101_01776_b200.problems import fourier_u0

    n = 128
    U = fourier_u0((n, n), 1, 16, 0.1, 0)
    a = 1.0 + U * U
    alpha, dt = 4.0, 0.2
    h = 1.0 / n
    S = operator("nldiff", n, n, [1 / h**2] * 2, [0.5 / h] * 2, a, 1.0, alpha, dt)
    b = np.random.default_rng(5).standard_normal(S.shape[0])
    mg = VCycle("nldiff", (n, n), (1.0, 1.0), a, 1.0, alpha, dt)
    d = S.diagonal()

    def jac4(r):
        x = np.zeros_like(r)
        for _ in range(4):
            x = x + (2.0 / 3.0) * ((r - S @ x) / d)
        return x

    x, rep_mg = irk.gmres(lambda x: S @ x, b, S.shape[0], mg.solve, 1, 1e-8, 3000, 200)
    _, rep_j = irk.gmres(lambda x: S @ x, b, S.shape[0], jac4, 1, 1e-8, 3000, 200)
    assert rep_mg.converged and rep_j.converged
    assert np.linalg.norm(S @ x - b) <= 1e-8 * np.linalg.norm(b) * 1.0001
    assert rep_mg.iterations <= 25 and rep_mg.iterations * 8 <= rep_j.iterations, (
        rep_mg.iterations, rep_j.iterations)
