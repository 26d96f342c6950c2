"""Oracle problem builders for the BASELINE configurations (test infrastructure).

None of the five BASELINE problems exists in the reference catalog
(``src/problems.py:318-326`` only has 1-D problems and a desk-scale shear
layer).  They are written here on the reference's own plugin API -- an
``OdeSystem(dim, rhs(u, t), linearize(u, t) -> SparseMatrix)``
(``src/nonlinear.py:35-48``) -- so that the real ``irkit`` and the oracle
restatement can both run them.  The CSR assembly follows the reference's
periodic grid operators (``src/problems.py:120-134`` central difference /
Laplacian, ``src/problems.py:233-242`` x-fastest Kronecker layout).

The CUDA kernels implement the same discretisations matrix-free:

* ``nldiff``  u_t = div((1+u^2) grad u) written in Kirchhoff form
  ``N(u) = Lap_h(u + u^3/3)`` (exact identity (1+u^2) grad u = grad(u+u^3/3)),
  Jacobian ``L(U) = Lap_h diag(1 + U^2)``.
* ``burgers`` u_t + div(u^2/2 (1,..,1)) = nu Lap u with central differences,
  ``N(u) = -Dsum(u^2/2) + nu Lap_h u``, ``L(U) = -Dsum diag(U) + nu Lap_h``
  (the 2-D analogue of ``burgers1d``, ``src/problems.py:175-200``).
* ``rad``     reaction-advection-diffusion with constant coefficients,
  ``N(u) = nu Lap_h u + c Dsum u + lam u + mu u^2`` -- covers the reference
  catalog's dahlquist / advection1d / advdiff1d and the logistic test system
  on periodic grids.

Domain: periodic box of side ``length`` (default 1) per axis, ``h = length/n``.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def _central_1d(n, h):
    # periodic central difference, src/problems.py:120-125
    if n == 1:
        return sp.csr_matrix((1, 1))
    i = np.arange(n)
    rows = np.concatenate([i, i])
    cols = np.concatenate([(i + 1) % n, (i - 1) % n])
    vals = np.concatenate([np.full(n, 1.0 / (2.0 * h)), np.full(n, -1.0 / (2.0 * h))])
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def _laplacian_1d(n, h):
    # periodic 3-point Laplacian, src/problems.py:128-134
    if n == 1:
        return sp.csr_matrix((1, 1))
    i = np.arange(n)
    rows = np.concatenate([i, i, i])
    cols = np.concatenate([i, (i + 1) % n, (i - 1) % n])
    vals = np.concatenate(
        [np.full(n, -2.0 / h**2), np.full(n, 1.0 / h**2), np.full(n, 1.0 / h**2)]
    )
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def _axis_embed(mat1d, axis, shape):
    """Kronecker embedding with x fastest: flat = (k*ny + j)*nx + i."""
    out = None
    # kron order: slowest axis first
    for ax in reversed(range(len(shape))):
        m = mat1d if ax == axis else sp.identity(shape[ax], format="csr")
        out = m if out is None else sp.kron(out, m, format="csr")
    return out.tocsr()


def grid_operators(shape, lengths=None):
    """(Dsum, Lap, h) for a periodic grid of ``shape`` (x fastest)."""
    shape = tuple(int(n) for n in shape)
    if lengths is None:
        lengths = (1.0,) * len(shape)
    hs = tuple(float(lengths[a]) / shape[a] for a in range(len(shape)))
    dsum = None
    lap = None
    for ax, n in enumerate(shape):
        d_ax = _axis_embed(_central_1d(n, hs[ax]), ax, shape)
        l_ax = _axis_embed(_laplacian_1d(n, hs[ax]), ax, shape)
        dsum = d_ax if dsum is None else dsum + d_ax
        lap = l_ax if lap is None else lap + l_ax
    return dsum.tocsr(), lap.tocsr(), hs


def band_hint(shape):
    """Bandwidth hint for the reference SparseMatrix (in-band stencil part)."""
    if len(shape) == 1:
        return 1
    return int(np.prod(shape[:-1]))


class ProblemDef:
    """Callables of one oracle problem: ``rhs(u, t)`` and ``linearize(u, t)``
    returning a scipy CSR matrix.  ``as_ode_system`` wraps them into the
    reference plugin types (irkit's or the oracle's own)."""

    def __init__(self, kind, shape, params, rhs, linearize):
        self.kind = kind
        self.shape = tuple(shape)
        self.params = dict(params)
        self.dim = int(np.prod(self.shape))
        self.rhs = rhs
        self.linearize_csr = linearize

    def as_ode_system(self, ode_cls, sparse_cls):
        bw = band_hint(self.shape)
        lin = self.linearize_csr
        return ode_cls(
            dim=self.dim,
            rhs=self.rhs,
            linearize=lambda u, t: sparse_cls(lin(u, t), bandwidth=bw),
            name=f"{self.kind}{len(self.shape)}d",
        )


def build_problem(kind, shape, **params):
    shape = tuple(int(n) for n in shape)
    lengths = params.get("lengths")
    dsum, lap, _ = grid_operators(shape, lengths)
    if kind == "nldiff":

        def rhs(u, t):
            return lap @ (u + u * u * u / 3.0)

        def linearize(u, t):
            return (lap @ sp.diags(1.0 + u * u)).tocsr()

    elif kind == "burgers":
        nu = float(params.get("nu", 1e-2))

        def rhs(u, t):
            return -(dsum @ (0.5 * u * u)) + nu * (lap @ u)

        def linearize(u, t):
            return (-(dsum @ sp.diags(u)) + nu * lap).tocsr()

    elif kind == "rad":
        nu = float(params.get("nu", 0.0))
        c = float(params.get("c", 0.0))
        lam = float(params.get("lam", 0.0))
        mu = float(params.get("mu", 0.0))
        base = (nu * lap + c * dsum).tocsr()

        def rhs(u, t):
            return base @ u + lam * u + mu * u * u

        def linearize(u, t):
            return (base + sp.diags(lam + 2.0 * mu * u)).tocsr()

    else:
        raise ValueError(f"unknown oracle problem kind {kind!r}")
    return ProblemDef(kind, shape, params, rhs, linearize)
