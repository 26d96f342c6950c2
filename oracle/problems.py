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


def _shift_index(nx, ny, dx, dy):
    """Flat index of the periodic neighbour (i+dx, j+dy) for every point (x fastest)."""
    j, i = np.divmod(np.arange(nx * ny), nx)
    return ((j + dy) % ny) * nx + (i + dx) % nx


def arakawa_jacobian_matrix(psi, nx, ny, hx, hy):
    """CSR of x -> J(psi, x), Arakawa's energy/enstrophy-conserving form
    J = (J++ + J+x + Jx+)/3 on a periodic grid (x fastest)."""
    n = nx * ny
    s = lambda dx, dy: _shift_index(nx, ny, dx, dy)  # noqa: E731
    pE, pW, pN, pS = psi[s(1, 0)], psi[s(-1, 0)], psi[s(0, 1)], psi[s(0, -1)]
    pNE, pNW, pSE, pSW = psi[s(1, 1)], psi[s(-1, 1)], psi[s(1, -1)], psi[s(-1, -1)]
    coef = {
        (0, 1): (pE - pW) + (pNE - pNW),
        (0, -1): -(pE - pW) - (pSE - pSW),
        (1, 0): -(pN - pS) - (pNE - pSE),
        (-1, 0): (pN - pS) + (pNW - pSW),
        (1, 1): pE - pN,
        (1, -1): -pE + pS,
        (-1, 1): -pW + pN,
        (-1, -1): pW - pS,
    }
    scale = 1.0 / (12.0 * hx * hy)
    rows = np.concatenate([np.arange(n)] * len(coef))
    cols = np.concatenate([s(dx, dy) for (dx, dy) in coef])
    vals = np.concatenate([c * scale for c in coef.values()])
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def arakawa_jacobian(psi, w, nx, ny, hx, hy):
    """J(psi, w) evaluated directly from the three Arakawa forms."""
    s = lambda dx, dy: _shift_index(nx, ny, dx, dy)  # noqa: E731
    P = {d: psi[s(*d)] for d in [(1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, 1), (1, -1), (-1, -1)]}
    W = {d: w[s(*d)] for d in P}
    j1 = (P[1, 0] - P[-1, 0]) * (W[0, 1] - W[0, -1]) - (P[0, 1] - P[0, -1]) * (W[1, 0] - W[-1, 0])
    j2 = (P[1, 0] * (W[1, 1] - W[1, -1]) - P[-1, 0] * (W[-1, 1] - W[-1, -1])
          - P[0, 1] * (W[1, 1] - W[-1, 1]) + P[0, -1] * (W[1, -1] - W[-1, -1]))
    j3 = (W[0, 1] * (P[1, 1] - P[-1, 1]) - W[0, -1] * (P[1, -1] - P[-1, -1])
          - W[1, 0] * (P[1, 1] - P[1, -1]) + W[-1, 0] * (P[-1, 1] - P[-1, -1]))
    return (j1 + j2 + j3) / (12.0 * hx * hy)


class DaeProblemDef:
    """Vorticity/streamfunction index-1 DAE on a periodic box (BASELINE
    configs[4]), on the reference plugin API DaeSystem(dim_u, dim_w, rhs,
    constraint, blocks) (src/dae.py:52-66), modelled on shear_layer_small
    (src/problems.py:245-315):

    * differential  w_t = N(w, psi) = -J(psi, w) + nu Lap w   (Arakawa J)
    * constraint    0 = G(w, psi) = h^2 (Lap psi + w), row 0 pinned: G_0 = psi_0
      (h^2-scaled rows: the 1e-10 consistency check of dae_integrate,
      src/dae.py:527-531, rejects unscaled rows at n >= 128 -- SURVEY 8a a19)
    * linearisation with lagged advection: L_u = -J(psi, .) + nu Lap,
      L_w = 0 (so the reordered mode applies), G_u = h^2 I (row 0 zero),
      G_w = h^2 Lap with row 0 replaced by e_0.
    """

    def __init__(self, shape, nu, length=1.0):
        nx, ny = (int(x) for x in shape)
        self.shape = (nx, ny)
        self.nu = float(nu)
        self.dim = nx * ny
        hx, hy = length / nx, length / ny
        self.h2 = hx * hy
        _, lap, _ = grid_operators((nx, ny), (length, length))
        self.lap = lap
        n = self.dim

        def rhs(u, w, t):
            return -arakawa_jacobian(w, u, nx, ny, hx, hy) + self.nu * (lap @ u)

        def constraint(u, w, t):
            g = self.h2 * (lap @ w + u)
            g[0] = w[0]
            return g

        gw = (self.h2 * lap).tolil()
        gw[0, :] = 0.0
        gw[0, 0] = 1.0
        self.gw = gw.tocsr()
        gu = (self.h2 * sp.identity(n, format="csr")).tolil()
        gu[0, :] = 0.0
        self.gu = gu.tocsr()
        self.lw = sp.csr_matrix((n, n))

        def blocks(u, w, t):
            lu = (-arakawa_jacobian_matrix(w, nx, ny, hx, hy) + self.nu * lap).tocsr()
            return lu, self.lw, self.gu, self.gw

        self.rhs = rhs
        self.constraint = constraint
        self.blocks_csr = blocks

    def as_dae_system(self, dae_cls, sparse_cls):
        nx = self.shape[0]
        blocks = self.blocks_csr

        def blocks_wrapped(u, w, t):
            lu, lw, gu, gw = blocks(u, w, t)
            return (sparse_cls(lu, bandwidth=nx + 1), sparse_cls(lw, bandwidth=0),
                    sparse_cls(gu, bandwidth=0), sparse_cls(gw, bandwidth=nx))

        return dae_cls(dim_u=self.dim, dim_w=self.dim, rhs=self.rhs,
                       constraint=self.constraint, blocks=blocks_wrapped, name="vorticity2d")


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
