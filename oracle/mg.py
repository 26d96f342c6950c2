"""Restatement of the device geometric-multigrid inner solve (test infrastructure only).

``PrecondSpec(inner="mg")`` is an extension beyond the reference (SURVEY 8f
row f1; the paper uses one AMG/AIR iteration, where the
reference substitutes Jacobi-k, src/irk_core.py:103-123).  There is no
reference golden for it, so this numpy/scipy restatement of
``csrc/mg.cu`` is the checker: one V-cycle of cell-centred multigrid for
S = alpha I - dt L(a, sigma) on a periodic 2-D grid --

* level l: S_l rediscretised with h_l = 2^l h, a_l = 2x2 cell average of a_{l-1};
* 2 damped-Jacobi sweeps (omega = 2/3) from zero, residual restricted by 2x2
  averaging, bilinear (9/3/3/1)/16 prolongation, 2 post-sweeps;
* coarsest level (<= 64 points, or when a side would drop below 8): exact solve.

Operators follow kinds.cuh (the same stencils the oracle's problem builders
assemble at level 0).  Parity unpinned against the reference (no reference
counterpart); pinned against a dense solve at two levels and by linearity.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

OMEGA = 2.0 / 3.0


def operator(kind, nx, ny, ih2, i2h, a, sigma, alpha, dt, nu=0.0, c=0.0):
    """CSR of S = alpha I - dt L_eff(a, sigma) on a periodic nx x ny grid
    (x fastest), kinds.cuh / stencil_row."""
    n = nx * ny
    p = np.arange(n)
    ix, iy = p % nx, p // nx
    nb = [p + np.where(ix == 0, nx - 1, -1), p + np.where(ix == nx - 1, 1 - nx, 1),
          p + np.where(iy == 0, (ny - 1) * nx, -nx), p + np.where(iy == ny - 1, -(ny - 1) * nx, nx)]
    lapdiag = -2.0 * (ih2[0] + ih2[1])
    if kind == "nldiff":
        cc = lapdiag * a
        cn = [ih2[0] * a[nb[0]], ih2[0] * a[nb[1]], ih2[1] * a[nb[2]], ih2[1] * a[nb[3]]]
    elif kind == "burgers":
        cc = np.full(n, sigma * nu * lapdiag)
        cn = [i2h[0] * a[nb[0]] + sigma * nu * ih2[0], -i2h[0] * a[nb[1]] + sigma * nu * ih2[0],
              i2h[1] * a[nb[2]] + sigma * nu * ih2[1], -i2h[1] * a[nb[3]] + sigma * nu * ih2[1]]
    else:  # rad
        cc = sigma * nu * lapdiag + a
        cn = [np.full(n, sigma * (nu * ih2[0] - c * i2h[0])),
              np.full(n, sigma * (nu * ih2[0] + c * i2h[0])),
              np.full(n, sigma * (nu * ih2[1] - c * i2h[1])),
              np.full(n, sigma * (nu * ih2[1] + c * i2h[1]))]
    rows = np.concatenate([p] * 5)
    cols = np.concatenate([p] + nb)
    vals = np.concatenate([alpha - dt * cc] + [-dt * v for v in cn])
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def restrict(f, nx, ny):
    g = f.reshape(ny, nx)
    return 0.25 * ((g[0::2, 0::2] + g[0::2, 1::2]) + (g[1::2, 0::2] + g[1::2, 1::2])).ravel()


def prolong(xc, nxc, nyc):
    """Bilinear cell-centred prolongation to (2 nxc) x (2 nyc)."""
    g = xc.reshape(nyc, nxc)
    nx, ny = 2 * nxc, 2 * nyc
    i = np.arange(nx)
    j = np.arange(ny)
    I, J = i // 2, j // 2
    I2 = (I + np.where(i % 2 == 1, 1, -1)) % nxc
    J2 = (J + np.where(j % 2 == 1, 1, -1)) % nyc
    out = (9.0 * g[J[:, None], I[None, :]] + 3.0 * g[J[:, None], I2[None, :]]
           + 3.0 * g[J2[:, None], I[None, :]] + g[J2[:, None], I2[None, :]])
    return (out * 0.0625).ravel()


class VCycle:
    """One V-cycle as a fixed linear operator (mirrors Engine::mg_setup/mg_vcycle)."""

    def __init__(self, kind, shape, lengths, a, sigma, alpha, dt, nu=0.0, c=0.0):
        nx, ny = shape
        h = (lengths[0] / nx, lengths[1] / ny)
        ih2 = [1.0 / h[0] ** 2, 1.0 / h[1] ** 2]
        i2h = [0.5 / h[0], 0.5 / h[1]]
        self.levels = []
        af = np.asarray(a, dtype=float)
        while True:
            S = operator(kind, nx, ny, ih2, i2h, af, sigma, alpha, dt, nu, c)
            self.levels.append((nx, ny, S, S.diagonal()))
            if not (nx % 2 == 0 and ny % 2 == 0 and nx // 2 >= 8 and ny // 2 >= 8
                    and nx * ny > 64):
                break
            af = restrict(af, nx, ny)
            nx, ny = nx // 2, ny // 2
            ih2 = [v * 0.25 for v in ih2]
            i2h = [v * 0.5 for v in i2h]
        if len(self.levels) < 2:
            raise ValueError("grid too small to coarsen")
        self.coarse = spla.splu(self.levels[-1][2].tocsc())

    def _cycle(self, l, b):
        nx, ny, S, d = self.levels[l]
        if l == len(self.levels) - 1:
            return self.coarse.solve(b)
        t = OMEGA * (b / d)
        x = t + OMEGA * ((b - S @ t) / d)
        r = b - S @ x
        bc = restrict(r, nx, ny)
        xc = self._cycle(l + 1, bc)
        x = x + prolong(xc, nx // 2, ny // 2)
        t = x + OMEGA * ((b - S @ x) / d)
        return t + OMEGA * ((b - S @ t) / d)

    def solve(self, b):
        return self._cycle(0, np.asarray(b, dtype=float))
