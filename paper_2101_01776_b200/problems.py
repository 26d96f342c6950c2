"""Grid problem descriptors for the device stage solver (the problem plugin).

A descriptor plays the role of the reference's ``OdeSystem``
(``src/nonlinear.py:35-48``): it has ``dim``, ``mass`` (always ``None``, the
identity, for the BASELINE configurations) and ``name``; but instead of
host callables ``rhs``/``linearize`` it names a *kind* whose nonlinear
operator N(u) and Jacobian-vector product are implemented matrix-free in the
CUDA kernels (``csrc/kinds.cuh``):

========  ==========================================  ===========================
kind      N(u)                                        L(U) x  (exact Jacobian)
========  ==========================================  ===========================
nldiff    Lap_h(u + u^3/3)   [= div((1+u^2) grad u)]  Lap_h((1 + U^2) x)
burgers   -Dsum(u^2/2) + nu Lap_h u                   -Dsum(U x) + nu Lap_h x
rad       nu Lap_h u + c Dsum u + lam u + mu u^2      nu Lap_h x + c Dsum x + (lam + 2 mu U) x
========  ==========================================  ===========================

``Lap_h`` is the periodic 2d+1-point Laplacian and ``Dsum`` the sum over
axes of periodic central differences on a box of side ``length`` per axis,
``h = length / n``; DOFs are ordered x fastest (``src/problems.py:238-239``).

Because every Jacobian above is affine in a single pointwise function of the
stage state, the weighted operator sums the reference materialises with
``combine`` (``src/sparsela.py:106-128``) collapse to one coefficient field
``a = sum_k w_k f(U_k)`` plus the scalar ``sigma = sum_k w_k``; the device
keeps only those fields ("operator fields").
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

KINDS = ("nldiff", "burgers", "rad")
KIND_CODE = {"nldiff": 0, "burgers": 1, "rad": 2, "arakawa": 3}


@dataclass(frozen=True)
class GridProblem:
    kind: str
    shape: tuple
    nu: float = 0.0
    c: float = 0.0
    lam: float = 0.0
    mu: float = 0.0
    length: float = 1.0
    name: str = ""
    lengths: tuple = None  # per-axis box sides (default: ``length`` on every axis)

    def __post_init__(self):
        if self.lengths is not None:
            object.__setattr__(self, "lengths", tuple(float(x) for x in self.lengths))
        if self.kind not in KINDS:
            raise ValueError(f"unknown problem kind {self.kind!r}; available: {KINDS}")
        shape = tuple(int(n) for n in self.shape)
        if not (1 <= len(shape) <= 3) or min(shape) < 1:
            raise ValueError(f"shape must have 1-3 positive extents, got {self.shape}")
        object.__setattr__(self, "shape", shape)
        if not self.name:
            object.__setattr__(self, "name", f"{self.kind}{len(shape)}d")

    @property
    def dim(self):
        return int(np.prod(self.shape))

    @property
    def mass(self):
        return None

    @property
    def ndim(self):
        return len(self.shape)

    @property
    def box(self):
        return self.lengths if self.lengths is not None else (self.length,) * self.ndim

    @property
    def h(self):
        return tuple(L / n for L, n in zip(self.box, self.shape))

    # ---- the OdeSystem protocol (src/nonlinear.py:35-48): dim, rhs,
    # linearize, mass, name -- so a GridProblem is itself a valid irkit
    # OdeSystem whose callables run on the device (irkg_rhs; the Jacobian is
    # a matrix-free OperatorField whose ``@`` / ``matvec`` is
    # irkg_operator_apply)
    def rhs(self, u, t=0.0):
        """N(u, t) by the device stencil kernel; numpy in -> numpy out."""
        from .solver import problem_rhs

        return problem_rhs(self, u, t)

    def linearize(self, u, t=0.0):
        """The exact Jacobian dN/du at u as a device ``OperatorField``."""
        from .solver import OperatorField

        return OperatorField.linearize(self, u)

    def oracle_params(self):
        """Keyword arguments for ``oracle.problems.build_problem`` (tests only)."""
        p = {"lengths": self.box}
        if self.kind == "burgers":
            p["nu"] = self.nu
        elif self.kind == "rad":
            p.update(nu=self.nu, c=self.c, lam=self.lam, mu=self.mu)
        return p


def fourier_modes(ndim, k_lo, k_hi):
    """Integer wavevectors k != 0 with k_lo <= |k| <= k_hi, lexicographic
    (first axis outermost), each component over -k_hi..k_hi."""
    rng = range(-k_hi, k_hi + 1)
    out = []
    if ndim == 1:
        grid = ((a,) for a in rng)
    elif ndim == 2:
        grid = ((a, b) for a in rng for b in rng)
    else:
        grid = ((a, b, c) for a in rng for b in rng for c in rng)
    for k in grid:
        k2 = sum(x * x for x in k)
        if k2 == 0:
            continue
        if k_lo * k_lo <= k2 <= k_hi * k_hi:
            out.append(k)
    return out


def fourier_u0(shape, k_lo=1, k_hi=4, sigma=0.1, seed=0):
    """Seeded random Fourier-mode field on the periodic unit box.

    ``u(x) = sum_k a_k cos(2 pi k.x) + b_k sin(2 pi k.x)`` at cell centres
    ``x_i = (i + 1/2)/n``, with ``(a_k, b_k) ~ N(0, sigma)`` drawn in mode
    order from ``np.random.default_rng(seed)``; k = (kx, ky, kz) pairs with
    the (x, y, z) axes.  Evaluated separably as the real part of a complex
    product so 4096^2 / 256^3 grids take seconds.  Returns a flat x-fastest
    float64 array.
    """
    shape = tuple(int(n) for n in shape)
    ndim = len(shape)
    modes = fourier_modes(ndim, k_lo, k_hi)
    rng = np.random.default_rng(seed)
    ab = rng.normal(0.0, sigma, size=(len(modes), 2))
    kr = 2 * k_hi + 1
    coef = np.zeros((kr,) * ndim, dtype=complex)
    for (k, (a, b)) in zip(modes, ab):
        coef[tuple(x + k_hi for x in k)] += complex(a, -b)
    ks = np.arange(-k_hi, k_hi + 1)

    def basis(n):
        x = (np.arange(n) + 0.5) / n
        return np.exp(2j * np.pi * np.outer(ks, x))  # (kr, n)

    if ndim == 1:
        u = (coef @ basis(shape[0])).real
    elif ndim == 2:
        ex, ey = basis(shape[0]), basis(shape[1])
        # coef[kx, ky]; u[j, i] = Re sum coef[kx,ky] ex[kx,i] ey[ky,j]
        t = coef.T @ ex  # (ky, nx)
        u = (ey.T @ t).real  # (ny, nx)
    else:
        ex, ey, ez = basis(shape[0]), basis(shape[1]), basis(shape[2])
        t = np.einsum("abc,ai->bci", coef, ex)  # (ky, kz, nx)
        t = np.einsum("bci,bj->cji", t, ey)  # (kz, ny, nx)
        u = np.einsum("cji,ck->kji", t, ez).real  # (nz, ny, nx)
    return np.ascontiguousarray(u, dtype=np.float64).ravel()


@dataclass(frozen=True)
class VorticityProblem:
    """2-D incompressible Navier-Stokes in vorticity/streamfunction DAE form
    (BASELINE configs[4]) -- the device analogue of the reference's
    ``DaeSystem`` plugin (src/dae.py:52-66), modelled on shear_layer_small
    (src/problems.py:245-315):

    * differential u = omega:  omega_t = -J(psi, omega) + nu Lap_h omega
      (Arakawa Jacobian J = (J++ + J+x + Jx+)/3);
    * algebraic    w = psi:    0 = G = h^2 (Lap_h psi + omega), row 0 pinned
      to psi_0 (h^2-scaled so the reference's absolute 1e-10 consistency
      check holds at every n);
    * linearisation with lagged advection: L_u = -J(psi, .) + nu Lap_h,
      L_w = 0 (reordered mode), G_u = h^2 I (row 0 zero), G_w = h^2 Lap_h
      with row 0 replaced by e_0.
    """

    shape: tuple
    nu: float = 1e-4
    length: float = 1.0
    name: str = "vorticity2d"

    def __post_init__(self):
        shape = tuple(int(n) for n in self.shape)
        if len(shape) != 2 or min(shape) < 3:
            raise ValueError(f"vorticity problem needs a 2-D grid >= 3x3, got {self.shape}")
        object.__setattr__(self, "shape", shape)

    kind = "arakawa"

    @property
    def dim_u(self):
        return self.shape[0] * self.shape[1]

    @property
    def dim_w(self):
        return self.dim_u

    @property
    def dim(self):
        return self.dim_u

    @property
    def mass(self):
        return None

    @property
    def ndim(self):
        return 2

    c = 0.0
    lam = 0.0
    mu = 0.0


def pinned_poisson(f, shape, pin_value=0.0, length=1.0):
    """Solve Lap_h y = f on rows i != 0 with y_0 = pin_value (periodic, x fastest).

    The rows of Lap_h sum to zero, so row 0 of Lap_h y is -sum_{i != 0} f_i; the
    zero-mean periodic problem is solved spectrally and shifted so y_0 equals
    the pin.  Used to build the consistent initial streamfunction."""
    nx, ny = shape
    fl = np.array(f, dtype=float).ravel()
    fl[0] = -(fl[1:].sum())
    hx, hy = length / nx, length / ny
    kx = np.arange(nx)
    ky = np.arange(ny)
    lam = (-4.0 / hx**2) * np.sin(np.pi * kx / nx)[None, :] ** 2 + (
        -4.0 / hy**2) * np.sin(np.pi * ky / ny)[:, None] ** 2
    lam[0, 0] = 1.0
    yh = np.fft.fft2(fl.reshape(ny, nx)) / lam
    yh[0, 0] = 0.0
    y = np.real(np.fft.ifft2(yh)).ravel()
    return y - y[0] + pin_value


def vorticity_initial_state(prob, k_lo=2, k_hi=10, sigma=1.0, seed=0):
    """(omega0, psi0): seeded Fourier-mode vorticity and the streamfunction
    satisfying the pinned constraint G(omega0, psi0) = 0."""
    omega0 = fourier_u0(prob.shape, k_lo, k_hi, sigma, seed)
    psi0 = pinned_poisson(-omega0, prob.shape, 0.0, prob.length)
    return omega0, psi0


# --------------------------------------------------------------- catalog


@dataclass(frozen=True)
class RunSpec:
    """One BASELINE configuration: problem, initial state, scheme, manifest."""

    name: str
    problem: GridProblem
    family: str
    s: int
    dt: float
    nsteps: int
    u0_args: dict
    solver: dict = field(default_factory=dict)

    def u0(self):
        return fourier_u0(self.problem.shape, **self.u0_args)


#: Manifest pinned for every config: variant 3, gamma*, Jacobi-4
#: inner solves, restart 200, krylov_maxit raised to 5000, newton_maxit 30.
BASE_SOLVER = dict(variant=3, inner=4, restart=200, krylov_maxit=5000, newton_maxit=30)


def baseline_config(index, n=None, nsteps=None, family=None, s=None):
    """BASELINE.json ``configs[index]`` (optionally at a reduced grid size)."""
    if index == 0:
        nn = n or 64
        prob = GridProblem("nldiff", (nn, nn))
        spec = RunSpec("cfg0_nldiff2d", prob, family or "gauss", s or 2, 1e-3, nsteps or 10,
                       dict(k_lo=1, k_hi=4, sigma=0.1, seed=0),
                       dict(BASE_SOLVER, newton_rtol=1e-10, krylov_rtol=1e-10))
    elif index == 1:
        nn = n or 1024
        prob = GridProblem("burgers", (nn, nn), nu=1e-2)
        spec = RunSpec("cfg1_burgers2d", prob, family or "gauss", s or 3, 5e-4, nsteps or 20,
                       dict(k_lo=1, k_hi=8, sigma=0.5, seed=0), dict(BASE_SOLVER))
    elif index == 2:
        nn = n or 4096
        prob = GridProblem("nldiff", (nn, nn))
        spec = RunSpec("cfg2_nldiff2d", prob, family or "gauss", s or 2, 2e-4, nsteps or 10,
                       dict(k_lo=1, k_hi=16, sigma=0.1, seed=0), dict(BASE_SOLVER))
    elif index == 3:
        nn = n or 256
        prob = GridProblem("nldiff", (nn, nn, nn))
        spec = RunSpec("cfg3_nldiff3d", prob, family or "gauss", s or 5, 1e-3, nsteps or 5,
                       dict(k_lo=1, k_hi=6, sigma=0.1, seed=0), dict(BASE_SOLVER))
    elif index == 4:
        nn = n or 2048
        prob = VorticityProblem((nn, nn), nu=1e-4)
        spec = RunSpec("cfg4_vorticity2d", prob, family or "gauss", s or 2, 1e-3, nsteps or 10,
                       dict(k_lo=2, k_hi=10, sigma=1.0, seed=0), dict(BASE_SOLVER))
    else:
        raise ValueError(f"no baseline config {index}")
    return spec
