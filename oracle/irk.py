"""Restatement of irkit's stage-solve hot path (test infrastructure only).

Follows, function by function, the reference package
(``/root/reference/pkg/src/irkit``; paths below are relative to it):

* ``gmres``                   src/sparsela.py:176-280
* ``jacobi_solver``           src/irk_core.py:103-123 (ShiftedSolver, inner=k)
* ``block2x2_apply``          src/irk_core.py:126-140
* ``block2x2_precond``        src/irk_core.py:147-165
* ``solve_transformed``       src/irk_core.py:225-338
* ``variant_weights``         src/nonlinear.py:99-126
* ``stage_residual``          src/nonlinear.py:145-152
* ``newton_like_step``        src/nonlinear.py:186-236
* ``step`` / ``integrate``    src/nonlinear.py:299-314, 331-374
* ``dirk_step``               src/nonlinear.py:239-296 (the SDIRK baseline)

Matrices are scipy CSR; ``mass`` is the identity throughout (all BASELINE
configurations have M = I).  Exact inner solves use a sparse LU
(scipy ``splu``) in place of the reference's banded LU + SMW wrap
(src/sparsela.py:283-359): both are exact to rounding.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class OracleError(Exception):
    pass


class StageSolveError(OracleError):
    def __init__(self, msg, block_offset=None, report=None):
        super().__init__(msg)
        self.block_offset = block_offset
        self.report = report


class StepFailureError(OracleError):
    def __init__(self, msg, stats=None, partial=None):
        super().__init__(msg)
        self.stats = stats
        self.partial = partial


class KrylovBreakdownError(OracleError):
    pass


@dataclass
class OdeSystem:
    """Plugin type of src/nonlinear.py:35-48 (identity mass only)."""

    dim: int
    rhs: object
    linearize: object
    mass: object = None
    name: str = ""


def _csr(m):
    return m.csr if hasattr(m, "csr") else sp.csr_matrix(m)


# --------------------------------------------------------------------- GMRES


@dataclass
class KrylovReport:
    iterations: int
    converged: bool
    residuals: list = field(default_factory=list)
    precond_applications: int = 0


def gmres(apply_op, rhs, n, apply_m=None, spa=0, rtol=1e-5, maxit=200, restart=200):
    """Restarted right-preconditioned GMRES with CGS2 (src/sparsela.py:176-280).

    Control flow is the reference's: Givens estimate test (253-256), the
    breakdown threshold ``1e-14*max(wnorm0, 1e-300)`` (229-233), the dead
    column exit (238-246), and a true-residual recheck per cycle (262-272).
    """
    rhs = np.asarray(rhs, dtype=float)
    if rhs.shape != (n,):
        raise ValueError(f"rhs has shape {rhs.shape}, expected ({n},)")
    if not (0.0 < rtol < 1.0):
        raise ValueError(f"rtol must lie in (0, 1), got {rtol}")
    if apply_m is None:
        apply_m = lambda v: v  # noqa: E731
    bnorm = np.linalg.norm(rhs)
    if bnorm == 0.0:
        return np.zeros(n), KrylovReport(0, True, [0.0], 0)
    x = np.zeros(n)
    r = rhs.copy()
    beta = np.linalg.norm(r)
    residuals = [beta / bnorm]
    total_it = 0
    converged = residuals[0] <= rtol
    while not converged and total_it < maxit:
        m = min(restart, maxit - total_it)
        v = np.zeros((n, m + 1))
        z = np.zeros((n, m))
        h = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        v[:, 0] = r / beta
        g[0] = beta
        breakdown = False
        j = -1
        for j in range(m):
            zj = apply_m(v[:, j])
            z[:, j] = zj
            w = apply_op(zj)
            wnorm0 = np.linalg.norm(w)
            for _ in range(2):  # CGS with one re-orthogonalisation (224-227)
                coef = v[:, : j + 1].T @ w
                w -= v[:, : j + 1] @ coef
                h[: j + 1, j] += coef
            hj = np.linalg.norm(w)
            h[j + 1, j] = hj
            if hj <= 1e-14 * max(wnorm0, 1e-300):
                breakdown = True
            else:
                v[:, j + 1] = w / hj
            for i in range(j):
                tmp = cs[i] * h[i, j] + sn[i] * h[i + 1, j]
                h[i + 1, j] = -sn[i] * h[i, j] + cs[i] * h[i + 1, j]
                h[i, j] = tmp
            denom = np.hypot(h[j, j], h[j + 1, j])
            if denom == 0.0:
                breakdown = True
                j -= 1
                total_it += 1
                residuals.append(residuals[-1])
                break
            cs[j], sn[j] = h[j, j] / denom, h[j + 1, j] / denom
            h[j, j] = denom
            h[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total_it += 1
            est = abs(g[j + 1]) / bnorm
            residuals.append(est)
            if est <= rtol or breakdown or total_it >= maxit:
                break
        k = j + 1
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - h[i, i + 1 : k] @ y[i + 1 : k]) / h[i, i]
        x = x + z[:, :k] @ y
        r = rhs - apply_op(x)
        true_rel = np.linalg.norm(r) / bnorm
        residuals[-1] = true_rel
        if true_rel <= rtol:
            converged = True
        elif breakdown:
            raise KrylovBreakdownError(
                f"Arnoldi breakdown with residual {true_rel:.3e} above rtol {rtol:.3e}"
            )
        beta = np.linalg.norm(r)
    return x, KrylovReport(total_it, converged, residuals, total_it * spa)


# ------------------------------------------------------- shifted inner solves


def combine(coeffs, mats):
    """Weighted CSR sum in stage order, zero weights skipped (src/sparsela.py:106-128)."""
    shape = next(m.shape for m in mats if m is not None)
    acc = sp.csr_matrix(shape)
    for ck, mk in zip(coeffs, mats):
        if ck == 0.0:
            continue
        if mk is None:
            acc = acc + ck * sp.identity(shape[0], format="csr")
        else:
            acc = acc + ck * _csr(mk)
    return acc.tocsr()


class ShiftedSolver:
    """``(alpha*I - dt*L)^{-1}`` by k damped-Jacobi sweeps from zero
    (src/irk_core.py:103-123, omega = 2/3) or exactly."""

    def __init__(self, alpha, lmat, dt, inner):
        self.mat = combine([alpha, -dt], [None, lmat])
        self.inner = inner
        if inner == "exact":
            self._lu = spla.splu(self.mat.tocsc())
        else:
            diag = self.mat.diagonal()
            if np.any(diag == 0.0):
                raise ValueError("Jacobi inner solver needs a nonzero diagonal")
            self._invdiag = 1.0 / diag

    def solve(self, r):
        if self.inner == "exact":
            return self._lu.solve(r)
        x = np.zeros_like(r)
        for _ in range(self.inner):
            x = x + (2.0 / 3.0) * (self._invdiag * (r - self.mat @ x))
        return x


def gamma_of(gamma_mode, eta, beta):
    """PrecondSpec.gamma (src/irk_core.py:63-68)."""
    if gamma_mode == "star":
        return eta + beta * beta / eta
    if gamma_mode == "eta":
        return eta
    return float(gamma_mode)


def block2x2_apply(eta, beta, phi, l1, l2, dt, x, c12=None, c21=None):
    """src/irk_core.py:126-140 with M = I."""
    n = l1.shape[0]
    x1, x2 = x[:n], x[n:]
    top = eta * x1 - dt * (l1 @ x1) + phi * x2
    bot = -(beta**2 / phi) * x1 + eta * x2 - dt * (l2 @ x2)
    if c12 is not None:
        top -= dt * (c12 @ x2)
    if c21 is not None:
        bot -= dt * (c21 @ x1)
    return np.concatenate([top, bot])


def block2x2_precond(eta, beta, phi, l1, l2, dt, gamma_mode, inner):
    """Block lower-triangular preconditioner (src/irk_core.py:147-165)."""
    gamma = gamma_of(gamma_mode, eta, beta)
    s1 = ShiftedSolver(eta, l1, dt, inner)
    s2 = ShiftedSolver(gamma, l2, dt, inner)
    n = l1.shape[0]
    coupling = beta**2 / phi

    def apply(r):
        z1 = s1.solve(r[:n])
        z2 = s2.solve(r[n:] + coupling * z1)
        return np.concatenate([z1, z2])

    return apply


# -------------------------------------------------------------- transformed


@dataclass
class SolveStats:
    reports: list = field(default_factory=list)

    @property
    def krylov_iterations(self):
        return sum(rep.iterations for _, rep in self.reports)

    @property
    def precond_applications(self):
        return sum(rep.precond_applications for _, rep in self.reports)


def variant_weights(prep, variant, variant0_stage=0):
    """src/nonlinear.py:99-126."""
    s = prep.tableau.s
    d = prep.d
    diag = np.zeros((s, s))
    offdiag = {}
    if variant == 0:
        diag[:, variant0_stage] = 1.0
        return diag, offdiag
    if variant == 1:
        for i in range(s):
            diag[i, int(np.argmax(np.abs(d[i, i])))] = 1.0
        return diag, offdiag
    for i in range(s):
        diag[i] = d[i, i]
    if variant == 2:
        return diag, offdiag
    for i in range(s):
        for j in range(i + 1, s):
            offdiag[(i, j)] = d[i, j]
    for blk in prep.blocks:
        if blk.size == 2:
            offdiag[(blk.offset + 1, blk.offset)] = d[blk.offset + 1, blk.offset]
    return diag, offdiag


def build_variant_jacobian(prep, stage_ops, variant, variant0_stage=0):
    """src/nonlinear.py:129-142 -> (diag tuple, offdiag dict) of CSR."""
    dw, ow = variant_weights(prep, variant, variant0_stage)
    ops = [_csr(o) for o in stage_ops]
    diag = tuple(combine(dw[i], ops) for i in range(prep.tableau.s))
    offdiag = {key: combine(w, ops) for key, w in ow.items()}
    return diag, offdiag


def solve_transformed(prep, vjac, dt, rhs_stages, gamma_mode="star", inner=4,
                      krylov_rtol=1e-5, krylov_maxit=200, restart=200):
    """Backward block sweep of the Schur-transformed stage system
    (src/irk_core.py:225-338), identity mass."""
    diag, offdiag = vjac
    rhs = np.asarray(rhs_stages, dtype=float)
    s = prep.tableau.s
    q, r0 = prep.q, prep.r
    g = q.T @ rhs
    y = np.zeros_like(g)
    stats = SolveStats()
    for blk in reversed(prep.blocks):
        rows = list(range(blk.offset, blk.offset + blk.size))
        acc = g[rows].copy()
        for local, ri in enumerate(rows):
            for j in range(blk.offset + blk.size, s):
                coef = r0[ri, j]
                if coef != 0.0:
                    acc[local] -= coef * y[j]
                od = offdiag.get((ri, j))
                if od is not None:
                    acc[local] += dt * (od @ y[j])
        if blk.size == 1:
            lmat = diag[blk.offset]
            n = lmat.shape[0]
            eta = blk.eta
            solver = ShiftedSolver(eta, lmat, dt, inner)
            sol, rep = gmres(
                lambda x, lmat=lmat, eta=eta: eta * x - dt * (lmat @ x),
                acc[0], n, solver.solve, 1, krylov_rtol, krylov_maxit, restart,
            )
            if not rep.converged:
                raise StageSolveError(
                    f"1x1 block at offset {blk.offset} did not converge",
                    block_offset=blk.offset, report=rep,
                )
            y[rows[0]] = sol
        else:
            l1, l2 = diag[blk.offset], diag[blk.offset + 1]
            c12 = offdiag.get((blk.offset, blk.offset + 1))
            c21 = offdiag.get((blk.offset + 1, blk.offset))
            n = l1.shape[0]
            pre = block2x2_precond(blk.eta, blk.beta, blk.phi, l1, l2, dt, gamma_mode, inner)
            sol, rep = gmres(
                lambda x, b=blk: block2x2_apply(b.eta, b.beta, b.phi, l1, l2, dt, x, c12, c21),
                np.concatenate([acc[0], acc[1]]), 2 * n, pre, 2,
                krylov_rtol, krylov_maxit, restart,
            )
            if not rep.converged:
                raise StageSolveError(
                    f"2x2 block at offset {blk.offset} did not converge",
                    block_offset=blk.offset, report=rep,
                )
            y[rows[0]] = sol[:n]
            y[rows[1]] = sol[n:]
        stats.reports.append((blk.offset, rep))
    return (q @ r0) @ y, stats


# ------------------------------------------------------------------- Newton


@dataclass
class StepStats:
    newton_iterations: int = 0
    krylov_iterations: int = 0
    precond_applications: int = 0
    jacobian_assemblies: int = 0
    converged: bool = False
    residual_history: list = field(default_factory=list)
    block_iterations: dict = field(default_factory=dict)
    wall_time: float = 0.0

    def add_solve(self, st):
        self.krylov_iterations += st.krylov_iterations
        self.precond_applications += st.precond_applications
        for off, rep in st.reports:
            self.block_iterations.setdefault(off, []).append(rep.iterations)


@dataclass
class Config:
    """SolverConfig + PrecondSpec fields (src/nonlinear.py:61-83, src/irk_core.py:39-68)."""

    variant: int = 3
    newton_rtol: float = 1e-9
    newton_maxit: int = 30
    newton_abs_floor: float = 1e-14
    krylov_rtol: float = 1e-5
    krylov_maxit: int = 200
    restart: int = 200
    gamma_mode: object = "star"
    inner: object = 4
    jacobian_refresh: str = "every"
    variant0_stage: int = 0


def stage_residual(sys, u, k, t, dt, tableau):
    """src/nonlinear.py:145-152 (identity mass)."""
    u_stage = u[None, :] + dt * (tableau.a0 @ k)
    out = np.empty_like(k)
    for i in range(tableau.s):
        out[i] = sys.rhs(u_stage[i], t + tableau.c0[i] * dt)
        out[i] -= k[i]
    return out


def newton_like_step(sys, u, k, t, dt, prep, cfg):
    """src/nonlinear.py:186-236; returns (k, StepStats)."""
    tab = prep.tableau
    stats = StepStats()
    tic = time.perf_counter()
    res = stage_residual(sys, u, k, t, dt, tab)
    f0 = np.linalg.norm(res)
    stats.residual_history.append(f0)
    tol = max(cfg.newton_rtol * f0, cfg.newton_abs_floor)
    vjac = None
    while stats.newton_iterations < cfg.newton_maxit:
        if np.linalg.norm(res) <= tol:
            stats.converged = True
            break
        if vjac is None or cfg.jacobian_refresh == "every":
            times = t + tab.c0 * dt
            u_stage = u[None, :] + dt * (tab.a0 @ k)
            ops = [sys.linearize(u_stage[i], times[i]) for i in range(tab.s)]
            stats.jacobian_assemblies += tab.s
            vjac = build_variant_jacobian(prep, ops, cfg.variant, cfg.variant0_stage)
        dk, sst = solve_transformed(
            prep, vjac, dt, res, cfg.gamma_mode, cfg.inner,
            cfg.krylov_rtol, cfg.krylov_maxit, cfg.restart,
        )
        k = k + dk
        stats.newton_iterations += 1
        stats.add_solve(sst)
        res = stage_residual(sys, u, k, t, dt, tab)
        stats.residual_history.append(np.linalg.norm(res))
    else:
        if np.linalg.norm(res) > tol:
            stats.wall_time = time.perf_counter() - tic
            raise StepFailureError("stage solve stalled", stats=stats)
        stats.converged = True
    stats.wall_time = time.perf_counter() - tic
    return k, stats


def dirk_step(sys, u, t, dt, tableau, cfg):
    """src/nonlinear.py:239-296: sequential stage solves of an SDIRK tableau;
    returns (u_next, k, StepStats) with block_iterations keyed by stage."""
    s, n = tableau.s, sys.dim
    k = np.zeros((s, n))
    stats = StepStats()
    tic = time.perf_counter()
    for i in range(s):
        base = u + dt * (tableau.a0[i, :i] @ k[:i]) if i else u.copy()
        aii = tableau.a0[i, i]
        ti = t + tableau.c0[i] * dt
        ki = np.zeros(n)
        res = sys.rhs(base + dt * aii * ki, ti) - ki
        f0 = np.linalg.norm(res)
        stats.residual_history.append(f0)
        tol = max(cfg.newton_rtol * f0, cfg.newton_abs_floor)
        it = 0
        while np.linalg.norm(res) > tol:
            if it >= cfg.newton_maxit:
                stats.wall_time = time.perf_counter() - tic
                raise StepFailureError(f"DIRK stage {i} stalled", stats=stats)
            lmat = _csr(sys.linearize(base + dt * aii * ki, ti))
            stats.jacobian_assemblies += 1
            solver = ShiftedSolver(1.0, lmat, dt * aii, cfg.inner)
            dk, rep = gmres(lambda x: x - dt * aii * (lmat @ x), res, n, solver.solve, 1,
                            cfg.krylov_rtol, cfg.krylov_maxit, cfg.restart)
            ki += dk
            it += 1
            stats.newton_iterations += 1
            stats.krylov_iterations += rep.iterations
            stats.precond_applications += rep.precond_applications
            stats.block_iterations.setdefault(i, []).append(rep.iterations)
            res = sys.rhs(base + dt * aii * ki, ti) - ki
            stats.residual_history.append(np.linalg.norm(res))
        k[i] = ki
    stats.converged = True
    stats.wall_time = time.perf_counter() - tic
    return u + dt * (tableau.b0 @ k), k, stats


def step(sys, u, t, dt, prep, cfg):
    """src/nonlinear.py:299-314 (collocation tableaux only)."""
    k = np.zeros((prep.tableau.s, sys.dim))
    k, stats = newton_like_step(sys, np.asarray(u, dtype=float), k, t, dt, prep, cfg)
    return u + dt * (prep.tableau.b0 @ k), stats


def integrate(sys, u0, t0, t_final, dt, prep, cfg, max_steps=None):
    """src/nonlinear.py:331-374 (every state kept).  ``max_steps`` bounds the
    march for CPU-baseline sampling."""
    span = t_final - t0
    nsteps_f = span / dt
    nsteps = int(round(nsteps_f))
    if abs(nsteps_f - nsteps) > 1e-8 * max(1.0, abs(nsteps_f)):
        raise ValueError("(t_final - t0)/dt is not an integer step count")
    if max_steps is not None:
        nsteps = min(nsteps, max_steps)
    u = np.array(u0, dtype=float)
    states = [u.copy()]
    all_stats = []
    for j in range(nsteps):
        u, stats = step(sys, u, t0 + j * dt, dt, prep, cfg)
        all_stats.append(stats)
        states.append(u.copy())
    return states, all_stats
