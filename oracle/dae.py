"""Restatement of irkit's index-1 DAE stage solve (test infrastructure only).

Follows src/dae.py of the reference:

* ``dae_stage_residual``      src/dae.py:94-105
* ``ConstraintSolver``        src/dae.py:108-126 (exact solves with G_w; splu
                              in place of BandedLU, both exact to rounding)
* ``solve_block4x4_reordered`` src/dae.py:195-279, 307-315 (mode="reordered":
                              differential 2x2 GMRES with the block
                              preconditioner, then two constraint solves,
                              then the composite true-residual recheck)
* ``build_dae_variant``       src/dae.py:318-333
* ``solve_dae_transformed``   src/dae.py:336-420 (2x2 eigen-blocks)
* ``dae_newton_step`` / ``dae_step`` / ``dae_integrate``  src/dae.py:423-564

Only the reordered mode is restated: SURVEY 8a a18 -- the coupled mode
hard-codes exact differential solves (src/dae.py:140) and ignores inner=k.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse.linalg as spla

from . import irk


class IndexViolationError(irk.OracleError):
    pass


@dataclass
class DaeSystem:
    dim_u: int
    dim_w: int
    rhs: object
    constraint: object
    blocks: object
    mass: object = None
    name: str = ""


@dataclass
class DaeCounters:
    differential: int = 0
    constraint: int = 0


@dataclass
class DaeStepStats(irk.StepStats):
    constraint_residual: float = 0.0
    differential_solves: int = 0
    constraint_solves: int = 0


def dae_stage_residual(sys, u, w, k, ell, t, dt, tab):
    """src/dae.py:94-105 (identity mass)."""
    u_stage = u[None, :] + dt * (tab.a0 @ k)
    w_stage = w[None, :] + dt * (tab.a0 @ ell)
    out = np.empty((tab.s, sys.dim_u + sys.dim_w))
    for i in range(tab.s):
        ti = t + tab.c0[i] * dt
        out[i, : sys.dim_u] = sys.rhs(u_stage[i], w_stage[i], ti) - k[i]
        out[i, sys.dim_u:] = sys.constraint(u_stage[i], w_stage[i], ti)
    return out


class ConstraintSolver:
    """Exact solves with G_w (src/dae.py:108-126)."""

    def __init__(self, gw, counters):
        self.counters = counters
        try:
            self._lu = spla.splu(gw.tocsc())
        except RuntimeError as exc:
            raise IndexViolationError(f"constraint Jacobian is singular: {exc}") from exc

    def solve(self, r):
        self.counters.constraint += 1
        return self._lu.solve(r)


def build_dae_variant(prep, stage_ops, variant, variant0_stage=0):
    """src/dae.py:318-333: componentwise weighted sums (lu, lw, gu, gw)."""
    dw, ow = irk.variant_weights(prep, variant, variant0_stage)

    def comb(weights):
        return tuple(irk.combine(weights, [op[c] for op in stage_ops]) for c in range(4))

    diag = tuple(comb(dw[i]) for i in range(prep.tableau.s))
    offdiag = {key: comb(w) for key, w in ow.items()}
    return diag, offdiag


def solve_block4x4_reordered(ops_i, ops_j, eta, beta, phi, dt, rhs, gamma_mode, inner,
                             counters, rtol, maxit, restart):
    """src/dae.py:255-279 + true-residual recheck 307-315."""
    lu_i, lw_i, gu_i, gw_i = ops_i
    lu_j, lw_j, gu_j, gw_j = ops_j
    nu, nw = lu_i.shape[0], gw_i.shape[0]
    n = nu + nw
    if lw_i.nnz or lw_j.nnz:
        raise irk.OracleError("reordered mode requires structurally zero L_w blocks")
    pre = irk.block2x2_precond(eta, beta, phi, lu_i, lu_j, dt, gamma_mode, inner)
    rdiff = np.concatenate([rhs[:nu], rhs[n: n + nu]])
    sol, rep = irk.gmres(
        lambda x: irk.block2x2_apply(eta, beta, phi, lu_i, lu_j, dt, x), rdiff, 2 * nu, pre, 2,
        rtol, maxit, restart)
    counters.differential += rep.precond_applications
    k1, k2 = sol[:nu], sol[nu:]
    c1 = ConstraintSolver(gw_i, counters)
    c2 = ConstraintSolver(gw_j, counters)
    l1 = -c1.solve(rhs[nu:n] + dt * (gu_i @ k1)) / dt
    l2 = -c2.solve(rhs[n + nu:] + dt * (gu_j @ k2)) / dt
    x = np.concatenate([k1, l1, k2, l2])

    def apply_full(x):
        x1u, x1w = x[:nu], x[nu:n]
        x2u, x2w = x[n: n + nu], x[n + nu:]
        top1 = eta * x1u - dt * (lu_i @ x1u) - dt * (lw_i @ x1w) + phi * x2u
        bot1 = -dt * (gu_i @ x1u) - dt * (gw_i @ x1w)
        top2 = eta * x2u - dt * (lu_j @ x2u) - dt * (lw_j @ x2w) - (beta**2 / phi) * x1u
        bot2 = -dt * (gu_j @ x2u) - dt * (gw_j @ x2w)
        return np.concatenate([top1, bot1, top2, bot2])

    rnorm = np.linalg.norm(rhs)
    if rnorm > 0.0:
        true_rel = np.linalg.norm(rhs - apply_full(x)) / rnorm
        if true_rel > rtol:
            raise irk.StageSolveError(
                f"composite block residual {true_rel:.3e} above rtol {rtol:.3e}", report=rep)
    return x, rep


def solve_dae_transformed(prep, diag, offdiag, dt, rhs, cfg, counters):
    """src/dae.py:336-420 for 2x2 eigen-blocks (reordered mode)."""
    s = prep.tableau.s
    nu = diag[0][0].shape[0]
    nw = diag[0][3].shape[0]
    n = nu + nw
    q, r0 = prep.q, prep.r
    g = q.T @ rhs
    y = np.zeros_like(g)
    stats = irk.SolveStats()
    for blk in reversed(prep.blocks):
        rows = list(range(blk.offset, blk.offset + blk.size))
        acc = g[rows].copy()
        for local, ri in enumerate(rows):
            for j in range(blk.offset + blk.size, s):
                coef = r0[ri, j]
                if coef != 0.0:
                    acc[local, :nu] -= coef * y[j, :nu]
                od = offdiag.get((ri, j))
                if od is not None:
                    xu, xw = y[j, :nu], y[j, nu:]
                    acc[local, :nu] += dt * (od[0] @ xu) + dt * (od[1] @ xw)
                    acc[local, nu:] += dt * (od[2] @ xu) + dt * (od[3] @ xw)
        if blk.size == 1:
            raise irk.OracleError("composite 1x1 blocks use exact reduced solves (src/dae.py:140)")
        sol, rep = solve_block4x4_reordered(
            diag[blk.offset], diag[blk.offset + 1], blk.eta, blk.beta, blk.phi, dt,
            np.concatenate([acc[0], acc[1]]), cfg.gamma_mode, cfg.inner, counters,
            cfg.krylov_rtol, cfg.krylov_maxit, cfg.restart)
        if not rep.converged:
            raise irk.StageSolveError(
                f"composite 2x2 block at offset {blk.offset} did not converge",
                block_offset=blk.offset, report=rep)
        y[rows[0]] = sol[:n]
        y[rows[1]] = sol[n:]
        stats.reports.append((blk.offset, rep))
    return (q @ r0) @ y, stats


def dae_newton_step(sys, u, w, k, ell, t, dt, prep, cfg):
    """src/dae.py:423-471 (reordered mode)."""
    tab = prep.tableau
    stats = DaeStepStats()
    counters = DaeCounters()
    tic = time.perf_counter()
    res = dae_stage_residual(sys, u, w, k, ell, t, dt, tab)
    f0 = np.linalg.norm(res)
    stats.residual_history.append(f0)
    tol = max(cfg.newton_rtol * f0, cfg.newton_abs_floor)
    ops = None
    nu = sys.dim_u
    while stats.newton_iterations < cfg.newton_maxit:
        if np.linalg.norm(res) <= tol:
            stats.converged = True
            break
        if ops is None or cfg.jacobian_refresh == "every":
            u_stage = u[None, :] + dt * (tab.a0 @ k)
            w_stage = w[None, :] + dt * (tab.a0 @ ell)
            ops = [sys.blocks(u_stage[i], w_stage[i], t + tab.c0[i] * dt) for i in range(tab.s)]
            stats.jacobian_assemblies += tab.s
            diag, offdiag = build_dae_variant(prep, ops, cfg.variant, cfg.variant0_stage)
        dx, sst = solve_dae_transformed(prep, diag, offdiag, dt, res, cfg, counters)
        k = k + dx[:, :nu]
        ell = ell + dx[:, nu:]
        stats.newton_iterations += 1
        stats.add_solve(sst)
        res = dae_stage_residual(sys, u, w, k, ell, t, dt, tab)
        stats.residual_history.append(np.linalg.norm(res))
    else:
        if np.linalg.norm(res) > tol:
            raise irk.StepFailureError("DAE stage solve stalled", stats=stats)
        stats.converged = True
    stats.wall_time = time.perf_counter() - tic
    stats.differential_solves = counters.differential
    stats.constraint_solves = counters.constraint
    return k, ell, stats


def dae_step(sys, u, w, t, dt, prep, cfg):
    """src/dae.py:474-498."""
    tab = prep.tableau
    k = np.zeros((tab.s, sys.dim_u))
    ell = np.zeros((tab.s, sys.dim_w))
    k, ell, stats = dae_newton_step(sys, u, w, k, ell, t, dt, prep, cfg)
    u_next = u + dt * (tab.b0 @ k)
    w_next = w + dt * (tab.b0 @ ell)
    stats.constraint_residual = float(np.linalg.norm(sys.constraint(u_next, w_next, t + dt)))
    return u_next, w_next, stats


def dae_integrate(sys, u0, w0, t0, t_final, dt, prep, cfg):
    """src/dae.py:520-564; returns (u_states, w_states, step_stats)."""
    g0 = np.linalg.norm(sys.constraint(np.asarray(u0, float), np.asarray(w0, float), t0))
    if g0 > 1e-10:
        raise irk.OracleError(f"inconsistent initial condition: |G(u0, w0, t0)| = {g0:.3e}")
    nsteps = int(round((t_final - t0) / dt))
    u = np.array(u0, dtype=float)
    w = np.array(w0, dtype=float)
    us, ws, sts = [u.copy()], [w.copy()], []
    for j in range(nsteps):
        u, w, st = dae_step(sys, u, w, t0 + j * dt, dt, prep, cfg)
        us.append(u.copy())
        ws.append(w.copy())
        sts.append(st)
    return us, ws, sts
