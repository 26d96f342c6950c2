"""irkit-compatible solver entry points, running on the B200 engine.

Same names, argument meaning and error behaviour as the reference
(``/root/reference/pkg/src/irkit``):

* ``stage_residual``           src/nonlinear.py:145-152
* ``newton_like_step``         src/nonlinear.py:186-236
* ``step``                     src/nonlinear.py:299-314
* ``integrate``                src/nonlinear.py:331-374
* ``solve_transformed_system`` src/irk_core.py:225-338
* ``apply_block2x2`` / ``precond_block2x2`` / ``ShiftedSolver`` /
  ``block_gmres``              src/irk_core.py:71-165, src/sparsela.py:176-280

``sys`` is a :class:`~paper_2101_01776_b200.problems.GridProblem` (the
device-side analogue of ``OdeSystem``).  State arrays may be numpy arrays
(results come back as numpy, like the reference) or CUDA torch tensors
(results stay on the device).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import PrecondSpec, SolverConfig, inner_sweeps
from .engine import _raise, as_device, context_for, opfield, ptr, torch
from .errors import ConfigurationError, StepFailureError
from .stats import IntegrationResult, KrylovReport, SolveStats
from .tableau import SDIRK_FAMILIES, prepare_stages


def _check_sys(sys):
    if getattr(sys, "mass", None) is not None:
        raise ConfigurationError("the device engine supports identity mass only (M = I)")
    if not hasattr(sys, "kind"):
        raise ConfigurationError(
            "device solves need a GridProblem (paper_2101_01776_b200.problems); "
            "host-callable OdeSystems run on the reference"
        )


def problem_rhs(sys, u, t=0.0):
    """``OdeSystem.rhs`` of a GridProblem on the device (irkg_rhs)."""
    _check_sys(sys)
    ctx = context_for(sys)
    ud = as_device(u).reshape(-1)
    if ud.numel() != sys.dim:
        raise ValueError(f"u has {ud.numel()} entries, the system has {sys.dim}")
    f = torch().empty_like(ud)
    rc = ctx.lib.irkg_rhs(ctx.h, ptr(ud), float(t), ptr(f))
    if rc:
        _raise(rc)
    return _out(f, u)


def _is_torch(x):
    try:
        return isinstance(x, torch().Tensor)
    except ImportError:
        return False


def _pinned(n):
    """A numpy float64 view of ``n`` page-locked doubles from torch's caching
    host allocator: host<->device copies of step states run at full DMA speed
    and the block returns to the cache when the array dies (no per-step
    cudaHostAlloc)."""
    return torch().empty(int(n), dtype=torch().float64, pin_memory=True).numpy()


def _host_copy(x_dev):
    """Device vector -> new (pinned) numpy array."""
    out = _pinned(x_dev.numel()).reshape(tuple(x_dev.shape))
    torch().from_numpy(out).copy_(x_dev)
    return out


def _out(x_dev, like):
    if _is_torch(like):
        return x_dev
    return _host_copy(x_dev)


@dataclass
class StageState:
    """Current stage vectors and step context (src/nonlinear.py:51-58)."""

    k: object  # (s, dim)
    u: object
    t: float
    dt: float


def _sdirk_guard(tableau):
    if str(tableau.family) in SDIRK_FAMILIES:
        raise ConfigurationError(
            f"{tableau.family} is an SDIRK baseline (src/nonlinear.py:239-296), "
            "outside the device stage-solve path"
        )


def stage_residual(sys, st: StageState, tableau):
    """``N(u + dt * sum_j a_ij k_j, t + c_i dt) - k_i`` per stage."""
    _check_sys(sys)
    ctx = context_for(sys)
    ctx.set_prep(_prep_for(tableau))
    u = as_device(st.u)
    k = as_device(st.k).reshape(tableau.s, sys.dim)
    f = torch().empty_like(k)
    ctx.stage_residual(u, k, st.t, st.dt, f)
    return _out(f, st.k)


_PREP_CACHE = {}


def _prep_for(tableau, prep=None):
    if prep is not None:
        return prep
    key = (str(tableau.family), int(tableau.s), np.asarray(tableau.a0).tobytes())
    p = _PREP_CACHE.get(key)
    if p is None:
        p = prepare_stages(tableau)
        _PREP_CACHE[key] = p
    return p


def newton_like_step(sys, st: StageState, prep, cfg: SolverConfig):
    """Drive the stage vectors to the residual tolerance on the device.

    Returns ``(st, StepStats)`` with ``st.k`` rebound (not mutated), like the
    reference; exhausting ``newton_maxit`` raises StepFailureError(stats).
    """
    _check_sys(sys)
    _sdirk_guard(prep.tableau)
    ctx = context_for(sys)
    ctx.set_prep(prep)
    ctx.set_config(cfg)
    u = as_device(st.u)
    k = as_device(st.k).reshape(prep.tableau.s, sys.dim).clone()
    stats = ctx.newton(u, k, st.t, st.dt)
    st.k = _out(k, st.k)
    return st, stats


def step(sys, u, t, dt, tableau, cfg=SolverConfig(), prep=None):
    """Advance one step: solve the stages, then ``u + dt * sum b_i k_i``.

    Returns ``(u_next, StepStats)``.
    """
    _check_sys(sys)
    if str(tableau.family) in SDIRK_FAMILIES:  # src/nonlinear.py:304-306
        return _dirk_step(sys, u, t, dt, tableau, cfg)
    prep = _prep_for(tableau, prep)
    ctx = context_for(sys)
    ctx.set_prep(prep)
    ctx.set_config(cfg)
    if _is_torch(u):
        ud = as_device(u).clone()
        stats = ctx.step_device(ud, t, dt)
        return ud, stats
    # u_next lives in page-locked memory (and so does u when it came from a
    # previous step): both copies of irkg_step_host_out are DMA transfers
    uin = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
    if uin.size != sys.dim:
        raise ValueError(f"u has {uin.size} entries, the system has {sys.dim}")
    uh = _pinned(sys.dim)
    stats = ctx.step_host_out(uin, uh, t, dt)
    return uh, stats


def _dirk_step(sys, u, t, dt, tableau, cfg):
    """Sequential stage solves of an SDIRK tableau on the device
    (src/nonlinear.py:239-296): returns (u_next, StepStats) with
    ``block_iterations`` keyed by stage."""
    ctx = context_for(sys)
    ctx.set_dirk_tableau(tableau)
    ctx.set_config(cfg)
    if _is_torch(u):
        ud = as_device(u).clone()
        stats = ctx.dirk_step_device(ud, t, dt)
        return ud, stats
    ud = as_device(np.asarray(u, dtype=np.float64)).clone()
    stats = ctx.dirk_step_device(ud, t, dt)
    return _host_copy(ud), stats


def integrate(sys, u0, t0, t_final, dt, tableau, cfg=SolverConfig(), snapshot_every=None):
    """Fixed-step march from ``t0`` to ``t_final`` (src/nonlinear.py:331-374).

    The state stays resident on the device between steps; snapshots are
    copied back to the host.  The first failing step raises
    StepFailureError with ``partial`` attached.
    """
    _check_sys(sys)
    span = t_final - t0
    nsteps_f = span / dt
    nsteps = int(round(nsteps_f))
    if abs(nsteps_f - nsteps) > 1e-8 * max(1.0, abs(nsteps_f)):
        raise ConfigurationError(f"(t_final - t0)/dt = {nsteps_f} is not an integer step count")
    dirk = str(tableau.family) in SDIRK_FAMILIES  # prep = None (src/nonlinear.py:355)
    ctx = context_for(sys)
    if dirk:
        ctx.set_dirk_tableau(tableau)
    else:
        ctx.set_prep(_prep_for(tableau))
    ctx.set_config(cfg)
    advance = ctx.dirk_step_device if dirk else ctx.step_device
    on_dev = _is_torch(u0)
    u = as_device(u0).clone()
    host = (lambda x: x.clone()) if on_dev else (lambda x: x.cpu().numpy())
    times = [t0]
    states = [host(u)]
    step_stats = []
    for j in range(nsteps):
        t = t0 + j * dt
        try:
            stats = advance(u, t, dt)
        except StepFailureError as exc:
            exc.partial = IntegrationResult(times=np.array(times), states=states,
                                            step_stats=step_stats)
            raise
        step_stats.append(stats)
        keep = snapshot_every is None or ((j + 1) % snapshot_every == 0)
        if keep or j == nsteps - 1:
            times.append(t0 + (j + 1) * dt)
            states.append(host(u))
    return IntegrationResult(times=np.array(times), states=states, step_stats=step_stats)


# ------------------------------------------------------ operator level


class OperatorField:
    """A device linearisation ``sum_k w_k L(U_k)`` held as its coefficient
    field ``a`` (CUDA tensor, N) and weight sum ``sigma`` -- the engine's
    replacement for the CSR ``SparseMatrix`` returned by ``linearize`` and
    summed by ``combine`` (src/sparsela.py:106-128)."""

    def __init__(self, problem, a, sigma=1.0):
        self.problem = problem
        self.a = None if a is None else as_device(a)
        self.sigma = float(sigma)

    @classmethod
    def linearize(cls, problem, u_stages, weights=None):
        """Field of ``sum_k w_k L(U_k)`` for stage values ``u_stages`` (m, N)."""
        ctx = context_for(problem)
        U = as_device(u_stages)
        if U.dim() == 1:
            U = U.reshape(1, -1)
        if weights is None:
            weights = [1.0] + [0.0] * (U.shape[0] - 1)
        a, sig = ctx.linearize(U.contiguous(), weights)
        return cls(problem, a, sig)

    @property
    def n(self):
        return self.problem.dim

    def matvec(self, x):
        """``L x`` on the device (SparseMatrix.matvec, src/sparsela.py:29-103)."""
        xd = as_device(x)
        if tuple(xd.shape) != (self.n,):
            raise ValueError(f"x has shape {tuple(xd.shape)}, expected ({self.n},)")
        ctx = context_for(self.problem)
        y = torch().empty_like(xd)
        rc = ctx.lib.irkg_operator_apply(ctx.h, opfield(self), ptr(xd), ptr(y))
        if rc:
            _raise(rc)
        return _out(y, x)

    def __matmul__(self, x):
        return self.matvec(x)


def combine(coeffs, fields):
    """``sum_k c_k L_k`` of operator fields of one problem
    (src/sparsela.py:106-128): zero weights skipped, summed in order k = 0..,
    the same association the reference's CSR sum uses; None when every
    weight is zero (the reference's empty matrix)."""
    coeffs = [float(c) for c in coeffs]
    fields = list(fields)
    if len(coeffs) != len(fields):
        raise ValueError("coefficient / operator count mismatch")
    a, sig, prob = None, 0.0, None
    for c, f in zip(coeffs, fields):
        if c == 0.0:
            continue
        prob = f.problem
        term = None if f.a is None else c * f.a
        a = term if a is None else (a if term is None else a + term)
        sig += c * f.sigma
    if prob is None:
        return None
    return OperatorField(prob, a, sig)


def _opfield_value(f):
    """OperatorField (or None: a skipped, all-zero key) -> irkg_opfield value."""
    out = _lib.OpField()
    if f is None:
        out.a_dev = None
        out.sigma = 0.0
        return out
    if f.a is not None and not f.a.is_contiguous():
        f.a = f.a.contiguous()
    out.a_dev = C.c_void_p(f.a.data_ptr()) if f.a is not None else None
    out.sigma = float(f.sigma)
    return out


@dataclass
class VariantJacobian:
    """The variant's diagonal and coupling operators (src/nonlinear.py:86-96)
    as device operator fields: ``diag`` one per stage row, ``offdiag``
    keyed ``(i, j)``."""

    diag: tuple
    offdiag: dict


def variant_weights(prep, variant, variant0_stage=0):
    """Per-row stage weights and coupling weights of each variant
    (src/nonlinear.py:99-126): the same index logic (argmax |d_ii| first on
    ties, variant-3 keys i<j plus the sub-diagonal of every 2x2 block)."""
    s = prep.tableau.s
    d = np.asarray(prep.d, dtype=float)
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
    for blk in prep.schur.blocks:
        if blk.size == 2:
            i = blk.offset
            offdiag[(i + 1, i)] = d[i + 1, i]
    return diag, offdiag


def build_variant_jacobian(prep, stage_ops, variant, variant0_stage=0):
    """src/nonlinear.py:129-142 over device operator fields (one per stage,
    e.g. ``OperatorField.linearize(sys, U_i)`` or ``sys.linearize(U_i, t_i)``)."""
    stage_ops = list(stage_ops)
    s = prep.tableau.s
    if len(stage_ops) != s:
        raise ValueError(f"expected {s} stage operators, got {len(stage_ops)}")
    dw, ow = variant_weights(prep, variant, variant0_stage)
    diag = tuple(combine(dw[i], stage_ops) for i in range(s))
    offdiag = {key: combine(w, stage_ops) for key, w in ow.items()}
    return VariantJacobian(diag=diag, offdiag=offdiag)


@dataclass(frozen=True)
class Block2x2System:
    """One complex eigen-block system (src/irk_core.py:71-95), identity mass."""

    eta: float
    beta: float
    phi: float
    mass: object
    l1: OperatorField
    l2: OperatorField
    dt: float
    offdiag12: OperatorField = None
    offdiag21: OperatorField = None

    @property
    def n(self):
        return self.l1.problem.dim


def apply_block2x2(sys2: Block2x2System, x):
    """Matrix action of the 2x2 eigen-block system on ``x`` (length 2n)."""
    n = sys2.n
    xd = as_device(x)
    if tuple(xd.shape) != (2 * n,):
        raise ValueError(f"x has shape {tuple(xd.shape)}, expected ({2 * n},)")
    ctx = context_for(sys2.l1.problem)
    y = torch().empty_like(xd)
    rc = ctx.lib.irkg_block2x2_apply(
        ctx.h, sys2.eta, sys2.beta, sys2.phi, sys2.dt, opfield(sys2.l1), opfield(sys2.l2),
        opfield(sys2.offdiag12), opfield(sys2.offdiag21), ptr(xd), ptr(y))
    if rc:
        _raise(rc)
    return _out(y, x)


def precond_block2x2(sys2: Block2x2System, spec: PrecondSpec, r):
    """One application of the block lower-triangular preconditioner."""
    rd = as_device(r)
    ctx = context_for(sys2.l1.problem)
    z = torch().empty_like(rd)
    rc = ctx.lib.irkg_block2x2_precond(
        ctx.h, sys2.eta, sys2.beta, sys2.phi, spec.gamma(sys2.eta, sys2.beta), sys2.dt,
        inner_sweeps(spec), opfield(sys2.l1), opfield(sys2.l2), ptr(rd), ptr(z))
    if rc:
        _raise(rc)
    return _out(z, r)


class ShiftedSolver:
    """Applies ``(alpha*I - dt*L)^{-1}`` exactly (banded LU + SMW, the
    reference default) or by k damped-Jacobi sweeps (src/irk_core.py:103-123)."""

    def __init__(self, alpha, mass, lmat: OperatorField, dt, inner="exact"):
        if mass is not None:
            raise ConfigurationError("identity mass only")
        self.alpha = float(alpha)
        self.lmat = lmat
        self.dt = float(dt)
        self.inner = inner_sweeps(PrecondSpec(inner=inner))

    def solve(self, r):
        rd = as_device(r)
        ctx = context_for(self.lmat.problem)
        x = torch().empty_like(rd)
        rc = ctx.lib.irkg_shifted_solve(ctx.h, self.alpha, self.dt, self.inner,
                                        opfield(self.lmat), ptr(rd), ptr(x))
        if rc:
            _raise(rc)
        return _out(x, r)


def block_gmres(sys2, rhs, spec=PrecondSpec(inner=4), rtol=1e-5, maxit=200, restart=200):
    """GMRES on one eigen-block with its reference preconditioner.

    ``sys2`` is a Block2x2System (block preconditioner, src/irk_core.py:
    303-333) or a ``(eta, OperatorField, dt)`` tuple for a 1x1 block
    (``_solve_1x1``, src/irk_core.py:215-222).  Returns ``(x, KrylovReport)``.
    """
    rd = as_device(rhs)
    if isinstance(sys2, Block2x2System):
        size, eta, beta, phi, dt = 2, sys2.eta, sys2.beta, sys2.phi, sys2.dt
        l1, l2, c12, c21 = sys2.l1, sys2.l2, sys2.offdiag12, sys2.offdiag21
        gamma = spec.gamma(eta, beta)
    else:
        eta, l1, dt = sys2
        size, beta, phi, gamma, l2, c12, c21 = 1, 0.0, 1.0, float(eta), None, None, None
    n = l1.problem.dim
    if tuple(rd.shape) != (size * n,):
        raise ValueError(f"rhs has shape {tuple(rd.shape)}, expected ({size * n},)")
    ctx = context_for(l1.problem)
    x = torch().empty_like(rd)
    res = (C.c_double * (int(maxit) + 4))()
    rep = _lib.KrylovReportC()
    rep.residuals = C.cast(res, C.POINTER(C.c_double))
    rep.residual_capacity = len(res)
    rc = ctx.lib.irkg_block_gmres(
        ctx.h, size, float(eta), float(beta), float(phi), float(gamma), float(dt),
        inner_sweeps(spec), opfield(l1), opfield(l2), opfield(c12), opfield(c21), ptr(rd),
        ptr(x), float(rtol), int(maxit), int(restart), C.byref(rep))
    if rc:
        _raise(rc)
    report = KrylovReport(int(rep.iterations), bool(rep.converged),
                          list(res[: min(rep.n_residuals, len(res))]),
                          int(rep.precond_applications))
    return _out(x, rhs), report


class LinearOperator:
    """Abstract linear action ``y = A x`` of dimension ``n`` on the device
    (src/sparsela.py:131-152): ``apply`` maps a CUDA float64 tensor (n,) to
    one; ``solves_per_apply`` is the preconditioner-work unit the Krylov
    report counts (src/sparsela.py:192, 278)."""

    def __init__(self, n, apply, solves_per_apply=1):
        self.n = int(n)
        self._apply = apply
        self.solves_per_apply = solves_per_apply

    def __call__(self, x):
        return self._apply(x)

    def matvec(self, x):
        return self._apply(x)


def _as_device_apply(op):
    """src/sparsela.py:165-173 for device operands: a LinearOperator, an
    OperatorField, or a dense square matrix (numpy or CUDA tensor)."""
    if isinstance(op, LinearOperator):
        return op.n, op.matvec
    if isinstance(op, OperatorField):
        return op.n, op.matvec
    t = torch()
    if isinstance(op, t.Tensor) or isinstance(op, np.ndarray):
        a = as_device(op)
        if a.dim() == 2 and a.shape[0] == a.shape[1]:
            return int(a.shape[0]), (lambda x: a @ x)
    raise TypeError(f"cannot interpret {type(op)!r} as a linear operator")


_RC_HOSTS = {}


def gmres(op, rhs, right_precond=None, rtol=1e-5, maxit=200, restart=200, x0=None):
    """Restarted right-preconditioned GMRES over a caller's operator
    (src/sparsela.py:176-280): the engine runs the Arnoldi process (fused
    CGS2 sweeps, Givens, back-substitution, the true-residual recheck, Z
    stored) and calls back ``op`` / ``right_precond`` on CUDA tensors
    through the reverse-communication C entries (irkg_rc_gmres_*).
    Returns ``(x, KrylovReport)``; breakdown above rtol raises
    KrylovBreakdownError."""
    n, apply_op = _as_device_apply(op)
    t = torch()
    b = as_device(rhs).reshape(-1)
    if tuple(b.shape) != (n,):
        raise ValueError(f"rhs has shape {tuple(b.shape)}, expected ({n},)")
    if not (0.0 < rtol < 1.0):
        raise ValueError(f"rtol must lie in (0, 1), got {rtol}")
    spa = 0
    apply_m = None
    if right_precond is not None:
        spa = int(getattr(right_precond, "solves_per_apply", 1))
        apply_m = right_precond.matvec if hasattr(right_precond, "matvec") else right_precond
    b = b.contiguous()
    if float(t.linalg.vector_norm(b)) == 0.0:  # src/sparsela.py:196-198
        return _out(t.zeros_like(b), rhs), KrylovReport(0, True, [0.0], 0)
    key = (n, t.cuda.current_device())
    host = _RC_HOSTS.get(key)
    if host is None:
        from .problems import GridProblem

        host = _RC_HOSTS[key] = GridProblem("rad", (n,), name=f"krylov{n}")
    ctx = context_for(host)
    x = t.empty_like(b)
    vin, vout = t.empty_like(b), t.empty_like(b)
    xd = None if x0 is None else as_device(x0).reshape(-1).contiguous()
    rc = ctx.lib.irkg_rc_gmres_begin(ctx.h, n, ptr(b), ptr(xd) if xd is not None else None,
                                     ptr(x), ptr(vin), ptr(vout), float(rtol), int(maxit),
                                     int(restart), spa)
    if rc:
        _raise(rc)
    act = C.c_int()
    while True:
        rc = ctx.lib.irkg_rc_gmres_next(ctx.h, C.byref(act))
        if rc:
            _raise(rc)
        if act.value == 0:
            break
        y = apply_m(vin) if act.value == 1 else apply_op(vin)
        vout.copy_(as_device(y).reshape(-1))
    res = (C.c_double * (int(maxit) + 4))()
    rep = _lib.KrylovReportC()
    rep.residuals = C.cast(res, C.POINTER(C.c_double))
    rep.residual_capacity = len(res)
    rc = ctx.lib.irkg_rc_gmres_report(ctx.h, C.byref(rep))
    if rc:
        _raise(rc)
    report = KrylovReport(int(rep.iterations), bool(rep.converged),
                          list(res[: min(rep.n_residuals, len(res))]),
                          int(rep.precond_applications))
    return _out(x, rhs), report


class StageLinearization:
    """The s stage linearisations of ``sys`` at ``u + dt A0 K`` -- the device
    analogue of the ``stage_ops`` list of CSR matrices the reference passes
    to ``solve_transformed_system``."""

    def __init__(self, sys, u, k, dt):
        self.sys = sys
        self.u = as_device(u)
        self.k = as_device(k)
        self.dt = float(dt)


def solve_transformed_system(prep, stage_ops=None, variant=None, dt=None, rhs_stages=None,
                             mass=None, precond=PrecondSpec(inner=4), krylov_rtol=1e-5,
                             krylov_maxit=200, restart=200, variant_jacobian=None):
    """Solve one linearised stage system through the Schur transform.

    The operators come as in the reference (src/irk_core.py:225-237): either
    ``variant_jacobian`` (a :class:`VariantJacobian` of operator fields, e.g.
    from :func:`build_variant_jacobian`), or ``stage_ops`` + ``variant`` with
    ``stage_ops`` a list of s :class:`OperatorField` (the device analogue of
    the list of CSR stage operators) or a :class:`StageLinearization` (stage
    values; the fields are formed on the device).  Returns ``(k,
    SolveStats)``; a non-convergent block solve raises
    StageSolveError(block_offset, report).
    """
    if mass is not None:
        raise ConfigurationError("identity mass only")
    if dt is None or dt <= 0.0:
        raise ValueError("dt must be positive")
    s = prep.tableau.s
    rhs = as_device(rhs_stages)
    if rhs.shape[0] != s:
        raise ValueError(f"rhs has {rhs.shape[0]} stage rows, expected {s}")
    if variant_jacobian is None and not isinstance(stage_ops, StageLinearization):
        if stage_ops is None or variant is None:
            raise ValueError("need variant_jacobian or stage_ops with variant")
        variant_jacobian = build_variant_jacobian(prep, stage_ops, variant)
    cfg = SolverConfig(variant=3 if variant is None else variant, krylov_rtol=krylov_rtol,
                       krylov_maxit=krylov_maxit, restart=restart, precond=precond)
    if variant_jacobian is not None:
        vj = variant_jacobian
        if len(vj.diag) != s:
            raise ValueError(f"variant_jacobian has {len(vj.diag)} diagonal operators, "
                             f"expected {s}")
        present = [f for f in list(vj.diag) + list(vj.offdiag.values()) if f is not None]
        if not present:
            raise ValueError("variant_jacobian has no operators")
        ctx = context_for(present[0].problem)
        ctx.set_prep(prep)
        ctx.set_config(cfg)
        keys = list(vj.offdiag.items())
        diag = (_lib.OpField * s)(*[_opfield_value(f) for f in vj.diag])
        off = (_lib.OpField * max(1, len(keys)))(*[_opfield_value(f) for _, f in keys])
        oi = (C.c_int * max(1, len(keys)))(*[int(k[0]) for k, _ in keys])
        oj = (C.c_int * max(1, len(keys)))(*[int(k[1]) for k, _ in keys])
        rc = ctx.lib.irkg_set_variant_jacobian(ctx.h, diag, len(keys), oi, oj, off)
        if rc:
            _raise(rc)
    else:
        lin = stage_ops
        ctx = context_for(lin.sys)
        ctx.set_prep(prep)
        ctx.set_config(cfg)
        ctx.prepare_linearization(lin.u, lin.k.reshape(s, -1), lin.dt)
    dk = torch().empty_like(rhs)
    st = ctx.transformed_solve(dt, rhs.contiguous(), dk)
    stats = SolveStats()
    for i in range(st.n_block_records):
        its = int(st.block_iterations[i])
        size = 2 if any(b.offset == st.block_offset[i] and b.size == 2 for b in prep.blocks) else 1
        stats.reports.append(
            (int(st.block_offset[i]), KrylovReport(its, True, [], its * size)))
    return _out(dk, rhs_stages), stats


# ------------------------------------------------------------------ DAE


@dataclass
class DaeIntegrationResult:
    """src/dae.py:501-517."""

    times: np.ndarray
    u_states: list
    w_states: list
    step_stats: list

    @property
    def u_final(self):
        return self.u_states[-1]

    @property
    def w_final(self):
        return self.w_states[-1]

    def total(self, attr):
        return sum(getattr(s, attr) for s in self.step_stats)


def _check_dae(sys, mode):
    if getattr(sys, "kind", None) != "arakawa":
        raise ConfigurationError("device DAE solves need a VorticityProblem (problems.py)")
    if mode != "reordered":
        raise ConfigurationError(
            "only mode='reordered' runs on the device: the reference's coupled mode hard-codes "
            "exact differential solves (src/dae.py:140) and ignores PrecondSpec.inner"
        )


def dae_step(sys, u, w, t, dt, tableau, cfg=SolverConfig(), prep=None, mode="reordered"):
    """One DAE step (src/dae.py:474-498); returns ``(u_next, w_next, StepStats)``."""
    _check_dae(sys, mode)
    if str(tableau.family) in SDIRK_FAMILIES:
        raise ConfigurationError(
            "DIRK tableaux are not supported on DAE systems; use a fully implicit "
            "collocation scheme")
    prep = _prep_for(tableau, prep)
    ctx = context_for(sys)
    ctx.set_prep(prep)
    ctx.set_config(cfg)
    n = sys.dim_u
    if _is_torch(u):
        uw = torch().cat([as_device(u), as_device(w)]).contiguous()
        stats = ctx.dae_step_device(uw, t, dt)
        return uw[:n].clone(), uw[n:].clone(), stats
    uw = _pinned(n + sys.dim_w)
    uw[:n] = np.asarray(u, float).reshape(-1)
    uw[n:] = np.asarray(w, float).reshape(-1)
    stats = ctx.dae_step_host(uw, t, dt)
    return uw[:n], uw[n:], stats


def dae_integrate(sys, u0, w0, t0, t_final, dt, tableau, cfg=SolverConfig(), mode="reordered"):
    """Fixed-step DAE march (src/dae.py:520-564) with the device-resident state.

    The initial state must satisfy the constraint to 1e-10 (ConfigurationError
    otherwise); a failing step raises StepFailureError with ``partial``.
    """
    _check_dae(sys, mode)
    prep = _prep_for(tableau)
    ctx = context_for(sys)
    ctx.set_prep(prep)
    ctx.set_config(cfg)
    n = sys.dim_u
    uw = torch().cat([as_device(u0), as_device(w0)]).contiguous()
    g0 = ctx.dae_constraint_norm(uw)
    if g0 > 1e-10:
        raise ConfigurationError(f"inconsistent initial condition: |G(u0, w0, t0)| = {g0:.3e}")
    span = t_final - t0
    nsteps_f = span / dt
    nsteps = int(round(nsteps_f))
    if abs(nsteps_f - nsteps) > 1e-8 * max(1.0, abs(nsteps_f)):
        raise ConfigurationError(f"(t_final - t0)/dt = {nsteps_f} is not an integer step count")
    if str(tableau.family) in SDIRK_FAMILIES:
        raise ConfigurationError("DIRK tableaux are not supported on DAE systems")
    on_dev = _is_torch(u0)
    host = (lambda x: x.clone()) if on_dev else (lambda x: x.cpu().numpy())
    times, us, ws, sts = [t0], [host(uw[:n])], [host(uw[n:])], []
    for j in range(nsteps):
        try:
            st = ctx.dae_step_device(uw, t0 + j * dt, dt)
        except StepFailureError as exc:
            exc.partial = DaeIntegrationResult(np.array(times), us, ws, sts)
            raise
        sts.append(st)
        times.append(t0 + (j + 1) * dt)
        us.append(host(uw[:n]))
        ws.append(host(uw[n:]))
    return DaeIntegrationResult(np.array(times), us, ws, sts)
