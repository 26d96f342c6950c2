"""Device context: one libirkg context per (problem, device, stream).

Wraps the C ABI (include/irkg.h) and maps its status codes onto the
reference's exception types (src/errors.py).  Device memory for the
caller-facing arrays is PyTorch's (plumbing only); the compute is the
CUDA engine.  There is no CPU path: construction fails loudly without the
shared library or a CUDA device.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .config import gamma_code, inner_sweeps
from .errors import (
    SingularMatrixError,
    ConfigurationError,
    IndexViolationError,
    KrylovBreakdownError,
    StageSolveError,
    StepFailureError,
)
from .problems import KIND_CODE
from .stats import KrylovReport, step_stats_from_c

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t

        _torch = _t
    return _torch


def _raise(rc, stats_c=None, fail_res=None):
    msg = _lib.last_error()
    if rc == _lib.ERR_VALUE:
        raise ValueError(msg)
    if rc == _lib.ERR_CONFIG:
        raise ConfigurationError(msg)
    if rc == _lib.ERR_STAGE_SOLVE:
        rep = None
        off = None
        if stats_c is not None:
            fr = stats_c.fail_report
            n = min(fr.n_residuals, fr.residual_capacity)
            res = list(fail_res[:n]) if fail_res is not None else []
            rep = KrylovReport(int(fr.iterations), bool(fr.converged), res,
                               int(fr.precond_applications))
            off = int(stats_c.fail_block_offset)
        raise StageSolveError(msg, block_offset=off, report=rep)
    if rc == _lib.ERR_STEP_FAILURE:
        st = step_stats_from_c(stats_c) if stats_c is not None else None
        raise StepFailureError(msg, stats=st)
    if rc == _lib.ERR_BREAKDOWN:
        raise KrylovBreakdownError(msg)
    if rc == _lib.ERR_INDEX:
        raise IndexViolationError(msg)
    if rc == _lib.ERR_SINGULAR:
        raise SingularMatrixError(msg)
    raise RuntimeError(f"irkg CUDA failure: {msg}")


def as_device(x, dtype=None):
    """numpy / torch -> contiguous float64 CUDA tensor (no copy if already one)."""
    t = torch()
    if isinstance(x, t.Tensor):
        if not x.is_cuda:
            x = x.cuda()
        return x.to(t.float64).contiguous()
    return t.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def ptr(t):
    return C.c_void_p(t.data_ptr())


def dirk_tableau_struct(tab):
    """An SDIRK ButcherTableau as irkg_tableau: coefficients only, nblocks = 0."""
    s = int(tab.s)
    S = _lib.MAX_STAGES
    if s > S:
        raise ConfigurationError(f"s = {s} exceeds {S}")
    out = _lib.Tableau()
    out.s = s
    a0 = np.asarray(tab.a0, dtype=float)
    for i in range(s):
        out.b0[i] = float(tab.b0[i])
        out.c0[i] = float(tab.c0[i])
        for j in range(s):
            out.a0[i * S + j] = a0[i, j]
    out.nblocks = 0
    return out


def tableau_struct(prep):
    """Pack a (reference or mirror) StagePrep into the C irkg_tableau."""
    tab = prep.tableau
    s = int(tab.s)
    S = _lib.MAX_STAGES
    if s > S:
        raise ConfigurationError(f"s = {s} exceeds {S}")
    out = _lib.Tableau()
    out.s = s
    a0 = np.asarray(tab.a0, dtype=float)
    q = np.asarray(prep.schur.q, dtype=float)
    r = np.asarray(prep.schur.r, dtype=float)
    d = np.asarray(prep.d, dtype=float)
    for i in range(s):
        out.b0[i] = float(tab.b0[i])
        out.c0[i] = float(tab.c0[i])
        for j in range(s):
            out.a0[i * S + j] = a0[i, j]
            out.q[i * S + j] = q[i, j]
            out.r[i * S + j] = r[i, j]
            for k in range(s):
                out.d[(i * S + j) * S + k] = d[i, j, k]
    blocks = list(prep.schur.blocks)
    out.nblocks = len(blocks)
    for b, blk in enumerate(blocks):
        out.blk_offset[b] = int(blk.offset)
        out.blk_size[b] = int(blk.size)
        out.blk_eta[b] = float(blk.eta)
        out.blk_beta[b] = float(blk.beta)
        out.blk_phi[b] = float(blk.phi)
    return out


def problem_struct(problem):
    """Pack a GridProblem / VorticityProblem into the C irkg_problem."""
    shape = tuple(problem.shape) + (1,) * (3 - len(problem.shape))
    p = _lib.Problem()
    p.kind = KIND_CODE[problem.kind]
    p.nx, p.ny, p.nz = (int(x) for x in shape)
    box = getattr(problem, "box", None) or (problem.length,) * len(problem.shape)
    box = tuple(box) + (problem.length,) * (3 - len(box))
    p.length = float(box[0])
    p.length_y = float(box[1])
    p.length_z = float(box[2])
    p.nu = float(problem.nu)
    p.c = float(problem.c)
    p.lam = float(problem.lam)
    p.mu = float(problem.mu)
    return p


def solver_struct(cfg):
    out = _lib.Solver()
    out.variant = int(cfg.variant)
    out.newton_rtol = float(cfg.newton_rtol)
    out.newton_maxit = int(cfg.newton_maxit)
    out.newton_abs_floor = float(cfg.newton_abs_floor)
    out.krylov_rtol = float(cfg.krylov_rtol)
    out.krylov_maxit = int(cfg.krylov_maxit)
    out.restart = int(cfg.restart)
    gm, gc = gamma_code(cfg.precond)
    out.gamma_mode = gm
    out.gamma_custom = gc
    out.inner = inner_sweeps(cfg.precond)
    out.jacobian_refresh = 0 if cfg.jacobian_refresh == "every" else 1
    out.variant0_stage = int(cfg.variant0_stage)
    return out


class Context:
    """One engine context bound to a grid problem, a CUDA device and stream."""

    def __init__(self, problem, device=None):
        t = torch()
        if not t.cuda.is_available():
            raise RuntimeError("paper_2101_01776_b200 needs a CUDA device (no CPU fallback)")
        self.lib = _lib.load()
        self.problem = problem
        dev = t.cuda.current_device() if device is None else int(device)
        self.device = dev
        self.stream = t.cuda.current_stream(dev)
        p = problem_struct(problem)
        h = C.c_void_p()
        rc = self.lib.irkg_create(C.byref(h), C.byref(p), dev,
                                  C.c_void_p(self.stream.cuda_stream), None, 0, 1)
        if rc != 0:
            _raise(rc)
        self.h = h
        self.n = int(problem.dim)
        self._prep_key = None
        self._cfg_key = None
        self._fail_res = None

    def close(self):
        if getattr(self, "h", None) is not None:
            self.lib.irkg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ config
    def set_prep(self, prep):
        key = id(prep)
        if key == self._prep_key:
            return
        ts = tableau_struct(prep)
        rc = self.lib.irkg_set_tableau(self.h, C.byref(ts))
        if rc != 0:
            _raise(rc)
        self._prep_key = key
        self._prep_ref = prep

    def set_dirk_tableau(self, tab):
        key = ("dirk", str(tab.family), np.asarray(tab.a0, dtype=float).tobytes())
        if key == self._prep_key:
            return
        ts = dirk_tableau_struct(tab)
        rc = self.lib.irkg_set_tableau(self.h, C.byref(ts))
        if rc != 0:
            _raise(rc)
        self._prep_key = key
        self._prep_ref = tab

    def dirk_step_device(self, u_dev, t, dt):
        """_dirk_step (src/nonlinear.py:239-296) on a device state, in place."""
        st = self._new_stats()
        rc = self.lib.irkg_dirk_step(self.h, ptr(u_dev), float(t), float(dt), C.byref(st))
        self._check(rc, st)
        return step_stats_from_c(st)

    def set_config(self, cfg):
        key = (cfg.variant, cfg.newton_rtol, cfg.newton_maxit, cfg.newton_abs_floor,
               cfg.krylov_rtol, cfg.krylov_maxit, cfg.restart, cfg.precond.gamma_mode,
               cfg.precond.inner, cfg.jacobian_refresh, cfg.variant0_stage)
        if key == self._cfg_key:
            return
        ss = solver_struct(cfg)
        rc = self.lib.irkg_set_solver(self.h, C.byref(ss))
        if rc != 0:
            _raise(rc)
        self._cfg_key = key
        self._fail_res = (C.c_double * (int(cfg.krylov_maxit) + 4))()

    def set_timing(self, on):
        self.lib.irkg_set_timing(self.h, 1 if on else 0)

    def counters(self):
        c = _lib.Counters()
        self.lib.irkg_get_counters(self.h, C.byref(c))
        return {f: getattr(c, f) for f, _ in _lib.Counters._fields_}

    def _new_stats(self):
        st = _lib.StepStatsC()
        if self._fail_res is not None:
            st.fail_report.residuals = C.cast(self._fail_res, C.POINTER(C.c_double))
            st.fail_report.residual_capacity = len(self._fail_res)
        return st

    def _check(self, rc, st=None):
        if rc != 0:
            _raise(rc, st, self._fail_res)

    # ----------------------------------------------------------- solves
    def step_device(self, u_dev, t, dt):
        st = self._new_stats()
        rc = self.lib.irkg_step(self.h, ptr(u_dev), float(t), float(dt), C.byref(st))
        self._check(rc, st)
        return step_stats_from_c(st)

    def step_host(self, u_host, t, dt):
        """u_host: C-contiguous float64 numpy array, updated in place."""
        st = self._new_stats()
        rc = self.lib.irkg_step_host(self.h, u_host.ctypes.data_as(C.c_void_p), float(t),
                                     float(dt), C.byref(st))
        self._check(rc, st)
        return step_stats_from_c(st)

    def step_host_out(self, u_host, u_next_host, t, dt):
        """u_host -> u_next_host (C-contiguous float64 numpy arrays; u_host untouched)."""
        st = self._new_stats()
        rc = self.lib.irkg_step_host_out(self.h, u_host.ctypes.data_as(C.c_void_p),
                                         u_next_host.ctypes.data_as(C.c_void_p), float(t),
                                         float(dt), C.byref(st))
        self._check(rc, st)
        return step_stats_from_c(st)

    def newton(self, u_dev, k_dev, t, dt):
        st = self._new_stats()
        rc = self.lib.irkg_newton_step(self.h, ptr(u_dev), ptr(k_dev), float(t), float(dt),
                                       C.byref(st))
        self._check(rc, st)
        return step_stats_from_c(st)

    def stage_residual(self, u_dev, k_dev, t, dt, f_dev):
        nrm = C.c_double()
        rc = self.lib.irkg_stage_residual(self.h, ptr(u_dev), ptr(k_dev), float(t), float(dt),
                                          ptr(f_dev), C.byref(nrm))
        self._check(rc)
        return float(nrm.value)

    def prepare_linearization(self, u_dev, k_dev, dt):
        rc = self.lib.irkg_prepare_linearization(self.h, ptr(u_dev), ptr(k_dev), float(dt))
        self._check(rc)

    def transformed_solve(self, dt, rhs_dev, dk_dev):
        st = self._new_stats()
        rc = self.lib.irkg_transformed_solve(self.h, float(dt), ptr(rhs_dev), ptr(dk_dev),
                                             C.byref(st))
        self._check(rc, st)
        return st

    # ------------------------------------------------------------- DAE
    def dae_step_device(self, uw_dev, t, dt):
        st = self._new_stats()
        rc = self.lib.irkg_dae_step(self.h, ptr(uw_dev), float(t), float(dt), C.byref(st))
        self._check(rc, st)
        return step_stats_from_c(st)

    def dae_step_host(self, uw_host, t, dt):
        st = self._new_stats()
        rc = self.lib.irkg_dae_step_host(self.h, uw_host.ctypes.data_as(C.c_void_p), float(t),
                                         float(dt), C.byref(st))
        self._check(rc, st)
        return step_stats_from_c(st)

    def dae_constraint_norm(self, uw_dev):
        nrm = C.c_double()
        rc = self.lib.irkg_dae_constraint_norm(self.h, ptr(uw_dev), C.byref(nrm))
        self._check(rc)
        return float(nrm.value)

    def dae_stage_residual(self, uw_dev, k2_dev, t, dt, f2_dev):
        nrm = C.c_double()
        rc = self.lib.irkg_dae_stage_residual(self.h, ptr(uw_dev), ptr(k2_dev), float(t),
                                              float(dt), ptr(f2_dev), C.byref(nrm))
        self._check(rc)
        return float(nrm.value)

    def linearize(self, U_dev, weights):
        m = U_dev.shape[0]
        w = (C.c_double * m)(*[float(x) for x in weights])
        a = torch().empty(self.n, dtype=torch().float64, device=U_dev.device)
        sig = C.c_double()
        rc = self.lib.irkg_linearize(self.h, ptr(U_dev), m, w, ptr(a), C.byref(sig))
        self._check(rc)
        return a, float(sig.value)


def opfield(op):
    """OperatorField -> C struct (None stays None)."""
    if op is None:
        return None
    f = _lib.OpField()
    f.a_dev = C.c_void_p(op.a.data_ptr()) if op.a is not None else None
    f.sigma = float(op.sigma)
    return C.byref(f)


_CONTEXTS = {}


def context_for(problem, device=None):
    t = torch()
    dev = t.cuda.current_device() if device is None else int(device)
    key = (problem, dev, t.cuda.current_stream(dev).cuda_stream)
    ctx = _CONTEXTS.get(key)
    if ctx is None:
        if len(_CONTEXTS) >= 8:
            old = next(iter(_CONTEXTS))
            _CONTEXTS.pop(old).close()
        ctx = Context(problem, dev)
        _CONTEXTS[key] = ctx
    return ctx


def release_contexts():
    while _CONTEXTS:
        _CONTEXTS.popitem()[1].close()
