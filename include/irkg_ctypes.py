"""Reference-side ctypes binding of ``include/irkg.h`` (the stub INTEGRATION.md
documents, kept as a runnable file so a test executes it exactly as written).

A maintainer who wants irkit itself to hand its hot path to the B200 engine
drops this file next to ``irkit/nonlinear.py`` and calls ``step_on_gpu``
where ``step`` (src/nonlinear.py:299-314) would run.  It needs only ctypes
and numpy -- none of ``paper_2101_01776_b200`` -- and takes irkit's own
``StagePrep`` (src/tableau.py:84-101) and ``SolverConfig``
(src/nonlinear.py:61-83) objects.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

MAX_STAGES = 8          # IRKG_MAX_STAGES
MAX_NEWTON = 512        # IRKG_MAX_NEWTON
MAX_BLOCK_RECORDS = 4096  # IRKG_MAX_BLOCK_RECORDS
KINDS = {"nldiff": 0, "burgers": 1, "rad": 2, "arakawa": 3}  # IRKG_KIND_*
INNER_EXACT, INNER_MG = 0, -1


class Problem(C.Structure):          # irkg_problem
    _fields_ = [("kind", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("length", C.c_double), ("nu", C.c_double), ("c", C.c_double),
                ("lam", C.c_double), ("mu", C.c_double),
                ("length_y", C.c_double), ("length_z", C.c_double)]


class Tableau(C.Structure):          # irkg_tableau
    _S = MAX_STAGES
    _fields_ = [("s", C.c_int), ("a0", C.c_double * (_S * _S)), ("b0", C.c_double * _S),
                ("c0", C.c_double * _S), ("q", C.c_double * (_S * _S)),
                ("r", C.c_double * (_S * _S)), ("d", C.c_double * (_S * _S * _S)),
                ("nblocks", C.c_int), ("blk_offset", C.c_int * _S), ("blk_size", C.c_int * _S),
                ("blk_eta", C.c_double * _S), ("blk_beta", C.c_double * _S),
                ("blk_phi", C.c_double * _S)]


class Solver(C.Structure):           # irkg_solver
    _fields_ = [("variant", C.c_int), ("newton_rtol", C.c_double), ("newton_maxit", C.c_int),
                ("newton_abs_floor", C.c_double), ("krylov_rtol", C.c_double),
                ("krylov_maxit", C.c_int), ("restart", C.c_int), ("gamma_mode", C.c_int),
                ("gamma_custom", C.c_double), ("inner", C.c_int),
                ("jacobian_refresh", C.c_int), ("variant0_stage", C.c_int)]


class KrylovReport(C.Structure):     # irkg_krylov_report
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int),
                ("precond_applications", C.c_int), ("n_residuals", C.c_int),
                ("residual_capacity", C.c_int), ("residuals", C.POINTER(C.c_double))]


class StepStats(C.Structure):        # irkg_step_stats
    _fields_ = [("newton_iterations", C.c_int), ("krylov_iterations", C.c_int),
                ("precond_applications", C.c_int), ("jacobian_assemblies", C.c_int),
                ("converged", C.c_int), ("n_residuals", C.c_int),
                ("residual_history", C.c_double * (MAX_NEWTON + 1)),
                ("n_block_records", C.c_int),
                ("block_offset", C.c_int * MAX_BLOCK_RECORDS),
                ("block_iterations", C.c_int * MAX_BLOCK_RECORDS),
                ("wall_time", C.c_double), ("fail_block_offset", C.c_int),
                ("fail_report", KrylovReport), ("differential_solves", C.c_int),
                ("constraint_solves", C.c_int), ("constraint_residual", C.c_double)]


def load(path="libirkg.so"):
    lib = C.CDLL(path)
    vp, dp, ip = C.c_void_p, C.c_double, C.c_int
    lib.irkg_last_error.restype = C.c_char_p
    lib.irkg_create.argtypes = [C.POINTER(vp), C.POINTER(Problem), ip, vp, vp, ip, ip]
    lib.irkg_destroy.argtypes = [vp]
    lib.irkg_set_tableau.argtypes = [vp, C.POINTER(Tableau)]
    lib.irkg_set_solver.argtypes = [vp, C.POINTER(Solver)]
    lib.irkg_step_host_out.argtypes = [vp, vp, vp, dp, dp, C.POINTER(StepStats)]
    return lib


def pack_tableau(prep):
    """irkit StagePrep -> irkg_tableau (constants copied bit-exactly)."""
    S, tab, out = MAX_STAGES, prep.tableau, Tableau()
    s = out.s = int(tab.s)
    a0, q, r, d = (np.asarray(x, dtype=np.float64)
                   for x in (tab.a0, prep.schur.q, prep.schur.r, prep.d))
    for i in range(s):
        out.b0[i], out.c0[i] = float(tab.b0[i]), float(tab.c0[i])
        for j in range(s):
            out.a0[i * S + j], out.q[i * S + j], out.r[i * S + j] = a0[i, j], q[i, j], r[i, j]
            for k in range(s):
                out.d[(i * S + j) * S + k] = d[i, j, k]
    blocks = list(prep.schur.blocks)
    out.nblocks = len(blocks)
    for b, blk in enumerate(blocks):
        out.blk_offset[b], out.blk_size[b] = int(blk.offset), int(blk.size)
        out.blk_eta[b], out.blk_beta[b], out.blk_phi[b] = (float(blk.eta), float(blk.beta),
                                                           float(blk.phi))
    return out


def pack_solver(cfg):
    """irkit SolverConfig + PrecondSpec -> irkg_solver."""
    pc, out = cfg.precond, Solver()
    out.variant, out.newton_rtol, out.newton_maxit = int(cfg.variant), cfg.newton_rtol, int(
        cfg.newton_maxit)
    out.newton_abs_floor = float(getattr(cfg, "newton_abs_floor", 1e-14))
    out.krylov_rtol, out.krylov_maxit, out.restart = (cfg.krylov_rtol, int(cfg.krylov_maxit),
                                                      int(cfg.restart))
    gm = pc.gamma_mode              # "star" | "eta" | a positive float (custom)
    out.gamma_mode = {"star": 0, "eta": 1}.get(gm, 2) if isinstance(gm, str) else 2
    out.gamma_custom = 0.0 if isinstance(gm, str) else float(gm)
    out.inner = INNER_EXACT if pc.inner == "exact" else (INNER_MG if pc.inner == "mg"
                                                        else int(pc.inner))
    out.jacobian_refresh = 0 if cfg.jacobian_refresh == "every" else 1
    out.variant0_stage = int(cfg.variant0_stage)
    return out


def step_on_gpu(lib, kind, shape, params, u, t, dt, prep, cfg, device=0):
    """irkit.step() on the device: returns (u_next, StepStats); u untouched."""
    nx, ny, nz = (tuple(shape) + (1, 1))[:3]
    p = Problem(KINDS[kind], nx, ny, nz, params.get("length", 1.0), params.get("nu", 0.0),
                params.get("c", 0.0), params.get("lam", 0.0), params.get("mu", 0.0),
                0.0, 0.0)                      # length_y/z = 0: same as length
    ctx = C.c_void_p()
    if lib.irkg_create(C.byref(ctx), C.byref(p), device, None, None, 0, 1) != 0:
        raise RuntimeError(lib.irkg_last_error().decode())
    try:
        tab, sol, stats = pack_tableau(prep), pack_solver(cfg), StepStats()
        for rc in (lib.irkg_set_tableau(ctx, C.byref(tab)), lib.irkg_set_solver(ctx, C.byref(sol))):
            if rc != 0:
                raise RuntimeError(lib.irkg_last_error().decode())
        uh = np.ascontiguousarray(u, dtype=np.float64)
        un = np.empty_like(uh)    # irkit's step() returns a new array, u untouched
        rc = lib.irkg_step_host_out(ctx, uh.ctypes.data, un.ctypes.data, float(t), float(dt),
                                    C.byref(stats))
        if rc == -3:   # IRKG_ERR_STAGE_SOLVE -> irkit.errors.StageSolveError(block_offset, ...)
            raise RuntimeError(f"StageSolveError at block {stats.fail_block_offset}: "
                               f"{lib.irkg_last_error().decode()}")
        if rc == -4:   # IRKG_ERR_STEP_FAILURE -> irkit.errors.StepFailureError(stats=...)
            raise RuntimeError(f"StepFailureError: {lib.irkg_last_error().decode()}")
        if rc != 0:
            raise RuntimeError(lib.irkg_last_error().decode())
        return un, stats
    finally:
        lib.irkg_destroy(ctx)
