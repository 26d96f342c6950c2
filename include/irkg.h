/*
 * irkg.h -- C ABI of the B200 IRK stage-solve engine (libirkg.so).
 *
 * Drop-in boundary for the hot path of the reference package `irkit`
 * (paths relative to /root/reference/pkg/src/irkit).  The reference has no
 * FFI: its "plugin/operator API" is Python.  Each entry point
 * below replaces one reference function; the Python mirror
 * `paper_2101_01776_b200` binds them with ctypes.
 *
 * Conventions
 *  - plain pointers and sizes only; all vectors are fp64.
 *  - `*_dev` pointers are CUDA device pointers owned by the caller; stage
 *    arrays are (s, N) row-major (stage-major, C order), N = nx*ny*nz with x
 *    fastest -- the reference's layout (src/nonlinear.py:310, problems.py:238).
 *  - work is enqueued on the context's stream; calls return after the
 *    result is on the device (scalars / stats are copied back to the host).
 *  - return value: IRKG_OK or a negative IRKG_ERR_* code; the Python shim
 *    maps them to the reference exception types (src/errors.py:6-58) with the
 *    same payload fields.  irkg_last_error() gives a message.
 *  - one context per GPU / rank, not thread-safe per context.
 */
#ifndef IRKG_H
#define IRKG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IRKG_OK 0
#define IRKG_ERR_VALUE -1          /* ValueError (shape/domain, zero Jacobi diagonal) */
#define IRKG_ERR_CONFIG -2         /* ConfigurationError */
#define IRKG_ERR_STAGE_SOLVE -3    /* StageSolveError(block_offset, report) */
#define IRKG_ERR_STEP_FAILURE -4   /* StepFailureError(stats) */
#define IRKG_ERR_BREAKDOWN -5      /* KrylovBreakdownError */
#define IRKG_ERR_CUDA -6           /* CUDA / NCCL runtime failure */
#define IRKG_ERR_INDEX -7          /* IndexViolationError (singular constraint block) */
#define IRKG_ERR_SINGULAR -8       /* SingularMatrixError (exact inner solve: singular band) */

/* irkg_solver.inner: damped-Jacobi sweeps (> 0) or IRKG_INNER_EXACT for the
 * reference's default PrecondSpec(inner="exact") banded LU (1-D / 2-D, one rank) */
#define IRKG_INNER_EXACT 0
/* ... or IRKG_INNER_MG: one geometric-multigrid V-cycle per inner solve
 * (beyond the reference; 2-D grids, one rank) */
#define IRKG_INNER_MG -1

#define IRKG_MAX_STAGES 8
#define IRKG_MAX_NEWTON 512
#define IRKG_MAX_BLOCK_RECORDS 4096

/* Problem kinds (paper_2101_01776_b200/problems.py, csrc/kinds.cuh). */
#define IRKG_KIND_NLDIFF 0   /* N(u) = Lap_h(u + u^3/3) */
#define IRKG_KIND_BURGERS 1  /* N(u) = -Dsum(u^2/2) + nu Lap_h u */
#define IRKG_KIND_RAD 2      /* N(u) = nu Lap_h u + c Dsum u + lam u + mu u^2 */
#define IRKG_KIND_ARAKAWA 3  /* DAE: w_t = -J(psi,w) + nu Lap w, 0 = h^2(Lap psi + w) */

typedef struct irkg_ctx irkg_ctx;

/* Grid + problem plugin: replaces OdeSystem(dim, rhs, linearize)
 * (src/nonlinear.py:35-48) for the matrix-free stencil kinds.
 * rank/nranks describe the slab partition along the slowest axis
 * (ny_global split into contiguous slabs); nranks = 1 on one GPU. */
typedef struct {
  int kind;
  int nx, ny, nz;        /* global extents; 1 for absent axes */
  double length;         /* periodic box side per axis (h = length / n) */
  double nu, c, lam, mu; /* kind parameters */
  double length_y, length_z; /* per-axis box sides (0: same as length) */
} irkg_problem;

/* Prepared stage constants: ButcherTableau + StagePrep
 * (src/tableau.py:66-101, 364-379); consumed bit-exactly, never recomputed. */
typedef struct {
  int s;
  double a0[IRKG_MAX_STAGES * IRKG_MAX_STAGES];
  double b0[IRKG_MAX_STAGES];
  double c0[IRKG_MAX_STAGES];
  double q[IRKG_MAX_STAGES * IRKG_MAX_STAGES];
  double r[IRKG_MAX_STAGES * IRKG_MAX_STAGES];
  double d[IRKG_MAX_STAGES * IRKG_MAX_STAGES * IRKG_MAX_STAGES]; /* d[k][l][i] */
  int nblocks;
  int blk_offset[IRKG_MAX_STAGES];
  int blk_size[IRKG_MAX_STAGES];
  double blk_eta[IRKG_MAX_STAGES];
  double blk_beta[IRKG_MAX_STAGES];
  double blk_phi[IRKG_MAX_STAGES];
} irkg_tableau;

/* SolverConfig + PrecondSpec (src/nonlinear.py:61-83, src/irk_core.py:39-68). */
typedef struct {
  int variant;            /* 0..3 */
  double newton_rtol;
  int newton_maxit;
  double newton_abs_floor;
  double krylov_rtol;
  int krylov_maxit;
  int restart;
  int gamma_mode;         /* 0 = star, 1 = eta, 2 = custom */
  double gamma_custom;
  int inner;              /* Jacobi sweeps (>0), IRKG_INNER_EXACT (banded LU), IRKG_INNER_MG */
  int jacobian_refresh;   /* 0 = every, 1 = frozen */
  int variant0_stage;
} irkg_solver;

/* KrylovReport (src/sparsela.py:155-162); residuals into a caller buffer. */
typedef struct {
  int iterations;
  int converged;
  int precond_applications;
  int n_residuals;        /* entries written (may exceed capacity: truncated) */
  int residual_capacity;  /* set by caller */
  double *residuals;      /* host buffer, caller-owned (may be NULL) */
} irkg_krylov_report;

/* StepStats (src/nonlinear.py:155-179) plus the failure payload. */
typedef struct {
  int newton_iterations;
  int krylov_iterations;
  int precond_applications;
  int jacobian_assemblies;
  int converged;
  int n_residuals;
  double residual_history[IRKG_MAX_NEWTON + 1];
  int n_block_records;                      /* one per (Newton it, block) */
  int block_offset[IRKG_MAX_BLOCK_RECORDS]; /* in solve order */
  int block_iterations[IRKG_MAX_BLOCK_RECORDS];
  double wall_time;
  /* StageSolveError payload (valid when a call returned IRKG_ERR_STAGE_SOLVE) */
  int fail_block_offset;
  irkg_krylov_report fail_report;
  /* DAE paths (src/nonlinear.py:170-172 fields; zero on ODE paths) */
  int differential_solves;
  int constraint_solves;
  double constraint_residual;
} irkg_step_stats;

/* Engine counters since creation (bench.py: launches / algorithmic bytes). */
typedef struct {
  int64_t kernel_launches;
  int64_t arnoldi_iterations;
  double cgs_bytes;       /* algorithmic bytes moved by the CGS2 sweeps */
  double cgs_time_ms;     /* device time of the CGS2 sweeps (if timing on) */
  int64_t cgs_launches;
  double precond_bytes;
  double op_bytes;
  double precond_time_ms; /* device time of the inner solves (if timing on) */
  double op_time_ms;      /* device time of the block operator (if timing on) */
  int64_t halo_exchanges; /* slab-partition halo exchanges issued */
  /* with IRKG_GRAPH_TIMING=1 (one event pair per restart cycle): device time
   * of the Arnoldi-loop graphs of 1x1 / 2x2 blocks and of the cycle ends */
  double arnoldi_ms_1x1;
  double arnoldi_ms_2x2;
  double cycle_end_ms;
  /* ... and the device idle time across the host round trips: residual norm
   * read -> next Newton iteration, block solve end -> next block */
  double newton_gap_ms;
  double block_gap_ms;
} irkg_counters;

/* Host-callback transport for the slab partition (alternative to NCCL):
 * allreduce: in-place sum of `count` doubles at device pointer `dev`;
 * halo: send my first planes (send_lo) to rank-1 and my last (send_hi) to
 * rank+1 (periodic ring), receive rank+1's first into recv_hi and rank-1's
 * last into recv_lo; `count` doubles each.  Called with the stream drained;
 * must complete before returning. */
typedef void (*irkg_allreduce_fn)(void *user, double *dev, int count);
typedef void (*irkg_halo_fn)(void *user, const double *send_lo, const double *send_hi,
                             double *recv_lo, double *recv_hi, long long count);
/* alltoall: block p (`count` doubles) of `send` goes to rank p, block p of
 * `recv` arrives from rank p (device pointers; the slab -> pencil transposes
 * of the DAE constraint solve, replacing _ConstraintSolver.solve,
 * src/dae.py:108-126, across ranks). */
typedef void (*irkg_alltoall_fn)(void *user, const double *send, double *recv, long long count);

const char *irkg_last_error(void);
const char *irkg_version(void);

/* Context: owns the stream binding, workspaces (V basis sized by restart)
 * and the stage arrays.  `stream` is a cudaStream_t (0 = legacy default);
 * `nccl_id` (128 bytes) may be NULL when nranks == 1.
 * Replaces the per-call workspaces of gmres (src/sparsela.py:208-213). */
int irkg_create(irkg_ctx **out, const irkg_problem *prob, int device, void *stream,
                const void *nccl_id, int rank, int nranks);
/* Multi-rank context over host callbacks (nccl_id-free variant of irkg_create):
 * the slab partition is the same; only the transport differs. */
int irkg_create_callback(irkg_ctx **out, const irkg_problem *prob, int device, void *stream,
                         int rank, int nranks, irkg_allreduce_fn allreduce, irkg_halo_fn halo,
                         void *user);
/* All-to-all of a callback-transport context (same `user` as its other
 * callbacks); needed only by DAE contexts with nranks > 1. */
int irkg_set_alltoall_callback(irkg_ctx *ctx, irkg_alltoall_fn alltoall);
int irkg_destroy(irkg_ctx *ctx);
int irkg_get_local_extent(irkg_ctx *ctx, int *n_local, int *y0, int *ny_local);
int irkg_nccl_unique_id(void *out128);

int irkg_set_tableau(irkg_ctx *ctx, const irkg_tableau *tab);
int irkg_set_solver(irkg_ctx *ctx, const irkg_solver *cfg);
int irkg_set_timing(irkg_ctx *ctx, int on);
int irkg_get_counters(irkg_ctx *ctx, irkg_counters *out);
/* Diagnostics (no reference counterpart): average device time in us of one
 * hot-path phase replayed `reps` times on the state the last block solve left
 * (0 precond, 1/2 first/second Jacobi chain, 3 block operator, 6 CGS2 sweeps,
 * 7 index pin alone, 8 whole Arnoldi step, 10 x += V y).  Destroys the Krylov
 * state. */
int irkg_probe_phase(irkg_ctx *ctx, int phase, int j, int reps, double *us);

/* stage_residual (src/nonlinear.py:145-152): F = N(u + dt A0 K) - K.
 * u_dev (N), k_dev (s,N), f_dev (s,N) out; *norm = ||F||_F. */
int irkg_stage_residual(irkg_ctx *ctx, const double *u_dev, const double *k_dev, double t,
                        double dt, double *f_dev, double *norm);

/* newton_like_step (src/nonlinear.py:186-236): k_dev (s,N) in/out. */
int irkg_newton_step(irkg_ctx *ctx, const double *u_dev, double *k_dev, double t, double dt,
                     irkg_step_stats *stats);

/* step (src/nonlinear.py:299-314): u_dev (N) in/out, u <- u + dt b0^T K. */
int irkg_step(irkg_ctx *ctx, double *u_dev, double t, double dt, irkg_step_stats *stats);

/* _dirk_step (src/nonlinear.py:239-296), the stepper the reference's step()
 * uses for SDIRK tableaux (304-306): sequential stage solves, each a Newton
 * loop over 1x1 GMRES on (I - dt a_ii L) with the Jacobi-k ShiftedSolver.
 * The tableau comes through irkg_set_tableau with nblocks = 0 (a0 lower
 * triangular, b0, c0).  u_dev (N) in/out.  Block records are keyed by stage. */
int irkg_dirk_step(irkg_ctx *ctx, double *u_dev, double t, double dt, irkg_step_stats *stats);

/* Same as irkg_step with host buffers: H2D copy of u, step, D2H copy
 * (the end-to-end path timed by bench.py's e2e leg). */
int irkg_step_host(irkg_ctx *ctx, double *u_host, double t, double dt, irkg_step_stats *stats);

/* step() with the reference's value semantics on host arrays
 * (src/nonlinear.py:299-314 returns a new u_next and leaves u untouched):
 * H2D copy of u_host, step, D2H copy into u_next_host (may equal u_host).
 * Page-locked buffers make both copies DMA transfers. */
int irkg_step_host_out(irkg_ctx *ctx, const double *u_host, double *u_next_host, double t,
                       double dt, irkg_step_stats *stats);

/* ---- operator-level entry points (parity tests; src/irk_core.py) ----
 * An operator "field" is the coefficient field a (device, N) + scalar sigma
 * of the collapsed weighted linearisation sum_k w_k L_k (see problems.py). */
typedef struct {
  const double *a_dev; /* may be NULL for kinds whose L does not read a */
  double sigma;
} irkg_opfield;

/* linearize + combine (src/nonlinear.py:204-209, src/sparsela.py:106-128):
 * the operator field of sum_k w_k L(U_k) for m stage values U_dev (m,N):
 * a_out_dev (N) = sum_k w_k f(U_k), *sigma_out = sum_k w_k. */
int irkg_linearize(irkg_ctx *ctx, const double *U_dev, int m, const double *weights,
                   double *a_out_dev, double *sigma_out);

/* apply_block2x2 (src/irk_core.py:126-140): y = A x, x,y (2N). c12/c21 may be NULL. */
int irkg_block2x2_apply(irkg_ctx *ctx, double eta, double beta, double phi, double dt,
                        const irkg_opfield *l1, const irkg_opfield *l2,
                        const irkg_opfield *c12, const irkg_opfield *c21,
                        const double *x_dev, double *y_dev);

/* make_block2x2_preconditioner(...)(r) (src/irk_core.py:147-165), Jacobi-k inner. */
int irkg_block2x2_precond(irkg_ctx *ctx, double eta, double beta, double phi, double gamma,
                          double dt, int inner, const irkg_opfield *l1,
                          const irkg_opfield *l2, const double *r_dev, double *z_dev);

/* ShiftedSolver(alpha, I, L, dt, inner=k).solve(r) (src/irk_core.py:103-123). */
int irkg_shifted_solve(irkg_ctx *ctx, double alpha, double dt, int inner,
                       const irkg_opfield *l, const double *r_dev, double *x_dev);

/* gmres on one eigen-block system (src/sparsela.py:176-280 driving
 * src/irk_core.py:215-222 / 303-333): size 1 (eta*I - dt*L1, ShiftedSolver
 * preconditioner) or 2 (Block2x2System + block preconditioner).
 * rhs_dev, x_dev: size*N.  x0 = 0 (as every reference block solve). */
int irkg_block_gmres(irkg_ctx *ctx, int size, double eta, double beta, double phi,
                     double gamma, double dt, int inner, const irkg_opfield *l1,
                     const irkg_opfield *l2, const irkg_opfield *c12,
                     const irkg_opfield *c21, const double *rhs_dev, double *x_dev,
                     double rtol, int maxit, int restart, irkg_krylov_report *report);

/* solve_transformed_system (src/irk_core.py:225-338) at the linearisation
 * last set by irkg_newton_step / irkg_prepare_linearization.
 * rhs_dev (s,N) -> dk_dev (s,N); per-block records into stats. */
int irkg_prepare_linearization(irkg_ctx *ctx, const double *u_dev, const double *k_dev,
                               double dt);
int irkg_transformed_solve(irkg_ctx *ctx, double dt, const double *rhs_dev, double *dk_dev,
                           irkg_step_stats *stats);

/* solve_transformed_system(..., variant_jacobian=vj) (src/irk_core.py:225-237)
 * with a VariantJacobian (src/nonlinear.py:86-96) supplied by the caller
 * instead of irkg_prepare_linearization: `diag` holds the s diagonal
 * operators, (off_i[q], off_j[q]) -> off[q] the coupling operators; a field
 * with a_dev = NULL and sigma = 0 is a skipped (zero) key.  The fields are
 * copied; the next irkg_transformed_solve uses them. */
int irkg_set_variant_jacobian(irkg_ctx *ctx, const irkg_opfield *diag, int n_off,
                              const int *off_i, const int *off_j, const irkg_opfield *off);

/* y = L x for one operator field: the matvec of a stage operator / a
 * combine()d sum (SparseMatrix.__matmul__, src/sparsela.py:29-103). */
int irkg_operator_apply(irkg_ctx *ctx, const irkg_opfield *l, const double *x_dev,
                        double *y_dev);

/* OdeSystem.rhs (src/nonlinear.py:35-48): f = N(u, t) (autonomous kinds; one rank). */
int irkg_rhs(irkg_ctx *ctx, const double *u_dev, double t, double *f_dev);

/* Reverse-communication GMRES over a caller-supplied operator and right
 * preconditioner: the reference's gmres(op, rhs, right_precond, rtol, maxit,
 * restart, x0) (src/sparsela.py:176-280) with its LinearOperator plugin
 * (src/sparsela.py:131-152).  The engine runs the restarted Arnoldi process
 * (fused CGS2 sweeps, Givens, back-substitution, x += Z y with Z stored,
 * true-residual recheck) and returns to the caller for every operator
 * application: after irkg_rc_gmres_next() reports IRKG_RC_APPLY_PRECOND or
 * IRKG_RC_APPLY_OP, the caller writes M^{-1} vin (resp. A vin) into vout and
 * calls next() again; IRKG_RC_DONE ends the solve (x_dev holds x; the
 * report comes from irkg_rc_gmres_report).  All vectors are n doubles on the
 * device (n <= 2 * the context's N); x0_dev may be NULL (x0 = 0);
 * solves_per_apply = 0 means no preconditioner.  Breakdown with a residual
 * above rtol returns IRKG_ERR_BREAKDOWN from next(). */
#define IRKG_RC_DONE 0
#define IRKG_RC_APPLY_PRECOND 1
#define IRKG_RC_APPLY_OP 2
int irkg_rc_gmres_begin(irkg_ctx *ctx, long long n, const double *rhs_dev, const double *x0_dev,
                        double *x_dev, double *vin_dev, double *vout_dev, double rtol, int maxit,
                        int restart, int solves_per_apply);
int irkg_rc_gmres_next(irkg_ctx *ctx, int *action);
int irkg_rc_gmres_report(irkg_ctx *ctx, irkg_krylov_report *report);

/* ---- index-1 DAE (vorticity/streamfunction, IRKG_KIND_ARAKAWA) ----
 * State uw = [u; w] (2N: vorticity then streamfunction), stage arrays
 * (s, 2N) with rows [k_i; l_i] -- the reference's composite layout
 * (src/dae.py:98).  Reordered mode only (coupled mode hard-codes exact
 * differential solves, src/dae.py:140). */

/* dae_stage_residual (src/dae.py:94-105) */
int irkg_dae_stage_residual(irkg_ctx *ctx, const double *uw_dev, const double *k2_dev, double t,
                            double dt, double *f2_dev, double *norm);
/* dae_step (src/dae.py:474-498): uw_dev in/out; stats->constraint_residual set */
int irkg_dae_step(irkg_ctx *ctx, double *uw_dev, double t, double dt, irkg_step_stats *stats);
/* same with host buffers (H2D + step + D2H) */
int irkg_dae_step_host(irkg_ctx *ctx, double *uw_host, double t, double dt,
                       irkg_step_stats *stats);
/* ||G(u, w, t)||_2 -- the consistency check of dae_integrate (src/dae.py:527-531) */
int irkg_dae_constraint_norm(irkg_ctx *ctx, const double *uw_dev, double *norm);

#ifdef __cplusplus
}
#endif
#endif /* IRKG_H */
