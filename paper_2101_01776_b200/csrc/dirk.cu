// dirk.cu -- (S)DIRK baseline on the device: sequential stage solves.
//
// Restates the reference's _dirk_step (src/nonlinear.py:239-296), the
// stepper its step() routes SDIRK tableaux to (304-306): for stage i
//     base = u + dt sum_{j<i} a_ij k_j
//     Newton on  N(base + dt a_ii k_i) - k_i = 0  from k_i = 0, each
//     correction from right-preconditioned GMRES on (I - dt a_ii L) with the
//     ShiftedSolver(1, I, L, dt a_ii, inner) preconditioner,
// then u_next = u + dt b^T K.  The linear solves are this engine's 1x1 block
// GMRES (eta = 1, shift dt a_ii) with the same Jacobi chains, operator and
// CGS2 sweeps as the collocation path; only the outer control differs.
// As in the reference, a GMRES solve that stops short of rtol is not an
// error here (only breakdown is), and stalling Newton raises
// StepFailureError.
#include <chrono>
#include <cmath>
#include <cstdio>

#include "engine.h"

namespace irkg {

// out = u + dt * sum_{j < i} a_j K_j
__global__ void k_dirk_base(int n, int i, StageConsts A, double dt, const double *__restrict__ u,
                            const double *__restrict__ K, double *__restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < i; ++j) acc += A.v[j] * K[(size_t)j * n + p];
    out[p] = i ? u[p] + dt * acc : u[p];
  }
}

// U = base + h k  (stage value at the current iterate)
__global__ void k_dirk_stage(int n, double h, const double *__restrict__ base,
                             const double *__restrict__ k, double *__restrict__ U) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    U[p] = base[p] + h * k[p];
}

void Engine::dirk_step(double *u, double t, double dt, irkg_step_stats *stats) {
  (void)t;  // the supported problem kinds are autonomous
  for (int i = 0; i < s; ++i)
    for (int j = i + 1; j < s; ++j)
      if (tab.a0[i * IRKG_MAX_STAGES + j] != 0.0)
        throw SolveError(IRKG_ERR_CONFIG, "dirk_step needs a lower-triangular tableau");
  auto tic = std::chrono::steady_clock::now();
  double *base = DK;  // (row 0)
  double *dk = Y;     // GMRES correction (row 0)
  check(cudaMemsetAsync(Kst, 0, (size_t)s * N * sizeof(double), stream));
  // one operator slot: a = f(U), sigma = 1 (the stage's own linearisation)
  OpWeights w1{};
  w1.nops = 1;
  w1.s = 1;
  w1.w[0] = 1.0;
  if (nops_cap < 1) {
    dalloc_raw((void **)&opA, sizeof(double) * (size_t)N);
    nops_cap = 1;
  }
  const int gb = grid_for(N);
  stats->n_residuals = 0;
  for (int i = 0; i < s; ++i) {
    StageConsts A{};
    A.s = s;
    for (int j = 0; j < i; ++j) A.v[j] = tab.a0[i * IRKG_MAX_STAGES + j];
    k_dirk_base<<<gb, 256, 0, stream>>>((int)N, i, A, dt, u, Kst, base);
    count(1);
    const double aii = tab.a0[i * IRKG_MAX_STAGES + i];
    const double h = dt * aii;
    double *ki = Kst + (size_t)i * N;
    k_dirk_stage<<<gb, 256, 0, stream>>>((int)N, h, base, ki, U);
    count(1);
    double fn = std::sqrt(residual(U, ki, F, 1));
    if (stats->n_residuals <= IRKG_MAX_NEWTON) stats->residual_history[stats->n_residuals++] = fn;
    const double tol = std::max(cfg.newton_rtol * fn, cfg.newton_abs_floor);
    int it = 0;
    while (fn > tol) {
      if (it >= cfg.newton_maxit) {
        stats->wall_time =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - tic).count();
        char msg[96];
        snprintf(msg, sizeof msg, "DIRK stage %d stalled after %d iterations", i,
                 cfg.newton_maxit);
        throw SolveError(IRKG_ERR_STEP_FAILURE, msg);
      }
      opfields(U, w1, opA);  // L at the current stage value
      if (slab()) exchange(R_OP, opA, inhalo());
      stats->jacobian_assemblies += 1;
      BlockSpec B{};
      B.size = 1;
      B.eta = 1.0;
      B.dt = h;
      B.inner = cfg.inner;
      B.l1 = Op{opA, 1.0, 1};
      KrylovOut rep = gmres(B, F, dk, cfg.krylov_rtol, cfg.krylov_maxit, cfg.restart, false);
      axpy(N, 1.0, dk, ki);
      it += 1;
      stats->newton_iterations += 1;
      stats->krylov_iterations += rep.iterations;
      stats->precond_applications += rep.precond_applications;
      if (stats->n_block_records < IRKG_MAX_BLOCK_RECORDS) {
        stats->block_offset[stats->n_block_records] = i;  // keyed by stage
        stats->block_iterations[stats->n_block_records] = rep.iterations;
        stats->n_block_records++;
      }
      k_dirk_stage<<<gb, 256, 0, stream>>>((int)N, h, base, ki, U);
      count(1);
      fn = std::sqrt(residual(U, ki, F, 1));
      if (stats->n_residuals <= IRKG_MAX_NEWTON) stats->residual_history[stats->n_residuals++] = fn;
    }
  }
  step_update(dt, Kst, u);
  stats->converged = 1;
  stats->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - tic).count();
}

}  // namespace irkg
