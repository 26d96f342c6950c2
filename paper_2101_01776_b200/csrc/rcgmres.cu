// rcgmres.cu -- reverse-communication GMRES: the reference's generic
// gmres(op, rhs, right_precond, rtol, maxit, restart, x0)
// (src/sparsela.py:176-280) over a caller-supplied operator and right
// preconditioner (its LinearOperator plugin, src/sparsela.py:131-152).
//
// The engine owns everything of the Krylov solve that is the same for every
// operator -- the basis V, the fused CGS2 sweeps + Hessenberg/Givens finish
// (cgs.cu), the back-substitution, x += Z y, the true-residual recheck and
// the restart logic -- and hands the two operator applications back to the
// caller: irkg_rc_gmres_next() returns APPLY_PRECOND / APPLY_OP with the
// input vector in the caller's `vin` buffer and expects the result in `vout`
// before the next call.  Unlike the block solves (engine.cu, which apply the
// fixed Jacobi-k preconditioner a second time at the cycle end), the
// preconditioned basis Z is stored, as the reference stores it, since a
// caller's preconditioner need not be a fixed linear map (flexible GMRES).
#include "engine.h"

namespace irkg {

namespace {

// V slot j materialised: out = alpha_j * s_j
__global__ void k_rc_slot(int n, const double *__restrict__ V, long long pitch, int j,
                          const double *__restrict__ alpha, double *__restrict__ out) {
  const double a = alpha[j];
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    out[r] = a * V[(size_t)j * pitch + r];
}

// out = b - ax
__global__ void k_rc_sub(int n, const double *__restrict__ b, const double *__restrict__ ax,
                         double *__restrict__ out) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    out[r] = b[r] - ax[r];
}

// control block of a solve with an initial guess (src/sparsela.py:194-204):
// bnorm = ||b||, beta = ||b - A x0||, residuals[0] = beta / bnorm
__global__ void k_rc_init(GWork W, const double *bn2, const double *rn2, int maxit, double rtol) {
  GCtrl *c = W.ctrl;
  const double bnorm = sqrt(*bn2);
  const double beta = rn2 ? sqrt(*rn2) : bnorm;
  GCtrl z{};
  z.maxit = maxit;
  z.rtol = rtol;
  z.bnorm = bnorm;
  z.beta = beta;
  z.n_res = 1;
  const double r0 = bnorm == 0.0 ? 0.0 : beta / bnorm;
  z.converged = (bnorm == 0.0 || r0 <= rtol) ? 1 : 0;
  *c = z;
  W.res[0] = r0;
}

__global__ void k_rc_set_rr(GCtrl *c, const double *rr) { c->rr = *rr; }

// x += sum_{l<k} y_l z_l  (src/sparsela.py:262, z stored: flexible GMRES)
__global__ void k_rc_zupdate(int n, const double *__restrict__ Z, const GCtrl *ctrl,
                             const double *__restrict__ y, double *__restrict__ x) {
  const int k = ctrl->k;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double a0 = 0.0, a1 = 0.0;
    int l = 0;
    for (; l + 2 <= k; l += 2) {
      a0 += Z[(size_t)l * n + r] * y[l];
      a1 += Z[(size_t)(l + 1) * n + r] * y[l + 1];
    }
    if (l < k) a0 += Z[(size_t)l * n + r] * y[l];
    x[r] = x[r] + (a0 + a1);
  }
}

}  // namespace

void Engine::rc_copy(double *dst, const double *src, long long n) {
  check(cudaMemcpyAsync(dst, src, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice, stream),
        "rc copy");
}

void Engine::rc_begin(long long n, const double *b, const double *x0, double *x, double *vin,
                      double *vout, double rtol, int maxit, int restart, int spa) {
  if (!(rtol > 0.0 && rtol < 1.0)) throw SolveError(IRKG_ERR_VALUE, "rtol must lie in (0, 1)");
  if (n < 1 || n > 2 * N) throw SolveError(IRKG_ERR_VALUE, "vector length exceeds the context");
  if (restart < 1) throw SolveError(IRKG_ERR_VALUE, "restart must be positive");
  if (slab()) throw SolveError(IRKG_ERR_CONFIG, "reverse-communication GMRES: one rank only");
  ensure_basis(restart);
  ensure_res(maxit);
  if (rc.zcap < restart) {
    dalloc_raw((void **)&rc.Z, (size_t)restart * (size_t)n * sizeof(double));
    rc.zcap = restart;
    rc.zn = n;
  } else if (rc.zn != n) {
    dalloc_raw((void **)&rc.Z, (size_t)rc.zcap * (size_t)n * sizeof(double));
    rc.zn = n;
  }
  rc.active = true;
  rc.n = n;
  rc.b = b;
  rc.x = x;
  rc.vin = vin;
  rc.vout = vout;
  rc.rtol = rtol;
  rc.maxit = maxit;
  rc.restart = restart;
  rc.spa = spa;
  rc.j = 0;
  rc.its = 0;
  // ||b||^2 -> scal_dev[1] (kept there across the caller's applications); x = x0 or 0
  norm2_dev(b, n);
  check(cudaMemcpyAsync(&scal_dev[1], &scal_dev[0], sizeof(double), cudaMemcpyDeviceToDevice,
                        stream), "rc scal");
  if (x0) {
    if (x0 != x) rc_copy(x, x0, n);
    rc_copy(vin, x, n);
    rc.phase = RC_R0;  // the caller applies A to x0 first
  } else {
    check(cudaMemsetAsync(x, 0, (size_t)n * sizeof(double), stream), "rc x0");
    rc_copy(V, b, n);
    k_rc_init<<<1, 1, 0, stream>>>(W, &scal_dev[1], nullptr, maxit, rtol);
    count(1);
    rc.phase = RC_CYCLE;
  }
}

int Engine::rc_next() {
  if (!rc.active) throw SolveError(IRKG_ERR_CONFIG, "no reverse-communication solve in progress");
  const long long n = rc.n;
  const int gb = grid_for(n);
  for (;;) {
    switch (rc.phase) {
      case RC_R0:  // caller: vin = x0 -> A x0 (return to it)
        rc.phase = RC_R0_DONE;
        return IRKG_RC_APPLY_OP;
      case RC_R0_DONE: {
        k_rc_sub<<<gb, 256, 0, stream>>>((int)n, rc.b, rc.vout, V);  // r0 into slot 0
        norm2_dev(V, n);  // ||r0||^2 -> scal_dev[0]; ||b||^2 is in scal_dev[1]
        k_rc_init<<<1, 1, 0, stream>>>(W, &scal_dev[1], &scal_dev[0], rc.maxit, rc.rtol);
        count(2);
        rc.phase = RC_CYCLE;
        break;
      }
      case RC_CYCLE: {
        read_ctrl();
        if (ctrl_host->converged || ctrl_host->total_it >= rc.maxit) {
          rc.phase = RC_DONE;
          break;
        }
        const int m = std::min(rc.restart, rc.maxit - ctrl_host->total_it);
        cycle_init(m);
        rc.j = 0;
        rc.phase = RC_PREC;
        break;
      }
      case RC_PREC: {  // vin = v_j
        k_rc_slot<<<gb, 256, 0, stream>>>((int)n, V, vpitch, rc.j, W.alpha, rc.vin);
        count(1);
        if (rc.spa == 0) {  // no preconditioner: z_j = v_j
          rc_copy(rc.Z + (size_t)rc.j * n, rc.vin, n);
          rc.phase = RC_OP;
          break;
        }
        rc.phase = RC_PREC_DONE;
        return IRKG_RC_APPLY_PRECOND;
      }
      case RC_PREC_DONE:
        rc_copy(rc.Z + (size_t)rc.j * n, rc.vout, n);
        rc.phase = RC_OP;
        break;
      case RC_OP:
        rc_copy(rc.vin, rc.Z + (size_t)rc.j * n, n);
        rc.phase = RC_OP_DONE;
        return IRKG_RC_APPLY_OP;
      case RC_OP_DONE: {
        rc_copy(wbuf, rc.vout, n);
        cgs(n);  // CGS2 + Hessenberg column / Givens / exit test (cgs.cu)
        counters.arnoldi_iterations += 1;
        read_ctrl();
        if (ctrl_host->cycle_done) {
          rc.phase = RC_CYCLE_END;
        } else {
          rc.j = ctrl_host->j;
          rc.phase = RC_PREC;
        }
        break;
      }
      case RC_CYCLE_END:
        // x += Z y (src/sparsela.py:258-262), then the true residual
        backsolve();
        k_rc_zupdate<<<gb, 256, 0, stream>>>((int)n, rc.Z, ctrl_dev, W.y, rc.x);
        count(1);
        rc_copy(rc.vin, rc.x, n);
        rc.phase = RC_RESID;
        return IRKG_RC_APPLY_OP;
      case RC_RESID: {  // r = b - A x into slot 0, its norm -> rr
        k_rc_sub<<<gb, 256, 0, stream>>>((int)n, rc.b, rc.vout, V);
        norm2_dev(V, n);
        k_rc_set_rr<<<1, 1, 0, stream>>>(ctrl_dev, &scal_dev[0]);
        count(2);
        cycle_end();
        read_ctrl();
        if (ctrl_host->err_breakdown) {
          rc.active = false;
          char msg[160];
          snprintf(msg, sizeof msg, "Arnoldi breakdown with residual %.3e above rtol %.3e",
                   std::sqrt(ctrl_host->rr) / ctrl_host->bnorm, rc.rtol);
          throw SolveError(IRKG_ERR_BREAKDOWN, msg);
        }
        rc.phase = RC_CYCLE;
        break;
      }
      case RC_DONE:
      default:
        rc.active = false;
        rc.phase = RC_DONE;
        return IRKG_RC_DONE;
    }
  }
}

void Engine::rc_report(irkg_krylov_report *rep) {
  read_ctrl();
  rep->iterations = ctrl_host->total_it;
  rep->converged = ctrl_host->converged;
  rep->precond_applications = ctrl_host->total_it * rc.spa;
  const int nres = ctrl_host->n_res;
  rep->n_residuals = nres;
  if (rep->residuals && rep->residual_capacity > 0) {
    const int k = std::min(nres, rep->residual_capacity);
    check(cudaMemcpyAsync(rep->residuals, W.res, (size_t)k * sizeof(double),
                          cudaMemcpyDeviceToHost, stream), "rc residuals");
    check(cudaStreamSynchronize(stream), "sync");
  }
}

}  // namespace irkg
