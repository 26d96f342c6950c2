// kernels.cuh -- fp64 device kernels of the IRK stage solve (sm_100a).
//
// All kernels are HBM-bound (<1 flop/byte); none is a dense
// contraction, so there is no tensor-core work here.  Design rules:
//  * coalesced, x-fastest streaming over the N local points;
//  * the s x s Butcher / Schur mixes are register-level matvecs fused into
//    the pointwise passes (north star (2));
//  * reductions are deterministic: per-CTA partials, then the last CTA to
//    finish (atomic ticket) folds them in fixed CTA order -- no fp atomics;
//  * Krylov-loop kernels read the Arnoldi index j and the cycle state from a
//    device-resident control block, so an iteration is a fixed launch
//    sequence (graph-capturable, no host round trip for scalars).
#pragma once
#include <cuda_runtime.h>

#include "kinds.cuh"

namespace irkg {

// Programmatic dependent launch (PDL).  Kernels of the Arnoldi body are
// launched with programmatic stream serialisation: a kernel may start while
// its predecessor drains.  Convention: every PDL kernel calls pdl_wait()
// before touching anything its predecessor writes, and pdl_trigger() only
// after its own pdl_wait(), so the code before pdl_wait() may read anything
// written two or more launches back.  (No-ops for ordinary launches.)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

constexpr int MAXS = 8;       // max stages
constexpr int MAXR = 256;     // max restart length
constexpr int MAXOPS = 48;    // max operator fields per linearisation
constexpr double OMEGA = 2.0 / 3.0;  // damped-Jacobi weight, src/irk_core.py:123

struct Op {
  const double *a;
  double sigma;
  int present;
  const double *alo = nullptr;  // ghost planes of a (slab mode)
  const double *ahi = nullptr;
};

__device__ __forceinline__ FRef fref(const Op &o) { return FRef{o.a, o.alo, o.ahi}; }

// Device-resident GMRES control block (src/sparsela.py:206-272 state).
struct GCtrl {
  int j;            // Arnoldi index within the current cycle
  int m;            // current cycle length
  int k;            // columns to assemble at cycle end
  int total_it;
  int maxit;
  int cycle_done;   // Arnoldi loop of this cycle finished
  int breakdown;
  int converged;
  int err_breakdown;  // KrylovBreakdownError to raise
  int n_res;          // residual history length
  int zero_diag;      // Jacobi met a zero diagonal
  int pad_;
  double bnorm, beta, rtol;
  double wn2;   // ||w||^2 before orthogonalisation
  double hn2;   // ||w||^2 after CGS2
  double rr;    // ||r||^2 at cycle end
  double scalar;  // generic reduction output
};

// Workspace pointers of one Krylov solve
struct GWork {
  GCtrl *ctrl;
  double *H;      // (MAXR+1) x MAXR, column j at H + j*(MAXR+1)
  double *cs, *sn, *g, *alpha, *y;
  double *c1, *c2;
  double *res;    // residual history (maxit + 2)
};

struct StageConsts {
  int s;
  double a[MAXS * MAXS];  // generic s x s matrix (row-major)
  double v[MAXS];         // generic vector
};

struct OpWeights {
  int nops;
  int s;
  double w[MAXOPS * MAXS];
};

// back-substitution terms for one eigen-block (src/irk_core.py:273-283)
struct BacksubTerms {
  int rows;      // 1 or 2
  int row0;      // first stage row of the block
  int njs;       // number of later stages
  int j[MAXS];
  double coef[2][MAXS];   // R0[r, j]
  Op od[2][MAXS];         // variant-3 coupling operators (present flag)
  const double *ylo[MAXS];  // ghost planes of y_j (slab mode)
  const double *yhi[MAXS];
};

// Resolve the input vector of a preconditioner: a fixed pointer, or the
// basis slot j of the control block scaled by alpha[j] (v_j = alpha_j s_j).
struct VecIn {
  const double *base;
  long long pitch;   // slot pitch when ctrl != null
  const GCtrl *ctrl; // if set: base + j*pitch, scale alpha[j]
  const double *alpha;
  const double *scale_ptr = nullptr;       // fixed-pointer input scaled by *scale_ptr
  const double *lo[2] = {nullptr, nullptr};  // ghost planes of the two halves (slab mode)
  const double *hi[2] = {nullptr, nullptr};
};

// ghost planes of the s stage fields (slab mode; unused otherwise)
struct StageGhosts {
  const double *lo[MAXS];
  const double *hi[MAXS];
};

// Input of an inner solve: basis slot j of the control block scaled by
// alpha[j] (v_j = alpha_j s_j), or a fixed pointer (scaled by *scale_ptr);
// returns the half selected by in_off together with its ghost planes.
__device__ __forceinline__ FRef vin_resolve(const VecIn &vi, int in_off, double &scale) {
  const double *p;
  if (vi.ctrl) {
    const int j = vi.ctrl->j;
    p = vi.base + (size_t)j * vi.pitch;
    scale = vi.alpha[j];
  } else {
    p = vi.base;
    scale = vi.scale_ptr ? *vi.scale_ptr : 1.0;
  }
  const int h = in_off ? 1 : 0;
  return FRef{p + in_off, vi.lo[h], vi.hi[h]};
}

}  // namespace irkg
