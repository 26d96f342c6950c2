// mg.cu -- geometric-multigrid inner solves: PrecondSpec(inner="mg").
//
// the paper preconditions each (gamma M - dt L) with one
// AMG/AIR iteration; the reference substitutes damped
// Jacobi (src/irk_core.py:103-123).  This mode replaces the inner solve by
// ONE V-cycle of cell-centred geometric multigrid on the periodic grid:
//   level l: S_l = alpha I - dt L(a_l, sigma) rediscretised with h_l = 2^l h
//            and a_l the 2x2 cell average of a_{l-1};
//   pre-smoothing  nu1 = 2 damped-Jacobi sweeps (omega = 2/3) from zero,
//   residual restricted by 2x2 averaging, coarse correction prolonged
//   bilinearly, post-smoothing nu2 = 2 sweeps;
//   coarsest level (<= 64 points, normally 8x8): exact banded LU + SMW
//   (banded.cu) -- the sequential band substitutions make a large coarsest
//   level the V-cycle's latency floor.
// Every piece is a fixed linear map, so the V-cycle is a fixed linear
// preconditioner: right-preconditioned GMRES, and x += M^{-1}(V y) at the
// cycle end, stay valid.  Beyond reference parity (the reference has no MG):
// pinned by the oracle's restatement (oracle/mg.py), not by reference goldens.
// 2-D grids, one rank.
#include <algorithm>

#include "engine.h"

namespace irkg {

constexpr int MG_COARSE = 64;  // coarsen while a level has more points than this

namespace {

__device__ __forceinline__ void nbr2d(const Grid &g, int p, int nb[4]) {
  const int nx = g.nx, ix = p % nx, iy = p / nx;
  nb[0] = p + (ix == 0 ? nx - 1 : -1);
  nb[1] = p + (ix == nx - 1 ? 1 - nx : 1);
  nb[2] = p + (iy == 0 ? (g.ny - 1) * nx : -nx);
  nb[3] = p + (iy == g.ny - 1 ? -(g.ny - 1) * nx : nx);
}

// (S x)(p) and the diagonal of S = alpha I - dt L(a, sigma)
template <int KIND>
__device__ __forceinline__ double apply_s(const Grid &g, const KindParams &kp,
                                          const double *__restrict__ a, double sig, double alpha,
                                          double dt, const double *__restrict__ x, int p,
                                          double &diag) {
  int nb[4];
  nbr2d(g, p, nb);
  double cc, cn[4];
  stencil_row<KIND>(g, kp, a, sig, p, nb, cc, cn);
  diag = alpha - dt * cc;
  double lx = cc * x[p];
#pragma unroll
  for (int k = 0; k < 4; ++k) lx += cn[k] * x[nb[k]];
  return alpha * x[p] - dt * lx;
}

}  // namespace

// one damped-Jacobi sweep: xout = xin + omega D^{-1} (b - S xin)  (xin == null: 0)
template <int KIND>
__global__ void k_mg_sweep(Grid g, KindParams kp, const double *__restrict__ a, double sig,
                           double alpha, double dt, const double *__restrict__ b,
                           const double *__restrict__ xin, double *__restrict__ xout,
                           const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < g.n; p += gridDim.x * blockDim.x) {
    if (xin) {
      double d;
      const double sx = apply_s<KIND>(g, kp, a, sig, alpha, dt, xin, p, d);
      xout[p] = xin[p] + OMEGA * ((b[p] - sx) / d);
    } else {
      int nb[4];
      nbr2d(g, p, nb);
      double cc, cn[4];
      stencil_row<KIND>(g, kp, a, sig, p, nb, cc, cn);
      xout[p] = OMEGA * (b[p] / (alpha - dt * cc));
    }
  }
}

// bc = R (b - S x): the 2x2 average of the fine residual
template <int KIND>
__global__ void k_mg_resid_restrict(Grid gf, Grid gc, KindParams kp, const double *__restrict__ a,
                                    double sig, double alpha, double dt,
                                    const double *__restrict__ b, const double *__restrict__ x,
                                    double *__restrict__ bc, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < gc.n; q += gridDim.x * blockDim.x) {
    const int I = q % gc.nx, J = q / gc.nx;
    double acc = 0.0;
#pragma unroll
    for (int dj = 0; dj < 2; ++dj)
#pragma unroll
      for (int di = 0; di < 2; ++di) {
        const int p = (2 * J + dj) * gf.nx + 2 * I + di;
        double d;
        acc += b[p] - apply_s<KIND>(gf, kp, a, sig, alpha, dt, x, p, d);
      }
    bc[q] = 0.25 * acc;
  }
}

// fc = 2x2 average of f
__global__ void k_mg_restrict(Grid gf, Grid gc, const double *__restrict__ f,
                              double *__restrict__ fc) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < gc.n; q += gridDim.x * blockDim.x) {
    const int I = q % gc.nx, J = q / gc.nx;
    const int p = 2 * J * gf.nx + 2 * I;
    fc[q] = 0.25 * ((f[p] + f[p + 1]) + (f[p + gf.nx] + f[p + gf.nx + 1]));
  }
}

// xf += P xc, bilinear on cell centres: (9 xc[I,J] + 3 xc[I+di,J] + 3 xc[I,J+dj]
// + xc[I+di,J+dj]) / 16 with (di, dj) pointing to the fine cell's side
__global__ void k_mg_prolong_add(Grid gc, Grid gf, const double *__restrict__ xc,
                                 double *__restrict__ xf, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < gf.n; p += gridDim.x * blockDim.x) {
    const int i = p % gf.nx, j = p / gf.nx;
    const int I = i >> 1, J = j >> 1;
    int I2 = (i & 1) ? I + 1 : I - 1;
    int J2 = (j & 1) ? J + 1 : J - 1;
    I2 = I2 < 0 ? I2 + gc.nx : (I2 >= gc.nx ? I2 - gc.nx : I2);
    J2 = J2 < 0 ? J2 + gc.ny : (J2 >= gc.ny ? J2 - gc.ny : J2);
    const double v = 9.0 * xc[J * gc.nx + I] + 3.0 * xc[J * gc.nx + I2] +
                     3.0 * xc[J2 * gc.nx + I] + xc[J2 * gc.nx + I2];
    xf[p] += v * 0.0625;
  }
}

__global__ void k_mg_copy(int n, const double *__restrict__ src, double *__restrict__ dst,
                          const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    dst[p] = src[p];
}

// ------------------------------------------------------------------ host

static Grid coarse_grid(const Grid &f) {
  Grid c = f;
  c.nx = f.nx / 2;
  c.ny = f.ny / 2;
  c.nz = 1;
  c.nxy = c.nx * c.ny;
  c.n = c.nxy;
  for (int d = 0; d < 2; ++d) {
    c.ih2[d] = f.ih2[d] * 0.25;
    c.i2h[d] = f.i2h[d] * 0.5;
  }
  c.ih2[2] = c.i2h[2] = 0.0;
  c.lapdiag = -2.0 * (c.ih2[0] + c.ih2[1]);
  c.slab = 0;
  c.pin = 0;
  return c;
}

template <class F>
static void dispatch_ode_kind(int kind, F f) {
  switch (kind) {
    case KIND_NLDIFF: f(std::integral_constant<int, KIND_NLDIFF>{}); break;
    case KIND_BURGERS: f(std::integral_constant<int, KIND_BURGERS>{}); break;
    case KIND_RAD: f(std::integral_constant<int, KIND_RAD>{}); break;
    default: throw SolveError(IRKG_ERR_CONFIG, "multigrid inner solves: ODE kinds only");
  }
}

// Level hierarchy, restricted coefficient fields and coarsest factors for
// the block's inner operators (S1 = eta I - dt L1 [, S2 = gamma I - dt L2]).
void Engine::mg_setup(const BlockSpec &B) {
  if (ndim != 2 || slab())
    throw SolveError(IRKG_ERR_CONFIG, "PrecondSpec(inner='mg') covers single-rank 2-D grids");
  // levels: halve while both extents stay even and the coarse grid keeps >= 8 cells a side
  std::vector<Grid> gs{grid};
  while (gs.back().nx % 2 == 0 && gs.back().ny % 2 == 0 && gs.back().nx / 2 >= 8 &&
         gs.back().ny / 2 >= 8 && gs.back().n > MG_COARSE)
    gs.push_back(coarse_grid(gs.back()));
  const int L = (int)gs.size();
  if (L < 2) throw SolveError(IRKG_ERR_CONFIG, "multigrid: grid too small to coarsen");
  if (mg.nlev != L || mg.lev[0].g.n != grid.n) {
    for (int l = 0; l < mg.nlev; ++l)
      for (double *p : {mg.lev[l].a[0], mg.lev[l].a[1], mg.lev[l].b, mg.lev[l].x, mg.lev[l].t})
        if (p) cudaFree(p);
    mg = MgHier{};
    mg.nlev = L;
    for (int l = 0; l < L; ++l) {
      MgLevel &v = mg.lev[l];
      v.g = gs[l];
      const size_t n = (size_t)gs[l].n;
      if (l > 0) {
        dalloc_raw((void **)&v.a[0], sizeof(double) * n);
        dalloc_raw((void **)&v.a[1], sizeof(double) * n);
        dalloc_raw((void **)&v.b, sizeof(double) * n);
        dalloc_raw((void **)&v.x, sizeof(double) * n);
      }
      dalloc_raw((void **)&v.t, sizeof(double) * n);
    }
  }
  const Op ops[2] = {B.l1, B.size == 2 ? B.l2 : B.l1};
  const double alphas[2] = {B.eta, B.size == 2 ? B.gamma : B.eta};
  const int nops = B.size;
  for (int o = 0; o < nops; ++o) {
    mg.alpha[o] = alphas[o];
    mg.sigma[o] = ops[o].sigma;
    mg.lev[0].a[o] = const_cast<double *>(ops[o].a);
    for (int l = 1; l < L; ++l) {
      k_mg_restrict<<<grid_for(gs[l].n), 256, 0, stream>>>(gs[l - 1], gs[l], mg.lev[l - 1].a[o],
                                                          mg.lev[l].a[o]);
      count(1);
    }
    Op oc{mg.lev[L - 1].a[o], ops[o].sigma, 1};
    band_factor(mg.coarse[o], oc, alphas[o], B.dt, &gs[L - 1]);
  }
  mg.dt = B.dt;
}

// x = V-cycle(S_o) b on the fine level (b is not modified)
void Engine::mg_vcycle(int o, const double *b, double *x, const GCtrl *skip) {
  const int L = mg.nlev;
  const double al = mg.alpha[o], sg = mg.sigma[o], dt = mg.dt;
  dispatch_ode_kind(prob.kind, [&](auto KD) {
    constexpr int K_ = decltype(KD)::value;
    for (int l = 0; l < L - 1; ++l) {
      MgLevel &v = mg.lev[l], &c = mg.lev[l + 1];
      const double *bl = l == 0 ? b : v.b;
      double *xl = l == 0 ? x : v.x;
      const int gb = grid_for(v.g.n);
      k_mg_sweep<K_><<<gb, 256, 0, stream>>>(v.g, kp, v.a[o], sg, al, dt, bl, nullptr, v.t, skip);
      k_mg_sweep<K_><<<gb, 256, 0, stream>>>(v.g, kp, v.a[o], sg, al, dt, bl, v.t, xl, skip);
      k_mg_resid_restrict<K_><<<grid_for(c.g.n), 256, 0, stream>>>(v.g, c.g, kp, v.a[o], sg, al,
                                                                    dt, bl, xl, c.b, skip);
      count(3);
    }
    MgLevel &cl = mg.lev[L - 1];
    k_mg_copy<<<grid_for(cl.g.n), 256, 0, stream>>>(cl.g.n, cl.b, cl.x, skip);
    count(1);
    band_apply(mg.coarse[o], cl.x, skip);
    for (int l = L - 2; l >= 0; --l) {
      MgLevel &v = mg.lev[l], &c = mg.lev[l + 1];
      const double *bl = l == 0 ? b : v.b;
      double *xl = l == 0 ? x : v.x;
      const int gb = grid_for(v.g.n);
      k_mg_prolong_add<<<gb, 256, 0, stream>>>(c.g, v.g, c.x, xl, skip);
      k_mg_sweep<K_><<<gb, 256, 0, stream>>>(v.g, kp, v.a[o], sg, al, dt, bl, xl, v.t, skip);
      k_mg_sweep<K_><<<gb, 256, 0, stream>>>(v.g, kp, v.a[o], sg, al, dt, bl, v.t, xl, skip);
      count(3);
    }
  });
}

// z1 = MG(S1) r1 ; z2 = MG(S2) (r2 + beta^2/phi z1)
void Engine::precond_mg(const BlockSpec &B, const VecIn &vin, double *z, const GCtrl *skip) {
  if (!mg_rhs) dalloc_raw((void **)&mg_rhs, sizeof(double) * (size_t)N);
  const int gb = grid_for(N);
  k_vin_rhs<<<gb, 256, 0, stream>>>((int)N, vin, 0, nullptr, 0.0, mg_rhs, skip);
  count(1);
  mg_vcycle(0, mg_rhs, z, skip);
  if (B.size == 2) {
    k_vin_rhs<<<gb, 256, 0, stream>>>((int)N, vin, (int)N, z, B.beta * B.beta / B.phi, mg_rhs,
                                       skip);
    count(1);
    mg_vcycle(1, mg_rhs, z + N, skip);
  }
}

}  // namespace irkg
