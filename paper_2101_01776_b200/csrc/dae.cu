// dae.cu -- index-1 DAE stage solve for the vorticity/streamfunction system
// (BASELINE configs[4]) on the device.
//
// Restates src/dae.py of the reference for the reordered mode:
//   dae_stage_residual      94-105     k_dae_residual
//   _build_dae_variant      318-333    opfields of Psi stage values + sigma
//   _solve_dae_transformed  336-420    Engine::dae_transformed_solve
//   solve_dae_block4x4      255-279    differential 2x2 GMRES (shared block
//                          + 307-315   machinery, kind = Arakawa) then two
//                                      exact constraint solves, then the
//                                      composite true-residual recheck
//   _ConstraintSolver       108-126    FFT-diagonalised pinned Poisson solve
//   dae_newton_step / dae_step 423-498 Engine::dae_newton / dae_step
//
// Operator (VorticityProblem, problems.py):
//   N(w, psi) = -J(psi, w) + nu Lap w   (Arakawa J, 9-point)
//   G(w, psi) = h^2 (Lap psi + w), row 0: psi_0
//   L_u(Psi) x = -J(Psi, x) + nu Lap x;  L_w = 0;  G_u = h^2 I_p;  G_w = h^2 Lap_p
// Weighted sums collapse to a = sum_k w_k Psi_k (J is linear in psi), sigma.
#include <cufft.h>

#include <chrono>
#include <cmath>
#include <cstdio>

#include "engine.h"

namespace irkg {

namespace {

struct P9 {
  double c, E, W, N, S, NE, NW, SE, SW;
};

struct Off9 {
  int dxm, dxp, dym, dyp;
};

__device__ __forceinline__ Off9 off9(const Grid &g, int ix, int iy) {
  Off9 o;
  o.dxm = (ix == 0) ? g.nx - 1 : -1;
  o.dxp = (ix == g.nx - 1) ? 1 - g.nx : 1;
  o.dym = (iy == 0) ? (g.ny - 1) * g.nx : -g.nx;
  o.dyp = (iy == g.ny - 1) ? -(g.ny - 1) * g.nx : g.nx;
  return o;
}

__device__ __forceinline__ P9 load9(const double *__restrict__ f, int p, const Off9 &o) {
  P9 v;
  v.c = f[p];
  v.E = f[p + o.dxp];
  v.W = f[p + o.dxm];
  v.N = f[p + o.dyp];
  v.S = f[p + o.dym];
  v.NE = f[p + o.dyp + o.dxp];
  v.NW = f[p + o.dyp + o.dxm];
  v.SE = f[p + o.dym + o.dxp];
  v.SW = f[p + o.dym + o.dxm];
  return v;
}

// 12 hx hy * J(psi, w): Arakawa's three forms summed
__device__ __forceinline__ double jac_sum(const P9 &P, const P9 &W) {
  const double j1 = (P.E - P.W) * (W.N - W.S) - (P.N - P.S) * (W.E - W.W);
  const double j2 = P.E * (W.NE - W.SE) - P.W * (W.NW - W.SW) - P.N * (W.NE - W.NW) +
                    P.S * (W.SE - W.SW);
  const double j3 = W.N * (P.NE - P.NW) - W.S * (P.SE - P.SW) - W.E * (P.NE - P.SE) +
                    W.W * (P.NW - P.SW);
  return (j1 + j2) + j3;
}

__device__ __forceinline__ double lap9(const Grid &g, const P9 &f) {
  return g.ih2[0] * (f.E + f.W - 2.0 * f.c) + g.ih2[1] * (f.N + f.S - 2.0 * f.c);
}

__device__ __forceinline__ double jscale(const Grid &g) {
  // 1 / (12 hx hy) with i2h = 1/(2h): 4 i2h_x i2h_y / 12
  return g.i2h[0] * g.i2h[1] / 3.0;
}

// L_eff(a, sigma) x = -J(a, x) + sigma nu Lap x
__device__ __forceinline__ double ara_lx(const Grid &g, double nu, const double *a, double sigma,
                                         const double *x, int p, const Off9 &o) {
  const P9 A = load9(a, p, o), X = load9(x, p, o);
  return -jscale(g) * jac_sum(A, X) + sigma * nu * lap9(g, X);
}

__device__ __forceinline__ double wsum3(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fold per-CTA (a, b) pairs via the last-CTA ticket; out[0] = sum a, out[1] = sum b
template <int BS>
__device__ void reduce2(double a, double b, double *part, int nblk, unsigned *counter,
                        double *out) {
  __shared__ double ra[BS / 32], rb[BS / 32];
  __shared__ bool last;
  a = wsum3(a);
  b = wsum3(b);
  if ((threadIdx.x & 31) == 0) {
    ra[threadIdx.x >> 5] = a;
    rb[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = 0.0, tb = 0.0;
    for (int w = 0; w < BS / 32; ++w) {
      ta += ra[w];
      tb += rb[w];
    }
    part[2 * blockIdx.x] = ta;
    part[2 * blockIdx.x + 1] = tb;
    __threadfence();
    last = (atomicAdd(counter, 1u) == (unsigned)(nblk - 1));
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    double sa = 0.0, sb = 0.0;
    for (int c = threadIdx.x; c < nblk; c += 32) {
      sa += __ldcg(part + 2 * c);
      sb += __ldcg(part + 2 * c + 1);
    }
    sa = wsum3(sa);
    sb = wsum3(sb);
    if (threadIdx.x == 0) {
      out[0] = sa;
      out[1] = sb;
      *counter = 0u;
    }
  }
}

constexpr int DBS = 256;

}  // namespace

#define ROWS_LOOP(g)                                                  \
  for (int iy = blockIdx.x; iy < (g).ny; iy += gridDim.x)             \
    for (int ix = threadIdx.x; ix < (g).nx; ix += blockDim.x)

// composite residual per stage: [N(U_i, W_i) - k_i ; G(U_i, W_i)] and ||.||^2
__global__ void k_dae_residual(Grid g, double nu, double h2, int s, const double *__restrict__ UW,
                               const double *__restrict__ K2, double *__restrict__ F2,
                               double *part, unsigned *counter, double *out) {
  const int n = g.n;
  double acc = 0.0;
  ROWS_LOOP(g) {
    const int p = iy * g.nx + ix;
    const Off9 o = off9(g, ix, iy);
    for (int i = 0; i < s; ++i) {
      const double *U = UW + (size_t)i * 2 * n, *Wp = U + n;
      const P9 u = load9(U, p, o), w = load9(Wp, p, o);
      const double fu = (-jscale(g) * jac_sum(w, u) + nu * lap9(g, u)) - K2[(size_t)i * 2 * n + p];
      const double fw = (p == 0) ? w.c : h2 * (lap9(g, w) + u.c);
      F2[(size_t)i * 2 * n + p] = fu;
      F2[(size_t)i * 2 * n + n + p] = fw;
      acc += fu * fu + fw * fw;
    }
  }
  reduce2<DBS>(acc, 0.0, part, gridDim.x, counter, out);
}

// ||G(u, w)||^2 for the state uw = [u; w]
__global__ void k_dae_gnorm(Grid g, double h2, const double *__restrict__ UW, double *part,
                            unsigned *counter, double *out) {
  const int n = g.n;
  double acc = 0.0;
  ROWS_LOOP(g) {
    const int p = iy * g.nx + ix;
    const Off9 o = off9(g, ix, iy);
    const P9 w = load9(UW + n, p, o);
    const double fw = (p == 0) ? w.c : h2 * (lap9(g, w) + UW[p]);
    acc += fw * fw;
  }
  reduce2<DBS>(acc, 0.0, part, gridDim.x, counter, out);
}

// a_o = sum_k w[o][k] Psi_k  (Psi_k = second half of stage row k of UW)
__global__ void k_dae_opfields(int n, OpWeights W, const double *__restrict__ UW,
                               double *__restrict__ A) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    double f[MAXS];
#pragma unroll
    for (int k = 0; k < MAXS; ++k)
      if (k < W.s) f[k] = UW[(size_t)k * 2 * n + n + p];
    for (int o = 0; o < W.nops; ++o) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < MAXS; ++k) {
        if (k < W.s) {
          const double wk = W.w[o * MAXS + k];
          if (wk != 0.0) acc += wk * f[k];
        }
      }
      A[(size_t)o * n + p] = acc;
    }
  }
}

// Jacobi on (alpha I - dt L_eff); first sweep from zero when x == nullptr
__global__ void k_ara_jac(Grid g, double nu, Op L, double alpha, double dt, VecIn vin, int in_off,
                          const double *__restrict__ zc, double cpl, double *__restrict__ t_out,
                          const double *__restrict__ t_in, const double *__restrict__ x,
                          double *__restrict__ x_out, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  double scale = 1.0;
  const double *in = t_in ? nullptr : vin_resolve(vin, in_off, scale).base;
  const double D = alpha - dt * (L.sigma * nu * g.lapdiag);
  const double invD = 1.0 / D;
  ROWS_LOOP(g) {
    const int p = iy * g.nx + ix;
    double r;
    if (t_in) {
      r = t_in[p];
    } else {
      r = scale * in[p];
      if (zc) {
        r = r + cpl * zc[p];
        if (t_out) t_out[p] = r;
      }
    }
    if (!x) {
      x_out[p] = OMEGA * (invD * r);
    } else {
      const Off9 o = off9(g, ix, iy);
      const double xc = x[p];
      const double sx = alpha * xc - dt * ara_lx(g, nu, L.a, L.sigma, x, p, o);
      x_out[p] = xc + OMEGA * (invD * (r - sx));
    }
  }
}

// 1x1 / 2x2 block operator with the Arakawa L (apply_block2x2); b != null: residual + norm
template <int SIZE>
__global__ void k_ara_block_op(Grid g, double nu, double eta, double beta, double phi, double dt,
                               Op l1, Op l2, Op c12, Op c21, const double *__restrict__ z,
                               double *__restrict__ w, const double *__restrict__ b, double *part,
                               unsigned *counter, double *out_norm, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  const int n = g.n;
  double nrm = 0.0;
  ROWS_LOOP(g) {
    const int p = iy * g.nx + ix;
    const Off9 o = off9(g, ix, iy);
    if (SIZE == 1) {
      double v = eta * z[p] - dt * ara_lx(g, nu, l1.a, l1.sigma, z, p, o);
      if (b) {
        v = b[p] - v;
        nrm += v * v;
      }
      w[p] = v;
    } else {
      const double *z1 = z, *z2 = z + n;
      double top = eta * z1[p] - dt * ara_lx(g, nu, l1.a, l1.sigma, z1, p, o) + phi * z2[p];
      double bot = -(beta * beta / phi) * z1[p] + eta * z2[p] -
                   dt * ara_lx(g, nu, l2.a, l2.sigma, z2, p, o);
      if (c12.present) top -= dt * ara_lx(g, nu, c12.a, c12.sigma, z2, p, o);
      if (c21.present) bot -= dt * ara_lx(g, nu, c21.a, c21.sigma, z1, p, o);
      if (b) {
        top = b[p] - top;
        bot = b[p + n] - bot;
        nrm += top * top + bot * bot;
      }
      w[p] = top;
      w[p + n] = bot;
    }
  }
  if (b) reduce2<DBS>(nrm, 0.0, part, gridDim.x, counter, out_norm);
}

// composite block rhs rows (src/dae.py:349-360): for r in block rows
//   acc_u = g_u - sum_j R0[r,j] y_u,j + dt sum_j L_od y_u,j
//   acc_w = g_w + dt sum_j sigma_od (h^2 I_p y_u,j + h^2 Lap_p y_w,j)
struct DaeBacksub {
  int rows, row0, njs;
  int j[MAXS];
  double coef[2][MAXS];
  Op od[2][MAXS];
};

__global__ void k_dae_backsub(Grid g, double nu, double h2, double dt, DaeBacksub T,
                              const double *__restrict__ G2, const double *__restrict__ Y2,
                              double *__restrict__ ACC) {
  const int n = g.n;
  ROWS_LOOP(g) {
    const int p = iy * g.nx + ix;
    const Off9 o = off9(g, ix, iy);
    for (int r = 0; r < T.rows; ++r) {
      double au = G2[(size_t)(T.row0 + r) * 2 * n + p];
      double aw = G2[(size_t)(T.row0 + r) * 2 * n + n + p];
      for (int q = 0; q < T.njs; ++q) {
        const double *yu = Y2 + (size_t)T.j[q] * 2 * n, *yw = yu + n;
        const double c = T.coef[r][q];
        if (c != 0.0) au -= c * yu[p];
        const Op od = T.od[r][q];
        if (od.present) {
          au += dt * ara_lx(g, nu, od.a, od.sigma, yu, p, o);
          const P9 w9 = load9(yw, p, o);
          const double gu = (p == 0) ? 0.0 : h2 * yu[p];
          const double gw = (p == 0) ? w9.c : h2 * lap9(g, w9);
          aw += dt * (od.sigma * gu + od.sigma * gw);
        }
      }
      ACC[(size_t)r * 2 * n + p] = au;
      ACC[(size_t)r * 2 * n + n + p] = aw;
    }
  }
}

// constraint rhs c = acc_w + dt * sigma * G_u y_u  (G_u row 0 is zero)
__global__ void k_dae_crhs(int n, double dt, double sigma_h2, const double *__restrict__ accw,
                           const double *__restrict__ yu, double *__restrict__ c) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    c[p] = (p == 0) ? accw[0] : accw[p] + dt * (sigma_h2 * yu[p]);
}

// Poisson step 1: f = c / (sigma h^2) off the pin; f_0 = -sum_{i != 0} f_i
__global__ void k_pois_sum(int n, double inv, const double *__restrict__ c, double *part,
                           unsigned *counter, double *out) {
  double acc = 0.0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    if (p != 0) acc += inv * c[p];
  reduce2<DBS>(acc, 0.0, part, gridDim.x, counter, out);
}

__global__ void k_pois_rhs(int n, double inv, const double *__restrict__ c,
                           const double *__restrict__ sum, double *__restrict__ f) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    f[p] = (p == 0) ? -sum[0] : inv * c[p];
}

// divide the half spectrum by the periodic Laplacian eigenvalues (mode 0 -> 0)
__global__ void k_pois_scale(int nx, int ny, double ih2x, double ih2y, cufftDoubleComplex *F) {
  const int nxh = nx / 2 + 1;
  const int tot = nxh * ny;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < tot; q += gridDim.x * blockDim.x) {
    const int kx = q % nxh, ky = q / nxh;
    const double sx = sin(M_PI * kx / nx), sy = sin(M_PI * ky / ny);
    const double lam = -4.0 * ih2x * sx * sx - 4.0 * ih2y * sy * sy;
    const double inv = (q == 0) ? 0.0 : 1.0 / (lam * (double)nx * (double)ny);
    F[q].x *= inv;
    F[q].y *= inv;
  }
}

// y = yt - yt_0 + c_0 / sigma;  out = post * y
__global__ void k_pois_fix(int n, double post, double inv_sigma, const double *__restrict__ yt,
                           const double *__restrict__ c, double *__restrict__ out) {
  const double y0 = yt[0], pin = c[0] * inv_sigma;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    out[p] = post * ((yt[p] - y0) + pin);
}

// composite true residual of the reordered 4x4 block (src/dae.py:238-253, 307-314):
// out[0] = ||rhs - A x||^2, out[1] = ||rhs||^2; rhs = ACC (2 x 2N), x = Y2 rows r0, r0+1
__global__ void k_dae_block_res(Grid g, double nu, double h2, double eta, double beta, double phi,
                                double dt, Op l1, Op l2, double sig1, double sig2,
                                const double *__restrict__ ACC, const double *__restrict__ X1,
                                const double *__restrict__ X2, double *part, unsigned *counter,
                                double *out) {
  const int n = g.n;
  double rr = 0.0, bb = 0.0;
  ROWS_LOOP(g) {
    const int p = iy * g.nx + ix;
    const Off9 o = off9(g, ix, iy);
    const double *x1u = X1, *x1w = X1 + n, *x2u = X2, *x2w = X2 + n;
    const double top1 = eta * x1u[p] - dt * ara_lx(g, nu, l1.a, l1.sigma, x1u, p, o) + phi * x2u[p];
    const double top2 = eta * x2u[p] - dt * ara_lx(g, nu, l2.a, l2.sigma, x2u, p, o) -
                        (beta * beta / phi) * x1u[p];
    const P9 w1 = load9(x1w, p, o), w2 = load9(x2w, p, o);
    const double gu1 = (p == 0) ? 0.0 : h2 * x1u[p], gu2 = (p == 0) ? 0.0 : h2 * x2u[p];
    const double gw1 = (p == 0) ? w1.c : h2 * lap9(g, w1);
    const double gw2 = (p == 0) ? w2.c : h2 * lap9(g, w2);
    const double bot1 = -dt * (sig1 * gu1) - dt * (sig1 * gw1);
    const double bot2 = -dt * (sig2 * gu2) - dt * (sig2 * gw2);
    const double r[4] = {ACC[p], ACC[n + p], ACC[2 * n + p], ACC[3 * n + p]};
    const double ax[4] = {top1, bot1, top2, bot2};
    for (int k = 0; k < 4; ++k) {
      const double d = r[k] - ax[k];
      rr += d * d;
      bb += r[k] * r[k];
    }
  }
  reduce2<DBS>(rr, bb, part, gridDim.x, counter, out);
}

// ============================================================ engine side

void Engine::dae_init() {
  if (!dae) return;
  dalloc_raw((void **)&ACC, sizeof(double) * 4 * N);
  dalloc_raw((void **)&XU, sizeof(double) * 2 * N);
  dalloc_raw((void **)&CR, sizeof(double) * N);
  dalloc_raw((void **)&PT, sizeof(double) * N);
  dalloc_raw((void **)&fft_buf, sizeof(cufftDoubleComplex) * (size_t)grid.ny * (grid.nx / 2 + 1));
  h2 = (prob.length / grid.nx) *
       ((prob.length_y > 0.0 ? prob.length_y : prob.length) / grid.ny);
  cufftHandle p1, p2;
  if (cufftPlan2d(&p1, grid.ny, grid.nx, CUFFT_D2Z) != CUFFT_SUCCESS ||
      cufftPlan2d(&p2, grid.ny, grid.nx, CUFFT_Z2D) != CUFFT_SUCCESS)
    throw CudaError("cufftPlan2d failed");
  fft_fwd = (int)p1;
  fft_inv = (int)p2;
}

void Engine::dae_fini() {
  if (fft_fwd >= 0) cufftDestroy((cufftHandle)fft_fwd);
  if (fft_inv >= 0) cufftDestroy((cufftHandle)fft_inv);
  void *bufs[] = {ACC, XU, CR, PT, fft_buf};
  for (void *b : bufs)
    if (b) cudaFree(b);
}

int Engine::dae_grid() const { return grid.ny < sms * 8 ? grid.ny : sms * 8; }

// out = post * (sigma G_w)^{-1} c  -- _ConstraintSolver.solve, src/dae.py:122-126
void Engine::constraint_solve(double sigma, const double *c, double *out, double post) {
  if (sigma == 0.0) throw SolveError(IRKG_ERR_INDEX, "constraint Jacobian is singular");
  const int n = (int)N;
  const double inv = 1.0 / (sigma * h2);
  k_pois_sum<<<dae_grid(), DBS, 0, stream>>>(n, inv, c, part, counter, &scal_dev[4]);
  k_pois_rhs<<<grid_for(N), 256, 0, stream>>>(n, inv, c, &scal_dev[4], PT);
  cufftSetStream((cufftHandle)fft_fwd, stream);
  cufftSetStream((cufftHandle)fft_inv, stream);
  if (cufftExecD2Z((cufftHandle)fft_fwd, PT, (cufftDoubleComplex *)fft_buf) != CUFFT_SUCCESS)
    throw CudaError("cufftExecD2Z failed");
  k_pois_scale<<<grid_for((long long)grid.ny * (grid.nx / 2 + 1)), 256, 0, stream>>>(
      grid.nx, grid.ny, grid.ih2[0], grid.ih2[1], (cufftDoubleComplex *)fft_buf);
  if (cufftExecZ2D((cufftHandle)fft_inv, (cufftDoubleComplex *)fft_buf, PT) != CUFFT_SUCCESS)
    throw CudaError("cufftExecZ2D failed");
  k_pois_fix<<<grid_for(N), 256, 0, stream>>>(n, post, 1.0 / sigma, PT, c, out);
  count(4);

}

void Engine::ara_jacobi_chain(const Op &L, double alpha, double dt, int inner, const VecIn &vin,
                              int in_off, const double *zc, double cpl, double *x_out,
                              const GCtrl *skip) {
  const int gb = dae_grid();
  double *tbuf = zc ? tmp_t : nullptr;
  auto dst = [&](int i) { return ((inner - i) % 2 == 0) ? x_out : tmp_x; };
  k_ara_jac<<<gb, DBS, 0, stream>>>(grid, kp.nu, L, alpha, dt, vin, in_off, zc, cpl, tbuf, nullptr,
                                    nullptr, dst(1), skip);
  count(1);
  for (int i = 2; i <= inner; ++i) {
    k_ara_jac<<<gb, DBS, 0, stream>>>(grid, kp.nu, L, alpha, dt, vin, in_off, nullptr, 0.0, nullptr,
                                      tbuf, dst(i - 1), dst(i), skip);
    count(1);
  }
}

void Engine::ara_block_op(const BlockSpec &B, const double *z, double *w, const double *b,
                          double *out_norm, const GCtrl *skip) {
  const int gb = dae_grid();
  if (B.size == 1)
    k_ara_block_op<1><<<gb, DBS, 0, stream>>>(grid, kp.nu, B.eta, B.beta, B.phi, B.dt, B.l1, B.l2,
                                              B.c12, B.c21, z, w, b, part, counter, out_norm, skip);
  else
    k_ara_block_op<2><<<gb, DBS, 0, stream>>>(grid, kp.nu, B.eta, B.beta, B.phi, B.dt, B.l1, B.l2,
                                              B.c12, B.c21, z, w, b, part, counter, out_norm, skip);
  count(1);
}

double Engine::dae_residual(const double *UW, const double *K2, double *F2) {
  k_dae_residual<<<dae_grid(), DBS, 0, stream>>>(grid, kp.nu, h2, s, UW, K2, F2, part, counter,
                                                 &scal_dev[0]);
  count(1);
  double v = 0.0;
  check(cudaMemcpyAsync(&v, &scal_dev[0], sizeof(double), cudaMemcpyDeviceToHost, stream));
  check(cudaStreamSynchronize(stream));
  return v;
}

double Engine::dae_gnorm(const double *UW) {
  k_dae_gnorm<<<dae_grid(), DBS, 0, stream>>>(grid, h2, UW, part, counter, &scal_dev[0]);
  count(1);
  double v = 0.0;
  check(cudaMemcpyAsync(&v, &scal_dev[0], sizeof(double), cudaMemcpyDeviceToHost, stream));
  check(cudaStreamSynchronize(stream));
  return std::sqrt(v);
}

// _solve_dae_transformed (src/dae.py:336-420), reordered 4x4 blocks
void Engine::dae_transformed_solve(double dt, const double *rhs, double *dk,
                                   irkg_step_stats *stats) {
  const long long n2 = 2 * N;
  std::vector<double> qt(s * s), qr(s * s);
  for (int i = 0; i < s; ++i)
    for (int k = 0; k < s; ++k) qt[i * s + k] = tab.q[k * IRKG_MAX_STAGES + i];
  stage_mix_n(qt.data(), rhs, Gs, false, n2);
  check(cudaMemsetAsync(Y, 0, (size_t)s * n2 * sizeof(double), stream));
  for (int b = tab.nblocks - 1; b >= 0; --b) {
    const int off = tab.blk_offset[b], size = tab.blk_size[b];
    if (size != 2)
      throw SolveError(IRKG_ERR_CONFIG,
                       "composite 1x1 DAE blocks need exact reduced solves (src/dae.py:140); "
                       "use a tableau with complex eigen-pairs only (e.g. Gauss(2), Gauss(4))");
    DaeBacksub T{};
    T.rows = 2;
    T.row0 = off;
    for (int j = off + 2; j < s; ++j) {
      int q = T.njs++;
      T.j[q] = j;
      for (int r = 0; r < 2; ++r) {
        T.coef[r][q] = tab.r[(off + r) * IRKG_MAX_STAGES + j];
        T.od[r][q] = op_of(od_slot[off + r][j]);
      }
    }
    k_dae_backsub<<<dae_grid(), DBS, 0, stream>>>(grid, kp.nu, h2, dt, T, Gs, Y, ACC);
    count(1);
    // differential 2x2: rdiff = [acc0_u ; acc1_u]
    check(cudaMemcpyAsync(RHS, ACC, N * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    check(cudaMemcpyAsync(RHS + N, ACC + n2, N * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    BlockSpec B{};
    B.size = 2;
    B.eta = tab.blk_eta[b];
    B.beta = tab.blk_beta[b];
    B.phi = tab.blk_phi[b];
    B.gamma = gamma_of(B.eta, B.beta);
    B.dt = dt;
    B.inner = cfg.inner;
    B.l1 = op_of(diag_slot[off]);
    B.l2 = op_of(diag_slot[off + 1]);
    B.l1.present = B.l2.present = 1;  // reordered drops C12/C21 (src/dae.py:232-233)
    KrylovOut rep = gmres(B, RHS, XU, cfg.krylov_rtol, cfg.krylov_maxit, cfg.restart);
    const long long diff_solves = rep.precond_applications;
    // y_u -> Y rows; constraint solves for y_w (src/dae.py:274-278)
    double *Y1 = Y + (size_t)off * n2, *Y2r = Y + (size_t)(off + 1) * n2;
    check(cudaMemcpyAsync(Y1, XU, N * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    check(cudaMemcpyAsync(Y2r, XU + N, N * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    const double sig1 = op_sigma[diag_slot[off]], sig2 = op_sigma[diag_slot[off + 1]];
    k_dae_crhs<<<grid_for(N), 256, 0, stream>>>((int)N, dt, sig1 * h2, ACC + N, XU, CR);
    constraint_solve(sig1, CR, Y1 + N, -1.0 / dt);
    k_dae_crhs<<<grid_for(N), 256, 0, stream>>>((int)N, dt, sig2 * h2, ACC + n2 + N, XU + N, CR);
    constraint_solve(sig2, CR, Y2r + N, -1.0 / dt);
    count(2);
    if (stats) {
      if (stats->n_block_records < IRKG_MAX_BLOCK_RECORDS) {
        stats->block_offset[stats->n_block_records] = off;
        stats->block_iterations[stats->n_block_records] = rep.iterations;
        stats->n_block_records++;
      }
      stats->krylov_iterations += rep.iterations;
      stats->precond_applications += rep.precond_applications;
      stats->differential_solves += (int)diff_solves;
      stats->constraint_solves += 2;
    }
    if (!rep.converged) {
      if (stats) {
        stats->fail_block_offset = off;
        irkg_krylov_report &fr = stats->fail_report;
        fr.iterations = rep.iterations;
        fr.converged = 0;
        fr.precond_applications = rep.precond_applications;
        fr.n_residuals = (int)rep.residuals.size();
        if (fr.residuals)
          for (int i = 0; i < (int)rep.residuals.size() && i < fr.residual_capacity; ++i)
            fr.residuals[i] = rep.residuals[i];
      }
      char msg[96];
      snprintf(msg, sizeof msg, "composite 2x2 block at offset %d did not converge", off);
      throw SolveError(IRKG_ERR_STAGE_SOLVE, msg);
    }
    // composite true-residual recheck (src/dae.py:307-314)
    k_dae_block_res<<<dae_grid(), DBS, 0, stream>>>(grid, kp.nu, h2, B.eta, B.beta, B.phi, dt,
                                                    B.l1, B.l2, sig1, sig2, ACC, Y1, Y2r, part,
                                                    counter, &scal_dev[6]);
    count(1);
    double rb[2];
    check(cudaMemcpyAsync(rb, &scal_dev[6], 2 * sizeof(double), cudaMemcpyDeviceToHost, stream));
    check(cudaStreamSynchronize(stream));
    if (rb[1] > 0.0) {
      const double true_rel = std::sqrt(rb[0]) / std::sqrt(rb[1]);
      if (true_rel > cfg.krylov_rtol) {
        if (stats) {
          stats->fail_block_offset = -1;
          stats->fail_report.iterations = rep.iterations;
          stats->fail_report.converged = rep.converged;
          stats->fail_report.precond_applications = rep.precond_applications;
          stats->fail_report.n_residuals = 0;
        }
        char msg[128];
        snprintf(msg, sizeof msg, "composite block residual %.3e above rtol %.3e", true_rel,
                 cfg.krylov_rtol);
        throw SolveError(IRKG_ERR_STAGE_SOLVE, msg);
      }
    }
  }
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j) {
      double acc = 0.0;
      for (int k = 0; k < s; ++k) acc += tab.q[i * IRKG_MAX_STAGES + k] * tab.r[k * IRKG_MAX_STAGES + j];
      qr[i * s + j] = acc;
    }
  stage_mix_n(qr.data(), Y, dk, false, n2);
}

// dae_newton_step (src/dae.py:423-471): uw = [u; w] (2N), K2 = (s, 2N) [k_i; l_i]
void Engine::dae_newton(const double *uw, double *K2, double t, double dt, irkg_step_stats *stats) {
  auto tic = std::chrono::steady_clock::now();
  const long long n2 = 2 * N;
  stage_values_n(uw, K2, dt, U, n2);
  double f0 = std::sqrt(dae_residual(U, K2, F));
  stats->n_residuals = 0;
  stats->residual_history[stats->n_residuals++] = f0;
  const double tol = std::max(cfg.newton_rtol * f0, cfg.newton_abs_floor);
  double fn = f0;
  bool have_ops = false;
  auto finish = [&]() {
    stats->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - tic).count();
  };
  while (stats->newton_iterations < cfg.newton_maxit) {
    if (fn <= tol) {
      stats->converged = 1;
      finish();
      return;
    }
    if (!have_ops || cfg.jacobian_refresh == 0) {
      build_weights();
      k_dae_opfields<<<grid_for(N), 256, 0, stream>>>((int)N, weights, U, opA);
      count(1);
      stats->jacobian_assemblies += s;
      have_ops = true;
    }
    dae_transformed_solve(dt, F, DK, stats);
    std::vector<double> eye(s * s, 0.0);
    for (int i = 0; i < s; ++i) eye[i * s + i] = 1.0;
    stage_mix_n(eye.data(), DK, K2, true, n2);
    stats->newton_iterations += 1;
    stage_values_n(uw, K2, dt, U, n2);
    fn = std::sqrt(dae_residual(U, K2, F));
    if (stats->n_residuals <= IRKG_MAX_NEWTON) stats->residual_history[stats->n_residuals++] = fn;
  }
  if (fn > tol) {
    finish();
    char msg[160];
    snprintf(msg, sizeof msg, "DAE stage solve stalled after %d iterations (residual %.3e, tol %.3e)",
             cfg.newton_maxit, fn, tol);
    throw SolveError(IRKG_ERR_STEP_FAILURE, msg);
  }
  stats->converged = 1;
  finish();
}

}  // namespace irkg
