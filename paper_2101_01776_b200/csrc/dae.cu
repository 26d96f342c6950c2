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

#include <cstddef>

#include <chrono>
#include <cmath>
#include <cstdio>

#include "engine.h"

namespace irkg {

namespace {

struct P9 {
  double c, E, W, N, S, NE, NW, SE, SW;
};

// rows iy-1, iy, iy+1 of a field: ghost planes in slab mode, periodic wrap
// otherwise (plane_ptr) -- the same values as flat periodic offsets
struct R3 {
  const double *m, *c, *p;
};

__device__ __forceinline__ R3 rows3(const FRef &f, const Grid &g, int iy) {
  R3 r;
  r.c = f.base + (size_t)iy * g.nx;
  r.m = plane_ptr(f, iy - 1, g.ny, g.nx, g.slab);
  r.p = plane_ptr(f, iy + 1, g.ny, g.nx, g.slab);
  return r;
}

// a column and its periodic x-neighbours
struct XO {
  int c, m, p;
};

__device__ __forceinline__ XO xo_of(const Grid &g, int ix) {
  return XO{ix, ix == 0 ? g.nx - 1 : ix - 1, ix == g.nx - 1 ? 0 : ix + 1};
}

__device__ __forceinline__ P9 load9(const R3 &r, const XO &x) {
  P9 v;
  v.c = r.c[x.c];
  v.E = r.c[x.p];
  v.W = r.c[x.m];
  v.N = r.p[x.c];
  v.S = r.m[x.c];
  v.NE = r.p[x.p];
  v.NW = r.p[x.m];
  v.SE = r.m[x.p];
  v.SW = r.m[x.m];
  return v;
}

__device__ __forceinline__ P9 load9(const FRef &f, const Grid &g, int iy, const XO &x) {
  return load9(rows3(f, g, iy), x);
}

// the pinned constraint row: global point 0 (on the rank that holds it)
__device__ __forceinline__ bool pinned(const Grid &g, int p) { return g.pin && p == 0; }

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
__device__ __forceinline__ double ara_lx(const Grid &g, double nu, const FRef &a, double sigma,
                                         const FRef &x, int iy, const XO &o) {
  const P9 A = load9(a, g, iy, o), X = load9(x, g, iy, o);
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

// Traversals of the 9-point kernels.  ROWS_LOOP: one grid row per CTA trip.
// STRIP_LOOP: column strips of DBS points x bands of rows, a CTA walking its
// band row by row with one column per thread, so rows iy-1, iy, iy+1 of its
// strip stay in L1.  Measured at 2048^2 (profiles/r2s4_cfg4_traversal_ab.txt):
// the strips help the stage residual (few fields live per strip: 164 -> 97 us)
// and hurt the 2x2 block operator (six fields: 78 -> 111 us) -- each kernel
// keeps the traversal that is faster for it.
#define ROWS_LOOP(g)                                                  \
  for (int iy = blockIdx.x; iy < (g).ny; iy += gridDim.x)             \
    for (int ix = threadIdx.x; ix < (g).nx; ix += blockDim.x)

struct RowsIter {
  int strips, bands, rows;  // rows per band
};
__device__ __forceinline__ RowsIter rows_iter(const Grid &g) {
  RowsIter r;
  r.strips = (g.nx + DBS - 1) / DBS;
  r.bands = max(1, min(g.ny, (int)gridDim.x / r.strips));
  r.rows = (g.ny + r.bands - 1) / r.bands;
  return r;
}
#define STRIP_LOOP(g)                                                                      \
  for (int sb_ = blockIdx.x, ns_ = rows_iter(g).strips, nr_ = rows_iter(g).rows,           \
           nt_ = rows_iter(g).strips * rows_iter(g).bands;                                 \
       sb_ < nt_; sb_ += gridDim.x)                                                        \
    for (int ix = (sb_ % ns_) * DBS + threadIdx.x, iy = (sb_ / ns_) * nr_,                 \
             ye_ = min((g).ny, (sb_ / ns_ + 1) * nr_);                                     \
         iy < ye_ && ix < (g).nx; ++iy)

// stage fields U_i, W_i (rows of UW) with their ghost planes
struct DaeStageRefs {
  FRef u[MAXS], w[MAXS];
};

// composite residual per stage: [N(U_i, W_i) - k_i ; G(U_i, W_i)] and ||.||^2
__global__ void k_dae_residual(Grid g, double nu, double h2, int s, DaeStageRefs R,
                               const double *__restrict__ K2, double *__restrict__ F2,
                               double *part, unsigned *counter, double *out) {
  const int n = g.n;
  double acc = 0.0;
  STRIP_LOOP(g) {
    const int p = iy * g.nx + ix;
    const XO o = xo_of(g, ix);
    for (int i = 0; i < s; ++i) {
      const P9 u = load9(R.u[i], g, iy, o), w = load9(R.w[i], g, iy, o);
      const double fu = (-jscale(g) * jac_sum(w, u) + nu * lap9(g, u)) - K2[(size_t)i * 2 * n + p];
      const double fw = pinned(g, p) ? w.c : h2 * (lap9(g, w) + u.c);
      F2[(size_t)i * 2 * n + p] = fu;
      F2[(size_t)i * 2 * n + n + p] = fw;
      acc += fu * fu + fw * fw;
    }
  }
  reduce2<DBS>(acc, 0.0, part, gridDim.x, counter, out);
}

// ||G(u, w)||^2 for the state uw = [u; w]
__global__ void k_dae_gnorm(Grid g, double h2, const double *__restrict__ UW, FRef wr, double *part,
                            unsigned *counter, double *out) {
  double acc = 0.0;
  ROWS_LOOP(g) {
    const int p = iy * g.nx + ix;
    const XO o = xo_of(g, ix);
    const P9 w = load9(wr, g, iy, o);
    const double fw = pinned(g, p) ? w.c : h2 * (lap9(g, w) + UW[p]);
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
                          const double *__restrict__ t_in, FRef xr,
                          double *__restrict__ x_out, const GCtrl *skip) {
  const double *x = xr.base;
  const FRef ar = fref(L);
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
      const XO o = xo_of(g, ix);
      const double xc = x[p];
      const double sx = alpha * xc - dt * ara_lx(g, nu, ar, L.sigma, xr, iy, o);
      x_out[p] = xc + OMEGA * (invD * (r - sx));
    }
  }
}

// 1x1 / 2x2 block operator with the Arakawa L (apply_block2x2); b != null: residual + norm
template <int SIZE>
__global__ void k_ara_block_op(Grid g, double nu, double eta, double beta, double phi, double dt,
                               Op l1, Op l2, Op c12, Op c21, FRef z1r, FRef z2r,
                               double *__restrict__ w, const double *__restrict__ b, double *part,
                               unsigned *counter, double *out_norm, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  const int n = g.n;
  const FRef a1 = fref(l1), a2 = fref(l2), a12 = fref(c12), a21 = fref(c21);
  double nrm = 0.0;
  ROWS_LOOP(g) {
    const int p = iy * g.nx + ix;
    const XO o = xo_of(g, ix);
    if (SIZE == 1) {
      const double *z = z1r.base;
      double v = eta * z[p] - dt * ara_lx(g, nu, a1, l1.sigma, z1r, iy, o);
      if (b) {
        v = b[p] - v;
        nrm += v * v;
      }
      w[p] = v;
    } else {
      const double *z1 = z1r.base, *z2 = z2r.base;
      double top = eta * z1[p] - dt * ara_lx(g, nu, a1, l1.sigma, z1r, iy, o) + phi * z2[p];
      double bot = -(beta * beta / phi) * z1[p] + eta * z2[p] -
                   dt * ara_lx(g, nu, a2, l2.sigma, z2r, iy, o);
      if (c12.present) top -= dt * ara_lx(g, nu, a12, c12.sigma, z2r, iy, o);
      if (c21.present) bot -= dt * ara_lx(g, nu, a21, c21.sigma, z1r, iy, o);
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
  FRef yu[MAXS], yw[MAXS];  // y_u,j / y_w,j with ghost planes
};

__global__ void k_dae_backsub(Grid g, double nu, double h2, double dt, DaeBacksub T,
                              const double *__restrict__ G2, const double *__restrict__ Y2,
                              double *__restrict__ ACC) {
  const int n = g.n;
  ROWS_LOOP(g) {
    const int p = iy * g.nx + ix;
    const XO o = xo_of(g, ix);
    for (int r = 0; r < T.rows; ++r) {
      double au = G2[(size_t)(T.row0 + r) * 2 * n + p];
      double aw = G2[(size_t)(T.row0 + r) * 2 * n + n + p];
      for (int q = 0; q < T.njs; ++q) {
        const double *yu = T.yu[q].base;
        const double c = T.coef[r][q];
        if (c != 0.0) au -= c * yu[p];
        const Op od = T.od[r][q];
        if (od.present) {
          au += dt * ara_lx(g, nu, fref(od), od.sigma, T.yu[q], iy, o);
          const P9 w9 = load9(T.yw[q], g, iy, o);
          const double gu = pinned(g, p) ? 0.0 : h2 * yu[p];
          const double gw = pinned(g, p) ? w9.c : h2 * lap9(g, w9);
          aw += dt * (od.sigma * gu + od.sigma * gw);
        }
      }
      ACC[(size_t)r * 2 * n + p] = au;
      ACC[(size_t)r * 2 * n + n + p] = aw;
    }
  }
}

// constraint rhs c = acc_w + dt * sigma * G_u y_u  (G_u row 0 is zero)
__global__ void k_dae_crhs(int n, int pin, double dt, double sigma_h2,
                           const double *__restrict__ accw, const double *__restrict__ yu,
                           double *__restrict__ c) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    c[p] = (pin && p == 0) ? accw[0] : accw[p] + dt * (sigma_h2 * yu[p]);
}

// first row and row count of rank r's slab (the rule of Engine::Engine /
// distributed.slab_range)
__host__ __device__ inline void slab_rows(int planes, int r, int nranks, int &p0, int &nl) {
  const int base = planes / nranks, rem = planes % nranks;
  nl = base + (r < rem ? 1 : 0);
  p0 = r * base + (r < rem ? r : rem);
}

// Poisson step 1: f = c / (sigma h^2) off the pin; f_0 = -sum_{i != 0} f_i
// (pin: this rank's local point 0 is the global pinned point)
__global__ void k_pois_sum(int n, int pin, double inv, const double *__restrict__ c, double *part,
                           unsigned *counter, double *out) {
  double acc = 0.0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    if (!(pin && p == 0)) acc += inv * c[p];
  reduce2<DBS>(acc, 0.0, part, gridDim.x, counter, out);
}

// the pinned point's value on the rank that owns it, 0 elsewhere (summed over ranks)
__global__ void k_pois_pin(int pin, const double *__restrict__ v, double *out) {
  *out = pin ? v[0] : 0.0;
}

__global__ void k_pois_rhs(int n, int pin, double inv, const double *__restrict__ c,
                           const double *__restrict__ sum, double *__restrict__ f) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    f[p] = (pin && p == 0) ? -sum[0] : inv * c[p];
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

// the same division on a pencil: `cols` lines of ny values, line kc = wavenumber kx0 + kc
__global__ void k_pois_scale_cols(int nx, int ny, int kx0, int cols, double ih2x, double ih2y,
                                  cufftDoubleComplex *F) {
  const long long tot = (long long)cols * ny;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tot;
       q += (long long)gridDim.x * blockDim.x) {
    const int kx = kx0 + (int)(q / ny), ky = (int)(q % ny);
    const double sx = sin(M_PI * kx / nx), sy = sin(M_PI * ky / ny);
    const double lam = -4.0 * ih2x * sx * sx - 4.0 * ih2y * sy * sy;
    const double inv = (kx == 0 && ky == 0) ? 0.0 : 1.0 / (lam * (double)nx * (double)ny);
    F[q].x *= inv;
    F[q].y *= inv;
  }
}

// Transposes of the slab -> pencil FFT.  All-to-all block d (sent to / received
// from rank d) holds nylmax x C complex values, row-major [row][wavenumber].
// rows -> send: block d = my rows x the wavenumbers rank d owns
__global__ void k_tr_pack_rows(int nranks, int nyl, int nxh, int C, int nylmax,
                               const cufftDoubleComplex *__restrict__ F,
                               cufftDoubleComplex *__restrict__ S) {
  const long long blk = (long long)nylmax * C, tot = blk * nranks;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const int d = (int)(i / blk);
    const long long r = i % blk;
    const int iy = (int)(r / C), kc = (int)(r % C), kx = d * C + kc;
    cufftDoubleComplex v = {0.0, 0.0};
    if (iy < nyl && kx < nxh) v = F[(size_t)iy * nxh + kx];
    S[i] = v;
  }
}

// recv -> pencil lines: block s = rank s's rows x my wavenumbers; line kc holds all gny rows
__global__ void k_tr_unpack_cols(int nranks, int gny, int C, int cols, int nylmax,
                                 const cufftDoubleComplex *__restrict__ R,
                                 cufftDoubleComplex *__restrict__ Lb) {
  const long long blk = (long long)nylmax * C, tot = blk * nranks;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(i / blk);
    const long long r = i % blk;
    const int iy = (int)(r / C), kc = (int)(r % C);
    int p0, nl;
    slab_rows(gny, s, nranks, p0, nl);
    if (iy < nl && kc < cols) Lb[(size_t)kc * gny + p0 + iy] = R[i];
  }
}

// pencil lines -> send: block d = rank d's rows x my wavenumbers
__global__ void k_tr_pack_cols(int nranks, int gny, int C, int cols, int nylmax,
                               const cufftDoubleComplex *__restrict__ Lb,
                               cufftDoubleComplex *__restrict__ S) {
  const long long blk = (long long)nylmax * C, tot = blk * nranks;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const int d = (int)(i / blk);
    const long long r = i % blk;
    const int iy = (int)(r / C), kc = (int)(r % C);
    int p0, nl;
    slab_rows(gny, d, nranks, p0, nl);
    cufftDoubleComplex v = {0.0, 0.0};
    if (iy < nl && kc < cols) v = Lb[(size_t)kc * gny + p0 + iy];
    S[i] = v;
  }
}

// recv -> rows: block s = my rows x the wavenumbers rank s owns
__global__ void k_tr_unpack_rows(int nranks, int nyl, int nxh, int C, int nylmax,
                                 const cufftDoubleComplex *__restrict__ R,
                                 cufftDoubleComplex *__restrict__ F) {
  const long long blk = (long long)nylmax * C, tot = blk * nranks;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(i / blk);
    const long long r = i % blk;
    const int iy = (int)(r / C), kc = (int)(r % C), kx = s * C + kc;
    if (iy < nyl && kx < nxh) F[(size_t)iy * nxh + kx] = R[i];
  }
}

// y = yt - yt_0 + c_0 / sigma;  out = post * y  (yt0, c0: values at the global pinned point)
__global__ void k_pois_fix(int n, double post, double inv_sigma, const double *__restrict__ yt,
                           const double *__restrict__ yt0, const double *__restrict__ c0,
                           double *__restrict__ out) {
  const double y0 = yt0[0], pin = c0[0] * inv_sigma;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    out[p] = post * ((yt[p] - y0) + pin);
}

// composite true residual of the reordered 4x4 block (src/dae.py:238-253, 307-314):
// out[0] = ||rhs - A x||^2, out[1] = ||rhs||^2; rhs = ACC (2 x 2N), x = Y2 rows r0, r0+1
__global__ void k_dae_block_res(Grid g, double nu, double h2, double eta, double beta, double phi,
                                double dt, Op l1, Op l2, double sig1, double sig2,
                                const double *__restrict__ ACC, FRef x1ur, FRef x1wr, FRef x2ur,
                                FRef x2wr, double *part, unsigned *counter, double *out) {
  const int n = g.n;
  const FRef a1 = fref(l1), a2 = fref(l2);
  double rr = 0.0, bb = 0.0;
  ROWS_LOOP(g) {
    const int p = iy * g.nx + ix;
    const XO o = xo_of(g, ix);
    const double *x1u = x1ur.base, *x2u = x2ur.base;
    const double top1 = eta * x1u[p] - dt * ara_lx(g, nu, a1, l1.sigma, x1ur, iy, o) + phi * x2u[p];
    const double top2 = eta * x2u[p] - dt * ara_lx(g, nu, a2, l2.sigma, x2ur, iy, o) -
                        (beta * beta / phi) * x1u[p];
    const P9 w1 = load9(x1wr, g, iy, o), w2 = load9(x2wr, g, iy, o);
    const double gu1 = pinned(g, p) ? 0.0 : h2 * x1u[p], gu2 = pinned(g, p) ? 0.0 : h2 * x2u[p];
    const double gw1 = pinned(g, p) ? w1.c : h2 * lap9(g, w1);
    const double gw2 = pinned(g, p) ? w2.c : h2 * lap9(g, w2);
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
  const int gny = gplanes;
  dalloc_raw((void **)&ACC, sizeof(double) * 4 * N);
  dalloc_raw((void **)&XU, sizeof(double) * 2 * N);
  dalloc_raw((void **)&CR, sizeof(double) * N);
  dalloc_raw((void **)&PT, sizeof(double) * N);
  h2 = (prob.length / grid.nx) * ((prob.length_y > 0.0 ? prob.length_y : prob.length) / gny);
  const int nxh = grid.nx / 2 + 1;
  cufftHandle p1, p2;
  if (!slab()) {
    dalloc_raw((void **)&fft_buf, sizeof(cufftDoubleComplex) * (size_t)gny * nxh);
    if (cufftPlan2d(&p1, gny, grid.nx, CUFFT_D2Z) != CUFFT_SUCCESS ||
        cufftPlan2d(&p2, gny, grid.nx, CUFFT_Z2D) != CUFFT_SUCCESS)
      throw CudaError("cufftPlan2d failed");
    fft_fwd = (int)p1;
    fft_inv = (int)p2;
    return;
  }
  // slab -> pencil layout: rank r transforms x-wavenumbers [r C, (r+1) C)
  tr_C = (nxh + nranks - 1) / nranks;
  tr_cols = std::max(0, std::min(tr_C, nxh - rank * tr_C));
  tr_nylmax = (gny + nranks - 1) / nranks;
  const size_t blk = (size_t)tr_nylmax * tr_C;  // complex values per all-to-all block
  dalloc_raw((void **)&fft_buf, sizeof(cufftDoubleComplex) * (size_t)grid.ny * nxh);
  dalloc_raw((void **)&tr_send, sizeof(cufftDoubleComplex) * blk * nranks);
  dalloc_raw((void **)&tr_recv, sizeof(cufftDoubleComplex) * blk * nranks);
  dalloc_raw((void **)&tr_lines, sizeof(cufftDoubleComplex) * (size_t)tr_C * gny);
  int nrow = grid.nx, ncol = gny;
  if (cufftPlanMany(&p1, 1, &nrow, nullptr, 1, grid.nx, nullptr, 1, nxh, CUFFT_D2Z, grid.ny) !=
          CUFFT_SUCCESS ||
      cufftPlanMany(&p2, 1, &nrow, nullptr, 1, nxh, nullptr, 1, grid.nx, CUFFT_Z2D, grid.ny) !=
          CUFFT_SUCCESS)
    throw CudaError("cufftPlanMany (rows) failed");
  fft_fwd = (int)p1;
  fft_inv = (int)p2;
  if (tr_cols > 0) {
    cufftHandle p3;
    if (cufftPlanMany(&p3, 1, &ncol, nullptr, 1, gny, nullptr, 1, gny, CUFFT_Z2Z, tr_cols) !=
        CUFFT_SUCCESS)
      throw CudaError("cufftPlanMany (columns) failed");
    fft_col = (int)p3;
  }
}

void Engine::dae_fini() {
  if (fft_fwd >= 0) cufftDestroy((cufftHandle)fft_fwd);
  if (fft_inv >= 0) cufftDestroy((cufftHandle)fft_inv);
  if (fft_col >= 0) cufftDestroy((cufftHandle)fft_col);
  void *bufs[] = {ACC, XU, CR, PT, fft_buf, tr_send, tr_recv, tr_lines};
  for (void *b : bufs)
    if (b) cudaFree(b);
}

int Engine::dae_grid() const { return grid.ny < sms * 8 ? grid.ny : sms * 8; }

// out = post * (sigma G_w)^{-1} c  -- _ConstraintSolver.solve, src/dae.py:122-126.
void Engine::constraint_solve(double sigma, const double *c, double *out, double post) {
  if (sigma == 0.0) throw SolveError(IRKG_ERR_INDEX, "constraint Jacobian is singular");
  if (slab()) {
    constraint_solve_slab(sigma, c, out, post);
    return;
  }
  const int n = (int)N;
  const double inv = 1.0 / (sigma * h2);
  k_pois_sum<<<dae_grid(), DBS, 0, stream>>>(n, 1, inv, c, part, counter, &scal_dev[4]);
  k_pois_rhs<<<grid_for(N), 256, 0, stream>>>(n, 1, inv, c, &scal_dev[4], PT);
  cufftSetStream((cufftHandle)fft_fwd, stream);
  cufftSetStream((cufftHandle)fft_inv, stream);
  if (cufftExecD2Z((cufftHandle)fft_fwd, PT, (cufftDoubleComplex *)fft_buf) != CUFFT_SUCCESS)
    throw CudaError("cufftExecD2Z failed");
  k_pois_scale<<<grid_for((long long)grid.ny * (grid.nx / 2 + 1)), 256, 0, stream>>>(
      grid.nx, grid.ny, grid.ih2[0], grid.ih2[1], (cufftDoubleComplex *)fft_buf);
  if (cufftExecZ2D((cufftHandle)fft_inv, (cufftDoubleComplex *)fft_buf, PT) != CUFFT_SUCCESS)
    throw CudaError("cufftExecZ2D failed");
  k_pois_fix<<<grid_for(N), 256, 0, stream>>>(n, post, 1.0 / sigma, PT, PT, c, out);
  count(4);
}

// The same solve on y-slabs: a slab -> pencil transpose FFT.  Every rank
// transforms its own rows along x, one all-to-all gives rank r the
// x-wavenumbers [r C, (r+1) C) with all of y (blocks padded to the largest
// slab), the y transforms and the division by the Laplacian's eigenvalues
// run on those pencils, and the way back mirrors it: O(N/P) work and
// 2 x 16 N/P bytes on the links per rank and solve, no global vector
// anywhere.  The zero-mean shift and the pinned row (global point 0, owned by
// the rank with grid.pin) travel in two small all-reduces.
void Engine::constraint_solve_slab(double sigma, const double *c, double *out, double post) {
  const int n = (int)N, nx = grid.nx, nyl = grid.ny, gny = gplanes, nxh = nx / 2 + 1;
  const double inv = 1.0 / (sigma * h2);
  auto *FB = (cufftDoubleComplex *)fft_buf;
  auto *SB = (cufftDoubleComplex *)tr_send, *RB = (cufftDoubleComplex *)tr_recv;
  auto *LB = (cufftDoubleComplex *)tr_lines;
  const long long blk = (long long)tr_nylmax * tr_C;
  // scal[4] = sum_{i != 0} f_i, scal[5] = c at global point 0 (pin rank only)
  k_pois_sum<<<dae_grid(), DBS, 0, stream>>>(n, grid.pin, inv, c, part, counter, &scal_dev[4]);
  k_pois_pin<<<1, 1, 0, stream>>>(grid.pin, c, &scal_dev[5]);
  allreduce(&scal_dev[4], 2);
  k_pois_rhs<<<grid_for(N), 256, 0, stream>>>(n, grid.pin, inv, c, &scal_dev[4], PT);
  cufftSetStream((cufftHandle)fft_fwd, stream);
  cufftSetStream((cufftHandle)fft_inv, stream);
  if (cufftExecD2Z((cufftHandle)fft_fwd, PT, FB) != CUFFT_SUCCESS)
    throw CudaError("cufftExecD2Z (rows) failed");
  const int gp = grid_for((long long)nranks * blk);
  k_tr_pack_rows<<<gp, 256, 0, stream>>>(nranks, nyl, nxh, tr_C, tr_nylmax, FB, SB);
  comm->alltoall(tr_send, tr_recv, 2 * blk, stream);
  k_tr_unpack_cols<<<gp, 256, 0, stream>>>(nranks, gny, tr_C, tr_cols, tr_nylmax, RB, LB);
  if (tr_cols > 0) {
    cufftSetStream((cufftHandle)fft_col, stream);
    if (cufftExecZ2Z((cufftHandle)fft_col, LB, LB, CUFFT_FORWARD) != CUFFT_SUCCESS)
      throw CudaError("cufftExecZ2Z failed");
    k_pois_scale_cols<<<grid_for((long long)tr_cols * gny), 256, 0, stream>>>(
        nx, gny, rank * tr_C, tr_cols, grid.ih2[0], grid.ih2[1], LB);
    if (cufftExecZ2Z((cufftHandle)fft_col, LB, LB, CUFFT_INVERSE) != CUFFT_SUCCESS)
      throw CudaError("cufftExecZ2Z failed");
  }
  k_tr_pack_cols<<<gp, 256, 0, stream>>>(nranks, gny, tr_C, tr_cols, tr_nylmax, LB, SB);
  comm->alltoall(tr_send, tr_recv, 2 * blk, stream);
  k_tr_unpack_rows<<<gp, 256, 0, stream>>>(nranks, nyl, nxh, tr_C, tr_nylmax, RB, FB);
  if (cufftExecZ2D((cufftHandle)fft_inv, FB, PT) != CUFFT_SUCCESS)
    throw CudaError("cufftExecZ2D (rows) failed");
  // scal[8] = yt at global point 0
  k_pois_pin<<<1, 1, 0, stream>>>(grid.pin, PT, &scal_dev[8]);
  allreduce(&scal_dev[8], 1);
  k_pois_fix<<<grid_for(N), 256, 0, stream>>>(n, post, 1.0 / sigma, PT, &scal_dev[8],
                                              &scal_dev[5], out);
  count(9);
  counters.halo_exchanges += 2;
}

void Engine::ara_jacobi_chain(const Op &L, double alpha, double dt, int inner, const VecIn &vin,
                              int in_off, const double *zc, double cpl, double *x_out,
                              const GCtrl *skip) {
  if (ara_chain_fused(L, alpha, dt, inner, vin, in_off, zc, cpl, x_out, skip)) return;
  const int gb = dae_grid();
  double *tbuf = zc ? tmp_t : nullptr;
  auto dst = [&](int i) { return ((inner - i) % 2 == 0) ? x_out : tmp_x; };
  const Op Lr = opref(L);
  k_ara_jac<<<gb, DBS, 0, stream>>>(grid, kp.nu, Lr, alpha, dt, vin, in_off, zc, cpl, tbuf, nullptr,
                                    FRef{nullptr, nullptr, nullptr}, dst(1), skip);
  count(1);
  for (int i = 2; i <= inner; ++i) {
    if (slab()) exchange(R_JX, dst(i - 1), 1);
    k_ara_jac<<<gb, DBS, 0, stream>>>(grid, kp.nu, Lr, alpha, dt, vin, in_off, nullptr, 0.0, nullptr,
                                      tbuf, ref(dst(i - 1)), dst(i), skip);
    count(1);
  }
}

void Engine::ara_block_op(const BlockSpec &B, const double *z, double *w, const double *b,
                          double *out_norm, const GCtrl *skip) {
  const int gb = dae_grid();
  if (slab()) {
    exchange(R_X0, z, 1);
    if (B.size == 2) exchange(R_X1, z + N, 1);
  }
  const FRef z1 = ref(z), z2 = B.size == 2 ? ref(z + N) : FRef{nullptr, nullptr, nullptr};
  const Op l1 = opref(B.l1), l2 = opref(B.l2), c12 = opref(B.c12), c21 = opref(B.c21);
  if (B.size == 1)
    k_ara_block_op<1><<<gb, DBS, 0, stream>>>(grid, kp.nu, B.eta, B.beta, B.phi, B.dt, l1, l2,
                                              c12, c21, z1, z2, w, b, part, counter, out_norm,
                                              skip);
  else
    k_ara_block_op<2><<<gb, DBS, 0, stream>>>(grid, kp.nu, B.eta, B.beta, B.phi, B.dt, l1, l2,
                                              c12, c21, z1, z2, w, b, part, counter, out_norm,
                                              skip);
  count(1);
  if (b) allreduce(out_norm, 1);
}

double Engine::dae_residual(const double *UW, const double *K2, double *F2) {
  DaeStageRefs R{};
  for (int i = 0; i < s; ++i) {
    const double *u = UW + (size_t)i * 2 * N, *w = u + N;
    if (slab()) {
      exchange(R_STAGE + i, u, 1);
      exchange(R_DW + i, w, 1);
    }
    R.u[i] = ref(u);
    R.w[i] = ref(w);
  }
  k_dae_residual<<<dae_grid(), DBS, 0, stream>>>(grid, kp.nu, h2, s, R, K2, F2, part, counter,
                                                 &scal_dev[0]);
  count(1);
  allreduce(&scal_dev[0], 1);
  double v = 0.0;
  v = read_scalar();
  return v;
}

double Engine::dae_gnorm(const double *UW) {
  if (slab()) exchange(R_DG, UW + N, 1);
  k_dae_gnorm<<<dae_grid(), DBS, 0, stream>>>(grid, h2, UW, ref(UW + N), part, counter,
                                              &scal_dev[0]);
  count(1);
  allreduce(&scal_dev[0], 1);
  double v = 0.0;
  v = read_scalar();
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
      bool any_od = false;
      for (int r = 0; r < 2; ++r) {
        T.coef[r][q] = tab.r[(off + r) * IRKG_MAX_STAGES + j];
        T.od[r][q] = opref(op_of(od_slot[off + r][j]));
        any_od |= T.od[r][q].present != 0;
      }
      const double *yu = Y + (size_t)j * n2, *yw = yu + N;
      if (slab() && any_od) {
        exchange(R_Y + j, yu, 1);
        exchange(R_DYW + j, yw, 1);
      }
      T.yu[q] = any_od ? ref(yu) : FRef{yu, nullptr, nullptr};
      T.yw[q] = any_od ? ref(yw) : FRef{yw, nullptr, nullptr};
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
    KrylovOut rep = gmres(B, RHS, XU, cfg.krylov_rtol, cfg.krylov_maxit, cfg.restart, false);
    const long long diff_solves = rep.precond_applications;
    // y_u -> Y rows; constraint solves for y_w (src/dae.py:274-278)
    double *Y1 = Y + (size_t)off * n2, *Y2r = Y + (size_t)(off + 1) * n2;
    check(cudaMemcpyAsync(Y1, XU, N * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    check(cudaMemcpyAsync(Y2r, XU + N, N * sizeof(double), cudaMemcpyDeviceToDevice, stream));
    const double sig1 = op_sigma[diag_slot[off]], sig2 = op_sigma[diag_slot[off + 1]];
    k_dae_crhs<<<grid_for(N), 256, 0, stream>>>((int)N, grid.pin, dt, sig1 * h2, ACC + N, XU, CR);
    constraint_solve(sig1, CR, Y1 + N, -1.0 / dt);
    k_dae_crhs<<<grid_for(N), 256, 0, stream>>>((int)N, grid.pin, dt, sig2 * h2, ACC + n2 + N,
                                                XU + N, CR);
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
    if (slab()) {
      exchange(R_DB + 0, Y1, 1);
      exchange(R_DB + 1, Y1 + N, 1);
      exchange(R_DB + 2, Y2r, 1);
      exchange(R_DB + 3, Y2r + N, 1);
    }
    k_dae_block_res<<<dae_grid(), DBS, 0, stream>>>(grid, kp.nu, h2, B.eta, B.beta, B.phi, dt,
                                                    opref(B.l1), opref(B.l2), sig1, sig2, ACC,
                                                    ref(Y1), ref(Y1 + N), ref(Y2r), ref(Y2r + N),
                                                    part, counter, &scal_dev[6]);
    count(1);
    allreduce(&scal_dev[6], 2);
    // (through the pinned control-block mirror: a pageable destination staged the copy)
    double *rb = &ctrl_host->rr;  // rr, scalar: two adjacent doubles of the host mirror
    static_assert(offsetof(GCtrl, scalar) == offsetof(GCtrl, rr) + sizeof(double), "GCtrl layout");
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
      if (slab())  // operator fields feed the 9-point stencils
        for (int o = 0; o < nops; ++o)
          if (!op_zero[o]) exchange(R_OP + o, opA + (size_t)o * N, jhalo());
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
