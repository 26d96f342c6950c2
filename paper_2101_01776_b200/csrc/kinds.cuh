// kinds.cuh -- matrix-free problem kinds: N(u), L(a, sigma) x, diag L, f(U).
//
// Replaces the reference's problem callbacks OdeSystem.rhs / .linearize
// (src/nonlinear.py:35-48) and the CSR weighted sums of
// build_variant_jacobian / combine (src/nonlinear.py:129-142,
// src/sparsela.py:106-128).  Every Jacobian of the supported kinds is affine
// in one pointwise function f(U) of the stage state, so
//      sum_k w_k L(U_k)  ==  L_eff(a, sigma),  a = sum_k w_k f(U_k),
//                                              sigma = sum_k w_k,
// and an operator is carried on the device as one coefficient field a plus
// the scalar sigma.
//
//   kind     N(u)                              L_eff(a,sigma) x                f(U)
//   nldiff   Lap(u + u^3/3)                    Lap(a x)                        1 + U^2
//   burgers  -Dsum(u^2/2) + nu Lap u           -Dsum(a x) + sigma nu Lap x     U
//   rad      nu Lap u + c Dsum u + lam u       sigma (nu Lap x + c Dsum x)     lam + 2 mu U
//              + mu u^2                          + a x
//
// Lap = periodic 2d+1-point Laplacian, Dsum = sum of periodic central
// differences, x fastest: p = (iz*ny + iy)*nx + ix (src/problems.py:238-239).
#pragma once
#include <cuda_runtime.h>

// Checked build (python -m paper_2101_01776_b200._build --checked, -DIRKG_CHECKED):
// device-side bounds/invariant checks that trap with the failing line -- the
// stand-in for compute-sanitizer, which this GPU pool does not allow.  They
// compile to nothing in the production library.
#ifdef IRKG_CHECKED
#include <cstdio>
#define IRKG_DCHECK(cond)                                                               \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("IRKG_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,   \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                              \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define IRKG_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace irkg {

enum { KIND_NLDIFF = 0, KIND_BURGERS = 1, KIND_RAD = 2, KIND_ARAKAWA = 3 };

struct Grid {
  int nx, ny, nz;  // local extents (ny or nz is the slab axis when partitioned)
  int nxy;         // nx*ny
  int n;           // nx*ny*nz local points
  double ih2[3];   // 1/h^2 per axis, 0 for an axis of extent 1
  double i2h[3];   // 1/(2h) per axis, 0 for an axis of extent 1
  double lapdiag;  // diagonal of Lap: -2 * sum ih2
  int slab;        // 1: slab-partitioned (ghost planes), 0: periodic wrap locally
  int pin;         // 1: this rank holds global point 0 (the DAE constraint's pinned row)
};

// Depth of the ghost-plane buffers (>= Jacobi halo K-1 for K <= 6, and the
// extended halo 2(K-1)+1 of the communication-avoiding 2-D chains for K <= 4).
constexpr int GH = 8;

// A field and its ghost planes along the slab (slowest) axis.  In slab mode
// plane -d (1 <= d <= GH) is lo + (GH - d) * P and plane nl + e is hi + e * P;
// in single-rank mode the accessor wraps periodically inside base.
struct FRef {
  const double *base;
  const double *lo;
  const double *hi;
};

__device__ __forceinline__ const double *plane_ptr(const FRef &f, int s, int nl, int P, int slab) {
  if (!slab) {
    s = s < 0 ? s + nl : (s >= nl ? s - nl : s);
    IRKG_DCHECK(s >= 0 && s < nl);
    return f.base + (size_t)s * P;
  }
  IRKG_DCHECK(s >= -GH && s < nl + GH);
  if (s < 0) {
    IRKG_DCHECK(f.lo != nullptr);
    return f.lo + (size_t)(s + GH) * P;
  }
  if (s >= nl) {
    IRKG_DCHECK(f.hi != nullptr);
    return f.hi + (size_t)(s - nl) * P;
  }
  return f.base + (size_t)s * P;
}

struct KindParams {
  double nu, c, lam, mu;
};

// Row-structured traversal: a "row" is one x-line (fixed iy, iz).  Kernels
// loop rows across CTAs and x across threads, so the periodic neighbour
// offsets are computed once per row (no per-element integer division).
struct RowCtx {
  int base;      // row * nx
  int dym, dyp;  // element offsets to the y-neighbour rows
  int dzm, dzp;  // element offsets to the z-neighbour planes
};

template <int NDIM>
__device__ __forceinline__ RowCtx row_ctx(const Grid &g, int row) {
  RowCtx rc;
  rc.base = row * g.nx;
  rc.dym = rc.dyp = rc.dzm = rc.dzp = 0;
  if (NDIM >= 2) {
    const int iy = (NDIM == 3) ? row % g.ny : row;
    rc.dym = (iy == 0) ? (g.ny - 1) * g.nx : -g.nx;
    rc.dyp = (iy == g.ny - 1) ? -(g.ny - 1) * g.nx : g.nx;
    if (NDIM == 3) {
      const int iz = row / g.ny;
      rc.dzm = (iz == 0) ? (g.nz - 1) * g.nxy : -g.nxy;
      rc.dzp = (iz == g.nz - 1) ? -(g.nz - 1) * g.nxy : g.nxy;
    }
  }
  return rc;
}

template <int NDIM>
__device__ __forceinline__ int row_neighbours(const Grid &g, const RowCtx &rc, int ix, int nb[6]) {
  const int p = rc.base + ix;
  nb[0] = p + (ix == 0 ? g.nx - 1 : -1);
  nb[1] = p + (ix == g.nx - 1 ? 1 - g.nx : 1);
  nb[2] = p + rc.dym;
  nb[3] = p + rc.dyp;
  nb[4] = p + rc.dzm;
  nb[5] = p + rc.dzp;
  return p;
}

// Periodic neighbours of p: [xm, xp, ym, yp, zm, zp].
template <int NDIM>
__device__ __forceinline__ void neighbours(const Grid &g, int p, int nb[6]) {
  int ix = p % g.nx;
  nb[0] = p + (ix == 0 ? g.nx - 1 : -1);
  nb[1] = p + (ix == g.nx - 1 ? 1 - g.nx : 1);
  if (NDIM >= 2) {
    int r = p / g.nx;
    int iy = (NDIM == 3) ? r % g.ny : r;
    nb[2] = p + (iy == 0 ? (g.ny - 1) * g.nx : -g.nx);
    nb[3] = p + (iy == g.ny - 1 ? -(g.ny - 1) * g.nx : g.nx);
    if (NDIM == 3) {
      int iz = r / g.ny;
      nb[4] = p + (iz == 0 ? (g.nz - 1) * g.nxy : -g.nxy);
      nb[5] = p + (iz == g.nz - 1 ? -(g.nz - 1) * g.nxy : g.nxy);
    }
  }
}

// sum over axes of ih2 * (v[p+e] + v[p-e] - 2 v[p]) for a value functor
template <int NDIM, class F>
__device__ __forceinline__ double lap_of(const Grid &g, const int nb[6], double vp, F v) {
  double s = g.ih2[0] * (v(nb[0]) + v(nb[1]) - 2.0 * vp);
  if (NDIM >= 2) s += g.ih2[1] * (v(nb[2]) + v(nb[3]) - 2.0 * vp);
  if (NDIM == 3) s += g.ih2[2] * (v(nb[4]) + v(nb[5]) - 2.0 * vp);
  return s;
}

template <int NDIM, class F>
__device__ __forceinline__ double dsum_of(const Grid &g, const int nb[6], F v) {
  double s = g.i2h[0] * (v(nb[1]) - v(nb[0]));
  if (NDIM >= 2) s += g.i2h[1] * (v(nb[3]) - v(nb[2]));
  if (NDIM == 3) s += g.i2h[2] * (v(nb[5]) - v(nb[4]));
  return s;
}

// N(u)[p]
template <int KIND, int NDIM>
__device__ __forceinline__ double rhs_at(const Grid &g, const KindParams &kp,
                                         const double *__restrict__ u, int p, const int nb[6]) {
  double up = u[p];
  if (KIND == KIND_NLDIFF) {
    auto phi = [&](int q) {
      double v = u[q];
      return v + v * v * v / 3.0;
    };
    return lap_of<NDIM>(g, nb, up + up * up * up / 3.0, phi);
  } else if (KIND == KIND_BURGERS) {
    auto half_sq = [&](int q) {
      double v = u[q];
      return 0.5 * v * v;
    };
    auto val = [&](int q) { return u[q]; };
    return -dsum_of<NDIM>(g, nb, half_sq) + kp.nu * lap_of<NDIM>(g, nb, up, val);
  } else {
    auto val = [&](int q) { return u[q]; };
    return kp.nu * lap_of<NDIM>(g, nb, up, val) + kp.c * dsum_of<NDIM>(g, nb, val) +
           kp.lam * up + kp.mu * up * up;
  }
}

// f(U): the pointwise function whose weighted sum is the operator field
template <int KIND>
__device__ __forceinline__ double field_of(const KindParams &kp, double U) {
  if (KIND == KIND_NLDIFF) return 1.0 + U * U;
  if (KIND == KIND_BURGERS) return U;
  return kp.lam + 2.0 * kp.mu * U;
}

// (L_eff(a, sigma) x)[p]
template <int KIND, int NDIM>
__device__ __forceinline__ double lx_at(const Grid &g, const KindParams &kp,
                                        const double *__restrict__ a, double sigma,
                                        const double *__restrict__ x, int p, const int nb[6]) {
  if (KIND == KIND_NLDIFF) {
    auto ax = [&](int q) { return a[q] * x[q]; };
    return lap_of<NDIM>(g, nb, a[p] * x[p], ax);
  } else if (KIND == KIND_BURGERS) {
    auto ax = [&](int q) { return a[q] * x[q]; };
    auto xv = [&](int q) { return x[q]; };
    return -dsum_of<NDIM>(g, nb, ax) + sigma * kp.nu * lap_of<NDIM>(g, nb, x[p], xv);
  } else {
    auto xv = [&](int q) { return x[q]; };
    return sigma * (kp.nu * lap_of<NDIM>(g, nb, x[p], xv) + kp.c * dsum_of<NDIM>(g, nb, xv)) +
           a[p] * x[p];
  }
}

// ---- value-based forms (register-sliding kernels, stencil.cu) ----------
// A field sampled at a point and its periodic neighbours [xm, xp, ym, yp, zm, zp].
struct Nb {
  double c;
  double v[6];
};

template <int NDIM, class F>
__device__ __forceinline__ double lap_nb(const Grid &g, const Nb &f, F op) {
  double cp = op(f.c, 6);
  double s = g.ih2[0] * (op(f.v[0], 0) + op(f.v[1], 1) - 2.0 * cp);
  if (NDIM >= 2) s += g.ih2[1] * (op(f.v[2], 2) + op(f.v[3], 3) - 2.0 * cp);
  if (NDIM == 3) s += g.ih2[2] * (op(f.v[4], 4) + op(f.v[5], 5) - 2.0 * cp);
  return s;
}

template <int NDIM, class F>
__device__ __forceinline__ double dsum_nb(const Grid &g, const Nb &f, F op) {
  double s = g.i2h[0] * (op(f.v[1], 1) - op(f.v[0], 0));
  if (NDIM >= 2) s += g.i2h[1] * (op(f.v[3], 3) - op(f.v[2], 2));
  if (NDIM == 3) s += g.i2h[2] * (op(f.v[5], 5) - op(f.v[4], 4));
  return s;
}

// N(u) from neighbour values
template <int KIND, int NDIM>
__device__ __forceinline__ double rhs_nb(const Grid &g, const KindParams &kp, const Nb &u) {
  if (KIND == KIND_NLDIFF) {
    return lap_nb<NDIM>(g, u, [](double v, int) { return v + v * v * v / 3.0; });
  } else if (KIND == KIND_BURGERS) {
    return -dsum_nb<NDIM>(g, u, [](double v, int) { return 0.5 * v * v; }) +
           kp.nu * lap_nb<NDIM>(g, u, [](double v, int) { return v; });
  } else {
    const double up = u.c;
    return kp.nu * lap_nb<NDIM>(g, u, [](double v, int) { return v; }) +
           kp.c * dsum_nb<NDIM>(g, u, [](double v, int) { return v; }) + kp.lam * up +
           kp.mu * up * up;
  }
}

// L_eff(a, sigma) x from neighbour values of a and x
template <int KIND, int NDIM>
__device__ __forceinline__ double lx_nb(const Grid &g, const KindParams &kp, const Nb &a,
                                        double sigma, const Nb &x) {
  if (KIND == KIND_NLDIFF) {
    return lap_nb<NDIM>(g, x, [&](double v, int k) { return (k == 6 ? a.c : a.v[k]) * v; });
  } else if (KIND == KIND_BURGERS) {
    return -dsum_nb<NDIM>(g, x, [&](double v, int k) { return (k == 6 ? a.c : a.v[k]) * v; }) +
           sigma * kp.nu * lap_nb<NDIM>(g, x, [](double v, int) { return v; });
  } else {
    return sigma * (kp.nu * lap_nb<NDIM>(g, x, [](double v, int) { return v; }) +
                    kp.c * dsum_nb<NDIM>(g, x, [](double v, int) { return v; })) +
           a.c * x.c;
  }
}

// whether L_eff reads the coefficient field at neighbour points
template <int KIND>
__device__ __forceinline__ constexpr bool a_stencil() {
  return KIND != KIND_RAD;
}

// diagonal entry of L_eff(a, sigma) at p
template <int KIND>
__device__ __forceinline__ double ldiag_at(const Grid &g, const KindParams &kp,
                                           const double *__restrict__ a, double sigma, int p) {
  if (KIND == KIND_NLDIFF) return g.lapdiag * a[p];
  if (KIND == KIND_BURGERS) return sigma * kp.nu * g.lapdiag;
  return sigma * kp.nu * g.lapdiag + a[p];
}

// coefficients of L_eff(a, sigma) at point p: centre and neighbours
// [xm, xp, ym, yp] (2-D) -- the same operators as kinds.cuh / lx_nb
template <int KIND>
__device__ __forceinline__ void stencil_row(const Grid &g, const KindParams &kp, const double *a,
                                            double sig, int p, const int nb[4], double &cc,
                                            double cn[4]) {
  const double ih2[2] = {g.ih2[0], g.ih2[1]};
  const double i2h[2] = {g.i2h[0], g.i2h[1]};
  if (KIND == KIND_NLDIFF) {  // Lap(a x)
    cc = g.lapdiag * a[p];
    for (int d = 0; d < 2; ++d) {
      cn[2 * d] = ih2[d] * a[nb[2 * d]];
      cn[2 * d + 1] = ih2[d] * a[nb[2 * d + 1]];
    }
  } else if (KIND == KIND_BURGERS) {  // -Dsum(a x) + sigma nu Lap x
    cc = sig * kp.nu * g.lapdiag;
    for (int d = 0; d < 2; ++d) {
      cn[2 * d] = i2h[d] * a[nb[2 * d]] + sig * kp.nu * ih2[d];
      cn[2 * d + 1] = -i2h[d] * a[nb[2 * d + 1]] + sig * kp.nu * ih2[d];
    }
  } else {  // sigma (nu Lap x + c Dsum x) + a x
    cc = sig * kp.nu * g.lapdiag + a[p];
    for (int d = 0; d < 2; ++d) {
      cn[2 * d] = sig * (kp.nu * ih2[d] - kp.c * i2h[d]);
      cn[2 * d + 1] = sig * (kp.nu * ih2[d] + kp.c * i2h[d]);
    }
  }
}


}  // namespace irkg
