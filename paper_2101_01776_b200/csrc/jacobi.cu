// jacobi.cu -- temporally blocked damped-Jacobi inner solves (2-D).
//
// ShiftedSolver(alpha, I, L, dt, inner=K).solve(r) (src/irk_core.py:117-123):
//     x_0 = 0;  x_m = x_{m-1} + (2/3) D^{-1} (r - (alpha I - dt L) x_{m-1}),  m = 1..K
// computed in ONE pass over the grid instead of K: every warp owns a strip of
// 32 columns and slides along y; sweep m runs one row behind sweep m-1 and
// keeps its last three output rows in registers, so all K sweeps are fused
// with no intermediate x written to memory (temporal blocking, halo K-1).
// x-neighbours come from warp shuffles; the valid columns shrink by one per
// sweep on each side, so a warp emits 34-2K columns.  The inputs r (= scale *
// basis slot j [+ coupling * z1 for the second block row]) and the operator
// field a are read once; x_K is written once:  3-4 passes of N instead of
// 4K-1.  Inputs are prefetched PF rows ahead (register FIFO) for HBM MLP.
#include "engine.h"

namespace irkg {

namespace {

constexpr int JW = 4;   // warps per CTA
constexpr int JPF = 4;  // prefetch depth (rows)

__device__ __forceinline__ double shfl_up1(double v) {
  return __shfl_sync(0xffffffffu, v, (threadIdx.x + 31) & 31);
}
__device__ __forceinline__ double shfl_dn1(double v) {
  return __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31);
}

// (L_eff x) at a point from own-column rows (m, c, p) and x-neighbours
template <int KIND>
__device__ __forceinline__ double lx_col(const Grid &g, const KindParams &kp, double sigma,
                                         double am, double ac, double ap, double xm, double xc,
                                         double xp) {
  if (KIND == KIND_NLDIFF) {
    const double axc = ac * xc;
    const double axl = shfl_up1(axc), axr = shfl_dn1(axc);
    return g.ih2[0] * (axl + axr - 2.0 * axc) + g.ih2[1] * (am * xm + ap * xp - 2.0 * axc);
  } else if (KIND == KIND_BURGERS) {
    const double axc = ac * xc;
    const double axl = shfl_up1(axc), axr = shfl_dn1(axc);
    const double xl = shfl_up1(xc), xr = shfl_dn1(xc);
    const double adv = g.i2h[0] * (axr - axl) + g.i2h[1] * (ap * xp - am * xm);
    const double lap = g.ih2[0] * (xl + xr - 2.0 * xc) + g.ih2[1] * (xm + xp - 2.0 * xc);
    return -adv + sigma * kp.nu * lap;
  } else {
    const double xl = shfl_up1(xc), xr = shfl_dn1(xc);
    const double lap = g.ih2[0] * (xl + xr - 2.0 * xc) + g.ih2[1] * (xm + xp - 2.0 * xc);
    const double ds = g.i2h[0] * (xr - xl) + g.i2h[1] * (xp - xm);
    return sigma * (kp.nu * lap + kp.c * ds) + ac * xc;
  }
}

template <int KIND>
__device__ __forceinline__ double diag_of(const Grid &g, const KindParams &kp, double a,
                                          double sigma) {
  if (KIND == KIND_NLDIFF) return g.lapdiag * a;
  if (KIND == KIND_BURGERS) return sigma * kp.nu * g.lapdiag;
  return sigma * kp.nu * g.lapdiag + a;
}

}  // namespace

template <int KIND, int K>
__global__ void __launch_bounds__(JW * 32)
    k_jacobi_chain2d(Grid g, KindParams kp, Op L, double alpha, double dt, VecIn vin, int in_off,
                     FRef zcr, double cpl, double *__restrict__ x_out,
                     int span, GCtrl *flag_ctrl, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  constexpr int H = K - 1;
  constexpr int WCOLS = 32 - 2 * H;  // valid output columns per warp
  double scale;
  const FRef inr = vin_resolve(vin, in_off, scale);
  const FRef ar = fref(L);
  const bool has_zc = zcr.base != nullptr;
  const int lane = threadIdx.x & 31;
  const int wtile = blockIdx.x * JW + (threadIdx.x >> 5);
  const int x0 = wtile * WCOLS;
  if (x0 >= g.nx) return;  // whole warp idle
  int col = x0 - H + lane;
  col = col < 0 ? col + g.nx : (col >= g.nx ? col - g.nx : col);
  // degenerate tiny grids: a column may alias another lane's; still correct
  // because every lane computes its own column's values.
  const bool valid_lane = (lane >= H) && (lane < 32 - H) && (x0 - H + lane < g.nx);
  const int y0 = blockIdx.y * span;
  const int y1 = min(g.ny, y0 + span);
  const double sig = L.sigma;
  const int ny = g.ny;

  // windows (rows relative to the current input row t)
  double A[K + 1];   // a rows t-K .. t
  double ID[K + 1];  // 1/D rows t-K .. t (D = alpha - dt diag L)
  double R[K];       // r rows t-K+1 .. t
  double X[K][3];    // X[m][.]: sweep m (1..K-1) outputs rows rho_m-2, rho_m-1, rho_m
#pragma unroll
  for (int i = 0; i <= K; ++i) A[i] = ID[i] = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) R[i] = 0.0;
#pragma unroll
  for (int m = 0; m < K; ++m) X[m][0] = X[m][1] = X[m][2] = 0.0;
  // two statically named prefetch banks of JPF rows each (no register moves
  // of in-flight load destinations, which would stall on the scoreboard)
  double pa[JPF], pr[JPF], qa[JPF], qr[JPF];
  const int t0 = y0 - H, t1 = y1 + H;  // input rows [t0, t1)
  auto load_row = [&](int t, double &av, double &rv) {
    if (t < t1) {
      double r;
      if (!g.slab) {
        const int p = (t < 0 ? t + ny : (t >= ny ? t - ny : t)) * g.nx + col;
        av = ar.base[p];
        r = scale * inr.base[p];
        if (has_zc) r = r + cpl * zcr.base[p];
      } else {
        av = plane_ptr(ar, t, ny, g.nx, 1)[col];
        r = scale * plane_ptr(inr, t, ny, g.nx, 1)[col];
        if (has_zc) r = r + cpl * plane_ptr(zcr, t, ny, g.nx, 1)[col];
      }
      rv = r;
    } else {
      av = 0.0;
      rv = 0.0;
    }
  };
#pragma unroll
  for (int i = 0; i < JPF; ++i) load_row(t0 + i, pa[i], pr[i]);

  bool zero_diag = false;
  auto step = [&](int t, double a_in, double r_in) {
    // shift windows and take row t
#pragma unroll
    for (int i = 0; i < K; ++i) {
      A[i] = A[i + 1];
      ID[i] = ID[i + 1];
    }
#pragma unroll
    for (int i = 0; i < K - 1; ++i) R[i] = R[i + 1];
    A[K] = a_in;
    R[K - 1] = r_in;
    {
      const double D = alpha - dt * diag_of<KIND>(g, kp, A[K], sig);
      zero_diag |= (D == 0.0);
      ID[K] = 1.0 / D;
    }
    // sweep 1 at row t (pointwise from x_0 = 0)
    double xnew = OMEGA * (ID[K] * R[K - 1]);
    // sweeps 2..K: sweep m at row rho = t - m + 1
#pragma unroll
    for (int m = 2; m <= K; ++m) {
      // sweep m-1's window gets its newest row
      X[m - 1][0] = X[m - 1][1];
      X[m - 1][1] = X[m - 1][2];
      X[m - 1][2] = xnew;
      const double am = A[K - m], ac = A[K - m + 1], ap = A[K - m + 2];
      const double xm = X[m - 1][0], xc = X[m - 1][1], xp = X[m - 1][2];
      const double lx = lx_col<KIND>(g, kp, sig, am, ac, ap, xm, xc, xp);
      const double sx = alpha * xc - dt * lx;
      xnew = xc + OMEGA * (ID[K - m + 1] * (R[K - m] - sx));
    }
    // sweep K output row t - H
    const int yo = t - H;
    if (valid_lane && yo >= y0 && yo < y1) x_out[yo * g.nx + col] = xnew;
  };
  for (int t = t0; t < t1; t += 2 * JPF) {
#pragma unroll
    for (int i = 0; i < JPF; ++i) load_row(t + JPF + i, qa[i], qr[i]);
#pragma unroll
    for (int i = 0; i < JPF; ++i)
      if (t + i < t1) step(t + i, pa[i], pr[i]);
#pragma unroll
    for (int i = 0; i < JPF; ++i) load_row(t + 2 * JPF + i, pa[i], pr[i]);
#pragma unroll
    for (int i = 0; i < JPF; ++i)
      if (t + JPF + i < t1) step(t + JPF + i, qa[i], qr[i]);
  }
  if (zero_diag && flag_ctrl) flag_ctrl->zero_diag = 1;
}

// ---------------------------------------------------------------------------
// Column-pair variant (nx even, nx >= 64): lane l owns the aligned column pair
// (c, c+1), c = strip start + 2l, so a warp covers a 64-column strip and emits
// 64 - 2*HS columns (HS = halo rounded up to even, keeping the pairs 16-byte
// aligned for double2 loads/stores).  Against the one-column kernel: twice the
// independent work per lane (the sweep chain is latency-bound), one shuffle
// per neighbour per pair instead of per point, no per-row reciprocal when the
// diagonal is constant (Burgers), and sweep m skips the rows outside the band
// it must supply to sweep m+1 ([y0-(K-m), y1+(K-m))) -- all warp-uniform.
// The input rows (a, r, coupling field) stream through a per-warp ring of
// JRING rows in shared memory filled with cp.async, so the loads run JRING
// rows ahead without holding registers (the sweep chain is load-latency bound).
constexpr int JPW = 4;   // warps per CTA
constexpr int JRING = 8; // rows in flight per warp (cp.async ring in shared memory)
// the split-operator chain runs one warp per CTA: every loop bound is then
// block-uniform, so the compiler emits the x-neighbour shuffles as plain
// SHFL (a 4-warp CTA made the bounds thread-dependent in its eyes, and each
// shuffle grew a WARPSYNC + divergent-collective fallback path)
constexpr int JSPW = 1;

namespace {

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int KIND>
__device__ __forceinline__ void lx_pair(const Grid &g, const KindParams &kp, double sigma,
                                        const double *am, const double *ac, const double *ap,
                                        const double *xm, const double *xc, const double *xp,
                                        double *lx) {
  // same expression order as lx_col (left + right - 2 centre) for each column
  if (KIND == KIND_NLDIFF) {
    const double ax0 = ac[0] * xc[0], ax1 = ac[1] * xc[1];
    const double axl = shfl_up1(ax1), axr = shfl_dn1(ax0);
    lx[0] = g.ih2[0] * (axl + ax1 - 2.0 * ax0) + g.ih2[1] * (am[0] * xm[0] + ap[0] * xp[0] - 2.0 * ax0);
    lx[1] = g.ih2[0] * (ax0 + axr - 2.0 * ax1) + g.ih2[1] * (am[1] * xm[1] + ap[1] * xp[1] - 2.0 * ax1);
  } else if (KIND == KIND_BURGERS) {
    const double ax0 = ac[0] * xc[0], ax1 = ac[1] * xc[1];
    const double axl = shfl_up1(ax1), axr = shfl_dn1(ax0);
    const double xl = shfl_up1(xc[1]), xr = shfl_dn1(xc[0]);
    const double adv0 = g.i2h[0] * (ax1 - axl) + g.i2h[1] * (ap[0] * xp[0] - am[0] * xm[0]);
    const double adv1 = g.i2h[0] * (axr - ax0) + g.i2h[1] * (ap[1] * xp[1] - am[1] * xm[1]);
    const double lap0 = g.ih2[0] * (xl + xc[1] - 2.0 * xc[0]) + g.ih2[1] * (xm[0] + xp[0] - 2.0 * xc[0]);
    const double lap1 = g.ih2[0] * (xc[0] + xr - 2.0 * xc[1]) + g.ih2[1] * (xm[1] + xp[1] - 2.0 * xc[1]);
    lx[0] = -adv0 + sigma * kp.nu * lap0;
    lx[1] = -adv1 + sigma * kp.nu * lap1;
  } else {
    const double xl = shfl_up1(xc[1]), xr = shfl_dn1(xc[0]);
    const double lap0 = g.ih2[0] * (xl + xc[1] - 2.0 * xc[0]) + g.ih2[1] * (xm[0] + xp[0] - 2.0 * xc[0]);
    const double lap1 = g.ih2[0] * (xc[0] + xr - 2.0 * xc[1]) + g.ih2[1] * (xm[1] + xp[1] - 2.0 * xc[1]);
    const double ds0 = g.i2h[0] * (xc[1] - xl) + g.i2h[1] * (xp[0] - xm[0]);
    const double ds1 = g.i2h[0] * (xr - xc[0]) + g.i2h[1] * (xp[1] - xm[1]);
    lx[0] = sigma * (kp.nu * lap0 + kp.c * ds0) + ac[0] * xc[0];
    lx[1] = sigma * (kp.nu * lap1 + kp.c * ds1) + ac[1] * xc[1];
  }
}

}  // namespace

template <int KIND, int K>
__global__ void __launch_bounds__(JPW * 32)
    k_jacobi_pair2d(Grid g, KindParams kp, Op L, double alpha, double dt, VecIn vin, int in_off,
                    FRef zcr, double cpl, double *__restrict__ x_out, int span, int strips,
                    int nwarps, GCtrl *flag_ctrl, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  constexpr int H = K - 1;
  constexpr int HS = (H + 1) & ~1;
  constexpr int WC = 64 - 2 * HS;
  constexpr bool CONST_D = (KIND == KIND_BURGERS);
  const int gw = blockIdx.x * JPW + (threadIdx.x >> 5);
  if (gw >= nwarps) return;  // whole warp idle
  const int strip = gw % strips, band = gw / strips;
  double scale;
  const FRef inr = vin_resolve(vin, in_off, scale);
  const FRef ar = fref(L);
  const bool has_zc = zcr.base != nullptr;
  const int lane = threadIdx.x & 31;
  const int nx = g.nx, ny = g.ny;
  const int x0 = strip * WC;
  const int li = 2 * lane;  // strip-local index of the pair's first column
  int c0 = x0 - HS + li;
  c0 = c0 < 0 ? c0 + nx : (c0 >= nx ? c0 - nx : c0);
  const bool valid = li >= HS && li < 64 - HS && x0 - HS + li < nx;
  const int y0 = band * span;
  const int y1 = min(ny, y0 + span);
  const double sig = L.sigma;

  double A[K + 1][2];               // a rows t-K .. t
  double ID[K + 1][2];              // 1/D rows t-K .. t (unused if CONST_D)
  double R[K][2];                   // r rows t-K+1 .. t
  double X[K][3][2];                // sweep m (1..K-1): rows rho_m-2 .. rho_m
#pragma unroll
  for (int i = 0; i <= K; ++i) A[i][0] = A[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i <= K; ++i) ID[i][0] = ID[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) R[i][0] = R[i][1] = 0.0;
#pragma unroll
  for (int m = 0; m < K; ++m)
#pragma unroll
    for (int i = 0; i < 3; ++i) X[m][i][0] = X[m][i][1] = 0.0;
  bool zero_diag = false;
  double idc = 0.0;
  if (CONST_D) {
    const double D = alpha - dt * diag_of<KIND>(g, kp, 0.0, sig);
    zero_diag = (D == 0.0);
    idc = 1.0 / D;
  }

  const int t0 = y0 - H, t1 = y1 + H;  // input rows [t0, t1)
  auto rowp = [&](const FRef &f, int t) -> const double * {
    if (!g.slab) {
      const int s = t < 0 ? t + ny : (t >= ny ? t - ny : t);
      return f.base + (size_t)s * nx;
    }
    return plane_ptr(f, t, ny, nx, 1);
  };
  // ring slot layout per warp: [JRING][3 fields][64 columns]
  extern __shared__ __align__(16) double jring[];
  double *ring = jring + (size_t)(threadIdx.x >> 5) * JRING * 3 * 64;
  const int nf = has_zc ? 3 : 2;
  auto issue_row = [&](int t, int slot) {
    if (t < t1) {
      double *d = ring + slot * 3 * 64 + 2 * lane;
      cp_async16(d, rowp(ar, t) + c0);
      cp_async16(d + 64, rowp(inr, t) + c0);
      if (nf == 3) cp_async16(d + 128, rowp(zcr, t) + c0);
    }
    cp_async_commit();  // (empty groups past the end keep the count uniform)
  };
  auto read_row = [&](int slot, double2 &av, double2 &rv) {
    const double *d = ring + slot * 3 * 64 + 2 * lane;
    av = *reinterpret_cast<const double2 *>(d);
    const double2 in = *reinterpret_cast<const double2 *>(d + 64);
    double r0 = scale * in.x, r1 = scale * in.y;
    if (nf == 3) {
      const double2 z = *reinterpret_cast<const double2 *>(d + 128);
      r0 = r0 + cpl * z.x;
      r1 = r1 + cpl * z.y;
    }
    rv = make_double2(r0, r1);
  };
#pragma unroll
  for (int i = 0; i < JRING; ++i) issue_row(t0 + i, i);

  auto step = [&](int t, double2 a_in, double2 r_in) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      A[i][0] = A[i + 1][0];
      A[i][1] = A[i + 1][1];
      if (!CONST_D) {
        ID[i][0] = ID[i + 1][0];
        ID[i][1] = ID[i + 1][1];
      }
    }
#pragma unroll
    for (int i = 0; i < K - 1; ++i) {
      R[i][0] = R[i + 1][0];
      R[i][1] = R[i + 1][1];
    }
    A[K][0] = a_in.x;
    A[K][1] = a_in.y;
    R[K - 1][0] = r_in.x;
    R[K - 1][1] = r_in.y;
    if (!CONST_D) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double D = alpha - dt * diag_of<KIND>(g, kp, A[K][c], sig);
        zero_diag |= (D == 0.0);
        ID[K][c] = 1.0 / D;
      }
    }
    // sweep 1 at row t (pointwise from x_0 = 0)
    double xn[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) xn[c] = OMEGA * ((CONST_D ? idc : ID[K][c]) * R[K - 1][c]);
    // sweeps 2..K: sweep m at row rho = t - m + 1
#pragma unroll
    for (int m = 2; m <= K; ++m) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        X[m - 1][0][c] = X[m - 1][1][c];
        X[m - 1][1][c] = X[m - 1][2][c];
        X[m - 1][2][c] = xn[c];
      }
      const int rho = t - m + 1;
      if (rho >= y0 - (K - m) && rho < y1 + (K - m)) {  // warp-uniform
        double lx[2];
        lx_pair<KIND>(g, kp, sig, A[K - m], A[K - m + 1], A[K - m + 2], X[m - 1][0], X[m - 1][1],
                      X[m - 1][2], lx);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const double xc = X[m - 1][1][c];
          const double sx = alpha * xc - dt * lx[c];
          const double id = CONST_D ? idc : ID[K - m + 1][c];
          xn[c] = xc + OMEGA * (id * (R[K - m][c] - sx));
        }
      } else {
        xn[0] = xn[1] = 0.0;
      }
    }
    const int yo = t - H;
    if (valid && yo >= y0 && yo < y1)
      *reinterpret_cast<double2 *>(x_out + (size_t)yo * nx + c0) = make_double2(xn[0], xn[1]);
  };
  int slot = 0;
  for (int t = t0; t < t1; ++t) {
    cp_async_wait<JRING - 1>();  // row t (the oldest group) has landed
    double2 av, rv;
    read_row(slot, av, rv);
    issue_row(t + JRING, slot);  // refill the slot just read (own lane only)
    slot = slot + 1 == JRING ? 0 : slot + 1;
    step(t, av, rv);
  }
  cp_async_wait<0>();
  if (zero_diag && flag_ctrl) flag_ctrl->zero_diag = 1;
}

// ---------------------------------------------------------------------------
// Split-operator variant of the column-pair chain (the default).  With D the
// diagonal of S = alpha I - dt L and O = S - D its off-diagonal part, one
// damped-Jacobi sweep is
//     x_m = (1 - w) x_{m-1} + c (r - O x_{m-1}),   c = w / D,
// and sweep 1 (x_0 = 0) is x_1 = c r.  O is written with per-kernel constants
// on the products p = a x (the advective / Kirchhoff part) and on x (the
// viscous part), so a sweep costs ~11 FP64 operations per point instead of
// ~22 for the textbook "x + w D^{-1}(r - S x)" form; c r is formed once per
// point and reused by all K sweeps.  The row loop is unrolled over the
// cp.async ring so the sliding register windows are renamed, not copied.
// Rounding differs from the reference's CSR sweep at the 1e-16 level (the
// parity contract is 1e-10 on the solution and +/-1 on iteration counts).
struct JacCoef {
  double om1;         // 1 - omega
  double c;           // omega / D when D is constant (burgers)
  double dalpha;      // D = dalpha + dcoef * a   (nldiff, rad)
  double dcoef;
  double pxl, pxr;    // O x += pxl p_l + pxr p_r + pym p_m + pyp p_p
  double pym, pyp;
  double xx, xy;      // O x += xx (x_l + x_r) + xy (x_m + x_p)   (symmetric part)
  double xxa, xya;    // O x += xxa (x_r - x_l) + xya (x_p - x_m) (rad: advective)
  double xym, xyp;    // the y-terms regrouped: xym x_m + xyp x_p
};

#ifndef IRKG_JSP_MINB
#define IRKG_JSP_MINB 12  // resident one-warp CTAs per SM the compiler must allow (register cap)
#endif
template <int KIND, int K, bool SLAB>
__global__ void __launch_bounds__(JSPW * 32, IRKG_JSP_MINB / JSPW)
    k_jacobi_sp2d(Grid g, Op L, JacCoef jc, VecIn vin, int in_off, FRef zcr, double cpl,
                  double *__restrict__ x_out, int span, int strips, int nwarps, int band0,
                  GCtrl *flag_ctrl, const GCtrl *skip, int ylo, int yhi, double *out_lo,
                  double *out_hi) {
  constexpr int H = K - 1;
  constexpr int HS = (H + 1) & ~1;
  constexpr int WC = 64 - 2 * HS;
  constexpr bool CONST_D = (KIND == KIND_BURGERS);
  constexpr bool USE_P = (KIND != KIND_RAD);   // O acts on p = a x
  constexpr bool USE_XS = (KIND != KIND_NLDIFF);  // O acts on x (viscous / rad)
  const int gw = JSPW == 1 ? (int)blockIdx.x : (int)(blockIdx.x * JSPW + (threadIdx.x >> 5));
  if (gw >= nwarps) return;  // whole warp idle
  const int strip = gw % strips, band = band0 + gw / strips;
  double scale = 1.0;
  FRef inr{};  // v_j (the predecessor's output): resolved after pdl_wait()
  const FRef ar = fref(L);
  const bool has_zc = zcr.base != nullptr;
  const int lane = threadIdx.x & 31;
  const int nx = g.nx, ny = g.ny;
  const int x0 = strip * WC;
  const int li = 2 * lane;
  int c0 = x0 - HS + li;
  c0 = c0 < 0 ? c0 + nx : (c0 >= nx ? c0 - nx : c0);
  const bool valid = li >= HS && li < 64 - HS && x0 - HS + li < nx;
  // output rows [ylo, yhi): the local rows [0, ny), or (slab mode, extended
  // halo) E rows beyond them on either side, computed redundantly from a
  // deeper halo of the input and stored into the output's ghost planes -- the
  // consumer then needs no halo exchange of this chain's result
  // (single rank: ylo = 0, yhi = ny, folded at compile time -- the recompiled kernel with the
  // run-time bounds cost 1.6 us per launch inside the step graph, 2 % of a configs[1] step)
  const int y0 = (SLAB ? ylo : 0) + band * span;
  const int y1 = min(SLAB ? yhi : ny, y0 + span);

  // sliding windows (index K-1 / 2 = newest row)
  double AW[K][2];      // a, rows t-K+1 .. t
  double CW[K][2];      // omega / D, rows t-K+1 .. t (varying-D kinds)
  double RW[K][2];      // c r, rows t-K+1 .. t
  double XW[K][3][2];   // sweep m (1..K-1): x rows rho-2 .. rho
  double PW[K][3][2];   // sweep m: p = a x, same rows
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int c = 0; c < 2; ++c) AW[i][c] = CW[i][c] = RW[i][c] = 0.0;
#pragma unroll
  for (int m = 0; m < K; ++m)
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int c = 0; c < 2; ++c) XW[m][i][c] = PW[m][i][c] = 0.0;
  bool zero_diag = false;

  const int t0 = y0 - H, t1 = y1 + H;  // input rows [t0, t1)
  auto rowp = [&](const FRef &f, int t) -> const double * {
    if (!SLAB) {
      const int s = t < 0 ? t + ny : (t >= ny ? t - ny : t);
      return f.base + (size_t)s * nx;
    }
    return plane_ptr(f, t, ny, nx, 1);
  };
  extern __shared__ __align__(16) double jring[];
  double *ring = jring + (JSPW == 1 ? 0 : (size_t)(threadIdx.x >> 5) * JRING * 3 * 64);
  // periodic (single-rank) rows: the element offset of the next row to issue
  // advances by nx and wraps once at ny, so a refill is three cp.async with
  // one add -- no per-row wrap branches or 64-bit multiplies in the hot loop
  const long long nloc = (long long)nx * ny;
  long long ioff = 0;  // offset (wrapped row * nx + c0) of row t0 + JRING
  if (!SLAB) {
    int w = t0 + JRING;
    w = w < 0 ? w + ny : (w >= ny ? w - ny : w);
    ioff = (long long)w * nx + c0;
  }
  const double *pa = ar.base, *pr = nullptr, *pz = zcr.base;
  auto issue_row = [&](int t, int slot) {
    double *d = ring + slot * 3 * 64 + 2 * lane;
    if (!SLAB) {
      if (t < t1) {
        IRKG_DCHECK(ioff >= 0 && ioff + 2 <= nloc && (ioff & 1) == 0);
        IRKG_DCHECK(slot >= 0 && slot < JRING);
        cp_async16(d, pa + ioff);
        cp_async16(d + 64, pr + ioff);
        if (has_zc) cp_async16(d + 128, pz + ioff);
      }
      ioff += nx;
      if (ioff >= nloc) ioff -= nloc;
    } else if (t < t1) {
      cp_async16(d, rowp(ar, t) + c0);
      cp_async16(d + 64, rowp(inr, t) + c0);
      if (has_zc) cp_async16(d + 128, rowp(zcr, t) + c0);
    }
    cp_async_commit();
  };
  // the operator-field rows of the first ring group go out before the
  // dependency wait (no predecessor writes them; v_j / z1 only after it) --
  // they join the first commit group
#pragma unroll
  for (int i = 0; i < JRING; ++i)
    if (t0 + i < t1) cp_async16(ring + i * 3 * 64 + 2 * lane, rowp(ar, t0 + i) + c0);
  pdl_wait();  // inputs: v_j / z1 from the predecessors
  pdl_trigger();
  if (skip && skip->cycle_done) {
    cp_async_commit();
    cp_async_wait<0>();
    return;
  }
  inr = vin_resolve(vin, in_off, scale);
  pr = inr.base;
#pragma unroll
  for (int i = 0; i < JRING; ++i) {
    const int t = t0 + i;
    if (t < t1) {
      double *d = ring + i * 3 * 64 + 2 * lane;
      cp_async16(d + 64, rowp(inr, t) + c0);
      if (has_zc) cp_async16(d + 128, rowp(zcr, t) + c0);
    }
    cp_async_commit();
  }

  auto step = [&](int t, int slot) {
    cp_async_wait<JRING - 1>();
    const double *d = ring + slot * 3 * 64 + 2 * lane;
    const double2 av = *reinterpret_cast<const double2 *>(d);
    const double2 in = *reinterpret_cast<const double2 *>(d + 64);
    double r0 = scale * in.x, r1 = scale * in.y;
    if (has_zc) {
      const double2 z = *reinterpret_cast<const double2 *>(d + 128);
      r0 = r0 + cpl * z.x;
      r1 = r1 + cpl * z.y;
    }
    issue_row(t + JRING, slot);
    // shift the per-row windows (renamed away by the unrolled loop)
#pragma unroll
    for (int i = 0; i < K - 1; ++i)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        AW[i][c] = AW[i + 1][c];
        RW[i][c] = RW[i + 1][c];
        if (!CONST_D) CW[i][c] = CW[i + 1][c];
      }
    AW[K - 1][0] = av.x;
    AW[K - 1][1] = av.y;
    const double rr[2] = {r0, r1};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      double cc;
      if (CONST_D) {
        cc = jc.c;
      } else {
        const double D = jc.dalpha + jc.dcoef * AW[K - 1][c];
        zero_diag |= (D == 0.0);
        cc = OMEGA / D;
        CW[K - 1][c] = cc;
      }
      RW[K - 1][c] = cc * rr[c];
    }
    // sweep 1 at row t: x_1 = c r
    double xn[2], pn[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      xn[c] = RW[K - 1][c];
      pn[c] = USE_P ? AW[K - 1][c] * xn[c] : 0.0;
    }
    // sweeps 2..K: sweep m at row rho = t - m + 1 from sweep m-1's window
#pragma unroll
    for (int m = 2; m <= K; ++m) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        XW[m - 1][0][c] = XW[m - 1][1][c];
        XW[m - 1][1][c] = XW[m - 1][2][c];
        XW[m - 1][2][c] = xn[c];
        if (USE_P) {
          PW[m - 1][0][c] = PW[m - 1][1][c];
          PW[m - 1][1][c] = PW[m - 1][2][c];
          PW[m - 1][2][c] = pn[c];
        }
      }
      const double *xm = XW[m - 1][0], *xc = XW[m - 1][1], *xp = XW[m - 1][2];
      const double *pm = PW[m - 1][0], *pc = PW[m - 1][1], *pp = PW[m - 1][2];
      // x-neighbours: lane-1's second column, lane+1's first column.  The
      // rows produced this step (xp, pp: sweep m-1's newest) enter last, so
      // the per-step dependency chain through the K sweeps is three FMAs and
      // a multiply per sweep; everything else is off the chain.
      double off[2] = {0.0, 0.0};
      if (USE_P) {
        const double pl = shfl_up1(pc[1]), pr = shfl_dn1(pc[0]);
        off[0] = jc.pxl * pl + jc.pxr * pc[1] + jc.pym * pm[0];
        off[1] = jc.pxl * pc[0] + jc.pxr * pr + jc.pym * pm[1];
      }
      if (USE_XS) {
        const double xl = shfl_up1(xc[1]), xr = shfl_dn1(xc[0]);
        off[0] += jc.xx * (xl + xc[1]) + jc.xym * xm[0];
        off[1] += jc.xx * (xc[0] + xr) + jc.xym * xm[1];
        if (KIND == KIND_RAD) {
          off[0] += jc.xxa * (xc[1] - xl);
          off[1] += jc.xxa * (xr - xc[0]);
        }
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double cc = CONST_D ? jc.c : CW[K - m][c];
        const double base = jc.om1 * xc[c] + RW[K - m][c];
        double ox = off[c];
        if (USE_XS) ox = fma(jc.xyp, xp[c], ox);
        if (USE_P) ox = fma(jc.pyp, pp[c], ox);
        xn[c] = fma(-cc, ox, base);
        pn[c] = (USE_P && m < K) ? AW[K - m][c] * xn[c] : 0.0;
      }
    }
    const int yo = t - H;
    if (valid && yo >= y0 && yo < y1) {
      double *orow;
      if (!SLAB || (yo >= 0 && yo < ny))
        orow = x_out + (size_t)yo * nx;
      else if (yo < 0)
        orow = out_lo + (size_t)(GH + yo) * nx;
      else
        orow = out_hi + (size_t)(yo - ny) * nx;
      *reinterpret_cast<double2 *>(orow + c0) = make_double2(xn[0], xn[1]);
    }
  };
  for (int tg = t0; tg < t1; tg += JRING) {
#pragma unroll
    for (int i = 0; i < JRING; ++i) step(tg + i, i);
  }
  cp_async_wait<0>();
  if (zero_diag && flag_ctrl) flag_ctrl->zero_diag = 1;
}

__global__ void k_flag_zero_diag(GCtrl *c, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  c->zero_diag = 1;
}

// launcher: returns false when the fused path does not apply
bool Engine::jacobi_chain_fused(const Op &L, double alpha, double dt, int inner, const VecIn &vin,
                                int in_off, const double *zc, double cpl, double *x_out,
                                const GCtrl *skip) {
  if (!fused_jacobi || ndim != 2 || inner < 1 || inner > 6 || grid.nx < 32 ||
      grid.ny < 2 * inner)
    return false;
  if (pair_jacobi && grid.nx % 2 == 0 && grid.nx >= 64) {
    const int wc = 64 - 2 * (inner & ~1);  // 64 - 2*HS, HS = (H+1) & ~1 with H = inner-1
    const int strips = (grid.nx + wc - 1) / wc;
    long long target = (long long)sms * jwarps_per_sm;
    long long bands = target / strips;
    bands = bands < 1 ? 1 : bands;
    int span = (int)((grid.ny + bands - 1) / bands);
    span = span < 8 ? 8 : (span > 128 ? 128 : span);
    if (jacobi_split) {
      // the split kernel walks span + 2(K-1) input rows in unrolled groups of
      // JRING: take spans that fill whole groups, the longest (least halo
      // redundancy) that still leaves ~6 resident warps per SM
      const int h2 = 2 * (inner - 1);
      int k = 2;
      while (k < 16) {
        const int nxt = JRING * (k + 1) - h2;
        const long long nw = (long long)strips * ((grid.ny + nxt - 1) / nxt);
        if (nw < 6LL * sms) break;
        ++k;
      }
      span = JRING * k - h2;
    }
    if (jspan_override > 0) span = jspan_override;
    if (span > grid.ny) span = grid.ny;
    // slab mode, extended halo: E rows beyond the slab on either side (chain_ext)
    const int E = (grid.slab && jacobi_split) ? chain_ext : 0;
    const int ylo = -E, yhi = grid.ny + E;
    double *out_lo = nullptr, *out_hi = nullptr;
    if (E > 0) {
      Ghost &og = role(chain_out_role);
      if (og.field && og.field != x_out) {
        auto it = owner.find(og.field);
        if (it != owner.end() && it->second == chain_out_role) owner.erase(it);
      }
      og.field = x_out;
      owner[x_out] = chain_out_role;
      out_lo = og.lo;
      out_hi = og.hi;
    }
    const int nb = (grid.ny + 2 * E + span - 1) / span;
    const int nwarps = strips * nb;
    const int blocks = (nwarps + JPW - 1) / JPW;
    // band ranges to launch: all, or (slab halo overlap, band_sel) the
    // interior bands that read no ghost plane / the edge bands that do
    int br[2][2] = {{0, nb}, {0, 0}};
    if (band_sel != 0) {
      int lo, hi;
      interior_bands(nb, span, inner - 1, lo, hi, ylo);
      if (band_sel == 1) {
        br[0][0] = lo;
        br[0][1] = hi;
      } else {
        br[0][0] = 0;
        br[0][1] = lo;
        br[1][0] = hi;
        br[1][1] = nb;
      }
    }
    const Op Lr = opref(L);
    auto go3 = [&](auto KD, auto KK) {
      constexpr int KIND_ = decltype(KD)::value;
      const double sig = Lr.sigma;
      JacCoef jc{};
      jc.om1 = 1.0 - OMEGA;
      if (KIND_ == KIND_BURGERS) {
        const double D = alpha - dt * sig * kp.nu * grid.lapdiag;
        jc.c = OMEGA / D;
        if (D == 0.0) jc.c = 0.0;
        jc.pxl = -dt * grid.i2h[0];
        jc.pxr = dt * grid.i2h[0];
        jc.pym = -dt * grid.i2h[1];
        jc.pyp = dt * grid.i2h[1];
        jc.xx = -dt * sig * kp.nu * grid.ih2[0];
        jc.xy = -dt * sig * kp.nu * grid.ih2[1];
        if (D == 0.0) {  // the reference raises for a zero diagonal
          k_flag_zero_diag<<<1, 1, 0, stream>>>(ctrl_dev, skip);
        }
      } else if (KIND_ == KIND_NLDIFF) {
        jc.dalpha = alpha;
        jc.dcoef = -dt * grid.lapdiag;
        jc.pxl = jc.pxr = -dt * grid.ih2[0];
        jc.pym = jc.pyp = -dt * grid.ih2[1];
      } else {
        jc.dalpha = alpha - dt * sig * kp.nu * grid.lapdiag;
        jc.dcoef = -dt;
        jc.xx = -dt * sig * kp.nu * grid.ih2[0];
        jc.xy = -dt * sig * kp.nu * grid.ih2[1];
        jc.xxa = -dt * sig * kp.c * grid.i2h[0];
        jc.xya = -dt * sig * kp.c * grid.i2h[1];
      }
      jc.xym = jc.xy - jc.xya;
      jc.xyp = jc.xy + jc.xya;
      auto go_s = [&](auto SL) {
        constexpr bool SLAB_ = decltype(SL)::value;
        auto kfn = k_jacobi_sp2d<KIND_, decltype(KK)::value, SLAB_>;
        static bool attr = false;  // one per instantiation
        if (!attr) {
          check(cudaFuncSetAttribute((const void *)kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     JSPW * JRING * 3 * 64 * 8),
                "jacobi ring smem");
          attr = true;
        }
        for (int r = 0; r < 2; ++r) {
          const int nbr = br[r][1] - br[r][0];
          if (nbr <= 0) continue;
          const int nw = strips * nbr;
          launch_pdl(kfn, dim3((nw + JSPW - 1) / JSPW), dim3(JSPW * 32),
                     (size_t)JSPW * JRING * 3 * 64 * sizeof(double), grid, Lr, jc, vin, in_off,
                     zc ? ref(zc) : FRef{nullptr, nullptr, nullptr}, cpl, x_out, span, strips,
                     nw, br[r][0], ctrl_dev, skip, ylo, yhi, out_lo, out_hi);
        }
      };
      if (grid.slab)
        go_s(std::true_type{});
      else
        go_s(std::false_type{});
    };
    auto go2 = [&](auto KD, auto KK) {
      if (jacobi_split) {
        go3(KD, KK);
        return;
      }
      static bool attr = false;  // one per instantiation
      if (!attr) {
        check(cudaFuncSetAttribute(
                  (const void *)k_jacobi_pair2d<decltype(KD)::value, decltype(KK)::value>,
                  cudaFuncAttributeMaxDynamicSharedMemorySize, JPW * JRING * 3 * 64 * 8),
              "jacobi ring smem");
        attr = true;
      }
      k_jacobi_pair2d<decltype(KD)::value, decltype(KK)::value>
          <<<blocks, JPW * 32, JPW * JRING * 3 * 64 * sizeof(double), stream>>>(
          grid, kp, opref(L), alpha, dt, vin, in_off,
          zc ? ref(zc) : FRef{nullptr, nullptr, nullptr}, cpl, x_out, span, strips, nwarps,
          ctrl_dev, skip);
    };
    auto with_k2 = [&](auto KD) {
      switch (inner) {
        case 1: go2(KD, std::integral_constant<int, 1>{}); break;
        case 2: go2(KD, std::integral_constant<int, 2>{}); break;
        case 3: go2(KD, std::integral_constant<int, 3>{}); break;
        case 4: go2(KD, std::integral_constant<int, 4>{}); break;
        case 5: go2(KD, std::integral_constant<int, 5>{}); break;
        default: go2(KD, std::integral_constant<int, 6>{}); break;
      }
    };
    switch (prob.kind) {
      case KIND_NLDIFF: with_k2(std::integral_constant<int, KIND_NLDIFF>{}); break;
      case KIND_BURGERS: with_k2(std::integral_constant<int, KIND_BURGERS>{}); break;
      default: with_k2(std::integral_constant<int, KIND_RAD>{}); break;
    }
    count(1);
    counters.precond_bytes += 8.0 * N * (zc ? 4.0 : 3.0);
    return true;
  }
  const int H = inner - 1;
  const int wcols = 32 - 2 * H;
  const int xt = (grid.nx + wcols - 1) / wcols;
  const int bx = (xt + JW - 1) / JW;
  long long target = (long long)sms * 16 / JW;  // ~16 warps per SM
  int span = (int)((long long)bx * grid.ny / target);
  span = span < 8 ? 8 : (span > 64 ? 64 : span);
  if (jspan_override > 0) span = jspan_override;
  if (span > grid.ny) span = grid.ny;
  const dim3 gr(bx, (grid.ny + span - 1) / span);
  auto go = [&](auto KD, auto KK) {
    k_jacobi_chain2d<decltype(KD)::value, decltype(KK)::value><<<gr, JW * 32, 0, stream>>>(
        grid, kp, opref(L), alpha, dt, vin, in_off, zc ? ref(zc) : FRef{nullptr, nullptr, nullptr},
        cpl, x_out, span, ctrl_dev, skip);
  };
  auto with_k = [&](auto KD) {
    switch (inner) {
      case 1: go(KD, std::integral_constant<int, 1>{}); break;
      case 2: go(KD, std::integral_constant<int, 2>{}); break;
      case 3: go(KD, std::integral_constant<int, 3>{}); break;
      case 4: go(KD, std::integral_constant<int, 4>{}); break;
      case 5: go(KD, std::integral_constant<int, 5>{}); break;
      default: go(KD, std::integral_constant<int, 6>{}); break;
    }
  };
  switch (prob.kind) {
    case KIND_NLDIFF: with_k(std::integral_constant<int, KIND_NLDIFF>{}); break;
    case KIND_BURGERS: with_k(std::integral_constant<int, KIND_BURGERS>{}); break;
    default: with_k(std::integral_constant<int, KIND_RAD>{}); break;
  }
  count(1);
  counters.precond_bytes += 8.0 * N * (zc ? 4.0 : 3.0);
  return true;
}

}  // namespace irkg
