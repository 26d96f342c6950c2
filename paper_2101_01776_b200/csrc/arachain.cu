// arachain.cu -- temporally blocked damped-Jacobi inner solves for the
// vorticity DAE's differential operator (BASELINE configs[4]).
//
// ShiftedSolver(alpha, I, L_u, dt, inner=K).solve(r) (src/irk_core.py:117-123)
// with L_u(Psi) x = -J(Psi, x) + sigma nu Lap x, J the 9-point Arakawa Jacobian
// (src/dae.py's blocks; csrc/dae.cu ara_lx):
//     x_0 = 0;  x_m = x_{m-1} + (2/3) D^{-1} (r - (alpha I - dt L_u) x_{m-1}),  m = 1..K
// in ONE pass over the grid instead of K (the unfused path launches K 9-point
// sweeps, each re-reading Psi, x and r: half of a configs[4] step).  Two
// forms: warp strips of column pairs (k_ara_sp2d, further down: the default
// for even nx >= 64) and, for the other grids, CTA strips (k_ara_chain): a CTA of
// 256 threads owns a strip of 256 columns (halo K-1 on each side: 258-2K
// columns out) and slides along y through a band of rows, one column per
// thread.  Sweep m runs two rows behind sweep m-1, so everything a step reads
// from shared memory was written in an earlier step: one CTA barrier per row.
// Shared memory holds, per strip: the rows of Psi a sweep may still need (ring,
// filled by cp.async three rows ahead of use), the scaled right-hand side
// c r of the last 2K-1 rows, and the last four rows of every sweep's output.
// The diagonal of alpha I - dt L_u is constant (J has a zero diagonal), so the
// split form of the 2-D chain applies: x_m = (1-w) x_{m-1} + c (r - O x_{m-1}).
// HBM traffic: Psi, r [, the coupling field] read once, x_K written once.
#include <type_traits>

#include "engine.h"

namespace irkg {

namespace {

constexpr int AC_SW = 256;  // strip width = threads per CTA
constexpr int AC_PF = 3;    // input rows in flight beyond the one being consumed

__device__ __forceinline__ void ac_cp8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void ac_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void ac_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace

struct AraCoef {
  double om1;  // 1 - omega
  double c;    // omega / D
  double cj;   // c dt / (12 hx hy)
  double cx;   // c dt sigma nu / hx^2
  double cy;   // c dt sigma nu / hy^2
};

template <int K, bool SLAB>
__global__ void __launch_bounds__(AC_SW, 2)
    k_ara_chain(Grid g, Op L, AraCoef ac, VecIn vin, int in_off, FRef zcr, double cpl,
                double *__restrict__ x_out, int span, int strips, const GCtrl *skip) {
  constexpr int H = K - 1;
  constexpr int WV = AC_SW - 2 * H;       // valid columns per strip
  constexpr int DA = AC_PF + 2 * K + 1;   // Psi ring (rows t + PF + 1 - DA .. t + PF)
  constexpr int DL = AC_PF + 1;           // landing ring of the raw rhs rows
  constexpr int DR = 2 * K;               // c r ring (rows t - 2(K-1) .. t)
  constexpr int DX = 4;                   // rows kept of each sweep's output
  constexpr int NST = K > 1 ? K - 1 : 1;
  const int i = threadIdx.x;
  const int strip = blockIdx.x % strips, band = blockIdx.x / strips;
  const int nx = g.nx, ny = g.ny;
  int gc = (strip * WV - H + i) % nx;
  if (gc < 0) gc += nx;
  const bool valid = i >= H && i < AC_SW - H && strip * WV + (i - H) < nx;
  const int y0 = band * span, y1 = min(ny, y0 + span);
  const int t0 = y0 - H, t1 = y1 + H;        // input rows [t0, t1)
  const int tlast = y1 - 1 + 2 * (K - 1);    // last step: sweep K reaches row y1 - 1

  extern __shared__ __align__(16) double acsm[];
  double *ringA = acsm;                           // [DA][SW]
  double *landR = ringA + DA * AC_SW;             // [DL][SW] raw rhs rows
  double *landZ = landR + DL * AC_SW;             // [DL][SW] coupling field rows
  double *ringR = landZ + DL * AC_SW;             // [DR][SW] c r
  double *ringX = ringR + DR * AC_SW;             // [NST][DX][SW]
  for (int q = i; q < (DA + 2 * DL + DR + NST * DX) * AC_SW; q += AC_SW) acsm[q] = 0.0;

  const FRef ar = fref(L);
  const bool has_zc = zcr.base != nullptr;
  auto rowp = [&](const FRef &f, int t) -> const double * {
    if (!SLAB) {
      const int s = t < 0 ? t + ny : (t >= ny ? t - ny : t);
      return f.base + (size_t)s * nx;
    }
    return plane_ptr(f, t, ny, nx, 1);
  };
  double scale = 1.0;
  FRef inr{};
  // row t lives in slot (t - t0) % depth of its ring
  auto issue_a = [&](int t) {
    if (t < t1) ac_cp8(ringA + ((t - t0) % DA) * AC_SW + i, rowp(ar, t) + gc);
  };
  auto issue_r = [&](int t) {
    if (t < t1) {
      const int sl = ((t - t0) % DL) * AC_SW + i;
      ac_cp8(landR + sl, rowp(inr, t) + gc);
      if (has_zc) ac_cp8(landZ + sl, rowp(zcr, t) + gc);
    }
  };
  __syncthreads();  // rings zeroed before the first copies land
  // Psi rows of the first group go out before the dependency wait (nothing in
  // the Arnoldi body writes the operator fields)
#pragma unroll
  for (int d = 0; d <= AC_PF; ++d) issue_a(t0 + d);
  pdl_wait();
  pdl_trigger();
  if (skip && skip->cycle_done) {
    ac_commit();
    ac_wait<0>();
    return;
  }
  inr = vin_resolve(vin, in_off, scale);
#pragma unroll
  for (int d = 0; d <= AC_PF; ++d) {
    issue_r(t0 + d);
    ac_commit();
  }
  const int il = (i + AC_SW - 1) & (AC_SW - 1), ir = (i + 1) & (AC_SW - 1);

  for (int t = t0; t <= tlast; ++t) {
    ac_wait<AC_PF>();  // this thread's copies of row t have landed
    __syncthreads();   // ... everyone's; and the previous step's ring writes are visible
    const int u = t - t0;
    // sweep 1 at row t (pointwise from x_0 = 0): x_1 = c r
    {
      const int sl = (u % DL) * AC_SW + i;
      double r = scale * landR[sl];
      if (has_zc) r = r + cpl * landZ[sl];
      const double rw = (t < t1) ? ac.c * r : 0.0;
      ringR[(u % DR) * AC_SW + i] = rw;
      if (K > 1)
        ringX[(u % DX) * AC_SW + i] = rw;
      else if (valid && t >= y0 && t < y1)
        x_out[(size_t)t * nx + gc] = rw;
    }
    issue_a(t + AC_PF + 1);
    issue_r(t + AC_PF + 1);
    ac_commit();
#pragma unroll
    for (int m = 2; m <= K; ++m) {
      const int rho = t - 2 * (m - 1);  // sweep m's row
      if (rho < y0 - (K - m) || rho >= y1 + (K - m)) continue;  // block-uniform
      const int ur = rho - t0;                                  // >= m - 1 >= 1
      const double *X = ringX + (size_t)(m - 2) * DX * AC_SW;
      const double *xs = X + ((ur - 1) % DX) * AC_SW, *xc = X + (ur % DX) * AC_SW,
                   *xn = X + ((ur + 1) % DX) * AC_SW;
      const double *as = ringA + ((ur - 1) % DA) * AC_SW, *am = ringA + (ur % DA) * AC_SW,
                   *an = ringA + ((ur + 1) % DA) * AC_SW;
      // Psi: S / N = rows rho -+ 1, W / E = columns -+ 1
      const double aS = as[i], aN = an[i], aW = am[il], aE = am[ir];
      const double aSW = as[il], aSE = as[ir], aNW = an[il], aNE = an[ir];
      const double xS = xs[i], xN = xn[i], xW = xc[il], xE = xc[ir], xC = xc[i];
      const double xSW = xs[il], xSE = xs[ir], xNW = xn[il], xNE = xn[ir];
      // 12 hx hy J(Psi, x): the three Arakawa forms collected per neighbour of x
      const double dEW = aE - aW, dNS = aN - aS;
      double J = xN * (dEW + (aNE - aNW)) - xS * (dEW + (aSE - aSW));
      J += xW * (dNS + (aNW - aSW)) - xE * (dNS + (aNE - aSE));
      J += xNE * (aE - aN) + xSE * (aS - aE);
      J += xNW * (aN - aW) + xSW * (aW - aS);
      const double base = ac.om1 * xC + ringR[(ur % DR) * AC_SW + i];
      double v = fma(ac.cx, xE + xW, base);
      v = fma(ac.cy, xN + xS, v);
      v = fma(-ac.cj, J, v);
      if (m < K) {
        ringX[((size_t)(m - 1) * DX + (ur % DX)) * AC_SW + i] = v;
      } else if (valid && rho >= y0 && rho < y1) {
        IRKG_DCHECK(rho >= 0 && rho < ny && gc >= 0 && gc < nx);
        x_out[(size_t)rho * nx + gc] = v;
      }
    }
  }
  ac_wait<0>();
}

// ---------------------------------------------------------------------------
// Warp-strip form (nx even, nx >= 64; the default): the layout of the 2-D
// Burgers/diffusion chain (jacobi.cu k_jacobi_sp2d).  One warp per CTA owns a
// 64-column strip of aligned column pairs and slides along y; sweep m runs
// one row behind sweep m-1.  Every sweep's last three rows of x live in
// registers (own pair + the two x-neighbour values, fetched by one shuffle
// pair when the row is produced), as rings of statically indexed registers in
// a row loop unrolled PER times, and so do the K + 1 rows of Psi the sweeps
// read (one shuffle pair when the row arrives); shared memory is only the
// landing zone of the cp.async copies (two rows ahead, every lane its own
// pair) and the c r ring.  No barrier anywhere: per point-sweep 26 FP64
// operations, one shared-memory load and 2 shuffles.  (ncu, 2048^2, K = 4: with
// Psi re-read from a shared-memory ring by every sweep the shared-memory pipe
// sat at 75 % of its peak and the FP64 pipe at 46 %.)
constexpr int AW_PF = 2;   // input rows in flight beyond the one being consumed
constexpr int AW_DL = 4;   // landing ring of the raw rhs rows (>= AW_PF + 1)

__device__ __forceinline__ void aw_cp16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ double aw_up(double v) {
  return __shfl_sync(0xffffffffu, v, (threadIdx.x + 31) & 31);
}
__device__ __forceinline__ double aw_dn(double v) {
  return __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31);
}

template <int K, bool SLAB>
__global__ void __launch_bounds__(32, 10)
    k_ara_sp2d(Grid g, Op L, AraCoef ac, VecIn vin, int in_off, FRef zcr, double cpl,
               double *__restrict__ x_out, int span, int strips, const GCtrl *skip) {
  constexpr int H = K - 1;
  constexpr int HS = (H + 1) & ~1;
  constexpr int WC = 64 - 2 * HS;
  // unroll / register-ring period: the Psi ring holds rows t-K .. t (K + 1 live entries)
  constexpr int PER = K + 1 <= 4 ? 4 : 8;
  constexpr int DR = PER;  // c r ring rows in shared memory (>= K)
  const int lane = threadIdx.x;
  const int strip = blockIdx.x % strips, band = blockIdx.x / strips;
  const int nx = g.nx, ny = g.ny;
  const int li = 2 * lane;
  int c0 = strip * WC - HS + li;
  c0 = c0 < 0 ? c0 + nx : (c0 >= nx ? c0 - nx : c0);
  const bool valid = li >= HS && li < 64 - HS && strip * WC - HS + li < nx;
  const int y0 = band * span, y1 = min(ny, y0 + span);
  const int t0 = y0 - H, t1 = y1 + H;  // input rows [t0, t1)

  extern __shared__ __align__(16) double awsm[];
  double *landA = awsm;                    // [AW_DL][64] Psi rows
  double *landR = landA + AW_DL * 64;      // [AW_DL][64] raw rhs rows
  double *landZ = landR + AW_DL * 64;      // [AW_DL][64] coupling field rows
  double *ringR = landZ + AW_DL * 64;      // [DR][64] c r
  for (int q = lane; q < (3 * AW_DL + DR) * 64; q += 32) awsm[q] = 0.0;
  __syncwarp();

  const FRef ar = fref(L);
  const bool has_zc = zcr.base != nullptr;
  auto rowp = [&](const FRef &f, int t) -> const double * {
    if (!SLAB) {
      const int s = t < 0 ? t + ny : (t >= ny ? t - ny : t);
      return f.base + (size_t)s * nx;
    }
    return plane_ptr(f, t, ny, nx, 1);
  };
  double scale = 1.0;
  FRef inr{};
  auto issue_a = [&](int t, int u) {  // row t = t0 + u
    if (t < t1) aw_cp16(landA + (u & (AW_DL - 1)) * 64 + li, rowp(ar, t) + c0);
  };
  auto issue_r = [&](int t, int u) {
    if (t < t1) {
      const int sl = (u & (AW_DL - 1)) * 64 + li;
      aw_cp16(landR + sl, rowp(inr, t) + c0);
      if (has_zc) aw_cp16(landZ + sl, rowp(zcr, t) + c0);
    }
  };
#pragma unroll
  for (int d = 0; d <= AW_PF; ++d) issue_a(t0 + d, d);
  pdl_wait();
  pdl_trigger();
  if (skip && skip->cycle_done) {
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    return;
  }
  inr = vin_resolve(vin, in_off, scale);
#pragma unroll
  for (int d = 0; d <= AW_PF; ++d) {
    issue_r(t0 + d, d);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }

  // register rings (index = the row's step number mod PER): Psi rows t-K .. t
  // and, per sweep m = 1 .. K-1, its last three output rows -- each as the
  // own pair plus the value left of / right of it
  double AWn[PER][2], AL[PER], AR[PER];
  double XW[K][PER][2], XL[K][PER], XR[K][PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) AWn[q][0] = AWn[q][1] = AL[q] = AR[q] = 0.0;
#pragma unroll
  for (int m = 0; m < K; ++m)
#pragma unroll
    for (int q = 0; q < PER; ++q) XW[m][q][0] = XW[m][q][1] = XL[m][q] = XR[m][q] = 0.0;

  auto step = [&](int t, int ub, auto UC) {
    constexpr int U = decltype(UC)::value;  // (t - t0) % PER
    const int u = ub + U;                   // t - t0
    asm volatile("cp.async.wait_group %0;" ::"n"(AW_PF) : "memory");
    double xn[2];
    {
      const int sl = (u & (AW_DL - 1)) * 64 + li;
      const double2 a = *reinterpret_cast<const double2 *>(landA + sl);
      AWn[U][0] = a.x;
      AWn[U][1] = a.y;
      AL[U] = aw_up(a.y);
      AR[U] = aw_dn(a.x);
      const double2 in = *reinterpret_cast<const double2 *>(landR + sl);
      double r0 = scale * in.x, r1 = scale * in.y;
      if (has_zc) {
        const double2 z = *reinterpret_cast<const double2 *>(landZ + sl);
        r0 = r0 + cpl * z.x;
        r1 = r1 + cpl * z.y;
      }
      xn[0] = (t < t1) ? ac.c * r0 : 0.0;  // sweep 1 at row t: x_1 = c r
      xn[1] = (t < t1) ? ac.c * r1 : 0.0;
      *reinterpret_cast<double2 *>(ringR + (u & (DR - 1)) * 64 + li) = make_double2(xn[0], xn[1]);
    }
    // (every lane copies and reads only its own pair of the landing rows: no warp barrier)
    issue_a(t + AW_PF + 1, u + AW_PF + 1);
    issue_r(t + AW_PF + 1, u + AW_PF + 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
#pragma unroll
    for (int m = 2; m <= K; ++m) {
      constexpr int IN = U;                    // sweep m-1's row rho + 1 (produced now)
      constexpr int IC = (U + PER - 1) % PER;  // ... row rho
      constexpr int IS = (U + PER - 2) % PER;  // ... row rho - 1
      XW[m - 1][IN][0] = xn[0];
      XW[m - 1][IN][1] = xn[1];
      XL[m - 1][IN] = aw_up(xn[1]);
      XR[m - 1][IN] = aw_dn(xn[0]);
      const int rho = t - (m - 1);  // sweep m's row (warp-uniform test)
      if (rho >= y0 - (K - m) && rho < y1 + (K - m)) {
        // Psi rows rho + 1, rho, rho - 1 = steps t - (m - 2), t - (m - 1), t - m
        const int an_ = (U + 2 * PER - (m - 2)) % PER, am_ = (U + 2 * PER - (m - 1)) % PER,
                  as_ = (U + 2 * PER - m) % PER;
        const double *aN = AWn[an_], *aM = AWn[am_], *aS = AWn[as_];
        const double aNl = AL[an_], aNr = AR[an_], aMl = AL[am_], aMr = AR[am_], aSl = AL[as_],
                     aSr = AR[as_];
        const int ur = u - (m - 1);
        const double2 rw = *reinterpret_cast<const double2 *>(ringR + (ur & (DR - 1)) * 64 + li);
        const double *xS = XW[m - 1][IS], *xC = XW[m - 1][IC], *xN = XW[m - 1][IN];
        const double xSl = XL[m - 1][IS], xSr = XR[m - 1][IS], xCl = XL[m - 1][IC],
                     xCr = XR[m - 1][IC], xNl = XL[m - 1][IN], xNr = XR[m - 1][IN];
        // column li: W = li-1, E = li+1;  column li+1: W = li, E = li+2
        double v[2];
        {
          const double dEW = aM[1] - aMl, dNS = aN[0] - aS[0];
          double J = xN[0] * (dEW + (aN[1] - aNl)) - xS[0] * (dEW + (aS[1] - aSl));
          J += xCl * (dNS + (aNl - aSl)) - xC[1] * (dNS + (aN[1] - aS[1]));
          J += xN[1] * (aM[1] - aN[0]) + xS[1] * (aS[0] - aM[1]);
          J += xNl * (aN[0] - aMl) + xSl * (aMl - aS[0]);
          double w = fma(ac.cx, xC[1] + xCl, ac.om1 * xC[0] + rw.x);
          w = fma(ac.cy, xN[0] + xS[0], w);
          v[0] = fma(-ac.cj, J, w);
        }
        {
          const double dEW = aMr - aM[0], dNS = aN[1] - aS[1];
          double J = xN[1] * (dEW + (aNr - aN[0])) - xS[1] * (dEW + (aSr - aS[0]));
          J += xC[0] * (dNS + (aN[0] - aS[0])) - xCr * (dNS + (aNr - aSr));
          J += xNr * (aMr - aN[1]) + xSr * (aS[1] - aMr);
          J += xN[0] * (aN[1] - aM[0]) + xS[0] * (aM[0] - aS[1]);
          double w = fma(ac.cx, xCr + xC[0], ac.om1 * xC[1] + rw.y);
          w = fma(ac.cy, xN[1] + xS[1], w);
          v[1] = fma(-ac.cj, J, w);
        }
        xn[0] = v[0];
        xn[1] = v[1];
      } else {
        xn[0] = xn[1] = 0.0;
      }
    }
    const int yo = t - H;
    if (valid && yo >= y0 && yo < y1) {
      IRKG_DCHECK(yo >= 0 && yo < ny && c0 >= 0 && c0 + 1 < nx);
      *reinterpret_cast<double2 *>(x_out + (size_t)yo * nx + c0) = make_double2(xn[0], xn[1]);
    }
  };
  // (steps past t1 in the last group read stale landing rows and store nothing)
  for (int tg = t0, ub = 0; tg < t1; tg += PER, ub += PER) {
    step(tg + 0, ub, std::integral_constant<int, 0>{});
    step(tg + 1, ub, std::integral_constant<int, 1>{});
    step(tg + 2, ub, std::integral_constant<int, 2>{});
    step(tg + 3, ub, std::integral_constant<int, 3>{});
    if (PER == 8) {
      step(tg + 4, ub, std::integral_constant<int, 4 % PER>{});
      step(tg + 5, ub, std::integral_constant<int, 5 % PER>{});
      step(tg + 6, ub, std::integral_constant<int, 6 % PER>{});
      step(tg + 7, ub, std::integral_constant<int, 7 % PER>{});
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

__global__ void k_flag_zero_diag_ara(GCtrl *c, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  c->zero_diag = 1;
}

// launcher: returns false when the fused path does not apply
bool Engine::ara_chain_fused(const Op &L, double alpha, double dt, int inner, const VecIn &vin,
                             int in_off, const double *zc, double cpl, double *x_out,
                             const GCtrl *skip) {
  if (!fused_ara || inner < 1 || inner > 6 || grid.ny < 2 * inner + 2 || grid.nx < 8) return false;
  const int H = inner - 1;
  // warp strips (aligned column pairs) need an even nx >= 64; otherwise the CTA-strip kernel
  const bool warp_form = ara_warp_form && grid.nx % 2 == 0 && grid.nx >= 64;
  const int wv = warp_form ? 64 - 2 * ((H + 1) & ~1) : AC_SW - 2 * H;
  const int strips = (grid.nx + wv - 1) / wv;
  // rows a band spends beyond its span: halo rows (+ pipeline drain of the CTA form)
  const int extra = warp_form ? 2 * H : 2 * H + 2 * (inner - 1);
  const int per = warp_form ? (inner + 1 <= 4 ? 4 : 8) : 1;  // row-loop unroll of the warp form
  const double cap = warp_form ? 10.0 * sms : 2.0 * sms;   // resident CTAs
  int best_nb = 1;
  double best = 0.0;
  for (int nb = 1; nb <= 1024 && nb <= grid.ny / 4; ++nb) {
    const int sp = (grid.ny + nb - 1) / nb;
    const int nbe = (grid.ny + sp - 1) / sp;
    const double waves = (double)strips * nbe / cap;
    const int steps = (sp + extra + per - 1) / per * per;
    const double eff = waves / std::ceil(waves) * sp / (double)steps;
    if (eff > best * 1.0001) {
      best = eff;
      best_nb = nbe;
    }
  }
  int span = (grid.ny + best_nb - 1) / best_nb;
  if (jspan_override > 0) span = jspan_override;
  if (span > grid.ny) span = grid.ny;
  const int nb = (grid.ny + span - 1) / span;
  const Op Lr = opref(L);
  const double D = alpha - dt * (Lr.sigma * kp.nu * grid.lapdiag);
  if (D == 0.0) {  // the reference raises for a zero diagonal
    k_flag_zero_diag_ara<<<1, 1, 0, stream>>>(ctrl_dev, skip);
  }
  AraCoef ac{};
  ac.om1 = 1.0 - OMEGA;
  ac.c = D == 0.0 ? 0.0 : OMEGA / D;
  ac.cj = ac.c * dt * (grid.i2h[0] * grid.i2h[1] / 3.0);
  ac.cx = ac.c * dt * Lr.sigma * kp.nu * grid.ih2[0];
  ac.cy = ac.c * dt * Lr.sigma * kp.nu * grid.ih2[1];
  const FRef zr = zc ? ref(zc) : FRef{nullptr, nullptr, nullptr};
  auto go = [&](auto KK, auto SL) {
    constexpr int K_ = decltype(KK)::value;
    constexpr bool SLAB_ = decltype(SL)::value;
    if (warp_form) {
      constexpr int PER = K_ + 1 <= 4 ? 4 : 8;
      constexpr size_t smem = (size_t)(3 * AW_DL + PER) * 64 * sizeof(double);
      launch_pdl(k_ara_sp2d<K_, SLAB_>, dim3(strips * nb), dim3(32), smem, grid, Lr, ac, vin,
                 in_off, zr, cpl, x_out, span, strips, skip);
      return;
    }
    constexpr int NST = K_ > 1 ? K_ - 1 : 1;
    constexpr size_t smem =
        (size_t)(AC_PF + 2 * K_ + 1 + 2 * (AC_PF + 1) + 2 * K_ + NST * 4) * AC_SW * sizeof(double);
    auto kfn = k_ara_chain<K_, SLAB_>;
    static bool attr = false;  // one per instantiation
    if (!attr) {
      check(cudaFuncSetAttribute((const void *)kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem),
            "ara chain smem");
      attr = true;
    }
    launch_pdl(kfn, dim3(strips * nb), dim3(AC_SW), smem, grid, Lr, ac, vin, in_off, zr, cpl, x_out,
               span, strips, skip);
  };
  auto with_s = [&](auto KK) {
    if (grid.slab)
      go(KK, std::true_type{});
    else
      go(KK, std::false_type{});
  };
  switch (inner) {
    case 1: with_s(std::integral_constant<int, 1>{}); break;
    case 2: with_s(std::integral_constant<int, 2>{}); break;
    case 3: with_s(std::integral_constant<int, 3>{}); break;
    case 4: with_s(std::integral_constant<int, 4>{}); break;
    case 5: with_s(std::integral_constant<int, 5>{}); break;
    default: with_s(std::integral_constant<int, 6>{}); break;
  }
  count(1);
  counters.precond_bytes += 8.0 * N * (zc ? 4.0 : 3.0);
  return true;
}

}  // namespace irkg
