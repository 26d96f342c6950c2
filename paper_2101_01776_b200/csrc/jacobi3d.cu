// jacobi3d.cu -- temporally blocked damped-Jacobi inner solves (3-D, 7-point).
//
// ShiftedSolver(alpha, I, L, dt, inner=K).solve(r) (src/irk_core.py:117-123):
//     x_0 = 0;  x_m = x_{m-1} + (2/3) D^{-1} (r - (alpha I - dt L) x_{m-1}),  m = 1..K
// computed in ONE pass over the grid (3.5-D blocking) instead of K: a CTA owns
// a 32 x 32 in-plane tile (halo K-1 on every side, so it emits (34-2K)^2
// columns) and slides along z through a band of planes; sweep m runs one
// plane behind sweep m-1.  Along z every thread keeps the sliding windows of
// its two columns in registers (the 2-D chain's split-operator form,
// jacobi.cu: x_m = (1-w) x_{m-1} + c (r - O x_{m-1}), c = w/D, O on the
// products p = a x and on x); the four in-plane neighbours of a sweep's
// centre plane come from shared memory, where each sweep leaves the plane it
// produced in the previous step (double-buffered: one CTA barrier per plane).
// The input planes (a, r = scale * basis slot j [, coupling field]) stream
// through a cp.async ring JR planes ahead; every thread copies and reads only
// its own two points, so the ring needs no barrier.  HBM traffic: a, r
// [, zc] read once, x_K written once -- 3-4 passes of N instead of the 4K-1
// of K separate sweeps (configs[3]: 256^3, K = 4: 15 -> 3 passes).
#include <type_traits>

#include "engine.h"

namespace irkg {

namespace {

constexpr int T3 = 32;             // tile edge (points)
constexpr int T3P = T3 * T3;       // points per tile plane
constexpr int T3THREADS = T3P / 2; // two columns per thread

__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit3() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait3() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace

// per-kernel constants of the split sweep: O x = sum over the axes d of
//   pm[d] p_{-d} + pp[d] p_{+d} + xm[d] x_{-d} + xp[d] x_{+d}
struct JacCoef3 {
  double om1;            // 1 - omega
  double c;              // omega / D when D is constant (burgers)
  double dalpha, dcoef;  // D = dalpha + dcoef * a (nldiff, rad)
  double pm[3], pp[3];
  double xm[3], xp[3];
};

// 1 / d to full double precision: the 20-bit hardware seed and two Newton
// steps (5 FP64 operations instead of the ~25 of an IEEE division; within
// 1 ulp of it, and the reference's own Jacobi sweep rounds differently anyway)
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

template <int KIND, int K, bool SLAB, int JR>
__global__ void __launch_bounds__(T3THREADS, 1)
    k_jacobi_sp3d(Grid g, Op L, JacCoef3 jc, VecIn vin, int in_off, FRef zcr, double cpl,
                  double *__restrict__ x_out, int span, int tiles_x, GCtrl *flag_ctrl,
                  const GCtrl *skip) {
  constexpr int H = K - 1;
  constexpr int WV = T3 - 2 * H;  // valid columns per tile edge
  constexpr bool CONST_D = (KIND == KIND_BURGERS);
  constexpr bool USE_P = (KIND != KIND_RAD);      // O acts on p = a x
  constexpr bool USE_XS = (KIND != KIND_NLDIFF);  // O acts on x
  constexpr int NPL = (USE_P ? 1 : 0) + (USE_XS ? 1 : 0);
  constexpr int NST = K > 1 ? K - 1 : 1;  // sweeps whose planes feed a successor
  // the plane loop is unrolled PER times and every sliding window is a ring
  // of PER statically indexed registers: the windows are renamed, not copied
  // (only the live entries of a ring occupy registers)
  constexpr int PER = K <= 4 ? 4 : 8;
  static_assert(PER % JR == 0, "ring slots must be static in the unrolled loop");
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;  // ty in 0..15; columns (tx, ty) and (tx, ty + 16)
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int tile_x = blockIdx.x % tiles_x, tile_y = blockIdx.x / tiles_x;
  const int X0 = tile_x * WV, Y0 = tile_y * WV;
  int gx = X0 - H + tx;
  gx = gx < 0 ? gx + nx : (gx >= nx ? gx - nx : gx);
  int q[2];
  bool valid[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int ly = ty + 16 * c;
    int gy = Y0 - H + ly;
    gy = gy < 0 ? gy + ny : (gy >= ny ? gy - ny : gy);
    q[c] = gy * nx + gx;
    valid[c] = tx >= H && tx < T3 - H && X0 + tx - H < nx && ly >= H && ly < T3 - H &&
               Y0 + ly - H < ny;
  }
  const int z0 = blockIdx.y * span;
  const int z1 = min(nz, z0 + span);
  const int t0 = z0 - H, t1 = z1 + H;  // input planes [t0, t1)

  extern __shared__ __align__(16) double sm3[];
  // ring: [JR][3 fields][2 columns][512 threads]; planes: [NST][2 buffers][NPL][32*32]
  double *ring = sm3;
  double *planes = sm3 + (size_t)JR * 3 * T3P;
  for (int i = tid; i < NST * 2 * NPL * T3P; i += T3THREADS) planes[i] = 0.0;

  const FRef ar = fref(L);
  const bool has_zc = zcr.base != nullptr;
  const long long nxy = g.nxy;
  const long long nloc = nxy * nz;
  auto planep = [&](const FRef &f, int t) -> const double * {
    if (!SLAB) {
      const int s = t < 0 ? t + nz : (t >= nz ? t - nz : t);
      return f.base + (size_t)s * nxy;
    }
    return plane_ptr(f, t, nz, (int)nxy, 1);
  };
  double scale = 1.0;
  FRef inr{};
  const double *pr_base = nullptr;
  // single rank: the element offset of the next plane to issue advances by
  // nxy and wraps once at the end of the grid
  long long goff = 0;
  if (!SLAB) {
    int w = t0 + JR;
    w = w < 0 ? w + nz : (w >= nz ? w - nz : w);
    goff = (long long)w * nxy;
  }
  auto issue_a = [&](int t, int slot) {
    if (t < t1) {
      const double *pa = planep(ar, t);
      double *d = ring + (size_t)slot * 3 * T3P + tid;
      cp_async8(d, pa + q[0]);
      cp_async8(d + T3THREADS, pa + q[1]);
    }
  };
  auto issue_r = [&](int t, int slot) {
    if (t < t1) {
      double *d = ring + (size_t)slot * 3 * T3P + T3P + tid;
      const double *pr = planep(inr, t);
      cp_async8(d, pr + q[0]);
      cp_async8(d + T3THREADS, pr + q[1]);
      if (has_zc) {
        const double *pz = planep(zcr, t);
        cp_async8(d + T3P, pz + q[0]);
        cp_async8(d + T3P + T3THREADS, pz + q[1]);
      }
    }
  };
  // refill of ring slot `slot` with plane t (the plane at offset goff)
  auto refill = [&](int t, int slot) {
    if (!SLAB) {
      if (t < t1) {
        IRKG_DCHECK(goff >= 0 && goff + nxy <= nloc && slot >= 0 && slot < JR);
        IRKG_DCHECK(q[0] >= 0 && q[0] < nxy && q[1] >= 0 && q[1] < nxy);
        double *d = ring + (size_t)slot * 3 * T3P + tid;
        const double *pa = ar.base + goff, *pr = pr_base + goff;
        cp_async8(d, pa + q[0]);
        cp_async8(d + T3THREADS, pa + q[1]);
        cp_async8(d + T3P, pr + q[0]);
        cp_async8(d + T3P + T3THREADS, pr + q[1]);
        if (has_zc) {
          const double *pz = zcr.base + goff;
          cp_async8(d + 2 * T3P, pz + q[0]);
          cp_async8(d + 2 * T3P + T3THREADS, pz + q[1]);
        }
      }
      goff += nxy;
      if (goff >= nloc) goff -= nloc;
    } else {
      issue_a(t, slot);
      issue_r(t, slot);
    }
  };
  // operator-field planes of the first ring go out before the dependency
  // wait (nothing in the Arnoldi body writes them); they join the first group
#pragma unroll
  for (int i = 0; i < JR; ++i) issue_a(t0 + i, i);
  pdl_wait();
  pdl_trigger();
  if (skip && skip->cycle_done) {
    cp_async_commit3();
    cp_async_wait3<0>();
    return;
  }
  inr = vin_resolve(vin, in_off, scale);
  pr_base = inr.base;
#pragma unroll
  for (int i = 0; i < JR; ++i) {
    issue_r(t0 + i, i);
    cp_async_commit3();
  }

  // sliding windows along z as rings: the value of plane t sits at index t' = (t - t0) % PER
  double AW[PER][2], CW[PER][2], RW[PER][2];
  double XW[K][PER][2], PW[K][PER][2];  // sweep m's outputs (m = 1 .. K-1)
#pragma unroll
  for (int i = 0; i < PER; ++i)
#pragma unroll
    for (int c = 0; c < 2; ++c) AW[i][c] = CW[i][c] = RW[i][c] = 0.0;
#pragma unroll
  for (int m = 0; m < K; ++m)
#pragma unroll
    for (int i = 0; i < PER; ++i)
#pragma unroll
      for (int c = 0; c < 2; ++c) XW[m][i][c] = PW[m][i][c] = 0.0;
  bool zero_diag = false;
  __syncthreads();  // planes zeroed

  // tile-local neighbour indices (wrapped inside the tile: the wrapped reads
  // only reach points outside every sweep's valid region)
  int nbi[2][4];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int ly = ty + 16 * c;
    nbi[c][0] = ly * T3 + ((tx + 31) & 31);
    nbi[c][1] = ly * T3 + ((tx + 1) & 31);
    nbi[c][2] = ((ly + 31) & 31) * T3 + tx;
    nbi[c][3] = ((ly + 1) & 31) * T3 + tx;
  }
  const int own[2] = {ty * T3 + tx, (ty + 16) * T3 + tx};
  // shared planes: the buffer written at even / odd unrolled steps
  double *const buf_e = planes, *const buf_o = planes + (size_t)NPL * T3P;

  auto step = [&](int t, auto UC) {
    constexpr int U = decltype(UC)::value;     // (t - t0) % PER
    constexpr int SLOT = U % JR;
    cp_async_wait3<JR - 1>();  // this thread's copies of plane t have landed
    const double *d = ring + (size_t)SLOT * 3 * T3P + tid;
    double a_in[2], r_in[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      a_in[c] = d[c * T3THREADS];
      r_in[c] = scale * d[T3P + c * T3THREADS];
      if (has_zc) r_in[c] = r_in[c] + cpl * d[2 * T3P + c * T3THREADS];
    }
    refill(t + JR, SLOT);
    cp_async_commit3();

    IRKG_DCHECK(own[0] < T3P && own[1] < T3P && nbi[0][0] < T3P && nbi[1][3] < T3P);
    double *wr = (U & 1) ? buf_o : buf_e;        // planes produced now
    const double *rd = (U & 1) ? buf_e : buf_o;  // produced in the previous step
    double xn[2], pn[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      AW[U][c] = a_in[c];
      double cc;
      if (CONST_D) {
        cc = jc.c;
      } else {
        const double D = jc.dalpha + jc.dcoef * a_in[c];
        zero_diag |= (D == 0.0);
        cc = OMEGA * rcp_nr(D);
        CW[U][c] = cc;
      }
      RW[U][c] = cc * r_in[c];
      xn[c] = RW[U][c];  // sweep 1 at plane t: x_1 = c r
      pn[c] = USE_P ? a_in[c] * xn[c] : 0.0;
    }
#pragma unroll
    for (int m = 2; m <= K; ++m) {
      // sweep m-1's newest plane enters its window and its shared plane
      double *wp = wr + (size_t)(m - 2) * 2 * NPL * T3P;
      const double *rp = rd + (size_t)(m - 2) * 2 * NPL * T3P;
      const int IN = U;                          // index of sweep m-1's plane rho + 1
      const int IC = (U + PER - 1) % PER;        // ... plane rho (sweep m's centre)
      const int IM = (U + PER - 2) % PER;        // ... plane rho - 1
      const int IW = (U + PER - (m - 1)) % PER;  // input windows at plane rho
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        XW[m - 1][IN][c] = xn[c];
        if (USE_P) {
          PW[m - 1][IN][c] = pn[c];
          wp[own[c]] = pn[c];
        }
        if (USE_XS) wp[(USE_P ? T3P : 0) + own[c]] = xn[c];
      }
      const int rho = t - m + 1;  // sweep m's plane (block-uniform test)
      if (rho >= z0 - (K - m) && rho < z1 + (K - m)) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          double ox = 0.0;
          if (USE_P) {
            const double *pp = rp;
            ox = jc.pm[0] * pp[nbi[c][0]] + jc.pp[0] * pp[nbi[c][1]] + jc.pm[1] * pp[nbi[c][2]] +
                 jc.pp[1] * pp[nbi[c][3]] + jc.pm[2] * PW[m - 1][IM][c];
          }
          if (USE_XS) {
            const double *xp = rp + (USE_P ? T3P : 0);
            ox += jc.xm[0] * xp[nbi[c][0]] + jc.xp[0] * xp[nbi[c][1]] + jc.xm[1] * xp[nbi[c][2]] +
                  jc.xp[1] * xp[nbi[c][3]] + jc.xm[2] * XW[m - 1][IM][c];
            ox = fma(jc.xp[2], XW[m - 1][IN][c], ox);
          }
          if (USE_P) ox = fma(jc.pp[2], PW[m - 1][IN][c], ox);
          const double cc = CONST_D ? jc.c : CW[IW][c];
          const double base = jc.om1 * XW[m - 1][IC][c] + RW[IW][c];
          xn[c] = fma(-cc, ox, base);
          pn[c] = (USE_P && m < K) ? AW[IW][c] * xn[c] : 0.0;
        }
      } else {
        xn[0] = xn[1] = 0.0;
        pn[0] = pn[1] = 0.0;
      }
    }
    const int zo = t - H;
    if (zo >= z0 && zo < z1) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
        if (valid[c]) {
          IRKG_DCHECK(zo >= 0 && zo < nz && (long long)zo * nxy + q[c] < nloc);
          x_out[(size_t)zo * nxy + q[c]] = xn[c];
        }
    }
    if (K > 1) __syncthreads();
  };
  // (steps past t1 in the last group read stale ring slots and store nothing)
  for (int tg = t0; tg < t1; tg += PER) {
    step(tg + 0, std::integral_constant<int, 0>{});
    step(tg + 1, std::integral_constant<int, 1>{});
    step(tg + 2, std::integral_constant<int, 2>{});
    step(tg + 3, std::integral_constant<int, 3>{});
    if (PER == 8) {
      step(tg + 4, std::integral_constant<int, 4 % PER>{});
      step(tg + 5, std::integral_constant<int, 5 % PER>{});
      step(tg + 6, std::integral_constant<int, 6 % PER>{});
      step(tg + 7, std::integral_constant<int, 7 % PER>{});
    }
  }
  cp_async_wait3<0>();
  if (zero_diag && flag_ctrl) flag_ctrl->zero_diag = 1;
}

__global__ void k_flag_zero_diag3(GCtrl *c, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  c->zero_diag = 1;
}

// launcher: returns false when the fused 3-D path does not apply
bool Engine::jacobi_chain_fused3d(const Op &L, double alpha, double dt, int inner,
                                  const VecIn &vin, int in_off, const double *zc, double cpl,
                                  double *x_out, const GCtrl *skip) {
  if (!fused_jacobi3d || ndim != 3 || inner < 1 || inner > 6 || grid.nx < T3 || grid.ny < T3 ||
      grid.nz < 2 * inner)
    return false;
  const int H = inner - 1;
  const int wv = T3 - 2 * H;
  const int tiles_x = (grid.nx + wv - 1) / wv, tiles_y = (grid.ny + wv - 1) / wv;
  const int tiles = tiles_x * tiles_y;
  // bands along z: fill whole waves of one CTA per SM while keeping the
  // z-halo redundancy (span + 2H) / span low
  int best_nb = 1;
  double best = 0.0;
  for (int nb = 1; nb <= grid.nz / (2 * inner > 4 ? 2 * inner : 4) && nb <= 64; ++nb) {
    const int sp = (grid.nz + nb - 1) / nb;
    const int nbe = (grid.nz + sp - 1) / sp;
    const double waves = (double)tiles * nbe / sms;
    const double eff = waves / std::ceil(waves) * sp / (sp + 2.0 * H);
    if (eff > best * 1.0001) {
      best = eff;
      best_nb = nbe;
    }
  }
  int span = (grid.nz + best_nb - 1) / best_nb;
  if (jspan_override > 0) span = jspan_override;
  if (span > grid.nz) span = grid.nz;
  const int nb = (grid.nz + span - 1) / span;
  const Op Lr = opref(L);
  const double sig = Lr.sigma;
  JacCoef3 jc{};
  jc.om1 = 1.0 - OMEGA;
  bool zero_d = false;
  if (prob.kind == KIND_BURGERS) {
    const double D = alpha - dt * sig * kp.nu * grid.lapdiag;
    zero_d = (D == 0.0);
    jc.c = zero_d ? 0.0 : OMEGA / D;
    for (int d = 0; d < 3; ++d) {
      jc.pm[d] = -dt * grid.i2h[d];
      jc.pp[d] = dt * grid.i2h[d];
      jc.xm[d] = jc.xp[d] = -dt * sig * kp.nu * grid.ih2[d];
    }
  } else if (prob.kind == KIND_NLDIFF) {
    jc.dalpha = alpha;
    jc.dcoef = -dt * grid.lapdiag;
    for (int d = 0; d < 3; ++d) jc.pm[d] = jc.pp[d] = -dt * grid.ih2[d];
  } else {
    jc.dalpha = alpha - dt * sig * kp.nu * grid.lapdiag;
    jc.dcoef = -dt;
    for (int d = 0; d < 3; ++d) {
      jc.xm[d] = -dt * sig * (kp.nu * grid.ih2[d] - kp.c * grid.i2h[d]);
      jc.xp[d] = -dt * sig * (kp.nu * grid.ih2[d] + kp.c * grid.i2h[d]);
    }
  }
  if (zero_d) {  // the reference raises for a zero diagonal
    k_flag_zero_diag3<<<1, 1, 0, stream>>>(ctrl_dev, skip);
  }
  const FRef zr = zc ? ref(zc) : FRef{nullptr, nullptr, nullptr};
  auto go = [&](auto KD, auto KK, auto SL, auto JRc) {
    constexpr int KIND_ = decltype(KD)::value, K_ = decltype(KK)::value, JR_ = decltype(JRc)::value;
    constexpr bool SLAB_ = decltype(SL)::value;
    constexpr int NPL = (KIND_ != KIND_RAD ? 1 : 0) + (KIND_ != KIND_NLDIFF ? 1 : 0);
    constexpr int NST = K_ > 1 ? K_ - 1 : 1;
    constexpr size_t smem = ((size_t)JR_ * 3 * T3P + (size_t)NST * 2 * NPL * T3P) * sizeof(double);
    auto kfn = k_jacobi_sp3d<KIND_, K_, SLAB_, JR_>;
    static bool attr = false;  // one per instantiation
    if (!attr) {
      check(cudaFuncSetAttribute((const void *)kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem),
            "jacobi3d smem");
      attr = true;
    }
    launch_pdl(kfn, dim3(tiles, nb), dim3(T3THREADS), smem, grid, Lr, jc, vin, in_off, zr, cpl,
               x_out, span, tiles_x, ctrl_dev, skip);
  };
  auto with_jr = [&](auto KD, auto KK, auto SL) {
    constexpr int KIND_ = decltype(KD)::value, K_ = decltype(KK)::value;
    constexpr int NPL = (KIND_ != KIND_RAD ? 1 : 0) + (KIND_ != KIND_NLDIFF ? 1 : 0);
    constexpr int NST = K_ > 1 ? K_ - 1 : 1;
    // deepest input ring that fits beside the sweep planes (227 KB per CTA)
    if constexpr ((4 * 3 + NST * 2 * NPL) * T3P * 8 <= 227 * 1024)
      go(KD, KK, SL, std::integral_constant<int, 4>{});
    else
      go(KD, KK, SL, std::integral_constant<int, 2>{});
  };
  auto with_s = [&](auto KD, auto KK) {
    if (grid.slab)
      with_jr(KD, KK, std::true_type{});
    else
      with_jr(KD, KK, std::false_type{});
  };
  auto with_k = [&](auto KD) {
    switch (inner) {
      case 1: with_s(KD, std::integral_constant<int, 1>{}); break;
      case 2: with_s(KD, std::integral_constant<int, 2>{}); break;
      case 3: with_s(KD, std::integral_constant<int, 3>{}); break;
      case 4: with_s(KD, std::integral_constant<int, 4>{}); break;
      case 5: with_s(KD, std::integral_constant<int, 5>{}); break;
      default: with_s(KD, std::integral_constant<int, 6>{}); break;
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
