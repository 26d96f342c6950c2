// stencil.cu -- register-sliding stencil kernels (2-D / 3-D).
//
// Each thread owns one column along the slowest axis (y in 2-D, z in 3-D)
// and slides along it, keeping every input field's (-1, 0, +1) values in
// registers; in-plane neighbours are L1 hits (loaded by neighbouring lanes /
// warps of the same CTA).  Every field therefore crosses L2->SM roughly once
// instead of three times (the row-per-CTA layout re-fetched each y-neighbour
// row from L2).  Used by the Jacobi sweeps (ShiftedSolver inner solves,
// src/irk_core.py:117-123), the block operators (src/irk_core.py:126-140,
// 216-219) and the stage residual (src/nonlinear.py:145-152).
#include <cstdlib>

#include "engine.h"

namespace irkg {

namespace {

#ifndef IRKG_SBX
#define IRKG_SBX 128
#endif
constexpr int SBX = IRKG_SBX;  // threads per CTA (3-D: a 32 x SBX/32 in-plane tile)

// Geometry of the slide: plane size P, number of planes NS, in-plane extents.
struct Slide {
  int P, NS;
};

template <int NDIM>
__device__ __forceinline__ Slide slide_of(const Grid &g) {
  Slide s;
  if (NDIM == 2) {
    s.P = g.nx;
    s.NS = g.ny;
  } else {
    s.P = g.nxy;
    s.NS = g.nz;
  }
  return s;
}

// column owned by this thread: in-plane offset q, or -1 if outside
template <int NDIM>
__device__ __forceinline__ int column_q(const Grid &g, int &ix, int &iy) {
  if (NDIM == 2) {
    ix = blockIdx.x * SBX + threadIdx.x;
    iy = 0;
    return ix < g.nx ? ix : -1;
  } else {
    ix = blockIdx.x * 32 + (threadIdx.x & 31);
    iy = blockIdx.y * (SBX / 32) + (threadIdx.x >> 5);
    return (ix < g.nx && iy < g.ny) ? iy * g.nx + ix : -1;
  }
}

// in-plane neighbour offsets relative to the point (periodic)
struct InPlane {
  int dxm, dxp, dym, dyp;
};

template <int NDIM>
__device__ __forceinline__ InPlane in_plane(const Grid &g, int ix, int iy) {
  InPlane o;
  o.dxm = (ix == 0) ? g.nx - 1 : -1;
  o.dxp = (ix == g.nx - 1) ? 1 - g.nx : 1;
  o.dym = o.dyp = 0;
  if (NDIM == 3) {
    o.dym = (iy == 0) ? (g.ny - 1) * g.nx : -g.nx;
    o.dyp = (iy == g.ny - 1) ? -(g.ny - 1) * g.nx : g.nx;
  }
  return o;
}

struct Win {
  double m, c, p;
};

template <int NDIM>
__device__ __forceinline__ Nb gather(const Win &w, const double *f, int p, const InPlane &o) {
  Nb n;
  n.c = w.c;
  n.v[0] = f[p + o.dxm];
  n.v[1] = f[p + o.dxp];
  if (NDIM == 2) {
    n.v[2] = w.m;
    n.v[3] = w.p;
    n.v[4] = n.v[5] = 0.0;
  } else {
    n.v[2] = f[p + o.dym];
    n.v[3] = f[p + o.dyp];
    n.v[4] = w.m;
    n.v[5] = w.p;
  }
  return n;
}

__device__ __forceinline__ double wsum2(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fold one value per CTA through the last-CTA ticket (deterministic order)
template <int NWARP = SBX / 32>
__device__ void cta_reduce_store(double v, double *part, int nblk, unsigned *counter,
                                 double *out) {
  __shared__ double red[NWARP];
  __shared__ bool last;
  const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  v = wsum2(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < NWARP; ++w) t += red[w];
    part[bid] = t;
    __threadfence();
    last = (atomicAdd(counter, 1u) == (unsigned)(nblk - 1));
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    double s = 0.0;
    for (int c = threadIdx.x; c < nblk; c += 32) s += __ldcg(part + c);
    s = wsum2(s);
    if (threadIdx.x == 0) {
      *out = s;
      *counter = 0u;
    }
  }
}

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

}  // namespace

// ---------------------------------------------------------- Jacobi sweep
// x' = x + omega * (r - (alpha x - dt L x)) / D   (src/irk_core.py:121-123)
template <int KIND, int NDIM>
__global__ void __launch_bounds__(SBX) k_jac_sweep_s(Grid g, KindParams kp, Op L, double alpha,
                                                     double dt, VecIn vin, int in_off,
                                                     const double *__restrict__ t_in,
                                                     FRef xr, double *__restrict__ x_out,
                                                     int span, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  double scale = 1.0;
  const double *in = t_in ? nullptr : vin_resolve(vin, in_off, scale).base;
  int ix, iy;
  const int q = column_q<NDIM>(g, ix, iy);
  if (q < 0) return;
  const Slide sl = slide_of<NDIM>(g);
  const InPlane o = in_plane<NDIM>(g, ix, iy);
  const int s0 = (NDIM == 2 ? blockIdx.y : blockIdx.z) * span;
  const int s1 = min(sl.NS, s0 + span);
  const double *a = L.a;
  const double *x = xr.base;
  const FRef ar = fref(L);
  auto at = [&](const FRef &f, int s) { return plane_ptr(f, s, sl.NS, sl.P, g.slab)[q]; };
  Win wx, wa;
  wx.m = at(xr, s0 - 1);
  wx.c = x[s0 * sl.P + q];
  if (a_stencil<KIND>()) {
    wa.m = at(ar, s0 - 1);
    wa.c = a[s0 * sl.P + q];
  }
  for (int s = s0; s < s1; ++s) {
    const int p = s * sl.P + q;
    wx.p = at(xr, s + 1);
    if (a_stencil<KIND>()) wa.p = at(ar, s + 1);
    const double r = t_in ? t_in[p] : scale * in[p];
    Nb xn = gather<NDIM>(wx, x, p, o);
    Nb an;
    if (a_stencil<KIND>()) {
      an = gather<NDIM>(wa, a, p, o);
    } else {
      an.c = a[p];
    }
    const double lx = lx_nb<KIND, NDIM>(g, kp, an, L.sigma, xn);
    const double diag = ldiag_at<KIND>(g, kp, a, L.sigma, p);
    const double D = alpha - dt * diag;
    const double sx = alpha * wx.c - dt * lx;
    x_out[p] = wx.c + OMEGA * ((1.0 / D) * (r - sx));
    wx.m = wx.c;
    wx.c = wx.p;
    if (a_stencil<KIND>()) {
      wa.m = wa.c;
      wa.c = wa.p;
    }
  }
}

// --------------------------------------------------------- block operator
// SIZE 1: w = eta z - dt L1 z (src/irk_core.py:216-219)
// SIZE 2: apply_block2x2 (src/irk_core.py:126-140); b != null: w = b - A z, ||w||^2
template <int KIND, int NDIM, int SIZE>
__global__ void __launch_bounds__(SBX)
    k_block_op_s(Grid g, KindParams kp, double eta, double beta, double phi, double dt, Op l1,
                 Op l2, Op c12, Op c21, FRef z1r, FRef z2r, double *__restrict__ w,
                 const double *__restrict__ b, int span, double *part, unsigned *counter,
                 double *out_norm, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  const int n = g.n;
  int ix, iy;
  const int q = column_q<NDIM>(g, ix, iy);
  double nrm = 0.0;
  if (q >= 0) {
    const Slide sl = slide_of<NDIM>(g);
    const InPlane o = in_plane<NDIM>(g, ix, iy);
    const int s0 = (NDIM == 2 ? blockIdx.y : blockIdx.z) * span;
    const int s1 = min(sl.NS, s0 + span);
    const double *z1 = z1r.base, *z2 = z2r.base;
    constexpr bool AS = a_stencil<KIND>();
    const bool h12 = SIZE == 2 && c12.present, h21 = SIZE == 2 && c21.present;
    const FRef a1r = fref(l1), a2r = fref(l2), c12r = fref(c12), c21r = fref(c21);
    // plane s of field f: one wrapped index shared by all fields (single rank)
    // or the ghost-aware pointer (slab mode)
    int pw = 0;
    auto at = [&](const FRef &f, int s) {
      return g.slab ? plane_ptr(f, s, sl.NS, sl.P, 1)[q] : f.base[pw];
    };
    auto wrap_idx = [&](int s) {
      s = s < 0 ? s + sl.NS : (s >= sl.NS ? s - sl.NS : s);
      return s * sl.P + q;
    };
    Win w1{}, w2{}, wa1{}, wa2{}, wc12{}, wc21{};
    auto init = [&](Win &wv, const FRef &f) {
      wv.m = at(f, s0 - 1);
      wv.c = f.base[s0 * sl.P + q];
    };
    pw = wrap_idx(s0 - 1);
    init(w1, z1r);
    if (AS) init(wa1, a1r);
    if (SIZE == 2) {
      init(w2, z2r);
      if (AS) init(wa2, a2r);
      if (AS && h12) init(wc12, c12r);
      if (AS && h21) init(wc21, c21r);
    }
    for (int s = s0; s < s1; ++s) {
      const int p = s * sl.P + q;
      pw = wrap_idx(s + 1);
      w1.p = at(z1r, s + 1);
      if (AS) wa1.p = at(a1r, s + 1);
      if (SIZE == 2) {
        w2.p = at(z2r, s + 1);
        if (AS) wa2.p = at(a2r, s + 1);
        if (AS && h12) wc12.p = at(c12r, s + 1);
        if (AS && h21) wc21.p = at(c21r, s + 1);
      }
      auto field = [&](const Win &wv, const double *f) {
        Nb r;
        if (AS) {
          r = gather<NDIM>(wv, f, p, o);
        } else {
          r.c = f[p];
        }
        return r;
      };
      const Nb x1 = gather<NDIM>(w1, z1, p, o);
      if (SIZE == 1) {
        double v = eta * x1.c - dt * lx_nb<KIND, NDIM>(g, kp, field(wa1, l1.a), l1.sigma, x1);
        if (b) {
          v = b[p] - v;
          nrm += v * v;
        }
        w[p] = v;
      } else {
        const Nb x2 = gather<NDIM>(w2, z2, p, o);
        double top = eta * x1.c - dt * lx_nb<KIND, NDIM>(g, kp, field(wa1, l1.a), l1.sigma, x1) +
                     phi * x2.c;
        double bot = -(beta * beta / phi) * x1.c + eta * x2.c -
                     dt * lx_nb<KIND, NDIM>(g, kp, field(wa2, l2.a), l2.sigma, x2);
        if (h12) top -= dt * lx_nb<KIND, NDIM>(g, kp, field(wc12, c12.a), c12.sigma, x2);
        if (h21) bot -= dt * lx_nb<KIND, NDIM>(g, kp, field(wc21, c21.a), c21.sigma, x1);
        if (b) {
          top = b[p] - top;
          bot = b[p + n] - bot;
          nrm += top * top + bot * bot;
        }
        w[p] = top;
        w[p + n] = bot;
      }
      auto shift = [](Win &wv) {
        wv.m = wv.c;
        wv.c = wv.p;
      };
      shift(w1);
      if (AS) shift(wa1);
      if (SIZE == 2) {
        shift(w2);
        if (AS) shift(wa2);
        if (AS && h12) shift(wc12);
        if (AS && h21) shift(wc21);
      }
    }
  }
  if (b) {
    const int nblk = gridDim.x * gridDim.y * gridDim.z;
    cta_reduce_store(nrm, part, nblk, counter, out_norm);
  }
}

// ------------------------------------------- block operator, 2-D strips
// Same operator as k_block_op_s (identical lx_nb arithmetic), laid out for
// memory-level parallelism: a warp owns a 64-column strip of aligned column
// pairs (60 valid; x-neighbours by shuffle) and slides along y through a
// band of rows; every input row (z1 [, z2], a1 [, a2, c12, c21]) streams
// through a per-warp ring of BRING rows in shared memory filled by cp.async,
// BRING-2 rows ahead of the row being computed.  (The one-column slide keeps
// only one row in flight per thread and is load-latency bound.)
constexpr int BPW = 1;    // warps per CTA (one: every loop bound is block-uniform, so the
                          // x-neighbour shuffles compile without divergent-collective paths)
constexpr int BRING = 6;  // ring rows per warp (rows s-1..s+1 + BRING-3 ahead)
constexpr int BWC = 60;   // valid columns per strip (halo 2 keeps pairs aligned)

template <int SIZE>
constexpr int bop_nf() {
  return SIZE == 1 ? 2 : 6;  // ring fields: z1, a1 [, z2, a2, c12, c21]
}

#ifndef IRKG_BOP_MINB
#define IRKG_BOP_MINB 16  // resident one-warp CTAs per SM the compiler must allow (register cap)
#endif
template <int KIND, int SIZE, bool SLAB>
__global__ void __launch_bounds__(BPW * 32, IRKG_BOP_MINB / BPW)
    k_block_op_strip(Grid g, KindParams kp, double eta, double beta, double phi, double dt,
                     Op l1, Op l2, Op c12, Op c21, FRef z1r, FRef z2r, double *__restrict__ w,
                     const double *__restrict__ b, int span, int strips, int nwarps, int band0,
                     double *part, unsigned *counter, double *out_norm, const GCtrl *skip) {
  constexpr int NF = bop_nf<SIZE>();
  const int lane = threadIdx.x & 31;
  const int gw = BPW == 1 ? (int)blockIdx.x : (int)(blockIdx.x * BPW + (threadIdx.x >> 5));
  double nrm = 0.0;
  if (gw >= nwarps) {  // idle warp: nothing to prefetch
    pdl_wait();
    pdl_trigger();
    if (skip && skip->cycle_done) return;
  }
  if (gw < nwarps) {
    const int nx = g.nx, ny = g.ny, n = g.n;
    const int strip = gw % strips, band = band0 + gw / strips;
    const int x0 = strip * BWC;
    const int li = 2 * lane;
    int c0 = x0 - 2 + li;
    c0 = c0 < 0 ? c0 + nx : (c0 >= nx ? c0 - nx : c0);
    const bool valid = li >= 2 && li < 62 && x0 - 2 + li < nx;
    const int y0 = band * span, y1 = min(ny, y0 + span);
    const bool h12 = SIZE == 2 && c12.present, h21 = SIZE == 2 && c21.present;
    FRef fr[NF];
    fr[0] = z1r;
    fr[1] = fref(l1);
    if (SIZE == 2) {
      fr[2] = z2r;
      fr[3] = fref(l2);
      fr[4] = fref(c12);
      fr[5] = fref(c21);
    }
    bool have[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) have[f] = true;
    if (SIZE == 2) {
      have[4] = h12;
      have[5] = h21;
    }
    extern __shared__ __align__(16) double bring[];
    double *ring = bring + (BPW == 1 ? 0 : (size_t)(threadIdx.x >> 5) * BRING * NF * 64) + li;
    auto rowp = [&](const FRef &f, int t) -> const double * {
      if (!SLAB) {
        const int s = t < 0 ? t + ny : (t >= ny ? t - ny : t);
        return f.base + (size_t)s * nx;
      }
      return plane_ptr(f, t, ny, nx, 1);
    };
    // periodic (single-rank) refills: the element offset of the next row to
    // issue (row y0 + BRING - 2 first) advances by nx and wraps once at ny
    const long long nloc = (long long)nx * ny;
    long long ioff = 0;
    if (!SLAB) {
      int wr = y0 + BRING - 2;
      wr = wr >= ny ? wr - ny : wr;
      ioff = (long long)wr * nx + c0;
    }
    // the slot of row t is (t - y0 + 1) % BRING; in the unrolled row loop
    // below it is a compile-time constant
    auto issue_row_slot = [&](int t, int slot) {
      if (!SLAB) {
        if (t <= y1) {  // rows y0-1 .. y1 feed the band
          IRKG_DCHECK(ioff >= 0 && ioff + 2 <= nloc && slot >= 0 && slot < BRING);
          double *d = ring + slot * NF * 64;
#pragma unroll
          for (int f = 0; f < NF; ++f)
            if (have[f]) cp_async16(d + f * 64, fr[f].base + ioff);
        }
        ioff += nx;
        if (ioff >= nloc) ioff -= nloc;
      } else if (t <= y1) {
        double *d = ring + slot * NF * 64;
#pragma unroll
        for (int f = 0; f < NF; ++f)
          if (have[f]) cp_async16(d + f * 64, rowp(fr[f], t) + c0);
      }
      cp_async_commit();  // (empty groups past the end keep the count uniform)
    };
    // pair values of field f at row t (from the ring)
    auto rd = [&](int f, int t) {
      return *reinterpret_cast<const double2 *>(ring + (((t - y0 + 1) % BRING) * NF + f) * 64);
    };
    auto rds = [&](int f, int slot) {
      return *reinterpret_cast<const double2 *>(ring + (slot * NF + f) * 64);
    };
    // neighbourhoods of the two columns from rows (m, c, p) of one field
    auto nb2 = [&](double2 m, double2 c, double2 p, Nb &n0, Nb &n1) {
      n0.c = c.x;
      n0.v[0] = __shfl_sync(0xffffffffu, c.y, (lane + 31) & 31);
      n0.v[1] = c.y;
      n0.v[2] = m.x;
      n0.v[3] = p.x;
      n0.v[4] = n0.v[5] = 0.0;
      n1.c = c.y;
      n1.v[0] = c.x;
      n1.v[1] = __shfl_sync(0xffffffffu, c.x, (lane + 1) & 31);
      n1.v[2] = m.y;
      n1.v[3] = p.y;
      n1.v[4] = n1.v[5] = 0.0;
    };
    auto field_nb = [&](int f, int s, Nb &n0, Nb &n1) {
      nb2(rd(f, s - 1), rd(f, s), rd(f, s + 1), n0, n1);
    };
    // coefficient fields (a1 [, a2, c12, c21]) are not written by the
    // predecessors: their first rows go out before the dependency wait and
    // join the first commit group; z1 [, z2] only after it
    auto coef_field = [](int f) { return f == 1 || f == 3 || f == 4 || f == 5; };
#pragma unroll
    for (int i = 0; i < BRING - 1; ++i) {
      const int t = y0 - 1 + i;
      if (t <= y1) {
        double *d = ring + ((t - y0 + 1) % BRING) * NF * 64;
#pragma unroll
        for (int f = 0; f < NF; ++f)
          if (have[f] && coef_field(f)) cp_async16(d + f * 64, rowp(fr[f], t) + c0);
      }
    }
    pdl_wait();  // z from the preconditioner
    pdl_trigger();
    if (skip && skip->cycle_done) {
      cp_async_commit();
      cp_async_wait<0>();
      return;
    }
#pragma unroll
    for (int i = 0; i < BRING - 1; ++i) {  // rows y0-1 .. y0+BRING-3
      const int t = y0 - 1 + i;
      if (t <= y1) {
        double *d = ring + ((t - y0 + 1) % BRING) * NF * 64;
#pragma unroll
        for (int f = 0; f < NF; ++f)
          if (have[f] && !coef_field(f)) cp_async16(d + f * 64, rowp(fr[f], t) + c0);
      }
      cp_async_commit();
    }
    // per-row coefficient combinations of rows s-1, s, s+1 slide down the band
    // in registers: each row's combination is formed once, not three times
    double qtm[2], rtm[2], qbm[2], rbm[2], qtc[2], rtc[2], qbc[2], rbc[2], qtp[2], rtp[2],
        qbp[2], rbp[2];
    // the row loop is unrolled over the ring (BRING rows per trip), so every
    // ring slot below is a compile-time constant
    for (int sb = y0; sb < y1; sb += BRING) {
#pragma unroll
    for (int ii = 0; ii < BRING; ++ii) {
      const int s = sb + ii;
      if (s >= y1) break;  // block-uniform
      auto slot_of = [&](int d) { return (ii + 1 + d + BRING) % BRING; };  // slot of row s + d
      cp_async_wait<BRING - 4>();  // rows up to s+1 have landed (s+2 .. s+BRING-3 may pend)
      // The operator is linear in its coefficient fields, so the four
      // stencil applications of a 2x2 block collapse into two per row:
      //   top = eta z1 + phi z2 - dt [ K(q_t) + sig-part(r_t) ],
      //   q_t = a1 z1 + c12 z2,  r_t = s1 z1 + s12 z2   (bot likewise)
      // with K the kind's coefficient stencil (Lap for nldiff, -Dsum for
      // burgers, the centre for rad) and the sigma part nu Lap (+ c Dsum).
      constexpr bool CP = (KIND != KIND_RAD);  // coefficients enter the stencil
      const double s1 = l1.sigma, s2 = SIZE == 2 ? l2.sigma : 0.0;
      const double s12 = h12 ? c12.sigma : 0.0, s21 = h21 ? c21.sigma : 0.0;
      auto combo = [&](int sl, double (&qt)[2], double (&rt)[2], double (&qb)[2],
                       double (&rb)[2]) {
        const double2 z1 = rds(0, sl), A1 = rds(1, sl);
        const double zz1[2] = {z1.x, z1.y}, aa1[2] = {A1.x, A1.y};
        double zz2[2] = {0.0, 0.0}, aa2[2] = {0.0, 0.0}, cc12[2] = {0.0, 0.0},
               cc21[2] = {0.0, 0.0};
        if (SIZE == 2) {
          const double2 z2 = rds(2, sl), A2 = rds(3, sl);
          zz2[0] = z2.x;
          zz2[1] = z2.y;
          aa2[0] = A2.x;
          aa2[1] = A2.y;
          if (h12) {
            const double2 c = rds(4, sl);
            cc12[0] = c.x;
            cc12[1] = c.y;
          }
          if (h21) {
            const double2 c = rds(5, sl);
            cc21[0] = c.x;
            cc21[1] = c.y;
          }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          qt[c] = aa1[c] * zz1[c];
          rt[c] = s1 * zz1[c];
          if (SIZE == 2) {
            if (h12) qt[c] += cc12[c] * zz2[c];
            rt[c] += s12 * zz2[c];
            qb[c] = aa2[c] * zz2[c];
            if (h21) qb[c] += cc21[c] * zz1[c];
            rb[c] = s2 * zz2[c] + s21 * zz1[c];
          }
        }
      };
      if (s == y0) {
        combo(slot_of(-1), qtm, rtm, qbm, rbm);
        combo(slot_of(0), qtc, rtc, qbc, rbc);
      }
      combo(slot_of(1), qtp, rtp, qbp, rbp);
      // x-neighbours of a row-s combination (lane-1's second / lane+1's first column)
      auto lap = [&](const double (&m)[2], const double (&c)[2], const double (&p)[2], double out[2]) {
        const double l = __shfl_sync(0xffffffffu, c[1], (lane + 31) & 31);
        const double r = __shfl_sync(0xffffffffu, c[0], (lane + 1) & 31);
        out[0] = g.ih2[0] * (l + c[1] - 2.0 * c[0]) + g.ih2[1] * (m[0] + p[0] - 2.0 * c[0]);
        out[1] = g.ih2[0] * (c[0] + r - 2.0 * c[1]) + g.ih2[1] * (m[1] + p[1] - 2.0 * c[1]);
      };
      auto dsum = [&](const double (&m)[2], const double (&c)[2], const double (&p)[2], double out[2]) {
        const double l = __shfl_sync(0xffffffffu, c[1], (lane + 31) & 31);
        const double r = __shfl_sync(0xffffffffu, c[0], (lane + 1) & 31);
        out[0] = g.i2h[0] * (c[1] - l) + g.i2h[1] * (p[0] - m[0]);
        out[1] = g.i2h[0] * (r - c[0]) + g.i2h[1] * (p[1] - m[1]);
      };
      // L-part of one block row from its two combinations
      auto lpart = [&](const double (&qm)[2], const double (&qc)[2], const double (&qp)[2],
                       const double (&rm)[2], const double (&rc)[2], const double (&rp)[2],
                       double out[2]) {
        if (KIND == KIND_NLDIFF) {
          lap(qm, qc, qp, out);
        } else if (KIND == KIND_BURGERS) {
          double d[2], l[2];
          dsum(qm, qc, qp, d);
          lap(rm, rc, rp, l);
#pragma unroll
          for (int c = 0; c < 2; ++c) out[c] = -d[c] + kp.nu * l[c];
        } else {
          double d[2], l[2];
          dsum(rm, rc, rp, d);
          lap(rm, rc, rp, l);
#pragma unroll
          for (int c = 0; c < 2; ++c) out[c] = (kp.nu * l[c] + kp.c * d[c]) + qc[c];
        }
        (void)CP;
      };
      double top[2], bot[2];
      {
        const double2 z1 = rds(0, slot_of(0));
        const double zz1[2] = {z1.x, z1.y};
        double lt[2];
        lpart(qtm, qtc, qtp, rtm, rtc, rtp, lt);
        if (SIZE == 1) {
#pragma unroll
          for (int c = 0; c < 2; ++c) top[c] = eta * zz1[c] - dt * lt[c];
        } else {
          const double2 z2 = rds(2, slot_of(0));
          const double zz2[2] = {z2.x, z2.y};
          double lb[2];
          lpart(qbm, qbc, qbp, rbm, rbc, rbp, lb);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            top[c] = (eta * zz1[c] + phi * zz2[c]) - dt * lt[c];
            bot[c] = (-(beta * beta / phi) * zz1[c] + eta * zz2[c]) - dt * lb[c];
          }
        }
      }
      if (valid) {
        const size_t p = (size_t)s * nx + c0;
        if (b) {
          const double2 b1 = *reinterpret_cast<const double2 *>(b + p);
          top[0] = b1.x - top[0];
          top[1] = b1.y - top[1];
          nrm += top[0] * top[0] + top[1] * top[1];
          if (SIZE == 2) {
            const double2 b2 = *reinterpret_cast<const double2 *>(b + p + n);
            bot[0] = b2.x - bot[0];
            bot[1] = b2.y - bot[1];
            nrm += bot[0] * bot[0] + bot[1] * bot[1];
          }
        }
        *reinterpret_cast<double2 *>(w + p) = make_double2(top[0], top[1]);
        if (SIZE == 2) *reinterpret_cast<double2 *>(w + p + n) = make_double2(bot[0], bot[1]);
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        qtm[c] = qtc[c];
        rtm[c] = rtc[c];
        qbm[c] = qbc[c];
        rbm[c] = rbc[c];
        qtc[c] = qtp[c];
        rtc[c] = rtp[c];
        qbc[c] = qbp[c];
        rbc[c] = rbp[c];
      }
      issue_row_slot(s + BRING - 2, slot_of(BRING - 2));  // the slot of row s-2 (no longer read)
    }
    }
    cp_async_wait<0>();
  }
  if (b) {
    const int nblk = gridDim.x;
    cta_reduce_store<BPW>(nrm, part, nblk, counter, out_norm);
  }
}

// ------------------------------------------------------- stage residual
// F_i = N(U_i) - K_i, ||F||^2   (src/nonlinear.py:148-152)
template <int KIND, int NDIM>
__global__ void __launch_bounds__(SBX)
    k_residual_s(Grid g, KindParams kp, int s_st, const double *__restrict__ U, StageGhosts ug,
                 const double *__restrict__ K, double *__restrict__ F, int span, double *part,
                 unsigned *counter, double *out) {
  pdl_wait();  // (PDL launch; no early trigger: a bandwidth kernel keeps its SMs)
  const int n = g.n;
  int ix, iy;
  const int q = column_q<NDIM>(g, ix, iy);
  double acc = 0.0;
  if (q >= 0) {
    const Slide sl = slide_of<NDIM>(g);
    const InPlane o = in_plane<NDIM>(g, ix, iy);
    const int s0 = (NDIM == 2 ? blockIdx.y : blockIdx.z) * span;
    const int s1 = min(sl.NS, s0 + span);
    for (int i = 0; i < s_st; ++i) {
      const double *u = U + (size_t)i * n;
      const FRef ur{u, ug.lo[i], ug.hi[i]};
      auto at = [&](int s) { return plane_ptr(ur, s, sl.NS, sl.P, g.slab)[q]; };
      Win wu;
      wu.m = at(s0 - 1);
      wu.c = u[s0 * sl.P + q];
      for (int s = s0; s < s1; ++s) {
        const int p = s * sl.P + q;
        wu.p = at(s + 1);
        const Nb un = gather<NDIM>(wu, u, p, o);
        const double f = rhs_nb<KIND, NDIM>(g, kp, un) - K[(size_t)i * n + p];
        F[(size_t)i * n + p] = f;
        acc += f * f;
        wu.m = wu.c;
        wu.c = wu.p;
      }
    }
  }
  const int nblk = gridDim.x * gridDim.y * gridDim.z;
  cta_reduce_store(acc, part, nblk, counter, out);
}

// ------------------------------------------------ back-substitution rhs
// acc_r = g_r - sum_j R0[r,j] y_j + dt sum_j od(r,j) y_j (src/irk_core.py:273-283),
// neighbours gathered directly (called once per block per Newton iteration).
template <int NDIM>
__device__ __forceinline__ Nb gather_direct(const FRef &f, int s, int q, int p, const InPlane &o,
                                            const Slide &sl, int slab) {
  Nb n;
  n.c = f.base[p];
  n.v[0] = f.base[p + o.dxm];
  n.v[1] = f.base[p + o.dxp];
  const double m = plane_ptr(f, s - 1, sl.NS, sl.P, slab)[q];
  const double pp = plane_ptr(f, s + 1, sl.NS, sl.P, slab)[q];
  if (NDIM == 2) {
    n.v[2] = m;
    n.v[3] = pp;
    n.v[4] = n.v[5] = 0.0;
  } else {
    n.v[2] = f.base[p + o.dym];
    n.v[3] = f.base[p + o.dyp];
    n.v[4] = m;
    n.v[5] = pp;
  }
  return n;
}

template <int KIND, int NDIM>
__global__ void __launch_bounds__(SBX)
    k_backsub_s(Grid g, KindParams kp, double dt, BacksubTerms T, const double *__restrict__ gst,
                const double *__restrict__ y, double *__restrict__ rhs, int span) {
  pdl_wait();  // (PDL launch; no early trigger: a bandwidth kernel keeps its SMs)
  const int n = g.n;
  int ix, iy;
  const int q = column_q<NDIM>(g, ix, iy);
  if (q < 0) return;
  const Slide sl = slide_of<NDIM>(g);
  const InPlane o = in_plane<NDIM>(g, ix, iy);
  const int s0 = (NDIM == 2 ? blockIdx.y : blockIdx.z) * span;
  const int s1 = min(sl.NS, s0 + span);
  for (int s = s0; s < s1; ++s) {
    const int p = s * sl.P + q;
    for (int r = 0; r < T.rows; ++r) {
      double acc = gst[(size_t)(T.row0 + r) * n + p];
      for (int qq = 0; qq < T.njs; ++qq) {
        const FRef yr{y + (size_t)T.j[qq] * n, T.ylo[qq], T.yhi[qq]};
        const double c = T.coef[r][qq];
        if (c != 0.0) acc -= c * yr.base[p];
        const Op od = T.od[r][qq];
        if (od.present) {
          const Nb xn = gather_direct<NDIM>(yr, s, q, p, o, sl, g.slab);
          Nb an;
          if (a_stencil<KIND>())
            an = gather_direct<NDIM>(fref(od), s, q, p, o, sl, g.slab);
          else
            an.c = od.a[p];
          acc += dt * lx_nb<KIND, NDIM>(g, kp, an, od.sigma, xn);
        }
      }
      rhs[(size_t)r * n + p] = acc;
    }
  }
}

// ============================================================ launchers

template <class F>
static void dispatch_kd23(int kind, int ndim, F f) {
  auto with_dim = [&](auto K) {
    if (ndim == 2)
      f(K, std::integral_constant<int, 2>{});
    else
      f(K, std::integral_constant<int, 3>{});
  };
  switch (kind) {
    case KIND_NLDIFF: with_dim(std::integral_constant<int, KIND_NLDIFF>{}); break;
    case KIND_BURGERS: with_dim(std::integral_constant<int, KIND_BURGERS>{}); break;
    default: with_dim(std::integral_constant<int, KIND_RAD>{}); break;
  }
}

// grid + slide span for ~8 CTAs per SM
dim3 Engine::slide_grid(int &span) const {
  static int cps = -1;
  if (cps < 0) {
    const char *e = getenv("IRKG_SLIDE_CPS");
    cps = e && atoi(e) > 0 ? atoi(e) : 8;
  }
  if (ndim == 2) {
    const int bx = (grid.nx + SBX - 1) / SBX;
    long long target = (long long)sms * cps;
    int sp = (int)((long long)bx * grid.ny / target);
    sp = sp < 2 ? 2 : (sp > 32 ? 32 : sp);
    span = sp;
    return dim3(bx, (grid.ny + sp - 1) / sp, 1);
  }
  const int bx = (grid.nx + 31) / 32, by = (grid.ny + SBX / 32 - 1) / (SBX / 32);
  long long target = (long long)sms * cps;
  int sp = (int)((long long)bx * by * grid.nz / target);
  sp = sp < 2 ? 2 : (sp > 32 ? 32 : sp);
  span = sp;
  return dim3(bx, by, (grid.nz + sp - 1) / sp);
}

void Engine::jac_sweep_s(const Op &L, double alpha, double dt, const VecIn &vin, int in_off,
                         const double *t_in, const double *x, double *x_out, const GCtrl *skip) {
  int span;
  const dim3 gr = slide_grid(span);
  dispatch_kd23(prob.kind, ndim, [&](auto KD, auto ND) {
    k_jac_sweep_s<decltype(KD)::value, decltype(ND)::value>
        <<<gr, SBX, 0, stream>>>(grid, kp, opref(L), alpha, dt, vin, in_off, t_in, ref(x), x_out,
                                 span, skip);
  });
  count(1);
}

void Engine::block_op_s(const BlockSpec &B, const double *z, double *w, const double *b,
                        double *out_norm, const GCtrl *skip) {
  if (strip_op && ndim == 2 && grid.nx % 2 == 0 && grid.nx >= 64) {
    // strips of BWC columns x bands of rows: ~bop_wps resident warps per SM
    const int strips = (grid.nx + BWC - 1) / BWC;
    const int wps = B.size == 1 ? 2 * bop_wps : bop_wps;
    long long bands = (long long)sms * wps / strips;
    bands = bands < 1 ? 1 : bands;
    int span = (int)((grid.ny + bands - 1) / bands);
    span = span < 4 ? 4 : span;
    if (span > grid.ny) span = grid.ny;
    const int nb = (grid.ny + span - 1) / span;
    int br[2][2] = {{0, nb}, {0, 0}};
    if (band_sel != 0 && !b) {  // slab halo overlap (never for the residual form)
      int lo, hi;
      interior_bands(nb, span, 1, lo, hi);
      if (band_sel == 1) {
        br[0][0] = lo;
        br[0][1] = hi;
      } else {
        br[0][0] = 0;
        br[0][1] = lo;
        br[1][0] = hi;
        br[1][1] = nb;
      }
    } else if (band_sel == 2) {
      br[0][1] = 0;  // (band_sel 1 did all of them)
    }
    const FRef z1 = ref(z);
    auto launch2 = [&](auto KD, auto SL) {
      constexpr int K_ = decltype(KD)::value;
      constexpr bool S_ = decltype(SL)::value;
      // opt in above the 48 KB default (static + dynamic shared memory)
      static bool attr[2] = {false, false};
      auto opt_in = [&](const void *fn, int size, int bytes) {
        if (!attr[size - 1]) {
          check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
                "strip op smem");
          attr[size - 1] = true;
        }
      };
      opt_in((const void *)k_block_op_strip<K_, 1, S_>, 1, BPW * BRING * bop_nf<1>() * 64 * 8);
      opt_in((const void *)k_block_op_strip<K_, 2, S_>, 2, BPW * BRING * bop_nf<2>() * 64 * 8);
      for (int r = 0; r < 2; ++r) {
        const int nbr = br[r][1] - br[r][0];
        if (nbr <= 0) continue;
        const int nwarps = strips * nbr;
        const int blocks = (nwarps + BPW - 1) / BPW;
        if (B.size == 1)
          launch_pdl(k_block_op_strip<K_, 1, S_>, dim3(blocks), dim3(BPW * 32),
                     (size_t)BPW * BRING * bop_nf<1>() * 64 * 8, grid, kp, B.eta, B.beta, B.phi,
                     B.dt, opref(B.l1), opref(B.l2), opref(B.c12), opref(B.c21), z1,
                     FRef{nullptr, nullptr, nullptr}, w, b, span, strips, nwarps, br[r][0], part,
                     counter, out_norm, skip);
        else
          launch_pdl(k_block_op_strip<K_, 2, S_>, dim3(blocks), dim3(BPW * 32),
                     (size_t)BPW * BRING * bop_nf<2>() * 64 * 8, grid, kp, B.eta, B.beta, B.phi,
                     B.dt, opref(B.l1), opref(B.l2), opref(B.c12), opref(B.c21), z1, ref(z + N),
                     w, b, span, strips, nwarps, br[r][0], part, counter, out_norm, skip);
      }
    };
    auto launch = [&](auto KD) {
      if (grid.slab)
        launch2(KD, std::true_type{});
      else
        launch2(KD, std::false_type{});
    };
    switch (prob.kind) {
      case KIND_NLDIFF: launch(std::integral_constant<int, KIND_NLDIFF>{}); break;
      case KIND_BURGERS: launch(std::integral_constant<int, KIND_BURGERS>{}); break;
      default: launch(std::integral_constant<int, KIND_RAD>{}); break;
    }
    count(1);
    return;
  }
  int span;
  const dim3 gr = slide_grid(span);
  dispatch_kd23(prob.kind, ndim, [&](auto KD, auto ND) {
    constexpr int K_ = decltype(KD)::value, D_ = decltype(ND)::value;
    if (B.size == 1)
      k_block_op_s<K_, D_, 1><<<gr, SBX, 0, stream>>>(
          grid, kp, B.eta, B.beta, B.phi, B.dt, opref(B.l1), opref(B.l2), opref(B.c12),
          opref(B.c21), ref(z), FRef{nullptr, nullptr, nullptr}, w, b, span, part, counter,
          out_norm, skip);
    else
      k_block_op_s<K_, D_, 2><<<gr, SBX, 0, stream>>>(
          grid, kp, B.eta, B.beta, B.phi, B.dt, opref(B.l1), opref(B.l2), opref(B.c12),
          opref(B.c21), ref(z), ref(z + N), w, b, span, part, counter, out_norm, skip);
  });
  count(1);
}

void Engine::backsub_s(double dt, BacksubTerms T, const double *gst, const double *y,
                       double *rhs) {
  int span;
  const dim3 gr = slide_grid(span);
  for (int qq = 0; qq < T.njs; ++qq) {
    const FRef f = ref(y + (size_t)T.j[qq] * N);
    T.ylo[qq] = f.lo;
    T.yhi[qq] = f.hi;
    for (int r = 0; r < T.rows; ++r) T.od[r][qq] = opref(T.od[r][qq]);
  }
  dispatch_kd23(prob.kind, ndim, [&](auto KD, auto ND) {
    launch_pdl(k_backsub_s<decltype(KD)::value, decltype(ND)::value>, gr, dim3(SBX), 0, grid, kp, dt,
               T, gst, y, rhs, span);
  });
  count(1);
}

double Engine::residual_s(const double *Ust, const double *K, double *Fo, int nst) {
  int span;
  const dim3 gr = slide_grid(span);
  if (slab())
    for (int i = 0; i < nst; ++i) exchange(R_STAGE + i, Ust + (size_t)i * N, 1);
  dispatch_kd23(prob.kind, ndim, [&](auto KD, auto ND) {
    launch_pdl(k_residual_s<decltype(KD)::value, decltype(ND)::value>, gr, dim3(SBX), 0, grid, kp,
               nst, Ust, stage_ghosts(Ust, N, nst), K, Fo, span, part, counter, &scal_dev[0]);
  });
  count(1);
  allreduce(&scal_dev[0], 1);
  double v = 0.0;
  v = read_scalar();
  return v;
}

}  // namespace irkg
