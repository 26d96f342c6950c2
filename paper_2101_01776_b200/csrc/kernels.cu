// kernels.cu -- device kernels + host launchers (see kernels.cuh for the rules).
#include <cstdio>
#include <type_traits>

#include "engine.h"

namespace irkg {

// ------------------------------------------------------------ reductions

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int BS>
__device__ __forceinline__ double block_sum(double v, double *sm) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = (lane < BS / 32) ? sm[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;  // valid in thread 0
}

// Last-CTA ticket.  Every CTA calls it after writing its partials; returns
// true in all threads of the CTA that finished last.
__device__ __forceinline__ bool last_block(unsigned *counter, int G) {
  __shared__ bool is_last;
  __syncthreads();  // every thread's partials ordered before thread 0's fence
  if (threadIdx.x == 0) {
    __threadfence();
    is_last = (atomicAdd(counter, 1u) == (unsigned)(G - 1));
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

// Fold part[l*G + c] over c (fixed order per lane, fixed shuffle tree).
__device__ __forceinline__ double fold_partials(const double *part, int l, int G) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int c = lane; c < G; c += 32) s += __ldcg(part + (size_t)l * G + c);
  return warp_sum(s);
}

template <int BS>
__global__ void k_norm2(int n, const double *__restrict__ x, double *part, int G, double *out,
                        unsigned *counter, const GCtrl *ctrl) {
  pdl_wait();  // (PDL launch; no early trigger: a bandwidth kernel keeps its SMs)
  __shared__ double sm[32];
  if (ctrl && ctrl->cycle_done) return;
  double acc = 0.0;
  // four loads in flight per thread; summed in the order of the plain strided loop
  const long long st = (long long)G * BS;
  for (long long p = blockIdx.x * BS + threadIdx.x; p < n; p += 4 * st) {
    double v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = (p + j * st < n) ? x[p + j * st] : 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) acc += v[j] * v[j];
  }
  acc = block_sum<BS>(acc, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
  if (!last_block(counter, G)) return;
  if (threadIdx.x < 32) {
    double s = fold_partials(part, 0, G);
    if (threadIdx.x == 0) {
      *out = s;
      *counter = 0u;
    }
  }
}

// ------------------------------------------------------ stage-space passes

// U_i = u + dt * (A0 K)_i  (src/nonlinear.py:147)
// Newton update fused with the next stage values (src/nonlinear.py:221,
// 147): K_i += sum_k (Q R0)_ik y_k ;  U_i = u + dt sum_j A0_ij K_j.
// Same arithmetic as stage_mix (dk) + stage_mix (K += dk) + stage_values.
// V consecutive points per thread (V = 2: double2 loads/stores when the
// stage rows are 16-byte aligned); per point the same operations in the same
// order as the scalar form.
template <int V>
struct Vx {
  static __device__ __forceinline__ void ld(const double *__restrict__ p, double (&o)[V]) {
    if constexpr (V == 2) {
      const double2 t = *reinterpret_cast<const double2 *>(p);
      o[0] = t.x;
      o[1] = t.y;
    } else {
      o[0] = p[0];
    }
  }
  static __device__ __forceinline__ void st(double *__restrict__ p, const double (&o)[V]) {
    if constexpr (V == 2)
      *reinterpret_cast<double2 *>(p) = make_double2(o[0], o[1]);
    else
      p[0] = o[0];
  }
};

// S = the stage count as a template parameter: with a runtime s the register
// arrays were sized for MAXS = 8 stages (119-128 registers: two CTAs of 256
// threads per SM, and these passes ran at half the copy bandwidth).
template <int V, int S>
__global__ void k_newton_update(int n, StageConsts QR, StageConsts A, double dt,
                                const double *__restrict__ Y, const double *__restrict__ u,
                                double *__restrict__ K, double *__restrict__ U) {
  pdl_wait();  // (PDL launch; no early trigger: a bandwidth kernel keeps its SMs)
  const int np = n / V;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < np; q += gridDim.x * blockDim.x) {
    const size_t p = (size_t)q * V;
    double yv[S][V], kv[S][V], up[V];
#pragma unroll
    for (int k = 0; k < S; ++k) Vx<V>::ld(Y + (size_t)k * n + p, yv[k]);
#pragma unroll
    for (int i = 0; i < S; ++i) Vx<V>::ld(K + (size_t)i * n + p, kv[i]);
    Vx<V>::ld(u + p, up);
#pragma unroll
    for (int i = 0; i < S; ++i) {
#pragma unroll
      for (int e = 0; e < V; ++e) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < S; ++k) acc += QR.a[i * MAXS + k] * yv[k][e];
        kv[i][e] = kv[i][e] + acc;
      }
      Vx<V>::st(K + (size_t)i * n + p, kv[i]);
    }
#pragma unroll
    for (int i = 0; i < S; ++i) {
      double o[V];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < S; ++j) acc += A.a[i * MAXS + j] * kv[j][e];
        o[e] = up[e] + dt * acc;
      }
      Vx<V>::st(U + (size_t)i * n + p, o);
    }
  }
}

// UNR consecutive 32-point chunks per warp and trip: at small S a thread
// otherwise has only S loads in flight
template <int V, int S, int UNR>
__global__ void k_stage_values(int n, const double *__restrict__ u, const double *__restrict__ K,
                               StageConsts A, double dt, double *__restrict__ U) {
  pdl_wait();  // (PDL launch; no early trigger: a bandwidth kernel keeps its SMs)
  const int np = n / V;
  const int lane = threadIdx.x & 31;
  const int wst = (gridDim.x * blockDim.x) >> 5;
  for (int c0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * UNR; c0 * 32 < np;
       c0 += UNR * wst) {
    const int q0 = c0 * 32 + lane;
    double kv[UNR][S][V], up[UNR][V];
#pragma unroll
    for (int r = 0; r < UNR; ++r) {
      const int q = q0 + r * 32;
      if (q < np) {
        const size_t p = (size_t)q * V;
#pragma unroll
        for (int j = 0; j < S; ++j) Vx<V>::ld(K + (size_t)j * n + p, kv[r][j]);
        Vx<V>::ld(u + p, up[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < UNR; ++r) {
      const int q = q0 + r * 32;
      if (q < np) {
        const size_t p = (size_t)q * V;
#pragma unroll
        for (int i = 0; i < S; ++i) {
          double o[V];
#pragma unroll
          for (int e = 0; e < V; ++e) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < S; ++j) acc += A.a[i * MAXS + j] * kv[r][j][e];
            o[e] = up[r][e] + dt * acc;
          }
          Vx<V>::st(U + (size_t)i * n + p, o);
        }
      }
    }
  }
}

// F_i = N(U_i) - K_i and ||F||^2  (src/nonlinear.py:148-152)
template <int KIND, int NDIM, int BS>
__global__ void k_residual(Grid g, KindParams kp, int s, const double *__restrict__ U,
                           const double *__restrict__ K, double *__restrict__ F, double *part,
                           int G, double *out, unsigned *counter) {
  __shared__ double sm[32];
  const int n = g.n;
  const int nrows = g.ny * g.nz;
  double acc = 0.0;
  for (int row = blockIdx.x; row < nrows; row += G) {
    const RowCtx rc = row_ctx<NDIM>(g, row);
    for (int ix = threadIdx.x; ix < g.nx; ix += BS) {
      int nb[6];
      const int p = row_neighbours<NDIM>(g, rc, ix, nb);
      for (int i = 0; i < s; ++i) {
        double f = rhs_at<KIND, NDIM>(g, kp, U + (size_t)i * n, p, nb) - K[(size_t)i * n + p];
        F[(size_t)i * n + p] = f;
        acc += f * f;
      }
    }
  }
  acc = block_sum<BS>(acc, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
  if (!last_block(counter, G)) return;
  if (threadIdx.x < 32) {
    double t = fold_partials(part, 0, G);
    if (threadIdx.x == 0) {
      *out = t;
      *counter = 0u;
    }
  }
}

// a_o = sum_k w[o][k] f(U_k), zero weights skipped, stage order
// (combine, src/sparsela.py:120-127)
template <int KIND>
__global__ void k_opfields(int n, KindParams kp, OpWeights W, const double *__restrict__ U,
                           double *__restrict__ A) {
  pdl_wait();  // (PDL launch; no early trigger: a bandwidth kernel keeps its SMs)
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    double f[MAXS];
#pragma unroll
    for (int k = 0; k < MAXS; ++k)
      if (k < W.s) f[k] = field_of<KIND>(kp, U[(size_t)k * n + p]);
    for (int o = 0; o < W.nops; ++o) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < MAXS; ++k) {
        if (k < W.s) {
          double wk = W.w[o * MAXS + k];
          if (wk != 0.0) acc += wk * f[k];
        }
      }
      A[(size_t)o * n + p] = acc;
    }
  }
}

// out_i = sum_k M[i][k] in_k  (pointwise s x s mix; g = Q^T F, dk = (Q R0) y)
// mode 0: out = M in; mode 1: out += M in (Newton update K += dk)
template <int V, int S, int UNR>
__global__ void k_stage_mix(int n, StageConsts M, const double *__restrict__ in,
                            double *__restrict__ out, int accumulate) {
  pdl_wait();  // (PDL launch; no early trigger: a bandwidth kernel keeps its SMs)
  const int np = n / V;
  const int lane = threadIdx.x & 31;
  const int wst = (gridDim.x * blockDim.x) >> 5;
  for (int c0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * UNR; c0 * 32 < np;
       c0 += UNR * wst) {
    const int q0 = c0 * 32 + lane;
    double v[UNR][S][V];
#pragma unroll
    for (int r = 0; r < UNR; ++r) {
      const int q = q0 + r * 32;
      if (q < np) {
#pragma unroll
        for (int k = 0; k < S; ++k) Vx<V>::ld(in + (size_t)k * n + (size_t)q * V, v[r][k]);
      }
    }
#pragma unroll
    for (int r = 0; r < UNR; ++r) {
      const int q = q0 + r * 32;
      if (q < np) {
        const size_t p = (size_t)q * V;
#pragma unroll
        for (int i = 0; i < S; ++i) {
          double o[V];
          if (accumulate) Vx<V>::ld(out + (size_t)i * n + p, o);
#pragma unroll
          for (int e = 0; e < V; ++e) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < S; ++k) acc += M.a[i * MAXS + k] * v[r][k][e];
            o[e] = accumulate ? o[e] + acc : acc;
          }
          Vx<V>::st(out + (size_t)i * n + p, o);
        }
      }
    }
  }
}

// u <- u + dt * sum_i b_i K_i  (src/nonlinear.py:313)
__global__ void k_step_update(int n, int s, StageConsts B, double dt, const double *__restrict__ K,
                              double *__restrict__ u) {
  pdl_wait();  // (PDL launch; no early trigger: a bandwidth kernel keeps its SMs)
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < MAXS; ++i)
      if (i < s) acc += B.v[i] * K[(size_t)i * n + p];
    u[p] = u[p] + dt * acc;
  }
}

// Block right-hand side: acc_r = g_r - sum_j R0[r,j] y_j + dt * sum_j od(r,j) y_j
// (src/irk_core.py:273-283); writes rows contiguously into rhs (rows, N).
template <int KIND, int NDIM>
__global__ void k_backsub(Grid g, KindParams kp, double dt, BacksubTerms T,
                          const double *__restrict__ gst, const double *__restrict__ y,
                          double *__restrict__ rhs) {
  const int n = g.n;
  const int nrows = g.ny * g.nz;
  for (int row = blockIdx.x; row < nrows; row += gridDim.x)
  for (int ix = threadIdx.x; ix < g.nx; ix += blockDim.x) {
    int nb[6];
    const int p = row_neighbours<NDIM>(g, row_ctx<NDIM>(g, row), ix, nb);
    for (int r = 0; r < T.rows; ++r) {
      double acc = gst[(size_t)(T.row0 + r) * n + p];
      for (int q = 0; q < T.njs; ++q) {
        const double *yj = y + (size_t)T.j[q] * n;
        double c = T.coef[r][q];
        if (c != 0.0) acc -= c * yj[p];
        const Op od = T.od[r][q];
        if (od.present) acc += dt * lx_at<KIND, NDIM>(g, kp, od.a, od.sigma, yj, p, nb);
      }
      rhs[(size_t)r * n + p] = acc;
    }
  }
}

// ---------------------------------------------------- inner solves / ops

__device__ __forceinline__ void resolve_in(const VecIn &vi, const double *&ptr, double &scale) {
  ptr = vin_resolve(vi, 0, scale).base;
}

// First damped-Jacobi sweep from x = 0:  x = omega * (r / D)
// r = scale*in (+ cpl*zc, materialised into t_out when coupling).
template <int KIND>
__global__ void k_jac_first(Grid g, KindParams kp, Op L, double alpha, double dt, VecIn vin,
                            int in_off, const double *__restrict__ zc, double cpl,
                            double *__restrict__ t_out, double *__restrict__ x_out,
                            GCtrl *flag_ctrl, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  const double *in;
  double scale;
  resolve_in(vin, in, scale);
  in += in_off;
  const int n = g.n;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    double r = scale * in[p];
    if (zc) {
      r = r + cpl * zc[p];
      t_out[p] = r;
    }
    double D = alpha - dt * ldiag_at<KIND>(g, kp, L.a, L.sigma, p);
    if (D == 0.0) flag_ctrl->zero_diag = 1;
    x_out[p] = OMEGA * ((1.0 / D) * r);
  }
}

// Later sweeps: x' = x + omega * (r - (alpha x - dt L x)) / D
template <int KIND, int NDIM>
__global__ void k_jac_sweep(Grid g, KindParams kp, Op L, double alpha, double dt, VecIn vin,
                            int in_off, const double *__restrict__ t_in,
                            const double *__restrict__ x, double *__restrict__ x_out,
                            const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  const double *in = nullptr;
  double scale = 1.0;
  if (!t_in) {
    resolve_in(vin, in, scale);
    in += in_off;
  }
  const int nrows = g.ny * g.nz;
  for (int row = blockIdx.x; row < nrows; row += gridDim.x) {
    const RowCtx rc = row_ctx<NDIM>(g, row);
    for (int ix = threadIdx.x; ix < g.nx; ix += blockDim.x) {
    int nb[6];
    const int p = row_neighbours<NDIM>(g, rc, ix, nb);
    double r = t_in ? t_in[p] : scale * in[p];
    double xp = x[p];
    double sx = alpha * xp - dt * lx_at<KIND, NDIM>(g, kp, L.a, L.sigma, x, p, nb);
    double D = alpha - dt * ldiag_at<KIND>(g, kp, L.a, L.sigma, p);
    x_out[p] = xp + OMEGA * ((1.0 / D) * (r - sx));
    }
  }
}

// Block operator y = A z (size 1: eta z - dt L1 z; size 2: apply_block2x2,
// src/irk_core.py:126-140).  With b != null writes r = b - A z instead and
// reduces ||r||^2 into *out_norm.
template <int KIND, int NDIM, int SIZE, int BS>
__global__ void k_block_op(Grid g, KindParams kp, double eta, double beta, double phi, double dt,
                           Op l1, Op l2, Op c12, Op c21, const double *__restrict__ z,
                           double *__restrict__ w, const double *__restrict__ b, double *part,
                           int G, double *out_norm, unsigned *counter, const GCtrl *skip) {
  __shared__ double sm[32];
  if (skip && skip->cycle_done) return;
  const int n = g.n;
  double nrm = 0.0;
  const int nrows = g.ny * g.nz;
  for (int row = blockIdx.x; row < nrows; row += G)
  for (int ix = threadIdx.x; ix < g.nx; ix += BS) {
    int nb[6];
    const int p = row_neighbours<NDIM>(g, row_ctx<NDIM>(g, row), ix, nb);
    if (SIZE == 1) {
      double v = eta * z[p] - dt * lx_at<KIND, NDIM>(g, kp, l1.a, l1.sigma, z, p, nb);
      if (b) {
        v = b[p] - v;
        nrm += v * v;
      }
      w[p] = v;
    } else {
      const double *z1 = z, *z2 = z + n;
      double x1 = z1[p], x2 = z2[p];
      double top = eta * x1 - dt * lx_at<KIND, NDIM>(g, kp, l1.a, l1.sigma, z1, p, nb) + phi * x2;
      double bot = -(beta * beta / phi) * x1 + eta * x2 -
                   dt * lx_at<KIND, NDIM>(g, kp, l2.a, l2.sigma, z2, p, nb);
      if (c12.present) top -= dt * lx_at<KIND, NDIM>(g, kp, c12.a, c12.sigma, z2, p, nb);
      if (c21.present) bot -= dt * lx_at<KIND, NDIM>(g, kp, c21.a, c21.sigma, z1, p, nb);
      if (b) {
        top = b[p] - top;
        bot = b[p + n] - bot;
        nrm += top * top + bot * bot;
      }
      w[p] = top;
      w[p + n] = bot;
    }
  }
  if (!b) return;
  nrm = block_sum<BS>(nrm, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = nrm;
  if (!last_block(counter, G)) return;
  if (threadIdx.x < 32) {
    double t = fold_partials(part, 0, G);
    if (threadIdx.x == 0) {
      *out_norm = t;
      *counter = 0u;
    }
  }
}

// ----------------------------------------------------------- CGS2 sweeps



// ------------------------------------------------------ scalar control

// Start a restart cycle: v_0 = r / beta  (src/sparsela.py:207-216).
// Control block of a fresh solve from the device-side ||b||^2 (x0 = 0):
// no host round trip before the first cycle.  b = 0 is converged at once
// (src/sparsela.py:193-198); the cycles then run as no-ops.
__global__ void k_gmres_init(GWork W, const double *bn2, int maxit, double rtol) {
  pdl_wait();  // (launched with programmatic stream serialisation)
  pdl_trigger();
  GCtrl *c = W.ctrl;
  const double bnorm = sqrt(*bn2);
  GCtrl z{};
  z.maxit = maxit;
  z.rtol = rtol;
  z.bnorm = bnorm;
  z.beta = bnorm;
  z.n_res = 1;
  z.converged = (bnorm == 0.0) ? 1 : 0;
  *c = z;
  W.res[0] = (bnorm == 0.0) ? 0.0 : 1.0;
}

__global__ void k_cycle_init(GWork W, int m) {
  pdl_wait();  // (launched with programmatic stream serialisation)
  pdl_trigger();
  GCtrl *c = W.ctrl;
  if (c->bnorm == 0.0) {  // zero right-hand side: nothing to iterate
    c->k = 0;
    c->cycle_done = 1;
    return;
  }
  c->j = 0;
  c->m = m;
  c->k = 0;
  c->cycle_done = 0;
  c->breakdown = 0;
  W.g[0] = c->beta;
  W.alpha[0] = 1.0 / c->beta;
}


// y = H(:k,:k)^{-1} g(:k) by back substitution (src/sparsela.py:258-261),
// then fold alpha into y so that x += V (alpha .* y).
// Column-oriented on MAXR threads: thread l keeps the running r_l = g_l -
// sum_{i' > l} H(l,i') y_i' in a register; column i-1 of H is fetched while
// column i is applied, so the k sequential steps cost two barriers each
// instead of k dependent global loads.
__global__ void __launch_bounds__(MAXR) k_backsolve(GWork W) {
  pdl_wait();  // (launched with programmatic stream serialisation)
  pdl_trigger();
  __shared__ double ybc;
  const GCtrl *c = W.ctrl;
  const int k = c->k;
  const int t = threadIdx.x;
  double r = t < k ? W.g[t] : 0.0;
  double yt = 0.0;
  double hcol = (k > 0 && t < k) ? W.H[(size_t)(k - 1) * (MAXR + 1) + t] : 0.0;
  for (int i = k - 1; i >= 0; --i) {
    const double hnext = (i > 0 && t < i) ? W.H[(size_t)(i - 1) * (MAXR + 1) + t] : 0.0;
    if (t == i) {
      yt = r / hcol;  // hcol = H(i,i) in thread i
      ybc = yt;
    }
    __syncthreads();
    const double yi = ybc;
    if (t < i) r -= hcol * yi;
    __syncthreads();
    hcol = hnext;
  }
  if (t < k) {
    W.y[t] = yt;
    W.c1[t] = W.alpha[t] * yt;
  }
}

// out = sum_{l<k} s_l * coef_l
__global__ void k_vcombine(int n, const double *__restrict__ V, long long pitch, const GCtrl *ctrl,
                           const double *__restrict__ coef, double *__restrict__ out) {
  pdl_wait();  // (PDL launch; no early trigger: a bandwidth kernel keeps its SMs)
  const int k = ctrl->k;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double a0 = 0.0, a1 = 0.0;
    int l = 0;
    for (; l + 2 <= k; l += 2) {
      a0 += V[(size_t)l * pitch + r] * coef[l];
      a1 += V[(size_t)(l + 1) * pitch + r] * coef[l + 1];
    }
    if (l < k) a0 += V[(size_t)l * pitch + r] * coef[l];
    out[r] = a0 + a1;
  }
}

// y += a x; V values per access, 4 accesses of each vector in flight per thread
template <int V>
__global__ void k_axpy(int n, double a, const double *__restrict__ x, double *__restrict__ y) {
  pdl_wait();  // (PDL launch; no early trigger: a bandwidth kernel keeps its SMs)
  const int np = n / V;
  const int st = gridDim.x * blockDim.x;
  for (int q0 = blockIdx.x * blockDim.x + threadIdx.x; q0 < np; q0 += 4 * st) {
    double xv[4][V], yv[4][V];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (q0 + r * st < np) {
        Vx<V>::ld(x + (size_t)(q0 + r * st) * V, xv[r]);
        Vx<V>::ld(y + (size_t)(q0 + r * st) * V, yv[r]);
      }
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (q0 + r * st < np) {
#pragma unroll
        for (int e = 0; e < V; ++e) yv[r][e] = yv[r][e] + a * xv[r][e];
        Vx<V>::st(y + (size_t)(q0 + r * st) * V, yv[r]);
      }
  }
}

// True residual bookkeeping after x += Z y (src/sparsela.py:263-272).
__global__ void k_cycle_end(GWork W) {
  pdl_wait();  // (launched with programmatic stream serialisation)
  pdl_trigger();
  GCtrl *c = W.ctrl;
  if (c->bnorm == 0.0) return;
  double rn = sqrt(c->rr);
  double true_rel = rn / c->bnorm;
  W.res[c->n_res - 1] = true_rel;
  if (true_rel <= c->rtol)
    c->converged = 1;
  else if (c->breakdown)
    c->err_breakdown = 1;
  c->beta = rn;
}

// ============================================================ launchers

template <class F>
static void dispatch_kind(int kind, F f) {
  switch (kind) {
    case KIND_NLDIFF: f(std::integral_constant<int, KIND_NLDIFF>{}); break;
    case KIND_BURGERS: f(std::integral_constant<int, KIND_BURGERS>{}); break;
    default: f(std::integral_constant<int, KIND_RAD>{}); break;
  }
}

template <class F>
static void dispatch_kd(int kind, int ndim, F f) {
  dispatch_kind(kind, [&](auto K) {
    switch (ndim) {
      case 1: f(K, std::integral_constant<int, 1>{}); break;
      case 2: f(K, std::integral_constant<int, 2>{}); break;
      default: f(K, std::integral_constant<int, 3>{}); break;
    }
  });
}

// pair (double2) path of the stage-space kernels: even row length and
// 16-byte-aligned stage rows
// the stage count as a compile-time constant (register arrays of exactly s rows)
template <class F>
static void dispatch_stages(int s, F f) {
  switch (s) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 5: f(std::integral_constant<int, 5>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    case 7: f(std::integral_constant<int, 7>{}); break;
    default: f(std::integral_constant<int, 8>{}); break;
  }
}

static bool pair_ok(long long n, const void *a, const void *b, const void *c, const void *d) {
  auto al = [](const void *p) { return ((uintptr_t)p & 15u) == 0; };
  return n % 2 == 0 && al(a) && al(b) && al(c) && al(d);
}

int Engine::grid_for(long long n) const {
  long long b = (n + 255) / 256;
  long long cap = (long long)sms * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

// every launcher reports here: a failed launch (bad configuration, shared
// memory over the limit) surfaces immediately instead of as a stalled solve
void Engine::count(int k) {
  counters.kernel_launches += k;
  check(cudaPeekAtLastError(), "kernel launch");
}

double Engine::norm2(const double *x, long long n, const GCtrl *skip) {
  launch_pdl(k_norm2<256>, dim3(G), dim3(256), 0, (int)n, x, part, G, &scal_dev[0], counter, skip);
  count(1);
  allreduce(&scal_dev[0], 1);
  double v = 0.0;
  v = read_scalar();
  return v;
}

void Engine::newton_update(const double *QR_rowmajor_s, double dt, const double *Yv,
                           const double *u, double *K, double *Uo) {
  StageConsts QR{}, A{};
  QR.s = A.s = s;
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j) {
      QR.a[i * MAXS + j] = QR_rowmajor_s[i * s + j];
      A.a[i * MAXS + j] = tab.a0[i * IRKG_MAX_STAGES + j];
    }
  const bool pair = pair_ok(N, Yv, u, K, Uo);
  dispatch_stages(s, [&](auto SC) {
    constexpr int S_ = decltype(SC)::value;
    if (pair)
      launch_pdl(k_newton_update<2, S_>, dim3(grid_for(N / 2)), dim3(256), 0, (int)N, QR, A, dt, Yv,
                 u, K, Uo);
    else
      launch_pdl(k_newton_update<1, S_>, dim3(grid_for(N)), dim3(256), 0, (int)N, QR, A, dt, Yv, u,
                 K, Uo);
  });
  count(1);
}

// sum of squares into scal_dev[0] (all ranks), no host round trip
void Engine::norm2_dev(const double *x, long long n) {
  launch_pdl(k_norm2<256>, dim3(G), dim3(256), 0, (int)n, x, part, G, &scal_dev[0], counter,
             (const GCtrl *)nullptr);
  count(1);
  allreduce(&scal_dev[0], 1);
}

void Engine::stage_values(const double *u, const double *K, double dt, double *U) {
  stage_values_n(u, K, dt, U, N);
}

void Engine::stage_values_n(const double *u, const double *K, double dt, double *Uo, long long n) {
  StageConsts A{};
  A.s = s;
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j) A.a[i * MAXS + j] = tab.a0[i * IRKG_MAX_STAGES + j];
  const bool pair = pair_ok(n, u, K, Uo, Uo);
  dispatch_stages(s, [&](auto SC) {
    constexpr int S_ = decltype(SC)::value;
    constexpr int UNR = S_ <= 2 ? 4 : (S_ <= 4 ? 2 : 1);
    if (pair)
      launch_pdl(k_stage_values<2, S_, UNR>, dim3(grid_for(n / 2)), dim3(256), 0, (int)n, u, K, A,
                 dt, Uo);
    else
      launch_pdl(k_stage_values<1, S_, UNR>, dim3(grid_for(n)), dim3(256), 0, (int)n, u, K, A, dt,
                 Uo);
  });
  count(1);
}

double Engine::residual(const double *U, const double *K, double *F, int nst) {
  if (nst < 0) nst = s;
  if (ndim >= 2) return residual_s(U, K, F, nst);
  dispatch_kd(prob.kind, ndim, [&](auto KD, auto ND) {
    k_residual<decltype(KD)::value, decltype(ND)::value, 256>
        <<<G, 256, 0, stream>>>(grid, kp, nst, U, K, F, part, G, &scal_dev[0], counter);
  });
  count(1);
  double v = 0.0;
  v = read_scalar();
  return v;
}

void Engine::opfields(const double *U, const OpWeights &W, double *A) {
  dispatch_kind(prob.kind, [&](auto KD) {
    launch_pdl(k_opfields<decltype(KD)::value>, dim3(grid_for(N)), dim3(256), 0, (int)N, kp, W, U,
               A);
  });
  count(1);
}

void Engine::stage_mix(const double *M_rowmajor_s, const double *in, double *out, bool accumulate) {
  stage_mix_n(M_rowmajor_s, in, out, accumulate, N);
}

void Engine::stage_mix_n(const double *M_rowmajor_s, const double *in, double *out,
                         bool accumulate, long long n) {
  StageConsts M{};
  M.s = s;
  for (int i = 0; i < s; ++i)
    for (int k = 0; k < s; ++k) M.a[i * MAXS + k] = M_rowmajor_s[i * s + k];
  const bool pair = pair_ok(n, in, out, out, out);
  dispatch_stages(s, [&](auto SC) {
    constexpr int S_ = decltype(SC)::value;
    constexpr int UNR = S_ <= 2 ? 4 : (S_ <= 4 ? 2 : 1);
    if (pair)
      launch_pdl(k_stage_mix<2, S_, UNR>, dim3(grid_for(n / 2)), dim3(256), 0, (int)n, M, in, out,
                 accumulate ? 1 : 0);
    else
      launch_pdl(k_stage_mix<1, S_, UNR>, dim3(grid_for(n)), dim3(256), 0, (int)n, M, in, out,
                 accumulate ? 1 : 0);
  });
  count(1);
}

void Engine::step_update(double dt, const double *K, double *u) { step_update_n(dt, K, u, N); }

void Engine::step_update_n(double dt, const double *K, double *u, long long n) {
  StageConsts B{};
  B.s = s;
  for (int i = 0; i < s; ++i) B.v[i] = tab.b0[i];
  launch_pdl(k_step_update, dim3(grid_for(n)), dim3(256), 0, (int)n, s, B, dt, K, u);
  count(1);
}

void Engine::backsub(double dt, const BacksubTerms &T, const double *gst, const double *y,
                     double *rhs) {
  if (ndim >= 2) {
    if (slab()) {
      bool any_od = false;
      for (int q = 0; q < T.njs; ++q)
        for (int r = 0; r < T.rows; ++r) any_od |= (T.od[r][q].present != 0);
      for (int q = 0; q < T.njs && any_od; ++q)
        exchange(R_Y + T.j[q], y + (size_t)T.j[q] * N, 1);
    }
    backsub_s(dt, T, gst, y, rhs);
    return;
  }
  dispatch_kd(prob.kind, ndim, [&](auto KD, auto ND) {
    k_backsub<decltype(KD)::value, decltype(ND)::value>
        <<<row_grid(), 256, 0, stream>>>(grid, kp, dt, T, gst, y, rhs);
  });
  count(1);
}

// Jacobi-k chain on (alpha I - dt L): x_out = S^{-1}_k (scale*in [+cpl*zc])
void Engine::jacobi_chain(const Op &L, double alpha, double dt, int inner, const void *vin_p,
                          int in_off, const double *zc, double cpl, double *x_out,
                          const GCtrl *skip) {
  const VecIn &vin = *static_cast<const VecIn *>(vin_p);
  if (prob.kind == KIND_ARAKAWA) {
    ara_jacobi_chain(L, alpha, dt, inner, vin, in_off, zc, cpl, x_out, skip);
    return;
  }
  if (jacobi_chain_fused(L, alpha, dt, inner, vin, in_off, zc, cpl, x_out, skip)) return;
  if (jacobi_chain_fused3d(L, alpha, dt, inner, vin, in_off, zc, cpl, x_out, skip)) return;
  const int gb = grid_for(N);
  double *tbuf = zc ? tmp_t : nullptr;
  // sweep i (1-based) writes into out if (inner - i) even, else tmp_x
  auto dst = [&](int i) { return ((inner - i) % 2 == 0) ? x_out : tmp_x; };
  dispatch_kind(prob.kind, [&](auto KD) {
    k_jac_first<decltype(KD)::value><<<gb, 256, 0, stream>>>(grid, kp, L, alpha, dt, vin, in_off,
                                                               zc, cpl, tbuf, dst(1), ctrl_dev,
                                                               skip);
  });
  count(1);
  for (int i = 2; i <= inner; ++i) {
    const double *xin = dst(i - 1);
    double *xo = dst(i);
    if (ndim >= 2) {
      if (slab()) exchange(R_JX, xin, 1);
      jac_sweep_s(L, alpha, dt, vin, in_off, tbuf, xin, xo, skip);
      continue;
    }
    dispatch_kd(prob.kind, ndim, [&](auto KD, auto ND) {
      k_jac_sweep<decltype(KD)::value, decltype(ND)::value>
          <<<row_grid(), 256, 0, stream>>>(grid, kp, L, alpha, dt, vin, in_off, tbuf, xin, xo, skip);
    });
    count(1);
  }
  counters.precond_bytes += 8.0 * N * ((zc ? 4.0 : 3.0) + (inner - 1) * 4.0);
}

void Engine::precond(const BlockSpec &B, const void *vin_p, double *z, const GCtrl *skip) {
  VecIn vin = *static_cast<const VecIn *>(vin_p);
  if (B.inner == IRKG_INNER_EXACT) {  // factors prepared by gmres() (banded.cu)
    precond_exact(B, vin, z, skip);
    return;
  }
  if (B.inner == IRKG_INNER_MG) {  // hierarchy prepared by gmres() (mg.cu)
    precond_mg(B, vin, z, skip);
    return;
  }
  const bool ext = ext_halo_ok() && B.inner == cfg.inner;
  if (slab()) {
    // the input must be a fixed pointer here (the multi-rank loop resolves
    // slot j on the host); exchange the halves' boundary planes
    if (vin.ctrl) throw SolveError(IRKG_ERR_CONFIG, "internal: slot-indexed input in slab mode");
    const int H = ext ? inhalo() : jhalo();
    exchange(R_VIN0, vin.base, H);
    vin.lo[0] = role(R_VIN0).lo;
    vin.hi[0] = role(R_VIN0).hi;
    if (B.size == 2) {
      exchange(R_VIN1, vin.base + N, H);
      vin.lo[1] = role(R_VIN1).lo;
      vin.hi[1] = role(R_VIN1).hi;
    }
  }
  if (ext) {
    // the chains compute the ghost rows of z1 / z2 themselves (see arnoldi_iteration_slab)
    chain_ext = B.size == 2 ? B.inner : 1;  // chain 2's reach K-1, plus the operator's row
    chain_out_role = R_Z0;
    jacobi_chain(B.l1, B.eta, B.dt, B.inner, &vin, 0, nullptr, 0.0, z, skip);
    if (B.size == 2) {
      chain_ext = 1;
      chain_out_role = R_Z1;
      jacobi_chain(B.l2, B.gamma, B.dt, B.inner, &vin, (int)N, z, B.beta * B.beta / B.phi, z + N,
                   skip);
    }
    chain_ext = 0;
    return;
  }
  if (B.size == 1) {
    jacobi_chain(B.l1, B.eta, B.dt, B.inner, &vin, 0, nullptr, 0.0, z, skip);
  } else {
    jacobi_chain(B.l1, B.eta, B.dt, B.inner, &vin, 0, nullptr, 0.0, z, skip);
    if (slab()) exchange(R_Z0, z, jhalo());  // z1 feeds the second row's rhs
    jacobi_chain(B.l2, B.gamma, B.dt, B.inner, &vin, (int)N, z, B.beta * B.beta / B.phi, z + N,
                 skip);
  }
}

void Engine::block_op(const BlockSpec &B, const double *z, double *w, const double *b,
                      double *out_norm, const GCtrl *skip) {
  counters.op_bytes += 8.0 * N * B.size * 3.0;
  if (prob.kind == KIND_ARAKAWA) {
    ara_block_op(B, z, w, b, out_norm, skip);
    return;
  }
  if (ndim >= 2) {
    if (slab()) {
      exchange(R_X0, z, 1);
      if (B.size == 2) exchange(R_X1, z + N, 1);
    }
    block_op_s(B, z, w, b, out_norm, skip);
    if (b) allreduce(out_norm, 1);
    return;
  }
  dispatch_kd(prob.kind, ndim, [&](auto KD, auto ND) {
    constexpr int K_ = decltype(KD)::value, D_ = decltype(ND)::value;
    if (B.size == 1)
      k_block_op<K_, D_, 1, 256><<<G, 256, 0, stream>>>(grid, kp, B.eta, B.beta, B.phi, B.dt,
                                                         B.l1, B.l2, B.c12, B.c21, z, w, b, part,
                                                         G, out_norm, counter, skip);
    else
      k_block_op<K_, D_, 2, 256><<<G, 256, 0, stream>>>(grid, kp, B.eta, B.beta, B.phi, B.dt,
                                                         B.l1, B.l2, B.c12, B.c21, z, w, b, part,
                                                         G, out_norm, counter, skip);
  });
  count(1);
}



void Engine::gmres_init(int maxit, double rtol) {
  launch_pdl(k_gmres_init, dim3(1), dim3(1), 0, W, (const double *)&scal_dev[0], maxit, rtol);
  count(1);
}
void Engine::cycle_init(int m) {
  launch_pdl(k_cycle_init, dim3(1), dim3(1), 0, W, m);
  count(1);
}

void Engine::backsolve() {
  launch_pdl(k_backsolve, dim3(1), dim3(MAXR), 0, W);
  count(1);
}
void Engine::vcombine(long long n, const double *coef, double *out) {
  // (plain launch: with the PDL launch's maximum shared-memory carveout the
  // basis combination ran 25 % slower -- it streams its slots through L1)
  k_vcombine<<<grid_for(n), 256, 0, stream>>>((int)n, V, vpitch, ctrl_dev, coef, out);
  count(1);
}
void Engine::axpy(long long n, double a, const double *x, double *y) {
  if (pair_ok(n, x, y, y, y))
    launch_pdl(k_axpy<2>, dim3(grid_for(n / 2)), dim3(256), 0, (int)n, a, x, y);
  else
    launch_pdl(k_axpy<1>, dim3(grid_for(n)), dim3(256), 0, (int)n, a, x, y);
  count(1);
}
void Engine::cycle_end() {
  launch_pdl(k_cycle_end, dim3(1), dim3(1), 0, W);
  count(1);
}

}  // namespace irkg
