// banded.cu -- exact inner solves: banded LU with the periodic wrap through
// Sherman-Morrison-Woodbury, on the device.
//
// Restates BandedLU (src/sparsela.py:283-359), the reference's default
// PrecondSpec(inner="exact") path of ShiftedSolver (src/irk_core.py:103-123):
//  * the in-band part of S = alpha I - dt L (|row - col| <= bw, bw = nx in
//    2-D, 1 in 1-D: the reference's band hint) is stored LAPACK-style
//    (ab: (2kl+ku+1) x n, column-major) and factored with partial pivoting
//    exactly as dgbtf2 does it, by ONE CTA that keeps the (kl+1) x (kl+ku+1)
//    active block in a circular shared-memory window (or, when that does not
//    fit, in a global scratch buffer that stays in L2);
//  * out-of-band entries (the y-periodic wrap) form U (n x nb) against the
//    border columns; B^{-1} U is computed with nb parallel banded solves,
//    the capacitance I + E^T B^{-1} U is LU-factored with partial pivoting,
//    and a solve is  y = B^{-1} b;  y -= B^{-1}U cap^{-1} y[border].
// The matrix is assembled from the matrix-free operator kinds (kinds.cuh),
// so no CSR exists anywhere.  Only 1-D and 2-D grids (3-D bands are
// nx*ny wide: the reference calls that infeasible too).
#include <algorithm>
#include <cmath>

#include "engine.h"

namespace irkg {


// S = alpha I - dt L into band storage (+= so coinciding neighbours of tiny
// grids add up) and the out-of-band entries into U (n x nb, column-major).
template <int KIND>
__global__ void k_band_assemble(Grid g, KindParams kp, const double *__restrict__ a, double sig,
                                double alpha, double dt, double *__restrict__ ab, int ldab,
                                int kl, int ku, double *__restrict__ Ub, int nb) {
  const int n = g.n, nx = g.nx;
  const int kv = kl + ku;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const int ix = p % nx, iy = p / nx;
    int nbr[4];
    nbr[0] = p + (ix == 0 ? nx - 1 : -1);
    nbr[1] = p + (ix == nx - 1 ? 1 - nx : 1);
    nbr[2] = g.ny > 1 ? p + (iy == 0 ? (g.ny - 1) * nx : -nx) : p;
    nbr[3] = g.ny > 1 ? p + (iy == g.ny - 1 ? -(g.ny - 1) * nx : nx) : p;
    double cc, cn[4];
    stencil_row<KIND>(g, kp, a, sig, p, nbr, cc, cn);
    auto put = [&](int c, double v) {
      const int d = p - c;
      if (d <= kl && -d <= ku) {
        ab[(size_t)c * ldab + kv + d] += v;
      } else {  // border column: first grid row -> t = c, last grid row -> t = nb/2 + ...
        const int half = nb / 2;
        const int t = c < half ? c : half + (c - (n - half));
        Ub[(size_t)t * n + p] += v;
      }
    };
    put(p, alpha - dt * cc);
    const int nn = g.ny > 1 ? 4 : 2;
    for (int k = 0; k < nn; ++k) put(nbr[k], -dt * cn[k]);
  }
}

// dgbtf2 (partial pivoting, first maximal |pivot|) by one CTA on a circular
// window of R = kl+2 rows x C = kl+ku+2 columns: the active block of step j
// is rows j..j+kl x columns j..j+kl+ku; the extra row / column slot lets the
// admission of row j+kl+1 / column j+kl+ku+1 proceed while row and column j
// retire.  Warps own rows, lanes columns; slots advance incrementally (no
// integer division in the loop).  info[0] = first zero pivot + 1 (0: regular).
constexpr int BF_THREADS = 256;  // (more warps only add barrier and issue overhead per step)

__global__ void __launch_bounds__(BF_THREADS)
    k_band_factor(double *__restrict__ ab, int ldab, int n, int kl, int ku, int *__restrict__ piv,
                  int *__restrict__ info, double *__restrict__ wglob) {
  extern __shared__ double wsm[];
  __shared__ int s_jp;
  double *W = wglob ? wglob : wsm;
  const int kv = kl + ku;
  const int R = kl + 2, C = kv + 2;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
  auto band = [&](int r, int c) -> double {  // original entry a(r, c) (0 outside the band)
    const int d = r - c;
    return (d <= kl && -d <= kv) ? ab[(size_t)c * ldab + kv + d] : 0.0;
  };
  auto rs = [&](int slot0, int i) {  // row slot of row (j + i), slot0 = j % R
    const int v = slot0 + i;
    return v >= R ? v - R : v;
  };
  auto cs = [&](int slot0, int o) {  // column slot of column (j + o), o < C
    const int v = slot0 + o;
    return v >= C ? v - C : v;
  };
  for (int e = tid; e < R * C; e += nthr) {
    const int r = e / C, c = e % C;  // (once)
    W[e] = (r <= kl && c <= kv && r < n && c < n) ? band(r, c) : 0.0;
  }
  if (tid == 0) info[0] = 0;
  __syncthreads();
  int ju = 0;
  int jr = 0, jc = 0;  // j % R, j % C
  for (int j = 0; j < n; ++j) {
    const int km = min(kl, n - 1 - j);
    const int rn = j + kl + 1;
    double adm = 0.0;  // this step's admission row, read early (L2 latency off the chain)
    if (tid <= kv && rn < n && j + 1 + tid < n) adm = band(rn, j + 1 + tid);
    // pivot (warp 0): first index of max |a(j..j+km, j)|
    if (warp == 0) {
      double best = -1.0;
      int bi = 0x7fffffff;
      for (int i = lane; i <= km; i += 32) {
        const double v = fabs(W[rs(jr, i) * C + jc]);
        if (v > best) {
          best = v;
          bi = i;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
          best = ov;
          bi = oi;
        }
      }
      if (lane == 0) {
        s_jp = bi;
        piv[j] = j + bi;
      }
    }
    __syncthreads();
    const int jp = s_jp;
    const int rj = jr * C, rp = rs(jr, jp) * C;
    const double pvv = W[rp + jc];
    if (pvv != 0.0) {
      ju = max(ju, min(j + ku + jp, n - 1));
      if (jp != 0) {
        for (int o = tid; o <= ju - j; o += nthr) {
          const int c = cs(jc, o);
          const double t = W[rj + c];
          W[rj + c] = W[rp + c];
          W[rp + c] = t;
        }
        __syncthreads();
      }
      const double inv = 1.0 / W[rj + jc];
      const int ncol = ju - j;
      // rows j+1..j+km (warps) x columns j+1..ju (lanes); the owner of a row
      // also scales its multiplier once its row is updated
      for (int i = 1 + warp; i <= km; i += nwarp) {
        const int ri = rs(jr, i) * C;
        const double m = W[ri + jc] * inv;
        for (int o = 1 + lane; o <= ncol; o += 32) {
          const int c = cs(jc, o);
          W[ri + c] -= m * W[rj + c];
        }
        __syncwarp();
        if (lane == 0) W[ri + jc] = m;
      }
    } else if (tid == 0 && info[0] == 0) {
      info[0] = j + 1;
    }
    __syncthreads();
    // retire row j (U) and column j (multipliers) into ab; admit row j+kl+1
    // and column j+kv+1 into the spare slots
    for (int o = tid; o <= min(kv, n - 1 - j); o += nthr)
      ab[(size_t)(j + o) * ldab + kv - o] = W[rj + cs(jc, o)];
    for (int i = 1 + tid; i <= km; i += nthr) ab[(size_t)j * ldab + kv + i] = W[rs(jr, i) * C + jc];
    {
      const int rns = rs(jr, kl + 1) * C;
      if (tid <= kv) W[rns + cs(jc, 1 + tid)] = adm;
      for (int o = 1 + nthr; o <= kv + 1; o += nthr)  // (kv >= blockDim only)
        W[rns + cs(jc, o)] = (rn < n && j + o < n) ? band(rn, j + o) : 0.0;
      const int cns = cs(jc, kv + 1);
      for (int i = 1 + tid; i <= kl; i += nthr) W[rs(jr, i) * C + cns] = 0.0;
    }
    __syncthreads();
    jr = jr + 1 == R ? 0 : jr + 1;
    jc = jc + 1 == C ? 0 : jc + 1;
  }
}

// dgbtrs('N') on nrhs columns of b (n each, stride ldb), one warp per column,
// the column held in shared memory.  The substitutions are sequential, so
// the factor columns they walk through stream into a per-warp ring of BS_D
// columns with cp.async, BS_D steps ahead (the L2 latency is off the
// dependency chain); the pivot indices sit in shared memory.
constexpr int BS_D = 48;

__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

__host__ __device__ inline int band_seg(int kl, int ku) { return kl + ku + 1; }

__global__ void k_band_solve(const double *__restrict__ ab, int ldab, int n, int kl, int ku,
                             const int *__restrict__ piv, double *__restrict__ b, long long ldb,
                             int nrhs, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  extern __shared__ double bs[];
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kv = kl + ku;
  const int seg = band_seg(kl, ku);  // >= kl (L part) and = kv + 1 (U part)
  int *pv = reinterpret_cast<int *>(bs + (size_t)nw * (n + BS_D * seg));
  for (int i = threadIdx.x; i < n; i += blockDim.x) pv[i] = piv[i];
  __syncthreads();
  const int col = blockIdx.x * nw + warp;
  if (col >= nrhs) return;
  double *x = bs + (size_t)warp * (n + BS_D * seg);
  double *ring = x + n;
  double *bg = b + (size_t)col * ldb;
  for (int i = lane; i < n; i += 32) x[i] = bg[i];
  // forward: the kl multipliers of column jc; backward: rows 0..kv of column jc
  auto issue = [&](int jc, int slot, bool live, bool fwd) {
    if (live) {
      const double *src = ab + (size_t)jc * ldab + (fwd ? kv + 1 : 0);
      const int cnt = fwd ? kl : kv + 1;
      for (int i = lane; i < cnt; i += 32) cp_async8(ring + (size_t)slot * seg + i, src + i);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto wait_oldest = [&]() {
    asm volatile("cp.async.wait_group %0;" ::"n"(BS_D - 1) : "memory");
    __syncwarp();
  };
  for (int s = 0; s < BS_D; ++s) issue(s, s, s < n - 1, true);
  __syncwarp();
  int slot = 0;
  for (int j = 0; j < n - 1; ++j) {  // L with the row interchanges
    wait_oldest();
    const double *lc = ring + (size_t)slot * seg;
    const int lm = min(kl, n - 1 - j);
    const int l = pv[j];
    if (l != j && lane == 0) {
      const double t = x[l];
      x[l] = x[j];
      x[j] = t;
    }
    __syncwarp();
    const double xj = x[j];
    for (int i = lane; i < lm; i += 32) x[j + 1 + i] -= lc[i] * xj;
    __syncwarp();
    issue(j + BS_D, slot, j + BS_D < n - 1, true);
    slot = slot + 1 == BS_D ? 0 : slot + 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
  for (int s = 0; s < BS_D; ++s) issue(n - 1 - s, s, n - 1 - s >= 0, false);
  __syncwarp();
  slot = 0;
  for (int j = n - 1; j >= 0; --j) {  // U with kl+ku superdiagonals
    wait_oldest();
    const double *uc = ring + (size_t)slot * seg;
    const double xj = x[j] / uc[kv];
    __syncwarp();
    if (lane == 0) x[j] = xj;
    const int i0 = max(0, j - kv);
    for (int i = i0 + lane; i < j; i += 32) x[i] -= uc[kv + i - j] * xj;
    __syncwarp();
    issue(j - BS_D, slot, j - BS_D >= 0, false);
    slot = slot + 1 == BS_D ? 0 : slot + 1;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
  for (int i = lane; i < n; i += 32) bg[i] = x[i];
}

// cap = I + (B^{-1}U)[border rows, :]  (nb x nb, column-major)
__global__ void k_cap_assemble(const double *__restrict__ binvu, int n, int nb,
                               double *__restrict__ cap) {
  const int half = nb / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nb * nb; e += gridDim.x * blockDim.x) {
    const int r = e % nb, t = e / nb;
    const int row = r < half ? r : n - half + (r - half);
    cap[(size_t)t * nb + r] = (r == t ? 1.0 : 0.0) + binvu[(size_t)t * n + row];
  }
}

// dense LU with partial pivoting of cap (nb x nb, column-major), one CTA;
// ipiv in the interleaved (band-style) convention
__global__ void k_dense_lu(double *__restrict__ A, int m, int *__restrict__ ipiv,
                           int *__restrict__ info) {
  __shared__ int s_p;
  const int tid = threadIdx.x;
  for (int k = 0; k < m; ++k) {
    if (tid == 0) {
      int p = k;
      double best = fabs(A[(size_t)k * m + k]);
      for (int i = k + 1; i < m; ++i) {
        const double v = fabs(A[(size_t)k * m + i]);
        if (v > best) {
          best = v;
          p = i;
        }
      }
      s_p = p;
      ipiv[k] = p;
      if (best == 0.0 && info[0] == 0) info[0] = -(k + 1);
    }
    __syncthreads();
    const int p = s_p;
    // interchange the trailing part only (columns k..m-1, as dgbtf2 does):
    // the multipliers of earlier columns stay with their elimination step,
    // which is what the interleaved row interchanges in k_smw_mid assume
    if (p != k)
      for (int c = k + tid; c < m; c += blockDim.x) {
        const double t = A[(size_t)c * m + k];
        A[(size_t)c * m + k] = A[(size_t)c * m + p];
        A[(size_t)c * m + p] = t;
      }
    __syncthreads();
    const double d = A[(size_t)k * m + k];
    const double inv = d != 0.0 ? 1.0 / d : 0.0;
    const int rem = m - k - 1;
    for (int e = tid; e < rem * rem; e += blockDim.x) {
      const int i = k + 1 + e % rem, c = k + 1 + e / rem;
      A[(size_t)c * m + i] -= (A[(size_t)k * m + i] * inv) * A[(size_t)c * m + k];
    }
    __syncthreads();
    for (int i = k + 1 + tid; i < m; i += blockDim.x) A[(size_t)k * m + i] *= inv;
    __syncthreads();
  }
}

// y -= B^{-1}U cap^{-1} y[border]: one CTA solves the nb x nb system in
// shared memory (mid), then all CTAs apply the rank-nb update
__global__ void k_smw_mid(const double *__restrict__ cap, const int *__restrict__ ipiv, int nb,
                          const double *__restrict__ y, int n, double *__restrict__ mid,
                          const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  extern __shared__ double t[];
  const int half = nb / 2;
  for (int r = threadIdx.x; r < nb; r += blockDim.x)
    t[r] = y[r < half ? r : n - half + (r - half)];
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int k = 0; k < nb; ++k) {  // row interchanges + unit L
      if (lane == 0 && ipiv[k] != k) {
        const double s = t[k];
        t[k] = t[ipiv[k]];
        t[ipiv[k]] = s;
      }
      __syncwarp();
      const double tk = t[k];
      for (int i = k + 1 + lane; i < nb; i += 32) t[i] -= cap[(size_t)k * nb + i] * tk;
      __syncwarp();
    }
    for (int k = nb - 1; k >= 0; --k) {  // U
      const double tk = t[k] / cap[(size_t)k * nb + k];
      __syncwarp();
      if (lane == 0) t[k] = tk;
      for (int i = lane; i < k; i += 32) t[i] -= cap[(size_t)k * nb + i] * tk;
      __syncwarp();
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < nb; r += blockDim.x) mid[r] = t[r];
}

__global__ void k_smw_update(const double *__restrict__ binvu, int n, int nb,
                             const double *__restrict__ mid, double *__restrict__ y,
                             const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < nb; ++t) acc += binvu[(size_t)t * n + p] * mid[t];
    y[p] -= acc;
  }
}

// out = scale * in [+ cpl * zc]  (the inner solve's right-hand side)
__global__ void k_vin_rhs(int n, VecIn vin, int in_off, const double *__restrict__ zc, double cpl,
                          double *__restrict__ out, const GCtrl *skip) {
  if (skip && skip->cycle_done) return;
  double scale;
  const FRef in = vin_resolve(vin, in_off, scale);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    double v = scale * in.base[p];
    if (zc) v = v + cpl * zc[p];
    out[p] = v;
  }
}

// ------------------------------------------------------------------ host

void Engine::band_factor(BandFactor &F, const Op &L, double alpha, double dt, const Grid *gl) {
  const Grid &gg = gl ? *gl : grid;  // (a multigrid level, or the engine's grid)
  const int nd = gg.nz > 1 ? 3 : (gg.ny > 1 ? 2 : 1);
  if (nd > 2 || slab())
    throw SolveError(IRKG_ERR_CONFIG,
                     "PrecondSpec(inner='exact') covers single-rank 1-D / 2-D grids (banded LU)");
  const int n = gg.n;
  const int bw = nd == 1 ? 1 : gg.nx;
  const int kl = std::min(bw, n - 1), ku = kl;
  const int ldab = 2 * kl + ku + 1;
  // out-of-band wrap entries: the first and last grid rows (2-D) / points (1-D)
  const int lastrow = nd == 1 ? 1 : gg.nx;
  const int nb = (n - lastrow > bw) ? 2 * lastrow : 0;
  if (F.n != n || F.ldab != ldab || F.nb != nb) {
    for (void *p : {(void *)F.ab, (void *)F.piv, (void *)F.binvu, (void *)F.cap, (void *)F.cpiv,
                    (void *)F.info, (void *)F.mid, (void *)F.wglob})
      if (p) cudaFree(p);
    F = BandFactor{};
    F.n = n;
    F.kl = kl;
    F.ku = ku;
    F.ldab = ldab;
    F.nb = nb;
    dalloc_raw((void **)&F.ab, sizeof(double) * (size_t)ldab * n);
    dalloc_raw((void **)&F.piv, sizeof(int) * (size_t)n);
    dalloc_raw((void **)&F.info, 2 * sizeof(int));
    if (nb > 0) {
      dalloc_raw((void **)&F.binvu, sizeof(double) * (size_t)n * nb);
      dalloc_raw((void **)&F.cap, sizeof(double) * (size_t)nb * nb);
      dalloc_raw((void **)&F.cpiv, sizeof(int) * (size_t)nb);
      dalloc_raw((void **)&F.mid, sizeof(double) * (size_t)nb);
    }
    const size_t wbytes = sizeof(double) * (size_t)(kl + 2) * (kl + ku + 2);
    F.wsmem = wbytes <= 200 * 1024 ? wbytes : 0;
    if (!F.wsmem) dalloc_raw((void **)&F.wglob, wbytes);
  }
  check(cudaMemsetAsync(F.ab, 0, sizeof(double) * (size_t)ldab * n, stream));
  if (nb > 0) check(cudaMemsetAsync(F.binvu, 0, sizeof(double) * (size_t)n * nb, stream));
  const int gb = grid_for(n);
  auto assemble = [&](auto KD) {
    k_band_assemble<decltype(KD)::value><<<gb, 256, 0, stream>>>(
        gg, kp, L.a, L.sigma, alpha, dt, F.ab, ldab, kl, ku, F.binvu, nb);
  };
  switch (prob.kind) {
    case KIND_NLDIFF: assemble(std::integral_constant<int, KIND_NLDIFF>{}); break;
    case KIND_BURGERS: assemble(std::integral_constant<int, KIND_BURGERS>{}); break;
    case KIND_RAD: assemble(std::integral_constant<int, KIND_RAD>{}); break;
    default: throw SolveError(IRKG_ERR_CONFIG, "exact inner solves: ODE kinds only");
  }
  if (F.wsmem)
    check(cudaFuncSetAttribute(k_band_factor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)F.wsmem), "band factor smem");
  k_band_factor<<<1, BF_THREADS, F.wsmem, stream>>>(F.ab, ldab, n, kl, ku, F.piv, F.info,
                                                     F.wsmem ? nullptr : F.wglob);
  count(3);
  if (nb > 0) {
    band_solve(F, F.binvu, n, nb, nullptr);  // B^{-1} U
    k_cap_assemble<<<std::max(1, std::min(nb * nb / 256, 4 * sms)), 256, 0, stream>>>(
        F.binvu, n, nb, F.cap);
    k_dense_lu<<<1, 1024, 0, stream>>>(F.cap, nb, F.cpiv, F.info);
    count(2);
  }
  int info = 0;
  check(cudaMemcpyAsync(&info, F.info, sizeof(int), cudaMemcpyDeviceToHost, stream));
  check(cudaStreamSynchronize(stream), "band factor");
  if (info != 0) throw SolveError(IRKG_ERR_SINGULAR, "banded factorization failed (singular)");
}

void Engine::band_solve(const BandFactor &F, double *b, long long ldb, int nrhs,
                        const GCtrl *skip) {
  const size_t per = sizeof(double) * ((size_t)F.n + (size_t)BS_D * band_seg(F.kl, F.ku));
  const size_t pivb = sizeof(int) * (size_t)F.n;
  const size_t budget = 220 * 1024 - pivb;
  if (per > budget) throw SolveError(IRKG_ERR_CONFIG, "exact inner solve: grid too large");
  int wpc = (int)std::max<size_t>(1, std::min<size_t>(4, budget / per));
  wpc = std::min(wpc, std::max(1, nrhs));
  const size_t smem = per * wpc + pivb;
  check(cudaFuncSetAttribute(k_band_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem), "band solve smem");
  k_band_solve<<<(nrhs + wpc - 1) / wpc, 32 * wpc, smem, stream>>>(F.ab, F.ldab, F.n, F.kl, F.ku,
                                                                   F.piv, b, ldb, nrhs, skip);
  count(1);
}

// x <- S^{-1} x for a factored S (BandedLU.solve, src/sparsela.py:339-352)
void Engine::band_apply(const BandFactor &F, double *x, const GCtrl *skip) {
  band_solve(F, x, F.n, 1, skip);
  if (F.nb > 0) {
    k_smw_mid<<<1, 256, sizeof(double) * F.nb, stream>>>(F.cap, F.cpiv, F.nb, x, F.n, F.mid, skip);
    k_smw_update<<<grid_for(F.n), 256, 0, stream>>>(F.binvu, F.n, F.nb, F.mid, x, skip);
    count(2);
  }
}

// the exact branch of precond(): z1 = S1^{-1} r1 ; z2 = S2^{-1} (r2 + beta^2/phi z1)
void Engine::precond_exact(const BlockSpec &B, const VecIn &vin, double *z, const GCtrl *skip) {
  const int gb = grid_for(N);
  k_vin_rhs<<<gb, 256, 0, stream>>>((int)N, vin, 0, nullptr, 0.0, z, skip);
  count(1);
  band_apply(bfac[0], z, skip);
  if (B.size == 2) {
    k_vin_rhs<<<gb, 256, 0, stream>>>((int)N, vin, (int)N, z, B.beta * B.beta / B.phi, z + N,
                                       skip);
    count(1);
    band_apply(bfac[1], z + N, skip);
  }
  counters.precond_bytes += 8.0 * N * B.size * 3.0;
}

}  // namespace irkg
