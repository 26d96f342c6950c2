// cgs.cu -- fused classical Gram-Schmidt sweeps (CGS2) + Arnoldi finish.
//
// Replaces the reference's orthogonalisation (src/sparsela.py:222-233):
//     wnorm0 = ||w||; 2x { coef = V^T w ; w -= V coef ; h += coef }; h_{j+1,j} = ||w||
// as three sweeps over the basis instead of four:
//     DOT       c1 = V^T w, ||w||^2
//     UPD_DOT   w1 = w - V c1 (written back), c2 = V^T w1      (V tile read once)
//     UPD_NORM  s_{j+1} = w1 - V c2, ||s_{j+1}||^2; last CTA finishes the column
// Each CTA streams row tiles of all (j+1) basis slots + w into a shared-memory
// ring of up to CGS_MAXST tiles (one mbarrier each) with TMA bulk copies:
// 2-D tensor-map boxes (popcount(j+1) boxes of 2^b slots) or, per the
// IRKG_CGS_1D sweep mask (default: all three sweeps in tiles of >= 256
// rows), one 1-D cp.async.bulk per slot.  The only partial tile (the
// globally last) is loaded with generic zero-padded loads.  The tile is read
// once from HBM for both the update and the dots.  Per-CTA partials are
// folded in a fixed order (deterministic, no fp atomics) by every CTA of the
// NEXT sweep (UPD_DOT folds DOT's, UPD_NORM folds UPD_DOT's); UPD_NORM's are
// folded by its last CTA, which finishes the Hessenberg column.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "engine.h"

namespace irkg {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// plain arrival (no transaction bytes): completes the phase of a ring slot
// whose tile is not TMA-loaded (the zero-padded tail tile), so every slot
// advances exactly one phase per ring round and the parity waits stay in step
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// the same with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void tma_load_1d_hint(void *dst, const void *src, uint32_t bytes,
                                                 uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 2-D tile of the basis: box (rows x slots) at (row c0, slot c1), landing in
// shared memory slot-major, i.e. exactly the stage layout
__device__ __forceinline__ void tma_load_2d(void *dst, const void *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// generic-proxy writes to global memory -> later async-proxy (TMA) reads
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace

// Finish Arnoldi column j (src/sparsela.py:227-256), by one whole CTA.
// The column, the previous rotations and the coefficients are staged into
// shared memory (scr: >= 3 (MAXR + 2) doubles) by all threads at once, thread
// 0 applies the j earlier Givens rotations with the running entry in a
// register (the same operations in the same order as the textbook in-place
// loop, so H is bit-identical), and the finished column goes back to global
// memory in parallel.  A single-thread loop over global memory made the
// finish a chain of dependent L2 round trips that grew with j.
__device__ void arnoldi_finish_block(GWork W, double *scr) {
  GCtrl *c = W.ctrl;
  const int j = c->j;
  const int tid = threadIdx.x, nt = blockDim.x;
  double *hs = scr, *css = scr + (MAXR + 2), *sns = scr + 2 * (MAXR + 2);
  double *h = W.H + (size_t)j * (MAXR + 1);
  // thread 0's scalar inputs are loaded up front, all at once, alongside the
  // column staging (reading them between its stores made each one a
  // dependent L2 round trip on the serial tail of the sweep)
  GCtrl cl;
  double gj = 0.0;
  if (tid == 0) {
    cl = *c;
    gj = W.g[j];
  }
  for (int i = tid; i <= j; i += nt) {
    hs[i] = (0.0 + W.c1[i]) + W.c2[i];
    if (i < j) {
      css[i] = W.cs[i];
      sns[i] = W.sn[i];
    }
  }
  __syncthreads();
  if (tid == 0) {
    const double hj = sqrt(cl.hn2);
    const double wnorm0 = sqrt(cl.wn2);
    hs[j + 1] = hj;
    const bool breakdown = hj <= 1e-14 * fmax(wnorm0, 1e-300);
    if (!breakdown) W.alpha[j + 1] = 1.0 / hj;
    double hi = hs[0];
    for (int i = 0; i < j; ++i) {
      const double hn = hs[i + 1];
      const double tmp = css[i] * hi + sns[i] * hn;
      hi = -sns[i] * hi + css[i] * hn;
      hs[i] = tmp;
    }
    hs[j] = hi;
    const double denom = hypot(hs[j], hs[j + 1]);
    if (denom == 0.0) {  // dead column (src/sparsela.py:239-246)
      c->breakdown = 1;
      c->total_it = cl.total_it + 1;
      W.res[cl.n_res] = W.res[cl.n_res - 1];
      c->n_res = cl.n_res + 1;
      c->k = j;
      c->cycle_done = 1;
    } else {
      const double csj = hs[j] / denom, snj = hs[j + 1] / denom;
      W.cs[j] = csj;
      W.sn[j] = snj;
      hs[j] = denom;
      hs[j + 1] = 0.0;
      const double g1 = -snj * gj;
      W.g[j + 1] = g1;
      W.g[j] = csj * gj;
      const int total_it = cl.total_it + 1;
      c->total_it = total_it;
      const double est = fabs(g1) / cl.bnorm;
      W.res[cl.n_res] = est;
      c->n_res = cl.n_res + 1;
      if (breakdown) c->breakdown = 1;
      if (est <= cl.rtol || breakdown || total_it >= cl.maxit || j + 1 >= cl.m) {
        c->k = j + 1;
        c->cycle_done = 1;
      } else {
        c->j = j + 1;
      }
    }
  }
  __syncthreads();
  // (no fence: the consumers are later kernels -- a launch boundary, or a
  // griddepcontrol.wait, which waits for this grid's completion and flush)
  for (int i = tid; i <= j + 1; i += nt) h[i] = hs[i];
  __syncthreads();
}

constexpr int VM_TR = 4;  // tensor maps for tile rows 32, 64, 128, 256
constexpr int VM_B = 9;   // ... and slot boxes 1, 2, ..., 256
constexpr int CGS_BS = 256;
constexpr int CGS_NW = CGS_BS / 32;
constexpr int CGS_Q = (MAXR + 2 + CGS_NW - 1) / CGS_NW;  // slots per warp (<= 33)
constexpr int CGS_STAGE_MAX = (MAXR + 2) * 32;  // ring/2 upper bound: max doubles per tile
constexpr int CGS_MAXST = 8;                    // max tiles in flight per CTA

enum { CGS_DOT = 0, CGS_UPD_DOT = 1, CGS_UPD_NORM = 2 };

struct TileArgs {
  int n, L, G, ntiles;
  const double *V;
  long long pitch;
  const double *win;
  double *out;
  double *ring;      // NST tiles of (L+1) x TRC doubles
  int nst;
  uint64_t *bars;
  const double *cs;
  double *red;
  const char *maps;  // tensor maps of this tile height (null: 1-D copies)
  int rev;           // walk the row tiles last-to-first (L2 reuse between sweeps)
  int ef_from;       // basis slots >= ef_from are read evict-first (1-D copies)
  int st_mode;       // output store flavour (timing experiments): 0 default, 1 .cs, 2 .wt, 3 L2 evict_last
};

__device__ __forceinline__ void out_store(const TileArgs &A, long long i, double v) {
  IRKG_DCHECK(i >= 0 && i < A.n);
  double *p = A.out + i;
  if (A.st_mode == 1) {
    __stcs(p, v);
  } else if (A.st_mode == 2) {
    __stwt(p, v);
  } else if (A.st_mode == 3) {
    asm volatile("{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
                 " st.global.L2::cache_hint.f64 [%0], %1, pol;\n}\n" ::"l"(p), "d"(v)
                 : "memory");
  } else {
    *p = v;
  }
}

// Tile issue, out of line: one copy of the code for every tile height and
// call site (inlined, the unrolled copy loops made the kernels too large for
// the instruction cache of a short launch).
// TR <= 256: one thread moves the L basis segments with 2-D TMA boxes of 2^b
// slots (popcount(L) copies, one tensor map per box shape) and w with a 1-D
// copy.
// with_w = false: the basis part only (issued before pdl_wait(); the w
// segment follows with issue_w once the predecessor has finished)
__device__ __noinline__ void issue_boxed(double *dst, const char *maps, const double *win, int r0,
                                         int TR, int L, uint64_t *bar, bool with_w) {
  const uint32_t bytes = TR * 8u;
  mbar_expect_tx(bar, bytes * (uint32_t)(L + 1));
  int l0 = 0;
#pragma unroll 1
  for (int b = VM_B - 1; b >= 0; --b) {
    if (L & (1 << b)) {
      tma_load_2d(dst + l0 * TR, maps + b * sizeof(CUtensorMap), r0, l0, bar);
      l0 += 1 << b;
    }
  }
  if (with_w) tma_load_1d(dst + L * TR, win + r0, bytes, bar);
}

// Taller tiles (small j): one 1-D copy per slot, lane 0 of warp w issuing
// slots w, w+NW, ... (cp.async.bulk takes uniform operands: lane-divergent
// issue from one warp compiles to a serial waterfall).  Thread 0's expect_tx
// may land after some copies complete (the tx-count goes transiently
// negative); the phase cannot flip before its arrival.
// Slots at or above ef_from (past the L2-persisting window: re-read only
// after the whole basis has streamed through L2) go out evict-first, so they
// do not displace the lines the next kernels reuse.
__device__ __noinline__ void issue_slots(double *dst, const double *V, long long pitch,
                                         const double *win, int r0, int TR, int L, int warp,
                                         uint64_t *bar, bool with_w, int ef_from) {
  const uint32_t bytes = TR * 8u;
  const uint64_t pol = evict_first_policy();
  IRKG_DCHECK(r0 >= 0 && (long long)r0 + TR <= pitch && (TR & 1) == 0);
#pragma unroll 1
  for (int l = warp; l <= L - (with_w ? 0 : 1); l += CGS_NW) {
    const double *src = (l < L) ? V + (size_t)l * pitch + r0 : win + r0;
    if (l < L && l >= ef_from)
      tma_load_1d_hint(dst + l * TR, src, bytes, bar, pol);
    else
      tma_load_1d(dst + l * TR, src, bytes, bar);
  }
}

// Work on one tile in shared memory, specialised on the tile height TRC so
// the per-slot work is straight-line: a tile is (L+1) x TRC doubles (rows
// [0, L) basis slots, row L the w segment).  Phase A (update modes): w1 = w -
// sum_l s_l cs_l, written to A.out and back into the tile; phase B (dot
// modes): per-lane running dot products in registers.
template <int MODE, int TRC>
__device__ __forceinline__ void tile_compute(const TileArgs &A, double *buf, int r0, int rows,
                                             double (&acc)[CGS_Q], double &nrm) {
  constexpr int K = TRC / 32;                       // rows per lane in phase B
  constexpr int RPP = TRC < CGS_BS ? TRC : CGS_BS;  // rows per pass in phase A
  constexpr int PARTS = CGS_BS / RPP;
  // a tile holds at most CGS_STAGE_MAX doubles, so a tile of TRC rows has at
  // most CGS_STAGE_MAX/TRC slots: unroll only that many slot bodies per warp
  // (short launches at small j run from a cold instruction cache)
  constexpr int QMAX_ = (CGS_STAGE_MAX / TRC + CGS_NW - 1) / CGS_NW;
  constexpr int QMAX = QMAX_ < CGS_Q ? QMAX_ : CGS_Q;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int L = A.L;
  const int nd = (MODE == CGS_DOT) ? L + 1 : L;
  const int nq = (nd + CGS_NW - 1) / CGS_NW;
  double *wt = buf + L * TRC;
  if (MODE != CGS_DOT) {
    // PARTS threads share a row (slots split round-robin), two accumulators
    // break the DFMA chain
    const int pid = tid / RPP, rl = tid % RPP;
#pragma unroll
    for (int rb = 0; rb < TRC; rb += RPP) {
      const int r = rb + rl;
      const double *col = buf + r;
      double s0 = 0.0, s1 = 0.0;
      int l = pid;
      for (; l + PARTS < L; l += 2 * PARTS) {
        s0 += col[l * TRC] * A.cs[l];
        s1 += col[(l + PARTS) * TRC] * A.cs[l + PARTS];
      }
      if (l < L) s0 += col[l * TRC] * A.cs[l];
      double sum = s0 + s1;
      if (PARTS > 1) {
        A.red[tid] = sum;
        __syncthreads();
        if (pid == 0) {
          double tot = 0.0;
#pragma unroll
          for (int p = 0; p < PARTS; ++p) tot += A.red[p * RPP + rl];
          sum = tot;
        }
      }
      if (pid == 0) {
        double v = wt[r] - sum;
        if (r < rows) {
          if (MODE == CGS_UPD_NORM) nrm += v * v;
          out_store(A, r0 + r, v);
        } else {
          v = 0.0;
        }
        if (MODE == CGS_UPD_DOT) wt[r] = v;  // the second-pass dots read w1
      }
      if (PARTS > 1) __syncthreads();
    }
    __syncthreads();
  }
  if (MODE != CGS_UPD_NORM) {
    // warp w owns slots l = w + NW*q; each lane keeps its running partial sum
    // per owned slot in a register across rows and tiles (no per-tile shuffle
    // reductions; folded once after the tile loop).  w rows are cached in
    // registers for short tiles; tall tiles only occur at small j, where
    // re-reading them from shared memory is cheap.
    constexpr int KR = K <= 4 ? K : 1;
    double wr[KR];
#pragma unroll
    for (int k = 0; k < KR; ++k) wr[k] = wt[lane + 32 * k];
#pragma unroll
    for (int q = 0; q < QMAX; ++q) {
      if (q >= nq) break;
      const int l = warp + CGS_NW * q;
      if (l < nd) {
        const double *vl = buf + l * TRC + lane;
        double a = acc[q];
        if constexpr (K <= 4) {
#pragma unroll
          for (int k = 0; k < K; ++k) a += vl[32 * k] * wr[k];
        } else {  // keep the code small: 33 slot bodies x K rows would not fit the i-cache
          double a1 = 0.0;
#pragma unroll 2
          for (int k = 0; k < K; k += 2) {
            a += vl[32 * k] * wt[lane + 32 * k];
            a1 += vl[32 * k + 32] * wt[lane + 32 * k + 32];
          }
          a += a1;
        }
        acc[q] = a;
      }
    }
  }
}

// Row-owner form of the DOT / UPD_DOT tile work for short bases (L <= LMAX,
// tiles of >= CGS_BS rows): each thread owns rows tid, tid + CGS_BS, ...,
// reads each basis entry of its rows from shared memory once, forms w1 in a
// register (UPD_DOT: same association as tile_compute, so w1 is bit-identical)
// and keeps one running dot per slot (acc[l]; DOT: nrm = ||w||^2) across rows
// and tiles.  The slot-owner form above reads w once per slot, syncs the CTA
// between the update and the dots and leaves warps with uneven slot counts.
template <int MODE, int TRC, int LMAX>
__device__ __forceinline__ void tile_compute_ro(const TileArgs &A, const double (&csr)[LMAX],
                                                double *buf, int r0, int rows,
                                                double (&acc)[CGS_Q], double &nrm) {
  constexpr int RPT = TRC / CGS_BS;
  const int L = A.L;
  const double *wt = buf + L * TRC;
#pragma unroll(LMAX <= 8 ? 2 : 1)
  for (int m = 0; m < RPT; ++m) {
    const int r = threadIdx.x + CGS_BS * m;
    double v[LMAX];
#pragma unroll
    for (int l = 0; l < LMAX; ++l) v[l] = (l < L) ? buf[l * TRC + r] : 0.0;
    double w = wt[r];
    if (MODE != CGS_DOT) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int l = 0; l < LMAX; l += 2) {
        if (l < L) {
          if (l + 1 < L) {
            s0 += v[l] * csr[l];
            s1 += v[l + 1] * csr[l + 1];
          } else {
            s0 += v[l] * csr[l];
          }
        }
      }
      w = w - (s0 + s1);
      if (r < rows)
        out_store(A, r0 + r, w);
      else
        w = 0.0;
      if (MODE == CGS_UPD_NORM) nrm += w * w;
    } else {
      nrm += w * w;
    }
    if (MODE != CGS_UPD_NORM) {
#pragma unroll
      for (int l = 0; l < LMAX; ++l)
        if (l < L) acc[l] += v[l] * w;
    }
  }
}

// IRKG_CGS_RO mask (bits 24.. of the trmax word): bit m = row-owner tile work
// in sweep m (DOT, UPD_DOT, UPD_NORM); default 6 (the update sweeps; DOT, which
// has no update to fuse, measured the same either way)
template <int MODE>
__device__ __forceinline__ bool cgs_ro_on(int trmax_word) { return (trmax_word >> (24 + MODE)) & 1; }

template <int TRC>
__device__ __forceinline__ bool tile_full(const TileArgs &A, int t) {
  return (long long)(t + 1) * TRC <= (long long)A.n;
}

template <int TRC>
__device__ __forceinline__ void tile_issue(const TileArgs &A, int t, int s, bool with_w = true) {
  const int tid = threadIdx.x;
  IRKG_DCHECK(s >= 0 && s < A.nst && t >= 0 && (long long)(t + 1) * TRC <= A.n);
  double *dst = A.ring + (size_t)s * (A.L + 1) * TRC;
  if (A.maps) {
    if (tid == 0) issue_boxed(dst, A.maps, A.win, t * TRC, TRC, A.L, &A.bars[s], with_w);
  } else {
    if (tid == 0) mbar_expect_tx(&A.bars[s], TRC * 8u * (uint32_t)(A.L + 1));
    if ((tid & 31) == 0)
      issue_slots(dst, A.V, A.pitch, A.win, t * TRC, TRC, A.L, tid >> 5, &A.bars[s], with_w,
                  A.ef_from);
  }
}

// the w segment of a tile whose basis part went out before pdl_wait()
template <int TRC>
__device__ __forceinline__ void tile_issue_w(const TileArgs &A, int t, int s) {
  if (threadIdx.x == 0) {
    double *dst = A.ring + (size_t)s * (A.L + 1) * TRC;
    tma_load_1d(dst + A.L * TRC, A.win + t * TRC, TRC * 8u, &A.bars[s]);
  }
}

// partial tail tile (only the globally last one): generic loads, zero-padded
template <int TRC>
__device__ __forceinline__ void tile_load_tail(const TileArgs &A, double *buf, int r0, int rows) {
  IRKG_DCHECK(rows > 0 && rows < TRC && (long long)r0 + rows == A.n);
  for (int l = 0; l <= A.L; ++l) {
    const double *src = (l < A.L) ? A.V + (size_t)l * A.pitch + r0 : A.win + r0;
    for (int r = threadIdx.x; r < TRC; r += CGS_BS) buf[l * TRC + r] = (r < rows) ? src[r] : 0.0;
  }
  __syncthreads();
}

// Sum of the G per-CTA partials of one entry, by one warp, in a fixed order
// (identical wherever it runs: the last CTA of a sweep, or every CTA of the
// next sweep).
__device__ __forceinline__ double fold_partials(const double *pl, int G, int lane) {
  double f0 = 0.0, f1 = 0.0, f2 = 0.0, f3 = 0.0;
  constexpr int MAXK = 12;  // G <= 32 * MAXK: all of a lane's loads in flight at once
  if (G <= 32 * MAXK) {
    double v[MAXK];
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      const int c = lane + 32 * k;
      v[k] = c < G ? __ldcg(pl + c) : 0.0;
    }
    // the association of the loop below: blocks of 4 strided values while
    // c + 96 < G, then the tail into f0
    int nb = 0;
#pragma unroll
    for (int b = 0; b < MAXK / 4; ++b)
      if (nb == b && lane + 128 * b + 96 < G) {
        f0 += v[4 * b];
        f1 += v[4 * b + 1];
        f2 += v[4 * b + 2];
        f3 += v[4 * b + 3];
        nb = b + 1;
      }
#pragma unroll
    for (int k = 0; k < MAXK; ++k)
      if (k >= 4 * nb && lane + 32 * k < G) f0 += v[k];
    return wsum((f0 + f1) + (f2 + f3));
  }
  int c = lane;
  for (; c + 96 < G; c += 128) {
    f0 += __ldcg(pl + c);
    f1 += __ldcg(pl + c + 32);
    f2 += __ldcg(pl + c + 64);
    f3 += __ldcg(pl + c + 96);
  }
  for (; c < G; c += 32) f0 += __ldcg(pl + c);
  return wsum((f0 + f1) + (f2 + f3));
}

// One sweep's tile loop (grid-stride over row tiles, NST tiles in flight).
// LMAX > 0: the row-owner tile work (DOT / UPD_DOT with L <= LMAX).
// sync_point(): what the sweep must wait for before it touches w and the
// previous sweep's results -- pdl_wait() in a sweep of its own launch; in the
// fused three-sweep kernel the previous phase's partial stores + a grid barrier
struct PdlSync {
  __device__ __forceinline__ void operator()() const { pdl_wait(); }
};

template <int MODE, int TRC, int LMAX = 0, class SyncF = PdlSync>
__device__ __forceinline__ void cgs_tiles(const TileArgs &A, double (&acc)[CGS_Q], double &nrm,
                                          const GWork &W, const double *cin, const double *pin,
                                          SyncF sync_point = SyncF()) {
  const int G = A.G, ntiles = A.ntiles;
  const int t0 = blockIdx.x;
  const int NST = A.nst;
  // logical tile t -> row tile; consecutive sweeps walk the rows in opposite
  // directions so each starts on the tiles the previous one touched last
  // (still in L2) instead of the ones LRU evicted first
  auto ph = [&](int t) { return A.rev ? ntiles - 1 - t : t; };
  // PDL prologue: the basis slots were written >= 2 launches back, so their
  // part of the first NST tiles goes out while the predecessor drains; w
  // (and the coefficients) only after pdl_wait()
  for (int i = 0; i < NST; ++i)
    if (t0 + i * G < ntiles) {
      if (tile_full<TRC>(A, ph(t0 + i * G)))
        tile_issue<TRC>(A, ph(t0 + i * G), i, false);
      else if (threadIdx.x == 0)
        mbar_arrive(&A.bars[i]);  // the tail tile: generic loads at consumption
    }
  sync_point();
  fence_proxy_async_global();  // w was written through the generic proxy
  for (int i = 0; i < NST; ++i)
    if (t0 + i * G < ntiles && tile_full<TRC>(A, ph(t0 + i * G)))
      tile_issue_w<TRC>(A, ph(t0 + i * G), i);
  if (MODE != CGS_DOT) {
    if (pin) {
      // the previous sweep left only per-CTA partials: every CTA folds them
      // itself (same order everywhere), off the serial last-CTA path; CTA 0
      // publishes the coefficients (and DOT's ||w||^2) for the column finish
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const int nprev = (MODE == CGS_UPD_DOT) ? A.L + 1 : A.L;
      for (int l = warp; l < nprev; l += CGS_NW) {
        const double v = fold_partials(pin + (size_t)l * A.G, A.G, lane);
        if (lane == 0) {
          if (l < A.L) {
            const double c = W.alpha[l] * v;
            const_cast<double *>(A.cs)[l] = W.alpha[l] * c;
            if (blockIdx.x == 0) const_cast<double *>(cin)[l] = c;
          } else if (blockIdx.x == 0) {
            W.ctrl->wn2 = v;
          }
        }
      }
    } else {
      for (int l = threadIdx.x; l < A.L; l += CGS_BS)
        const_cast<double *>(A.cs)[l] = W.alpha[l] * cin[l];
    }
  }
  __syncthreads();
  pdl_trigger();
  constexpr int LR = LMAX > 0 ? LMAX : 1;
  double csr[LR];
  if constexpr (LMAX > 0) {
#pragma unroll
    for (int l = 0; l < LMAX; ++l) csr[l] = (MODE != CGS_DOT && l < A.L) ? A.cs[l] : 0.0;
  }

  int s = 0;
  uint32_t phase = 0;
  for (int t = t0; t < ntiles; t += G) {
    const int r0 = ph(t) * TRC;
    const int rows = min(TRC, A.n - r0);
    double *buf = A.ring + (size_t)s * (A.L + 1) * TRC;
    const bool full = tile_full<TRC>(A, ph(t));
    // every slot completes one phase per ring round (TMA bytes, or the plain
    // arrival issued for the tail tile), so the parity wait is uniform
    while (!mbar_try_wait(&A.bars[s], phase)) {
    }
    if (!full) tile_load_tail<TRC>(A, buf, r0, rows);
    if constexpr (LMAX > 0) {
      tile_compute_ro<MODE, TRC, LR>(A, csr, buf, r0, rows, acc, nrm);
    } else {
      tile_compute<MODE, TRC>(A, buf, r0, rows, acc, nrm);
    }
    // the slot is refilled by TMA below: order this thread's generic-proxy
    // writes to it (the zero-padded tail tile; the slot-owner UPD_DOT's w1)
    // before the async-proxy copy
    if (!full || (LMAX == 0 && MODE == CGS_UPD_DOT)) fence_proxy_async();
    __syncthreads();  // stage s consumed
    {
      const int tn = t + NST * G;
      if (tn < ntiles) {
        if (tile_full<TRC>(A, ph(tn)))
          tile_issue<TRC>(A, ph(tn), s);
        else if (threadIdx.x == 0)
          mbar_arrive(&A.bars[s]);
      }
    }
    if (++s == NST) {
      s = 0;
      phase ^= 1u;
    }
  }
}

// per-CTA partials of one sweep -> part[l * G + cta]
template <int MODE>
__device__ __forceinline__ void cgs_write_partials(int ro, int L, int nd, double (&acc)[CGS_Q],
                                                   double nrm, double *red, double *part, int G) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (ro && MODE != CGS_UPD_NORM) {
    // row-owner: every thread holds a partial of every entry; warp sums into
    // shared memory, then one thread per entry adds the warps in order
#pragma unroll
    for (int l = 0; l < 17; ++l) {
      if (l <= L && l < nd) {
        const double v = wsum(l == L ? nrm : acc[l]);
        if (lane == 0) red[warp * 17 + l] = v;
      }
    }
    __syncthreads();
    if (tid < nd) {
      double tot = 0.0;
      for (int w = 0; w < CGS_NW; ++w) tot += red[w * 17 + tid];
      part[(size_t)tid * G + blockIdx.x] = tot;
    }
  } else if (MODE != CGS_UPD_NORM) {
    const int nq = (nd + CGS_NW - 1) / CGS_NW;
#pragma unroll
    for (int q = 0; q < CGS_Q; ++q) {
      if (q >= nq) break;  // skip the dead slot blocks (cold code at small j)
      const int l = warp + CGS_NW * q;
      if (l < nd) {  // warp-uniform
        const double v = wsum(acc[q]);
        if (lane == 0) part[(size_t)l * G + blockIdx.x] = v;
      }
    }
  } else {
    double v = wsum(nrm);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < CGS_NW; ++w) tot += red[w];
      part[blockIdx.x] = tot;
    }
  }
}

// Tile layout: (L+1) x TR doubles; rows [0, L) are basis slots, row L is w.
template <int MODE>
__global__ void __launch_bounds__(CGS_BS, 2)
    k_cgs(int n, double *__restrict__ V, long long pitch, GWork W, const double *cin,
          const double *win, double *wout, double *part, int G, unsigned *counter,
          int ring_doubles, int use_cond, cudaGraphConditionalHandle cond,
          const char *__restrict__ vmaps, int trmax, const double *pin, int defer, int ef_from) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[CGS_MAXST];
  __shared__ double cs[MAXR + 1];
  __shared__ double red[CGS_BS];
  __shared__ bool is_last;

  GCtrl *ctrl = W.ctrl;
  if (ctrl->cycle_done) {
    // inside the graph WHILE body: make sure the loop terminates
    if (MODE == CGS_UPD_NORM && use_cond > 0 && blockIdx.x == 0 && threadIdx.x == 0)
      cudaGraphSetConditional(cond, 0);
    return;
  }
  const int L = ctrl->j + 1;
  const int trmax_raw = trmax;
  const int cgs_rev_mask = (trmax >> 16) & 0xff;
  trmax &= 0xffff;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double *out = (MODE == CGS_UPD_NORM && !wout) ? V + (size_t)L * pitch : wout;
  // tile rows: largest power of two with (L+1)*TR <= stage, within [32, 1024]
  int TR = trmax;
  while (TR > 32 && 2 * (L + 1) * TR > ring_doubles) TR >>= 1;
  // as many tiles in flight as the ring holds (short tiles at mid j would
  // otherwise leave most of the shared memory idle)
  int nst = ring_doubles / ((L + 1) * TR);
  nst = nst > CGS_MAXST ? CGS_MAXST : nst;
  IRKG_DCHECK(L >= 1 && L <= MAXR + 1 && nst >= 1 && nst * (L + 1) * TR <= ring_doubles);
  const int ntiles = (n + TR - 1) / TR;
  const int nd = (MODE == CGS_DOT) ? L + 1 : L;  // dot entries (DOT: + ||w||^2)
  if (TR <= 256 && vmaps) vmaps += (size_t)(__ffs(TR) - 6) * VM_B * sizeof(CUtensorMap);

  if (tid == 0) {
    for (int i = 0; i < nst; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // row-owner dots for short bases in tall tiles (all of configs[1]'s
  // typical cycle lengths); bucketed so the register arrays stay static
  const int ro = (TR >= CGS_BS && cgs_ro_on<MODE>(trmax_raw))
                     ? (L <= 4 ? 4 : L <= 8 ? 8 : L <= 16 ? 16 : 0)
                     : 0;
  // 1-D per-slot copies instead of tensor-map boxes (IRKG_CGS_1D, bits 28..30:
  // bit m = sweep m; default 7) in tiles of >= 256 rows (DOT: >= 128).
  // Same-box probe at configs[1], DOT j = 12 / 24 / 32: 35.1 / 63.8 / 86.3 ->
  // 30.2 / 55.5 / 73.3 us; the update sweeps lose in 128-row tiles
  // (UPD_DOT j = 32: 91.7 -> 114.8 us), so large j keeps the boxes there.
  const int m1d = (trmax_raw >> 28) & 7;
  const bool one_d = ((m1d >> MODE) & 1) && TR >= (MODE == CGS_DOT ? 128 : 256);
  TileArgs A{n, L, G, ntiles, V, pitch, win, out, sm, nst, bars, cs, red,
             (TR <= 256 && !one_d) ? vmaps : nullptr, (cgs_rev_mask >> MODE) & 1, ef_from & 0xffff,
             MODE == CGS_UPD_NORM ? (ef_from >> 16) : 0};
  double nrm = 0.0;
  double acc[CGS_Q];
#pragma unroll
  for (int q = 0; q < CGS_Q; ++q) acc[q] = 0.0;
  if (ro) {
    switch (TR * 100 + ro) {
      case 25604: cgs_tiles<MODE, 256, 4>(A, acc, nrm, W, cin, pin); break;
      case 25608: cgs_tiles<MODE, 256, 8>(A, acc, nrm, W, cin, pin); break;
      case 25616: cgs_tiles<MODE, 256, 16>(A, acc, nrm, W, cin, pin); break;
      case 51204: cgs_tiles<MODE, 512, 4>(A, acc, nrm, W, cin, pin); break;
      case 51208: cgs_tiles<MODE, 512, 8>(A, acc, nrm, W, cin, pin); break;
      case 51216: cgs_tiles<MODE, 512, 16>(A, acc, nrm, W, cin, pin); break;
      case 102404: cgs_tiles<MODE, 1024, 4>(A, acc, nrm, W, cin, pin); break;
      case 102408: cgs_tiles<MODE, 1024, 8>(A, acc, nrm, W, cin, pin); break;
      default: cgs_tiles<MODE, 1024, 16>(A, acc, nrm, W, cin, pin); break;
    }
  } else switch (TR) {
    case 32: cgs_tiles<MODE, 32>(A, acc, nrm, W, cin, pin); break;
    case 64: cgs_tiles<MODE, 64>(A, acc, nrm, W, cin, pin); break;
    case 128: cgs_tiles<MODE, 128>(A, acc, nrm, W, cin, pin); break;
    case 256: cgs_tiles<MODE, 256>(A, acc, nrm, W, cin, pin); break;
    case 512: cgs_tiles<MODE, 512>(A, acc, nrm, W, cin, pin); break;
    default: cgs_tiles<MODE, 1024>(A, acc, nrm, W, cin, pin); break;
  }

  cgs_write_partials<MODE>(ro, L, nd, acc, nrm, red, part, G);
  if (defer) return;  // the next sweep's CTAs fold these partials themselves
  // last-CTA ticket, the grid-sync pattern: the CTA barrier orders every
  // thread's partial store before thread 0's fence + atomic (fence
  // cumulativity), so one thread fences instead of all 256 -- a membar by
  // every thread waited out each thread's pending output stores
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    is_last = (atomicAdd(counter, 1u) == (unsigned)(G - 1));
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  const int nfold = (MODE == CGS_UPD_NORM) ? 1 : nd;
  for (int l = warp; l < nfold; l += CGS_NW) {
    const double v = fold_partials(part + (size_t)l * G, G, lane);
    if (lane == 0) {
      if (MODE == CGS_DOT) {
        if (l == L && use_cond < 0)
          W.c1[L] = v;  // multi-rank: all-reduced together with c1, then moved
        else if (l == L)
          ctrl->wn2 = v;
        else
          W.c1[l] = W.alpha[l] * v;
      } else if (MODE == CGS_UPD_DOT) {
        W.c2[l] = W.alpha[l] * v;
      } else {
        ctrl->hn2 = v;
      }
    }
  }
  __syncthreads();
  // use_cond < 0: multi-rank -- the column is finished after the all-reduce
  if (MODE == CGS_UPD_NORM && use_cond >= 0) {
    // ctrl->hn2 came from this CTA (the barrier suffices); the drained ring is scratch
    arnoldi_finish_block(W, sm);
    if (tid == 0 && use_cond > 0) cudaGraphSetConditional(cond, ctrl->cycle_done ? 0u : 1u);
  }
  if (tid == 0) *counter = 0u;
}

// ---------------------------------------------------------------------------
// The three sweeps of one orthogonalisation in ONE launch (single rank).  Same
// tiles, same per-CTA partials and folds as the three k_cgs launches (results
// bit-identical), with a grid barrier where a launch boundary was: all G = 2 x
// #SM CTAs are co-resident (two per SM by construction: the launcher checks the
// occupancy).  What it buys at short vectors, where a sweep is ~30 us of which
// ~5 are ramp and tail: the next sweep's first basis tiles are issued BEFORE
// the barrier (they depend on nothing the previous sweep computes), so they
// stream in while the partials are exchanged, and two launch transitions go.
__device__ __forceinline__ void mbar_inval(uint64_t *bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// monotone ticket barrier over all G CTAs (gbar never resets: every launch
// passes the same number of barriers with every CTA, so it is a multiple of G
// at launch boundaries); traps instead of hanging if a CTA never arrives
__device__ __forceinline__ void cgs_grid_barrier(unsigned long long *gbar, int G) {
  __syncthreads();  // every thread's stores ordered before thread 0's fence + ticket
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long old = atomicAdd(gbar, 1ULL);
    const unsigned long long target = (old / (unsigned long long)G + 1ULL) * (unsigned long long)G;
    const long long t0 = clock64();
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(gbar) : "memory");
      if (v < target && clock64() - t0 > (1LL << 32)) __trap();  // ~2 s: a CTA is not resident
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

struct GridSync {
  unsigned long long *gbar;
  int G;
  __device__ __forceinline__ void operator()() const { cgs_grid_barrier(gbar, G); }
};

__device__ __forceinline__ void cgs_ring_reset(uint64_t *bars, int nst) {
  __syncthreads();  // every tile of the finished sweep is consumed
  if (threadIdx.x == 0) {
    for (int i = 0; i < nst; ++i) {
      mbar_inval(&bars[i]);
      mbar_init(&bars[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

struct Cgs3Args {
  TileArgs dot, upd, nrmA;
  double *pdot, *pupd, *pnorm;
};

template <int TRC, int LMAX>
__device__ __forceinline__ void cgs3_run(const Cgs3Args &C, const GWork &W, int L, int G,
                                         unsigned long long *gbar, double *red) {
  double nrm = 0.0;
  double acc[CGS_Q];
#pragma unroll
  for (int q = 0; q < CGS_Q; ++q) acc[q] = 0.0;
  // sweep 1: c1 = V^T w, ||w||^2 (slot-owner dots, as k_cgs<DOT> with the default masks)
  cgs_tiles<CGS_DOT, TRC, 0>(C.dot, acc, nrm, W, nullptr, nullptr);
  cgs_write_partials<CGS_DOT>(0, L, L + 1, acc, nrm, red, C.pdot, G);
  cgs_ring_reset(C.dot.bars, C.dot.nst);
  nrm = 0.0;
#pragma unroll
  for (int q = 0; q < CGS_Q; ++q) acc[q] = 0.0;
  // sweep 2: w1 = w - V c1, c2 = V^T w1
  cgs_tiles<CGS_UPD_DOT, TRC, LMAX>(C.upd, acc, nrm, W, W.c1, C.pdot, GridSync{gbar, G});
  cgs_write_partials<CGS_UPD_DOT>(LMAX, L, L, acc, nrm, red, C.pupd, G);
  cgs_ring_reset(C.dot.bars, C.dot.nst);
  nrm = 0.0;
#pragma unroll
  for (int q = 0; q < CGS_Q; ++q) acc[q] = 0.0;
  // sweep 3: s_{j+1} = w1 - V c2, ||s_{j+1}||^2
  cgs_tiles<CGS_UPD_NORM, TRC, LMAX>(C.nrmA, acc, nrm, W, W.c2, C.pupd, GridSync{gbar, G});
  cgs_write_partials<CGS_UPD_NORM>(LMAX, L, L, acc, nrm, red, C.pnorm, G);
}

__global__ void __launch_bounds__(CGS_BS, 2)
    k_cgs3(int n, double *__restrict__ V, long long pitch, GWork W, double *wbuf, double *part,
           int G, unsigned *counter, unsigned long long *gbar, int ring_doubles, int use_cond,
           cudaGraphConditionalHandle cond, const char *__restrict__ vmaps, int trmax,
           int ef_from) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bars[CGS_MAXST];
  __shared__ double cs[MAXR + 1];
  __shared__ double red[CGS_BS];
  __shared__ bool is_last;

  GCtrl *ctrl = W.ctrl;
  if (ctrl->cycle_done) {  // (uniform over the grid: only this kernel's own finish sets it)
    if (use_cond > 0 && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0);
    return;
  }
  const int L = ctrl->j + 1;
  const int trmax_raw = trmax;
  const int cgs_rev_mask = (trmax >> 16) & 0xff;
  trmax &= 0xffff;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // tile geometry: exactly k_cgs's rule (it depends on L alone)
  int TR = trmax;
  while (TR > 32 && 2 * (L + 1) * TR > ring_doubles) TR >>= 1;
  int nst = ring_doubles / ((L + 1) * TR);
  nst = nst > CGS_MAXST ? CGS_MAXST : nst;
  IRKG_DCHECK(L >= 1 && L <= MAXR + 1 && nst >= 1 && nst * (L + 1) * TR <= ring_doubles);
  const int ntiles = (n + TR - 1) / TR;
  const char *vm = vmaps;
  if (TR <= 256 && vm) vm += (size_t)(__ffs(TR) - 6) * VM_B * sizeof(CUtensorMap);
  if (tid == 0) {
    for (int i = 0; i < nst; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // row-owner update sweeps for short bases in tall tiles (mask 6: the launcher
  // routes every other IRKG_CGS_RO setting to the three-launch path)
  const int ro = TR >= CGS_BS ? (L <= 4 ? 4 : L <= 8 ? 8 : L <= 16 ? 16 : 0) : 0;
  const int m1d = (trmax_raw >> 28) & 7;
  auto args = [&](int mode, double *out) {
    const bool one_d = ((m1d >> mode) & 1) && TR >= (mode == CGS_DOT ? 128 : 256);
    return TileArgs{n, L, G, ntiles, V, pitch, wbuf, out, sm, nst, bars, cs, red,
                    (TR <= 256 && !one_d) ? vm : nullptr, (cgs_rev_mask >> mode) & 1,
                    ef_from & 0xffff, 0};
  };
  Cgs3Args C{args(CGS_DOT, nullptr), args(CGS_UPD_DOT, wbuf),
             args(CGS_UPD_NORM, V + (size_t)L * pitch), part + (size_t)(MAXR + 2) * G,
             part + 2 * (size_t)(MAXR + 2) * G, part};
  switch (TR * 100 + ro) {
    case 25604: cgs3_run<256, 4>(C, W, L, G, gbar, red); break;
    case 25608: cgs3_run<256, 8>(C, W, L, G, gbar, red); break;
    case 25616: cgs3_run<256, 16>(C, W, L, G, gbar, red); break;
    case 51204: cgs3_run<512, 4>(C, W, L, G, gbar, red); break;
    case 51208: cgs3_run<512, 8>(C, W, L, G, gbar, red); break;
    case 51216: cgs3_run<512, 16>(C, W, L, G, gbar, red); break;
    case 102404: cgs3_run<1024, 4>(C, W, L, G, gbar, red); break;
    case 102408: cgs3_run<1024, 8>(C, W, L, G, gbar, red); break;
    case 102416: cgs3_run<1024, 16>(C, W, L, G, gbar, red); break;
    case 3200: cgs3_run<32, 0>(C, W, L, G, gbar, red); break;
    case 6400: cgs3_run<64, 0>(C, W, L, G, gbar, red); break;
    case 12800: cgs3_run<128, 0>(C, W, L, G, gbar, red); break;
    case 25600: cgs3_run<256, 0>(C, W, L, G, gbar, red); break;
    case 51200: cgs3_run<512, 0>(C, W, L, G, gbar, red); break;
    default: cgs3_run<1024, 0>(C, W, L, G, gbar, red); break;
  }
  // last-CTA ticket: fold ||s_{j+1}||^2 and finish the Hessenberg column (as k_cgs<UPD_NORM>)
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    is_last = (atomicAdd(counter, 1u) == (unsigned)(G - 1));
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (warp == 0) {
    const double v = fold_partials(part, G, lane);
    if (lane == 0) ctrl->hn2 = v;
  }
  __syncthreads();
  arnoldi_finish_block(W, sm);
  if (tid == 0 && use_cond > 0) cudaGraphSetConditional(cond, ctrl->cycle_done ? 0u : 1u);
  if (tid == 0) *counter = 0u;
}

// Tensor maps over the basis V viewed as a 2-D array (rows: vpitch, slots:
// vcap+1, slot stride vpitch doubles), one per (tile rows, slot box) shape.
void Engine::build_vmaps() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      dalloc_raw(&vmaps, 0);  // no tensor maps: the sweeps use 1-D copies only
      return;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  std::vector<CUtensorMap> maps(VM_TR * VM_B);
  const cuuint64_t dims[2] = {(cuuint64_t)vpitch, (cuuint64_t)(vcap + 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)vpitch * sizeof(double)};
  const cuuint32_t estr[2] = {1, 1};
  for (int a = 0; a < VM_TR; ++a)
    for (int b = 0; b < VM_B; ++b) {
      // shapes larger than a stage are never used (and boxes over 128 KB are
      // rejected by the encoder): leave those entries zero
      if ((1u << b) > (cuuint32_t)(vcap + 1) || (32u << a) * (1u << b) * 8u > (128u << 10)) {
        memset(&maps[a * VM_B + b], 0, sizeof(CUtensorMap));
        continue;
      }
      const cuuint32_t box[2] = {32u << a, 1u << b};
      CUresult r = encode(&maps[a * VM_B + b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, V, dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS)
        throw SolveError(IRKG_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) +
                                            ") box " + std::to_string(box[0]) + "x" +
                                            std::to_string(box[1]) + " dims " +
                                            std::to_string(dims[0]) + "x" + std::to_string(dims[1]));
    }
  dalloc_raw(&vmaps, maps.size() * sizeof(CUtensorMap));
  check(cudaMemcpy(vmaps, maps.data(), maps.size() * sizeof(CUtensorMap),
                   cudaMemcpyHostToDevice),
        "tensor maps");
}

static const char *cgs_maps(const void *vmaps) {
  static int nobox = -1;
  if (nobox < 0) nobox = getenv("IRKG_CGS_NOBOX") ? 1 : 0;
  return nobox ? nullptr : (const char *)vmaps;
}

static int cgs_trmax() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("IRKG_CGS_TRMAX");
    v = e ? atoi(e) : 1024;
    // bit m: sweep m (DOT, UPD_DOT, UPD_NORM) walks the row tiles backwards
    const char *r = getenv("IRKG_CGS_REV");
    v |= (r ? atoi(r) : 2) << 16;
    const char *ro = getenv("IRKG_CGS_RO");
    v |= ((ro ? atoi(ro) : 6) & 7) << 24;
    const char *o1 = getenv("IRKG_CGS_1D");
    v |= ((o1 ? atoi(o1) : 7) & 7) << 28;
  }
  return v;
}

// First basis slot read evict-first: the slots past the L2-persisting window
// (all of them when no window applies); IRKG_CGS_EF=0: none.
int Engine::cgs_ef_from() const {
  static int on = -1;
  if (on < 0) on = getenv("IRKG_CGS_EF") ? (atoi(getenv("IRKG_CGS_EF")) != 0) : 1;
  if (!on) return 1 << 30;
  return (int)(l2win.num_bytes / ((size_t)vpitch * sizeof(double)));
}

// Shared-memory ring per CTA, in doubles: 2 x 52 KB (2 CTAs per SM) unless
// the restart length needs two 32-row tiles of more slots.
int Engine::cgs_stage_doubles() const {
  static_assert(6656 <= CGS_STAGE_MAX, "ring floor above the unroll bound");
  int st = (vcap + 2) * 32;  // <= CGS_STAGE_MAX (vcap <= MAXR)
  return 2 * (st < 6656 ? 6656 : st);
}

// The fused three-sweep kernel needs every CTA resident (grid barriers): two
// CTAs per SM for G = 2 x #SM, checked once with the occupancy calculator;
// IRKG_CGS_FUSED=0, a non-default IRKG_CGS_RO mask, the phase probe's partial
// orthogonalisations (1 or 2 sweeps) and the multi-rank path use the three launches.
bool Engine::cgs_fused_ok(size_t smem, int trm, long long n) {
  if (!cgs_fused || ((trm >> 24) & 7) != 6) return false;
  if (cgs_fused_maxn > 0 && n > cgs_fused_maxn) return false;  // short vectors only
  if (cgs_fused_occ < 0 || cgs_fused_smem != smem) {
    check(cudaFuncSetAttribute(k_cgs3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
          "smem attr");
    max_carveout((const void *)k_cgs3);
    int nb = 0;
    check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_cgs3, CGS_BS, smem), "occupancy");
    cgs_fused_occ = nb;
    cgs_fused_smem = smem;
    if (!gbar) {
      dalloc_raw((void **)&gbar, sizeof(unsigned long long));
      check(cudaMemset(gbar, 0, sizeof(unsigned long long)), "memset");
    }
  }
  return (long long)cgs_fused_occ * sms >= G;
}

// One Arnoldi orthogonalisation: 3 fused sweeps; the last also finishes the
// Hessenberg column (Givens, estimate, exit test) in its final CTA.
void Engine::cgs(long long n, int nsweeps) {
  const int stage = cgs_stage_doubles();
  const size_t smem = (size_t)stage * sizeof(double);
  if (cgs_smem_set < smem) {
    check(cudaFuncSetAttribute(k_cgs<CGS_DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem), "smem attr");
    check(cudaFuncSetAttribute(k_cgs<CGS_UPD_DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem), "smem attr");
    check(cudaFuncSetAttribute(k_cgs<CGS_UPD_NORM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem), "smem attr");
    cgs_smem_set = smem;
  }
  const int uc = cond_active ? 1 : 0;
  const char *maps = cgs_maps(vmaps);
  const int ef = cgs_ef_from();
  const int trm = cgs_trmax();
  const double *cnull = nullptr;
  double *dnull = nullptr;
  if (nsweeps == 3 && cgs_fused_ok(smem, trm, n)) {
    // one launch for the three sweeps (grid barriers in between)
    launch_pdl_l2(true, k_cgs3, dim3(G), dim3(CGS_BS), smem, (int)n, V, vpitch, W, wbuf, part, G,
                  counter, gbar, stage, uc, cond_handle, maps, trm, ef);
    count(1);
    return;
  }
  // DOT and UPD_DOT leave per-CTA partials in their own regions of `part`;
  // the next sweep folds them in every CTA (no last-CTA fold between sweeps)
  double *pdot = part + (size_t)(MAXR + 2) * G, *pupd = part + 2 * (size_t)(MAXR + 2) * G;
  launch_pdl_l2(true, k_cgs<CGS_DOT>, dim3(G), dim3(CGS_BS), smem, (int)n, V, vpitch, W, cnull,
             (const double *)wbuf, dnull, pdot, G, counter, stage, 0, cond_handle, maps, trm,
             cnull, 1, ef);
  if (nsweeps < 2) {  // (phase probe)
    count(1);
    return;
  }
  launch_pdl_l2(true, k_cgs<CGS_UPD_DOT>, dim3(G), dim3(CGS_BS), smem, (int)n, V, vpitch, W,
             (const double *)W.c1, (const double *)wbuf, wbuf, pupd, G, counter, stage, 0,
             cond_handle, maps, trm, (const double *)pdot, 1, ef);
  if (nsweeps < 3) {
    count(2);
    return;
  }
  // (IRKG_CGS_EXP bit 0, timing experiments only -- wrong results: UPD_NORM
  // without its last-CTA finish)
  static const int exp_env = getenv("IRKG_CGS_EXP") ? atoi(getenv("IRKG_CGS_EXP")) : 0;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &cap);
  const int exp_bits = (probing && cap == cudaStreamCaptureStatusNone) ? exp_env : 0;
  launch_pdl_l2(true, k_cgs<CGS_UPD_NORM>, dim3(G), dim3(CGS_BS), smem, (int)n, V, vpitch, W,
             (const double *)W.c2, (const double *)wbuf, (exp_bits & 2) ? wbuf : dnull, part, G,
             counter, stage, uc, cond_handle, maps, trm, (const double *)pupd, exp_bits & 1,
             ef | (((exp_bits >> 2) & 3) << 16));
  count(3);
}

// Multi-rank CGS2: the same sweeps over the local slab with the partial
// dot products summed across ranks between them (fixed-length all-reduces,
// so the sequence is graph-capturable with the Arnoldi index on the device:
// c1 travels together with ||w||^2 in c1[L]); the Hessenberg column is then
// finished from the global sums by k_arnoldi_finish_slab.
__global__ void k_arnoldi_finish_slab(GWork W, int use_cond, cudaGraphConditionalHandle cond) {
  __shared__ double scr[3 * (MAXR + 2)];
  GCtrl *c = W.ctrl;
  const bool live = !c->cycle_done;  // block-uniform
  __syncthreads();
  if (live) {
    if (threadIdx.x == 0) c->wn2 = W.c1[c->j + 1];
    __syncthreads();
    arnoldi_finish_block(W, scr);
  }
  if (threadIdx.x == 0 && use_cond > 0) cudaGraphSetConditional(cond, c->cycle_done ? 0u : 1u);
}

void Engine::cgs_slab(long long n) {
  const int stage = cgs_stage_doubles();
  const size_t smem = (size_t)stage * sizeof(double);
  if (cgs_smem_set < smem) {
    check(cudaFuncSetAttribute(k_cgs<CGS_DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem), "smem attr");
    check(cudaFuncSetAttribute(k_cgs<CGS_UPD_DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem), "smem attr");
    check(cudaFuncSetAttribute(k_cgs<CGS_UPD_NORM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem), "smem attr");
    cgs_smem_set = smem;
  }
  const int cnt = vcap + 1;  // >= j + 2 for every j of the cycle
  const char *maps = cgs_maps(vmaps);
  const int ef = cgs_ef_from();
  const int trm = cgs_trmax();
  const double *cnull = nullptr;
  double *dnull = nullptr;
  launch_pdl_l2(true, k_cgs<CGS_DOT>, dim3(G), dim3(CGS_BS), smem, (int)n, V, vpitch, W, cnull,
             (const double *)wbuf, dnull, part, G, counter, stage, -1, cond_handle, maps, trm,
             cnull, 0, ef);
  allreduce(W.c1, cnt);
  launch_pdl_l2(true, k_cgs<CGS_UPD_DOT>, dim3(G), dim3(CGS_BS), smem, (int)n, V, vpitch, W,
             (const double *)W.c1, (const double *)wbuf, wbuf, part, G, counter, stage, -1,
             cond_handle, maps, trm, cnull, 0, ef);
  allreduce(W.c2, cnt);
  launch_pdl_l2(true, k_cgs<CGS_UPD_NORM>, dim3(G), dim3(CGS_BS), smem, (int)n, V, vpitch, W,
             (const double *)W.c2, (const double *)wbuf, dnull, part, G, counter, stage, -1,
             cond_handle, maps, trm, cnull, 0, ef);
  allreduce(&ctrl_dev->hn2, 1);
  k_arnoldi_finish_slab<<<1, 128, 0, stream>>>(W, cond_active ? 1 : 0, cond_handle);
  count(4);
}

}  // namespace irkg
