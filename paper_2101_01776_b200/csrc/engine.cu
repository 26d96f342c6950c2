// engine.cu -- solver drivers and the C ABI (include/irkg.h).
//
// The drivers restate the reference control flow exactly:
//   gmres                src/sparsela.py:176-280
//   transformed_solve    src/irk_core.py:225-338
//   newton               src/nonlinear.py:186-236
//   step                 src/nonlinear.py:299-314
// All vector work is on the device; the host reads back only scalars
// (norms, the GMRES control block) to steer the loops.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "engine.h"

namespace irkg {

static thread_local std::string g_last_error;

template <class T>
static void dalloc(T **p, size_t count) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  if (count == 0) return;
  check(cudaMalloc((void **)p, count * sizeof(T)), "cudaMalloc");
}

Engine::Engine(const irkg_problem &p, int dev, cudaStream_t st, int rank_, int nranks_,
               Comm *comm_, bool force_slab)
    : prob(p), device(dev), stream(st), comm(comm_), rank(rank_), nranks(nranks_),
      slab_forced(force_slab) {
  check(cudaSetDevice(dev), "cudaSetDevice");
  cudaDeviceProp prop;
  check(cudaGetDeviceProperties(&prop, dev), "props");
  sms = prop.multiProcessorCount;
  G = 2 * sms;
  l2_persist_max = prop.persistingL2CacheMaxSize > 0 ? (size_t)prop.persistingL2CacheMaxSize : 0;
  l2_window_max = prop.accessPolicyMaxWindowSize > 0 ? (size_t)prop.accessPolicyMaxWindowSize : 0;
  int ext[3] = {p.nx, p.ny, p.nz};
  ndim = (p.nz > 1) ? 3 : (p.ny > 1 ? 2 : 1);
  // slab partition of the slowest axis: rank r owns planes [p0, p0 + nl)
  gplanes = ndim == 3 ? p.nz : p.ny;
  {
    const int base = gplanes / nranks, rem = gplanes % nranks;
    const int nl = base + (rank < rem ? 1 : 0);
    p0 = rank * base + (rank < rem ? rank : rem);
    grid.nx = p.nx;
    grid.ny = ndim == 3 ? p.ny : nl;
    grid.nz = ndim == 3 ? nl : p.nz;
  }
  grid.slab = slab() ? 1 : 0;
  grid.pin = p0 == 0 ? 1 : 0;
  grid.nxy = grid.nx * grid.ny;
  grid.n = grid.nx * grid.ny * grid.nz;
  double lapdiag = 0.0;
  for (int a = 0; a < 3; ++a) {
    const double len = (a == 1 && p.length_y > 0.0) ? p.length_y
                       : (a == 2 && p.length_z > 0.0) ? p.length_z : p.length;
    double h = len / ext[a];
    if (ext[a] > 1) {
      grid.ih2[a] = 1.0 / (h * h);
      grid.i2h[a] = 1.0 / (2.0 * h);
      lapdiag += -2.0 * grid.ih2[a];
    } else {
      grid.ih2[a] = 0.0;
      grid.i2h[a] = 0.0;
    }
  }
  grid.lapdiag = lapdiag;
  kp.nu = p.nu;
  kp.c = p.c;
  kp.lam = p.lam;
  kp.mu = p.mu;
  N = grid.n;
  dalloc(&part, 3 * (size_t)(MAXR + 2) * G);  // 3 regions: CGS sweeps fold across launches
  dalloc(&counter, 1);
  check(cudaMemsetAsync(counter, 0, sizeof(unsigned), stream));
  dalloc(&scal_dev, 16);
  dalloc(&ctrl_dev, 1);
  check(cudaMemsetAsync(ctrl_dev, 0, sizeof(GCtrl), stream));
  W.ctrl = ctrl_dev;
  dalloc(&W.H, (size_t)(MAXR + 1) * MAXR);
  dalloc(&W.cs, MAXR);
  dalloc(&W.sn, MAXR);
  dalloc(&W.g, MAXR + 1);
  dalloc(&W.alpha, MAXR + 1);
  dalloc(&W.y, MAXR);
  dalloc(&W.c1, MAXR + 1);
  dalloc(&W.c2, MAXR + 1);
  check(cudaMallocHost((void **)&ctrl_host, sizeof(GCtrl)), "cudaMallocHost");
  dalloc(&wbuf, 2 * N);
  dalloc(&zbuf, 2 * N);
  dalloc(&ubuf, 2 * N);
  dalloc(&tmp_x, N);
  dalloc(&tmp_t, N);
  dalloc(&RHS, 2 * N);
  dae = (p.kind == KIND_ARAKAWA);
  dalloc(&ufield, Nst());
  dae_init();
  check(cudaEventCreate(&ev0), "event");
  check(cudaEventCreate(&ev1), "event");
  check(cudaEventCreate(&evp[0]), "event");
  check(cudaEventCreate(&evp[1]), "event");
  for (auto &e : evg) check(cudaEventCreate(&e), "event");
  for (auto &e : evh) check(cudaEventCreate(&e), "event");
  if (const char *e = getenv("IRKG_GRAPH_TIMING")) graph_timing = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_GRAPHS")) use_graphs = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_L2_MB")) l2_budget = atoi(e) > 0 ? ((size_t)atoi(e) << 20) : 0;
  if (const char *e = getenv("IRKG_FUSED_JACOBI")) fused_jacobi = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_FUSED_JACOBI3D")) fused_jacobi3d = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_FUSED_ARA")) fused_ara = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_ARA_WARP")) ara_warp_form = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_JSPAN")) jspan_override = atoi(e);
  if (const char *e = getenv("IRKG_PAIR_JACOBI")) pair_jacobi = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_JACOBI_SPLIT")) jacobi_split = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_PDL")) use_pdl = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_CARVEOUT")) use_carveout = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_SLAB_BATCH")) slab_batch = atoi(e) > 0 ? atoi(e) : 1;
  if (const char *e = getenv("IRKG_GRAPH_UNROLL")) graph_unroll = atoi(e) > 0 ? atoi(e) : 1;
  if (const char *e = getenv("IRKG_JWPS")) jwarps_per_sm = atoi(e) > 0 ? atoi(e) : 12;
  if (const char *e = getenv("IRKG_STRIP_OP")) strip_op = (atoi(e) != 0);
  // auto: on across real ranks (an inter-GPU exchange costs more than the
  // ~4 us a split adds: two launches + a fork/join); off on a 1-rank ring,
  // where the self-exchange is a local copy with nothing to hide
  // (profiles/r2_slab_probe_overlap.txt: 1.41x -> 1.73x of the plain path)
  halo_overlap = nranks > 1;
  if (const char *e = getenv("IRKG_HALO_OVERLAP")) halo_overlap = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_EXT_HALO")) ext_halo = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_CGS_FUSED")) cgs_fused = (atoi(e) != 0);
  if (const char *e = getenv("IRKG_CGS_FUSED_MAXN")) cgs_fused_maxn = atoll(e);
  if (const char *e = getenv("IRKG_BOP_WPS")) bop_wps = atoi(e) > 0 ? atoi(e) : 8;
  for (int i = 0; i < MAXS; ++i)
    for (int j = 0; j < MAXS; ++j) od_slot[i][j] = -1;
}

Engine::~Engine() {
  cudaStreamSynchronize(stream);
  void *bufs[] = {gbar, part, counter, scal_dev, ctrl_dev, W.H, W.cs, W.sn, W.g, W.alpha, W.y,
                  W.c1, W.c2, W.res, V, wbuf, zbuf, ubuf, tmp_x, tmp_t, U, F, Gs, Y, DK,
                  Kst, RHS, ufield, opA, vmaps, zero_n, rc.Z};
  for (void *b : bufs)
    if (b) cudaFree(b);
  if (ctrl_host) cudaFreeHost(ctrl_host);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  for (auto e : evg)
    if (e) cudaEventDestroy(e);
  for (auto e : evh)
    if (e) cudaEventDestroy(e);
  drop_graphs();
  if (cap_stream) cudaStreamDestroy(cap_stream);
  if (comm_stream) cudaStreamDestroy(comm_stream);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  dae_fini();
  free_ghosts();
  delete comm;
  release_l2_limit();
}

void Engine::ensure_stage_buffers() {
  if (U) return;
  const size_t ns = (size_t)s * Nst();
  dalloc(&U, ns);
  dalloc(&F, ns);
  dalloc(&Gs, ns);
  dalloc(&Y, ns);
  dalloc(&DK, ns);
  dalloc(&Kst, ns);
}

void Engine::dalloc_raw(void **p, size_t bytes) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  if (bytes) check(cudaMalloc(p, bytes), "cudaMalloc");
}

void Engine::ensure_basis(int restart) {
  if (restart > MAXR) throw SolveError(IRKG_ERR_CONFIG, "restart exceeds MAXR=256");
  if (V && restart <= vcap) return;
  vpitch = ((2 * N + 31) / 32) * 32;
  drop_graphs();  // graphs bake the basis pointer in
  dalloc(&V, (size_t)(restart + 1) * vpitch);
  vcap = restart;
  build_vmaps();
  set_l2_window();
}

// Every CGS sweep of an Arnoldi step re-reads slots 0..j, so the lowest slots
// are the hottest lines of the solve; a persisting access-policy window over
// them (on the CGS launches only) keeps them out of the streaming LRU churn
// once the basis outgrows L2.
//
// cudaLimitPersistingL2CacheSize is device-wide: the engines of a process
// share it through a per-device refcount; the first one records the limit it
// found, later ones only raise it, and the last one to go resets the
// persisting lines (cudaCtxResetPersistingL2Cache) and restores the limit, so
// nothing is left set aside for torch or other libraries on the GPU.
namespace {
constexpr int kMaxDev = 64;
int g_l2_users[kMaxDev] = {};
size_t g_l2_prev[kMaxDev] = {};
size_t g_l2_set[kMaxDev] = {};
}  // namespace

void Engine::release_l2_limit() {
  if (!l2_holder) return;
  l2_holder = false;
  if (device < 0 || device >= kMaxDev) return;
  if (--g_l2_users[device] == 0) {
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, g_l2_prev[device]);
    g_l2_set[device] = 0;
    cudaGetLastError();
  }
}

void Engine::set_l2_window() {
  l2win = cudaAccessPolicyWindow{};
  if (l2_budget == 0 || l2_persist_max == 0 || l2_window_max == 0 || !V) return;
  // only when whole low slots fit (slots larger than half the budget would
  // pin a fraction of slot 0 and just shrink the L2 left for the stencils)
  if (2 * (size_t)vpitch * sizeof(double) > l2_budget) return;
  size_t bytes = (size_t)(vcap + 1) * (size_t)vpitch * sizeof(double);
  bytes = std::min(std::min(bytes, l2_budget), l2_window_max);
  const size_t persist = std::min(bytes, l2_persist_max);
  if (device < 0 || device >= kMaxDev) return;
  if (!l2_holder) {
    if (g_l2_users[device]++ == 0) {
      if (cudaDeviceGetLimit(&g_l2_prev[device], cudaLimitPersistingL2CacheSize) != cudaSuccess) {
        cudaGetLastError();
        g_l2_prev[device] = 0;
      }
      g_l2_set[device] = 0;
    }
    l2_holder = true;
  }
  if (persist > g_l2_set[device]) {
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist) != cudaSuccess) {
      cudaGetLastError();
      release_l2_limit();
      return;
    }
    g_l2_set[device] = persist;
  }
  l2win.base_ptr = V;
  l2win.num_bytes = bytes;
  l2win.hitRatio = (float)std::min(1.0, (double)persist / (double)bytes);
  l2win.hitProp = cudaAccessPropertyPersisting;
  l2win.missProp = cudaAccessPropertyStreaming;
}

void Engine::set_tableau(const irkg_tableau &t) {
  if (t.s < 1 || t.s > MAXS) throw SolveError(IRKG_ERR_CONFIG, "stage count out of range");
  if (U && t.s != s) {
    void *bufs[] = {U, F, Gs, Y, DK, Kst};
    for (void *b : bufs) cudaFree(b);
    U = F = Gs = Y = DK = Kst = nullptr;
  }
  tab = t;
  s = t.s;
  have_tab = true;
  ensure_stage_buffers();
}

void Engine::set_solver(const irkg_solver &c) {
  if (c.variant < 0 || c.variant > 3) throw SolveError(IRKG_ERR_CONFIG, "variant must be 0..3");
  if (!(c.newton_rtol > 0.0 && c.newton_rtol < 1.0) || !(c.krylov_rtol > 0.0 && c.krylov_rtol < 1.0))
    throw SolveError(IRKG_ERR_CONFIG, "tolerance outside (0, 1)");
  if (c.inner < IRKG_INNER_MG)
    throw SolveError(IRKG_ERR_VALUE, "inner must be 'exact', 'mg' or a positive int");
  if (c.newton_maxit > IRKG_MAX_NEWTON) throw SolveError(IRKG_ERR_CONFIG, "newton_maxit too large");
  cfg = c;
  have_cfg = true;
  ensure_basis(c.restart);
  ensure_res(c.krylov_maxit);
}

void Engine::ensure_res(int maxit) {
  if (W.res && rescap >= maxit + 4) return;
  dalloc(&W.res, (size_t)maxit + 4);
  rescap = maxit + 4;
}

// scal_dev[0] -> host through the pinned control-block mirror (a pageable
// destination would make the runtime stage the copy)
double Engine::read_scalar() {
  gap_mark();
  check(cudaMemcpyAsync(&ctrl_host->scalar, &scal_dev[0], sizeof(double), cudaMemcpyDeviceToHost,
                        stream));
  check(cudaStreamSynchronize(stream), "sync");
  return ctrl_host->scalar;
}

void Engine::gap_mark() {
  if (!graph_timing) return;
  check(cudaEventRecord(evh[0], stream));
  gap_armed = true;
}

void Engine::gap_close(double &acc) {
  if (!graph_timing || !gap_armed) return;
  check(cudaEventRecord(evh[1], stream));
  check(cudaEventSynchronize(evh[1]), "sync");
  float ms = 0.f;
  check(cudaEventElapsedTime(&ms, evh[0], evh[1]), "elapsed");
  acc += ms;
  gap_armed = false;
}

void Engine::read_ctrl() {
  gap_mark();
  check(cudaMemcpyAsync(ctrl_host, ctrl_dev, sizeof(GCtrl), cudaMemcpyDeviceToHost, stream));
  check(cudaStreamSynchronize(stream), "sync");
}

// Boundary planes [0, H) and [nl-H, nl) of both halves of basis slot j
// (j read on the device) -> halo_pack, laid out [half][lo | hi][H planes].
__global__ void k_pack_slot_halo(const double *__restrict__ V, long long pitch, const GCtrl *ctrl,
                                 long long N, int nl, long long P, int H, int halves,
                                 double *__restrict__ out) {
  const double *s = V + (size_t)ctrl->j * pitch;
  const long long HP = (long long)H * P;
  const long long total = (long long)halves * 2 * HP;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long h = i / (2 * HP), r = i % (2 * HP);
    const long long q = r % HP;
    out[i] = s[h * N + (r < HP ? q : (long long)(nl - H) * P + q)];
  }
}

// Multi-rank Arnoldi step with the slot index on the device: pack + one
// NCCL round for the v_j halos, the two inner solves (z1's halo doubles as
// the block operator's), z2's halo, the block operator, CGS2 with
// fixed-length all-reduces and the column finish.  Only device work and
// NCCL calls: captured into the cycle graph like the single-rank step.
void Engine::arnoldi_iteration_slab(const BlockSpec &B, long long n, int j_host) {
  if (prob.kind == KIND_ARAKAWA) {
    // the DAE's 9-point kernels take the slot as a fixed pointer (host loop)
    if (j_host < 0) throw SolveError(IRKG_ERR_CONFIG, "internal: DAE slab step needs j");
    VecIn vj{V + (size_t)j_host * vpitch, 0, nullptr, nullptr};
    vj.scale_ptr = W.alpha + j_host;
    precond(B, &vj, zbuf, nullptr);
    block_op(B, zbuf, wbuf, nullptr, nullptr, nullptr);
    if (timing) check(cudaEventRecord(ev0, stream));
    cgs_slab(n);
    if (timing) check(cudaEventRecord(ev1, stream));
    return;
  }
  const bool ext = ext_halo_ok() && B.inner == cfg.inner;
  const int K1 = jhalo();              // stencil reach of one chain
  const int H = ext ? inhalo() : K1;   // depth of the v_j halo
  const long long P = plane_size();
  const int nl = local_planes();
  const int halves = B.size;
  if (!halo_pack) dalloc_raw((void **)&halo_pack, sizeof(double) * 4 * GH * (size_t)P);
  const long long tot = (long long)halves * 2 * H * P;
  int gb = (int)((tot + 255) / 256);
  gb = gb > sms * 4 ? sms * 4 : (gb < 1 ? 1 : gb);
  k_pack_slot_halo<<<gb, 256, 0, stream>>>(V, vpitch, ctrl_dev, N, nl, P, H, halves, halo_pack);
  count(1);
  Comm::Xfer xf[2];
  VecIn vslot{V, vpitch, ctrl_dev, W.alpha};
  for (int h = 0; h < halves; ++h) {
    Ghost &g = role(R_VIN0 + h);
    g.field = nullptr;  // indexed input: consumers get the planes through vslot.lo/hi
    xf[h] = Comm::Xfer{halo_pack + (size_t)h * 2 * H * P, halo_pack + ((size_t)h * 2 + 1) * H * P,
                       g.lo + (size_t)(GH - H) * P, g.hi, (long long)H * P};
    vslot.lo[h] = g.lo;
    vslot.hi[h] = g.hi;
  }
  counters.halo_exchanges += halves;
  const bool ovl = overlap_ok();
  cudaStream_t main = stream;
  auto on_comm = [&](auto &&f) {  // exchange() / halo_batch enqueue on `stream`
    stream = comm_stream;
    f();
    stream = main;
  };
  // every halo goes out on comm_stream while the bands that read no ghost
  // plane run; the edge bands follow the join (one split per stencil)
  auto overlapped = [&](auto &&send, auto &&compute) {
    fork_comm();
    send();
    band_sel = 1;
    compute();
    join_comm();
    band_sel = 2;
    compute();
    band_sel = 0;
  };
  if (ext) {
    // communication-avoiding step: one halo round (v_j, depth 2(K-1)+1); the
    // chains compute the ghost rows of z1 (K rows: chain 2's reach + the
    // operator's) and z2 (1 row) themselves, so neither needs an exchange
    auto chain1 = [&] {
      chain_ext = B.size == 2 ? B.inner : 1;  // chain 2's reach K-1, plus the operator's row
      chain_out_role = R_Z0;
      jacobi_chain(B.l1, B.eta, B.dt, B.inner, &vslot, 0, nullptr, 0.0, zbuf, ctrl_dev);
      chain_ext = 0;
    };
    if (ovl)
      overlapped([&] { on_comm([&] { comm->halo_batch(halves, xf, stream); }); }, chain1);
    else {
      comm->halo_batch(halves, xf, stream);
      chain1();
    }
    if (B.size == 2) {
      chain_ext = 1;
      chain_out_role = R_Z1;
      jacobi_chain(B.l2, B.gamma, B.dt, B.inner, &vslot, (int)N, zbuf, B.beta * B.beta / B.phi,
                   zbuf + N, ctrl_dev);
      chain_ext = 0;
    }
    counters.op_bytes += 8.0 * N * B.size * 3.0;
    block_op_s(B, zbuf, wbuf, nullptr, nullptr, ctrl_dev);
  } else if (!ovl) {
    comm->halo_batch(halves, xf, stream);
    jacobi_chain(B.l1, B.eta, B.dt, B.inner, &vslot, 0, nullptr, 0.0, zbuf, ctrl_dev);
    if (B.size == 2) {
      exchange(R_Z0, zbuf, H);  // z1 feeds the second row's rhs (and the operator below)
      jacobi_chain(B.l2, B.gamma, B.dt, B.inner, &vslot, (int)N, zbuf, B.beta * B.beta / B.phi,
                   zbuf + N, ctrl_dev);
      exchange(R_X1, zbuf + N, 1);
    } else {
      exchange(R_X0, zbuf, 1);
    }
    counters.op_bytes += 8.0 * N * B.size * 3.0;
    block_op_s(B, zbuf, wbuf, nullptr, nullptr, ctrl_dev);
  } else {
    overlapped([&] { on_comm([&] { comm->halo_batch(halves, xf, stream); }); },
               [&] { jacobi_chain(B.l1, B.eta, B.dt, B.inner, &vslot, 0, nullptr, 0.0, zbuf,
                                  ctrl_dev); });
    if (B.size == 2) {
      overlapped([&] { on_comm([&] { exchange(R_Z0, zbuf, H); }); },
                 [&] { jacobi_chain(B.l2, B.gamma, B.dt, B.inner, &vslot, (int)N, zbuf,
                                    B.beta * B.beta / B.phi, zbuf + N, ctrl_dev); });
      overlapped([&] { on_comm([&] { exchange(R_X1, zbuf + N, 1); }); },
                 [&] { block_op_s(B, zbuf, wbuf, nullptr, nullptr, ctrl_dev); });
    } else {
      overlapped([&] { on_comm([&] { exchange(R_X0, zbuf, 1); }); },
                 [&] { block_op_s(B, zbuf, wbuf, nullptr, nullptr, ctrl_dev); });
    }
    counters.op_bytes += 8.0 * N * B.size * 3.0;
  }
  if (timing) check(cudaEventRecord(ev0, stream));
  cgs_slab(n);
  if (timing) check(cudaEventRecord(ev1, stream));
}

// The split launches exist for the 2-D fused Jacobi chain and the strip
// block operator; the comm must enqueue device work only (NCCL) -- the host
// callback transport synchronises inside halo() anyway.
bool Engine::overlap_ok() const {
  return halo_overlap && slab() && comm->capturable() && ndim == 2 && fused_jacobi &&
         pair_jacobi && jacobi_split && strip_op && grid.nx % 2 == 0 && grid.nx >= 64;
}

// The 2-D fused chain can compute the ghost rows of its result itself
// (jacobi.cu, chain_ext) when the deeper input halo fits the ghost buffers.
bool Engine::ext_halo_ok() const {
  return ext_halo && slab() && ndim == 2 && prob.kind != KIND_ARAKAWA && fused_jacobi &&
         pair_jacobi && jacobi_split && grid.nx % 2 == 0 && grid.nx >= 64 && cfg.inner >= 1 &&
         cfg.inner <= 6 && 2 * (cfg.inner - 1) + 1 <= GH && grid.ny >= 2 * (cfg.inner - 1) + 1 &&
         grid.ny >= 2 * cfg.inner;
}

void Engine::fork_comm() {
  if (!comm_stream) {
    check(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking), "comm stream");
    check(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "event");
    check(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "event");
  }
  check(cudaEventRecord(ev_fork, stream), "fork");
  check(cudaStreamWaitEvent(comm_stream, ev_fork, 0), "fork wait");
}

void Engine::join_comm() {
  check(cudaEventRecord(ev_join, comm_stream), "join");
  check(cudaStreamWaitEvent(stream, ev_join, 0), "join wait");
}

// One Arnoldi step: z = M^{-1} v_j, w = A z, CGS2 + column finish.
void Engine::arnoldi_iteration(const BlockSpec &B, long long n) {
  if (slab()) {
    arnoldi_iteration_slab(B, n);
    return;
  }
  VecIn vslot{V, vpitch, ctrl_dev, W.alpha};
  precond(B, &vslot, zbuf, ctrl_dev);
  block_op(B, zbuf, wbuf, nullptr, nullptr, ctrl_dev);
  cgs(n);
}

void Engine::drop_graphs() {
  for (auto &kv : graphs) {
    if (kv.second.ex) cudaGraphExecDestroy(kv.second.ex);
    if (kv.second.g) cudaGraphDestroy(kv.second.g);
  }
  graphs.clear();
}

// Graph of one restart cycle: WHILE(cond) { Arnoldi step }.  Kernel
// arguments are fixed per block system (pointers, eta/beta/phi/gamma/dt,
// operator fields); the Arnoldi index and exit state live in the device
// control block, so the same executable serves every cycle and Newton
// iteration of that block.
// loop == false: a plain graph of ONE Arnoldi step, launched once per step
// by the host (multi-rank: NCCL's captured work is not allowed inside a
// conditional body).
Engine::CycleGraph &Engine::cycle_graph(const BlockSpec &B, long long n, bool loop) {
  char key[512];
  snprintf(key, sizeof key, "%c%d|%d|%a|%a|%a|%a|%a|%d|%p|%a|%d|%p|%a|%d|%p|%a|%d|%p|%a|%d|%lld|%p|%d",
           loop ? 'W' : 'S', loop ? graph_unroll : slab_batch, B.size, B.eta, B.beta, B.phi, B.gamma, B.dt, B.inner,
           (const void *)B.l1.a, B.l1.sigma, B.l1.present, (const void *)B.l2.a, B.l2.sigma,
           B.l2.present, (const void *)B.c12.a, B.c12.sigma, B.c12.present,
           (const void *)B.c21.a, B.c21.sigma, B.c21.present, n, (void *)V, vcap);
  auto it = graphs.find(key);
  if (it != graphs.end()) return it->second;
  if (graphs.size() > 64) drop_graphs();
  if (!cap_stream) check(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking), "stream");
  check(cudaStreamSynchronize(stream), "sync");
  CycleGraph cg;
  check(cudaGraphCreate(&cg.g, 0), "cudaGraphCreate");
  cudaGraph_t body = cg.g;
  if (loop) {
    check(cudaGraphConditionalHandleCreate(&cg.h, cg.g, 1, cudaGraphCondAssignDefault),
          "cond handle");
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cg.h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    check(cudaGraphAddNode(&node, cg.g, nullptr, 0, &np), "cond node");
    body = np.conditional.phGraph_out[0];
  }
  cudaStream_t saved = stream;
  stream = cap_stream;
  const long long launches0 = counters.kernel_launches;
  const double pb = counters.precond_bytes, ob = counters.op_bytes;
  check(cudaStreamBeginCaptureToGraph(cap_stream, body, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeRelaxed), "capture");
  cond_active = loop;
  cond_handle = cg.h;
  try {
    // the WHILE body holds `graph_unroll` Arnoldi steps: the conditional
    // re-launch of the body costs several us per trip, and a step after the
    // exit test fired is inert (every kernel checks cycle_done)
    for (int u = 0; u < (loop ? graph_unroll : slab_batch); ++u) arnoldi_iteration(B, n);
  } catch (...) {
    cond_active = false;
    stream = saved;
    cudaGraph_t tmp;
    cudaStreamEndCapture(cap_stream, &tmp);
    throw;
  }
  cond_active = false;
  cudaGraph_t captured;
  check(cudaStreamEndCapture(cap_stream, &captured), "end capture");
  stream = saved;
  cg.body_kernels = (int)(counters.kernel_launches - launches0);
  counters.kernel_launches = launches0;
  counters.precond_bytes = pb;
  counters.op_bytes = ob;
  check(cudaGraphInstantiate(&cg.ex, cg.g, 0), "cudaGraphInstantiate");
  auto res = graphs.emplace(key, cg);
  return res.first->second;
}

double Engine::gamma_of(double eta, double beta) const {
  if (cfg.gamma_mode == 0) return eta + beta * beta / eta;
  if (cfg.gamma_mode == 1) return eta;
  return cfg.gamma_custom;
}

// ------------------------------------------------------------------ GMRES
// src/sparsela.py:176-280 with x0 = 0.  V slot l stores s_l with
// v_l = alpha_l * s_l (no separate normalisation pass); the preconditioned
// basis Z is not stored: with the fixed linear preconditioner M^{-1}
// (Jacobi-k), x += Z y == x += M^{-1} (V y).
KrylovOut Engine::gmres(const BlockSpec &B, const double *rhs, double *x, double rtol, int maxit,
                        int restart, bool want_residuals) {
  if (!(rtol > 0.0 && rtol < 1.0)) throw SolveError(IRKG_ERR_VALUE, "rtol must lie in (0, 1)");
  ensure_basis(restart);
  ensure_res(maxit);
  last_block = B;
  have_last_block = true;
  if (B.inner == IRKG_INNER_EXACT) {
    // ShiftedSolver(..., "exact") factors its operator at construction, i.e.
    // once per block solve (src/irk_core.py:109-110, 155-156)
    band_factor(bfac[0], B.l1, B.eta, B.dt);
    if (B.size == 2) band_factor(bfac[1], B.l2, B.gamma, B.dt);
  } else if (B.inner == IRKG_INNER_MG) {
    mg_setup(B);  // restricted fields + coarsest factors, once per block solve
  }
  const long long n = (long long)B.size * N;
  const int spa = B.size;
  KrylovOut out;
  // ||b|| and the control block stay on the device: the first host round
  // trip of a solve is the end of its first restart cycle
  norm2_dev(rhs, n);
  gmres_init(maxit, rtol);
  check(cudaMemsetAsync(x, 0, n * sizeof(double), stream));
  check(cudaMemcpyAsync(V, rhs, n * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  int total_it = 0;
  int converged = 0;
  VecIn vslot{V, vpitch, ctrl_dev, W.alpha};
  VecIn vfix{ubuf, 0, nullptr, nullptr};
  while (!converged && total_it < maxit) {
    int m = std::min(restart, maxit - total_it);
    cycle_init(m);
    if (slab()) {
      // multi-rank: host-driven Arnoldi loop; with the NCCL transport each
      // step is one graph launch (captured NCCL halos + all-reduces)
      const bool g1 = use_graphs && !timing && comm->capturable() && prob.kind != KIND_ARAKAWA;
      if (g1) {
        // one graph launch = slab_batch steps, no host round trip in between; a
        // step after the exit test fired (or past the cycle length: the column
        // finish sets cycle_done at j + 1 >= m) is inert -- every kernel checks
        // cycle_done, the NCCL rounds move stale, unused values
        CycleGraph &cg = cycle_graph(B, n, false);
        int launched = 0;
        while (launched < m) {
          check(cudaGraphLaunch(cg.ex, stream), "cudaGraphLaunch");
          launched += slab_batch;
          read_ctrl();
          if (ctrl_host->cycle_done) break;
        }
        const int its = ctrl_host->j + 1;
        counters.kernel_launches += (long long)cg.body_kernels * (launched / slab_batch);
        counters.cgs_launches += 3LL * its;
        counters.arnoldi_iterations += its;
      }
      for (int it = 0; it < m && !g1; ++it) {
        {
          arnoldi_iteration_slab(B, n, it);  // (records ev0/ev1 around CGS2 when timing)
        }
        if (timing) {
          check(cudaEventSynchronize(ev1), "sync");
          float ms = 0.f;
          check(cudaEventElapsedTime(&ms, ev0, ev1), "elapsed");
          counters.cgs_time_ms += ms;
        }
        counters.cgs_launches += 3;
        counters.arnoldi_iterations += 1;
        read_ctrl();
        if (ctrl_host->cycle_done) break;
      }
    } else if (use_graphs && !timing) {
      // whole Arnoldi loop of this cycle as one graph launch (device-side WHILE)
      // (no host read here: the counters are settled after the cycle end)
      CycleGraph &cg = cycle_graph(B, n, true);
      if (graph_timing) check(cudaEventRecord(evg[0], stream));
      check(cudaGraphLaunch(cg.ex, stream), "cudaGraphLaunch");
      if (graph_timing) check(cudaEventRecord(evg[1], stream));
      graph_body_kernels = cg.body_kernels / graph_unroll;  // per Arnoldi step
    } else {
      for (int it = 0; it < m; ++it) {
        if (timing) check(cudaEventRecord(evp[0], stream));
        precond(B, &vslot, zbuf, ctrl_dev);                           // z = M^{-1} v_j
        if (timing) check(cudaEventRecord(evp[1], stream));
        block_op(B, zbuf, wbuf, nullptr, nullptr, ctrl_dev);          // w = A z
        if (timing) check(cudaEventRecord(ev0, stream));
        cgs(n);  // CGS2 in 3 fused sweeps + Hessenberg column / Givens / exit test
        if (timing) check(cudaEventRecord(ev1, stream));
        counters.cgs_launches += 3;
        counters.arnoldi_iterations += 1;
        read_ctrl();
        if (timing) {
          float ms = 0.f;
          check(cudaEventElapsedTime(&ms, ev0, ev1), "elapsed");
          counters.cgs_time_ms += ms;
          check(cudaEventElapsedTime(&ms, evp[0], evp[1]), "elapsed");
          counters.precond_time_ms += ms;
          check(cudaEventElapsedTime(&ms, evp[1], ev0), "elapsed");
          counters.op_time_ms += ms;
        }
        if (ctrl_host->cycle_done) break;
      }
    }
    {
      // algorithmic CGS2 bytes of this cycle: per iteration j, 4 sweeps over
      // (j+1) basis vectors + w traffic (2 reads, 1 rmw, 1 read + 1 write)
      double its = (double)(ctrl_host->j + 1);
      double sumj1 = its * (its + 1.0) / 2.0;  // sum_{j=0}^{its-1} (j+1)
      // 3 sweeps: DOT reads (j+1)+1 vectors, UPD_DOT reads (j+1)+1 and writes 1,
      // UPD_NORM reads (j+1)+1 and writes 1  ->  3(j+1) + 5 passes of n doubles
      counters.cgs_bytes += 8.0 * (double)n * (3.0 * sumj1 + 5.0 * its);
    }
    // cycle end: x += M^{-1} (V (alpha .* y)); r = b - A x (src/sparsela.py:258-272)
    backsolve();
    vcombine(n, W.c1, ubuf);
    precond(B, &vfix, zbuf, nullptr);
    axpy(n, 1.0, zbuf, x);
    block_op(B, x, V, rhs, &ctrl_dev->rr, nullptr);
    cycle_end();
    const bool timed_cycle = graph_timing && graph_body_kernels > 0;
    if (timed_cycle) check(cudaEventRecord(evg[2], stream));
    read_ctrl();
    if (timed_cycle) {
      float ms = 0.f;
      check(cudaEventSynchronize(evg[2]), "sync");
      check(cudaEventElapsedTime(&ms, evg[0], evg[1]), "elapsed");
      (B.size == 2 ? counters.arnoldi_ms_2x2 : counters.arnoldi_ms_1x1) += ms;
      check(cudaEventElapsedTime(&ms, evg[1], evg[2]), "elapsed");
      counters.cycle_end_ms += ms;
    }
    if (graph_body_kernels > 0) {  // WHILE-graph cycle: its = new iterations
      const int its = ctrl_host->total_it - total_it;
      counters.kernel_launches += (long long)graph_body_kernels * std::max(its, 1);
      counters.cgs_launches += 3LL * its;
      counters.arnoldi_iterations += its;
      graph_body_kernels = 0;
    }
    total_it = ctrl_host->total_it;
    converged = ctrl_host->converged;
    if (ctrl_host->zero_diag)
      throw SolveError(IRKG_ERR_VALUE, "Jacobi inner solver needs a nonzero diagonal");
    if (ctrl_host->err_breakdown) {
      char msg[160];
      double tr = std::sqrt(ctrl_host->rr) / ctrl_host->bnorm;
      snprintf(msg, sizeof msg, "Arnoldi breakdown with residual %.3e above rtol %.3e", tr, rtol);
      throw SolveError(IRKG_ERR_BREAKDOWN, msg);
    }
  }
  if (maxit <= 0) {  // no cycle ran: b = 0 is still converged (set by gmres_init)
    read_ctrl();
    converged = ctrl_host->converged;
  }
  out.iterations = total_it;
  out.converged = converged;
  out.precond_applications = total_it * spa;
  if (!want_residuals && converged) return out;
  int nres = ctrl_host->n_res;
  if (total_it == 0 && nres == 0) nres = 1;
  out.residuals.resize(nres);
  check(cudaMemcpyAsync(out.residuals.data(), W.res, nres * sizeof(double), cudaMemcpyDeviceToHost,
                        stream));
  check(cudaStreamSynchronize(stream));
  return out;
}

// ------------------------------------------------------- linearisation
// variant_weights (src/nonlinear.py:99-126) -> operator slots, then fields.
void Engine::build_linearization(const double *Ust) {
  build_weights();
  opfields(Ust, weights, opA);
  if (slab())  // operator fields feed stencils (fused Jacobi halo: K-1 planes)
    for (int o = 0; o < nops; ++o)
      if (!op_zero[o]) exchange(R_OP + o, opA + (size_t)o * N, inhalo());
}

void Engine::build_weights() {
  const int v = cfg.variant;
  double dw[MAXS][MAXS] = {};
  struct Key {
    int i, j;
  };
  std::vector<Key> keys;
  std::vector<std::vector<double>> ow;
  auto d = [&](int k, int l, int i) { return tab.d[(k * IRKG_MAX_STAGES + l) * IRKG_MAX_STAGES + i]; };
  if (v == 0) {
    for (int i = 0; i < s; ++i) dw[i][cfg.variant0_stage] = 1.0;
  } else if (v == 1) {
    for (int i = 0; i < s; ++i) {
      int best = 0;
      double bv = std::fabs(d(i, i, 0));
      for (int k = 1; k < s; ++k)
        if (std::fabs(d(i, i, k)) > bv) {
          bv = std::fabs(d(i, i, k));
          best = k;
        }
      dw[i][best] = 1.0;
    }
  } else {
    for (int i = 0; i < s; ++i)
      for (int k = 0; k < s; ++k) dw[i][k] = d(i, i, k);
    if (v == 3) {
      for (int i = 0; i < s; ++i)
        for (int j = i + 1; j < s; ++j) {
          keys.push_back({i, j});
          std::vector<double> w(s);
          for (int k = 0; k < s; ++k) w[k] = d(i, j, k);
          ow.push_back(w);
        }
      for (int b = 0; b < tab.nblocks; ++b)
        if (tab.blk_size[b] == 2) {
          int i = tab.blk_offset[b];
          keys.push_back({i + 1, i});
          std::vector<double> w(s);
          for (int k = 0; k < s; ++k) w[k] = d(i + 1, i, k);
          ow.push_back(w);
        }
    }
  }
  nops = s + (int)keys.size();
  if (nops > MAXOPS) throw SolveError(IRKG_ERR_CONFIG, "too many operator fields");
  if (nops > nops_cap) {
    dalloc(&opA, (size_t)nops * N);
    nops_cap = nops;
  }
  weights = OpWeights{};
  weights.nops = nops;
  weights.s = s;
  for (int i = 0; i < MAXS; ++i)
    for (int j = 0; j < MAXS; ++j) od_slot[i][j] = -1;
  for (int o = 0; o < nops; ++o) {
    const double *w = nullptr;
    std::vector<double> tmp(s);
    if (o < s) {
      for (int k = 0; k < s; ++k) tmp[k] = dw[o][k];
      diag_slot[o] = o;
    } else {
      tmp = ow[o - s];
      od_slot[keys[o - s].i][keys[o - s].j] = o;
    }
    w = tmp.data();
    double sig = 0.0;
    bool allzero = true;
    for (int k = 0; k < s; ++k) {
      weights.w[o * MAXS + k] = w[k];
      if (w[k] != 0.0) {
        sig += w[k];
        allzero = false;
      }
    }
    op_sigma[o] = sig;
    op_zero[o] = allzero;
  }
}

// A VariantJacobian given directly (src/nonlinear.py:86-96; the reference's
// solve_transformed_system(..., variant_jacobian=vj), src/irk_core.py:225-237):
// the s diagonal fields and the coupling fields keyed (i, j) are copied into
// the operator slots the transformed solve reads.  A field with a NULL
// coefficient array and sigma = 0 is the zero operator (a skipped key).
void Engine::set_variant_jacobian(const irkg_opfield *diag, int n_off, const int *oi,
                                  const int *oj, const irkg_opfield *off) {
  if (n_off < 0 || s + n_off > MAXOPS) throw SolveError(IRKG_ERR_CONFIG, "too many operator fields");
  nops = s + n_off;
  if (nops > nops_cap) {
    dalloc(&opA, (size_t)nops * N);
    nops_cap = nops;
  }
  for (int i = 0; i < MAXS; ++i)
    for (int j = 0; j < MAXS; ++j) od_slot[i][j] = -1;
  weights = OpWeights{};
  weights.nops = nops;
  weights.s = s;
  for (int o = 0; o < nops; ++o) {
    const irkg_opfield &f = o < s ? diag[o] : off[o - s];
    if (o < s) {
      diag_slot[o] = o;
    } else {
      const int i = oi[o - s], j = oj[o - s];
      if (i < 0 || i >= s || j < 0 || j >= s || i == j)
        throw SolveError(IRKG_ERR_VALUE, "coupling key out of range");
      od_slot[i][j] = o;
    }
    double *dst = opA + (size_t)o * N;
    if (f.a_dev)
      check(cudaMemcpyAsync(dst, f.a_dev, (size_t)N * sizeof(double), cudaMemcpyDeviceToDevice,
                            stream), "variant jacobian copy");
    else
      check(cudaMemsetAsync(dst, 0, (size_t)N * sizeof(double), stream), "variant jacobian zero");
    op_sigma[o] = f.sigma;
    op_zero[o] = (f.a_dev == nullptr && f.sigma == 0.0);
  }
  if (slab())
    for (int o = 0; o < nops; ++o)
      if (!op_zero[o]) exchange(R_OP + o, opA + (size_t)o * N, inhalo());
}

// N(u) for one state (OdeSystem.rhs): the stage residual kernel with one
// stage and K = 0.
void Engine::rhs(const double *u, double *f) {
  if (!zero_n) {
    dalloc(&zero_n, N);
    check(cudaMemsetAsync(zero_n, 0, (size_t)N * sizeof(double), stream), "zero");
  }
  residual(u, zero_n, f, 1);
}

Op Engine::op_of(int slot) const {
  Op o{};
  if (slot < 0 || op_zero[slot]) {
    o.present = 0;
    o.a = nullptr;
    o.sigma = 0.0;
    return o;
  }
  o.present = 1;
  o.a = opA + (size_t)slot * N;
  o.sigma = op_sigma[slot];
  return o;
}

// ---------------------------------------------------- transformed solve
// src/irk_core.py:225-338 (identity mass).
void Engine::transformed_solve(double dt, const double *rhs, double *dk, irkg_step_stats *stats) {
  // g = Q^T F
  std::vector<double> qt(s * s);
  for (int i = 0; i < s; ++i)
    for (int k = 0; k < s; ++k) qt[i * s + k] = tab.q[k * IRKG_MAX_STAGES + i];
  stage_mix(qt.data(), rhs, Gs, false);
  check(cudaMemsetAsync(Y, 0, (size_t)s * N * sizeof(double), stream));
  for (int b = tab.nblocks - 1; b >= 0; --b) {
    const int off = tab.blk_offset[b], size = tab.blk_size[b];
    BacksubTerms T{};
    T.rows = size;
    T.row0 = off;
    T.njs = 0;
    for (int j = off + size; j < s; ++j) {
      int q = T.njs++;
      T.j[q] = j;
      for (int r = 0; r < size; ++r) {
        T.coef[r][q] = tab.r[(off + r) * IRKG_MAX_STAGES + j];
        T.od[r][q] = op_of(od_slot[off + r][j]);
      }
    }
    gap_close(counters.block_gap_ms);
    backsub(dt, T, Gs, Y, RHS);
    BlockSpec B{};
    B.size = size;
    B.eta = tab.blk_eta[b];
    B.beta = tab.blk_beta[b];
    B.phi = tab.blk_phi[b];
    B.gamma = gamma_of(B.eta, B.beta);
    B.dt = dt;
    B.inner = cfg.inner;
    B.l1 = op_of(diag_slot[off]);
    if (size == 2) {
      B.l2 = op_of(diag_slot[off + 1]);
      B.c12 = op_of(od_slot[off][off + 1]);
      B.c21 = op_of(od_slot[off + 1][off]);
    }
    // the reference always applies the diagonal operators, even if zero
    B.l1.present = 1;
    if (!B.l1.a) B.l1.a = opA + (size_t)diag_slot[off] * N;
    if (size == 2) {
      B.l2.present = 1;
      if (!B.l2.a) B.l2.a = opA + (size_t)diag_slot[off + 1] * N;
    }
    KrylovOut rep = gmres(B, RHS, Y + (size_t)off * N, cfg.krylov_rtol, cfg.krylov_maxit, cfg.restart,
                          false);
    if (stats) {
      if (stats->n_block_records < IRKG_MAX_BLOCK_RECORDS) {
        stats->block_offset[stats->n_block_records] = off;
        stats->block_iterations[stats->n_block_records] = rep.iterations;
        stats->n_block_records++;
      }
      stats->krylov_iterations += rep.iterations;
      stats->precond_applications += rep.precond_applications;
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
      snprintf(msg, sizeof msg, "%dx%d block at offset %d did not converge", size, size, off);
      throw SolveError(IRKG_ERR_STAGE_SOLVE, msg);
    }
  }
  // dk = (Q R0) y
  if (dk) stage_mix(qr_matrix().data(), Y, dk, false);
}

std::vector<double> Engine::qr_matrix() const {
  std::vector<double> qr(s * s);
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j) {
      double acc = 0.0;
      for (int k = 0; k < s; ++k) acc += tab.q[i * IRKG_MAX_STAGES + k] * tab.r[k * IRKG_MAX_STAGES + j];
      qr[i * s + j] = acc;
    }
  return qr;
}

// ------------------------------------------------------------ phase probe
// Diagnostic: device time of one hot-path phase, replayed `reps` times
// back to back on the engine stream against the state the last gmres() call
// left (its block system, basis and fields).  Arnoldi index j is pinned by a
// one-thread kernel before each replay (its own time is probed as phase 7 and
// subtracted by the caller).  Destroys the Krylov state; diagnostics only.
__global__ void k_probe_setj(GCtrl *c, int j, int m) {
  c->j = j;
  c->m = m;
  c->k = j + 1;
  c->cycle_done = 0;
  c->converged = 0;
  c->total_it = 0;        // (phase 12: the cycle runs to m)
  c->maxit = 1 << 30;
  c->rtol = 0.0;
  c->breakdown = 0;
}

double Engine::probe_phase(int phase, int j, int reps) {
  if (!have_last_block) throw SolveError(IRKG_ERR_CONFIG, "probe: run a block solve first");
  const BlockSpec &B = last_block;
  const long long n = (long long)B.size * N;
  if (j < 0 || j + 1 >= vcap) throw SolveError(IRKG_ERR_VALUE, "probe: j out of range");
  VecIn vslot{V, vpitch, ctrl_dev, W.alpha};
  max_carveout((const void *)k_probe_setj);
  auto one = [&]() {
    // (phase 12: exactly 8 steps j .. j+7 of the WHILE graph)
    k_probe_setj<<<1, 1, 0, stream>>>(ctrl_dev, j, phase == 12 ? std::min(vcap, j + 8) : vcap);
    switch (phase) {
      case 0: precond(B, &vslot, zbuf, ctrl_dev); break;
      case 1: jacobi_chain(B.l1, B.eta, B.dt, B.inner, &vslot, 0, nullptr, 0.0, zbuf, ctrl_dev); break;
      case 2:
        jacobi_chain(B.size == 2 ? B.l2 : B.l1, B.size == 2 ? B.gamma : B.eta, B.dt, B.inner,
                     &vslot, B.size == 2 ? (int)N : 0, B.size == 2 ? zbuf : nullptr,
                     B.size == 2 ? B.beta * B.beta / B.phi : 0.0, zbuf + (B.size == 2 ? N : 0),
                     ctrl_dev);
        break;
      case 3: block_op(B, zbuf, wbuf, nullptr, nullptr, ctrl_dev); break;
      case 4: case 5: case 6: cgs(n, phase - 3); break;  // the first 1 / 2 / 3 sweeps
      case 7: break;
      case 8: arnoldi_iteration(B, n); break;
      case 9: {
        std::vector<double> eye(s * s, 0.0);
        for (int i = 0; i < s; ++i) eye[i * s + i] = 1.0;
        stage_mix(eye.data(), F, Gs, false);
        break;
      }
      case 10: vcombine(n, W.c1, ubuf); break;
      case 11: backsolve(); break;
      case 12: {  // the WHILE cycle graph from index j to the end of the cycle (m = vcap)
        CycleGraph &cg = cycle_graph(B, n, true);
        check(cudaGraphLaunch(cg.ex, stream), "cudaGraphLaunch");
        break;
      }
      default: throw SolveError(IRKG_ERR_VALUE, "probe: unknown phase");
    }
  };
  for (int i = 0; i < 2; ++i) one();  // warm
  check(cudaStreamSynchronize(stream), "probe sync");
  check(cudaEventRecord(ev0, stream));
  for (int i = 0; i < reps; ++i) one();
  check(cudaEventRecord(ev1, stream));
  check(cudaEventSynchronize(ev1), "probe sync");
  float ms = 0.f;
  check(cudaEventElapsedTime(&ms, ev0, ev1), "elapsed");
  return 1e3 * (double)ms / reps;
}

// -------------------------------------------------------------- Newton
// src/nonlinear.py:186-236.  K (s,N) in/out.
void Engine::newton(const double *u, double *K, double t, double dt, irkg_step_stats *stats) {
  auto tic = std::chrono::steady_clock::now();
  gap_armed = false;
  const std::vector<double> qrm = qr_matrix();
  stage_values(u, K, dt, U);
  double f0 = std::sqrt(residual(U, K, F));
  stats->n_residuals = 0;
  stats->residual_history[stats->n_residuals++] = f0;
  const double tol = std::max(cfg.newton_rtol * f0, cfg.newton_abs_floor);
  double fn = f0;
  bool have_ops = false;
  auto finish = [&]() {
    stats->wall_time =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - tic).count();
  };
  while (stats->newton_iterations < cfg.newton_maxit) {
    if (fn <= tol) {
      stats->converged = 1;
      finish();
      return;
    }
    gap_close(counters.newton_gap_ms);
    if (!have_ops || cfg.jacobian_refresh == 0) {
      build_linearization(U);  // U = u + dt A0 K at the current iterate
      stats->jacobian_assemblies += s;
      have_ops = true;
    }
    transformed_solve(dt, F, nullptr, stats);  // y (s,N) left in Y
    newton_update(qrm.data(), dt, Y, u, K, U);  // K += (Q R0) y ; U = u + dt A0 K
    stats->newton_iterations += 1;
    fn = std::sqrt(residual(U, K, F));
    if (stats->n_residuals <= IRKG_MAX_NEWTON) stats->residual_history[stats->n_residuals++] = fn;
  }
  if (fn > tol) {
    finish();
    char msg[160];
    snprintf(msg, sizeof msg, "stage solve stalled after %d iterations (residual %.3e, tol %.3e)",
             cfg.newton_maxit, fn, tol);
    throw SolveError(IRKG_ERR_STEP_FAILURE, msg);
  }
  stats->converged = 1;
  finish();
}

}  // namespace irkg

// ================================================================ C ABI
using namespace irkg;

struct irkg_ctx {
  Engine *eng;
};

static int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

#define IRKG_GUARD(...)                                           \
  try {                                                           \
    __VA_ARGS__;                                                  \
    return IRKG_OK;                                               \
  } catch (const SolveError &e) {                                 \
    return fail(e.code, e.what());                                \
  } catch (const CudaError &e) {                                  \
    return fail(IRKG_ERR_CUDA, e.what());                         \
  } catch (const std::exception &e) {                             \
    return fail(IRKG_ERR_CUDA, e.what());                         \
  }

static void validate_problem(const irkg_problem *prob, int rank, int nranks) {
  if (prob->kind < 0 || prob->kind > 3) throw SolveError(IRKG_ERR_CONFIG, "unknown problem kind");
  if (prob->kind == IRKG_KIND_ARAKAWA && (prob->nz != 1 || prob->nx < 3 || prob->ny < 3))
    throw SolveError(IRKG_ERR_CONFIG, "the vorticity DAE needs a 2-D grid >= 3x3");
  if (prob->nx < 1 || prob->ny < 1 || prob->nz < 1)
    throw SolveError(IRKG_ERR_VALUE, "grid extents must be positive");
  if (nranks < 1 || rank < 0 || rank >= nranks) throw SolveError(IRKG_ERR_VALUE, "bad rank/nranks");
  if (nranks > 1) {
    const int nd = (prob->nz > 1) ? 3 : (prob->ny > 1 ? 2 : 1);
    if (nd == 1) throw SolveError(IRKG_ERR_CONFIG, "slab partition needs a 2-D or 3-D grid");
    if (prob->kind == IRKG_KIND_ARAKAWA && nd != 2)
      throw SolveError(IRKG_ERR_CONFIG, "the vorticity DAE is 2-D");
    const int planes = nd == 3 ? prob->nz : prob->ny;
    if (planes / nranks < GH)
      throw SolveError(IRKG_ERR_CONFIG, "slabs must hold at least 6 planes per rank");
  }
  // local points incl. one plane of slack for the uneven split
  const long long nl = (long long)prob->nx * prob->ny * prob->nz / nranks + (long long)prob->nx * prob->ny;
  if (2 * nl >= (1LL << 31)) throw SolveError(IRKG_ERR_VALUE, "grid too large for one rank");
}

extern "C" {

const char *irkg_last_error(void) { return g_last_error.c_str(); }
const char *irkg_version(void) { return "irkg 0.1 sm_100a"; }

int irkg_create(irkg_ctx **out, const irkg_problem *prob, int device, void *stream,
                const void *nccl_id, int rank, int nranks) {
  IRKG_GUARD({
    validate_problem(prob, rank, nranks);
    Comm *comm = nullptr;
    // IRKG_FORCE_SLAB=1 with one rank: slab mode over a 1-rank NCCL ring (self
    // send/recv) -- exercises the NCCL transport on a single GPU
    const char *fs = getenv("IRKG_FORCE_SLAB");
    const bool force = nranks == 1 && nccl_id && fs && atoi(fs) != 0;
    if (nranks > 1 || force) {
      if (!nccl_id) throw SolveError(IRKG_ERR_VALUE, "nccl_id required when nranks > 1");
      check(cudaSetDevice(device), "cudaSetDevice");
      comm = make_nccl_comm(nccl_id, rank, nranks);
    }
    auto *c = new irkg_ctx;
    Engine *e = new Engine(*prob, device, (cudaStream_t)stream, rank, nranks, comm, force);
    c->eng = e;
    *out = c;
  });
}

int irkg_create_callback(irkg_ctx **out, const irkg_problem *prob, int device, void *stream,
                         int rank, int nranks, irkg_allreduce_fn allreduce, irkg_halo_fn halo,
                         void *user) {
  IRKG_GUARD({
    validate_problem(prob, rank, nranks);
    if (!allreduce || !halo) throw SolveError(IRKG_ERR_VALUE, "callbacks required");
    Comm *comm = nranks > 1 ? make_callback_comm(rank, nranks, allreduce, halo, user) : nullptr;
    auto *c = new irkg_ctx;
    c->eng = new Engine(*prob, device, (cudaStream_t)stream, rank, nranks, comm);
    *out = c;
  });
}

int irkg_set_alltoall_callback(irkg_ctx *ctx, irkg_alltoall_fn alltoall) {
  IRKG_GUARD({
    if (ctx->eng->comm) comm_set_alltoall(ctx->eng->comm, alltoall);
  });
}

int irkg_destroy(irkg_ctx *ctx) {
  IRKG_GUARD({
    if (ctx) {
      delete ctx->eng;
      delete ctx;
    }
  });
}

int irkg_get_local_extent(irkg_ctx *ctx, int *n_local, int *y0, int *ny_local) {
  IRKG_GUARD({
    *n_local = (int)ctx->eng->N;
    *y0 = ctx->eng->p0;
    *ny_local = ctx->eng->local_planes();
  });
}

int irkg_nccl_unique_id(void *out128) { IRKG_GUARD(nccl_unique_id(out128)); }

int irkg_set_tableau(irkg_ctx *ctx, const irkg_tableau *tab) { IRKG_GUARD(ctx->eng->set_tableau(*tab)); }
int irkg_set_solver(irkg_ctx *ctx, const irkg_solver *cfg) { IRKG_GUARD(ctx->eng->set_solver(*cfg)); }
int irkg_set_timing(irkg_ctx *ctx, int on) { IRKG_GUARD(ctx->eng->timing = (on != 0)); }
int irkg_get_counters(irkg_ctx *ctx, irkg_counters *out) { IRKG_GUARD(*out = ctx->eng->counters); }
int irkg_probe_phase(irkg_ctx *ctx, int phase, int j, int reps, double *us) {
  IRKG_GUARD({
    struct Flag {
      bool &f;
      ~Flag() { f = false; }
    } guard{ctx->eng->probing};
    ctx->eng->probing = true;
    *us = ctx->eng->probe_phase(phase, j, reps);
  });
}

int irkg_stage_residual(irkg_ctx *ctx, const double *u_dev, const double *k_dev, double t, double dt,
                        double *f_dev, double *norm) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (!e.have_tab) throw SolveError(IRKG_ERR_CONFIG, "tableau not set");
    (void)t;
    e.stage_values(u_dev, k_dev, dt, e.U);
    double v = e.residual(e.U, k_dev, f_dev);
    *norm = std::sqrt(v);
  });
}

int irkg_newton_step(irkg_ctx *ctx, const double *u_dev, double *k_dev, double t, double dt,
                     irkg_step_stats *stats) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (!e.have_tab || !e.have_cfg) throw SolveError(IRKG_ERR_CONFIG, "tableau/solver not set");
    if (e.dae) throw SolveError(IRKG_ERR_CONFIG, "DAE context: use the irkg_dae_* entry points");
    irkg_krylov_report fr = stats->fail_report;
    memset(stats, 0, offsetof(irkg_step_stats, fail_report));
    stats->fail_report = fr;
    e.newton(u_dev, k_dev, t, dt, stats);
  });
}

int irkg_step(irkg_ctx *ctx, double *u_dev, double t, double dt, irkg_step_stats *stats) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (!e.have_tab || !e.have_cfg) throw SolveError(IRKG_ERR_CONFIG, "tableau/solver not set");
    if (e.dae) throw SolveError(IRKG_ERR_CONFIG, "DAE context: use the irkg_dae_* entry points");
    irkg_krylov_report fr = stats->fail_report;
    memset(stats, 0, offsetof(irkg_step_stats, fail_report));
    stats->fail_report = fr;
    check(cudaMemsetAsync(e.Kst, 0, (size_t)e.s * e.N * sizeof(double), e.stream));
    e.newton(u_dev, e.Kst, t, dt, stats);
    e.step_update(dt, e.Kst, u_dev);
    check(cudaStreamSynchronize(e.stream));
  });
}

int irkg_dirk_step(irkg_ctx *ctx, double *u_dev, double t, double dt, irkg_step_stats *stats) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (!e.have_tab || !e.have_cfg) throw SolveError(IRKG_ERR_CONFIG, "tableau/solver not set");
    if (e.dae) throw SolveError(IRKG_ERR_CONFIG, "DIRK tableaux are not supported on DAE systems");
    irkg_krylov_report fr = stats->fail_report;
    memset(stats, 0, offsetof(irkg_step_stats, fail_report));
    stats->fail_report = fr;
    e.dirk_step(u_dev, t, dt, stats);
    check(cudaStreamSynchronize(e.stream));
  });
}

int irkg_step_host_out(irkg_ctx *ctx, const double *u_host, double *u_next_host, double t,
                       double dt, irkg_step_stats *stats) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (!e.have_tab || !e.have_cfg) throw SolveError(IRKG_ERR_CONFIG, "tableau/solver not set");
    if (e.dae) throw SolveError(IRKG_ERR_CONFIG, "DAE context: use the irkg_dae_* entry points");
    irkg_krylov_report fr = stats->fail_report;
    memset(stats, 0, offsetof(irkg_step_stats, fail_report));
    stats->fail_report = fr;
    check(cudaMemcpyAsync(e.ufield, u_host, e.N * sizeof(double), cudaMemcpyHostToDevice, e.stream));
    check(cudaMemsetAsync(e.Kst, 0, (size_t)e.s * e.N * sizeof(double), e.stream));
    e.newton(e.ufield, e.Kst, t, dt, stats);
    e.step_update(dt, e.Kst, e.ufield);
    check(cudaMemcpyAsync(u_next_host, e.ufield, e.N * sizeof(double), cudaMemcpyDeviceToHost,
                          e.stream));
    check(cudaStreamSynchronize(e.stream));
  });
}

int irkg_step_host(irkg_ctx *ctx, double *u_host, double t, double dt, irkg_step_stats *stats) {
  return irkg_step_host_out(ctx, u_host, u_host, t, dt, stats);
}

static Op to_op(const irkg_opfield *f) {
  Op o{};
  if (!f) return o;
  o.a = f->a_dev;
  o.sigma = f->sigma;
  o.present = 1;
  return o;
}

int irkg_linearize(irkg_ctx *ctx, const double *U_dev, int m, const double *weights,
                   double *a_out_dev, double *sigma_out) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (m < 1 || m > MAXS) throw SolveError(IRKG_ERR_VALUE, "stage count out of range");
    OpWeights W{};
    W.nops = 1;
    W.s = m;
    double sig = 0.0;
    for (int k = 0; k < m; ++k) {
      W.w[k] = weights[k];
      if (weights[k] != 0.0) sig += weights[k];
    }
    e.opfields(U_dev, W, a_out_dev);
    *sigma_out = sig;
    check(cudaStreamSynchronize(e.stream));
  });
}

int irkg_block2x2_apply(irkg_ctx *ctx, double eta, double beta, double phi, double dt,
                        const irkg_opfield *l1, const irkg_opfield *l2, const irkg_opfield *c12,
                        const irkg_opfield *c21, const double *x_dev, double *y_dev) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    BlockSpec B{};
    B.size = 2;
    B.eta = eta;
    B.beta = beta;
    B.phi = phi;
    B.dt = dt;
    B.l1 = to_op(l1);
    B.l2 = to_op(l2);
    B.c12 = to_op(c12);
    B.c21 = to_op(c21);
    e.block_op(B, x_dev, y_dev, nullptr, nullptr, nullptr);
    check(cudaStreamSynchronize(e.stream));
  });
}

int irkg_block2x2_precond(irkg_ctx *ctx, double eta, double beta, double phi, double gamma, double dt,
                          int inner, const irkg_opfield *l1, const irkg_opfield *l2,
                          const double *r_dev, double *z_dev) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (inner < IRKG_INNER_MG)
      throw SolveError(IRKG_ERR_VALUE, "inner must be 'exact', 'mg' or a positive int");
    BlockSpec B{};
    B.size = 2;
    B.eta = eta;
    B.beta = beta;
    B.phi = phi;
    B.gamma = gamma;
    B.dt = dt;
    B.inner = inner;
    B.l1 = to_op(l1);
    B.l2 = to_op(l2);
    VecIn vin{r_dev, 0, nullptr, nullptr};
    check(cudaMemsetAsync(e.ctrl_dev, 0, sizeof(GCtrl), e.stream));
    if (inner == IRKG_INNER_EXACT) {
      e.band_factor(e.bfac[0], B.l1, eta, dt);
      e.band_factor(e.bfac[1], B.l2, gamma, dt);
    } else if (inner == IRKG_INNER_MG) {
      e.mg_setup(B);
    }
    e.precond(B, &vin, z_dev, nullptr);
    e.read_ctrl();
    if (e.ctrl_host->zero_diag) throw SolveError(IRKG_ERR_VALUE, "Jacobi inner solver needs a nonzero diagonal");
  });
}

int irkg_shifted_solve(irkg_ctx *ctx, double alpha, double dt, int inner, const irkg_opfield *l,
                       const double *r_dev, double *x_dev) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (inner < IRKG_INNER_MG)
      throw SolveError(IRKG_ERR_VALUE, "inner must be 'exact', 'mg' or a positive int");
    VecIn vin{r_dev, 0, nullptr, nullptr};
    check(cudaMemsetAsync(e.ctrl_dev, 0, sizeof(GCtrl), e.stream));
    if (inner <= IRKG_INNER_EXACT) {
      BlockSpec B{};
      B.size = 1;
      B.eta = alpha;
      B.dt = dt;
      B.inner = inner;
      B.l1 = to_op(l);
      if (inner == IRKG_INNER_EXACT)
        e.band_factor(e.bfac[0], B.l1, alpha, dt);
      else
        e.mg_setup(B);
      e.precond(B, &vin, x_dev, nullptr);
    } else {
      e.jacobi_chain(to_op(l), alpha, dt, inner, &vin, 0, nullptr, 0.0, x_dev, nullptr);
    }
    e.read_ctrl();
    if (e.ctrl_host->zero_diag) throw SolveError(IRKG_ERR_VALUE, "Jacobi inner solver needs a nonzero diagonal");
  });
}

int irkg_block_gmres(irkg_ctx *ctx, int size, double eta, double beta, double phi, double gamma,
                     double dt, int inner, const irkg_opfield *l1, const irkg_opfield *l2,
                     const irkg_opfield *c12, const irkg_opfield *c21, const double *rhs_dev,
                     double *x_dev, double rtol, int maxit, int restart,
                     irkg_krylov_report *report) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (size != 1 && size != 2) throw SolveError(IRKG_ERR_VALUE, "block size must be 1 or 2");
    if (inner < IRKG_INNER_MG)
      throw SolveError(IRKG_ERR_VALUE, "inner must be 'exact', 'mg' or a positive int");
    BlockSpec B{};
    B.size = size;
    B.eta = eta;
    B.beta = beta;
    B.phi = phi;
    B.gamma = gamma;
    B.dt = dt;
    B.inner = inner;
    B.l1 = to_op(l1);
    B.l2 = to_op(l2);
    B.c12 = to_op(c12);
    B.c21 = to_op(c21);
    KrylovOut rep = e.gmres(B, rhs_dev, x_dev, rtol, maxit, restart);
    report->iterations = rep.iterations;
    report->converged = rep.converged;
    report->precond_applications = rep.precond_applications;
    report->n_residuals = (int)rep.residuals.size();
    if (report->residuals)
      for (int i = 0; i < (int)rep.residuals.size() && i < report->residual_capacity; ++i)
        report->residuals[i] = rep.residuals[i];
  });
}

int irkg_prepare_linearization(irkg_ctx *ctx, const double *u_dev, const double *k_dev, double dt) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (!e.have_tab || !e.have_cfg) throw SolveError(IRKG_ERR_CONFIG, "tableau/solver not set");
    if (e.dae) throw SolveError(IRKG_ERR_CONFIG, "DAE context: use the irkg_dae_* entry points");
    e.stage_values(u_dev, k_dev, dt, e.U);
    e.build_linearization(e.U);
    check(cudaStreamSynchronize(e.stream));
  });
}

int irkg_set_variant_jacobian(irkg_ctx *ctx, const irkg_opfield *diag, int n_off,
                              const int *off_i, const int *off_j, const irkg_opfield *off) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (!e.have_tab) throw SolveError(IRKG_ERR_CONFIG, "tableau not set");
    if (e.dae) throw SolveError(IRKG_ERR_CONFIG, "DAE context: use the irkg_dae_* entry points");
    e.set_variant_jacobian(diag, n_off, off_i, off_j, off);
    check(cudaStreamSynchronize(e.stream));
  });
}

int irkg_operator_apply(irkg_ctx *ctx, const irkg_opfield *l, const double *x_dev,
                        double *y_dev) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (e.dae) throw SolveError(IRKG_ERR_CONFIG, "DAE context: use the irkg_dae_* entry points");
    BlockSpec B{};
    B.size = 1;
    B.eta = 0.0;  // y = eta x - dt L x with eta = 0, dt = -1
    B.beta = 0.0;
    B.phi = 1.0;
    B.dt = -1.0;
    B.l1 = to_op(l);
    B.l1.present = 1;
    e.block_op(B, x_dev, y_dev, nullptr, nullptr, nullptr);
    check(cudaStreamSynchronize(e.stream));
  });
}

int irkg_rc_gmres_begin(irkg_ctx *ctx, long long n, const double *rhs_dev, const double *x0_dev,
                        double *x_dev, double *vin_dev, double *vout_dev, double rtol, int maxit,
                        int restart, int solves_per_apply) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    e.rc_begin(n, rhs_dev, x0_dev, x_dev, vin_dev, vout_dev, rtol, maxit, restart,
               solves_per_apply);
  });
}

int irkg_rc_gmres_next(irkg_ctx *ctx, int *action) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    *action = e.rc_next();
    if (*action != IRKG_RC_DONE) check(cudaStreamSynchronize(e.stream), "rc sync");
  });
}

int irkg_rc_gmres_report(irkg_ctx *ctx, irkg_krylov_report *report) {
  IRKG_GUARD(ctx->eng->rc_report(report));
}

int irkg_rhs(irkg_ctx *ctx, const double *u_dev, double t, double *f_dev) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    (void)t;  // every supported kind is autonomous
    if (e.dae) throw SolveError(IRKG_ERR_CONFIG, "DAE context: use the irkg_dae_* entry points");
    if (e.nranks > 1) throw SolveError(IRKG_ERR_CONFIG, "irkg_rhs: one rank only");
    e.rhs(u_dev, f_dev);
    check(cudaStreamSynchronize(e.stream));
  });
}

int irkg_transformed_solve(irkg_ctx *ctx, double dt, const double *rhs_dev, double *dk_dev,
                           irkg_step_stats *stats) {
  IRKG_GUARD({
    Engine &e = *ctx->eng;
    if (!e.have_tab || !e.have_cfg) throw SolveError(IRKG_ERR_CONFIG, "tableau/solver not set");
    if (e.dae) throw SolveError(IRKG_ERR_CONFIG, "DAE context: use the irkg_dae_* entry points");
    if (!(dt > 0.0)) throw SolveError(IRKG_ERR_VALUE, "dt must be positive");
    irkg_krylov_report fr = stats->fail_report;
    memset(stats, 0, offsetof(irkg_step_stats, fail_report));
    stats->fail_report = fr;
    e.transformed_solve(dt, rhs_dev, dk_dev, stats);
    check(cudaStreamSynchronize(e.stream));
  });
}

// ------------------------------------------------------------------- DAE

static Engine &dae_engine(irkg_ctx *ctx, bool need_solver) {
  Engine &e = *ctx->eng;
  if (!e.dae) throw SolveError(IRKG_ERR_CONFIG, "not a DAE context (kind IRKG_KIND_ARAKAWA)");
  if (need_solver && (!e.have_tab || !e.have_cfg))
    throw SolveError(IRKG_ERR_CONFIG, "tableau/solver not set");
  return e;
}

static void reset_stats(irkg_step_stats *stats) {
  irkg_krylov_report fr = stats->fail_report;
  memset(stats, 0, sizeof(irkg_step_stats));
  stats->fail_report = fr;
}

int irkg_dae_stage_residual(irkg_ctx *ctx, const double *uw_dev, const double *k2_dev, double t,
                            double dt, double *f2_dev, double *norm) {
  IRKG_GUARD({
    Engine &e = dae_engine(ctx, false);
    if (!e.have_tab) throw SolveError(IRKG_ERR_CONFIG, "tableau not set");
    (void)t;
    e.stage_values_n(uw_dev, k2_dev, dt, e.U, 2 * e.N);
    *norm = std::sqrt(e.dae_residual(e.U, k2_dev, f2_dev));
  });
}

int irkg_dae_step(irkg_ctx *ctx, double *uw_dev, double t, double dt, irkg_step_stats *stats) {
  IRKG_GUARD({
    Engine &e = dae_engine(ctx, true);
    reset_stats(stats);
    check(cudaMemsetAsync(e.Kst, 0, (size_t)e.s * 2 * e.N * sizeof(double), e.stream));
    e.dae_newton(uw_dev, e.Kst, t, dt, stats);
    e.step_update_n(dt, e.Kst, uw_dev, 2 * e.N);
    stats->constraint_residual = e.dae_gnorm(uw_dev);
  });
}

int irkg_dae_step_host(irkg_ctx *ctx, double *uw_host, double t, double dt,
                       irkg_step_stats *stats) {
  IRKG_GUARD({
    Engine &e = dae_engine(ctx, true);
    reset_stats(stats);
    const size_t bytes = 2 * e.N * sizeof(double);
    check(cudaMemcpyAsync(e.ufield, uw_host, bytes, cudaMemcpyHostToDevice, e.stream));
    check(cudaMemsetAsync(e.Kst, 0, (size_t)e.s * bytes, e.stream));
    e.dae_newton(e.ufield, e.Kst, t, dt, stats);
    e.step_update_n(dt, e.Kst, e.ufield, 2 * e.N);
    stats->constraint_residual = e.dae_gnorm(e.ufield);
    check(cudaMemcpyAsync(uw_host, e.ufield, bytes, cudaMemcpyDeviceToHost, e.stream));
    check(cudaStreamSynchronize(e.stream));
  });
}

int irkg_dae_constraint_norm(irkg_ctx *ctx, const double *uw_dev, double *norm) {
  IRKG_GUARD({
    Engine &e = dae_engine(ctx, false);
    *norm = e.dae_gnorm(uw_dev);
  });
}

}  // extern "C"
