// engine.h -- host-side engine: device buffers, launchers and the solver
// drivers (GMRES control, transformed solve, Newton loop).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <set>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/irkg.h"
#include "kernels.cuh"

namespace irkg {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Error carrying an irkg status code (mapped to reference exception types).
struct SolveError : std::runtime_error {
  int code;
  SolveError(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

inline void check(cudaError_t e, const char *what = "cuda") {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// One eigen-block system (Block2x2System / the 1x1 shifted system) plus
// the preconditioner parameters (src/irk_core.py:71-95, 147-165, 215-222).
struct BlockSpec {
  int size;
  double eta, beta, phi, gamma, dt;
  int inner;
  Op l1, l2, c12, c21;
};

// Transport of the slab partition (comm.cu)
struct Comm {
  int rank = 0, nranks = 1;
  virtual ~Comm() {}
  virtual void allreduce_sum(double *dev, int count, cudaStream_t st) = 0;
  // send my first `count` values (send_lo) to rank-1 and my last (send_hi) to
  // rank+1 (periodic); receive rank+1's first into recv_hi, rank-1's last into recv_lo
  virtual void halo(const double *send_lo, const double *send_hi, double *recv_lo,
                    double *recv_hi, long long count, cudaStream_t st) = 0;
  struct Xfer {
    const double *send_lo, *send_hi;
    double *recv_lo, *recv_hi;
    long long count;
  };
  // several halo exchanges in one round (one NCCL group)
  virtual void halo_batch(int nx, const Xfer *x, cudaStream_t st) {
    for (int i = 0; i < nx; ++i)
      halo(x[i].send_lo, x[i].send_hi, x[i].recv_lo, x[i].recv_hi, x[i].count, st);
  }
  // personalised all-to-all: block p of `send` (count doubles) goes to rank p,
  // block p of `recv` arrives from rank p (the pencil transposes of the DAE
  // constraint solve, dae.cu)
  virtual void alltoall(const double *send, double *recv, long long count, cudaStream_t st) = 0;
  // enqueues only device work (no host round trip): graph-capturable
  virtual bool capturable() const { return false; }
};
void comm_set_alltoall(Comm *c, irkg_alltoall_fn fn);
Comm *make_nccl_comm(const void *id128, int rank, int nranks);
Comm *make_callback_comm(int rank, int nranks, irkg_allreduce_fn a, irkg_halo_fn h, void *u);
void nccl_unique_id(void *out128);

// ghost-buffer roles (one ghost pair per role, re-pointed by exchange())
enum GhostRole {
  R_VIN0 = 0, R_VIN1 = 1, R_Z0 = 2, R_Z1 = 3, R_X0 = 4, R_X1 = 5, R_JX = 6,
  R_DG = 7,      // DAE: psi of the state (constraint norm)
  R_DB = 8,      // DAE: 4 fields of the composite block residual (8..11)
  R_STAGE = 16,  // stage values U_i (16..23)
  R_DW = 24,     // DAE: stage values W_i (24..31)
  R_Y = 32,      // back-substitution y_j (DAE: y_u,j) (32..39)
  R_DYW = 40,    // DAE back-substitution y_w,j (40..47)
  R_OP = 64      // operator fields
};

// Banded LU + SMW factor of one shifted operator (banded.cu)
struct BandFactor {
  int n = 0, kl = 0, ku = 0, ldab = 0, nb = 0;
  double *ab = nullptr;     // ldab x n, column-major (LAPACK band layout)
  int *piv = nullptr;
  double *binvu = nullptr;  // n x nb: B^{-1} U
  double *cap = nullptr;    // nb x nb LU of I + E^T B^{-1} U
  int *cpiv = nullptr;
  int *info = nullptr;
  double *mid = nullptr;    // nb
  double *wglob = nullptr;  // factor window when it does not fit in shared memory
  size_t wsmem = 0;
};

// Geometric-multigrid hierarchy of the block's inner operators (mg.cu)
constexpr int MG_MAXLEV = 16;
struct MgLevel {
  Grid g{};
  double *a[2] = {nullptr, nullptr};  // coefficient field of S1 / S2 on this level
  double *b = nullptr, *x = nullptr, *t = nullptr;
};
struct MgHier {
  int nlev = 0;
  MgLevel lev[MG_MAXLEV];
  BandFactor coarse[2];
  double alpha[2] = {0.0, 0.0}, sigma[2] = {0.0, 0.0}, dt = 0.0;
};

// out = scale * in [+ cpl * zc] (an inner solve's right-hand side; banded.cu)
__global__ void k_vin_rhs(int n, VecIn vin, int in_off, const double *__restrict__ zc, double cpl,
                          double *__restrict__ out, const GCtrl *skip);

struct KrylovOut {
  int iterations = 0;
  int converged = 0;
  int precond_applications = 0;
  std::vector<double> residuals;
};

struct Engine {
  // configuration
  irkg_problem prob{};
  Grid grid{};
  KindParams kp{};
  int ndim = 1;
  long long N = 0;
  int device = 0;
  int sms = 148;
  int G = 296;  // CTAs of the reduction kernels (partials per value)
  cudaStream_t stream = nullptr;
  bool timing = false;
  irkg_counters counters{};

  // tableau + solver
  bool have_tab = false, have_cfg = false;
  irkg_tableau tab{};
  irkg_solver cfg{};
  int s = 0;

  // device buffers
  double *part = nullptr;       // 3 x (MAXR+2) * G reduction partials
  unsigned *counter = nullptr;  // last-CTA ticket
  double *scal_dev = nullptr;   // scalar outputs
  GCtrl *ctrl_dev = nullptr;
  GWork W{};
  double *V = nullptr;          // basis, (restart+1) slots of 2N
  long long vpitch = 0;
  int vcap = 0;                 // allocated restart capacity
  void *vmaps = nullptr;        // CUtensorMap[4][9] over V: boxes (32<<a rows, 1<<b slots)
  void build_vmaps();
  double *wbuf = nullptr;       // 2N: w
  double *zbuf = nullptr;       // 2N: z / cycle-end scratch
  double *ubuf = nullptr;       // 2N: V y combination
  double *tmp_x = nullptr;      // N: Jacobi ping-pong
  double *tmp_t = nullptr;      // N: coupled rhs of the second inner solve
  // stage arrays (s, N)
  double *U = nullptr, *F = nullptr, *Gs = nullptr, *Y = nullptr, *DK = nullptr, *Kst = nullptr;
  double *RHS = nullptr;        // (2, N) block rhs
  double *ufield = nullptr;     // N (step_host staging)
  double *opA = nullptr;        // (nops, N) operator fields
  double *zero_n = nullptr;     // N zeros (irkg_rhs: K = 0)
  int nops_cap = 0;
  GCtrl *ctrl_host = nullptr;   // pinned mirror
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evp[2] = {nullptr, nullptr};
  cudaEvent_t evg[3] = {nullptr, nullptr, nullptr};  // cycle graph / cycle end (IRKG_GRAPH_TIMING)
  cudaEvent_t evh[2] = {nullptr, nullptr};  // host round-trip gaps (IRKG_GRAPH_TIMING)
  bool gap_armed = false;
  void gap_mark();              // before a host sync: the device work enqueued so far
  void gap_close(double &acc);  // after it: first work of the next phase
  bool graph_timing = false;

  // current linearisation: operator slot per diag row and per offdiag key
  int nops = 0;
  int diag_slot[MAXS];
  int od_slot[MAXS][MAXS];  // -1 if absent
  double op_sigma[MAXOPS];
  bool op_zero[MAXOPS];
  OpWeights weights{};

  // slab partition (comm.cu); nranks == 1: periodic wrap, no communication
  Comm *comm = nullptr;
  int rank = 0, nranks = 1;
  int gplanes = 1, p0 = 0;  // global planes along the slab axis, my first plane
  struct Ghost {
    double *lo = nullptr, *hi = nullptr;
    const double *field = nullptr;
  };
  std::map<int, Ghost> ghosts;
  std::map<const double *, int> owner;
  bool slab_forced = false;  // 1-rank slab mode over the transport (tests the NCCL path)
  bool slab() const { return nranks > 1 || slab_forced; }
  int local_planes() const { return ndim == 3 ? grid.nz : grid.ny; }
  int plane_size() const;
  Ghost &role(int r);
  void exchange(int role, const double *f, int depth);
  void allreduce(double *dev, int count);
  FRef ref(const double *p) const;
  Op opref(const Op &o) const;
  StageGhosts stage_ghosts(const double *Ub, long long stride, int nst = -1) const;
  void free_ghosts();
  int jhalo() const { return cfg.inner > 1 ? cfg.inner - 1 : 1; }
  // halo depth of the inner solves' inputs (v_j, operator fields): K-1, or 2(K-1)+1 when
  // the chains compute their results' ghost rows themselves (ext_halo_ok)
  int inhalo() const { return ext_halo_ok() ? 2 * (cfg.inner - 1) + 1 : jhalo(); }

  Engine(const irkg_problem &p, int dev, cudaStream_t st, int rank_ = 0, int nranks_ = 1,
         Comm *comm_ = nullptr, bool force_slab = false);
  ~Engine();

  void set_tableau(const irkg_tableau &t);
  void set_solver(const irkg_solver &c);
  void ensure_stage_buffers();
  void ensure_basis(int restart);
  void ensure_res(int maxit);
  int rescap = 0;
  size_t cgs_smem_set = 0;
  // CUDA-graph execution of the Arnoldi loop: one graph per block system,
  // a WHILE conditional node whose condition the last CGS kernel clears.
  struct CycleGraph {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ex = nullptr;
    cudaGraphConditionalHandle h{};
    int body_kernels = 0;
  };
  std::map<std::string, CycleGraph> graphs;
  bool use_graphs = true;
  bool cond_active = false;
  cudaGraphConditionalHandle cond_handle{};
  cudaStream_t cap_stream = nullptr;
  CycleGraph &cycle_graph(const BlockSpec &B, long long n, bool loop);
  void arnoldi_iteration(const BlockSpec &B, long long n);
  void drop_graphs();
  int cgs_stage_doubles() const;  // CGS shared-memory ring per CTA (doubles)
  void cgs(long long n, int nsweeps = 3);  // cgs.cu
  // the three sweeps in one launch with grid barriers (k_cgs3, IRKG_CGS_FUSED=1).  Off by
  // default: bit-identical, faster in isolation at j <= 4 (37.8 vs 46.5 us at j = 2) but not
  // at the step's mean Arnoldi index -- configs[1] 27.36 vs 27.01 ms/step on the same box
  // (profiles/r2s4_cgs_fused_ab.txt)
  bool cgs_fused = false;
  int cgs_fused_occ = -1;
  size_t cgs_fused_smem = 0;
  unsigned long long *gbar = nullptr;
  long long cgs_fused_maxn = 0;  // IRKG_CGS_FUSED_MAXN: fuse only sweeps over at most this many rows
  bool cgs_fused_ok(size_t smem, int trm, long long n);
  // stencil.cu (register-sliding 2-D / 3-D kernels)
  dim3 slide_grid(int &span) const;
  void jac_sweep_s(const Op &L, double alpha, double dt, const VecIn &vin, int in_off,
                   const double *t_in, const double *x, double *x_out, const GCtrl *skip);
  void block_op_s(const BlockSpec &B, const double *z, double *w, const double *b,
                  double *out_norm, const GCtrl *skip);
  double residual_s(const double *U, const double *K, double *F, int nst);
  void backsub_s(double dt, BacksubTerms T, const double *gst, const double *y, double *rhs);
  void cgs_slab(long long n);  // CGS2 with all-reduces between sweeps (multi-rank)
  void arnoldi_iteration_slab(const BlockSpec &B, long long n, int j_host = -1);
  double *halo_pack = nullptr;  // packed boundary planes of basis slot j (2 halves x lo/hi)
  int slab_batch = 4;           // multi-rank Arnoldi steps launched per host check (IRKG_SLAB_BATCH)
  // Arnoldi steps per WHILE-body trip (IRKG_GRAPH_UNROLL); configs[1]:
  // 1 / 2 / 3 / 4 -> 32.09 / 31.83 / 31.76 / 31.72 ms per IRK step
  int graph_unroll = 4;
  // dae.cu (vorticity/streamfunction DAE, reordered mode)
  bool dae = false;
  double h2 = 0.0;
  double *ACC = nullptr, *XU = nullptr, *CR = nullptr, *PT = nullptr;
  void *fft_buf = nullptr;
  int fft_fwd = -1, fft_inv = -1;
  // slab mode: the constraint solve as a slab -> pencil transpose FFT.  Rows
  // (x) are transformed where they live, an all-to-all hands every rank a
  // pencil of tr_cols x-wavenumbers with all of y, the y transforms and the
  // eigenvalue division run there, and the way back mirrors it.
  int tr_C = 0;       // x-wavenumbers per rank (the last ranks may own fewer / none)
  int tr_cols = 0;    // ... owned by this rank
  int tr_nylmax = 0;  // most rows any rank owns (all-to-all blocks are padded to it)
  int fft_col = -1;
  double *tr_send = nullptr, *tr_recv = nullptr, *tr_lines = nullptr;
  void constraint_solve_slab(double sigma, const double *c, double *out, double post);
  void dae_init();
  void dae_fini();
  int dae_grid() const;
  void constraint_solve(double sigma, const double *c, double *out, double post);
  void ara_jacobi_chain(const Op &L, double alpha, double dt, int inner, const VecIn &vin,
                        int in_off, const double *zc, double cpl, double *x_out,
                        const GCtrl *skip);
  void ara_block_op(const BlockSpec &B, const double *z, double *w, const double *b,
                    double *out_norm, const GCtrl *skip);
  double dae_residual(const double *UW, const double *K2, double *F2);
  double dae_gnorm(const double *UW);
  void dae_transformed_solve(double dt, const double *rhs, double *dk, irkg_step_stats *stats);
  void dae_newton(const double *uw, double *K2, double t, double dt, irkg_step_stats *stats);
  // generic helpers
  long long Nst() const { return dae ? 2 * N : N; }
  void stage_mix_n(const double *M_rowmajor_s, const double *in, double *out, bool accumulate,
                   long long n);
  void stage_values_n(const double *u, const double *K, double dt, double *Uo, long long n);
  void step_update_n(double dt, const double *K, double *u, long long n);
  void build_weights();
  static void dalloc_raw(void **p, size_t bytes);
  // jacobi.cu (temporally blocked inner solves, 2-D)
  bool fused_jacobi = true;
  int jspan_override = 0;
  bool pair_jacobi = true;
  bool jacobi_split = true;  // split-operator pair kernel (IRKG_JACOBI_SPLIT=0: textbook form)   // column-pair Jacobi kernel (IRKG_PAIR_JACOBI=0: one column per lane)
  int jwarps_per_sm = 12;    // pair kernel: target resident warps per SM (IRKG_JWPS)
  bool strip_op = true;      // 2-D block operator on column-pair strips (IRKG_STRIP_OP=0: slide)
  int bop_wps = 8;           // strip block operator: target warps per SM (IRKG_BOP_WPS)
  bool jacobi_chain_fused(const Op &L, double alpha, double dt, int inner, const VecIn &vin,
                          int in_off, const double *zc, double cpl, double *x_out,
                          const GCtrl *skip);
  // arachain.cu (temporally blocked inner solves of the vorticity DAE; IRKG_FUSED_ARA=0: K launches)
  bool fused_ara = true;
  bool ara_warp_form = true;  // IRKG_ARA_WARP=0: the CTA-strip kernel on every grid
  bool ara_chain_fused(const Op &L, double alpha, double dt, int inner, const VecIn &vin,
                       int in_off, const double *zc, double cpl, double *x_out, const GCtrl *skip);
  // jacobi3d.cu (3.5-D blocked inner solves, 3-D grids; IRKG_FUSED_JACOBI3D=0: K launches)
  bool fused_jacobi3d = true;
  bool jacobi_chain_fused3d(const Op &L, double alpha, double dt, int inner, const VecIn &vin,
                            int in_off, const double *zc, double cpl, double *x_out,
                            const GCtrl *skip);

  // PDL launch of an Arnoldi-body kernel (IRKG_PDL=0: ordinary launch)
  bool use_pdl = true;
  template <typename... KArgs, typename... Args>
  void launch_pdl(void (*kern)(KArgs...), dim3 grid_, dim3 block_, size_t smem, Args &&...args) {
    launch_pdl_l2(false, kern, grid_, block_, smem, std::forward<Args>(args)...);
  }
  // basis_l2: the launch carries the access-policy window that keeps the
  // lowest basis slots persisting in L2 (the slots every CGS sweep re-reads)
  template <typename... KArgs, typename... Args>
  void launch_pdl_l2(bool basis_l2, void (*kern)(KArgs...), dim3 grid_, dim3 block_, size_t smem,
                     Args &&...args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid_;
    lc.blockDim = block_;
    lc.dynamicSmemBytes = smem;
    lc.stream = stream;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (use_pdl) {
      at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    if (basis_l2 && l2win.num_bytes > 0) {
      at[na].id = cudaLaunchAttributeAccessPolicyWindow;
      at[na].val.accessPolicyWindow = l2win;
      ++na;
    }
    lc.attrs = at;
    lc.numAttrs = na;
    max_carveout((const void *)kern);
    check(cudaLaunchKernelEx(&lc, kern, std::forward<Args>(args)...), "PDL launch");
  }
  // L2 persistence of the lowest l2_budget bytes of the basis (IRKG_L2_MB;
  // 0 = off).  configs[1] (16.8 MB slots): 1 / 2 / 3 / 4 / 5 slots ->
  // 31.72 / 31.35 / 31.07 / 31.93 / 32.78 ms per IRK step (none: 31.73);
  // 40 / 50 / 60 MB -> 31.21 / 31.02 / 30.93; with the row-owner CGS update
  // sweeps (session 4) 34 / 51 / 60 MB -> 29.68 / 29.68 / 29.80
  size_t l2_budget = 51u << 20;
  size_t l2_persist_max = 0, l2_window_max = 0;
  cudaAccessPolicyWindow l2win{};
  bool l2_holder = false;
  bool probing = false;     // inside irkg_probe_phase (timing experiments)
  // slab halo / interior overlap (IRKG_HALO_OVERLAP): the 2-D fused chain and
  // strip operator launch only the bands that read no ghost plane
  // (band_sel 1) while the halo is in flight on comm_stream, then the edge
  // bands (band_sel 2) after the join
  // reverse-communication GMRES (rcgmres.cu; irkg_rc_gmres_*)
  enum RcPhase { RC_R0, RC_R0_DONE, RC_CYCLE, RC_PREC, RC_PREC_DONE, RC_OP, RC_OP_DONE,
                 RC_CYCLE_END, RC_RESID, RC_DONE };
  struct RcState {
    bool active = false;
    long long n = 0, zn = 0;
    int zcap = 0;
    double *Z = nullptr;  // stored preconditioned basis (restart x n)
    const double *b = nullptr;
    double *x = nullptr, *vin = nullptr, *vout = nullptr;
    double rtol = 0.0;
    int maxit = 0, restart = 0, spa = 0, j = 0, its = 0;
    RcPhase phase = RC_DONE;
  } rc;
  void rc_copy(double *dst, const double *src, long long n);
  void rc_begin(long long n, const double *b, const double *x0, double *x, double *vin,
                double *vout, double rtol, int maxit, int restart, int spa);
  int rc_next();
  void rc_report(irkg_krylov_report *rep);
  int band_sel = 0;
  bool halo_overlap = true;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // bands [lo, hi) of nb bands of `span` rows (local ny) read only local rows
  // when the stencil reaches h rows beyond the band
  // (bands start at row ylo <= 0 when the chain also computes ghost rows)
  void interior_bands(int nb, int span, int h, int &lo, int &hi, int ylo = 0) const {
    lo = 0;
    while (lo < nb && ylo + lo * span < h) ++lo;
    hi = nb;
    while (hi > lo && ylo + hi * span + h > grid.ny) --hi;
  }
  // Extended-halo chains (slab mode, 2-D fused chain): a chain also computes
  // chain_ext rows beyond the slab on either side, from a deeper halo of its
  // input, into the ghost planes of role chain_out_role -- the Arnoldi step
  // then exchanges only v_j (depth 2(K-1)+1) instead of v_j, z1 and z2
  int chain_ext = 0, chain_out_role = 0;
  bool ext_halo = true;  // IRKG_EXT_HALO=0: exchange z1 / z2 instead
  bool ext_halo_ok() const;
  bool overlap_ok() const;  // the slab step can split its stencils
  void fork_comm();
  void join_comm();  // counted in the per-device persisting-limit refcount
  void release_l2_limit();
  void set_l2_window();
  int cgs_ef_from() const;
  // All Arnoldi-body kernels ask for the maximum shared-memory carveout, so
  // consecutive kernels never force an L1/shared reconfiguration of the SMs
  // (IRKG_CARVEOUT=0: driver default).
  bool use_carveout = true;
  std::set<const void *> carved;
  void max_carveout(const void *fn) {
    if (!use_carveout || carved.count(fn)) return;
    check(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                               (int)cudaSharedmemCarveoutMaxShared),
          "carveout");
    carved.insert(fn);
  }
  // launch helpers (kernels.cu)
  int grid_for(long long n) const;
  int row_grid() const {  // CTAs of row-structured stencil kernels
    int rows = grid.ny * grid.nz;
    return rows < sms * 8 ? rows : sms * 8;
  }
  void count(int k);
  double norm2(const double *x, long long n, const GCtrl *skip = nullptr);
  void stage_values(const double *u, const double *K, double dt, double *U);
  double residual(const double *U, const double *K, double *F, int nst = -1);
  void opfields(const double *U, const OpWeights &W, double *A);
  void stage_mix(const double *M_rowmajor_s, const double *in, double *out, bool accumulate);
  void step_update(double dt, const double *K, double *u);
  void backsub(double dt, const BacksubTerms &T, const double *gst, const double *y, double *rhs);
  void jacobi_chain(const Op &L, double alpha, double dt, int inner, const void *vin, int in_off,
                    const double *zc, double cpl, double *x_out, const GCtrl *skip);
  void precond(const BlockSpec &B, const void *vin, double *z, const GCtrl *skip);
  void block_op(const BlockSpec &B, const double *z, double *w, const double *b,
                double *out_norm, const GCtrl *skip);
  void cycle_init(int m);
  void gmres_init(int maxit, double rtol);
  void norm2_dev(const double *x, long long n);
  void newton_update(const double *QR_rowmajor_s, double dt, const double *Yv, const double *u,
                     double *K, double *Uo);
  void backsolve();
  void vcombine(long long n, const double *coef, double *out);
  void axpy(long long n, double a, const double *x, double *y);
  void cycle_end();

  // drivers (engine.cu)
  BlockSpec last_block{};  // block system of the last gmres() call (phase probe)
  bool have_last_block = false;
  double probe_phase(int phase, int j, int reps);
  void read_ctrl();
  double read_scalar();
  int graph_body_kernels = 0;  // body size of the WHILE graph launched this cycle
  std::vector<double> qr_matrix() const;  // Q R0, row-major s x s
  // want_residuals = false: the residual history is copied back only when
  // the solve failed (the stage solves report it in StageSolveError alone),
  // saving a host round trip per block solve
  KrylovOut gmres(const BlockSpec &B, const double *rhs, double *x, double rtol, int maxit,
                  int restart, bool want_residuals = true);
  void build_linearization(const double *U);
  Op op_of(int slot) const;
  void set_variant_jacobian(const irkg_opfield *diag, int n_off, const int *oi, const int *oj,
                            const irkg_opfield *off);
  void rhs(const double *u, double *f);
  double gamma_of(double eta, double beta) const;
  // dk == nullptr: leave y in Y (the Newton loop fuses dk = (Q R0) y into its update)
  void transformed_solve(double dt, const double *rhs, double *dk, irkg_step_stats *stats);
  void newton(const double *u, double *K, double t, double dt, irkg_step_stats *stats);
  // banded.cu: exact inner solves (PrecondSpec(inner="exact"), cfg.inner == 0)
  BandFactor bfac[2];
  void band_factor(BandFactor &F, const Op &L, double alpha, double dt, const Grid *gl = nullptr);
  void band_solve(const BandFactor &F, double *b, long long ldb, int nrhs, const GCtrl *skip);
  void band_apply(const BandFactor &F, double *x, const GCtrl *skip);
  void precond_exact(const BlockSpec &B, const VecIn &vin, double *z, const GCtrl *skip);
  // mg.cu: one V-cycle per inner solve (PrecondSpec(inner="mg"), cfg.inner == -1)
  MgHier mg;
  double *mg_rhs = nullptr;
  void mg_setup(const BlockSpec &B);
  void mg_vcycle(int o, const double *b, double *x, const GCtrl *skip);
  void precond_mg(const BlockSpec &B, const VecIn &vin, double *z, const GCtrl *skip);
  // dirk.cu: sequential stage solves of an (S)DIRK tableau (src/nonlinear.py:239-296)
  void dirk_step(double *u, double t, double dt, irkg_step_stats *stats);
};

}  // namespace irkg
