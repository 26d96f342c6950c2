// comm.cu -- slab partition communication: halo exchange + global sums.
//
// The grid is split into contiguous slabs along its slowest axis (y in 2-D,
// z in 3-D); rank r owns planes [p0, p0 + nl).  Stencil consumers read the
// GH planes on either side from per-role ghost buffers filled here.  Global
// inner products / norms are per-rank deterministic partial sums combined
// with an all-reduce, so every rank takes the identical control decisions
// (GMRES exits, Newton tolerance) from identical scalars.
//
// Two transports behind one interface:
//  * NcclComm     -- ncclSend/ncclRecv (grouped) + ncclAllReduce over NVLink;
//                    libnccl is dlopen'ed (RTLD_NOLOAD first: reuse the copy
//                    torch.distributed already loaded).
//  * CallbackComm -- host callbacks supplied through the C ABI; the Python
//                    layer implements them with torch.distributed (used by
//                    the multi-process tests on one GPU; no kernel ever
//                    waits on another rank).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "engine.h"

namespace irkg {

// ------------------------------------------------------------- NCCL via dlopen
struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;

  void load() {
    if (h) return;
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
      if (h) break;
    }
    if (!h) {
      const char *env = getenv("IRKG_NCCL_LIB");
      if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw CudaError(std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char *n) {
      void *p = dlsym(h, n);
      if (!p) throw CudaError(std::string("libnccl missing symbol ") + n);
      return p;
    };
    GetUniqueId = (decltype(GetUniqueId))sym("ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))sym("ncclCommInitRank");
    CommDestroy = (decltype(CommDestroy))sym("ncclCommDestroy");
    AllReduce = (decltype(AllReduce))sym("ncclAllReduce");
    Send = (decltype(Send))sym("ncclSend");
    Recv = (decltype(Recv))sym("ncclRecv");
    GroupStart = (decltype(GroupStart))sym("ncclGroupStart");
    GroupEnd = (decltype(GroupEnd))sym("ncclGroupEnd");
    GetErrorString = (decltype(GetErrorString))sym("ncclGetErrorString");
  }
  void ck(ncclResult_t r, const char *what) {
    if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + GetErrorString(r));
  }
};

static NcclApi g_nccl;

void nccl_unique_id(void *out128) {
  g_nccl.load();
  ncclUniqueId id;
  g_nccl.ck(g_nccl.GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, sizeof id);
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  NcclComm(const void *id128, int rank_, int nranks_) {
    rank = rank_;
    nranks = nranks_;
    g_nccl.load();
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    g_nccl.ck(g_nccl.CommInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm) g_nccl.CommDestroy(comm);
  }
  void allreduce_sum(double *dev, int count, cudaStream_t st) override {
    g_nccl.ck(g_nccl.AllReduce(dev, dev, count, ncclFloat64, ncclSum, comm, st), "ncclAllReduce");
  }
  void halo(const double *send_lo, const double *send_hi, double *recv_lo, double *recv_hi,
            long long count, cudaStream_t st) override {
    const int prev = (rank + nranks - 1) % nranks, next = (rank + 1) % nranks;
    g_nccl.ck(g_nccl.GroupStart(), "ncclGroupStart");
    g_nccl.ck(g_nccl.Send(send_lo, count, ncclFloat64, prev, comm, st), "ncclSend");
    g_nccl.ck(g_nccl.Send(send_hi, count, ncclFloat64, next, comm, st), "ncclSend");
    g_nccl.ck(g_nccl.Recv(recv_hi, count, ncclFloat64, next, comm, st), "ncclRecv");
    g_nccl.ck(g_nccl.Recv(recv_lo, count, ncclFloat64, prev, comm, st), "ncclRecv");
    g_nccl.ck(g_nccl.GroupEnd(), "ncclGroupEnd");
  }
  void halo_batch(int nx, const Xfer *x, cudaStream_t st) override {
    const int prev = (rank + nranks - 1) % nranks, next = (rank + 1) % nranks;
    g_nccl.ck(g_nccl.GroupStart(), "ncclGroupStart");
    for (int i = 0; i < nx; ++i) {
      g_nccl.ck(g_nccl.Send(x[i].send_lo, x[i].count, ncclFloat64, prev, comm, st), "ncclSend");
      g_nccl.ck(g_nccl.Send(x[i].send_hi, x[i].count, ncclFloat64, next, comm, st), "ncclSend");
      g_nccl.ck(g_nccl.Recv(x[i].recv_hi, x[i].count, ncclFloat64, next, comm, st), "ncclRecv");
      g_nccl.ck(g_nccl.Recv(x[i].recv_lo, x[i].count, ncclFloat64, prev, comm, st), "ncclRecv");
    }
    g_nccl.ck(g_nccl.GroupEnd(), "ncclGroupEnd");
  }
  void alltoall(const double *send, double *recv, long long count, cudaStream_t st) override {
    g_nccl.ck(g_nccl.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < nranks; ++p) {
      g_nccl.ck(g_nccl.Send(send + (size_t)p * count, count, ncclFloat64, p, comm, st), "ncclSend");
      g_nccl.ck(g_nccl.Recv(recv + (size_t)p * count, count, ncclFloat64, p, comm, st), "ncclRecv");
    }
    g_nccl.ck(g_nccl.GroupEnd(), "ncclGroupEnd");
  }
  bool capturable() const override { return true; }
};

struct CallbackComm : Comm {
  irkg_allreduce_fn ar;
  irkg_halo_fn hf;
  irkg_alltoall_fn a2a = nullptr;
  void *user;
  CallbackComm(int rank_, int nranks_, irkg_allreduce_fn a, irkg_halo_fn h, void *u)
      : ar(a), hf(h), user(u) {
    rank = rank_;
    nranks = nranks_;
  }
  void allreduce_sum(double *dev, int count, cudaStream_t st) override {
    check(cudaStreamSynchronize(st), "sync");
    ar(user, dev, count);
  }
  void halo(const double *send_lo, const double *send_hi, double *recv_lo, double *recv_hi,
            long long count, cudaStream_t st) override {
    check(cudaStreamSynchronize(st), "sync");
    hf(user, send_lo, send_hi, recv_lo, recv_hi, count);
  }
  void alltoall(const double *send, double *recv, long long count, cudaStream_t st) override {
    if (!a2a)
      throw SolveError(IRKG_ERR_CONFIG,
                       "callback transport without an all-to-all (irkg_set_alltoall_callback)");
    check(cudaStreamSynchronize(st), "sync");
    a2a(user, send, recv, count);
  }
};

void comm_set_alltoall(Comm *c, irkg_alltoall_fn fn) {
  if (auto *cb = dynamic_cast<CallbackComm *>(c)) cb->a2a = fn;
}

Comm *make_nccl_comm(const void *id128, int rank, int nranks) {
  return new NcclComm(id128, rank, nranks);
}
Comm *make_callback_comm(int rank, int nranks, irkg_allreduce_fn a, irkg_halo_fn h, void *u) {
  return new CallbackComm(rank, nranks, a, h, u);
}

// --------------------------------------------------------------- ghost roles

int Engine::plane_size() const { return ndim == 3 ? grid.nxy : grid.nx; }

Engine::Ghost &Engine::role(int r) {
  Ghost &g = ghosts[r];
  if (!g.lo) {
    const size_t bytes = sizeof(double) * (size_t)GH * plane_size();
    check(cudaMalloc((void **)&g.lo, bytes), "cudaMalloc ghost");
    check(cudaMalloc((void **)&g.hi, bytes), "cudaMalloc ghost");
  }
  return g;
}

// fill role r's ghost planes with the neighbours' boundary planes of field f
void Engine::exchange(int r, const double *f, int depth) {
  if (!slab()) return;
  Ghost &g = role(r);
  if (g.field && g.field != f) {
    auto it = owner.find(g.field);
    if (it != owner.end() && it->second == r) owner.erase(it);
  }
  g.field = f;
  owner[f] = r;
  const long long P = plane_size();
  const int nl = local_planes();
  if (depth > GH) depth = GH;
  if (depth > nl) throw SolveError(IRKG_ERR_CONFIG, "slab thinner than the stencil halo");
  comm->halo(f, f + (size_t)(nl - depth) * P, g.lo + (size_t)(GH - depth) * P, g.hi, depth * P,
             stream);
  counters.halo_exchanges += 1;
}

void Engine::allreduce(double *dev, int count) {
  if (!slab()) return;
  comm->allreduce_sum(dev, count, stream);
}

FRef Engine::ref(const double *p) const {
  FRef f{p, nullptr, nullptr};
  if (!slab() || !p) return f;
  auto it = owner.find(p);
  if (it == owner.end())
    throw SolveError(IRKG_ERR_CONFIG, "internal: stencil input without halo exchange");
  const Ghost &g = ghosts.at(it->second);
  f.lo = g.lo;
  f.hi = g.hi;
  return f;
}

Op Engine::opref(const Op &o) const {
  Op r = o;
  if (slab() && o.present && o.a) {
    FRef f = ref(o.a);
    r.alo = f.lo;
    r.ahi = f.hi;
  }
  return r;
}

StageGhosts Engine::stage_ghosts(const double *Ub, long long stride, int nst) const {
  StageGhosts sg{};
  if (!slab()) return sg;
  if (nst < 0) nst = s;
  for (int i = 0; i < nst; ++i) {
    FRef f = ref(Ub + (size_t)i * stride);
    sg.lo[i] = f.lo;
    sg.hi[i] = f.hi;
  }
  return sg;
}

void Engine::free_ghosts() {
  for (auto &kv : ghosts) {
    if (kv.second.lo) cudaFree(kv.second.lo);
    if (kv.second.hi) cudaFree(kv.second.hi);
  }
  ghosts.clear();
  owner.clear();
}

}  // namespace irkg
