// Multi-GPU slab decomposition: one process per GPU, each owning a contiguous z-slab of
// element layers. The node plane between two slabs is held by both ranks and owned by the lower
// one. The matrix-free operator applies the local stencil (the slab's own elements only, so the
// shared planes receive partial sums — the z-face families of stencil.cu are exactly the one-sided
// sums), then adds the neighbour's partial plane (one plane exchanged with each neighbour) and
// re-imposes the unit Dirichlet rows. Dot products run over owned dofs and are summed across
// ranks. The collectives are the only data-path communication: a plane exchange per apply and
// scalar allreduces in the Krylov loop, over NCCL (NVLink/NVSwitch) — or, for single-GPU tests
// of the same algorithm, over a threads backend (several subdomains on one device).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "afem_impl.hpp"
#include "dist.hpp"
#include "reduce.cuh"

namespace afem {

unsigned red_grid(int64_t n);

// ------------------------------------------------------------------ NCCL (dlopen: reuse the copy
// the process already loaded, e.g. torch's, else the system one)
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool loaded = false;
  if (loaded) return api;
  // the process's NCCL if one is loaded (e.g. torch's), else AFEM_NCCL_LIBRARY, else the default
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h && std::getenv("AFEM_NCCL_LIBRARY")) h = dlopen(std::getenv("AFEM_NCCL_LIBRARY"), RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw std::runtime_error(std::string("NCCL unavailable: ") + dlerror());
  auto sym = [&](const char* n) {
    void* f = dlsym(h, n);
    if (!f) throw std::runtime_error(std::string("NCCL symbol missing: ") + n);
    return f;
  };
  api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(sym("ncclGetUniqueId"));
  api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(sym("ncclCommInitRank"));
  api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(sym("ncclCommDestroy"));
  api.allReduce = reinterpret_cast<decltype(api.allReduce)>(sym("ncclAllReduce"));
  api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
  api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
  api.groupStart = reinterpret_cast<decltype(api.groupStart)>(sym("ncclGroupStart"));
  api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(sym("ncclGroupEnd"));
  api.errorString = reinterpret_cast<decltype(api.errorString)>(sym("ncclGetErrorString"));
  loaded = true;
  return api;
}

#define AFEM_NCCL(x)                                                                           \
  do {                                                                                         \
    ncclResult_t r_ = (x);                                                                     \
    if (r_ != ncclSuccess) throw NcclError(std::string("NCCL: ") + nccl().errorString(r_));   \
  } while (0)

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  AFEM_NCCL(nccl().getUniqueId(&id));
  std::memcpy(out, &id, sizeof id);
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  NcclComm(const void* uid, int r, int n) {
    rank = r;
    size = n;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    AFEM_NCCL(nccl().commInitRank(&comm, n, id, r));
  }
  ~NcclComm() override {
    if (comm) nccl().commDestroy(comm);
  }
  void allreduce_sum(double* d, int n, cudaStream_t s) override {
    if (size == 1) return;  // the local sum is the global one
    AFEM_NCCL(nccl().allReduce(d, d, n, ncclFloat64, ncclSum, comm, s));
  }
  void exchange(const double* send_lo, double* recv_lo, const double* send_hi, double* recv_hi, size_t n,
                cudaStream_t s) override {
    AFEM_NCCL(nccl().groupStart());
    if (send_lo) {
      AFEM_NCCL(nccl().send(send_lo, n, ncclFloat64, rank - 1, comm, s));
      AFEM_NCCL(nccl().recv(recv_lo, n, ncclFloat64, rank - 1, comm, s));
    }
    if (send_hi) {
      AFEM_NCCL(nccl().send(send_hi, n, ncclFloat64, rank + 1, comm, s));
      AFEM_NCCL(nccl().recv(recv_hi, n, ncclFloat64, rank + 1, comm, s));
    }
    AFEM_NCCL(nccl().groupEnd());
  }
};

// ------------------------------------------------------------------ threads backend
struct ThreadGroup {
  int n = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<double> vals;
  std::vector<const double*> lo, hi;
  explicit ThreadGroup(int size) : n(size), lo(size, nullptr), hi(size, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> l(m);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(l, [&] { return gen != g; });
    }
  }
};

struct ThreadComm : Comm {
  ThreadGroup* g;
  ThreadComm(ThreadGroup* grp, int r) : g(grp) {
    rank = r;
    size = grp->n;
  }
  void allreduce_sum(double* d, int n, cudaStream_t s) override {
    std::vector<double> h(n);
    AFEM_CK(cudaMemcpyAsync(h.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    AFEM_CK(cudaStreamSynchronize(s));
    {
      std::lock_guard<std::mutex> l(g->m);
      if (g->vals.size() < static_cast<size_t>(g->n * n)) g->vals.resize(g->n * n);
      std::memcpy(&g->vals[rank * n], h.data(), n * sizeof(double));
    }
    g->barrier();
    for (int k = 0; k < n; ++k) {  // fixed rank order: identical on every rank
      double t = 0.0;
      for (int r = 0; r < g->n; ++r) t += g->vals[r * n + k];
      h[k] = t;
    }
    g->barrier();
    AFEM_CK(cudaMemcpyAsync(d, h.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
    AFEM_CK(cudaStreamSynchronize(s));
  }
  void exchange(const double* send_lo, double* recv_lo, const double* send_hi, double* recv_hi, size_t n,
                cudaStream_t s) override {
    AFEM_CK(cudaStreamSynchronize(s));
    g->lo[rank] = send_lo;
    g->hi[rank] = send_hi;
    g->barrier();
    if (recv_lo) AFEM_CK(cudaMemcpyAsync(recv_lo, g->hi[rank - 1], n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    if (recv_hi) AFEM_CK(cudaMemcpyAsync(recv_hi, g->lo[rank + 1], n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    AFEM_CK(cudaStreamSynchronize(s));
    g->barrier();
  }
};

ThreadGroup* thread_group_create(int n) {
  if (n < 1) throw std::invalid_argument("thread group: size must be >= 1");
  return new ThreadGroup(n);
}
void thread_group_destroy(ThreadGroup* g) { delete g; }
Comm* comm_create_nccl(const void* uid, int rank, int size) {
  if (size < 1 || rank < 0 || rank >= size) throw std::invalid_argument("dist: bad rank/size");
  return new NcclComm(uid, rank, size);
}
Comm* comm_create_threads(ThreadGroup* g, int rank) {
  if (!g || rank < 0 || rank >= g->n) throw std::invalid_argument("dist: bad rank for thread group");
  return new ThreadComm(g, rank);
}

// ------------------------------------------------------------------ slab partition
void slab_range(int nz, int size, int rank, int* z0, int* z1) {
  if (size < 1 || rank < 0 || rank >= size) throw std::invalid_argument("slab: bad rank/size");
  if (nz < size) throw std::invalid_argument("slab: fewer element layers than ranks");
  const int base = nz / size, extra = nz % size;  // the first `extra` ranks take one more layer
  *z0 = rank * base + std::min(rank, extra);
  *z1 = *z0 + base + (rank < extra ? 1 : 0);
}

// benchmark_bcs of the global grid restricted to a slab (3D twin of mesh.hpp:89-101).
std::vector<Constraint> slab_benchmark_bcs(const System& s, int rank, int size, double strain, double lx_global) {
  if (!s.grid || s.dim != 3) throw std::invalid_argument("slab bcs: 3D grid system required");
  std::vector<Constraint> c;
  const int nx = s.nx, ny = s.ny, nz = s.nz;
  auto node = [&](int i, int j, int k) { return i + (nx + 1) * (j + (ny + 1) * k); };
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j) c.push_back({node(0, j, k), 0, 0.0});
  if (rank == 0) {
    c.push_back({node(0, 0, 0), 1, 0.0});
    c.push_back({node(0, 0, 0), 2, 0.0});
  }
  if (rank == size - 1) c.push_back({node(0, 0, nz), 1, 0.0});
  const double u_right = strain * lx_global;
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j) c.push_back({node(nx, j, k), 0, u_right});
  return c;
}

// ------------------------------------------------------------------ distributed operator
namespace {

// The received neighbour partial sums added into the two shared node planes of v in one launch
// (index i < np: the bottom plane, else the top plane); constrained rows reset (mode 1: unit
// diagonal, mode 2: x); dot_out != nullptr: the owned top plane's x.v is added to dot_out[0]
// (fixed-order grid reduction; the bottom plane belongs to rank - 1).
__global__ void k_halo_fin(double* __restrict__ v, int64_t n, int64_t np, const double* __restrict__ recv_lo,
                           const double* __restrict__ recv_hi, const double* __restrict__ x,
                           const uint8_t* __restrict__ mask, int mode, double* partials, unsigned* counter,
                           double* dot_out, const int* skip) {
  if (skip && *skip) return;
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * np; i += (int64_t)gridDim.x * blockDim.x) {
    const bool top = i >= np;
    const double* rv = top ? recv_hi : recv_lo;
    if (!rv) continue;
    const int64_t k = top ? i - np : i, d = top ? n - np + k : k;
    double t = v[d] + rv[k];
    if (mode && mask[d]) t = mode == 1 ? 1.0 : x[d];
    v[d] = t;
    if (top && dot_out) s += x[d] * t;
  }
  if (!dot_out) return;
  double a[1] = {s};
  if (grid_reduce<1>(a, partials, counter))
    if (threadIdx.x == 0) dot_out[0] += a[0];
}

}  // namespace

DistMfOp::~DistMfOp() = default;

void DistMfOp::halo_add(double* v, const double* x_for_mask, bool diag_mode) {
  Ctx& c = *sys->ctx;
  if (comm->size == 1) return;
  const int64_t np = plane;
  const bool lo = comm->rank > 0, hi = comm->rank < comm->size - 1;
  double* top = v + (n - np);
  if (lo) copy(c, v, send_lo.p, np);
  if (hi) copy(c, top, send_hi.p, np);
  comm->exchange(lo ? send_lo.p : nullptr, lo ? recv_lo.p : nullptr, hi ? send_hi.p : nullptr,
                 hi ? recv_hi.p : nullptr, static_cast<size_t>(np), c.stream);
  halo_finish(v, x_for_mask, diag_mode);
}

void DistMfOp::halo_finish(double* v, const double* x_for_mask, bool diag_mode, double* dot_out) {
  Ctx& c = *sys->ctx;
  const bool lo = comm->rank > 0, hi = comm->rank < comm->size - 1;
  if (!lo && !hi) return;
  const int mode = diag_mode ? 1 : x_for_mask ? 2 : 0;  // neither: plain assembly of partial sums
  const unsigned g = dot_out ? red_grid(2 * plane) : grid_for(2 * plane, 256, 148 * 4);
  launch(c, k_halo_fin, g, dot_out ? kRedThreads : 256, 0, v, n, plane, lo ? recv_lo.p : nullptr,
         hi ? recv_hi.p : nullptr, x_for_mask, mask(), mode, c.red_partials.p, c.red_counter.p, dot_out,
         dot_out ? skip : nullptr);
}

// Halo exchange overlapped with the interior: the two shared node planes are applied first on a
// second stream (a one-plane launch each, main kernel + their correction items), sent to the
// neighbours from y there (NCCL send/recv), while the interior planes run as one balanced wave on
// the context stream, which then waits for the exchange and adds the received partial sums. The
// boundary launches fit beside the interior wave (a fifth CTA per SM), so the exchange is hidden
// under the interior. Same arithmetic as apply + halo_add. AFEM_DIST_OVERLAP=0: apply, then halo.
void DistMfOp::apply(const double* x, double* y) { apply_impl(x, y, nullptr); }

// Fused owned x.y: the interior wave's stencil dot covers every owned plane but the top shared one,
// whose rows are complete only after the halo add (k_halo_fin adds its share). Needs the overlapped
// stencil schedule (or no neighbours); false otherwise (the caller runs an owned-dot kernel).
bool DistMfOp::apply_dot(const double* x, double* y, double* dot_out) {
  static const char* ov = std::getenv("AFEM_DIST_OVERLAP");
  static const bool overlap = !(ov && ov[0] == '0');
  static const bool force = std::getenv("AFEM_DIST_FORCE_PIECES") != nullptr;
  static const bool disabled = std::getenv("AFEM_NO_FUSED_DOT") != nullptr;
  if (!local || !local->stencil || disabled || force) return false;
  if (comm->size == 1) {
    local->set_skip(skip);
    ScopeExit unset([&] { local->set_skip(nullptr); });
    return local->apply_dot(x, y, dot_out);
  }
  if (!overlap || sys->nz + 1 < 3) return false;
  apply_impl(x, y, dot_out);
  return true;
}

void DistMfOp::apply_impl(const double* x, double* y, double* dot_out) {
  if (!local) {  // assembled: local SpMV (partial sums on the shared planes) + halo
    csr_apply(*sys, vals.p, x, y);
    halo_add(y, x, false);
    return;
  }
  StencilPlan* pl = local->stencil;
  const int nzn = sys->nz + 1;  // node planes of the slab
  static const char* ov = std::getenv("AFEM_DIST_OVERLAP");
  static const bool overlap = !(ov && ov[0] == '0');
  // measurement switch (scripts/dist_apply_probe.py): the split schedule even without neighbours
  static const bool force = std::getenv("AFEM_DIST_FORCE_PIECES") != nullptr;
  if (!pl || nzn < 3 || !overlap || (comm->size == 1 && !force)) {
    local->apply(x, y);
    halo_add(y, x, false);
    return;
  }
  Ctx& c = *sys->ctx;
  const int64_t np = plane;
  const bool lo = comm->rank > 0, hi = comm->rank < comm->size - 1;
  const bool lo_b = lo || force, hi_b = hi || force;
  c.copy_streams(2);
  AFEM_CK(cudaEventRecord(c.events[0], c.stream));
  AFEM_CK(cudaStreamWaitEvent(c.s_in, c.events[0], 0));
  {
    cudaStream_t main_stream = c.stream;
    ScopeExit restore([&] { c.stream = main_stream; });
    c.stream = c.s_in;
    if (lo_b) stencil_apply_planes(*pl, *local, x, y, 0, 1, nullptr, skip);
    if (hi_b) stencil_apply_planes(*pl, *local, x, y, nzn - 1, nzn, nullptr, skip);
    comm->exchange(lo ? y : nullptr, lo ? recv_lo.p : nullptr, hi ? y + (n - np) : nullptr,
                   hi ? recv_hi.p : nullptr, static_cast<size_t>(np), c.s_in);
  }
  AFEM_CK(cudaEventRecord(c.events[1], c.s_in));
  stencil_apply_planes(*pl, *local, x, y, lo_b ? 1 : 0, hi_b ? nzn - 1 : nzn, dot_out, skip);
  AFEM_CK(cudaStreamWaitEvent(c.stream, c.events[1], 0));
  halo_finish(y, x, false, dot_out && hi ? dot_out : nullptr);
}

void DistMfOp::diagonal(double* d) { copy(*sys->ctx, diag.p, d, n); }

std::unique_ptr<DistMfOp> make_dist_mf_op(System& s, Comm* comm, std::unique_ptr<MfOp> local) {
  if (!s.grid || s.dim != 3) throw std::invalid_argument("dist operator: 3D grid (slab) system required");
  auto op = std::make_unique<DistMfOp>();
  op->sys = &s;
  op->kind = 1;
  op->n = s.n_dof;
  op->comm = comm;
  op->plane = static_cast<int64_t>(s.nx + 1) * (s.ny + 1) * 3;
  op->owned_offset = comm->rank > 0 ? op->plane : 0;
  op->send_lo.alloc(op->plane);
  op->recv_lo.alloc(op->plane);
  op->send_hi.alloc(op->plane);
  op->recv_hi.alloc(op->plane);
  op->local = std::move(local);
  op->diag.alloc(s.n_dof);
  op->local->diagonal(op->diag.p);
  op->halo_add(op->diag.p, nullptr, true);  // Jacobi diagonal of the global operator, unit on constraints
  AFEM_CK(cudaStreamSynchronize(s.ctx->stream));
  return op;
}

std::unique_ptr<DistMfOp> make_dist_csr_op(System& s, Comm* comm, const double* d_values) {
  if (!s.grid || s.dim != 3) throw std::invalid_argument("dist operator: 3D grid (slab) system required");
  auto op = std::make_unique<DistMfOp>();
  op->sys = &s;
  op->kind = 0;
  op->n = s.n_dof;
  op->comm = comm;
  op->plane = static_cast<int64_t>(s.nx + 1) * (s.ny + 1) * 3;
  op->owned_offset = comm->rank > 0 ? op->plane : 0;
  op->send_lo.alloc(op->plane);
  op->recv_lo.alloc(op->plane);
  op->send_hi.alloc(op->plane);
  op->recv_hi.alloc(op->plane);
  op->vals.alloc(s.nnz);
  copy(*s.ctx, d_values, op->vals.p, s.nnz);
  op->diag.alloc(s.n_dof);
  csr_diagonal(s, op->vals.p, op->diag.p);
  op->halo_add(op->diag.p, nullptr, true);  // Jacobi diagonal of the global operator, unit on constraints
  AFEM_CK(cudaStreamSynchronize(s.ctx->stream));
  return op;
}

// ------------------------------------------------------------------ distributed CG (krylov.hpp:350-408)
namespace {

// Single-reduction (Chronopoulos-Gear) preconditioned CG: the same iterates as krylov.hpp:350-408
// in exact arithmetic, with the three inner products of an iteration — (r, u), (r, r) and
// (u, w = A u), u = M r — summed across the ranks by ONE allreduce instead of two (p.Ap, then r.r
// and r.z): p = u + beta p, s = w + beta s (s = A p by recurrence), x += alpha p, r -= alpha s,
// with p.Ap = (u, w) - beta gamma / alpha_prev. Stopping rules are the reference's: recurrence
// test on ||r|| / ||b||, p.Ap <= 0 failure, max_iter; the caller re-verifies the true residual.
struct DcgDev {
  double gamma, alpha, denom, rtol;
  double loc[3];  // (r, u), (r, r), (u, w) of the current iterate: partial, then allreduced
  int it, max_iter, done, fail, conv;
  int fresh;  // the next step is the first after a (re)start: beta = 0, p.Ap = (u, w)
};

__global__ void k_owned_dot(const double* a, const double* b, int64_t n, double* partials, unsigned* counter,
                            double* out) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  double v[1] = {s};
  if (grid_reduce<1>(v, partials, counter))
    if (threadIdx.x == 0) out[0] = v[0];
}

// r = b - Ax (all dofs); out = owned sum of r^2
__global__ void k_dres(const double* b, const double* ax, double* r, int64_t n, int64_t off, double* partials,
                       unsigned* counter, double* out) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = b[i] - ax[i];
    if (r) r[i] = d;
    if (i >= off) s += d * d;
  }
  double v[1] = {s};
  if (grid_reduce<1>(v, partials, counter))
    if (threadIdx.x == 0) out[0] = v[0];
}

// start (or restart): u = M r, p = s = 0; loc[0] = owned (r, u), loc[1] = owned (r, r)
__global__ void k_dcg_start(const double* r, const double* inv, double* u, double* p, double* s, int64_t n,
                            int64_t off, double* partials, unsigned* counter, DcgDev* st) {
  double ru = 0.0, rr = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = r[i], z = inv ? ri * inv[i] : ri;
    u[i] = z;
    p[i] = 0.0;
    s[i] = 0.0;
    if (i >= off) {
      ru += ri * z;
      rr += ri * ri;
    }
  }
  double v[2] = {ru, rr};
  if (grid_reduce<2>(v, partials, counter))
    if (threadIdx.x == 0) {
      st->loc[0] = v[0];
      st->loc[1] = v[1];
      st->done = 0;
      st->fail = 0;
      st->conv = 0;
      st->fresh = 1;
    }
}

// One iteration. Preamble (every thread, identical scalars from the allreduced loc): the previous
// iteration's stopping test and the step's beta / alpha; then the fused vector update
//   p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s, u = M r
// with the owned (r, u), (r, r) partials. u is recomputed from r (the same product, so the same
// value the apply read) instead of re-read: 11 vector passes (88 B/dof). The last block (every other block has read st by then)
// commits the scalars: it, gamma, alpha, hist[it], the flags and the new partial sums.
__global__ void k_dcg_step(double* __restrict__ x, double* __restrict__ r, double* __restrict__ u,
                           double* __restrict__ p, double* __restrict__ s, const double* __restrict__ w,
                           const double* __restrict__ inv, int64_t n, int64_t off, double* partials,
                           unsigned* counter, DcgDev* st, double* hist) {
  if (st->done) return;
  const int it = st->it;
  const double gnew = st->loc[0], rr = st->loc[1], delta = st->loc[2];
  const double h = sqrt(rr) / st->denom;
  int stop = 0;  // 1 converged, 2 p.Ap <= 0, 3 max_iter
  double beta = 0.0, pap = delta;
  const bool fresh = st->fresh;  // (re)start: the host has tested this residual already
  if (!fresh) {
    if (h <= st->rtol) stop = 1;
    else if (it >= st->max_iter) stop = 3;
    else {
      beta = gnew / st->gamma;
      pap = delta - beta * gnew / st->alpha;
    }
  }
  if (!stop && !(pap > 0.0)) stop = 2;  // krylov.hpp:377-381
  const double alpha = stop ? 0.0 : gnew / pap;
  double ru = 0.0, rn = 0.0;
  if (!stop)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      const double iv = inv ? inv[i] : 1.0, r0 = r[i];
      const double pi = (inv ? r0 * iv : r0) + beta * p[i], si = w[i] + beta * s[i];  // u = M r, not re-read
      p[i] = pi;
      s[i] = si;
      x[i] += alpha * pi;
      const double ri = r0 - alpha * si, zi = inv ? ri * iv : ri;
      r[i] = ri;
      u[i] = zi;
      if (i >= off) {
        ru += ri * zi;
        rn += ri * ri;
      }
    }
  double v[2] = {ru, rn};
  if (grid_reduce<2>(v, partials, counter) && threadIdx.x == 0) {
    if (!fresh) hist[it] = h;
    st->fresh = 0;
    if (stop) {
      st->done = 1;
      st->conv = stop == 1;
      st->fail = stop == 2;
    } else {
      st->it = it + 1;
      st->gamma = gnew;
      st->alpha = alpha;
      st->loc[0] = v[0];
      st->loc[1] = v[1];
    }
  }
}

__global__ void k_inv(const double* d, double* inv, int64_t n, unsigned long long* first_zero) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (d[i] == 0.0) atomicMin(first_zero, static_cast<unsigned long long>(i));
    inv[i] = 1.0 / d[i];
  }
}

template <class T>
T fetch_dev(Ctx& c, const T* d) {
  T h{};
  AFEM_CK(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  return h;
}

}  // namespace

// Global ||b - A x|| over owned dofs (keeps r when given).
static double dist_residual_norm(DistMfOp& op, const double* b, const double* x, double* scratch, double* r,
                                 double* scal) {
  Ctx& c = *op.sys->ctx;
  op.apply(x, scratch);
  launch(c, k_dres, red_grid(op.n), kRedThreads, 0, b, scratch, r, op.n, op.owned_offset, c.red_partials.p,
         c.red_counter.p, scal);
  op.comm->allreduce_sum(scal, 1, c.stream);
  return std::sqrt(fetch_dev(c, scal));
}

void dist_solve(DistMfOp& op, const SolverCfg& cfg, const double* b, const double* x0, double* x, SolveReport& rep) {
  validate_cfg(cfg);
  if (cfg.method != 0) throw CapabilityError("distributed run_solver: CG, GMRES or BiCGStab");
  if (cfg.precond != 0 && cfg.precond != 1) throw CapabilityError("distributed run_solver: NONE or JACOBI");
  const auto t0 = std::chrono::steady_clock::now();
  Ctx& c = *op.sys->ctx;
  const int64_t n = op.n, off = op.owned_offset;
  const unsigned rg = red_grid(n), eg = grid_for(n, 256, 148 * 16);
  DevArray<double> inv, r(n), u(n), w(n), p(n), sv(n), scratch(n), hist(cfg.max_iter + 2), scal(4);
  if (cfg.precond == 1) {
    inv.alloc(n);
    DevArray<unsigned long long> fz(1);
    const unsigned long long init = ~0ull;
    AFEM_CK(cudaMemcpyAsync(fz.p, &init, 8, cudaMemcpyHostToDevice, c.stream));
    launch(c, k_inv, eg, 256, 0, op.diag.p, inv.p, n, fz.p);
    const unsigned long long z = fetch_dev(c, fz.p);
    if (z != ~0ull) throw FactorizationError("jacobi: zero diagonal at local row " + std::to_string(z));
  }
  if (x0) copy(c, x0, x, n);
  else fill(c, 0.0, x, n);
  // ||b|| over owned dofs, summed across ranks
  launch(c, k_owned_dot, rg, kRedThreads, 0, b + off, b + off, n - off, c.red_partials.p, c.red_counter.p, scal.p);
  op.comm->allreduce_sum(scal.p, 1, c.stream);
  const double bnorm = std::sqrt(fetch_dev(c, scal.p));
  const double denom = bnorm > 0.0 ? bnorm : 1.0;
  rep.history.assign(1, dist_residual_norm(op, b, x, w.p, r.p, scal.p) / denom);
  DevArray<DcgDev> st(1);
  DcgDev hs{};
  hs.denom = denom;
  hs.rtol = cfg.rtol;
  hs.max_iter = cfg.max_iter;
  hs.done = 1;
  AFEM_CK(cudaMemcpyAsync(st.p, &hs, sizeof hs, cudaMemcpyHostToDevice, c.stream));
  double* loc = reinterpret_cast<double*>(reinterpret_cast<char*>(st.p) + offsetof(DcgDev, loc));
  const int* done_dev = reinterpret_cast<const int*>(reinterpret_cast<const char*>(st.p) + offsetof(DcgDev, done));
  // w = A u with the owned (u, w) into loc[2]: fused into the stencil apply where the operator can
  auto apply_uw = [&] {
    if (!op.apply_dot(u.p, w.p, loc + 2)) {
      op.apply(u.p, w.p);
      launch(c, k_owned_dot, rg, kRedThreads, 0, u.p + off, w.p + off, n - off, c.red_partials.p, c.red_counter.p,
             loc + 2);
    }
    op.comm->allreduce_sum(loc, 3, c.stream);  // the iteration's one collective
  };
  ScopeExit unset([&] { op.set_skip(nullptr); });
  while (true) {
    if (rep.history.back() > cfg.rtol && rep.iterations < cfg.max_iter) {
      const int it0 = rep.iterations;
      hs.it = it0;
      AFEM_CK(cudaMemcpyAsync(reinterpret_cast<char*>(st.p) + offsetof(DcgDev, it), &hs.it, sizeof(int),
                              cudaMemcpyHostToDevice, c.stream));
      launch(c, k_dcg_start, rg, kRedThreads, 0, r.p, inv.p, u.p, p.p, sv.p, n, off, c.red_partials.p,
             c.red_counter.p, st.p);
      op.set_skip(done_dev);  // chunk iterations past convergence skip the apply
      apply_uw();
      int chunk = 4;
      while (true) {
        for (int k = 0; k < chunk; ++k) {
          launch(c, k_dcg_step, rg, kRedThreads, 0, x, r.p, u.p, p.p, sv.p, w.p, inv.p, n, off, c.red_partials.p,
                 c.red_counter.p, st.p, hist.p);
          apply_uw();
        }
        hs = fetch_dev(c, st.p);
        if (hs.done) break;
        chunk = std::min(chunk * 2, 64);
      }
      op.set_skip(nullptr);
      rep.iterations = hs.it;
      if (hs.it > it0) {
        rep.history.resize(hs.it + 1);
        AFEM_CK(cudaMemcpyAsync(rep.history.data() + it0 + 1, hist.p + it0 + 1, (hs.it - it0) * sizeof(double),
                                cudaMemcpyDeviceToHost, c.stream));
        AFEM_CK(cudaStreamSynchronize(c.stream));
      }
      if (hs.fail)
        rep.failure = "cg: operator not positive definite (p^T A p <= 0 at iteration " +
                      std::to_string(rep.iterations + 1) + ")";
    }
    const double true_rres = dist_residual_norm(op, b, x, scratch.p, nullptr, scal.p) / denom;
    rep.history.back() = true_rres;
    if (true_rres <= cfg.rtol) {
      rep.converged = rep.failure.empty();
      break;
    }
    if (!rep.failure.empty() || rep.iterations >= cfg.max_iter) break;
    dist_residual_norm(op, b, x, w.p, r.p, scal.p);  // recurrence drifted: restart (krylov.hpp:402-404)
  }
  AFEM_CK(cudaStreamSynchronize(c.stream));
  rep.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Global owned dot (tests / drivers).
double dist_dot(DistMfOp& op, const double* a, const double* b) {
  Ctx& c = *op.sys->ctx;
  DevArray<double> s(1);
  const int64_t off = op.owned_offset;
  launch(c, k_owned_dot, red_grid(op.n - off), kRedThreads, 0, a + off, b + off, op.n - off, c.red_partials.p,
         c.red_counter.p, s.p);
  op.comm->allreduce_sum(s.p, 1, c.stream);
  return fetch_dev(c, s.p);
}

double DistMfOp::inner(const double* a, const double* b) { return dist_dot(*this, a, b); }

void DistMfOp::inner_dev(const double* a, const double* b, double* out_dev) {
  Ctx& c = *sys->ctx;
  launch(c, k_owned_dot, red_grid(n - owned_offset), kRedThreads, 0, a + owned_offset, b + owned_offset,
         n - owned_offset, c.red_partials.p, c.red_counter.p, out_dev);
  comm->allreduce_sum(out_dev, 1, c.stream);
}

double DistMfOp::resid(const double* b, const double* x, double* scratch, double* r) {
  Ctx& c = *sys->ctx;
  apply(x, scratch);
  DevArray<double> s(1);
  launch(c, k_dres, red_grid(n), kRedThreads, 0, b, scratch, r, n, owned_offset, c.red_partials.p, c.red_counter.p,
         s.p);
  comm->allreduce_sum(s.p, 1, c.stream);
  return std::sqrt(fetch_dev(c, s.p));
}

}  // namespace afem
