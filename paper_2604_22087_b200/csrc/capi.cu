// extern "C" boundary (include/afem.h): handle management, host/device pointer staging, exception
// -> status mapping, the lease protocol (backend.hpp:26-111) and the Newton drivers
// (newton.hpp:59-186).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "../../include/afem.h"
#include "../../include/afem_testing.h"
#include "afem_impl.hpp"
#include "dist.hpp"

struct afem_ctx_s {
  afem::Ctx c;
};
struct afem_system_s {
  std::unique_ptr<afem::System> s;
};
struct afem_values_s {
  afem::Values v;
};
struct afem_buffer_s {
  afem::Buffer b;
};
struct afem_op_s {
  std::unique_ptr<afem::Operator> op;
};
struct afem_dist_s {
  afem::Ctx* ctx = nullptr;
  std::unique_ptr<afem::Comm> comm;
};
struct afem_thread_group_s {
  afem::ThreadGroup* g = nullptr;
};

namespace afem {

void scal(Ctx& c, double a, double* y, int64_t n);

// ------------------------------------------------------------------ operators
void ExplicitOp::validate() const {  // backend.hpp:176-181
  if (buf->state != 1) throw LeaseError("explicit operator used while the buffer lease is not held");
  if (buf->epoch != epoch) throw StaleEpochError("explicit operator built from a stale assembly epoch");
}
void ExplicitOp::apply(const double* x, double* y) { csr_apply(*sys, buf->store.p, x, y, skip); }
void ExplicitOp::diagonal(double* d) { csr_diagonal(*sys, buf->store.p, d); }

MfOp::~MfOp() { destroy_stencil_plan(stencil); }
void MfOp::apply(const double* x, double* y) {
  if (stencil) stencil_apply(*stencil, *this, x, y, nullptr, skip);
  else if (qpt.p) grid_mf_apply_cached(*sys, qpt.p, mask.p, x, y, skip);
  else mf_apply_general(*sys, state.p, mask.p, x, y);
}
bool MfOp::apply_dot(const double* x, double* y, double* dot_out) {
  static const bool disabled = std::getenv("AFEM_NO_FUSED_DOT") != nullptr;
  if (disabled) return false;
  if (stencil) stencil_apply(*stencil, *this, x, y, dot_out, skip);
  else if (qpt.p) grid_mf_apply_cached(*sys, qpt.p, mask.p, x, y, skip, dot_out);  // dot fused into the gather
  else if (grid_elem_path(*sys)) grid_mf_apply(*sys, state.p, mask.p, x, y, dot_out);  // (any law on a grid)
  else return false;
  return true;
}
void MfOp::diagonal(double* d) { copy(*sys->ctx, diag.p, d, n); }

__global__ void k_unit_on_mask(const uint8_t* mask, double* d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (mask[i]) d[i] = 1.0;
}

__global__ void k_scal(double a, double* y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] *= a;
}

void scal(Ctx& c, double a, double* y, int64_t n) { launch(c, k_scal, grid_for(n, 256, 148 * 16), 256, 0, a, y, n); }

// FP64 FMA throughput probe: 8 independent DFMA chains per thread (the roofline denominator for
// FP64-bound kernels; MEASURED_PEAKS.json only carries HBM and bf16 peaks).
__global__ void __launch_bounds__(256) k_dfma_probe(double* out, int iters, double a, double b) {
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = fma(r[k], a, b);
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

double probe_fp64(Ctx& c) {
  DevArray<double> o(1);
  const int iters = 4096, blocks = c.num_sms * 8;
  cudaEvent_t e0, e1;
  AFEM_CK(cudaEventCreate(&e0));
  AFEM_CK(cudaEventCreate(&e1));
  launch(c, k_dfma_probe, blocks, 256, 0, o.p, iters, 0.999999, 1e-7);  // warm-up
  AFEM_CK(cudaEventRecord(e0, c.stream));
  const int reps = 5;
  for (int r = 0; r < reps; ++r) launch(c, k_dfma_probe, blocks, 256, 0, o.p, iters, 0.999999, 1e-7);
  AFEM_CK(cudaEventRecord(e1, c.stream));
  AFEM_CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  AFEM_CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = 2.0 * 8.0 * iters * 256.0 * blocks * reps;
  return flops / (ms * 1e-3) / 1e12;
}

// matrix_free_operator (backend.hpp:222-236)
std::unique_ptr<MfOp> make_mf_op(System& s, const double* d_u) {
  auto op = std::make_unique<MfOp>();
  op->sys = &s;
  op->kind = 1;
  op->n = s.n_dof;
  op->state.alloc(s.n_dof);
  copy(*s.ctx, d_u, op->state.p, s.n_dof);
  op->mask.alloc(s.n_dof);
  AFEM_CK(cudaMemcpyAsync(op->mask.p, s.mask.p, s.n_dof, cudaMemcpyDeviceToDevice, s.ctx->stream));
  op->diag.alloc(s.n_dof);
  diagonal(s, op->state.p, op->diag.p);  // validates the state (detJ, det F) like the reference's AD pass
  launch(*s.ctx, k_unit_on_mask, grid_for(s.n_dof, 256, 148 * 16), 256, 0, op->mask.p, op->diag.p, s.n_dof);
  op->stencil = make_stencil_plan(s, *op);
  if (!op->stencil && grid_tangent_cacheable(s)) grid_tangent_cache(s, op->state.p, op->qpt);
  return op;
}

}  // namespace afem

namespace {

using namespace afem;

thread_local std::string g_err;

template <class F>
afem_status guarded(F&& f) {
  try {
    f();
    return AFEM_OK;
  } catch (const LeaseError& e) { g_err = e.what(); return AFEM_E_LEASE;
  } catch (const StaleEpochError& e) { g_err = e.what(); return AFEM_E_STALE_EPOCH;
  } catch (const CapabilityError& e) { g_err = e.what(); return AFEM_E_CAPABILITY;
  } catch (const FactorizationError& e) { g_err = e.what(); return AFEM_E_FACTORIZATION;
  } catch (const InvertedElementError& e) { g_err = e.what(); return AFEM_E_INVERTED_ELEMENT;
  } catch (const CudaError& e) { g_err = e.what(); return AFEM_E_CUDA;
  } catch (const NcclError& e) { g_err = e.what(); return AFEM_E_NCCL;
  } catch (const NomemError& e) { g_err = e.what(); return AFEM_E_NOMEM;
  } catch (const std::invalid_argument& e) { g_err = e.what(); return AFEM_E_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) { g_err = e.what(); return AFEM_E_OUT_OF_RANGE;
  } catch (const std::domain_error& e) { g_err = e.what(); return AFEM_E_DOMAIN;
  } catch (const std::logic_error& e) { g_err = e.what(); return AFEM_E_LOGIC;
  } catch (const std::bad_alloc& e) { g_err = e.what(); return AFEM_E_NOMEM;
  } catch (const std::exception& e) { g_err = e.what(); return AFEM_E_RUNTIME;
  } catch (...) { g_err = "unknown error"; return AFEM_E_RUNTIME; }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null argument: ") + what);
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Read-only argument: device pointer used in place; host data staged in (grow-only ctx buffers).
template <class T>
struct In {
  const T* d = nullptr;
  In(Ctx& c, const T* p, size_t n) {
    if (!p) return;
    if (is_device_ptr(p)) { d = p; return; }
    T* buf = static_cast<T*>(c.stage(n * sizeof(T)));
    if (n) AFEM_CK(cudaMemcpyAsync(buf, p, n * sizeof(T), cudaMemcpyHostToDevice, c.stream));
    d = buf;
  }
};

// Written argument (optionally read first): staged out on finish().
template <class T>
struct Out {
  T* d = nullptr;
  T* host = nullptr;
  size_t n = 0;
  Ctx* c;
  Out(Ctx& cc, T* p, size_t count, bool read_first) : n(count), c(&cc) {
    if (!p) return;
    if (is_device_ptr(p)) { d = p; return; }
    host = p;
    T* buf = static_cast<T*>(c->stage(n * sizeof(T)));
    if (read_first && n) AFEM_CK(cudaMemcpyAsync(buf, p, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    d = buf;
  }
  void finish() {
    if (host && n) AFEM_CK(cudaMemcpyAsync(host, d, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
    AFEM_CK(cudaStreamSynchronize(c->stream));
  }
};

// Start of an ABI call on a context: select the device, recycle the staging slots.
Ctx& begin(Ctx& c) {
  AFEM_CK(cudaSetDevice(c.device));
  c.staging_next = 0;
  return c;
}

System& SYS(afem_system s) {
  need(s, "system");
  begin(*s->s->ctx);
  return *s->s;
}

std::vector<DMat> to_dmats(int32_t n, const afem_material* m) {
  if (n < 0 || (n > 0 && !m)) throw std::invalid_argument("materials: bad table");
  std::vector<DMat> out;
  for (int i = 0; i < n; ++i) out.push_back(make_dmat(m[i].model, m[i].E, m[i].nu, m[i].sigma_y, m[i].hardening));
  return out;
}

SolverCfg to_cfg(const afem_solver_cfg* c) {
  SolverCfg s;
  s.method = c->method;
  s.precond = c->precond;
  s.rtol = c->rtol;
  s.max_iter = c->max_iter;
  s.restart = c->restart;
  return s;
}

void fill_report(const SolveReport& r, afem_solve_report* out, double* hist, int32_t cap) {
  if (!out) return;
  out->converged = r.converged;
  out->iterations = r.iterations;
  out->n_history = static_cast<int32_t>(r.history.size());
  out->wall_time = r.wall_time;
  std::snprintf(out->failure, sizeof out->failure, "%s", r.failure.c_str());
  if (hist)
    for (int32_t i = 0; i < cap && i < out->n_history; ++i) hist[i] = r.history[i];
}

struct NewtonReport {
  bool converged = false;
  int iterations = 0;
  std::vector<double> norms;
  std::vector<SolveReport> linear;
  double total_time = 0.0;
  std::string failure;
};

void validate_newton(const afem_newton_cfg* cfg) {  // NewtonConfig::validate (newton.hpp:27-32)
  if (!(cfg->rtol > 0.0) || !(cfg->atol > 0.0)) throw std::invalid_argument("newton config: tolerances must be > 0");
  if (cfg->max_iter < 1) throw std::invalid_argument("newton config: max_iter must be >= 1");
  validate_cfg(to_cfg(&cfg->linear));
}

// solve_bvp (newton.hpp:59-152); u is a device array of n_dof (in: initial guess, out: solution).
void newton(System& s, const afem_newton_cfg* cfg, double* u, NewtonReport& rep) {
  validate_newton(cfg);
  Ctx& c = *s.ctx;
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t n = s.n_dof;
  impose_dirichlet(s, u);
  DevArray<double> R(n), rhs(n), du(n), vals;
  Buffer buf;
  buf.sys = &s;
  residual(s, u, R.p);
  double rnorm = free_norm(c, R.p, s.mask.p, n);
  const double r0 = rnorm;
  rep.norms.push_back(rnorm);
  const double target = std::max(cfg->rtol * r0, cfg->atol);
  const SolverCfg lcfg = to_cfg(&cfg->linear);
  while (true) {
    if (!std::isfinite(rnorm)) {
      rep.failure = "newton: non-finite residual norm at iteration " + std::to_string(rep.iterations);
      break;
    }
    if (rnorm <= target) {
      rep.converged = true;
      break;
    }
    if (rep.iterations >= cfg->max_iter) {
      rep.failure = "newton: no convergence within " + std::to_string(cfg->max_iter) + " iterations (residual " +
                    std::to_string(rnorm) + ")";
      break;
    }
    copy(c, R.p, rhs.p, n);
    SolveReport lin;
    if (cfg->operator_kind == 0) {
      if (!buf.store.p) buf.store.alloc(s.nnz);
      jacobian(s, u, buf.store.p);
      eliminate(s, buf.store.p, rhs.p, u);
      scal(c, -1.0, rhs.p, n);
      buf.state = 1;  // handoff (backend.hpp:50-66): values stay in place, epoch advances
      ++buf.epoch;
      ExplicitOp op;
      op.sys = &s;
      op.kind = 0;
      op.n = n;
      op.buf = &buf;
      op.epoch = buf.epoch;
      solve(op, lcfg, rhs.p, nullptr, du.p, lin);
      buf.state = 0;  // LeaseGuard release
    } else {
      constrain_residual(s, rhs.p, u);
      scal(c, -1.0, rhs.p, n);
      auto op = make_mf_op(s, u);
      solve(*op, lcfg, rhs.p, nullptr, du.p, lin);
    }
    rep.linear.push_back(lin);
    if (!lin.converged) {
      rep.failure = "newton: linear solve failed at iteration " + std::to_string(rep.iterations + 1) +
                    (lin.failure.empty() ? " (tolerance not reached)" : " (" + lin.failure + ")");
      break;
    }
    axpy(c, 1.0, du.p, u, n);
    impose_dirichlet(s, u);
    residual(s, u, R.p);
    rnorm = free_norm(c, R.p, s.mask.p, n);
    ++rep.iterations;
    rep.norms.push_back(rnorm);
  }
  AFEM_CK(cudaStreamSynchronize(c.stream));
  rep.total_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

__global__ void k_zero_masked(const uint8_t* mask, const double* v, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = mask[i] ? 0.0 : v[i];
}

// run_solver (backend.hpp:241-286) over a slab operator: CG runs the distributed device-scalar PCG
// loop; GMRES and BiCGStab run the single-GPU methods over the operator's owned-dof inner products
// (one allreduce each). Preconditioners: NONE or JACOBI. Collective.
void dist_run_solver(DistMfOp& op, const SolverCfg& sc, const double* b, const double* x0, double* x,
                     SolveReport& r) {
  if (sc.method == 1 || sc.method == 2) {
    if (sc.precond != 0 && sc.precond != 1) throw CapabilityError("distributed run_solver: NONE or JACOBI");
    solve(op, sc, b, x0, x, r);
  } else {
    dist_solve(op, sc, b, x0, x, r);
  }
}

// solve_bvp (newton.hpp:59-152) over a z-slab decomposition: each rank holds its slab's u (shared
// node planes duplicated and kept identical); the residual's shared planes are summed over the
// neighbours, the free norm is a global dot over owned dofs, and each Newton step solves the
// distributed tangent system — matrix-free, or (EXPLICIT) every slab's own assembled and eliminated
// tangent with the same plane halo — with the configured Krylov method (dist_run_solver).
// Collective: every rank calls it.
void dist_newton(System& s, Comm* comm, const afem_newton_cfg* cfg, double* u, NewtonReport& rep) {
  validate_newton(cfg);
  Ctx& c = *s.ctx;
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t n = s.n_dof;
  const unsigned eg = grid_for(n, 256, 148 * 16);
  impose_dirichlet(s, u);
  DevArray<double> R(n), rhs(n), du(n), Rm(n);
  // tangent operator at u: matrix-free, or (EXPLICIT) each slab's assembled tangent eliminated on
  // the slab (assemble_jacobian + apply_dirichlet, newton.hpp:93-104) with the plane halo
  const bool explicit_op = cfg->operator_kind == 0;
  DevArray<double> vals, scratch;
  if (explicit_op) {
    vals.alloc(s.nnz);
    scratch.alloc(n);
  }
  auto tangent = [&]() -> std::unique_ptr<DistMfOp> {
    if (!explicit_op) return make_dist_mf_op(s, comm, make_mf_op(s, u));
    jacobian(s, u, vals.p);
    fill(c, 0.0, scratch.p, n);
    eliminate(s, vals.p, scratch.p, u);  // u satisfies the constraints: only the matrix changes
    return make_dist_csr_op(s, comm, vals.p);
  };
  std::unique_ptr<DistMfOp> op = tangent();
  auto global_residual = [&]() -> double {
    residual(s, u, R.p);
    op->halo_add(R.p, nullptr, false);  // sum the shared planes' partial sums
    launch(c, k_zero_masked, eg, 256, 0, s.mask.p, R.p, Rm.p, n);
    return std::sqrt(dist_dot(*op, Rm.p, Rm.p));  // free_norm (newton.hpp:46-51), owned dofs
  };
  double rnorm = global_residual();
  const double r0 = rnorm;
  rep.norms.push_back(rnorm);
  const double target = std::max(cfg->rtol * r0, cfg->atol);
  const SolverCfg lcfg = to_cfg(&cfg->linear);
  while (true) {
    if (!std::isfinite(rnorm)) {
      rep.failure = "newton: non-finite residual norm at iteration " + std::to_string(rep.iterations);
      break;
    }
    if (rnorm <= target) {
      rep.converged = true;
      break;
    }
    if (rep.iterations >= cfg->max_iter) {
      rep.failure = "newton: no convergence within " + std::to_string(cfg->max_iter) + " iterations (residual " +
                    std::to_string(rnorm) + ")";
      break;
    }
    copy(c, R.p, rhs.p, n);
    constrain_residual(s, rhs.p, u);
    scal(c, -1.0, rhs.p, n);
    SolveReport lin;
    dist_run_solver(*op, lcfg, rhs.p, nullptr, du.p, lin);
    rep.linear.push_back(lin);
    if (!lin.converged) {
      rep.failure = "newton: linear solve failed at iteration " + std::to_string(rep.iterations + 1) +
                    (lin.failure.empty() ? " (tolerance not reached)" : " (" + lin.failure + ")");
      break;
    }
    axpy(c, 1.0, du.p, u, n);
    impose_dirichlet(s, u);
    op = tangent();
    rnorm = global_residual();
    ++rep.iterations;
    rep.norms.push_back(rnorm);
  }
  AFEM_CK(cudaStreamSynchronize(c.stream));
  rep.total_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void fill_newton(const NewtonReport& r, afem_newton_report* out, double* norms, int32_t cap) {
  if (!out) return;
  out->converged = r.converged;
  out->iterations = r.iterations;
  out->n_norms = static_cast<int32_t>(r.norms.size());
  int tot = 0;
  for (const auto& l : r.linear) tot += l.iterations;
  out->total_linear_iterations = tot;
  out->total_time = r.total_time;
  std::snprintf(out->failure, sizeof out->failure, "%s", r.failure.c_str());
  if (norms)
    for (int32_t i = 0; i < cap && i < out->n_norms; ++i) norms[i] = r.norms[i];
}

}  // namespace

extern "C" {

const char* afem_last_error(void) { return g_err.c_str(); }
int32_t afem_abi_version(void) { return AFEM_ABI_VERSION; }

afem_status afem_ctx_create(int32_t device, afem_ctx* out) {
  return guarded([&] {
    need(out, "out");
    auto c = std::make_unique<afem_ctx_s>();
    AFEM_CK(cudaSetDevice(device));
    c->c.device = device;
    AFEM_CK(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
    c->c.own_stream = true;
    AFEM_CK(cudaDeviceGetAttribute(&c->c.num_sms, cudaDevAttrMultiProcessorCount, device));
    c->c.red_partials.alloc(kRedBlocks * 4);
    c->c.red_out.alloc(64);
    c->c.red_counter.alloc(1);
    AFEM_CK(cudaMemsetAsync(c->c.red_counter.p, 0, sizeof(unsigned), c->c.stream));
    AFEM_CK(cudaStreamSynchronize(c->c.stream));
    *out = c.release();
  });
}

afem_status afem_ctx_destroy(afem_ctx ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    ctx->c.release_copy_streams();
    ctx->c.release_graph_resources();
    if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
    delete ctx;
  });
}

afem_status afem_ctx_set_stream(afem_ctx ctx, void* stream) {
  return guarded([&] {
    need(ctx, "ctx");
    AFEM_CK(cudaStreamSynchronize(ctx->c.stream));
    if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
    ctx->c.own_stream = false;
    ctx->c.stream = static_cast<cudaStream_t>(stream);
  });
}

afem_status afem_ctx_synchronize(afem_ctx ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    AFEM_CK(cudaStreamSynchronize(ctx->c.stream));
  });
}

afem_status afem_ctx_launch_count(afem_ctx ctx, int64_t* count) {
  return guarded([&] {
    need(ctx, "ctx");
    *count = ctx->c.launches;
  });
}

afem_status afem_probe_fp64(afem_ctx ctx, double* tflops) {
  return guarded([&] {
    need(ctx, "ctx");
    need(tflops, "tflops");
    *tflops = probe_fp64(begin(ctx->c));
  });
}

afem_status afem_fibres(uint64_t seed, int32_t n, double lx, double ly, double* out) {
  return guarded([&] {
    need(out, "out");
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> ux(0.0, lx), uy(0.0, ly);
    for (int i = 0; i < n; ++i) {
      const double x = ux(rng);
      const double y = uy(rng);
      out[2 * i] = x;
      out[2 * i + 1] = y;
    }
  });
}

afem_status afem_system_create(afem_ctx ctx, int32_t dim, int64_t n_nodes, int64_t n_elem, const double* coords,
                               const int32_t* conn, const int32_t* phase, int32_t n_mat, const afem_material* mats,
                               afem_system* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    need(coords, "coords");
    need(conn, "conn");
    need(phase, "phase");
    Ctx& c = begin(ctx->c);
    if (dim != 2 && dim != 3) throw std::invalid_argument("system: dim must be 2 (quad4) or 3 (hex8)");
    const int npe = dim == 2 ? 4 : 8;
    In<double> dc(c, coords, n_nodes * dim);
    In<int32_t> dn(c, conn, n_elem * npe), dp(c, phase, n_elem);
    auto s = std::make_unique<afem_system_s>();
    s->s = make_system(c, dim, n_nodes, n_elem, dc.d, dn.d, dp.d, to_dmats(n_mat, mats));
    *out = s.release();
  });
}

afem_status afem_system_create_grid(afem_ctx ctx, int32_t dim, int32_t nx, int32_t ny, int32_t nz, double lx,
                                    double ly, double lz, int32_t n_incl, const double* incl_xy, double radius,
                                    int32_t n_mat, const afem_material* mats, afem_system* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(out, "out");
    if (n_incl < 0 || (n_incl > 0 && !incl_xy)) throw std::invalid_argument("mesh: bad inclusion list");
    Ctx& c = begin(ctx->c);
    std::vector<double> incl(incl_xy, incl_xy + 2 * n_incl);
    auto s = std::make_unique<afem_system_s>();
    s->s = make_grid_system(c, dim, nx, ny, nz, lx, ly, lz, incl, radius, to_dmats(n_mat, mats));
    *out = s.release();
  });
}

afem_status afem_system_destroy(afem_system sys) {
  return guarded([&] {
    if (!sys) return;
    cudaSetDevice(sys->s->ctx->device);
    cudaStreamSynchronize(sys->s->ctx->stream);
    delete sys;
  });
}

afem_status afem_system_get_info(afem_system sys, afem_system_info* out) {
  return guarded([&] {
    System& s = SYS(sys);
    need(out, "out");
    out->dim = s.dim;
    out->nodes_per_elem = s.npe;
    out->n_nodes = s.n_nodes;
    out->n_elem = s.n_elem;
    out->n_dof = s.n_dof;
    out->nnz = s.nnz;
    out->n_batches = static_cast<int32_t>(std::count_if(s.phase_count.begin(), s.phase_count.end(),
                                                        [](int64_t k) { return k > 0; }));
    out->structured = s.grid ? 1 : 0;
    out->nx = s.nx;
    out->ny = s.ny;
    out->nz = s.nz;
    out->device_bytes = s.device_bytes();
  });
}

__global__ void k_phase_to_i32(const uint8_t* a, int32_t* b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

afem_status afem_system_mesh(afem_system sys, double* coords, int32_t* conn, int32_t* phase) {
  return guarded([&] {
    System& s = SYS(sys);
    Ctx& c = *s.ctx;
    if (coords) {
      Out<double> o(c, coords, s.coords.n, false);
      copy(c, s.coords.p, o.d, s.coords.n);
      o.finish();
    }
    if (conn) {
      Out<int32_t> o(c, conn, s.conn.n, false);
      AFEM_CK(cudaMemcpyAsync(o.d, s.conn.p, s.conn.bytes(), cudaMemcpyDeviceToDevice, c.stream));
      o.finish();
    }
    if (phase) {
      Out<int32_t> o(c, phase, s.n_elem, false);
      launch(c, k_phase_to_i32, grid_for(s.n_elem, 256, 148 * 16), 256, 0, s.phase.p, o.d, s.n_elem);
      o.finish();
    }
  });
}

afem_status afem_system_batch(afem_system sys, int32_t b, int64_t* size, int32_t* ids, int32_t* dof_map) {
  return guarded([&] {
    System& s = SYS(sys);
    need(size, "size");
    batch_export(s, b, size, ids, dof_map);
  });
}

afem_status afem_set_dirichlet(afem_system sys, int64_t n, const int32_t* node, const int32_t* comp,
                               const double* value) {
  return guarded([&] {
    System& s = SYS(sys);
    if (n < 0 || (n > 0 && (!node || !comp || !value))) throw std::invalid_argument("dirichlet: bad arrays");
    std::vector<Constraint> cs(n);
    for (int64_t i = 0; i < n; ++i) cs[i] = Constraint{node[i], comp[i], value[i]};
    set_dirichlet(s, cs);
  });
}

afem_status afem_set_benchmark_dirichlet(afem_system sys, double strain) {
  return guarded([&] {
    System& s = SYS(sys);
    set_dirichlet(s, benchmark_bcs(s, strain));
  });
}

afem_status afem_impose_dirichlet(afem_system sys, double* u) {
  return guarded([&] {
    System& s = SYS(sys);
    need(u, "u");
    Out<double> o(*s.ctx, u, s.n_dof, true);
    impose_dirichlet(s, o.d);
    o.finish();
  });
}

afem_status afem_pattern_nnz(afem_system sys, int64_t* nnz) {
  return guarded([&] {
    System& s = SYS(sys);
    need(nnz, "nnz");
    *nnz = s.nnz;
  });
}

afem_status afem_pattern(afem_system sys, int64_t* row_ptr, int32_t* rows, int32_t* cols) {
  return guarded([&] {
    System& s = SYS(sys);
    Ctx& c = *s.ctx;
    Out<int64_t> rp(c, row_ptr, s.n_dof + 1, false);
    Out<int32_t> rw(c, rows, s.nnz, false), cl(c, cols, s.nnz, false);
    if (rp.d && s.n_nodes > 0) AFEM_CK(cudaMemsetAsync(rp.d, 0, sizeof(int64_t), c.stream));
    pattern_export(s, rp.d, rw.d, cl.d);
    rp.finish();
    rw.finish();
    cl.finish();
  });
}

afem_status afem_residual(afem_system sys, const double* u, double* r) {
  return guarded([&] {
    System& s = SYS(sys);
    need(u, "u");
    need(r, "r");
    In<double> du(*s.ctx, u, s.n_dof);
    Out<double> o(*s.ctx, r, s.n_dof, false);
    residual(s, du.d, o.d);
    o.finish();
  });
}

afem_status afem_jacobian(afem_system sys, const double* u, double* values) {
  return guarded([&] {
    System& s = SYS(sys);
    need(u, "u");
    need(values, "values");
    In<double> du(*s.ctx, u, s.n_dof);
    Out<double> o(*s.ctx, values, s.nnz, false);
    jacobian(s, du.d, o.d);
    o.finish();
  });
}

afem_status afem_diagonal(afem_system sys, const double* u, double* d) {
  return guarded([&] {
    System& s = SYS(sys);
    need(u, "u");
    need(d, "d");
    In<double> du(*s.ctx, u, s.n_dof);
    Out<double> o(*s.ctx, d, s.n_dof, false);
    diagonal(s, du.d, o.d);
    o.finish();
  });
}

afem_status afem_eliminate(afem_system sys, double* values, double* res, const double* u) {
  return guarded([&] {
    System& s = SYS(sys);
    need(values, "values");
    need(res, "residual");
    need(u, "u");
    In<double> du(*s.ctx, u, s.n_dof);
    Out<double> v(*s.ctx, values, s.nnz, true), r(*s.ctx, res, s.n_dof, true);
    eliminate(s, v.d, r.d, du.d);
    v.finish();
    r.finish();
  });
}

afem_status afem_constrain_residual(afem_system sys, double* res, const double* u) {
  return guarded([&] {
    System& s = SYS(sys);
    need(res, "residual");
    need(u, "u");
    In<double> du(*s.ctx, u, s.n_dof);
    Out<double> r(*s.ctx, res, s.n_dof, true);
    constrain_residual(s, r.d, du.d);
    r.finish();
  });
}

afem_status afem_csr_apply(afem_system sys, const double* values, const double* x, double* y) {
  return guarded([&] {
    System& s = SYS(sys);
    need(values, "values");
    need(x, "x");
    need(y, "y");
    In<double> dv(*s.ctx, values, s.nnz), dx(*s.ctx, x, s.n_dof);
    Out<double> o(*s.ctx, y, s.n_dof, false);
    csr_apply(s, dv.d, dx.d, o.d);
    o.finish();
  });
}

afem_status afem_free_norm(afem_system sys, const double* r, double* out) {
  return guarded([&] {
    System& s = SYS(sys);
    need(r, "r");
    need(out, "out");
    In<double> dr(*s.ctx, r, s.n_dof);
    *out = free_norm(*s.ctx, dr.d, s.mask.p, s.n_dof);
  });
}

// ---- values + handoff
afem_status afem_values_create(afem_system sys, afem_values* out) {
  return guarded([&] {
    System& s = SYS(sys);
    need(out, "out");
    auto v = std::make_unique<afem_values_s>();
    v->v.sys = &s;
    v->v.v.alloc(s.nnz);
    AFEM_CK(cudaMemsetAsync(v->v.v.p, 0, v->v.v.bytes(), s.ctx->stream));
    *out = v.release();
  });
}

afem_status afem_values_destroy(afem_values v) {
  return guarded([&] { delete v; });
}

afem_status afem_values_assemble(afem_values v, const double* u) {
  return guarded([&] {
    need(v, "values");
    System& s = *v->v.sys;
    begin(*s.ctx);
    need(u, "u");
    In<double> du(*s.ctx, u, s.n_dof);
    jacobian(s, du.d, v->v.v.p);
  });
}

afem_status afem_values_set(afem_values v, const double* values) {
  return guarded([&] {
    need(v, "values");
    need(values, "values data");
    System& s = *v->v.sys;
    begin(*s.ctx);
    In<double> dv(*s.ctx, values, s.nnz);
    copy(*s.ctx, dv.d, v->v.v.p, s.nnz);
    AFEM_CK(cudaStreamSynchronize(s.ctx->stream));
  });
}

afem_status afem_values_eliminate(afem_values v, double* res, const double* u) {
  return guarded([&] {
    need(v, "values");
    System& s = *v->v.sys;
    begin(*s.ctx);
    In<double> du(*s.ctx, u, s.n_dof);
    Out<double> r(*s.ctx, res, s.n_dof, true);
    eliminate(s, v->v.v.p, r.d, du.d);
    r.finish();
  });
}

afem_status afem_values_device_ptr(afem_values v, double** out) {
  return guarded([&] {
    need(v, "values");
    *out = v->v.v.p;
  });
}

afem_status afem_values_copy(afem_values v, double* out) {
  return guarded([&] {
    need(v, "values");
    System& s = *v->v.sys;
    begin(*s.ctx);
    Out<double> o(*s.ctx, out, s.nnz, false);
    copy(*s.ctx, v->v.v.p, o.d, s.nnz);
    o.finish();
  });
}

afem_status afem_buffer_create(afem_system sys, afem_buffer* out) {
  return guarded([&] {
    System& s = SYS(sys);
    need(out, "out");
    auto b = std::make_unique<afem_buffer_s>();
    b->b.sys = &s;
    *out = b.release();
  });
}

afem_status afem_buffer_destroy(afem_buffer b) {
  return guarded([&] { delete b; });
}

afem_status afem_buffer_handoff(afem_buffer b, afem_values* values) {
  return guarded([&] {
    need(b, "buffer");
    need(values, "values");
    if (b->b.state != 0) throw LeaseError("handoff: buffer is already leased to the solver");
    if (!*values || (*values)->v.sys != b->b.sys || (*values)->v.v.n != static_cast<size_t>(b->b.sys->nnz))
      throw std::invalid_argument("handoff: triplets do not match the precomputed pattern");
    b->b.store = std::move((*values)->v.v);  // buffer steal: the device storage is aliased, not copied
    delete *values;
    *values = nullptr;
    b->b.state = 1;
    ++b->b.epoch;
  });
}

afem_status afem_buffer_release(afem_buffer b) {
  return guarded([&] {
    need(b, "buffer");
    if (b->b.state != 1) throw LeaseError("release: buffer is not leased");
    b->b.state = 0;
  });
}

afem_status afem_buffer_state(afem_buffer b, int32_t* state, uint64_t* epoch) {
  return guarded([&] {
    need(b, "buffer");
    if (state) *state = b->b.state;
    if (epoch) *epoch = b->b.epoch;
  });
}

afem_status afem_buffer_assembly_values(afem_buffer b, double** out) {
  return guarded([&] {
    need(b, "buffer");
    if (b->b.state != 0) throw LeaseError("assembly-side access while the buffer is leased to the solver");
    *out = b->b.store.p;
  });
}

afem_status afem_buffer_solver_values(afem_buffer b, double** out) {
  return guarded([&] {
    need(b, "buffer");
    if (b->b.state != 1) throw LeaseError("solver-side access without an active lease");
    *out = b->b.store.p;
  });
}

// ---- operators
afem_status afem_op_create_explicit(afem_buffer b, afem_op* out) {
  return guarded([&] {
    need(b, "buffer");
    need(out, "out");
    if (b->b.state != 1) throw LeaseError("explicit_operator: buffer must be leased to the solver");
    auto op = std::make_unique<ExplicitOp>();
    op->sys = b->b.sys;
    op->kind = 0;
    op->n = b->b.sys->n_dof;
    op->buf = &b->b;
    op->epoch = b->b.epoch;
    auto h = std::make_unique<afem_op_s>();
    h->op = std::move(op);
    *out = h.release();
  });
}

afem_status afem_op_create_mf(afem_system sys, const double* u, afem_op* out) {
  return guarded([&] {
    System& s = SYS(sys);
    need(u, "u");
    need(out, "out");
    In<double> du(*s.ctx, u, s.n_dof);
    auto h = std::make_unique<afem_op_s>();
    h->op = make_mf_op(s, du.d);
    AFEM_CK(cudaStreamSynchronize(s.ctx->stream));
    *out = h.release();
  });
}

afem_status afem_op_destroy(afem_op op) {
  return guarded([&] { delete op; });
}

afem_status afem_op_kind(afem_op op, int32_t* kind) {
  return guarded([&] {
    need(op, "op");
    *kind = op->op->kind;
  });
}

afem_status afem_op_dim(afem_op op, int64_t* n) {
  return guarded([&] {
    need(op, "op");
    *n = op->op->n;
  });
}

// Host-buffer apply of a stencil operator, pipelined over z pieces: H2D of piece p+1 (copy stream),
// the apply of piece p (context stream, once its x planes and the halo plane have landed) and the
// D2H of piece p-1 (second copy stream) overlap; PCIe runs both directions at once.
static bool pipelined_host_apply(Operator& o, const double* x, double* y) {
  static const bool off = std::getenv("AFEM_NO_PIPELINE") != nullptr;
  auto* mf = dynamic_cast<MfOp*>(&o);
  if (off || !mf || !mf->stencil || is_device_ptr(x) || is_device_ptr(y)) return false;
  StencilPlan& pl = *mf->stencil;
  System& s = *o.sys;
  Ctx& c = *s.ctx;
  const int P = stencil_pieces(pl), zp = stencil_piece_planes(pl);
  if (P < 2) return false;
  const int64_t plane = 3 * (int64_t)(s.nx + 1) * (s.ny + 1);  // doubles per node plane
  const int NZ = s.nz + 1;
  double* dx = static_cast<double*>(c.stage(o.n * 8));
  double* dy = static_cast<double*>(c.stage(o.n * 8));
  c.copy_streams(2 * P + 1);
  cudaEvent_t start = c.events[2 * P];
  AFEM_CK(cudaEventRecord(start, c.stream));  // earlier work on the staging buffers is done
  AFEM_CK(cudaStreamWaitEvent(c.s_in, start, 0));
  AFEM_CK(cudaStreamWaitEvent(c.s_out, start, 0));
  for (int p = 0; p < P; ++p) {
    const int64_t a = (int64_t)p * zp * plane, b = std::min<int64_t>((int64_t)(p + 1) * zp, NZ) * plane;
    AFEM_CK(cudaMemcpyAsync(dx + a, x + a, (b - a) * 8, cudaMemcpyHostToDevice, c.s_in));
    AFEM_CK(cudaEventRecord(c.events[p], c.s_in));
  }
  for (int p = 0; p < P; ++p) {
    AFEM_CK(cudaStreamWaitEvent(c.stream, c.events[std::min(p + 1, P - 1)], 0));
    stencil_apply_pieces(pl, *mf, dx, dy, p, p + 1);
    AFEM_CK(cudaEventRecord(c.events[P + p], c.stream));
    AFEM_CK(cudaStreamWaitEvent(c.s_out, c.events[P + p], 0));
    const int64_t a = (int64_t)p * zp * plane, b = std::min<int64_t>((int64_t)(p + 1) * zp, NZ) * plane;
    AFEM_CK(cudaMemcpyAsync(y + a, dy + a, (b - a) * 8, cudaMemcpyDeviceToHost, c.s_out));
  }
  AFEM_CK(cudaStreamSynchronize(c.s_out));
  AFEM_CK(cudaStreamSynchronize(c.stream));
  return true;
}

afem_status afem_op_apply(afem_op op, const double* x, double* y) {
  return guarded([&] {
    need(op, "op");
    need(x, "x");
    need(y, "y");
    Operator& o = *op->op;
    Ctx& c = begin(*o.sys->ctx);
    o.validate();
    if (pipelined_host_apply(o, x, y)) return;
    In<double> dx(c, x, o.n);
    Out<double> dy(c, y, o.n, false);
    o.apply(dx.d, dy.d);
    dy.finish();
  });
}

afem_status afem_op_apply_async(afem_op op, const double* x, double* y) {
  return guarded([&] {
    need(op, "op");
    op->op->apply(x, y);
  });
}

afem_status afem_op_diagonal(afem_op op, double* d) {
  return guarded([&] {
    need(op, "op");
    Operator& o = *op->op;
    o.validate();
    Out<double> dd(begin(*o.sys->ctx), d, o.n, false);
    o.diagonal(dd.d);
    dd.finish();
  });
}

afem_status afem_op_csr_values(afem_op op, double** values) {
  return guarded([&] {
    need(op, "op");
    if (op->op->kind != 0) throw CapabilityError("assembled matrix required, but the operator is matrix-free");
    op->op->validate();
    *values = static_cast<ExplicitOp*>(op->op.get())->buf->store.p;
  });
}

afem_status afem_op_uses_stencil(afem_op op, int32_t* flag) {
  return guarded([&] {
    need(op, "op");
    *flag = op->op->uses_stencil() ? 1 : 0;
  });
}

afem_status afem_solve(afem_op op, const afem_solver_cfg* cfg, const double* b, const double* x0, double* x,
                       afem_solve_report* rep, double* history, int32_t hist_cap) {
  return guarded([&] {
    need(op, "op");
    need(cfg, "cfg");
    need(b, "b");
    need(x, "x");
    Operator& o = *op->op;
    Ctx& c = begin(*o.sys->ctx);
    In<double> db(c, b, o.n), dx0(c, x0, o.n);
    Out<double> dx(c, x, o.n, false);
    SolveReport r;
    solve(o, to_cfg(cfg), db.d, dx0.d, dx.d, r);
    dx.finish();
    fill_report(r, rep, history, hist_cap);
  });
}

afem_status afem_solve_bvp(afem_system sys, const afem_newton_cfg* cfg, const double* x0, double* u,
                           afem_newton_report* rep, double* norms, int32_t cap) {
  return guarded([&] {
    System& s = SYS(sys);
    need(cfg, "cfg");
    need(u, "u");
    Ctx& c = *s.ctx;
    Out<double> du(c, u, s.n_dof, false);
    if (x0) {
      In<double> dx0(c, x0, s.n_dof);
      copy(c, dx0.d, du.d, s.n_dof);
    } else {
      fill(c, 0.0, du.d, s.n_dof);
    }
    NewtonReport r;
    newton(s, cfg, du.d, r);
    du.finish();
    fill_newton(r, rep, norms, cap);
  });
}

afem_status afem_solve_bvp_ex(afem_system sys, const afem_newton_cfg* cfg, const double* x0, double* u,
                              afem_newton_report* rep, double* norms, int32_t cap, afem_solve_report* linear,
                              int32_t linear_cap) {
  return guarded([&] {
    System& s = SYS(sys);
    need(cfg, "cfg");
    need(u, "u");
    Ctx& c = *s.ctx;
    Out<double> du(c, u, s.n_dof, false);
    if (x0) {
      In<double> dx0(c, x0, s.n_dof);
      copy(c, dx0.d, du.d, s.n_dof);
    } else {
      fill(c, 0.0, du.d, s.n_dof);
    }
    NewtonReport r;
    newton(s, cfg, du.d, r);
    du.finish();
    fill_newton(r, rep, norms, cap);
    if (linear)
      for (int32_t k = 0; k < linear_cap && k < static_cast<int32_t>(r.linear.size()); ++k)
        fill_report(r.linear[k], &linear[k], nullptr, 0);
  });
}

afem_status afem_op_create_csr(afem_ctx ctx, int64_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* cols,
                               afem_op* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(row_ptr, "row_ptr");
    need(out, "out");
    if (nnz > 0) need(cols, "cols");
    Ctx& c = begin(ctx->c);
    if (is_device_ptr(row_ptr) || is_device_ptr(cols))
      throw std::invalid_argument("afem_op_create_csr: row_ptr / cols must be host arrays");
    auto h = std::make_unique<afem_op_s>();
    h->op = make_csr_op(c, n, nnz, row_ptr, cols);
    *out = h.release();
  });
}

afem_status afem_op_set_values(afem_op op, const double* values) {
  return guarded([&] {
    need(op, "op");
    Operator& o = *op->op;
    int64_t nnz = 0;
    double* dst = csr_op_values(o, &nnz);
    Ctx& c = begin(*o.sys->ctx);
    if (nnz > 0) {
      need(values, "values");
      AFEM_CK(cudaMemcpyAsync(dst, values, nnz * sizeof(double), cudaMemcpyDefault, c.stream));
      AFEM_CK(cudaStreamSynchronize(c.stream));
    }
  });
}

afem_status afem_eliminate_csr(afem_ctx ctx, int64_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* cols,
                               double* values, double* residual, const uint8_t* constrained,
                               const double* prescribed, const double* u) {
  return guarded([&] {
    need(ctx, "ctx");
    need(row_ptr, "row_ptr");
    need(residual, "residual");
    need(constrained, "constrained");
    need(prescribed, "prescribed");
    need(u, "u");
    if (nnz > 0) {
      need(cols, "cols");
      need(values, "values");
    }
    Ctx& c = begin(ctx->c);
    In<int32_t> drp(c, row_ptr, n + 1), dci(c, cols, nnz);
    In<uint8_t> dm(c, constrained, n);
    In<double> dp(c, prescribed, n), du(c, u, n);
    Out<double> dv(c, values, nnz, true), dr(c, residual, n, true);
    eliminate_csr(c, n, drp.d, dci.d, dv.d, dr.d, dm.d, dp.d, du.d);
    dv.finish();
    dr.finish();
  });
}

afem_status afem_constrain_masked(afem_ctx ctx, int64_t n, double* residual, const uint8_t* constrained,
                                  const double* prescribed, const double* u) {
  return guarded([&] {
    need(ctx, "ctx");
    need(residual, "residual");
    need(constrained, "constrained");
    need(prescribed, "prescribed");
    need(u, "u");
    Ctx& c = begin(ctx->c);
    In<uint8_t> dm(c, constrained, n);
    In<double> dp(c, prescribed, n), du(c, u, n);
    Out<double> dr(c, residual, n, true);
    constrain_masked(c, n, dr.d, dm.d, dp.d, du.d);
    dr.finish();
  });
}

afem_status afem_load_stepping(afem_system sys, double total_strain, int32_t n_steps, const afem_newton_cfg* cfg,
                               double* u, int32_t* failed_step, int32_t* converged, int32_t* step_iterations) {
  return guarded([&] {
    System& s = SYS(sys);
    need(cfg, "cfg");
    need(u, "u");
    if (n_steps < 1) throw std::invalid_argument("load_stepping: n_steps must be >= 1");
    Ctx& c = *s.ctx;
    Out<double> du(c, u, s.n_dof, false);
    fill(c, 0.0, du.d, s.n_dof);
    if (failed_step) *failed_step = -1;
    if (converged) *converged = 0;
    for (int st = 1; st <= n_steps; ++st) {
      const double strain = total_strain * st / n_steps;  // newton.hpp:171
      set_dirichlet(s, benchmark_bcs(s, strain));
      NewtonReport r;
      newton(s, cfg, du.d, r);
      if (step_iterations) step_iterations[st - 1] = r.iterations;
      if (!r.converged) {
        if (failed_step) *failed_step = st;
        du.finish();
        return;
      }
      history_commit(s, du.d);  // J2: the converged step becomes the committed history
    }
    if (converged) *converged = 1;
    du.finish();
  });
}

afem_status afem_history_size(afem_system sys, int64_t* n) {
  return guarded([&] {
    System& s = SYS(sys);
    need(n, "n");
    *n = static_cast<int64_t>(s.hist.n);
  });
}

afem_status afem_history_commit(afem_system sys, const double* u) {
  return guarded([&] {
    System& s = SYS(sys);
    need(u, "u");
    In<double> du(*s.ctx, u, s.n_dof);
    history_commit(s, du.d);
    AFEM_CK(cudaStreamSynchronize(s.ctx->stream));
  });
}

afem_status afem_history_reset(afem_system sys) {
  return guarded([&] {
    System& s = SYS(sys);
    history_reset(s);
    AFEM_CK(cudaStreamSynchronize(s.ctx->stream));
  });
}

afem_status afem_history_copy(afem_system sys, double* out) {
  return guarded([&] {
    System& s = SYS(sys);
    need(out, "out");
    if (!s.has_history()) throw std::invalid_argument("history: system has no J2 phase");
    Out<double> o(*s.ctx, out, s.hist.n, false);
    AFEM_CK(cudaMemcpyAsync(o.d, s.hist.p, s.hist.bytes(), cudaMemcpyDeviceToDevice, s.ctx->stream));
    o.finish();
  });
}

afem_status afem_history_set(afem_system sys, const double* in) {
  return guarded([&] {
    System& s = SYS(sys);
    need(in, "in");
    if (!s.has_history()) throw std::invalid_argument("history: system has no J2 phase");
    In<double> d(*s.ctx, in, s.hist.n);
    AFEM_CK(cudaMemcpyAsync(s.hist.p, d.d, s.hist.bytes(), cudaMemcpyDeviceToDevice, s.ctx->stream));
    AFEM_CK(cudaStreamSynchronize(s.ctx->stream));
  });
}

// ---- multi-GPU slab decomposition
afem_status afem_slab_range(int32_t nz, int32_t size, int32_t rank, int32_t* z0, int32_t* z1) {
  return guarded([&] {
    need(z0, "z0");
    need(z1, "z1");
    slab_range(nz, size, rank, z0, z1);
  });
}

afem_status afem_nccl_unique_id(void* out) {
  return guarded([&] {
    need(out, "out");
    nccl_unique_id(out);
  });
}

afem_status afem_dist_create_nccl(afem_ctx ctx, const void* uid, int32_t rank, int32_t size, afem_dist* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(uid, "uid");
    need(out, "out");
    begin(ctx->c);
    auto d = std::make_unique<afem_dist_s>();
    d->ctx = &ctx->c;
    d->comm.reset(comm_create_nccl(uid, rank, size));
    *out = d.release();
  });
}

afem_status afem_thread_group_create(int32_t size, afem_thread_group* out) {
  return guarded([&] {
    need(out, "out");
    auto g = std::make_unique<afem_thread_group_s>();
    g->g = thread_group_create(size);
    *out = g.release();
  });
}

afem_status afem_thread_group_destroy(afem_thread_group g) {
  return guarded([&] {
    if (!g) return;
    thread_group_destroy(g->g);
    delete g;
  });
}

afem_status afem_dist_create_threads(afem_ctx ctx, afem_thread_group g, int32_t rank, afem_dist* out) {
  return guarded([&] {
    need(ctx, "ctx");
    need(g, "group");
    need(out, "out");
    auto d = std::make_unique<afem_dist_s>();
    d->ctx = &ctx->c;
    d->comm.reset(comm_create_threads(g->g, rank));
    *out = d.release();
  });
}

afem_status afem_dist_destroy(afem_dist d) {
  return guarded([&] { delete d; });
}

afem_status afem_dist_set_benchmark_dirichlet(afem_dist d, afem_system slab, double strain, double lx_global) {
  return guarded([&] {
    need(d, "dist");
    System& s = SYS(slab);
    set_dirichlet(s, slab_benchmark_bcs(s, d->comm->rank, d->comm->size, strain, lx_global));
  });
}

afem_status afem_dist_op_create_mf(afem_dist d, afem_system slab, const double* u, afem_op* out) {
  return guarded([&] {
    need(d, "dist");
    need(u, "u");
    need(out, "out");
    System& s = SYS(slab);
    In<double> du(*s.ctx, u, s.n_dof);
    auto h = std::make_unique<afem_op_s>();
    h->op = make_dist_mf_op(s, d->comm.get(), make_mf_op(s, du.d));
    *out = h.release();
  });
}

afem_status afem_dist_op_create_explicit(afem_dist d, afem_system slab, const double* values, afem_op* out) {
  return guarded([&] {
    need(d, "dist");
    need(values, "values");
    need(out, "out");
    System& s = SYS(slab);
    In<double> dv(*s.ctx, values, s.nnz);
    auto h = std::make_unique<afem_op_s>();
    h->op = make_dist_csr_op(s, d->comm.get(), dv.d);
    *out = h.release();
  });
}

afem_status afem_dist_solve(afem_dist d, afem_op op, const afem_solver_cfg* cfg, const double* b, const double* x0,
                            double* x, afem_solve_report* rep, double* history, int32_t hist_cap) {
  return guarded([&] {
    need(d, "dist");
    need(op, "op");
    need(cfg, "cfg");
    need(b, "b");
    need(x, "x");
    auto* dop = dynamic_cast<DistMfOp*>(op->op.get());
    if (!dop) throw std::invalid_argument("afem_dist_solve: operator is not distributed");
    Ctx& c = begin(*dop->sys->ctx);
    In<double> db(c, b, dop->n), dx0(c, x0, dop->n);
    Out<double> dx(c, x, dop->n, false);
    SolveReport r;
    const SolverCfg sc = to_cfg(cfg);
    dist_run_solver(*dop, sc, db.d, dx0.d, dx.d, r);
    dx.finish();
    fill_report(r, rep, history, hist_cap);
  });
}

afem_status afem_dist_assemble(afem_dist d, afem_op op, double* v) {
  return guarded([&] {
    need(d, "dist");
    need(op, "op");
    need(v, "v");
    auto* dop = dynamic_cast<DistMfOp*>(op->op.get());
    if (!dop) throw std::invalid_argument("afem_dist_assemble: operator is not distributed");
    Ctx& c = begin(*dop->sys->ctx);
    Out<double> dv(c, v, dop->n, true);
    dop->halo_add(dv.d, nullptr, false);
    dv.finish();
  });
}

afem_status afem_dist_solve_bvp(afem_dist d, afem_system slab, const afem_newton_cfg* cfg, const double* x0, double* u,
                                afem_newton_report* rep, double* norms, int32_t norms_cap) {
  return guarded([&] {
    need(d, "dist");
    need(cfg, "cfg");
    need(u, "u");
    System& s = SYS(slab);
    Ctx& c = *s.ctx;
    Out<double> du(c, u, s.n_dof, false);
    if (x0) {
      In<double> dx0(c, x0, s.n_dof);
      copy(c, dx0.d, du.d, s.n_dof);
    } else {
      fill(c, 0.0, du.d, s.n_dof);
    }
    NewtonReport r;
    dist_newton(s, d->comm.get(), cfg, du.d, r);
    du.finish();
    fill_newton(r, rep, norms, norms_cap);
  });
}

afem_status afem_dist_load_stepping(afem_dist d, afem_system slab, double total_strain, int32_t n_steps,
                                    double lx_global, const afem_newton_cfg* cfg, double* u, int32_t* failed_step,
                                    int32_t* converged, int32_t* step_iterations) {
  return guarded([&] {
    need(d, "dist");
    need(cfg, "cfg");
    need(u, "u");
    if (n_steps < 1) throw std::invalid_argument("load_stepping: n_steps must be >= 1");
    System& s = SYS(slab);
    Ctx& c = *s.ctx;
    Out<double> du(c, u, s.n_dof, false);
    fill(c, 0.0, du.d, s.n_dof);
    if (failed_step) *failed_step = -1;
    if (converged) *converged = 0;
    for (int st = 1; st <= n_steps; ++st) {
      const double strain = total_strain * st / n_steps;  // newton.hpp:171
      set_dirichlet(s, slab_benchmark_bcs(s, d->comm->rank, d->comm->size, strain, lx_global));
      NewtonReport r;
      dist_newton(s, d->comm.get(), cfg, du.d, r);
      if (step_iterations) step_iterations[st - 1] = r.iterations;
      if (!r.converged) {
        if (failed_step) *failed_step = st;
        du.finish();
        return;
      }
      history_commit(s, du.d);  // J2 history is element-local: each rank commits its own slab
    }
    if (converged) *converged = 1;
    du.finish();
  });
}

afem_status afem_dist_dot(afem_dist d, afem_op op, const double* a, const double* b, double* out) {
  return guarded([&] {
    need(d, "dist");
    need(op, "op");
    need(out, "out");
    auto* dop = dynamic_cast<DistMfOp*>(op->op.get());
    if (!dop) throw std::invalid_argument("afem_dist_dot: operator is not distributed");
    Ctx& c = begin(*dop->sys->ctx);
    In<double> da(c, a, dop->n), dbb(c, b, dop->n);
    *out = dist_dot(*dop, da.d, dbb.d);
  });
}

}  // extern "C"
