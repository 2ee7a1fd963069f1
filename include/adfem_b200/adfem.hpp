// adfem_b200/adfem.hpp — C++ overlay of libafem_b200.so with the reference's own types and
// signatures (namespace adfem, /root/reference/proj/include/adfem). Header-only; include it after
// the reference's "adfem/adfem.hpp" is on the include path and link -lafem_b200.
//
// Drop-in surface (every function keeps the reference's parameter and return types):
//   adfem::b200::solve_bvp(mesh, materials, bcs, cfg, x0)          newton.hpp:59-152
//   adfem::b200::load_stepping(mesh, materials, strain, cfg, n)    newton.hpp:163-186
//   adfem::b200::run_solver(op, b, cfg)                            backend.hpp:241-286
// and, over a device-resident System built once from (Mesh, materials):
//   assemble_residual / assemble_jacobian (CooTriplets in pattern order, ready for the
//   reference's HandoffBuffer::handoff) / assemble_diagonal / apply_dirichlet /
//   precompute_sparsity (SparsityPattern, bit-exact) / matrix_free_operator / explicit_operator.
// b200::LinearOperator has the reference LinearOperator's public interface (kind, dim, apply,
// diagonal), so the reference's own cg<Op, Prec> / gmres<Op, Prec> templates (krylov.hpp:350,
// 415) can drive the device operator too.
// Errors: the C status codes are rethrown as the reference's exception types (errors.hpp:10-38);
// numerical non-convergence stays in the report structs, as in the reference.
#ifndef ADFEM_B200_ADFEM_HPP
#define ADFEM_B200_ADFEM_HPP

#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "adfem/adfem.hpp"
#include "afem.h"

namespace adfem::b200 {

// ------------------------------------------------------------------ errors
inline void check(afem_status s) {
  if (s == AFEM_OK) return;
  const std::string m = afem_last_error();
  switch (s) {
    case AFEM_E_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case AFEM_E_OUT_OF_RANGE: throw std::out_of_range(m);
    case AFEM_E_LOGIC: throw std::logic_error(m);
    case AFEM_E_DOMAIN: throw std::domain_error(m);
    case AFEM_E_LEASE: throw LeaseError(m);
    case AFEM_E_STALE_EPOCH: throw StaleEpochError(m);
    case AFEM_E_CAPABILITY: throw CapabilityError(m);
    case AFEM_E_FACTORIZATION: throw FactorizationError(m);
    case AFEM_E_INVERTED_ELEMENT: throw InvertedElementError(m);
    default: throw std::runtime_error(m);
  }
}

// ------------------------------------------------------------------ device context
// One context per (host thread, device), created on first use.
inline afem_ctx context(int device = 0) {
  struct Holder {
    afem_ctx h = nullptr;
    ~Holder() {
      if (h) afem_ctx_destroy(h);
    }
  };
  static thread_local Holder holder;
  if (!holder.h) check(afem_ctx_create(device, &holder.h));
  return holder.h;
}

inline afem_material to_afem(const Material& m) {
  afem_material a{};
  a.model = m.model == MaterialModel::StVenantKirchhoff ? 1 : 0;
  a.E = m.E;
  a.nu = m.nu;
  return a;
}

inline afem_solver_cfg to_afem(const SolverConfig& c) {
  afem_solver_cfg a{};
  switch (c.method) {  // krylov.hpp:20 order
    case SolverMethod::CG: a.method = 0; break;
    case SolverMethod::GMRES: a.method = 1; break;
    case SolverMethod::BICGSTAB: a.method = 2; break;
    case SolverMethod::DIRECT_CHOL: a.method = 3; break;
    case SolverMethod::DIRECT_LU: a.method = 4; break;
  }
  a.precond = c.preconditioner == PreconKind::JACOBI ? 1 : (c.preconditioner == PreconKind::ILU0 ? 2 : 0);
  a.rtol = c.rtol;
  a.max_iter = c.max_iter;
  a.restart = c.gmres_restart;
  return a;
}

inline afem_newton_cfg to_afem(const NewtonConfig& c) {
  afem_newton_cfg a{};
  a.rtol = c.rtol;
  a.atol = c.atol;
  a.max_iter = c.max_iter;
  a.operator_kind = c.operator_kind == OperatorKind::EXPLICIT ? 0 : 1;
  a.linear = to_afem(c.linear);
  return a;
}

// ------------------------------------------------------------------ device system
// Mesh + batches + sparsity pattern + Dirichlet table resident in HBM (build_batches,
// precompute_sparsity and constraint_table run on the device; assembly.hpp:36-99, 197-211).
class System {
 public:
  System(const Mesh& mesh, std::span<const Material> materials) {
    std::vector<double> xy;
    xy.reserve(2 * mesh.nodes.size());
    for (const auto& n : mesh.nodes) {
      xy.push_back(n[0]);
      xy.push_back(n[1]);
    }
    std::vector<int32_t> conn;
    conn.reserve(4 * mesh.elements.size());
    for (const auto& e : mesh.elements) conn.insert(conn.end(), e.begin(), e.end());
    std::vector<int32_t> phase(mesh.material_of.begin(), mesh.material_of.end());
    std::vector<afem_material> mats;
    for (const Material& m : materials) mats.push_back(to_afem(m));
    afem_system h = nullptr;
    check(afem_system_create(context(), 2, mesh.n_nodes(), mesh.n_elements(), xy.data(), conn.data(), phase.data(),
                             static_cast<int32_t>(mats.size()), mats.data(), &h));
    h_.reset(h);
    check(afem_system_get_info(h, &info_));
  }
  afem_system handle() const { return h_.get(); }
  int n_dof() const { return static_cast<int>(info_.n_dof); }
  std::int64_t nnz() const { return info_.nnz; }

  void set_dirichlet(const DirichletSpec& bcs) {
    std::vector<int32_t> node, comp;
    std::vector<double> val;
    for (const auto& c : bcs.constraints) {
      node.push_back(c.node);
      comp.push_back(c.component);
      val.push_back(c.value);
    }
    check(afem_set_dirichlet(h_.get(), static_cast<std::int64_t>(node.size()), node.data(), comp.data(), val.data()));
  }

 private:
  struct Del {
    void operator()(afem_system s) const { afem_system_destroy(s); }
  };
  std::unique_ptr<afem_system_s, Del> h_;
  afem_system_info info_{};
};

// precompute_sparsity (assembly.hpp:71-99): bit-exact rows / cols / row_ptr.
inline std::shared_ptr<const SparsityPattern> precompute_sparsity(const System& s) {
  auto p = std::make_shared<SparsityPattern>();
  p->n_dof = s.n_dof();
  std::vector<std::int64_t> rp(static_cast<std::size_t>(s.n_dof()) + 1);
  p->rows.resize(static_cast<std::size_t>(s.nnz()));
  p->cols.resize(static_cast<std::size_t>(s.nnz()));
  check(afem_pattern(s.handle(), rp.data(), p->rows.data(), p->cols.data()));
  p->row_ptr.assign(rp.begin(), rp.end());
  return p;
}

// assemble_residual (assembly.hpp:126-139).
inline std::vector<double> assemble_residual(const System& s, std::span<const double> u) {
  if (static_cast<int>(u.size()) != s.n_dof()) throw std::invalid_argument("assemble_residual: state size mismatch");
  std::vector<double> r(u.size());
  check(afem_residual(s.handle(), u.data(), r.data()));
  return r;
}

// assemble_jacobian (assembly.hpp:144-173): the sorted, deduplicated triplets in pattern order,
// exactly what the reference hands to HandoffBuffer::handoff.
inline CooTriplets assemble_jacobian(const System& s, std::span<const double> u, const SparsityPattern& pattern) {
  if (static_cast<int>(u.size()) != s.n_dof()) throw std::invalid_argument("assemble_jacobian: state size mismatch");
  if (static_cast<std::int64_t>(pattern.nnz()) != s.nnz())
    throw std::logic_error("assemble_jacobian: produced indices leave the precomputed pattern");
  CooTriplets c;
  c.n = s.n_dof();
  c.rows = pattern.rows;
  c.cols = pattern.cols;
  c.values.resize(pattern.nnz());
  check(afem_jacobian(s.handle(), u.data(), c.values.data()));
  return c;
}

// assemble_diagonal (assembly.hpp:177-188).
inline std::vector<double> assemble_diagonal(const System& s, std::span<const double> u) {
  std::vector<double> d(u.size());
  check(afem_diagonal(s.handle(), u.data(), d.data()));
  return d;
}

// apply_dirichlet(pattern, values, residual, spec, u) (assembly.hpp:242-249) with the system's table.
inline void apply_dirichlet(const System& s, std::span<double> values, std::span<double> residual,
                            std::span<const double> u) {
  check(afem_eliminate(s.handle(), values.data(), residual.data(), u.data()));
}

// ------------------------------------------------------------------ operators (backend.hpp:117-236)
class LinearOperator {
 public:
  OperatorKind kind() const { return kind_; }
  int dim() const { return n_; }
  void apply(std::span<const double> x, std::span<double> y) const {
    if (static_cast<int>(x.size()) != n_ || static_cast<int>(y.size()) != n_)
      throw std::invalid_argument("linear operator: dimension mismatch");
    check(afem_op_apply(h_.get(), x.data(), y.data()));
  }
  std::vector<double> diagonal() const {
    std::vector<double> d(static_cast<std::size_t>(n_));
    check(afem_op_diagonal(h_.get(), d.data()));
    return d;
  }
  bool uses_stencil() const {
    int32_t f = 0;
    check(afem_op_uses_stencil(h_.get(), &f));
    return f != 0;
  }
  afem_op handle() const { return h_.get(); }

  friend LinearOperator matrix_free_operator(const System& s, std::span<const double> u);
  friend class DeviceHandoff;

 private:
  struct Del {
    void operator()(afem_op o) const { afem_op_destroy(o); }
  };
  LinearOperator(afem_op h, OperatorKind k) : h_(h, Del{}) {
    kind_ = k;
    std::int64_t n = 0;
    check(afem_op_dim(h, &n));
    n_ = static_cast<int>(n);
  }
  std::shared_ptr<afem_op_s> h_;
  OperatorKind kind_ = OperatorKind::MATRIX_FREE;
  int n_ = 0;
};

// matrix_free_operator(batches, u, dirichlet) (backend.hpp:222-236): copies u and the system's
// constraint table; the structured stencil path is chosen automatically on grid systems.
inline LinearOperator matrix_free_operator(const System& s, std::span<const double> u) {
  afem_op h = nullptr;
  check(afem_op_create_mf(s.handle(), u.data(), &h));
  return LinearOperator(h, OperatorKind::MATRIX_FREE);
}

// HandoffBuffer (backend.hpp:33-111) over device-resident values: assemble, eliminate, hand off
// (lease + epoch), build the explicit operator, release.
class DeviceHandoff {
 public:
  explicit DeviceHandoff(const System& s) : sys_(&s) {
    afem_buffer b = nullptr;
    check(afem_buffer_create(s.handle(), &b));
    buf_.reset(b);
  }
  // assemble_jacobian + apply_dirichlet on the device; rhs = -R eliminated (newton.hpp:108-111).
  std::vector<double> assemble(std::span<const double> u) {
    afem_values v = nullptr;
    check(afem_values_create(sys_->handle(), &v));
    std::vector<double> r = assemble_residual(*sys_, u);
    check(afem_values_assemble(v, u.data()));
    check(afem_values_eliminate(v, r.data(), u.data()));
    pending_ = v;
    for (double& x : r) x = -x;
    return r;
  }
  // handoff(CooTriplets&&) (backend.hpp:50-66): moves the values (no copy), LeaseError if leased.
  void handoff() {
    check(afem_buffer_handoff(buf_.get(), &pending_));
    pending_ = nullptr;
  }
  void release() { check(afem_buffer_release(buf_.get())); }
  LeaseState state() const {
    int32_t st = 0;
    std::uint64_t ep = 0;
    check(afem_buffer_state(buf_.get(), &st, &ep));
    return st ? LeaseState::LeasedToSolver : LeaseState::OwnedByAssembly;
  }
  std::uint64_t epoch() const {
    int32_t st = 0;
    std::uint64_t ep = 0;
    check(afem_buffer_state(buf_.get(), &st, &ep));
    return ep;
  }
  // explicit_operator(buffer) (backend.hpp:199-214)
  LinearOperator explicit_operator() const {
    afem_op h = nullptr;
    check(afem_op_create_explicit(buf_.get(), &h));
    return LinearOperator(h, OperatorKind::EXPLICIT);
  }
  ~DeviceHandoff() {
    if (pending_) afem_values_destroy(pending_);
  }

 private:
  struct Del {
    void operator()(afem_buffer b) const { afem_buffer_destroy(b); }
  };
  const System* sys_;
  std::unique_ptr<afem_buffer_s, Del> buf_;
  afem_values pending_ = nullptr;
};

// ------------------------------------------------------------------ solve (backend.hpp:241-286)
inline std::pair<std::vector<double>, SolveReport> run_solver(const LinearOperator& op, std::span<const double> b,
                                                              const SolverConfig& cfg) {
  cfg.validate();
  const afem_solver_cfg c = to_afem(cfg);
  std::vector<double> x(b.size());
  std::vector<double> hist(static_cast<std::size_t>(cfg.max_iter) + 2);
  afem_solve_report rep{};
  check(afem_solve(op.handle(), &c, b.data(), nullptr, x.data(), &rep, hist.data(),
                   static_cast<int32_t>(hist.size())));
  SolveReport out;
  out.converged = rep.converged != 0;
  out.iterations = rep.iterations;
  out.residual_history.assign(hist.begin(), hist.begin() + std::min<std::size_t>(hist.size(), rep.n_history));
  out.wall_time = rep.wall_time;
  out.failure = rep.failure;
  return {std::move(x), std::move(out)};
}

// ------------------------------------------------------------------ Newton (newton.hpp:59-186)
inline std::pair<std::vector<double>, NewtonReport> solve_bvp(const Mesh& mesh, std::span<const Material> materials,
                                                              const DirichletSpec& bcs, const NewtonConfig& cfg,
                                                              std::span<const double> initial_guess = {}) {
  cfg.validate();
  validate_dirichlet(bcs, mesh);
  System s(mesh, materials);
  s.set_dirichlet(bcs);
  const afem_newton_cfg c = to_afem(cfg);
  std::vector<double> u(static_cast<std::size_t>(s.n_dof()), 0.0);
  std::vector<double> norms(static_cast<std::size_t>(cfg.max_iter) + 2);
  afem_newton_report rep{};
  check(afem_solve_bvp(s.handle(), &c, initial_guess.empty() ? nullptr : initial_guess.data(), u.data(), &rep,
                       norms.data(), static_cast<int32_t>(norms.size())));
  NewtonReport out;
  out.converged = rep.converged != 0;
  out.iterations = rep.iterations;
  out.residual_norms.assign(norms.begin(), norms.begin() + std::min<std::size_t>(norms.size(), rep.n_norms));
  out.total_time = rep.total_time;
  out.failure = rep.failure;
  if (cfg.log)
    for (std::size_t k = 1; k < out.residual_norms.size(); ++k)
      *cfg.log << "newton iter=" << k << " rnorm=" << out.residual_norms[k]
               << " rel=" << out.residual_norms[k] / out.residual_norms[0] << "\n";
  return {std::move(u), std::move(out)};
}

inline std::pair<std::vector<double>, LoadSteppingReport> load_stepping(const Mesh& mesh,
                                                                        std::span<const Material> materials,
                                                                        double total_strain, const NewtonConfig& cfg,
                                                                        int n_steps) {
  if (n_steps < 1) throw std::invalid_argument("load_stepping: n_steps must be >= 1");
  LoadSteppingReport rep;
  std::vector<double> u;
  for (int st = 1; st <= n_steps; ++st) {
    const DirichletSpec bcs = benchmark_bcs(mesh, total_strain * st / n_steps);
    auto [u_s, nrep] = ::adfem::b200::solve_bvp(mesh, materials, bcs, cfg, u);
    rep.steps.push_back(nrep);
    rep.total_time += nrep.total_time;
    u = std::move(u_s);
    if (!nrep.converged) {
      rep.failed_step = st;
      return {std::move(u), std::move(rep)};
    }
  }
  rep.converged = true;
  return {std::move(u), std::move(rep)};
}

}  // namespace adfem::b200

#endif  // ADFEM_B200_ADFEM_HPP
