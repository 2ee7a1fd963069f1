// adfem/backend.hpp — B200 drop-in for the reference's assembly -> solver boundary
// (proj/include/adfem/backend.hpp). Same namespace, types, signatures and error semantics:
//
//   HandoffBuffer / LeaseGuard   (backend.hpp:33-111) host value store with the lease + epoch
//                                protocol (the values are the reference's std::vector, moved in)
//   LinearOperator               (backend.hpp:117-194) EXPLICIT: a device CSR operator whose values
//                                are re-uploaded from the leased store whenever it may have been
//                                written (a handoff or a mutable view handed out: writes through
//                                solver_values() are seen, backend test WriteThrough);
//                                its SpMV is bitwise equal to CsrMatrix::apply. MATRIX_FREE: the
//                                device matrix-free operator of the batches' mirror (state u and
//                                the constraint mask copied at creation, backend.hpp:222-236)
//   explicit_operator / matrix_free_operator / run_solver (backend.hpp:199-286)
//
// run_solver runs the Krylov methods on the device (afem_solve). ILU(0) and the banded direct
// factorisations need the device system the pattern came from (any pattern produced by
// precompute_sparsity); CapabilityError on matrix-free operators as in the reference.
#ifndef ADFEM_BACKEND_HPP
#define ADFEM_BACKEND_HPP

#include <cstdint>
#include <memory>
#include <ostream>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

#include "adfem/assembly.hpp"
#include "adfem/b200_device.hpp"
#include "adfem/errors.hpp"
#include "adfem/krylov.hpp"
#include "adfem/sparse.hpp"

namespace adfem {

enum class OperatorKind { EXPLICIT, MATRIX_FREE };

inline const char* to_string(OperatorKind k) { return k == OperatorKind::EXPLICIT ? "EXPLICIT" : "MATRIX_FREE"; }

enum class LeaseState { OwnedByAssembly, LeasedToSolver };

/// The assembly -> solver boundary (backend.hpp:33-97).
class HandoffBuffer {
 public:
  explicit HandoffBuffer(std::shared_ptr<const SparsityPattern> pattern)
      : pattern_(std::move(pattern)), store_(std::make_shared<std::vector<double>>()) {
    if (!pattern_) throw std::invalid_argument("handoff buffer: null pattern");
  }

  LeaseState state() const { return state_; }
  std::uint64_t epoch() const { return epoch_; }
  const SparsityPattern& pattern() const { return *pattern_; }
  std::shared_ptr<const SparsityPattern> pattern_handle() const { return pattern_; }
  void set_trace(std::ostream* os) { trace_ = os; }

  /// Moves the assembled values in (no element copy) and leases them to the solver.
  void handoff(CooTriplets&& coo) {
    if (state_ != LeaseState::OwnedByAssembly) throw LeaseError("handoff: buffer is already leased to the solver");
    const bool same = coo.n == pattern_->n_dof && coo.size() == pattern_->nnz() && coo.rows == pattern_->rows &&
                      coo.cols == pattern_->cols;
    if (!same) throw std::invalid_argument("handoff: triplets do not match the precomputed pattern");
    *store_ = std::move(coo.values);
    state_ = LeaseState::LeasedToSolver;
    ++epoch_;
    ++version_;
    if (trace_) *trace_ << "lease handoff epoch=" << epoch_ << "\n";
  }

  void release() {
    if (state_ != LeaseState::LeasedToSolver) throw LeaseError("release: buffer is not leased");
    state_ = LeaseState::OwnedByAssembly;
    if (trace_) *trace_ << "lease release epoch=" << epoch_ << "\n";
  }

  std::span<double> assembly_values() {
    if (state_ != LeaseState::OwnedByAssembly)
      throw LeaseError("assembly-side access while the buffer is leased to the solver");
    ++version_;
    return {store_->data(), store_->size()};
  }

  std::span<double> solver_values() {
    if (state_ != LeaseState::LeasedToSolver) throw LeaseError("solver-side access without an active lease");
    ++version_;
    return {store_->data(), store_->size()};
  }

  std::shared_ptr<std::vector<double>> value_store() const {
    ++version_;
    return store_;
  }

  /// B200: bumped whenever the values may have been (re)written — a handoff or a mutable view
  /// handed out — so the explicit operator re-uploads its device copy only then.
  std::uint64_t values_version() const { return version_; }

 private:
  std::shared_ptr<const SparsityPattern> pattern_;
  std::shared_ptr<std::vector<double>> store_;
  LeaseState state_ = LeaseState::OwnedByAssembly;
  std::uint64_t epoch_ = 0;
  mutable std::uint64_t version_ = 0;
  std::ostream* trace_ = nullptr;
};

/// Releases the lease on scope exit (backend.hpp:100-111).
class LeaseGuard {
 public:
  explicit LeaseGuard(HandoffBuffer& b) : buffer_(&b) {}
  ~LeaseGuard() {
    if (buffer_ && buffer_->state() == LeaseState::LeasedToSolver) buffer_->release();
  }
  LeaseGuard(const LeaseGuard&) = delete;
  LeaseGuard& operator=(const LeaseGuard&) = delete;

 private:
  HandoffBuffer* buffer_;
};

class LinearOperator;
std::pair<std::vector<double>, SolveReport> run_solver(const LinearOperator& op, std::span<const double> b,
                                                       const SolverConfig& cfg);

/// x -> K(u) x, EXPLICIT or MATRIX_FREE (backend.hpp:117-194), executed on the device.
class LinearOperator {
 public:
  OperatorKind kind() const { return kind_; }
  int dim() const { return n_; }

  void apply(std::span<const double> x, std::span<double> y) const {
    if (static_cast<int>(x.size()) != n_ || static_cast<int>(y.size()) != n_)
      throw std::invalid_argument("linear operator: dimension mismatch");
    if (kind_ == OperatorKind::EXPLICIT) {
      validate_lease();
      sync_values();
    }
    b200_dropin::check(afem_op_apply(dev_->h, x.data(), y.data()));
  }

  const CsrMatrix& csr() const {
    if (kind_ != OperatorKind::EXPLICIT) throw CapabilityError("assembled matrix required, but the operator is matrix-free");
    validate_lease();
    return csr_;
  }

  std::vector<double> diagonal() const {
    if (kind_ == OperatorKind::EXPLICIT) {
      validate_lease();
      sync_values();
    }
    std::vector<double> d(static_cast<std::size_t>(n_));
    b200_dropin::check(afem_op_diagonal(dev_->h, d.data()));
    return d;
  }

  friend LinearOperator explicit_operator(const HandoffBuffer& buffer);
  friend LinearOperator matrix_free_operator(std::span<const ElementBatch> batches, std::span<const double> u,
                                             const DirichletSpec& dirichlet);
  friend std::pair<std::vector<double>, SolveReport> run_solver(const LinearOperator& op, std::span<const double> b,
                                                                const SolverConfig& cfg);

 private:
  LinearOperator() = default;

  void validate_lease() const {
    if (buffer_->state() != LeaseState::LeasedToSolver)
      throw LeaseError("explicit operator used while the buffer lease is not held");
    if (buffer_->epoch() != epoch_) throw StaleEpochError("explicit operator built from a stale assembly epoch");
  }
  // the solver-side storage may have been written since the last upload: reload it then
  void sync_values() const {
    const std::uint64_t v = buffer_->values_version();
    if (synced_ == v) return;
    b200_dropin::check(afem_op_set_values(dev_->h, csr_.values().data()));
    synced_ = v;
  }

  OperatorKind kind_ = OperatorKind::EXPLICIT;
  int n_ = 0;
  std::shared_ptr<b200_dropin::OpHandle> dev_;
  // explicit realization: the reference's aliasing CSR view + the buffer it leases from
  CsrMatrix csr_;
  const HandoffBuffer* buffer_ = nullptr;
  std::uint64_t epoch_ = 0;
  mutable std::uint64_t synced_ = ~0ull;  // values_version() of the device copy
  // matrix-free realization: the mirror keeps the device system alive
  std::shared_ptr<b200_dropin::Mirror> mirror_;
};

/// CSR view over a leased buffer (backend.hpp:199-214); pattern arrays alias the precomputed
/// pattern, values alias the handoff storage.
inline LinearOperator explicit_operator(const HandoffBuffer& buffer) {
  if (buffer.state() != LeaseState::LeasedToSolver) throw LeaseError("explicit_operator: buffer must be leased to the solver");
  const auto pattern = buffer.pattern_handle();
  LinearOperator op;
  op.kind_ = OperatorKind::EXPLICIT;
  op.n_ = pattern->n_dof;
  op.csr_ = CsrMatrix(pattern->n_dof, std::shared_ptr<const std::vector<int>>(pattern, &pattern->row_ptr),
                      std::shared_ptr<const std::vector<int>>(pattern, &pattern->cols), buffer.value_store());
  op.buffer_ = &buffer;
  op.epoch_ = buffer.epoch();
  afem_op h = nullptr;
  b200_dropin::check(afem_op_create_csr(b200_dropin::context(), pattern->n_dof,
                                        static_cast<std::int64_t>(pattern->cols.size()), pattern->row_ptr.data(),
                                        pattern->cols.data(), &h));
  op.dev_ = std::make_shared<b200_dropin::OpHandle>(h);
  return op;
}

/// Matrix-free operator at state u (backend.hpp:222-236): the device mirror of the batches with
/// the given constraint table; state and mask are copied, the Jacobi diagonal (unit on
/// constrained dofs) is assembled once.
inline LinearOperator matrix_free_operator(std::span<const ElementBatch> batches, std::span<const double> u,
                                           const DirichletSpec& dirichlet) {
  (void)detail::constraint_table(dirichlet, u.size());  // the reference's range / duplicate checks
  auto m = b200_dropin::mirror(batches, static_cast<int>(u.size()));
  std::vector<std::int32_t> node, comp;
  std::vector<double> val;
  for (const DirichletConstraint& c : dirichlet.constraints) {
    node.push_back(c.node);
    comp.push_back(c.component);
    val.push_back(c.value);
  }
  b200_dropin::check(afem_set_dirichlet(m->sys->h, static_cast<std::int64_t>(node.size()), node.data(), comp.data(),
                                        val.data()));
  afem_op h = nullptr;
  b200_dropin::check(afem_op_create_mf(m->sys->h, u.data(), &h));
  LinearOperator op;
  op.kind_ = OperatorKind::MATRIX_FREE;
  op.n_ = static_cast<int>(u.size());
  op.dev_ = std::make_shared<b200_dropin::OpHandle>(h);
  op.mirror_ = m;
  return op;
}

namespace b200_dropin {

inline std::pair<std::vector<double>, SolveReport> solve_on(afem_op h, std::span<const double> b,
                                                           const SolverConfig& cfg) {
  const afem_solver_cfg c = to_afem(cfg);
  std::vector<double> x(b.size(), 0.0);
  std::vector<double> hist(static_cast<std::size_t>(cfg.max_iter) + 4);
  afem_solve_report rep{};
  check(afem_solve(h, &c, b.data(), nullptr, x.data(), &rep, hist.data(), static_cast<std::int32_t>(hist.size())));
  return {std::move(x), from_afem(rep, hist)};
}

}  // namespace b200_dropin

/// One linear solve (backend.hpp:241-286) on the device.
inline std::pair<std::vector<double>, SolveReport> run_solver(const LinearOperator& op, std::span<const double> b,
                                                              const SolverConfig& cfg) {
  cfg.validate();
  if (static_cast<int>(b.size()) != op.dim()) throw std::invalid_argument("run_solver: dimension mismatch");
  if (op.kind() == OperatorKind::MATRIX_FREE) return b200_dropin::solve_on(op.dev_->h, b, cfg);
  const CsrMatrix& a = op.csr();  // lease + epoch checks
  const bool needs_system = cfg.method == SolverMethod::DIRECT_CHOL || cfg.method == SolverMethod::DIRECT_LU ||
                            cfg.preconditioner == PreconKind::ILU0;
  if (!needs_system) {
    op.sync_values();
    return b200_dropin::solve_on(op.dev_->h, b, cfg);
  }
  // ILU(0) / banded direct: on the device system the pattern was built from
  auto m = b200_dropin::mirror_of(op.buffer_->pattern_handle().get());
  if (!m)
    throw CapabilityError("run_solver (B200): ILU0 and direct factorisations need a pattern from precompute_sparsity");
  afem_values v = nullptr;
  b200_dropin::check(afem_values_create(m->sys->h, &v));
  afem_buffer buf = nullptr;
  afem_op h = nullptr;
  struct Cleanup {
    afem_values* v;
    afem_buffer* b;
    afem_op* h;
    ~Cleanup() {
      if (*h) afem_op_destroy(*h);
      if (*b) afem_buffer_destroy(*b);
      if (*v) afem_values_destroy(*v);
    }
  } cleanup{&v, &buf, &h};
  b200_dropin::check(afem_values_set(v, a.values().data()));
  b200_dropin::check(afem_buffer_create(m->sys->h, &buf));
  b200_dropin::check(afem_buffer_handoff(buf, &v));  // moves the values into the buffer (v -> null)
  b200_dropin::check(afem_op_create_explicit(buf, &h));
  return b200_dropin::solve_on(h, b, cfg);
}

}  // namespace adfem

#endif  // ADFEM_BACKEND_HPP
