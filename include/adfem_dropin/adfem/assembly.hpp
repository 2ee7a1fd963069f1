// adfem/assembly.hpp — B200 drop-in for the reference's assembly layer (proj/include/adfem/
// assembly.hpp). Same namespace, types and signatures; the hot-path functions run on the device:
//
//   precompute_sparsity   (assembly.hpp:71-99)   device pattern build, bit-exact rows/cols/row_ptr
//   assemble_residual     (assembly.hpp:126-139) element kernels + ordered node gather on the device
//   assemble_jacobian     (assembly.hpp:144-173) hand-derived tangents, slot-indexed, pattern order
//   assemble_diagonal     (assembly.hpp:177-188)
//   apply_dirichlet / detail::eliminate_dirichlet / constrain_residual (assembly.hpp:218-260)
//
// The batch-level API carries no mesh handle, so the device keeps a MIRROR of the batches: one
// device system per distinct batch content (elements laid out batch by batch, phase = batch index,
// so the device's (phase, element) scatter order is the reference's (batch, element) order), keyed
// by a hash of the batches' dof maps, coordinates and materials and built on first use.
// build_batches, the constraint table and write_triplets are host bookkeeping, as in the
// reference. detail::BatchKernel / gather_states keep the reference's CPU AD kernel for callers
// that differentiate a single element (tests, verify.hpp).
#ifndef ADFEM_ASSEMBLY_HPP
#define ADFEM_ASSEMBLY_HPP

#include <algorithm>
#include <array>
#include <cstdio>
#include <list>
#include <memory>
#include <mutex>
#include <ostream>
#include <span>
#include <stdexcept>
#include <vector>

#include "adfem/autodiff.hpp"
#include "adfem/b200_device.hpp"
#include "adfem/element.hpp"
#include "adfem/mesh.hpp"
#include "adfem/sparse.hpp"

namespace adfem {

/// Homogeneous group of elements (assembly.hpp:22-32).
struct ElementBatch {
  std::vector<int> element_ids;
  std::vector<std::array<int, 4>> connectivity;
  std::vector<std::array<int, 8>> dof_map;
  std::vector<ElementCoords> coords;
  Material material;
  int quadrature = 2;

  std::size_t size() const { return element_ids.size(); }
};

/// One batch per phase present, in phase order, mesh order inside a batch, empty phases dropped
/// (assembly.hpp:36-67).
inline std::vector<ElementBatch> build_batches(const Mesh& mesh, std::span<const Material> phase_materials) {
  int top = -1;
  for (int p : mesh.material_of) top = std::max(top, p);
  if (top >= static_cast<int>(phase_materials.size()))
    throw std::invalid_argument("build_batches: no material supplied for a mesh phase");
  for (const Material& m : phase_materials) m.validate();
  std::vector<ElementBatch> out(static_cast<std::size_t>(top + 1));
  for (std::size_t p = 0; p < out.size(); ++p) out[p].material = phase_materials[p];
  for (int e = 0; e < mesh.n_elements(); ++e) {
    ElementBatch& b = out[static_cast<std::size_t>(mesh.material_of[static_cast<std::size_t>(e)])];
    const std::array<int, 4>& q = mesh.elements[static_cast<std::size_t>(e)];
    std::array<int, 8> dofs{};
    ElementCoords xy{};
    for (int k = 0; k < 4; ++k) {
      dofs[2 * k] = 2 * q[k];
      dofs[2 * k + 1] = 2 * q[k] + 1;
      xy[k] = mesh.nodes[static_cast<std::size_t>(q[k])];
    }
    b.element_ids.push_back(e);
    b.connectivity.push_back(q);
    b.dof_map.push_back(dofs);
    b.coords.push_back(xy);
  }
  std::erase_if(out, [](const ElementBatch& b) { return b.size() == 0; });
  return out;
}

namespace b200_dropin {

// Device system mirroring a batch set (see the file comment).
struct Mirror {
  std::unique_ptr<SystemHandle> sys;
  int n_dof = 0;
  std::int64_t nnz = 0;
  std::shared_ptr<const SparsityPattern> pattern;  // host copy, built on first request
};

inline std::uint64_t batches_key(std::span<const ElementBatch> batches, int n_dof) {
  Fnv f;
  f.pod(context());  // mirrors are per thread context (a context's stream is not shared across threads)
  f.pod(n_dof);
  f.pod(batches.size());
  for (const ElementBatch& b : batches) {
    f.pod(b.material.model);
    f.pod(b.material.E);
    f.pod(b.material.nu);
    f.pod(b.quadrature);
    f.pod(b.size());
    f.add(b.dof_map.data(), b.dof_map.size() * sizeof(b.dof_map[0]));
    f.add(b.coords.data(), b.coords.size() * sizeof(b.coords[0]));
  }
  return f.h;
}

inline std::shared_ptr<Mirror> build_mirror(std::span<const ElementBatch> batches, int n_dof) {
  if (n_dof < 0 || n_dof % 2 != 0) throw std::invalid_argument("assembly: n_dof must be 2 x n_nodes");
  const std::int64_t n_nodes = n_dof / 2;
  std::int64_t n_elem = 0;
  for (const ElementBatch& b : batches) {
    if (b.quadrature != 2)
      throw std::invalid_argument("assembly (B200): only the 2x2 Gauss rule is implemented on the device");
    if (b.dof_map.size() != b.size() || b.coords.size() != b.size())
      throw std::invalid_argument("assembly: inconsistent batch arrays");
    n_elem += static_cast<std::int64_t>(b.size());
  }
  std::vector<double> xy(static_cast<std::size_t>(2 * n_nodes), 0.0);
  std::vector<std::int32_t> conn;
  std::vector<std::int32_t> phase;
  std::vector<afem_material> mats;
  conn.reserve(static_cast<std::size_t>(4 * n_elem));
  phase.reserve(static_cast<std::size_t>(n_elem));
  for (std::size_t bi = 0; bi < batches.size(); ++bi) {
    const ElementBatch& b = batches[bi];
    mats.push_back(to_afem(b.material));
    for (std::size_t e = 0; e < b.size(); ++e) {
      for (int k = 0; k < 4; ++k) {
        const int dx = b.dof_map[e][2 * k], dy = b.dof_map[e][2 * k + 1];
        if (dx < 0 || dy < 0 || dx >= n_dof || dy >= n_dof)
          throw std::out_of_range("assembly: dof index outside system");
        if (dx % 2 != 0 || dy != dx + 1)
          throw std::invalid_argument("assembly (B200): dof_map must interleave node components");
        const int node = dx / 2;
        conn.push_back(node);
        xy[static_cast<std::size_t>(2 * node)] = b.coords[e][static_cast<std::size_t>(k)][0];
        xy[static_cast<std::size_t>(2 * node + 1)] = b.coords[e][static_cast<std::size_t>(k)][1];
      }
      phase.push_back(static_cast<std::int32_t>(bi));
    }
  }
  afem_system h = nullptr;
  check(afem_system_create(context(), 2, n_nodes, n_elem, xy.data(), conn.data(), phase.data(),
                           static_cast<std::int32_t>(mats.size()), mats.data(), &h));
  auto m = std::make_shared<Mirror>();
  m->sys = std::make_unique<SystemHandle>(h);
  m->n_dof = n_dof;
  check(afem_pattern_nnz(h, &m->nnz));
  return m;
}

struct Registry {
  std::mutex mu;
  std::list<std::pair<std::uint64_t, std::shared_ptr<Mirror>>> mirrors;  // most recent first
  // patterns handed out by precompute_sparsity -> their mirror
  std::vector<std::pair<std::weak_ptr<const SparsityPattern>, std::weak_ptr<Mirror>>> patterns;
  static Registry& get() {
    static Registry r;
    return r;
  }
};

// The device mirror of (batches, n_dof), built on first use; a few recent ones stay resident.
inline std::shared_ptr<Mirror> mirror(std::span<const ElementBatch> batches, int n_dof) {
  const std::uint64_t key = batches_key(batches, n_dof);
  Registry& r = Registry::get();
  std::lock_guard<std::mutex> lk(r.mu);
  for (auto it = r.mirrors.begin(); it != r.mirrors.end(); ++it)
    if (it->first == key) {
      r.mirrors.splice(r.mirrors.begin(), r.mirrors, it);
      return r.mirrors.front().second;
    }
  auto m = build_mirror(batches, n_dof);
  r.mirrors.emplace_front(key, m);
  if (r.mirrors.size() > 8) r.mirrors.pop_back();
  return m;
}

inline std::shared_ptr<const SparsityPattern> device_pattern(Mirror& m) {
  if (m.pattern) return m.pattern;
  auto p = std::make_shared<SparsityPattern>();
  p->n_dof = m.n_dof;
  std::vector<std::int64_t> rp(static_cast<std::size_t>(m.n_dof) + 1);
  p->rows.resize(static_cast<std::size_t>(m.nnz));
  p->cols.resize(static_cast<std::size_t>(m.nnz));
  check(afem_pattern(m.sys->h, rp.data(), p->rows.data(), p->cols.data()));
  p->row_ptr.assign(rp.begin(), rp.end());
  m.pattern = p;
  return p;
}

inline void register_pattern(const std::shared_ptr<const SparsityPattern>& p, const std::shared_ptr<Mirror>& m) {
  Registry& r = Registry::get();
  std::lock_guard<std::mutex> lk(r.mu);
  std::erase_if(r.patterns, [](const auto& e) { return e.first.expired() || e.second.expired(); });
  r.patterns.emplace_back(p, m);
}

// The mirror a pattern object came from (nullptr for patterns built by hand).
inline std::shared_ptr<Mirror> mirror_of(const SparsityPattern* p) {
  Registry& r = Registry::get();
  std::lock_guard<std::mutex> lk(r.mu);
  for (const auto& e : r.patterns) {
    auto sp = e.first.lock();
    if (sp && sp.get() == p) return e.second.lock();
  }
  return nullptr;
}

}  // namespace b200_dropin

/// Union of the per-element blocks, sorted and duplicate-free (assembly.hpp:71-99): built on the
/// device (node adjacency, closed-form row pointers), bit-exact with the reference.
inline std::shared_ptr<const SparsityPattern> precompute_sparsity(std::span<const ElementBatch> batches, int n_dof) {
  for (const ElementBatch& b : batches)
    for (const auto& dofs : b.dof_map)
      for (int d : dofs)
        if (d >= n_dof) throw std::out_of_range("precompute_sparsity: dof index outside system");
  auto m = b200_dropin::mirror(batches, n_dof);
  // a fresh pattern object per call (callers own and compare them), same content every time
  auto p = std::make_shared<const SparsityPattern>(*b200_dropin::device_pattern(*m));
  b200_dropin::register_pattern(p, m);
  return p;
}

namespace detail {

/// The reference's element residual family over one batch (assembly.hpp:104-113), for callers that
/// differentiate single elements on the host (element tests, verify.hpp FD-vs-AD).
struct BatchKernel {
  const ElementBatch* batch;

  template <class T>
  std::vector<T> operator()(std::size_t e, std::span<const T> u) const {
    std::array<T, 8> r;
    element_internal_force<T>(batch->coords[e], batch->material, batch->quadrature, u, r);
    return std::vector<T>(r.begin(), r.end());
  }
};

inline std::vector<std::vector<double>> gather_states(const ElementBatch& b, std::span<const double> u) {
  std::vector<std::vector<double>> xs(b.size(), std::vector<double>(8));
  for (std::size_t e = 0; e < b.size(); ++e)
    for (std::size_t k = 0; k < 8; ++k) xs[e][k] = u[static_cast<std::size_t>(b.dof_map[e][k])];
  return xs;
}

}  // namespace detail

/// R(u) with the reference's (batch, element) summation order per dof (assembly.hpp:126-139).
inline std::vector<double> assemble_residual(std::span<const ElementBatch> batches, std::span<const double> u) {
  auto m = b200_dropin::mirror(batches, static_cast<int>(u.size()));
  std::vector<double> r(u.size(), 0.0);
  b200_dropin::check(afem_residual(m->sys->h, u.data(), r.data()));
  return r;
}

/// K(u) as sorted, deduplicated triplets in pattern order (assembly.hpp:144-173); the device writes
/// each element tangent block straight into its pattern slots (no sort). The produced pattern must
/// equal the given one, else logic_error, like the reference.
inline CooTriplets assemble_jacobian(std::span<const ElementBatch> batches, std::span<const double> u,
                                     const SparsityPattern& pattern) {
  auto m = b200_dropin::mirror(batches, static_cast<int>(u.size()));
  auto own = b200_dropin::device_pattern(*m);
  if (own->rows != pattern.rows || own->cols != pattern.cols)
    throw std::logic_error("assemble_jacobian: produced indices leave the precomputed pattern");
  CooTriplets coo;
  coo.n = pattern.n_dof;
  coo.rows = own->rows;
  coo.cols = own->cols;
  coo.values.resize(own->cols.size());
  b200_dropin::check(afem_jacobian(m->sys->h, u.data(), coo.values.data()));
  return coo;
}

/// diag K(u) (assembly.hpp:177-188).
inline std::vector<double> assemble_diagonal(std::span<const ElementBatch> batches, std::span<const double> u) {
  auto m = b200_dropin::mirror(batches, static_cast<int>(u.size()));
  std::vector<double> d(u.size(), 0.0);
  b200_dropin::check(afem_diagonal(m->sys->h, u.data(), d.data()));
  return d;
}

namespace detail {

struct ConstraintTable {
  std::vector<char> constrained;
  std::vector<double> prescribed;
};

/// Per-dof constraint table (assembly.hpp:197-211): range and duplicate checks.
inline ConstraintTable constraint_table(const DirichletSpec& spec, std::size_t n_dof) {
  ConstraintTable t;
  t.constrained.assign(n_dof, 0);
  t.prescribed.assign(n_dof, 0.0);
  for (const DirichletConstraint& c : spec.constraints) {
    const long dof = 2L * c.node + c.component;
    if (dof < 0 || dof >= static_cast<long>(n_dof)) throw std::out_of_range("dirichlet: constrained dof outside system");
    if (t.constrained[static_cast<std::size_t>(dof)])
      throw std::invalid_argument("dirichlet: duplicate (node, component) pair");
    t.constrained[static_cast<std::size_t>(dof)] = 1;
    t.prescribed[static_cast<std::size_t>(dof)] = c.value;
  }
  return t;
}

/// Symmetric elimination on CSR-ordered storage (assembly.hpp:218-240), on the device, in the
/// reference's operation order (bitwise identical results).
inline void eliminate_dirichlet(std::span<const int> row_ptr, std::span<const int> col_idx, std::span<double> values,
                                std::span<double> residual, const ConstraintTable& t, std::span<const double> u) {
  const std::int64_t n = static_cast<std::int64_t>(row_ptr.size()) - 1;
  if (n < 0) return;
  static_assert(sizeof(char) == sizeof(std::uint8_t));
  b200_dropin::check(afem_eliminate_csr(b200_dropin::context(), n, static_cast<std::int64_t>(col_idx.size()),
                                        row_ptr.data(), col_idx.data(), values.data(), residual.data(),
                                        reinterpret_cast<const std::uint8_t*>(t.constrained.data()),
                                        t.prescribed.data(), u.data()));
}

}  // namespace detail

/// apply_dirichlet on pattern-ordered values (assembly.hpp:242-249).
inline void apply_dirichlet(const SparsityPattern& pattern, std::span<double> values, std::span<double> residual,
                            const DirichletSpec& spec, std::span<const double> u) {
  if (values.size() != pattern.nnz()) throw std::invalid_argument("apply_dirichlet: value array does not match pattern");
  const auto t = detail::constraint_table(spec, u.size());
  detail::eliminate_dirichlet(pattern.row_ptr, pattern.cols, values, residual, t, u);
}

/// apply_dirichlet on a CSR matrix (assembly.hpp:251-254).
inline void apply_dirichlet(CsrMatrix& a, std::span<double> residual, const DirichletSpec& spec,
                            std::span<const double> u) {
  const auto t = detail::constraint_table(spec, u.size());
  detail::eliminate_dirichlet(a.row_ptr(), a.col_idx(), a.values(), residual, t, u);
}

/// Residual-only elimination (assembly.hpp:255-260).
inline void constrain_residual(std::span<double> residual, const DirichletSpec& spec, std::span<const double> u) {
  const auto t = detail::constraint_table(spec, u.size());
  if (residual.empty()) return;
  b200_dropin::check(afem_constrain_masked(b200_dropin::context(), static_cast<std::int64_t>(residual.size()),
                                           residual.data(), reinterpret_cast<const std::uint8_t*>(t.constrained.data()),
                                           t.prescribed.data(), u.data()));
}

/// `row col value` lines, 17 significant digits (assembly.hpp:264-271).
inline void write_triplets(std::ostream& os, const CooTriplets& coo) {
  char buf[96];
  for (std::size_t k = 0; k < coo.size(); ++k) {
    std::snprintf(buf, sizeof buf, "%d %d %.17g\n", coo.rows[k], coo.cols[k], coo.values[k]);
    os << buf;
  }
}

}  // namespace adfem

#endif  // ADFEM_ASSEMBLY_HPP
