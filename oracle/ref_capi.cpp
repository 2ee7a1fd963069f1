// TEST INFRASTRUCTURE ONLY — C ABI (oracle/orc_api.h) over the UNMODIFIED reference headers.
//
// Compiled by oracle/Makefile with -I/root/reference/proj/include into oracle/_ref/libadfem_ref.so.
// Nothing here re-implements the algorithm: every entry point forwards to the reference function
// named in its comment. 2D only (the reference is quad4/plane-strain only, element.hpp:16-54).
#include <cstring>
#include <memory>
#include <string>

#include "adfem/adfem.hpp"
#include "orc_api.h"

namespace {
thread_local std::string g_err;

template <class F>
int32_t guarded(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const adfem::LeaseError& e) { g_err = e.what(); return ORC_E_LEASE;
  } catch (const adfem::StaleEpochError& e) { g_err = e.what(); return ORC_E_STALE_EPOCH;
  } catch (const adfem::CapabilityError& e) { g_err = e.what(); return ORC_E_CAPABILITY;
  } catch (const adfem::FactorizationError& e) { g_err = e.what(); return ORC_E_FACTORIZATION;
  } catch (const adfem::InvertedElementError& e) { g_err = e.what(); return ORC_E_INVERTED_ELEMENT;
  } catch (const std::invalid_argument& e) { g_err = e.what(); return ORC_E_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) { g_err = e.what(); return ORC_E_OUT_OF_RANGE;
  } catch (const std::domain_error& e) { g_err = e.what(); return ORC_E_DOMAIN;
  } catch (const std::logic_error& e) { g_err = e.what(); return ORC_E_LOGIC;
  } catch (const std::exception& e) { g_err = e.what(); return ORC_E_RUNTIME; }
}

struct RefSystem {
  adfem::Mesh mesh;
  std::vector<adfem::Material> materials;
  std::vector<adfem::ElementBatch> batches;
  std::shared_ptr<const adfem::SparsityPattern> pattern;
  adfem::DirichletSpec bcs;
  std::size_t n() const { return static_cast<std::size_t>(mesh.n_dof()); }
};

RefSystem* S(void* p) { return static_cast<RefSystem*>(p); }

adfem::SolverConfig to_cfg(const orc_solver_cfg* c) {
  adfem::SolverConfig s;
  s.method = static_cast<adfem::SolverMethod>(c->method);
  s.preconditioner = static_cast<adfem::PreconKind>(c->precond);
  s.rtol = c->rtol;
  s.max_iter = c->max_iter;
  s.gmres_restart = c->restart;
  return s;
}

adfem::NewtonConfig to_ncfg(const orc_newton_cfg* c) {
  adfem::NewtonConfig n;
  n.rtol = c->rtol;
  n.atol = c->atol;
  n.max_iter = c->max_iter;
  n.operator_kind = c->operator_kind == 0 ? adfem::OperatorKind::EXPLICIT : adfem::OperatorKind::MATRIX_FREE;
  n.linear = to_cfg(&c->linear);
  return n;
}

void fill_report(const adfem::SolveReport& r, orc_solve_report* out, double* hist, int32_t cap) {
  out->converged = r.converged;
  out->iterations = r.iterations;
  out->n_history = static_cast<int32_t>(r.residual_history.size());
  out->wall_time = r.wall_time;
  std::snprintf(out->failure, sizeof out->failure, "%s", r.failure.c_str());
  if (hist)
    for (int32_t i = 0; i < cap && i < out->n_history; ++i) hist[i] = r.residual_history[i];
}

void fill_newton(const adfem::NewtonReport& r, orc_newton_report* out, double* norms, int32_t cap) {
  out->converged = r.converged;
  out->iterations = r.iterations;
  out->n_norms = static_cast<int32_t>(r.residual_norms.size());
  out->total_time = r.total_time;
  int tot = 0;
  for (const auto& l : r.linear_reports) tot += l.iterations;
  out->total_linear_iterations = tot;
  std::snprintf(out->failure, sizeof out->failure, "%s", r.failure.c_str());
  if (norms)
    for (int32_t i = 0; i < cap && i < out->n_norms; ++i) norms[i] = r.residual_norms[i];
}

template <class Op>
std::pair<std::vector<double>, adfem::SolveReport> solve_with(const Op& op, std::span<const double> b,
                                                              const adfem::SolverConfig& cfg, const double* x0) {
  if (!x0) return adfem::run_solver(op, b, cfg);  // backend.hpp:241
  std::span<const double> xs(x0, b.size());
  auto go = [&](const auto& m) {
    return cfg.method == adfem::SolverMethod::CG ? adfem::cg(op, b, cfg, m, xs) : adfem::gmres(op, b, cfg, m, xs);
  };
  if (cfg.preconditioner == adfem::PreconKind::JACOBI)
    return go(adfem::JacobiPreconditioner::from_diagonal(op.diagonal()));
  return go(adfem::IdentityPreconditioner{});
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int32_t orc_dims_supported(void) { return 1 << 2; }

int32_t orc_mesh2d(int32_t nx, int32_t ny, double lx, double ly, double cx, double cy, double radius,
                   double* coords, int32_t* conn, int32_t* phase) {
  return guarded([&] {
    const adfem::Mesh m = adfem::generate_two_phase_mesh(nx, ny, lx, ly, {cx, cy}, radius);  // mesh.hpp:47
    for (int i = 0; i < m.n_nodes(); ++i) { coords[2 * i] = m.nodes[i][0]; coords[2 * i + 1] = m.nodes[i][1]; }
    for (int e = 0; e < m.n_elements(); ++e) {
      for (int k = 0; k < 4; ++k) conn[4 * e + k] = m.elements[e][k];
      phase[e] = m.material_of[e];
    }
  });
}

int32_t orc_mesh3d(int32_t, int32_t, int32_t, double, double, double, int32_t, const double*, double, double*,
                   int32_t*, int32_t*) {
  g_err = "reference has no 3D mesh generator";
  return ORC_E_CAPABILITY;
}

int32_t orc_fibres(uint64_t, int32_t, double, double, double*) {
  g_err = "reference has no fibre generator";
  return ORC_E_CAPABILITY;
}

int64_t orc_bcs(int32_t dim, int32_t nx, int32_t ny, int32_t, double lx, double strain, int32_t* node,
                int32_t* comp, double* value) {
  int64_t n = -1;
  const int32_t st = guarded([&] {
    if (dim != 2) throw adfem::CapabilityError("reference benchmark_bcs is 2D only");
    adfem::Mesh m;  // benchmark_bcs reads only the grid metadata (mesh.hpp:89-101)
    m.nx = nx; m.ny = ny; m.lx = lx;
    const auto spec = adfem::benchmark_bcs(m, strain);
    n = static_cast<int64_t>(spec.constraints.size());
    if (node)
      for (std::size_t i = 0; i < spec.constraints.size(); ++i) {
        node[i] = spec.constraints[i].node; comp[i] = spec.constraints[i].component; value[i] = spec.constraints[i].value;
      }
  });
  return st == ORC_OK ? n : -static_cast<int64_t>(st);
}

void* orc_system_create(int32_t dim, int64_t n_nodes, int64_t n_elem, const double* coords, const int32_t* conn,
                        const int32_t* phase, int32_t n_mat, const orc_material* mats) {
  RefSystem* out = nullptr;
  guarded([&] {
    if (dim != 2) throw adfem::CapabilityError("reference is 2D only");
    auto s = std::make_unique<RefSystem>();
    for (int64_t i = 0; i < n_nodes; ++i) s->mesh.nodes.push_back({coords[2 * i], coords[2 * i + 1]});
    for (int64_t e = 0; e < n_elem; ++e) {
      s->mesh.elements.push_back({conn[4 * e], conn[4 * e + 1], conn[4 * e + 2], conn[4 * e + 3]});
      s->mesh.material_of.push_back(phase[e]);
    }
    for (int i = 0; i < n_mat; ++i)
      s->materials.push_back(adfem::Material{static_cast<adfem::MaterialModel>(mats[i].model), mats[i].E, mats[i].nu});
    s->batches = adfem::build_batches(s->mesh, s->materials);                  // assembly.hpp:36
    s->pattern = adfem::precompute_sparsity(s->batches, s->mesh.n_dof());      // assembly.hpp:71
    out = s.release();
  });
  return out;
}

void* orc_system_create_lite(int32_t dim, int64_t n_nodes, int64_t n_elem, const double* coords,
                             const int32_t* conn, const int32_t* phase, int32_t n_mat, const orc_material* mats) {
  return orc_system_create(dim, n_nodes, n_elem, coords, conn, phase, n_mat, mats);
}

int32_t orc_system_set_grid(void* sys, int32_t nx, int32_t ny, int32_t, double lx, double ly, double) {
  return guarded([&] {
    auto& m = S(sys)->mesh;
    m.nx = nx; m.ny = ny; m.lx = lx; m.ly = ly;
  });
}

void orc_system_destroy(void* sys) { delete S(sys); }
int64_t orc_n_dof(void* sys) { return S(sys)->mesh.n_dof(); }
int32_t orc_n_batches(void* sys) { return static_cast<int32_t>(S(sys)->batches.size()); }

int32_t orc_batch_info(void* sys, int32_t b, int64_t* size, int32_t* element_ids, int32_t* dof_map) {
  return guarded([&] {
    const auto& bb = S(sys)->batches.at(b);
    *size = static_cast<int64_t>(bb.size());
    for (std::size_t e = 0; e < bb.size(); ++e) {
      if (element_ids) element_ids[e] = bb.element_ids[e];
      if (dof_map) for (int k = 0; k < 8; ++k) dof_map[8 * e + k] = bb.dof_map[e][k];
    }
  });
}

int32_t orc_set_dirichlet(void* sys, int64_t n, const int32_t* node, const int32_t* comp, const double* value) {
  return guarded([&] {
    auto* s = S(sys);
    adfem::DirichletSpec spec;
    for (int64_t i = 0; i < n; ++i) spec.constraints.push_back({node[i], comp[i], value[i]});
    adfem::validate_dirichlet(spec, s->mesh);  // mesh.hpp:105
    s->bcs = std::move(spec);
  });
}

int64_t orc_pattern_nnz(void* sys) { return static_cast<int64_t>(S(sys)->pattern->nnz()); }

int32_t orc_pattern(void* sys, int64_t* row_ptr, int32_t* rows, int32_t* cols) {
  return guarded([&] {
    const auto& p = *S(sys)->pattern;
    if (row_ptr) for (std::size_t i = 0; i < p.row_ptr.size(); ++i) row_ptr[i] = p.row_ptr[i];
    if (rows) std::memcpy(rows, p.rows.data(), p.rows.size() * 4);
    if (cols) std::memcpy(cols, p.cols.data(), p.cols.size() * 4);
  });
}

int32_t orc_residual(void* sys, const double* u, double* r) {
  return guarded([&] {
    auto* s = S(sys);
    const auto out = adfem::assemble_residual(s->batches, std::span<const double>(u, s->n()));  // assembly.hpp:126
    std::memcpy(r, out.data(), out.size() * 8);
  });
}

int32_t orc_element_residual(void* sys, int64_t e, const double* ue, double* re) {
  return guarded([&] {
    auto* s = S(sys);
    adfem::ElementState st;
    for (int k = 0; k < 4; ++k) st.coords[k] = s->mesh.nodes[s->mesh.elements[e][k]];
    for (int k = 0; k < 8; ++k) st.u[k] = ue[k];
    st.material = s->materials.at(s->mesh.material_of[e]);
    const auto r = adfem::element_residual(st, 2);  // element.hpp:127
    for (int k = 0; k < 8; ++k) re[k] = r[k];
  });
}

int32_t orc_jacobian(void* sys, const double* u, double* values) {
  return guarded([&] {
    auto* s = S(sys);
    const auto coo = adfem::assemble_jacobian(s->batches, std::span<const double>(u, s->n()), *s->pattern);
    std::memcpy(values, coo.values.data(), coo.values.size() * 8);  // assembly.hpp:144
  });
}

int32_t orc_diagonal(void* sys, const double* u, double* d) {
  return guarded([&] {
    auto* s = S(sys);
    const auto out = adfem::assemble_diagonal(s->batches, std::span<const double>(u, s->n()));  // assembly.hpp:177
    std::memcpy(d, out.data(), out.size() * 8);
  });
}

int32_t orc_eliminate(void* sys, double* values, double* residual, const double* u) {
  return guarded([&] {
    auto* s = S(sys);
    adfem::apply_dirichlet(*s->pattern, std::span<double>(values, s->pattern->nnz()),
                           std::span<double>(residual, s->n()), s->bcs, std::span<const double>(u, s->n()));
  });
}

int32_t orc_constrain_residual(void* sys, double* residual, const double* u) {
  return guarded([&] {
    auto* s = S(sys);
    adfem::constrain_residual(std::span<double>(residual, s->n()), s->bcs, std::span<const double>(u, s->n()));
  });
}

int32_t orc_mf_apply(void* sys, const double* u, const double* x, double* y) {
  return guarded([&] {
    auto* s = S(sys);
    const auto op = adfem::matrix_free_operator(s->batches, std::span<const double>(u, s->n()), s->bcs);
    op.apply(std::span<const double>(x, s->n()), std::span<double>(y, s->n()));  // backend.hpp:122
  });
}

int32_t orc_mf_apply_mt(void* sys, const double* u, const double* x, double* y, int32_t) {
  return orc_mf_apply(sys, u, x, y);  // the reference is single-threaded
}

int32_t orc_mf_diagonal(void* sys, const double* u, double* d) {
  return guarded([&] {
    auto* s = S(sys);
    const auto op = adfem::matrix_free_operator(s->batches, std::span<const double>(u, s->n()), s->bcs);
    const auto dg = op.diagonal();
    std::memcpy(d, dg.data(), dg.size() * 8);
  });
}

int32_t orc_mf_diagonal_mt(void* sys, const double* u, double* d, int32_t) {
  return orc_mf_diagonal(sys, u, d);  // the reference is single-threaded
}

int32_t orc_csr_apply(void* sys, const double* values, const double* x, double* y) {
  return guarded([&] {
    auto* s = S(sys);
    const auto& p = *s->pattern;
    adfem::CsrMatrix a(p.n_dof, p.row_ptr, p.cols, std::vector<double>(values, values + p.nnz()));
    a.apply(std::span<const double>(x, s->n()), std::span<double>(y, s->n()));  // sparse.hpp:106
  });
}

int32_t orc_solve(void* sys, int32_t op_kind, const double* values_or_u, const orc_solver_cfg* cfg, const double* b,
                  const double* x0, double* x, orc_solve_report* rep, double* history, int32_t hist_cap) {
  return guarded([&] {
    auto* s = S(sys);
    const adfem::SolverConfig c = to_cfg(cfg);
    std::span<const double> bs(b, s->n());
    std::pair<std::vector<double>, adfem::SolveReport> res;
    if (op_kind == 0) {
      const auto& p = *s->pattern;
      adfem::CooTriplets coo;
      coo.n = p.n_dof; coo.rows = p.rows; coo.cols = p.cols;
      coo.values.assign(values_or_u, values_or_u + p.nnz());
      adfem::HandoffBuffer buffer(s->pattern);  // backend.hpp:33
      buffer.handoff(std::move(coo));
      adfem::LeaseGuard guard(buffer);
      const adfem::LinearOperator op = adfem::explicit_operator(buffer);
      res = solve_with(op, bs, c, x0);
    } else {
      const adfem::LinearOperator op =
          adfem::matrix_free_operator(s->batches, std::span<const double>(values_or_u, s->n()), s->bcs);
      res = solve_with(op, bs, c, x0);
    }
    std::memcpy(x, res.first.data(), res.first.size() * 8);
    fill_report(res.second, rep, history, hist_cap);
  });
}

int32_t orc_solve_bvp(void* sys, const orc_newton_cfg* cfg, const double* x0, double* u, orc_newton_report* rep,
                      double* norms, int32_t norms_cap) {
  return guarded([&] {
    auto* s = S(sys);
    std::span<const double> guess;
    if (x0) guess = std::span<const double>(x0, s->n());
    auto [uu, r] = adfem::solve_bvp(s->mesh, s->materials, s->bcs, to_ncfg(cfg), guess);  // newton.hpp:59
    std::memcpy(u, uu.data(), uu.size() * 8);
    fill_newton(r, rep, norms, norms_cap);
  });
}

int32_t orc_load_stepping(void* sys, double total_strain, int32_t n_steps, const orc_newton_cfg* cfg, double* u,
                          int32_t* failed_step, int32_t* converged, int32_t* step_iterations) {
  return guarded([&] {
    auto* s = S(sys);
    auto [uu, r] = adfem::load_stepping(s->mesh, s->materials, total_strain, to_ncfg(cfg), n_steps);  // newton.hpp:163
    std::memcpy(u, uu.data(), uu.size() * 8);
    *failed_step = r.failed_step;
    *converged = r.converged;
    if (step_iterations)
      for (std::size_t i = 0; i < r.steps.size(); ++i) step_iterations[i] = r.steps[i].iterations;
  });
}

}  // extern "C"
