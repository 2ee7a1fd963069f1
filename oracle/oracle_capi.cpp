// TEST INFRASTRUCTURE ONLY — C ABI (oracle/orc_api.h) over the CPU restatement in restate.hpp.
#include <cstring>
#include <string>

#include "orc_api.h"
#include "restate.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int32_t guarded(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const orc::LeaseError& e) { g_err = e.what(); return ORC_E_LEASE;
  } catch (const orc::StaleEpochError& e) { g_err = e.what(); return ORC_E_STALE_EPOCH;
  } catch (const orc::CapabilityError& e) { g_err = e.what(); return ORC_E_CAPABILITY;
  } catch (const orc::FactorizationError& e) { g_err = e.what(); return ORC_E_FACTORIZATION;
  } catch (const orc::InvertedElementError& e) { g_err = e.what(); return ORC_E_INVERTED_ELEMENT;
  } catch (const std::invalid_argument& e) { g_err = e.what(); return ORC_E_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) { g_err = e.what(); return ORC_E_OUT_OF_RANGE;
  } catch (const std::domain_error& e) { g_err = e.what(); return ORC_E_DOMAIN;
  } catch (const std::logic_error& e) { g_err = e.what(); return ORC_E_LOGIC;
  } catch (const std::exception& e) { g_err = e.what(); return ORC_E_RUNTIME; }
}

orc::System* S(void* p) { return static_cast<orc::System*>(p); }

orc::SolverConfig to_cfg(const orc_solver_cfg* c) {
  orc::SolverConfig s;
  s.method = c->method; s.precond = c->precond; s.rtol = c->rtol; s.max_iter = c->max_iter; s.restart = c->restart;
  return s;
}

void fill_report(const orc::SolveReport& r, orc_solve_report* out, double* hist, int32_t cap) {
  out->converged = r.converged;
  out->iterations = r.iterations;
  out->n_history = (int32_t)r.residual_history.size();
  out->wall_time = r.wall_time;
  std::snprintf(out->failure, sizeof out->failure, "%s", r.failure.c_str());
  if (hist)
    for (int32_t i = 0; i < cap && i < (int32_t)r.residual_history.size(); ++i) hist[i] = r.residual_history[i];
}

template <class F2, class F3>
void by_dim(orc::System* s, F2&& f2, F3&& f3) {
  if (s->dim() == 2) f2(); else f3();
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int32_t orc_dims_supported(void) { return (1 << 2) | (1 << 3); }

int32_t orc_mesh2d(int32_t nx, int32_t ny, double lx, double ly, double cx, double cy, double radius,
                   double* coords, int32_t* conn, int32_t* phase) {
  return guarded([&] {
    const orc::Mesh m = orc::mesh2d(nx, ny, lx, ly, cx, cy, radius);
    std::memcpy(coords, m.coords.data(), m.coords.size() * sizeof(double));
    std::memcpy(conn, m.conn.data(), m.conn.size() * sizeof(int32_t));
    std::memcpy(phase, m.phase.data(), m.phase.size() * sizeof(int32_t));
  });
}

int32_t orc_mesh3d(int32_t nx, int32_t ny, int32_t nz, double lx, double ly, double lz, int32_t n_fibres,
                   const double* fibres, double radius, double* coords, int32_t* conn, int32_t* phase) {
  return guarded([&] {
    std::vector<std::array<double, 2>> f;
    for (int i = 0; i < n_fibres; ++i) f.push_back({fibres[2 * i], fibres[2 * i + 1]});
    const orc::Mesh m = orc::mesh3d(nx, ny, nz, lx, ly, lz, f, radius);
    std::memcpy(coords, m.coords.data(), m.coords.size() * sizeof(double));
    std::memcpy(conn, m.conn.data(), m.conn.size() * sizeof(int32_t));
    std::memcpy(phase, m.phase.data(), m.phase.size() * sizeof(int32_t));
  });
}

int32_t orc_fibres(uint64_t seed, int32_t n, double lx, double ly, double* out) {
  return guarded([&] {
    const auto f = orc::fibres(seed, n, lx, ly);
    for (int i = 0; i < n; ++i) { out[2 * i] = f[i][0]; out[2 * i + 1] = f[i][1]; }
  });
}

int64_t orc_bcs(int32_t dim, int32_t nx, int32_t ny, int32_t nz, double lx, double strain, int32_t* node,
                int32_t* comp, double* value) {
  int64_t n = -1;
  const int32_t st = guarded([&] {
    const auto c = orc::benchmark_bcs(dim, nx, ny, nz, lx, strain);
    n = (int64_t)c.size();
    if (node)
      for (std::size_t i = 0; i < c.size(); ++i) { node[i] = c[i].node; comp[i] = c[i].comp; value[i] = c[i].value; }
  });
  return st == ORC_OK ? n : -(int64_t)st;
}

static void* create(int32_t dim, int64_t n_nodes, int64_t n_elem, const double* coords, const int32_t* conn,
                    const int32_t* phase, int32_t n_mat, const orc_material* mats, bool pattern);

void* orc_system_create(int32_t dim, int64_t n_nodes, int64_t n_elem, const double* coords, const int32_t* conn,
                        const int32_t* phase, int32_t n_mat, const orc_material* mats) {
  return create(dim, n_nodes, n_elem, coords, conn, phase, n_mat, mats, true);
}

void* orc_system_create_lite(int32_t dim, int64_t n_nodes, int64_t n_elem, const double* coords,
                             const int32_t* conn, const int32_t* phase, int32_t n_mat, const orc_material* mats) {
  return create(dim, n_nodes, n_elem, coords, conn, phase, n_mat, mats, false);
}

static void* create(int32_t dim, int64_t n_nodes, int64_t n_elem, const double* coords, const int32_t* conn,
                    const int32_t* phase, int32_t n_mat, const orc_material* mats, bool pattern) {
  orc::System* out = nullptr;
  guarded([&] {
    if (dim != 2 && dim != 3) throw std::invalid_argument("system: dim must be 2 or 3");
    auto s = std::make_unique<orc::System>();
    const int npe = dim == 2 ? 4 : 8;
    s->mesh.dim = dim;
    s->mesh.coords.assign(coords, coords + n_nodes * dim);
    s->mesh.conn.assign(conn, conn + n_elem * npe);
    s->mesh.phase.assign(phase, phase + n_elem);
    for (int i = 0; i < n_mat; ++i) {
      orc::Material m;
      m.model = mats[i].model; m.E = mats[i].E; m.nu = mats[i].nu;
      m.sigma_y = mats[i].sigma_y; m.hardening = mats[i].hardening;
      s->materials.push_back(m);
    }
    s->batches = orc::build_batches(s->mesh, s->materials);
    s->init_history();
    if (pattern) s->pattern = orc::precompute_sparsity(s->batches, s->n_dof(), dim);
    s->table = orc::constraint_table({}, s->n_dof(), dim);
    out = s.release();
  });
  return out;
}

int32_t orc_system_set_grid(void* sys, int32_t nx, int32_t ny, int32_t nz, double lx, double ly, double lz) {
  return guarded([&] {
    auto& m = S(sys)->mesh;
    m.nx = nx; m.ny = ny; m.nz = nz; m.lx = lx; m.ly = ly; m.lz = lz;
  });
}

void orc_system_destroy(void* sys) { delete S(sys); }
int64_t orc_n_dof(void* sys) { return S(sys)->n_dof(); }
int32_t orc_n_batches(void* sys) { return (int32_t)S(sys)->batches.size(); }

int32_t orc_batch_info(void* sys, int32_t b, int64_t* size, int32_t* element_ids, int32_t* dof_map) {
  return guarded([&] {
    const auto& bb = S(sys)->batches.at(b);
    *size = (int64_t)bb.size();
    if (element_ids) std::memcpy(element_ids, bb.element_ids.data(), bb.element_ids.size() * 4);
    if (dof_map) std::memcpy(dof_map, bb.dof_map.data(), bb.dof_map.size() * 4);
  });
}

int32_t orc_set_dirichlet(void* sys, int64_t n, const int32_t* node, const int32_t* comp, const double* value) {
  return guarded([&] {
    auto* s = S(sys);
    std::vector<orc::Constraint> c;
    for (int64_t i = 0; i < n; ++i) c.push_back({node[i], comp[i], value[i]});
    orc::validate_dirichlet(c, s->mesh.n_nodes(), s->dim());
    s->table = orc::constraint_table(c, s->n_dof(), s->dim());
    s->constraints = std::move(c);
  });
}

int64_t orc_pattern_nnz(void* sys) { return (int64_t)S(sys)->pattern.nnz(); }

int32_t orc_pattern(void* sys, int64_t* row_ptr, int32_t* rows, int32_t* cols) {
  return guarded([&] {
    const auto& p = S(sys)->pattern;
    if (row_ptr) std::memcpy(row_ptr, p.row_ptr.data(), p.row_ptr.size() * 8);
    if (rows) std::memcpy(rows, p.rows.data(), p.rows.size() * 4);
    if (cols) std::memcpy(cols, p.cols.data(), p.cols.size() * 4);
  });
}

int32_t orc_residual(void* sys, const double* u, double* r) {
  return guarded([&] {
    auto* s = S(sys);
    std::vector<double> out;
    by_dim(s, [&] { out = orc::assemble_residual<2>(s->batches, u, s->n_dof()); },
           [&] { out = orc::assemble_residual<3>(s->batches, u, s->n_dof()); });
    std::memcpy(r, out.data(), out.size() * 8);
  });
}

int32_t orc_element_residual(void* sys, int64_t e, const double* ue, double* re) {
  return guarded([&] {
    auto* s = S(sys);
    const int D = s->dim(), npe = D == 2 ? 4 : 8;
    std::vector<double> xc(npe * D);
    for (int k = 0; k < npe; ++k)
      for (int c = 0; c < D; ++c) xc[k * D + c] = s->mesh.coords[(size_t)s->mesh.conn[e * npe + k] * D + c];
    const orc::Material& m = s->materials.at(s->mesh.phase.at(e));
    const double* h = s->history.empty() ? nullptr : s->history.data() + (size_t)e * s->nq() * orc::kHist;
    if (D == 2) orc::element_internal_force<2, double>(xc.data(), m, 2, ue, re, h);
    else orc::element_internal_force<3, double>(xc.data(), m, 2, ue, re, h);
  });
}

int32_t orc_jacobian(void* sys, const double* u, double* values) {
  return guarded([&] {
    auto* s = S(sys);
    std::vector<double> v;
    by_dim(s, [&] { v = orc::assemble_jacobian<2>(*s, u); }, [&] { v = orc::assemble_jacobian<3>(*s, u); });
    std::memcpy(values, v.data(), v.size() * 8);
  });
}

int32_t orc_diagonal(void* sys, const double* u, double* d) {
  return guarded([&] {
    auto* s = S(sys);
    std::vector<double> v;
    by_dim(s, [&] { v = orc::assemble_diagonal<2>(s->batches, u, s->n_dof()); },
           [&] { v = orc::assemble_diagonal<3>(s->batches, u, s->n_dof()); });
    std::memcpy(d, v.data(), v.size() * 8);
  });
}

int32_t orc_eliminate(void* sys, double* values, double* residual, const double* u) {
  return guarded([&] {
    auto* s = S(sys);
    orc::eliminate_dirichlet(s->pattern, values, residual, s->table, u);
  });
}

int32_t orc_constrain_residual(void* sys, double* residual, const double* u) {
  return guarded([&] {
    auto* s = S(sys);
    for (int64_t d = 0; d < s->n_dof(); ++d)
      if (s->table.constrained[d]) residual[d] = u[d] - s->table.prescribed[d];
  });
}

int32_t orc_mf_apply_mt(void* sys, const double* u, const double* x, double* y, int32_t nthreads) {
  return guarded([&] {
    auto* s = S(sys);
    // The operator's own Jacobi diagonal is not needed for apply; build the action directly.
    if (s->dim() == 2) {
      orc::MatrixFreeOperator<2> op; op.s = s; op.state.assign(u, u + s->n_dof()); op.nthreads = nthreads;
      op.apply(x, y);
    } else {
      orc::MatrixFreeOperator<3> op; op.s = s; op.state.assign(u, u + s->n_dof()); op.nthreads = nthreads;
      op.apply(x, y);
    }
  });
}

int32_t orc_mf_apply(void* sys, const double* u, const double* x, double* y) {
  return orc_mf_apply_mt(sys, u, x, y, 1);
}

int32_t orc_mf_diagonal(void* sys, const double* u, double* d) {
  return guarded([&] {
    auto* s = S(sys);
    std::vector<double> v;
    by_dim(s, [&] { v = orc::make_mf<2>(*s, u).diag; }, [&] { v = orc::make_mf<3>(*s, u).diag; });
    std::memcpy(d, v.data(), v.size() * 8);
  });
}

int32_t orc_mf_diagonal_mt(void* sys, const double* u, double* d, int32_t nthreads) {
  return guarded([&] {
    auto* s = S(sys);
    std::vector<double> v;
    by_dim(s, [&] { v = orc::assemble_diagonal_mt<2>(s->batches, u, s->n_dof(), nthreads); },
           [&] { v = orc::assemble_diagonal_mt<3>(s->batches, u, s->n_dof(), nthreads); });
    for (int64_t k = 0; k < s->n_dof(); ++k)
      if (s->table.constrained[k]) v[k] = 1.0;
    std::memcpy(d, v.data(), v.size() * 8);
  });
}

int32_t orc_csr_apply(void* sys, const double* values, const double* x, double* y) {
  return guarded([&] {
    auto* s = S(sys);
    orc::ExplicitOperator op;
    op.p = &s->pattern;
    op.values.assign(values, values + s->pattern.nnz());
    op.apply(x, y);
  });
}

int32_t orc_solve(void* sys, int32_t op_kind, const double* values_or_u, const orc_solver_cfg* cfg, const double* b,
                  const double* x0, double* x, orc_solve_report* rep, double* history, int32_t hist_cap) {
  return guarded([&] {
    auto* s = S(sys);
    orc::SolveReport r;
    std::vector<double> out;
    const orc::SolverConfig c = to_cfg(cfg);
    if (op_kind == 0) {
      orc::ExplicitOperator op;
      op.p = &s->pattern;
      op.values.assign(values_or_u, values_or_u + s->pattern.nnz());
      out = orc::run_solver(op, b, c, x0, r);
    } else if (s->dim() == 2) {
      const auto op = orc::make_mf<2>(*s, values_or_u);
      out = orc::run_solver(op, b, c, x0, r);
    } else {
      const auto op = orc::make_mf<3>(*s, values_or_u);
      out = orc::run_solver(op, b, c, x0, r);
    }
    std::memcpy(x, out.data(), out.size() * 8);
    fill_report(r, rep, history, hist_cap);
  });
}

static orc::NewtonConfig to_ncfg(const orc_newton_cfg* c) {
  orc::NewtonConfig n;
  n.rtol = c->rtol; n.atol = c->atol; n.max_iter = c->max_iter; n.operator_kind = c->operator_kind;
  n.linear = to_cfg(&c->linear);
  return n;
}

static void fill_newton(const orc::NewtonReport& r, orc_newton_report* out, double* norms, int32_t cap) {
  out->converged = r.converged;
  out->iterations = r.iterations;
  out->n_norms = (int32_t)r.residual_norms.size();
  out->total_time = r.total_time;
  int tot = 0;
  for (const auto& l : r.linear_reports) tot += l.iterations;
  out->total_linear_iterations = tot;
  std::snprintf(out->failure, sizeof out->failure, "%s", r.failure.c_str());
  if (norms)
    for (int32_t i = 0; i < cap && i < (int32_t)r.residual_norms.size(); ++i) norms[i] = r.residual_norms[i];
}

int32_t orc_solve_bvp(void* sys, const orc_newton_cfg* cfg, const double* x0, double* u, orc_newton_report* rep,
                      double* norms, int32_t norms_cap) {
  return guarded([&] {
    auto* s = S(sys);
    orc::NewtonReport r;
    std::vector<double> out;
    const auto c = to_ncfg(cfg);
    if (s->dim() == 2) out = orc::solve_bvp<2>(*s, c, x0, r);
    else out = orc::solve_bvp<3>(*s, c, x0, r);
    std::memcpy(u, out.data(), out.size() * 8);
    fill_newton(r, rep, norms, norms_cap);
  });
}

// load_stepping (newton.hpp:163-186): regenerates benchmark_bcs per step from the grid metadata.
int32_t orc_load_stepping(void* sys, double total_strain, int32_t n_steps, const orc_newton_cfg* cfg, double* u,
                          int32_t* failed_step, int32_t* converged, int32_t* step_iterations) {
  return guarded([&] {
    if (n_steps < 1) throw std::invalid_argument("load_stepping: n_steps must be >= 1");
    auto* s = S(sys);
    const auto c = to_ncfg(cfg);
    std::vector<double> cur;
    *failed_step = -1;
    *converged = 0;
    for (int st = 1; st <= n_steps; ++st) {
      const double strain = total_strain * st / n_steps;
      const auto bcs = orc::benchmark_bcs(s->dim(), s->mesh.nx, s->mesh.ny, s->mesh.nz, s->mesh.lx, strain);
      orc::validate_dirichlet(bcs, s->mesh.n_nodes(), s->dim());
      s->table = orc::constraint_table(bcs, s->n_dof(), s->dim());
      s->constraints = bcs;
      orc::NewtonReport r;
      const double* x0 = cur.empty() ? nullptr : cur.data();
      cur = s->dim() == 2 ? orc::solve_bvp<2>(*s, c, x0, r) : orc::solve_bvp<3>(*s, c, x0, r);
      if (step_iterations) step_iterations[st - 1] = r.iterations;
      if (!r.converged) {
        *failed_step = st;
        std::memcpy(u, cur.data(), cur.size() * 8);
        return;
      }
      // J2: the converged step becomes the committed history (not in the reference, which has no state)
      if (s->dim() == 2) orc::commit_history<2>(*s, cur.data()); else orc::commit_history<3>(*s, cur.data());
    }
    *converged = 1;
    std::memcpy(u, cur.data(), cur.size() * 8);
  });
}

int64_t orc_history_size(void* sys) { return (int64_t)S(sys)->history.size(); }

int32_t orc_history_commit(void* sys, const double* u) {
  return guarded([&] {
    auto* s = S(sys);
    if (s->dim() == 2) orc::commit_history<2>(*s, u); else orc::commit_history<3>(*s, u);
  });
}

int32_t orc_history_copy(void* sys, double* out) {
  return guarded([&] {
    const auto& h = S(sys)->history;
    std::memcpy(out, h.data(), h.size() * 8);
  });
}

int32_t orc_history_set(void* sys, const double* in) {
  return guarded([&] {
    auto& h = S(sys)->history;
    std::memcpy(h.data(), in, h.size() * 8);
  });
}

}  // extern "C"
