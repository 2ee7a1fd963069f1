// adfem/newton.hpp — B200 drop-in for the reference's nonlinear drivers (proj/include/adfem/
// newton.hpp). Same namespace, types and signatures:
//
//   solve_bvp      (newton.hpp:59-152)  the whole Newton loop resident on the device
//                  (afem_solve_bvp_ex: residual, tangent or matrix-free operator, elimination,
//                  the linear solve and the update never leave HBM); the report, the per-iteration
//                  linear reports and the optional log lines are the reference's
//   load_stepping  (newton.hpp:154-186) the reference's ramp over solve_bvp
#ifndef ADFEM_NEWTON_HPP
#define ADFEM_NEWTON_HPP

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "adfem/assembly.hpp"
#include "adfem/b200_device.hpp"
#include "adfem/backend.hpp"
#include "adfem/mesh.hpp"

namespace adfem {

struct NewtonConfig {
  double rtol = 1e-10;
  double atol = 1e-14;
  int max_iter = 25;
  SolverConfig linear{};
  OperatorKind operator_kind = OperatorKind::EXPLICIT;
  std::ostream* log = nullptr;

  void validate() const {
    if (!(rtol > 0.0) || !(atol > 0.0)) throw std::invalid_argument("newton config: tolerances must be > 0");
    if (max_iter < 1) throw std::invalid_argument("newton config: max_iter must be >= 1");
    linear.validate();
  }
};

struct NewtonReport {
  bool converged = false;
  int iterations = 0;
  std::vector<double> residual_norms;
  std::vector<SolveReport> linear_reports;
  double total_time = 0.0;
  std::string failure;
};

namespace detail {

/// ||R|| over the free dofs (newton.hpp:45-50).
inline double free_norm(std::span<const double> r, const ConstraintTable& t) {
  double s = 0.0;
  for (std::size_t i = 0; i < r.size(); ++i)
    if (!t.constrained[i]) s += r[i] * r[i];
  return std::sqrt(s);
}

}  // namespace detail

namespace b200_dropin {

// Device system of a mesh (elements in mesh order, phase = material label: the device's
// (phase, element) scatter order is build_batches' (batch, element) order).
inline std::unique_ptr<SystemHandle> mesh_system(const Mesh& mesh, std::span<const Material> materials) {
  int top = -1;
  for (int p : mesh.material_of) top = std::max(top, p);
  if (top >= static_cast<int>(materials.size()))
    throw std::invalid_argument("build_batches: no material supplied for a mesh phase");
  for (const Material& m : materials) m.validate();
  std::vector<double> xy;
  xy.reserve(2 * mesh.nodes.size());
  for (const auto& n : mesh.nodes) {
    xy.push_back(n[0]);
    xy.push_back(n[1]);
  }
  std::vector<std::int32_t> conn;
  conn.reserve(4 * mesh.elements.size());
  for (const auto& e : mesh.elements) conn.insert(conn.end(), e.begin(), e.end());
  std::vector<std::int32_t> phase(mesh.material_of.begin(), mesh.material_of.end());
  std::vector<afem_material> mats;
  for (const Material& m : materials) mats.push_back(to_afem(m));
  afem_system h = nullptr;
  check(afem_system_create(context(), 2, mesh.n_nodes(), mesh.n_elements(), xy.data(), conn.data(), phase.data(),
                           static_cast<std::int32_t>(mats.size()), mats.data(), &h));
  return std::make_unique<SystemHandle>(h);
}

}  // namespace b200_dropin

/// Newton's method on R(u) = 0 (newton.hpp:59-152), resident on the device.
inline std::pair<std::vector<double>, NewtonReport> solve_bvp(const Mesh& mesh, std::span<const Material> materials,
                                                              const DirichletSpec& bcs, const NewtonConfig& cfg,
                                                              std::span<const double> initial_guess = {}) {
  cfg.validate();
  validate_dirichlet(bcs, mesh);
  const auto t0 = std::chrono::steady_clock::now();
  const std::size_t n = static_cast<std::size_t>(mesh.n_dof());
  if (!initial_guess.empty() && initial_guess.size() != n)
    throw std::invalid_argument("solve_bvp: initial guess dimension mismatch");
  auto sys = b200_dropin::mesh_system(mesh, materials);
  {
    std::vector<std::int32_t> node, comp;
    std::vector<double> val;
    for (const DirichletConstraint& c : bcs.constraints) {
      node.push_back(c.node);
      comp.push_back(c.component);
      val.push_back(c.value);
    }
    b200_dropin::check(afem_set_dirichlet(sys->h, static_cast<std::int64_t>(node.size()), node.data(), comp.data(),
                                          val.data()));
  }
  afem_newton_cfg c{};
  c.rtol = cfg.rtol;
  c.atol = cfg.atol;
  c.max_iter = cfg.max_iter;
  c.operator_kind = cfg.operator_kind == OperatorKind::EXPLICIT ? 0 : 1;
  c.linear = b200_dropin::to_afem(cfg.linear);
  std::vector<double> u(n, 0.0);
  std::vector<double> norms(static_cast<std::size_t>(cfg.max_iter) + 2);
  std::vector<afem_solve_report> lin(static_cast<std::size_t>(cfg.max_iter) + 1);
  for (auto& l : lin) l.iterations = -1;  // marks the slots the library did not fill
  afem_newton_report rep{};
  b200_dropin::check(afem_solve_bvp_ex(sys->h, &c, initial_guess.empty() ? nullptr : initial_guess.data(), u.data(),
                                       &rep, norms.data(), static_cast<std::int32_t>(norms.size()), lin.data(),
                                       static_cast<std::int32_t>(lin.size())));
  NewtonReport out;
  out.converged = rep.converged != 0;
  out.iterations = rep.iterations;
  out.residual_norms.assign(norms.begin(), norms.begin() + std::min<std::size_t>(norms.size(), rep.n_norms));
  for (const afem_solve_report& l : lin)
    if (l.iterations >= 0) out.linear_reports.push_back(b200_dropin::from_afem(l, {}));
  out.failure = rep.failure;
  if (cfg.log) {
    const double r0 = out.residual_norms.empty() ? 0.0 : out.residual_norms.front();
    for (int k = 1; k <= out.iterations && static_cast<std::size_t>(k) < out.residual_norms.size(); ++k) {
      char line[160];
      const SolveReport& l = out.linear_reports[static_cast<std::size_t>(k - 1)];
      std::snprintf(line, sizeof line, "newton iter=%d rnorm=%.6e rel=%.6e lin_iters=%d lin_time=%.3e\n", k,
                    out.residual_norms[static_cast<std::size_t>(k)],
                    r0 > 0.0 ? out.residual_norms[static_cast<std::size_t>(k)] / r0 : 0.0, l.iterations, l.wall_time);
      *cfg.log << line;
    }
  }
  out.total_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return {std::move(u), std::move(out)};
}

struct LoadSteppingReport {
  std::vector<NewtonReport> steps;
  bool converged = false;
  int failed_step = -1;
  double total_time = 0.0;
};

/// Strain ramp over solve_bvp, warm-started per step (newton.hpp:163-186).
inline std::pair<std::vector<double>, LoadSteppingReport> load_stepping(const Mesh& mesh,
                                                                        std::span<const Material> materials,
                                                                        double total_strain, const NewtonConfig& cfg,
                                                                        int n_steps) {
  if (n_steps < 1) throw std::invalid_argument("load_stepping: n_steps must be >= 1");
  const auto t0 = std::chrono::steady_clock::now();
  LoadSteppingReport rep;
  std::vector<double> u;
  for (int s = 1; s <= n_steps; ++s) {
    const DirichletSpec bcs = benchmark_bcs(mesh, total_strain * s / n_steps);
    auto [u_s, nrep] = solve_bvp(mesh, materials, bcs, cfg, u);
    const bool ok = nrep.converged;
    rep.steps.push_back(std::move(nrep));
    u = std::move(u_s);
    if (!ok) {
      rep.failed_step = s;
      rep.total_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      return {std::move(u), std::move(rep)};
    }
  }
  rep.converged = true;
  rep.total_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return {std::move(u), std::move(rep)};
}

}  // namespace adfem

#endif  // ADFEM_NEWTON_HPP
