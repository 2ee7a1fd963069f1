// afem_bench — GPU-backed counterpart of the reference's `bench` CLI (tools/bench_main.cpp:56-115,
// bench.hpp:189-406), written against the C ABI only (include/afem.h; no reference code).
//
//   afem_bench spmv     [opts]   100 CSR applies of the eliminated benchmark tangent per rep (cmd_spmv)
//   afem_bench mfapply  [opts]   100 matrix-free applies per rep (the bench.py metric, any mesh)
//   afem_bench solvers  [opts]   method x preconditioner grid on the benchmark system (cmd_solvers)
//   afem_bench direct   [opts]   banded Cholesky and LU on the benchmark system (cmd_direct)
//   afem_bench newton   [opts]   solve_bvp under EXPLICIT and MATRIX_FREE (cmd_newton)
//   afem_bench verify   [opts]   the five oracle checks of verify.hpp:62-308 through the ABI
//
// Options: --dim 2|3 (2: the reference's quad4 series; 3: hex8 fibre RVE), --n N (base cells per
// axis; 2D default 16), --levels L (refinement series n, 2n, 4n...; default 3 in 2D, 1 in 3D),
// --reps R (3), --seed S (12345), --strain e (0.01), --rtol r (1e-13), --max-iter m (5000),
// --restart k (30), --materials linear|svk|neohooke|j2 (matrix law; inclusion linear E=10),
// --fibres K --radius r (3D), --out FILE (CSV; default stdout).
// CSV: the reference schema (bench.hpp:201-218): a '#' metadata line, then
// experiment,dof,method,pc,operator,converged,iters,time_s,final_rres. Timing: steady_clock around
// device-synchronised calls, min over reps is left to the reader (one row per rep, as the reference).
// Exit codes (bench_main.cpp:76-114): 0 ok, 1 a check / run failed, 2 usage or configuration error.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "afem.h"

namespace {

struct Opts {
  std::string cmd;
  int dim = 2, n = 0, levels = 0, reps = 3, max_iter = 5000, restart = 30, fibres = 40;
  uint64_t seed = 12345;
  double strain = 0.01, rtol = 1e-13, radius = 0.05;
  std::string materials = "svk", out;
};

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(afem_status s) {
  if (s != AFEM_OK) throw std::runtime_error(std::string("afem: ") + afem_last_error());
}

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

Opts parse(int argc, char** argv) {
  if (argc < 2) throw UsageError("missing subcommand (spmv | mfapply | solvers | direct | newton | verify)");
  Opts o;
  o.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw UsageError("missing value for " + k);
      return argv[++i];
    };
    if (k == "--dim") o.dim = std::stoi(val());
    else if (k == "--n") o.n = std::stoi(val());
    else if (k == "--levels") o.levels = std::stoi(val());
    else if (k == "--reps") o.reps = std::stoi(val());
    else if (k == "--seed") o.seed = std::stoull(val());
    else if (k == "--strain") o.strain = std::stod(val());
    else if (k == "--rtol") o.rtol = std::stod(val());
    else if (k == "--max-iter") o.max_iter = std::stoi(val());
    else if (k == "--restart") o.restart = std::stoi(val());
    else if (k == "--materials") o.materials = val();
    else if (k == "--fibres") o.fibres = std::stoi(val());
    else if (k == "--radius") o.radius = std::stod(val());
    else if (k == "--out") o.out = val();
    else throw UsageError("unknown option " + k);
  }
  if (o.dim != 2 && o.dim != 3) throw UsageError("--dim must be 2 or 3");
  if (o.n == 0) o.n = o.dim == 2 ? 16 : 32;
  if (o.levels == 0) o.levels = o.dim == 2 ? 3 : 1;
  if (o.reps < 1 || o.levels < 1 || o.n < 1) throw UsageError("reps, levels and n must be >= 1");
  return o;
}

std::vector<afem_material> materials(const std::string& m) {
  afem_material mat{0, 1.0, 0.3, 0.0, 0.0}, inc{0, 10.0, 0.3, 0.0, 0.0};
  if (m == "linear") mat.model = 0;
  else if (m == "svk") mat.model = 1;
  else if (m == "neohooke") mat.model = 2;
  else if (m == "j2") {
    mat.model = 3;
    mat.sigma_y = 0.002;
    mat.hardening = 0.1;
  } else {
    throw UsageError("--materials must be linear | svk | neohooke | j2");
  }
  return {mat, inc};
}

// A refinement level of the configured mesh family, generated on the device.
struct Sys {
  afem_system h = nullptr;
  afem_system_info info{};
  ~Sys() {
    if (h) afem_system_destroy(h);
  }
};

void make_sys(afem_ctx ctx, const Opts& o, int n, const std::vector<afem_material>& mats, Sys& s) {
  if (o.dim == 2) {
    const double c[2] = {0.5, 0.5};  // generate_two_phase_mesh(n, n, 1, 1, {.5,.5}, .25) (bench defaults)
    ck(afem_system_create_grid(ctx, 2, n, n, 0, 1.0, 1.0, 0.0, 1, c, 0.25, (int)mats.size(), mats.data(), &s.h));
  } else {
    std::vector<double> fib(2 * o.fibres);
    ck(afem_fibres(o.seed, o.fibres, 1.0, 1.0, fib.data()));
    ck(afem_system_create_grid(ctx, 3, n, n, n, 1.0, 1.0, 1.0, o.fibres, fib.data(), o.radius, (int)mats.size(),
                               mats.data(), &s.h));
  }
  ck(afem_system_get_info(s.h, &s.info));
}

struct Record {
  std::string experiment, method, pc, op;
  long long dof;
  bool converged;
  long iters;
  double time_s, rres;
};

void write_csv(std::ostream& os, const std::vector<Record>& rs, const Opts& o) {
  char line[320];
  std::snprintf(line, sizeof line,
                "# afem_bench (libafem_b200, B200): experiment=%s dim=%d seed=%llu reps=%d timing=steady_clock "
                "summary=min_over_reps\n",
                o.cmd.c_str(), o.dim, static_cast<unsigned long long>(o.seed), o.reps);
  os << line << "experiment,dof,method,pc,operator,converged,iters,time_s,final_rres\n";
  for (const Record& r : rs) {
    std::snprintf(line, sizeof line, "%s,%lld,%s,%s,%s,%d,%ld,%.6e,%.17g\n", r.experiment.c_str(), r.dof,
                  r.method.c_str(), r.pc.c_str(), r.op.c_str(), r.converged ? 1 : 0, r.iters, r.time_s, r.rres);
    os << line;
  }
}

// assemble_benchmark_system (bench.hpp:233-251): u0 BC-consistent, K(u0) eliminated, rhs = -R(u0);
// the values stay on the device and are handed to the buffer (lease held by the caller).
struct Bench {
  std::vector<double> u0, rhs;
  afem_buffer buf = nullptr;
  afem_op op = nullptr;
  ~Bench() {
    if (op) afem_op_destroy(op);
    if (buf) {
      afem_buffer_release(buf);
      afem_buffer_destroy(buf);
    }
  }
};

void bench_system(const Opts& o, Sys& s, Bench& b) {
  ck(afem_set_benchmark_dirichlet(s.h, o.strain));
  b.u0.assign(s.info.n_dof, 0.0);
  ck(afem_impose_dirichlet(s.h, b.u0.data()));
  b.rhs.assign(s.info.n_dof, 0.0);
  afem_values v = nullptr;
  ck(afem_values_create(s.h, &v));
  ck(afem_residual(s.h, b.u0.data(), b.rhs.data()));
  ck(afem_values_assemble(v, b.u0.data()));
  ck(afem_values_eliminate(v, b.rhs.data(), b.u0.data()));
  for (double& x : b.rhs) x = -x;
  ck(afem_buffer_create(s.h, &b.buf));
  ck(afem_buffer_handoff(b.buf, &v));
  ck(afem_op_create_explicit(b.buf, &b.op));
}

std::vector<double> rand_vec(size_t n, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> d(-1.0, 1.0);
  std::vector<double> v(n);
  for (double& x : v) x = d(rng);
  return v;
}

int level_n(const Opts& o, int k) { return o.n << k; }

std::vector<Record> cmd_apply(afem_ctx ctx, const Opts& o, bool mf) {
  std::vector<Record> rs;
  const auto mats = materials(o.materials);
  for (int k = 0; k < o.levels; ++k) {
    Sys s;
    make_sys(ctx, o, level_n(o, k), mats, s);
    Bench b;
    bench_system(o, s, b);
    afem_op op = b.op;
    afem_op mfop = nullptr;
    if (mf) {
      ck(afem_op_create_mf(s.h, b.u0.data(), &mfop));
      op = mfop;
    }
    const auto x = rand_vec(s.info.n_dof, o.seed);
    std::vector<double> y(x.size());
    for (int r = 0; r < o.reps; ++r) {
      const double t0 = now();
      for (int it = 0; it < 100; ++it) ck(afem_op_apply(op, x.data(), y.data()));
      rs.push_back({mf ? "mfapply" : "spmv", mf ? "MFAPPLY" : "SPMV", "NONE", mf ? "MATRIX_FREE" : "EXPLICIT",
                    s.info.n_dof, true, 100, now() - t0, 0.0});
    }
    if (mfop) afem_op_destroy(mfop);
  }
  return rs;
}

const char* mname(int m) {
  static const char* names[] = {"CG", "GMRES", "BICGSTAB", "DIRECT_CHOL", "DIRECT_LU"};
  return names[m];
}
const char* pname(int p) { return p == 0 ? "NONE" : (p == 1 ? "JACOBI" : "ILU0"); }

std::vector<Record> cmd_solvers(afem_ctx ctx, const Opts& o) {
  std::vector<Record> rs;
  const auto mats = materials(o.materials);
  for (int k = 0; k < o.levels; ++k) {
    Sys s;
    make_sys(ctx, o, level_n(o, k), mats, s);
    Bench b;
    bench_system(o, s, b);
    std::vector<double> x(s.info.n_dof), hist(o.max_iter + 2);
    for (int m : {0, 1, 2})
      for (int p : {0, 1, 2})
        for (int r = 0; r < o.reps; ++r) {
          afem_solver_cfg cfg{m, p, o.rtol, o.max_iter, o.restart};
          afem_solve_report rep{};
          ck(afem_solve(b.op, &cfg, b.rhs.data(), nullptr, x.data(), &rep, hist.data(), (int32_t)hist.size()));
          const int nh = std::min<int>(rep.n_history, (int)hist.size());
          rs.push_back({"solvers", mname(m), pname(p), "EXPLICIT", s.info.n_dof, rep.converged != 0, rep.iterations,
                        rep.wall_time, nh > 0 ? hist[nh - 1] : NAN});
        }
  }
  return rs;
}

// cmd_direct (bench.hpp:321-342): failures recorded with final_rres = NaN, never dropped.
std::vector<Record> cmd_direct(afem_ctx ctx, const Opts& o) {
  std::vector<Record> rs;
  const auto mats = materials(o.materials);
  for (int k = 0; k < o.levels; ++k) {
    Sys s;
    make_sys(ctx, o, level_n(o, k), mats, s);
    Bench b;
    bench_system(o, s, b);
    std::vector<double> x(s.info.n_dof), hist(4);
    for (int m : {3, 4})
      for (int r = 0; r < o.reps; ++r) {
        afem_solver_cfg cfg{m, 0, o.rtol, 1, o.restart};
        afem_solve_report rep{};
        ck(afem_solve(b.op, &cfg, b.rhs.data(), nullptr, x.data(), &rep, hist.data(), (int32_t)hist.size()));
        const int nh = std::min<int>(rep.n_history, (int)hist.size());
        rs.push_back({"direct", mname(m), "NONE", "EXPLICIT", s.info.n_dof, rep.converged != 0, rep.iterations,
                      rep.wall_time, rep.failure[0] ? NAN : hist[nh - 1]});
      }
  }
  return rs;
}

std::vector<Record> cmd_newton(afem_ctx ctx, const Opts& o, std::ostream& log) {
  std::vector<Record> rs;
  const auto mats = materials(o.materials);
  for (int k = 0; k < o.levels; ++k)
    for (int kind : {0, 1}) {
      Sys s;
      make_sys(ctx, o, level_n(o, k), mats, s);
      ck(afem_set_benchmark_dirichlet(s.h, o.strain));
      afem_newton_cfg cfg{1e-10, 1e-14, 25, kind, {0, 1, o.rtol, 20000, o.restart}};
      std::vector<double> u(s.info.n_dof), norms(27);
      afem_newton_report rep{};
      log << "# newton dof=" << s.info.n_dof << " operator=" << (kind ? "MATRIX_FREE" : "EXPLICIT") << "\n";
      ck(afem_solve_bvp(s.h, &cfg, nullptr, u.data(), &rep, norms.data(), (int32_t)norms.size()));
      const int nn = std::min<int>(rep.n_norms, (int)norms.size());
      for (int i = 1; i < nn; ++i)
        log << "newton iter=" << i << " rnorm=" << norms[i] << " rel=" << norms[i] / norms[0] << "\n";
      log << "# done converged=" << rep.converged << " newton_iters=" << rep.iterations
          << " linear_iters_total=" << rep.total_linear_iterations << "\n";
      rs.push_back({"newton", "CG", "JACOBI", kind ? "MATRIX_FREE" : "EXPLICIT", s.info.n_dof, rep.converged != 0,
                    rep.iterations, rep.total_time, nn > 0 && norms[0] > 0 ? norms[nn - 1] / norms[0] : 0.0});
    }
  return rs;
}

// ---------------------------------------------------------------- verify (verify.hpp:62-308)
struct Check {
  std::string name;
  bool pass;
  std::string detail;
};

double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num = std::max(num, std::abs(a[i] - b[i]));
    den = std::max(den, std::abs(b[i]));
  }
  return num / (den > 0 ? den : 1.0);
}

std::string fmt(const char* f, double v) {
  char b[96];
  std::snprintf(b, sizeof b, f, v);
  return b;
}

// Dense K from the CSR values (small meshes only).
std::vector<double> dense(afem_system s, int64_t n, const std::vector<double>& vals) {
  int64_t nnz = 0;
  ck(afem_pattern_nnz(s, &nnz));
  std::vector<int64_t> rp(n + 1);
  std::vector<int32_t> rows(nnz), cols(nnz);
  ck(afem_pattern(s, rp.data(), rows.data(), cols.data()));
  std::vector<double> K(n * n, 0.0);
  for (int64_t k = 0; k < nnz; ++k) K[rows[k] * n + cols[k]] = vals[k];
  return K;
}

std::vector<Check> cmd_verify(afem_ctx ctx, const Opts& o) {
  std::vector<Check> out;
  const int dim = o.dim;
  const auto mats = materials(o.materials);
  Opts oo = o;
  // (1) analytic tangent vs central finite differences of the residual (check_fd_vs_ad, :62-97)
  {
    Sys s;
    make_sys(ctx, oo, dim == 2 ? 4 : 3, mats, s);
    const int64_t n = s.info.n_dof;
    std::vector<double> u = rand_vec(n, o.seed);
    for (double& x : u) x *= 0.01;
    std::vector<double> vals(s.info.nnz);
    ck(afem_jacobian(s.h, u.data(), vals.data()));
    const auto K = dense(s.h, n, vals);
    const double h = 1e-6;
    double err = 0, kmax = 0;
    std::vector<double> up(u), um(u), rp(n), rm(n);
    for (int64_t j = 0; j < n; j += std::max<int64_t>(1, n / 12)) {
      up = u;
      um = u;
      up[j] += h;
      um[j] -= h;
      ck(afem_residual(s.h, up.data(), rp.data()));
      ck(afem_residual(s.h, um.data(), rm.data()));
      for (int64_t i = 0; i < n; ++i) {
        err = std::max(err, std::abs((rp[i] - rm[i]) / (2 * h) - K[i * n + j]));
        kmax = std::max(kmax, std::abs(K[i * n + j]));
      }
    }
    out.push_back({"fd_vs_tangent", err <= 1e-5 * std::max(kmax, 1.0), fmt("max |FD - K| = %.2e", err)});
  }
  // (2) dense equivalence: K u == R(u) - R(0) for the linear law; K symmetric (check_dense_equivalence)
  {
    Sys s;
    auto lin = materials("linear");
    make_sys(ctx, oo, dim == 2 ? 6 : 3, lin, s);
    const int64_t n = s.info.n_dof;
    const auto u = rand_vec(n, o.seed + 1);
    std::vector<double> vals(s.info.nnz), r(n), ku(n);
    ck(afem_jacobian(s.h, u.data(), vals.data()));
    ck(afem_residual(s.h, u.data(), r.data()));
    ck(afem_csr_apply(s.h, vals.data(), u.data(), ku.data()));
    const auto K = dense(s.h, n, vals);
    double asym = 0, km = 0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) {
        asym = std::max(asym, std::abs(K[i * n + j] - K[j * n + i]));
        km = std::max(km, std::abs(K[i * n + j]));
      }
    const double e = rel(ku, r);
    out.push_back({"dense_equivalence", e <= 1e-12 && asym <= 1e-12 * km,
                   fmt("|Ku - R(u)|/|R| = %.2e", e) + fmt(", asym %.2e", asym / km)});
  }
  // (3) operator equivalence: matrix-free == eliminated explicit on random vectors (check_operator_equivalence)
  {
    Sys s;
    make_sys(ctx, oo, dim == 2 ? 16 : 6, mats, s);
    Bench b;
    bench_system(oo, s, b);
    afem_op mf = nullptr;
    ck(afem_op_create_mf(s.h, b.u0.data(), &mf));
    double worst = 0;
    for (int t = 0; t < 5; ++t) {
      const auto x = rand_vec(s.info.n_dof, o.seed + 10 + t);
      std::vector<double> ya(x.size()), yb(x.size());
      ck(afem_op_apply(b.op, x.data(), ya.data()));
      ck(afem_op_apply(mf, x.data(), yb.data()));
      worst = std::max(worst, rel(yb, ya));
    }
    afem_op_destroy(mf);
    out.push_back({"operator_equivalence", worst <= 1e-12, fmt("max rel diff %.2e over 5 vectors", worst)});
  }
  // (4) patch test: homogeneous linear body under the benchmark BCs reproduces the exact uniaxial
  // state u_x = e x, u_y (, u_z) = -nu' e y (check_patch_test, :182-216); nu' = nu/(1-nu) in plane strain
  {
    Sys s;
    const afem_material one{0, 1.0, 0.3, 0.0, 0.0};
    const int n = dim == 2 ? 5 : 3;
    if (dim == 2) {
      const double c[2] = {0.5, 0.5};
      ck(afem_system_create_grid(ctx, 2, n, n, 0, 1, 1, 0, 1, c, 0.0, 1, &one, &s.h));
    } else {
      ck(afem_system_create_grid(ctx, 3, n, n, n, 1, 1, 1, 0, nullptr, 0.0, 1, &one, &s.h));
    }
    ck(afem_system_get_info(s.h, &s.info));
    ck(afem_set_benchmark_dirichlet(s.h, o.strain));
    afem_newton_cfg cfg{1e-12, 1e-14, 5, 0, {0, 1, 1e-13, 10000, 30}};
    std::vector<double> u(s.info.n_dof), norms(8), xyz(s.info.n_nodes * dim);
    afem_newton_report rep{};
    ck(afem_solve_bvp(s.h, &cfg, nullptr, u.data(), &rep, norms.data(), 8));
    ck(afem_system_mesh(s.h, xyz.data(), nullptr, nullptr));
    const double nu = 0.3, lat = dim == 2 ? nu / (1 - nu) : nu;
    double err = 0;
    for (int64_t i = 0; i < s.info.n_nodes; ++i) {
      err = std::max(err, std::abs(u[dim * i] - o.strain * xyz[dim * i]));
      for (int c = 1; c < dim; ++c) err = std::max(err, std::abs(u[dim * i + c] + lat * o.strain * xyz[dim * i + c]));
    }
    out.push_back({"patch_test", rep.converged && err <= 1e-10, fmt("max nodal error %.2e", err)});
  }
  // (5) MMS: u = a (x^2 - y^2, -2xy[, 0]) is an exact equilibrium field of isotropic linear
  // elasticity; Dirichlet data on the whole boundary; L2 error by 3-point Gauss quadrature of the
  // interpolant on a 3-mesh series, mean log2 slope 2.0 +- 0.1 (check_mms_convergence, :218-291)
  {
    const afem_material one{0, 1.0, 0.3, 0.0, 0.0};
    const double a = 0.01;
    auto field = [&](const double* X, int c) {
      return c == 0 ? a * (X[0] * X[0] - X[1] * X[1]) : (c == 1 ? -2 * a * X[0] * X[1] : 0.0);
    };
    std::vector<double> errs;
    const std::vector<int> series = dim == 2 ? std::vector<int>{8, 16, 32} : std::vector<int>{4, 8, 16};
    for (int n : series) {
      Sys s;
      if (dim == 2) {
        const double c[2] = {0.5, 0.5};
        ck(afem_system_create_grid(ctx, 2, n, n, 0, 1, 1, 0, 1, c, 0.0, 1, &one, &s.h));
      } else {
        ck(afem_system_create_grid(ctx, 3, n, n, n, 1, 1, 1, 0, nullptr, 0.0, 1, &one, &s.h));
      }
      ck(afem_system_get_info(s.h, &s.info));
      const int npe = dim == 2 ? 4 : 8;
      std::vector<double> xyz(s.info.n_nodes * dim);
      std::vector<int32_t> conn(s.info.n_elem * npe);
      ck(afem_system_mesh(s.h, xyz.data(), conn.data(), nullptr));
      std::vector<int32_t> node, comp;
      std::vector<double> val;
      for (int64_t i = 0; i < s.info.n_nodes; ++i) {
        bool bnd = false;
        for (int c = 0; c < dim; ++c) bnd |= xyz[dim * i + c] < 1e-12 || xyz[dim * i + c] > 1 - 1e-12;
        if (!bnd) continue;
        for (int c = 0; c < dim; ++c) {
          node.push_back((int32_t)i);
          comp.push_back(c);
          val.push_back(field(&xyz[dim * i], c));
        }
      }
      ck(afem_set_dirichlet(s.h, (int64_t)node.size(), node.data(), comp.data(), val.data()));
      afem_newton_cfg cfg{1e-12, 1e-15, 5, 0, {0, 1, 1e-13, 20000, 30}};
      std::vector<double> u(s.info.n_dof), norms(8);
      afem_newton_report rep{};
      ck(afem_solve_bvp(s.h, &cfg, nullptr, u.data(), &rep, norms.data(), 8));
      // L2 error of the interpolant, 3-point Gauss per axis (the grid is affine: detJ = h^dim)
      const double g3[3] = {-0.77459666924148337704, 0.0, 0.77459666924148337704};
      const double w3[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
      const int nz3 = dim == 3 ? 3 : 1;
      double err2 = 0.0;
      for (int64_t e = 0; e < s.info.n_elem; ++e) {
        const int32_t* cn = &conn[e * npe];
        for (int qz = 0; qz < nz3; ++qz)
          for (int qy = 0; qy < 3; ++qy)
            for (int qx = 0; qx < 3; ++qx) {
              const double xi = g3[qx], eta = g3[qy], zeta = dim == 3 ? g3[qz] : 0.0;
              const double w = w3[qx] * w3[qy] * (dim == 3 ? w3[qz] : 1.0);
              double X[3] = {0, 0, 0}, uh[3] = {0, 0, 0};
              for (int k = 0; k < npe; ++k) {
                const double sx = ((k & 3) == 1 || (k & 3) == 2) ? 1 : -1, sy = (k & 3) >= 2 ? 1 : -1;
                const double sz = k >= 4 ? 1 : -1;
                double N = 0.25 * (1 + sx * xi) * (1 + sy * eta);
                if (dim == 3) N *= 0.5 * (1 + sz * zeta);
                for (int c = 0; c < dim; ++c) {
                  X[c] += N * xyz[(int64_t)dim * cn[k] + c];
                  uh[c] += N * u[(int64_t)dim * cn[k] + c];
                }
              }
              const double detj = std::pow(1.0 / n, dim) / (dim == 2 ? 4.0 : 8.0);
              for (int c = 0; c < dim; ++c) err2 += w * detj * (uh[c] - field(X, c)) * (uh[c] - field(X, c));
            }
      }
      errs.push_back(std::sqrt(err2));
    }
    double slope = 0.0;
    for (size_t k = 0; k + 1 < errs.size(); ++k) slope += std::log2(errs[k] / errs[k + 1]);
    slope /= static_cast<double>(errs.size() - 1);
    out.push_back({"mms_convergence", std::abs(slope - 2.0) <= 0.1,
                   fmt("L2 errors %.3e", errs[0]) + fmt(" %.3e", errs[1]) + fmt(" %.3e", errs[2]) +
                       fmt(", slope %.3f (target 2.0 +- 0.1)", slope)});
  }
  return out;
}

}  // namespace

int main(int argc, char** argv) {
  Opts o;
  try {
    o = parse(argc, argv);
    if (o.cmd != "spmv" && o.cmd != "mfapply" && o.cmd != "solvers" && o.cmd != "direct" && o.cmd != "newton" &&
        o.cmd != "verify")
      throw UsageError("unknown subcommand " + o.cmd);
    materials(o.materials);
  } catch (const std::exception& e) {
    std::cerr << "afem_bench: " << e.what() << "\n";
    return 2;
  }
  try {
    afem_ctx ctx = nullptr;
    ck(afem_ctx_create(0, &ctx));
    std::ofstream file;
    std::ostream& os = o.out.empty() ? std::cout : (file.open(o.out), file);
    int rc = 0;
    if (o.cmd == "verify") {
      const auto res = cmd_verify(ctx, o);
      os << "check                          status  detail\n";
      for (const auto& r : res) {
        char line[256];
        std::snprintf(line, sizeof line, "%-30s %-7s %s\n", r.name.c_str(), r.pass ? "PASS" : "FAIL", r.detail.c_str());
        os << line;
        rc |= r.pass ? 0 : 1;
      }
    } else {
      std::vector<Record> rs;
      std::ostringstream log;
      if (o.cmd == "spmv") rs = cmd_apply(ctx, o, false);
      else if (o.cmd == "mfapply") rs = cmd_apply(ctx, o, true);
      else if (o.cmd == "solvers") rs = cmd_solvers(ctx, o);
      else if (o.cmd == "direct") rs = cmd_direct(ctx, o);
      else rs = cmd_newton(ctx, o, log);
      write_csv(os, rs, o);
      if (!log.str().empty()) std::cerr << log.str();
    }
    afem_ctx_destroy(ctx);
    return rc;
  } catch (const std::exception& e) {
    std::cerr << "afem_bench: " << e.what() << "\n";
    return 1;
  }
}
