// TEST INFRASTRUCTURE — the reference's benchmark harness (proj/include/adfem/bench.hpp, compiled in
// place) driven from a small argument parser instead of bench_main.cpp (which needs CLI11, absent
// from this image). Built against the drop-in header tree, every cmd_* runs on the B200 backend;
// acceptance C10 (proj/tests/acceptance.cpp:305-371) executes this binary. Same subcommands,
// options and exit codes as proj/tools/bench_main.cpp: 0 success, 1 failure, 2 configuration error.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>

#include "adfem/bench.hpp"

namespace {

struct Args {
  std::string cmd, config, out = "results.csv";
  long long seed = -1;
  int reps = -1;
  bool parallel = false;
};

void write_records(const std::string& path, const std::vector<adfem::bench::BenchRecord>& recs,
                   const adfem::bench::BenchConfig& cfg, const std::string& experiment) {
  std::ofstream f(path);
  if (!f) throw std::runtime_error("cannot open output file '" + path + "'");
  adfem::bench::write_csv(f, recs, cfg, experiment);
  std::printf("%s: %zu records -> %s\n", experiment.c_str(), recs.size(), path.c_str());
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s verify|spmv|solvers|direct|newton [--config F] [--out F] [--seed N] [--reps N]\n",
                 argv[0]);
    return 2;
  }
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw std::invalid_argument(k + " needs a value");
      return argv[++i];
    };
    try {
      if (k == "--config") a.config = val();
      else if (k == "--out") a.out = val();
      else if (k == "--seed") a.seed = std::stoll(val());
      else if (k == "--reps") a.reps = std::stoi(val());
      else if (k == "--parallel") a.parallel = true;
      else throw std::invalid_argument("unknown option " + k);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "argument error: %s\n", e.what());
      return 2;
    }
  }
  try {
    if (a.cmd == "verify") {
      adfem::VerifyOptions opts;
      if (a.seed >= 0) opts.seed = static_cast<std::uint64_t>(a.seed);
      opts.parallel = a.parallel;
      return adfem::bench::cmd_verify(std::cout, opts);
    }
    adfem::bench::BenchConfig cfg;
    if (!a.config.empty()) cfg = adfem::bench::load_config(a.config);
    if (a.seed >= 0) cfg.seed = static_cast<std::uint64_t>(a.seed);
    if (a.reps >= 1) cfg.reps = a.reps;
    cfg.validate();
    if (a.cmd == "spmv") write_records(a.out, adfem::bench::cmd_spmv(cfg), cfg, "spmv");
    else if (a.cmd == "solvers") write_records(a.out, adfem::bench::cmd_solvers(cfg), cfg, "solvers");
    else if (a.cmd == "direct") write_records(a.out, adfem::bench::cmd_direct(cfg), cfg, "direct");
    else if (a.cmd == "newton") {
      const auto run = adfem::bench::cmd_newton(cfg);
      write_records(a.out, run.records, cfg, "newton");
      std::ofstream(a.out + ".log") << run.log_text;
    } else {
      std::fprintf(stderr, "unknown subcommand %s\n", a.cmd.c_str());
      return 2;
    }
  } catch (const adfem::bench::ConfigError& e) {
    std::cerr << "configuration error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
