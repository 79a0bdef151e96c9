// rdd_run — C++ host driver of the device pipeline through rannddm_gpu.hpp (no Python).
//
//   rdd_run <C1|C2|C3|C4|C5|C5s> [--seed S] [--reps K] [--solver cg|cgs|bicg|gmres|qr]
//           [--precond AS|SAS|RAS|none] [--restart M] [--resident]
//
// Runs run_single (runner.hpp:202-275) K times on one B200 and prints one row per run in the
// column order of the reference's summary.csv (runner.hpp:296-330 `run`), plus the device PCA and
// evaluation times. --resident reruns on the inputs already in HBM after the first run.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include "rannddm_gpu.hpp"

namespace {

const char* problem_name(int id) {
  switch (id) {
    case RDD_PROBLEM_EXAMPLE1: return "example1";
    case RDD_PROBLEM_EXAMPLE2: return "example2";
    case RDD_PROBLEM_EXAMPLE3: return "example3";
    case RDD_PROBLEM_POISSON: return "poisson";
    case RDD_PROBLEM_MULTISCALE: return "multiscale";
    case RDD_PROBLEM_HEAT: return "heat";
    case RDD_PROBLEM_ADVECTION: return "advection";
    default: return "?";
  }
}
const char* solver_name(int s) {
  static const char* names[] = {"qr", "cg", "cgs", "bicg", "gmres"};
  return s >= 0 && s <= 4 ? names[s] : "?";
}
const char* precond_name(int k) {
  static const char* names[] = {"AS", "SAS", "RAS"};
  return k >= 0 && k <= 2 ? names[k] : "none";
}
int parse_solver(const std::string& s) {
  const char* names[] = {"qr", "cg", "cgs", "bicg", "gmres"};
  for (int i = 0; i < 5; ++i)
    if (s == names[i]) return i;
  throw std::invalid_argument("unknown solver '" + s + "'");
}
int parse_precond(const std::string& s) {
  if (s == "AS") return RDD_PRECOND_AS;
  if (s == "SAS") return RDD_PRECOND_SAS;
  if (s == "RAS") return RDD_PRECOND_RAS;
  if (s == "none") return RDD_PRECOND_NONE;
  throw std::invalid_argument("unknown preconditioner '" + s + "'");
}

}  // namespace

int main(int argc, char** argv) {
  namespace G = rannddm::gpu;
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s <C1|C2|C3|C4|C5|C5s> [--seed S] [--reps K] [--solver NAME] [--precond NAME] "
                         "[--restart M] [--resident]\n", argv[0]);
    return 2;
  }
  try {
    rdd_config cfg = G::baseline_config(argv[1]);
    int reps = 1;
    bool resident = false;
    for (int i = 2; i < argc; ++i) {
      const std::string a = argv[i];
      auto next = [&]() -> std::string {
        if (i + 1 >= argc) throw std::invalid_argument("missing value after " + a);
        return argv[++i];
      };
      if (a == "--seed") cfg.seed = std::strtoull(next().c_str(), nullptr, 10);
      else if (a == "--reps") reps = std::atoi(next().c_str());
      else if (a == "--solver") cfg.solver = parse_solver(next());
      else if (a == "--precond") cfg.precond = parse_precond(next());
      else if (a == "--restart") cfg.gmres_restart = std::atoi(next().c_str());
      else if (a == "--resident") resident = true;
      else throw std::invalid_argument("unknown option " + a);
    }
    G::Pipeline dev(0);
    std::printf("seed,problem,J,DoF,N,solver,precond,tau,iter,converged,e_l2,e_l1n,t_assemble,t_precond,t_solve,"
                "t_pca,t_evaluate\n");
    for (int r = 0; r < reps; ++r) {
      const rdd_summary s = (resident && r > 0) ? dev.rerun_resident() : dev.run_single(cfg, cfg.seed);
      std::printf("%llu,%s,%d,%d,%d,%s,%s,%g,%d,%d,%.10g,%.10g,%.9g,%.9g,%.9g,%.9g,%.9g\n",
                  static_cast<unsigned long long>(s.seed), problem_name(cfg.problem), s.J, s.DoF, s.N,
                  solver_name(cfg.solver), precond_name(cfg.precond), cfg.tau, s.iterations, s.converged, s.e_l2,
                  s.e_l1n, s.t_assemble, s.t_precond, s.t_solve, s.t_pca, s.t_evaluate);
    }
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "invalid_argument: %s\n", e.what());
    return 1;
  } catch (const std::domain_error& e) {
    std::fprintf(stderr, "domain_error: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "runtime_error: %s\n", e.what());
    return 1;
  }
  return 0;
}
