// rannddm_gpu.hpp — C++ host interface over the C ABI (rdd.h), with the reference's phase names.
//
// The reference `rannddm` (proj/include/rannddm/*.hpp) is header-only C++ whose phases are free
// functions over Eigen value types. This header gives a C++ host the same phases on the device
// path, Eigen-free (std::vector, column-major like Eigen), with the reference's exception classes
// rethrown from the ABI status codes. The maintainer-side Eigen adapters
// (LinearMap plug-ins, run_single_gpu) are in INTEGRATION.md; examples/rdd_run.cpp is a C++
// driver built on this header.
#ifndef RANNDDM_GPU_HPP
#define RANNDDM_GPU_HPP

#include <cstdint>
#include <initializer_list>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rdd.h"

namespace rannddm::gpu {

// ABI status -> the reference's exception types (std::invalid_argument / runtime_error / domain_error)
inline void check(const rdd_ctx* c, int st) {
  if (st == RDD_OK) return;
  const std::string msg = c ? rdd_last_error(c) : "rdd: no context";
  if (st == RDD_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (st == RDD_DOMAIN_ERROR) throw std::domain_error(msg);
  throw std::runtime_error(msg);
}

// RunConfig defaults (config.hpp:23-68): example1, GMRES + AS, tol 1e-5, τ off, op_applied.
inline rdd_config default_config() {
  rdd_config c{};
  c.problem = RDD_PROBLEM_EXAMPLE1;
  c.n = 2;
  c.counts[0] = c.counts[1] = 2;
  c.decomposition = RDD_DECOMP_REFERENCE;
  c.delta = 2.0;
  c.m = 32;
  c.seed = 1000;
  c.colloc[0] = c.colloc[1] = 20;
  c.test[0] = c.test[1] = 350;
  c.tau_mode = RDD_TAU_OFF;
  c.pca_matrix = RDD_PCA_OP_APPLIED;
  c.solver = RDD_SOLVER_GMRES;
  c.precond = RDD_PRECOND_AS;
  c.rel_tol = 1e-5;
  c.op_form = RDD_OPERATOR_TWO_PASS;
  c.true_residual = 1;
  return c;
}

// The BASELINE.json configs C1..C5 (same values as paper_2412_19207_b200/configs.py):
// cell-centred boxes extended by 10% per side, PCA σ/σmax > 1e-6 on op_applied, tol 1e-10.
inline rdd_config baseline_config(const std::string& name) {
  rdd_config c = default_config();
  c.decomposition = RDD_DECOMP_CELL;
  c.delta = 0.1;
  c.tau_mode = RDD_TAU_RELATIVE;
  c.tau = 1e-6;
  c.rel_tol = 1e-10;
  c.solver = RDD_SOLVER_CG;
  c.precond = RDD_PRECOND_AS;
  auto grid = [&c](std::initializer_list<int> counts, int per, int test) {
    int a = 0;
    for (int k : counts) {
      c.counts[a] = k;
      c.colloc[a] = k * per;
      c.test[a] = test;
      ++a;
    }
    for (; a < 4; ++a) c.counts[a] = c.colloc[a] = c.test[a] = 0;
  };
  if (name == "C1") {  // 2-D Poisson, 4x4, m=200, 40^2 per subdomain + 4x160 boundary points
    c.problem = RDD_PROBLEM_POISSON;
    c.dim = 2;
    c.m = 200;
    grid({4, 4}, 40, 350);
    c.boundary_per_edge = 160;
  } else if (name == "C2") {  // 2-D multiscale Poisson, 16x16, m=300, 60^2 per subdomain
    c.problem = RDD_PROBLEM_MULTISCALE;
    c.m = 300;
    grid({16, 16}, 60, 350);
  } else if (name == "C3") {  // heat in space-time, 8x8x8, m=300, 16^3; RAS-GMRES(50)
    c.problem = RDD_PROBLEM_HEAT;
    c.m = 300;
    grid({8, 8, 8}, 16, 50);
    c.solver = RDD_SOLVER_GMRES;
    c.precond = RDD_PRECOND_RAS;
    c.gmres_restart = 50;
  } else if (name == "C4") {  // advection in space-time on [0,2]x[0,1], 64x16, m=250, 40^2; RAS-GMRES(50)
    c.problem = RDD_PROBLEM_ADVECTION;
    c.m = 250;
    grid({64, 16}, 40, 350);
    c.solver = RDD_SOLVER_GMRES;
    c.precond = RDD_PRECOND_RAS;
    c.gmres_restart = 50;
  } else if (name == "C5" || name == "C5s") {  // 3-D Poisson, 8^3 (C5s: 2^3), m=400, 20^3 per subdomain
    c.problem = RDD_PROBLEM_POISSON;
    c.dim = 3;
    c.m = 400;
    if (name == "C5") grid({8, 8, 8}, 20, 50);
    else grid({2, 2, 2}, 20, 50);
  } else {
    throw std::invalid_argument("unknown config '" + name + "' (C1..C5, C5s)");
  }
  return c;
}

// krylov.hpp:64-76 SolveReport (iterations, flags, residual histories)
struct SolveReport {
  int iterations = 0;
  bool converged = false;
  bool breakdown = false;
  std::vector<double> residual_history;       // preconditioned relative residual
  std::vector<double> true_residual_history;  // GMRES diagnostic true residual (krylov.hpp:360-367)
};

// One device context = one instance of the pipeline (the reference's Instance + BlockSystem +
// preconditioner + solution), resident in HBM between calls.
class Pipeline {
 public:
  explicit Pipeline(int device = 0) {
    if (rdd_create(&c_, device) != RDD_OK)  // the device path has no CPU fallback
      throw std::runtime_error("rdd_create: no usable CUDA device " + std::to_string(device));
  }
  ~Pipeline() {
    if (c_) rdd_destroy(c_);
  }
  Pipeline(const Pipeline&) = delete;
  Pipeline& operator=(const Pipeline&) = delete;
  Pipeline(Pipeline&& o) noexcept : c_(std::exchange(o.c_, nullptr)) {}
  rdd_ctx* handle() const { return c_; }

  // runner.hpp:40-70
  void build_instance(const rdd_config& cfg, std::uint64_t seed) { check(c_, rdd_build_instance(c_, &cfg, seed)); }
  // runner.hpp:89-101 (assemble + column equilibration)
  void assemble(bool equilibrate = true) { check(c_, rdd_assemble(c_, equilibrate ? 1 : 0)); }
  // assembly.hpp:148 normal_blocks + schwarz.hpp:39 build_index_sets + :93 build_preconditioner
  void build_preconditioner(int kind) { check(c_, rdd_build_preconditioner(c_, kind)); }

  int J() const { return geti("J").at(0); }
  int p() const { return geti("p").at(0); }
  int N() const { return geti("N").at(0); }
  std::vector<int> p_j() const { return geti("p_j"); }
  std::vector<int> rows(int j) const { return geti("rows", j); }  // assembly.hpp:58-64 rows_j

  // assembly.hpp:110 matvec, :123 matvec_transpose; runner.hpp:233 the normal operator
  std::vector<double> matvec(const std::vector<double>& w) const {
    std::vector<double> y(N());
    check(c_, rdd_matvec(c_, w.data(), static_cast<int64_t>(w.size()), y.data(), static_cast<int64_t>(y.size())));
    return y;
  }
  std::vector<double> matvec_transpose(const std::vector<double>& r) const {
    std::vector<double> out(p());
    check(c_, rdd_matvec_transpose(c_, r.data(), static_cast<int64_t>(r.size()), out.data(),
                                   static_cast<int64_t>(out.size())));
    return out;
  }
  std::vector<double> normal_apply(const std::vector<double>& w) const {
    std::vector<double> out(p());
    check(c_, rdd_normal_apply(c_, w.data(), static_cast<int64_t>(w.size()), out.data(),
                               static_cast<int64_t>(out.size())));
    return out;
  }
  // schwarz.hpp:153 apply, :189 apply_transpose
  std::vector<double> apply(const std::vector<double>& v, bool transpose = false) const {
    std::vector<double> z(p());
    check(c_, rdd_precond_apply(c_, v.data(), static_cast<int64_t>(v.size()), z.data(),
                                static_cast<int64_t>(z.size()), transpose ? 1 : 0));
    return z;
  }
  std::vector<double> apply_transpose(const std::vector<double>& v) const { return apply(v, true); }

  // krylov.hpp:391 solve_with over the assembled system (all right-hand-side components)
  SolveReport solve(int solver, double rel_tol, int max_iter = 0, int gmres_restart = 0) {
    check(c_, rdd_solve(c_, solver, rel_tol, max_iter, gmres_restart));
    SolveReport r;
    r.iterations = geti("iterations").at(0);
    r.converged = geti("converged").at(0) != 0;
    r.residual_history = getd("hist", 0);
    r.true_residual_history = getd("true_hist", 0);
    rdd_summary s{};
    check(c_, rdd_get_summary(c_, &s));
    r.breakdown = s.breakdown != 0;
    return r;
  }
  std::vector<double> solution(int component = 0) const { return getd("W", component); }  // W (unscaled)

  // runner.hpp:253-256 evaluate_solution + compute_errors; returns the summary with e_L2 / e_L1n
  rdd_summary evaluate(const int* test_res) {
    check(c_, rdd_evaluate(c_, test_res));
    rdd_summary s{};
    check(c_, rdd_get_summary(c_, &s));
    return s;
  }
  // runner.hpp:202-275 run_single
  rdd_summary run_single(const rdd_config& cfg, std::uint64_t seed) {
    rdd_summary s{};
    check(c_, rdd_run_single(c_, &cfg, seed, &s));
    return s;
  }
  // run_single again on the inputs already resident in HBM
  rdd_summary rerun_resident() {
    rdd_summary s{};
    check(c_, rdd_rerun_resident(c_, &s));
    return s;
  }

  std::vector<int> geti(const char* what, int index = 0) const {
    const int64_t n = rdd_get_i(c_, what, index, nullptr, 0);
    if (n < 0) check(c_, RDD_INVALID_ARGUMENT);
    std::vector<int> v(static_cast<size_t>(n));
    if (n > 0 && rdd_get_i(c_, what, index, reinterpret_cast<int32_t*>(v.data()), n) < 0) check(c_, RDD_INVALID_ARGUMENT);
    return v;
  }
  std::vector<double> getd(const char* what, int index = 0) const {
    const int64_t n = rdd_get_d(c_, what, index, nullptr, 0);
    if (n < 0) check(c_, RDD_INVALID_ARGUMENT);
    std::vector<double> v(static_cast<size_t>(n));
    if (n > 0 && rdd_get_d(c_, what, index, v.data(), n) < 0) check(c_, RDD_INVALID_ARGUMENT);
    return v;
  }

 private:
  rdd_ctx* c_ = nullptr;
};

// krylov.hpp:413-440 dense diagnostics on a column-major host matrix (cap as kDenseSpectrumCap)
inline std::pair<std::vector<double>, std::vector<double>> spectrum(Pipeline& dev, int64_t n, const double* A,
                                                                   int cap = 0) {
  std::vector<double> wr(static_cast<size_t>(n)), wi(static_cast<size_t>(n));
  check(dev.handle(), rdd_dense_spectrum(dev.handle(), n, n, A, cap, wr.data(), wi.data()));
  return {wr, wi};
}
inline std::vector<double> singular_values(Pipeline& dev, int64_t rows, int64_t cols, const double* A, int cap = 0) {
  std::vector<double> s(static_cast<size_t>(rows < cols ? rows : cols));
  check(dev.handle(), rdd_dense_singular_values(dev.handle(), rows, cols, A, cap, s.data()));
  return s;
}
inline double condition_number(Pipeline& dev, int64_t rows, int64_t cols, const double* A, int cap = 0) {
  double k = 0.0;
  check(dev.handle(), rdd_dense_condition_number(dev.handle(), rows, cols, A, cap, &k));
  return k;
}

}  // namespace rannddm::gpu

#endif  // RANNDDM_GPU_HPP
