// dropin.cpp — the level-2 drop-in test: the UNMODIFIED reference (compiled against
// the Eigen-subset shim) and the device path through include/rannddm_gpu_ref.hpp, side by side.
// Prints one JSON line per scenario; tests/test_dropin_gpu.py asserts on them.
//   A  a problem the reference does not ship (-Δu + 2u_x - u_y + u/2 = f, L = x(1-x)y(1-y)),
//      reference pipeline on the CPU vs the device pipeline fed the reference's own objects
//   B  the reference's own cg() and gmres() driving the device LinearMaps (normal operator,
//      Schwarz preconditioner) vs the device's solver and the reference on the CPU
//   C  rannddm::gpu::run_single(to_rdd_config(cfg)) vs rannddm::run_single(cfg)
#include <cstdio>
#include <string>
#include <vector>

#include "rannddm/runner.hpp"
#include "rannddm_gpu_ref.hpp"

using namespace rannddm;

static ProblemSpec custom_problem() {
  ProblemSpec prob;
  prob.name = "dropin_custom";
  prob.domain = make_box(2, {0.0, 0.0}, {1.0, 1.0});
  prob.components = 1;
  prob.op = {"conv_diff_react", [](const Point&, const Jet2& u) {
               return -(u.hess(0, 0) + u.hess(1, 1)) + 2.0 * u.g[0] - u.g[1] + 0.5 * u.v;
             }};
  auto ujet = [](const Point& x) {
    const double e = std::exp(0.5 * x[0]);
    Jet2 E = Jet2::constant(2, e);
    E.g[0] = 0.5 * e;
    E.hess_ref(0, 0) = 0.25 * e;
    return E * sin_of_linear(2, 0, x[0], kPi) * sin_of_linear(2, 1, x[1], 2.0 * kPi);
  };
  ScalarField ex;
  ex.value = [ujet](const Point& x) { return ujet(x).v; };
  ex.jet = ujet;
  prob.exact = {ex};
  prob.has_exact = true;
  const LinearOperator op = prob.op;
  prob.rhs = {[op, ujet](const Point& x) { return op.apply(x, ujet(x)); }};
  prob.constraint.L = [](const Point& x) {
    Jet2 L = Jet2::constant(2, x[0] * (1.0 - x[0]) * x[1] * (1.0 - x[1]));
    L.g[0] = (1.0 - 2.0 * x[0]) * x[1] * (1.0 - x[1]);
    L.g[1] = x[0] * (1.0 - x[0]) * (1.0 - 2.0 * x[1]);
    L.hess_ref(0, 0) = -2.0 * x[1] * (1.0 - x[1]);
    L.hess_ref(0, 1) = (1.0 - 2.0 * x[0]) * (1.0 - 2.0 * x[1]);
    L.hess_ref(1, 1) = -2.0 * x[0] * (1.0 - x[0]);
    return L;
  };
  prob.constraint.G = {[](const Point&) { return Jet2::constant(2, 0.0); }};
  return prob;
}

// runner.hpp:40-70 with a caller ProblemSpec, on the reference's own functions
static Instance reference_instance(const RunConfig& cfg, const ProblemSpec& prob, std::uint64_t seed) {
  Instance inst;
  inst.prob = prob;
  const int d = prob.domain.dim;
  inst.dec = build_decomposition(prob.domain, cfg.counts, cfg.delta);
  inst.collocation = uniform_grid(prob.domain, cfg.collocation, PointKind::collocation);
  const WindowSet ws = make_window_set(inst.dec);
  for (int j = 0; j < inst.dec.size(); ++j) {
    inst.bases.push_back(make_random_basis(subdomain_seed(seed, j), cfg.m, d, cfg.activation));
    if (cfg.tau_on)
      inst.reduced.push_back(truncate(build_operator_sample_matrix(prob.op, ws, j, inst.bases.back(), prob.constraint,
                                                                   inst.collocation),
                                      cfg.tau));
    else
      inst.reduced.push_back(identity_reduction(cfg.m));
  }
  inst.column_offsets = make_column_offsets(inst.reduced);
  inst.p = inst.column_offsets.back();
  return inst;
}

static std::string ivec(const std::vector<int>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}

static double rel_diff(const Eigen::MatrixXd& a, const Eigen::MatrixXd& b, const Eigen::MatrixXd& scale) {
  return (a - b).norm() / scale.norm();
}

static std::vector<int> device_pj(gpu::Context& dev) {
  int32_t J = 0;
  rdd_get_i(dev.get(), "J", 0, &J, 1);
  std::vector<int32_t> v(static_cast<size_t>(J));
  rdd_get_i(dev.get(), "p_j", 0, v.data(), J);
  return std::vector<int>(v.begin(), v.end());
}

int main() {
  gpu::Context dev(0);
  const std::uint64_t seed = 4242;

  // ---------------------------------------------------------------- A: caller ProblemSpec
  RunConfig cfg;
  cfg.counts = {3, 3};
  cfg.delta = 1.5;
  cfg.m = 60;
  cfg.collocation = {36, 36};
  cfg.test = {60, 60};
  cfg.tau_on = true;
  cfg.tau = 1e-4;
  cfg.solver = SolverKind::cg;
  cfg.preconditioner = SchwarzKind::AS;
  cfg.rel_tol = 1e-10;
  const ProblemSpec prob = custom_problem();
  const Instance inst = reference_instance(cfg, prob, seed);
  const EquilibratedSystem eq = assemble_equilibrated(inst, true);
  const NormalBlocks nb = normal_blocks(eq.sys, inst.dec.neighbor_sets);
  const SchwarzPreconditioner pre =
      build_preconditioner(SchwarzKind::AS, nb, build_index_sets(inst.dec, inst.column_offsets));
  LinearMap Aref{inst.p, [&eq](const Eigen::VectorXd& w) { return matvec_transpose(eq.sys, matvec(eq.sys, w)); },
                 nullptr, false};
  LinearMap Mref{inst.p, [&pre](const Eigen::VectorXd& v) { return apply(pre, v); },
                 [&pre](const Eigen::VectorXd& v) { return apply_transpose(pre, v); }, false};
  const SolveConfig scfg{cfg.solver, cfg.rel_tol, cfg.max_iter, cfg.gmres_restart};
  const SolveReport rref = solve_with(scfg, Aref, Mref, matvec_transpose(eq.sys, eq.sys.F.col(0)));
  Eigen::MatrixXd Wref(inst.p, 1);
  Wref.col(0) = rref.W;
  Wref.array().colwise() /= eq.scales.array();
  const PointSet test = uniform_grid(prob.domain, cfg.test, PointKind::test);
  const Eigen::MatrixXd uref = evaluate_solution(inst, Wref, test);
  const Eigen::MatrixXd uex = exact_values(prob, test, nullptr);
  const ErrorReport eref = compute_errors(uref, uex);
  std::vector<int> pref;
  for (const auto& r : inst.reduced) pref.push_back(r.p);

  gpu::build_instance(dev, cfg, prob, seed);
  gpu::assemble(dev, true);
  gpu::build_preconditioner(dev, SchwarzKind::AS);
  dev(rdd_solve(dev.get(), RDD_SOLVER_CG, cfg.rel_tol, 0, 0));
  int32_t its_dev = 0;
  rdd_get_i(dev.get(), "iterations", 0, &its_dev, 1);
  Eigen::MatrixXd Wdev(gpu::size(dev), 1);
  rdd_get_d(dev.get(), "W", 0, Wdev.data(), Wdev.size());
  const Eigen::MatrixXd udev = gpu::evaluate_solution(dev, Wdev, test, prob);
  const ErrorReport edev = compute_errors(udev, uex);
  std::printf("{\"scenario\": \"A\", \"p_j_ref\": %s, \"p_j_dev\": %s, \"its_ref\": %d, \"its_dev\": %d, "
              "\"e_l2_ref\": %.17g, \"e_l2_dev\": %.17g, \"u_rel_diff\": %.6g}\n",
              ivec(pref).c_str(), ivec(device_pj(dev)).c_str(), rref.iterations, its_dev, eref.rel_l2, edev.rel_l2,
              rel_diff(udev, uref, uex));

  // ---------------------------------------------------------------- B: the reference's Krylov over device maps
  const LinearMap Adev = gpu::normal_operator(dev), Mdev = gpu::preconditioner(dev);
  const Eigen::VectorXd bdev = gpu::rhs(dev, 0), sdev = gpu::scales(dev);
  for (SolverKind sk : {SolverKind::cg, SolverKind::gmres}) {
    const SolveConfig sc{sk, cfg.rel_tol, 0, 0};
    const SolveReport r = solve_with(sc, Adev, Mdev, bdev);
    const SolveReport rr = solve_with(sc, Aref, Mref, matvec_transpose(eq.sys, eq.sys.F.col(0)));
    Eigen::MatrixXd W(gpu::size(dev), 1);
    W.col(0) = r.W;
    W.array().colwise() /= sdev.array();
    const Eigen::MatrixXd u = gpu::evaluate_solution(dev, W, test, prob);
    dev(rdd_solve(dev.get(), sk == SolverKind::cg ? RDD_SOLVER_CG : RDD_SOLVER_GMRES, cfg.rel_tol, 0, 0));
    int32_t itd = 0;
    rdd_get_i(dev.get(), "iterations", 0, &itd, 1);
    std::printf("{\"scenario\": \"B\", \"solver\": \"%s\", \"its_refkrylov_devmaps\": %d, \"its_dev\": %d, "
                "\"its_ref\": %d, \"converged\": %d, \"e_l2\": %.17g, \"e_l2_ref\": %.17g, \"u_rel_diff_ref\": %.6g}\n",
                to_string(sk), r.iterations, itd, rr.iterations, r.converged ? 1 : 0,
                compute_errors(u, uex).rel_l2, eref.rel_l2, rel_diff(u, uref, uex));
  }

  // ---------------------------------------------------------------- C: run_single drop-in
  for (std::uint64_t s : {77ull, 78ull}) {
    RunConfig rc;  // test_runner.cpp:13-42 small_config
    rc.problem = "example1";
    rc.n = 1;
    rc.counts = {2, 2};
    rc.m = 8;
    rc.collocation = {12, 12};
    rc.test = {40, 40};
    rc.seed = s;
    const SeedResult a = run_single(rc, s);
    const SeedResult b = gpu::run_single(dev, rc, s);
    std::printf("{\"scenario\": \"C\", \"seed\": %llu, \"ref\": [%d, %d, %d, %d, %.17g], \"dev\": [%d, %d, %d, %d, %.17g]}\n",
                static_cast<unsigned long long>(s), a.summary.J, a.summary.DoF, a.summary.N, a.summary.iterations,
                a.summary.e_l2, b.summary.J, b.summary.DoF, b.summary.N, b.summary.iterations, b.summary.e_l2);
  }
  return 0;
}
