// rannddm_gpu_ref.hpp — the level-2 drop-in: the reference's own types and phase signatures
// (rannddm::RunConfig, ProblemSpec, CartesianDecomposition, PointSet, RandomBasis, LinearMap,
// SeedResult) over the device C ABI (rdd.h / librdd.so).
//
// A reference maintainer includes this AFTER the reference headers (it needs Eigen, or the
// Eigen-subset shim this repository builds the reference with, oracle/eigen_shim/), links
// librdd.so, and swaps the phases of run_single (runner.hpp:202-275) one by one:
//
//   rannddm::gpu::Context dev;                              // one device context (rdd_create)
//   rannddm::gpu::build_instance(dev, cfg, prob, seed);     // runner.hpp:40-70, any ProblemSpec
//   rannddm::gpu::assemble(dev, true);                      // runner.hpp:89-101
//   rannddm::gpu::build_preconditioner(dev, SchwarzKind::AS); // assembly.hpp:148 + schwarz.hpp:39,93
//   LinearMap A = rannddm::gpu::normal_operator(dev);       // runner.hpp:232-234
//   LinearMap M = rannddm::gpu::preconditioner(dev);        // schwarz.hpp:153-215
//   SolveReport rep = rannddm::cg(A, M, rannddm::gpu::rhs(dev, 0), scfg);   // the reference's own CG
//   Eigen::MatrixXd u = rannddm::gpu::evaluate_solution(dev, W, pts, prob); // runner.hpp:105-127
//
// or replaces run_single wholesale for the built-in problems (rannddm::gpu::run_single).
// Every function throws the reference's exception classes with the library's message.
#pragma once

#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "rannddm/runner.hpp"
#include "rdd.h"

namespace rannddm::gpu {

inline void check(rdd_ctx* h, int st) {
  if (st == RDD_OK) return;
  const std::string msg = h ? rdd_last_error(h) : "rdd: no context";
  switch (st) {
    case RDD_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case RDD_DOMAIN_ERROR: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

/// One device context (one CUDA stream); move-only.
class Context {
 public:
  explicit Context(int device = 0) {
    if (rdd_create(&h_, device) != RDD_OK || !h_) throw std::runtime_error("rdd_create: no usable CUDA device");
  }
  ~Context() {
    if (h_) rdd_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  rdd_ctx* get() const { return h_; }
  void operator()(int st) const { check(h_, st); }

 private:
  rdd_ctx* h_ = nullptr;
};

/// config.hpp:23-68 RunConfig -> rdd_config (the reference's problems, decomposition and
/// absolute PCA threshold; the BASELINE extensions keep their defaults).
inline rdd_config to_rdd_config(const RunConfig& r) {
  rdd_config c{};
  if (r.problem == "example1") c.problem = RDD_PROBLEM_EXAMPLE1;
  else if (r.problem == "example2") c.problem = RDD_PROBLEM_EXAMPLE2;
  else if (r.problem == "example3") c.problem = RDD_PROBLEM_EXAMPLE3;
  else throw std::invalid_argument("unknown problem: " + r.problem);  // problems.hpp:172
  c.n = r.n;
  const int d = make_problem(r.problem, r.n).domain.dim;
  c.dim = d;
  if (static_cast<int>(r.counts.size()) != d || static_cast<int>(r.collocation.size()) != d ||
      static_cast<int>(r.test.size()) != d)
    throw std::invalid_argument("point resolutions must match the problem dimension");
  for (int a = 0; a < d; ++a) {
    c.counts[a] = r.counts[static_cast<std::size_t>(a)];
    c.colloc[a] = r.collocation[static_cast<std::size_t>(a)];
    c.test[a] = r.test[static_cast<std::size_t>(a)];
  }
  c.decomposition = RDD_DECOMP_REFERENCE;
  c.delta = r.delta;
  c.m = r.m;
  c.activation = r.activation == Activation::Sin ? 1 : 0;
  c.seed = r.seed;
  c.boundary_per_edge = 0;
  c.tau_mode = r.tau_on ? RDD_TAU_ABSOLUTE : RDD_TAU_OFF;
  c.tau = r.tau;
  c.pca_matrix = r.pca_matrix == PcaMatrix::psi ? RDD_PCA_PSI : RDD_PCA_OP_APPLIED;
  c.solver = static_cast<int>(r.solver);  // SolverKind order = RDD_SOLVER_*
  c.precond = r.preconditioner ? static_cast<int>(*r.preconditioner) : RDD_PRECOND_NONE;
  c.rel_tol = r.rel_tol;
  c.max_iter = r.max_iter;
  c.gmres_restart = r.gmres_restart;
  c.op_form = RDD_OPERATOR_TWO_PASS;
  c.true_residual = 1;
  c.ref_resolution = r.ref_resolution;
  return c;
}

/// The operator's constant coefficients on the jet (value, gradient, Hessian upper triangle), by
/// applying the reference's LinearOperator to unit jets; checked at a few points of the domain.
inline std::vector<double> operator_coefficients(const ProblemSpec& prob) {
  const int d = prob.domain.dim, jl = 1 + d + d * (d + 1) / 2;
  auto probe = [&](const Point& x) {
    std::vector<double> c(static_cast<std::size_t>(jl));
    for (int k = 0; k < jl; ++k) {
      Jet2 e = Jet2::constant(d, 0.0);
      if (k == 0) e.v = 1.0;
      else if (k <= d) e.g[static_cast<std::size_t>(k - 1)] = 1.0;
      else e.h[static_cast<std::size_t>(k - 1 - d)] = 1.0;
      c[static_cast<std::size_t>(k)] = prob.op.apply(x, e);
    }
    return c;
  };
  Point x0{};
  for (int a = 0; a < d; ++a) x0[static_cast<std::size_t>(a)] = 0.5 * (prob.domain.lo[a] + prob.domain.hi[a]);
  const std::vector<double> c0 = probe(x0);
  for (double t : {0.17, 0.61, 0.93}) {
    Point x{};
    for (int a = 0; a < d; ++a)
      x[static_cast<std::size_t>(a)] = prob.domain.lo[a] + t * (prob.domain.hi[a] - prob.domain.lo[a]);
    if (probe(x) != c0) throw std::invalid_argument("device operators need constant coefficients: " + prob.op.name);
  }
  return c0;
}

/// Hands the reference's objects to the device: the decomposition, the collocation PointSet,
/// the RandomBasis of every subdomain and the ProblemSpec evaluated at the points (L jets,
/// F = f − A[G] as assembly.hpp:97-106).
inline void upload(Context& dev, const CartesianDecomposition& dec, const PointSet& pts,
                   const std::vector<RandomBasis>& bases, const ProblemSpec& prob) {
  const int d = dec.dim(), J = dec.size(), N = pts.size(), C = prob.components;
  const int jl = 1 + d + d * (d + 1) / 2;
  std::vector<double> dlo(d), dhi(d), lo, hi, ctr, half;
  for (int a = 0; a < d; ++a) {
    dlo[static_cast<std::size_t>(a)] = dec.domain.lo[a];
    dhi[static_cast<std::size_t>(a)] = dec.domain.hi[a];
  }
  std::vector<int32_t> counts(dec.per_axis_counts.begin(), dec.per_axis_counts.end()), nptr{0}, nidx;
  for (int j = 0; j < J; ++j) {
    const auto sj = static_cast<std::size_t>(j);
    for (int a = 0; a < d; ++a) {
      const auto sa = static_cast<std::size_t>(a);
      lo.push_back(dec.subdomains[sj].lo[sa]);
      hi.push_back(dec.subdomains[sj].hi[sa]);
      ctr.push_back(dec.centers[sj][sa]);
      half.push_back(dec.half_widths[sj][sa]);
    }
    for (int k : dec.neighbor_sets[sj]) nidx.push_back(k);
    nptr.push_back(static_cast<int32_t>(nidx.size()));
  }
  dev(rdd_set_decomposition(dev.get(), d, counts.data(), dlo.data(), dhi.data(), lo.data(), hi.data(), ctr.data(),
                            half.data(), nptr.data(), nidx.data()));
  std::vector<double> xs(static_cast<std::size_t>(N) * d);
  for (int i = 0; i < N; ++i)
    for (int a = 0; a < d; ++a)
      xs[static_cast<std::size_t>(i) * d + a] = pts.points[static_cast<std::size_t>(i)][static_cast<std::size_t>(a)];
  dev(rdd_set_points(dev.get(), N, xs.data()));
  const int m = bases.empty() ? 0 : bases[0].m;
  std::vector<double> R, b;
  for (const RandomBasis& B : bases) {
    if (B.m != m || B.dim != d || B.act != bases[0].act)
      throw std::invalid_argument("bases: one width, dimension and activation for every subdomain");
    for (int k = 0; k < m; ++k)
      for (int a = 0; a < d; ++a) R.push_back(B.R(k, a));
    for (int k = 0; k < m; ++k) b.push_back(B.b(k));
  }
  dev(rdd_set_bases(dev.get(), J, m, R.data(), b.data(), bases.empty() || bases[0].act == Activation::Tanh ? 0 : 1));
  const std::vector<double> coef = operator_coefficients(prob);
  std::vector<double> Lj(static_cast<std::size_t>(N) * jl), F(static_cast<std::size_t>(N) * C);
  for (int i = 0; i < N; ++i) {
    const Point& x = pts.points[static_cast<std::size_t>(i)];
    const Jet2 L = prob.constraint.L(x);
    double* row = Lj.data() + static_cast<std::size_t>(i) * jl;
    row[0] = L.v;
    for (int a = 0; a < d; ++a) row[1 + a] = L.g[static_cast<std::size_t>(a)];
    for (int k = 0; k < d * (d + 1) / 2; ++k) row[1 + d + k] = L.h[static_cast<std::size_t>(k)];
    for (int c = 0; c < C; ++c)
      F[static_cast<std::size_t>(c) * N + i] =
          prob.rhs[static_cast<std::size_t>(c)](x) - prob.op.apply(x, prob.constraint.G[static_cast<std::size_t>(c)](x));
  }
  dev(rdd_set_problem(dev.get(), C, coef.data(), Lj.data(), F.data()));
}

/// runner.hpp:40-70 build_instance for any ProblemSpec: the reference's own decomposition,
/// collocation grid and seeded bases, handed to the device, which runs the per-subdomain PCA.
inline void build_instance(Context& dev, const RunConfig& cfg, const ProblemSpec& prob, std::uint64_t seed) {
  const int d = prob.domain.dim;
  if (static_cast<int>(cfg.counts.size()) != d)
    throw std::invalid_argument("decomposition counts have dimension " + std::to_string(cfg.counts.size()) +
                                " but the problem is " + std::to_string(d) + "-dimensional");
  const CartesianDecomposition dec = build_decomposition(prob.domain, cfg.counts, cfg.delta);
  const PointSet pts = uniform_grid(prob.domain, cfg.collocation, PointKind::collocation);
  std::vector<RandomBasis> bases;
  for (int j = 0; j < dec.size(); ++j) bases.push_back(make_random_basis(subdomain_seed(seed, j), cfg.m, d, cfg.activation));
  upload(dev, dec, pts, bases, prob);
  rdd_config c{};
  c.tau_mode = cfg.tau_on ? RDD_TAU_ABSOLUTE : RDD_TAU_OFF;
  c.tau = cfg.tau;
  c.pca_matrix = cfg.pca_matrix == PcaMatrix::psi ? RDD_PCA_PSI : RDD_PCA_OP_APPLIED;
  c.solver = static_cast<int>(cfg.solver);
  c.precond = cfg.preconditioner ? static_cast<int>(*cfg.preconditioner) : RDD_PRECOND_NONE;
  c.rel_tol = cfg.rel_tol;
  c.max_iter = cfg.max_iter;
  c.gmres_restart = cfg.gmres_restart;
  c.true_residual = 1;
  c.seed = seed;
  dev(rdd_build_custom(dev.get(), &c));
}

/// runner.hpp:89-101 assemble_equilibrated (assembly.hpp:41-108, 186-204).
inline void assemble(Context& dev, bool equilibrate = true) { dev(rdd_assemble(dev.get(), equilibrate ? 1 : 0)); }

/// assembly.hpp:148-183 normal_blocks + schwarz.hpp:39-61 build_index_sets + :93-148 build_preconditioner.
inline void build_preconditioner(Context& dev, SchwarzKind kind) {
  dev(rdd_build_preconditioner(dev.get(), static_cast<int>(kind)));
}

inline int size(const Context& dev) {
  int32_t p = 0;
  rdd_get_i(dev.get(), "p", 0, &p, 1);
  return p;
}

/// The normal operator w -> Hᵀ(H w) of runner.hpp:232-234 as the reference's LinearMap.
inline LinearMap normal_operator(Context& dev) {
  const int p = size(dev);
  Context* d = &dev;
  return LinearMap{p,
                   [d, p](const Eigen::VectorXd& w) {
                     Eigen::VectorXd out(p);
                     (*d)(rdd_normal_apply(d->get(), w.data(), w.size(), out.data(), p));
                     return out;
                   },
                   nullptr, false};
}

/// The Schwarz preconditioner (schwarz.hpp:153-215 apply / apply_transpose) as a LinearMap.
inline LinearMap preconditioner(Context& dev) {
  const int p = size(dev);
  Context* d = &dev;
  auto ap = [d, p](bool tr) {
    return [d, p, tr](const Eigen::VectorXd& v) {
      Eigen::VectorXd z(p);
      (*d)(rdd_precond_apply(d->get(), v.data(), v.size(), z.data(), p, tr ? 1 : 0));
      return z;
    };
  };
  return LinearMap{p, ap(false), ap(true), false};
}

/// b_c = Hᵀ F_c (runner.hpp:242) on the equilibrated system.
inline Eigen::VectorXd rhs(Context& dev, int c) {
  int32_t N = 0, p = 0;
  rdd_get_i(dev.get(), "N", 0, &N, 1);
  rdd_get_i(dev.get(), "p", 0, &p, 1);
  std::vector<double> F(static_cast<std::size_t>(rdd_get_d(dev.get(), "F", 0, nullptr, 0)));
  rdd_get_d(dev.get(), "F", 0, F.data(), static_cast<int64_t>(F.size()));
  Eigen::VectorXd b(p);
  dev(rdd_matvec_transpose(dev.get(), F.data() + static_cast<std::size_t>(c) * N, N, b.data(), p));
  return b;
}

/// The equilibration scales (runner.hpp:96-99): W = W_eq ./ scales.
inline Eigen::VectorXd scales(Context& dev) {
  const int p = size(dev);
  Eigen::VectorXd s(p);
  dev(rdd_get_d(dev.get(), "scales", 0, s.data(), p) == p ? RDD_OK : RDD_RUNTIME_ERROR);
  return s;
}

/// runner.hpp:105-127 evaluate_solution(inst, W, pts): W unscaled (p x C).
inline Eigen::MatrixXd evaluate_solution(Context& dev, const Eigen::MatrixXd& W, const PointSet& pts,
                                         const ProblemSpec& prob) {
  const int d = prob.domain.dim, M = pts.size(), C = prob.components;
  if (W.rows() != size(dev) || W.cols() != C) throw std::invalid_argument("evaluate_solution: W has wrong shape");
  std::vector<double> xs(static_cast<std::size_t>(M) * d), Lv(static_cast<std::size_t>(M)),
      Gv(static_cast<std::size_t>(M) * C);
  for (int i = 0; i < M; ++i) {
    const Point& x = pts.points[static_cast<std::size_t>(i)];
    for (int a = 0; a < d; ++a) xs[static_cast<std::size_t>(i) * d + a] = x[static_cast<std::size_t>(a)];
    Lv[static_cast<std::size_t>(i)] = prob.constraint.L(x).v;
    for (int c = 0; c < C; ++c)
      Gv[static_cast<std::size_t>(c) * M + i] = prob.constraint.G[static_cast<std::size_t>(c)](x).v;
  }
  Eigen::MatrixXd out(M, C);
  dev(rdd_evaluate_at(dev.get(), M, xs.data(), W.data(), Lv.data(), Gv.data(), out.data()));
  return out;
}

/// runner.hpp:202-275 run_single on the device end to end (the reference's problems): the
/// summary row as the reference fills it; one SolveReport per component with the histories.
inline SeedResult run_single(Context& dev, const RunConfig& cfg, std::uint64_t seed) {
  rdd_config c = to_rdd_config(cfg);
  rdd_summary s{};
  dev(rdd_run_single(dev.get(), &c, seed, &s));
  SeedResult out;
  RunSummary& r = out.summary;
  r.seed = seed;
  r.problem = cfg.problem;
  r.J = s.J;
  r.DoF = s.DoF;
  r.N = s.N;
  r.solver = to_string(cfg.solver);
  r.precond = cfg.solver == SolverKind::qr_direct ? "none" : cfg.precond_label();
  r.tau = cfg.tau_label();
  r.iterations = s.iterations;
  r.converged = s.converged != 0;
  r.e_l2 = s.e_l2;
  r.e_l1n = s.e_l1n;
  r.t_assemble = s.t_assemble;
  r.t_precond = s.t_precond;
  r.t_solve = s.t_solve;
  if (cfg.solver != SolverKind::qr_direct) {
    int32_t C = 1;
    rdd_get_i(dev.get(), "C", 0, &C, 1);
    for (int k = 0; k < C; ++k) {
      SolveReport rep;
      auto get = [&](const char* what) {
        std::vector<double> v(static_cast<std::size_t>(std::max<int64_t>(0, rdd_get_d(dev.get(), what, k, nullptr, 0))));
        rdd_get_d(dev.get(), what, k, v.data(), static_cast<int64_t>(v.size()));
        return v;
      };
      rep.residual_history = get("hist");
      rep.true_residual_history = get("true_hist");
      rep.iterations = static_cast<int>(rep.residual_history.size()) - 1;
      rep.converged = r.converged;
      rep.final_preconditioned_residual = rep.residual_history.empty() ? 0.0 : rep.residual_history.back();
      const std::vector<double> w = get("W");
      rep.W = Eigen::VectorXd(static_cast<Eigen::Index>(w.size()));
      for (std::size_t q = 0; q < w.size(); ++q) rep.W(static_cast<Eigen::Index>(q)) = w[q];
      out.reports.push_back(std::move(rep));
    }
  }
  return out;
}

}  // namespace rannddm::gpu
