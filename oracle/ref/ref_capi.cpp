// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// C entry points over the UNMODIFIED reference (/root/reference/proj/include/rannddm, compiled
// here against the Eigen-subset shim in oracle/eigen_shim/). Built by oracle/ref/Makefile into
// oracle/_ref/libref.so; loaded only by tests/ (oracle/ref.py) and bench.py's CPU legs. It runs
// the reference's own run_single (runner.hpp:202-275) and its phase functions for the
// configurations the reference's RunConfig can express (problems example1/2/3, the reference
// decomposition, absolute or no PCA threshold).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <optional>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "rannddm/runner.hpp"
#include "../../include/rdd.h"

namespace {

struct Ref {
  std::string err;
  rannddm::RunConfig cfg;
  std::unique_ptr<rannddm::SeedResult> res;  // ref_run_single
  // ref_build
  std::unique_ptr<rannddm::Instance> inst;
  std::unique_ptr<rannddm::EquilibratedSystem> eq;
  std::unique_ptr<rannddm::NormalBlocks> nb;
  std::unique_ptr<rannddm::SchwarzPreconditioner> pre;
  std::vector<rannddm::SolveReport> base_reports;  // ref_run_baseline
};

rannddm::RunConfig to_run_config(const rdd_config& c) {
  if (c.problem < 1 || c.problem > 3)
    throw std::invalid_argument("reference RunConfig: only the reference's problems example1/2/3");
  if (c.decomposition != RDD_DECOMP_REFERENCE)
    throw std::invalid_argument("reference RunConfig: only the reference decomposition");
  if (c.boundary_per_edge != 0) throw std::invalid_argument("reference RunConfig: no extra boundary points");
  if (c.tau_mode == RDD_TAU_RELATIVE) throw std::invalid_argument("reference RunConfig: tau is absolute");
  if (c.solver < RDD_SOLVER_QR || c.solver > RDD_SOLVER_GMRES) throw std::invalid_argument("unknown solver");
  if (c.precond < RDD_PRECOND_NONE || c.precond > RDD_PRECOND_RAS) throw std::invalid_argument("unknown preconditioner");
  rannddm::RunConfig r;
  r.problem = "example" + std::to_string(c.problem);
  r.n = c.n;
  r.ref_resolution = c.ref_resolution > 0 ? c.ref_resolution : 2001;
  const int d = rannddm::make_problem(r.problem, r.n).domain.dim;
  r.counts.assign(c.counts, c.counts + d);
  r.delta = c.delta;
  r.m = c.m;
  r.activation = c.activation == 1 ? rannddm::Activation::Sin : rannddm::Activation::Tanh;
  r.seed = c.seed;
  r.collocation.assign(c.colloc, c.colloc + d);
  r.test.assign(c.test, c.test + d);
  r.tau_on = c.tau_mode != RDD_TAU_OFF;
  r.tau = c.tau;
  r.pca_matrix = c.pca_matrix == RDD_PCA_PSI ? rannddm::PcaMatrix::psi : rannddm::PcaMatrix::op_applied;
  r.solver = static_cast<rannddm::SolverKind>(c.solver);
  if (c.precond < 0) r.preconditioner.reset();
  else r.preconditioner = static_cast<rannddm::SchwarzKind>(c.precond);
  r.rel_tol = c.rel_tol;
  r.max_iter = c.max_iter;
  r.gmres_restart = c.gmres_restart;
  return r;
}

template <class F>
int guarded(Ref* h, F&& f) {
  try {
    f();
    return RDD_OK;
  } catch (const std::invalid_argument& e) {
    h->err = e.what();
    return RDD_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    h->err = e.what();
    return RDD_DOMAIN_ERROR;
  } catch (const std::exception& e) {
    h->err = e.what();
    return RDD_RUNTIME_ERROR;
  }
}

Eigen::VectorXd vec_in(const double* p, int n) {
  Eigen::VectorXd v(n);
  for (int i = 0; i < n; ++i) v(i) = p[i];
  return v;
}

// ---- BASELINE configurations on the reference's own types: the problems C1-C5 as
// ProblemSpecs built from the reference's operators and jet helpers, the cell-centred
// decomposition filled into a CartesianDecomposition (geometry.hpp:84-97; neighbour sets by the
// reference's interiors_intersect), the reference's uniform_grid plus C1's edge points, and the
// relative PCA threshold applied to the reference's JacobiSVD (truncate at τ·σmax).
rannddm::Jet2 ramp_L(int d, const rannddm::Point& x) {
  rannddm::Jet2 v = rannddm::Jet2::constant(d, 1.0);
  for (int a = 0; a < d; ++a)
    v = v * rannddm::tanh_of_linear(d, a, x[a], 1.0) * rannddm::tanh_of_linear(d, a, x[a], -1.0, 1.0);
  return v;
}
rannddm::Jet2 gauss_of_linear(int d, int axis, double x, double alpha, double beta) {  // exp(-100 q²)
  const rannddm::Jet2 q = rannddm::Jet2::variable(d, axis, alpha * x + beta, alpha);
  const rannddm::Jet2 s = -100.0 * (q * q);
  const double e = std::exp(s.v);
  return rannddm::compose(rannddm::ScalarTriple{e, e, e}, s);
}

rannddm::ProblemSpec baseline_problem(int id, int dim) {
  using namespace rannddm;
  ProblemSpec P;
  auto value_field = [](std::function<double(const Point&)> f) {
    ScalarField sf;
    sf.value = f;
    sf.jet = nullptr;
    return sf;
  };
  switch (id) {
    case RDD_PROBLEM_POISSON: {  // C1 (2-D) / C5 (3-D): -Δu = f, u = Π sin πx_a
      const int d = dim == 0 ? 2 : dim;
      P.name = "poisson";
      P.domain.dim = d;
      for (int a = 0; a < d; ++a) {
        P.domain.lo[a] = 0.0;
        P.domain.hi[a] = 1.0;
      }
      P.op = minus_laplacian();
      P.exact = {value_field([d](const Point& x) {
        double s = 1.0;
        for (int a = 0; a < d; ++a) s *= std::sin(kPi * x[a]);
        return s;
      })};
      P.rhs = {[d](const Point& x) {
        double s = 1.0;
        for (int a = 0; a < d; ++a) s *= std::sin(kPi * x[a]);
        return (static_cast<double>(d) * kPi * kPi) * s;
      }};
      P.constraint.L = [d](const Point& x) { return ramp_L(d, x); };
      P.constraint.G = {[d](const Point&) { return Jet2::constant(d, 0.0); }};
      break;
    }
    case RDD_PROBLEM_MULTISCALE: {  // C2
      P.name = "multiscale";
      P.domain = make_box(2, {0.0, 0.0}, {1.0, 1.0});
      P.op = minus_laplacian();
      P.exact = {value_field([](const Point& x) {
        return std::sin(2.0 * kPi * x[0]) * std::sin(2.0 * kPi * x[1]) +
               0.1 * (std::sin(50.0 * kPi * x[0]) * std::sin(50.0 * kPi * x[1]));
      })};
      P.rhs = {[](const Point& x) {
        return (8.0 * kPi * kPi) * (std::sin(2.0 * kPi * x[0]) * std::sin(2.0 * kPi * x[1])) +
               (500.0 * kPi * kPi) * (std::sin(50.0 * kPi * x[0]) * std::sin(50.0 * kPi * x[1]));
      }};
      P.constraint.L = [](const Point& x) { return ramp_L(2, x); };
      P.constraint.G = {[](const Point&) { return Jet2::constant(2, 0.0); }};
      break;
    }
    case RDD_PROBLEM_HEAT: {  // C3: u_t = 0.1 Δ_xy u, axis 2 = t
      P.name = "heat";
      P.domain = make_box(3, {0.0, 0.0, 0.0}, {1.0, 1.0, 1.0});
      P.op = {"heat", [](const Point&, const Jet2& u) { return u.g[2] - 0.1 * (u.hess(0, 0) + u.hess(1, 1)); }};
      P.exact = {value_field([](const Point& x) {
        return std::exp(-0.2 * kPi * kPi * x[2]) * (std::sin(kPi * x[0]) * std::sin(kPi * x[1]));
      })};
      P.rhs = {[](const Point&) { return 0.0; }};
      P.constraint.L = [](const Point& x) {
        return tanh_of_linear(3, 0, x[0], 1.0) * tanh_of_linear(3, 0, x[0], -1.0, 1.0) *
               tanh_of_linear(3, 1, x[1], 1.0) * tanh_of_linear(3, 1, x[1], -1.0, 1.0) * tanh_of_linear(3, 2, x[2], 1.0);
      };
      P.constraint.G = {[](const Point& x) { return sin_of_linear(3, 0, x[0], kPi) * sin_of_linear(3, 1, x[1], kPi); }};
      break;
    }
    case RDD_PROBLEM_ADVECTION: {  // C4: u_t + 2 u_x = 0 on [0,2] x [0,1], axis 1 = t
      P.name = "advection";
      P.domain = make_box(2, {0.0, 0.0}, {2.0, 1.0});
      P.op = {"advection", [](const Point&, const Jet2& u) { return u.g[1] + 2.0 * u.g[0]; }};
      P.exact = {value_field([](const Point& x) {
        const double q = x[0] - 2.0 * x[1] - 0.5;
        return std::exp(-100.0 * (q * q));
      })};
      P.rhs = {[](const Point&) { return 0.0; }};
      P.constraint.L = [](const Point& x) { return tanh_of_linear(2, 0, x[0], 1.0) * tanh_of_linear(2, 1, x[1], 1.0); };
      P.constraint.G = {[](const Point& x) {
        const Jet2 u0 = gauss_of_linear(2, 0, x[0], 1.0, -0.5);
        const Jet2 g = gauss_of_linear(2, 1, x[1], 2.0, 0.5);
        return (u0 + g) - Jet2::constant(2, std::exp(-25.0));
      }};
      break;
    }
    default:
      throw std::invalid_argument("not a BASELINE problem");
  }
  P.components = 1;
  P.has_exact = true;
  return P;
}

rannddm::CartesianDecomposition cell_decomposition(const rannddm::Box& domain, const std::vector<int>& counts,
                                                   double ext) {
  using namespace rannddm;
  const int d = domain.dim;
  CartesianDecomposition dec;
  dec.domain = domain;
  dec.per_axis_counts = counts;
  dec.overlap_ratio = ext;
  std::vector<std::vector<double>> ac(d);
  std::vector<double> ah(d);
  for (int a = 0; a < d; ++a) {
    const int l = counts[a];
    const double lo = domain.lo[a], len = domain.width(a);
    if (l == 1) {
      ac[a] = {lo + 0.5 * len};
      ah[a] = 0.5 * len;
    } else {
      ah[a] = (0.5 + ext) / static_cast<double>(l) * len;
      for (int j = 0; j < l; ++j) ac[a].push_back(lo + (static_cast<double>(j) + 0.5) / static_cast<double>(l) * len);
    }
  }
  int total = 1;
  for (int c : counts) total *= c;
  std::vector<int> idx(d, 0);
  for (int flat = 0; flat < total; ++flat) {  // axis 0 slowest, as geometry.hpp:146-167
    Box sub;
    sub.dim = d;
    Point c{}, h{};
    for (int a = 0; a < d; ++a) {
      c[a] = ac[a][idx[a]];
      h[a] = ah[a];
      sub.lo[a] = c[a] - h[a];
      sub.hi[a] = c[a] + h[a];
    }
    dec.subdomains.push_back(sub);
    dec.centers.push_back(c);
    dec.half_widths.push_back(h);
    for (int a = d - 1; a >= 0; --a) {
      if (++idx[a] < counts[a]) break;
      idx[a] = 0;
    }
  }
  dec.neighbor_sets.assign(total, {});
  for (int i = 0; i < total; ++i)
    for (int j = 0; j < total; ++j)
      if (detail::interiors_intersect(dec.subdomains[i], dec.subdomains[j])) dec.neighbor_sets[i].push_back(j);
  return dec;
}

rannddm::PointSet baseline_points(const rannddm::Box& domain, const std::vector<int>& res, int nb) {
  using namespace rannddm;
  PointSet pts = uniform_grid(domain, res, PointKind::collocation);
  if (nb > 0) {  // C1: 4 x nb cell-centred edge points after the grid (y=lo, y=hi, x=lo, x=hi)
    for (int e = 0; e < 4; ++e) {
      const int axis = e < 2 ? 0 : 1, fixed = 1 - axis;
      const double fv = (e % 2 == 0) ? domain.lo[fixed] : domain.hi[fixed];
      const double st = (domain.hi[axis] - domain.lo[axis]) / static_cast<double>(nb);
      for (int k = 0; k < nb; ++k) {
        Point x{};
        x[axis] = domain.lo[axis] + (static_cast<double>(k) + 0.5) * st;
        x[fixed] = fv;
        pts.points.push_back(x);
      }
    }
  }
  return pts;
}

}  // namespace

extern "C" {

void* ref_create(void) { return new Ref(); }
void ref_destroy(void* h) { delete static_cast<Ref*>(h); }
const char* ref_last_error(void* h) { return static_cast<Ref*>(h)->err.c_str(); }

// runner.hpp:202-275 run_single, as the reference's driver calls it (runner.hpp:295-330)
int ref_run_single(void* hv, const rdd_config* c, uint64_t seed, rdd_summary* out) {
  Ref* h = static_cast<Ref*>(hv);
  return guarded(h, [&] {
    h->cfg = to_run_config(*c);
    const auto ref = rannddm::maybe_reference(h->cfg);
    h->res = std::make_unique<rannddm::SeedResult>(rannddm::run_single(h->cfg, seed, ref.get()));
    const rannddm::RunSummary& s = h->res->summary;
    std::memset(out, 0, sizeof(*out));
    out->seed = s.seed;
    out->J = s.J;
    out->DoF = s.DoF;
    out->N = s.N;
    out->p = h->res->instance->p;
    out->iterations = s.iterations;
    out->converged = s.converged ? 1 : 0;
    for (const auto& r : h->res->reports) out->breakdown |= r.breakdown ? 1 : 0;
    out->e_l2 = s.e_l2;
    out->e_l1n = s.e_l1n;
    out->t_assemble = s.t_assemble;
    out->t_precond = s.t_precond;
    out->t_solve = s.t_solve;
    double fr = 0.0;
    for (const auto& r : h->res->reports)
      if (!r.residual_history.empty()) fr = std::max(fr, r.residual_history.back());
    out->final_residual = fr;
  });
}


// run_single (runner.hpp:202-275) for a BASELINE configuration, phase by phase on the reference's
// functions: build_instance's loop (runner.hpp:52-65) over the BASELINE objects, then
// assemble_equilibrated, normal_blocks, build_index_sets, build_preconditioner, solve_with,
// evaluate_solution and compute_errors.
int ref_run_baseline(void* hv, const rdd_config* c, uint64_t seed, rdd_summary* out) {
  Ref* h = static_cast<Ref*>(hv);
  return guarded(h, [&] {
    using namespace rannddm;
    if (c->solver < RDD_SOLVER_QR || c->solver > RDD_SOLVER_GMRES) throw std::invalid_argument("unknown solver");
    if (c->precond < RDD_PRECOND_NONE || c->precond > RDD_PRECOND_RAS) throw std::invalid_argument("unknown preconditioner");
    const auto t0 = std::chrono::steady_clock::now();
    auto inst = std::make_unique<Instance>();
    std::shared_ptr<ReferenceGrid> refgrid;
    if (c->problem >= RDD_PROBLEM_POISSON) {
      inst->prob = baseline_problem(c->problem, c->dim);
    } else {  // the reference's own problems, with the BASELINE extensions of the other fields
      inst->prob = make_problem("example" + std::to_string(c->problem), c->n);
      if (!inst->prob.has_exact)
        refgrid = std::make_shared<ReferenceGrid>(reference_example2(c->ref_resolution > 0 ? c->ref_resolution : 2001));
    }
    const int d = inst->prob.domain.dim;
    std::vector<int> counts(c->counts, c->counts + d), res(c->colloc, c->colloc + d), test(c->test, c->test + d);
    inst->dec = c->decomposition == RDD_DECOMP_CELL ? cell_decomposition(inst->prob.domain, counts, c->delta)
                                                    : build_decomposition(inst->prob.domain, counts, c->delta);
    inst->collocation = baseline_points(inst->prob.domain, res, c->boundary_per_edge);
    const WindowSet ws = make_window_set(inst->dec);
    const Activation act = c->activation == 1 ? Activation::Sin : Activation::Tanh;
    for (int j = 0; j < inst->dec.size(); ++j) {
      inst->bases.push_back(make_random_basis(subdomain_seed(seed, j), c->m, d, act));
      if (c->tau_mode == RDD_TAU_OFF) {
        inst->reduced.push_back(identity_reduction(c->m));
        continue;
      }
      const SampleMatrix sm = c->pca_matrix == RDD_PCA_PSI
                                  ? build_sample_matrix(ws, j, inst->bases.back(), inst->collocation)
                                  : build_operator_sample_matrix(inst->prob.op, ws, j, inst->bases.back(),
                                                                 inst->prob.constraint, inst->collocation);
      if (c->tau_mode == RDD_TAU_ABSOLUTE) {
        inst->reduced.push_back(truncate(sm, c->tau));
      } else {  // relative: the reference's truncate at τ·σmax (its SVD, its strict > and sign rule)
        ReducedLocalBasis r = truncate(sm, 0.0);
        const double thr = c->tau * r.singular_values(0);
        int keep = 0;
        for (Eigen::Index i = 0; i < r.singular_values.size(); ++i)
          if (r.singular_values(i) > thr) ++keep;
        if (keep == 0) keep = 1;
        r.V = Eigen::MatrixXd(r.V.leftCols(keep));
        r.p = keep;
        inst->reduced.push_back(std::move(r));
      }
    }
    inst->column_offsets = make_column_offsets(inst->reduced);
    inst->p = inst->column_offsets.back();
    const EquilibratedSystem eq = assemble_equilibrated(*inst, c->precond >= 0);
    const double t_assemble = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const int C = inst->prob.components;
    Eigen::MatrixXd W(inst->p, C);
    double t_precond = 0.0, t_solve = 0.0;
    int iterations = 0;
    bool converged = true;
    h->base_reports.clear();
    if (c->solver == RDD_SOLVER_QR) {
      const auto t1 = std::chrono::steady_clock::now();
      const Eigen::MatrixXd Hd = densify(eq.sys);
      Eigen::ColPivHouseholderQR<Eigen::MatrixXd> qr(Hd);
      W = qr.solve(eq.sys.F);
      t_solve = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    } else {
      std::optional<SchwarzPreconditioner> pre;
      if (c->precond >= 0) {
        const auto t1 = std::chrono::steady_clock::now();
        const NormalBlocks nb = normal_blocks(eq.sys, inst->dec.neighbor_sets);
        pre = build_preconditioner(static_cast<SchwarzKind>(c->precond), nb,
                                   build_index_sets(inst->dec, inst->column_offsets));
        t_precond = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
      }
      const BlockSystem& sys = eq.sys;
      LinearMap A{inst->p, [&sys](const Eigen::VectorXd& w) { return matvec_transpose(sys, matvec(sys, w)); },
                  nullptr, false};
      LinearMap M = pre ? LinearMap{inst->p, [&pre](const Eigen::VectorXd& v) { return apply(*pre, v); },
                                    [&pre](const Eigen::VectorXd& v) { return apply_transpose(*pre, v); }, false}
                        : identity_map(inst->p);
      const SolveConfig scfg{static_cast<SolverKind>(c->solver), c->rel_tol, c->max_iter, c->gmres_restart};
      const auto t1 = std::chrono::steady_clock::now();
      for (int k = 0; k < C; ++k) {
        const Eigen::VectorXd b = matvec_transpose(sys, sys.F.col(k));
        SolveReport rep = solve_with(scfg, A, M, b);
        W.col(k) = rep.W;
        iterations = std::max(iterations, rep.iterations);
        converged = converged && rep.converged;
        h->base_reports.push_back(std::move(rep));
      }
      t_solve = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    }
    W.array().colwise() /= eq.scales.array();
    PointSet tp = uniform_grid(inst->prob.domain, test, PointKind::test);
    const Eigen::MatrixXd approx = evaluate_solution(*inst, W, tp);
    const Eigen::MatrixXd exact = exact_values(inst->prob, tp, refgrid.get());
    const ErrorReport err = compute_errors(approx, exact);
    std::memset(out, 0, sizeof(*out));
    out->seed = seed;
    out->J = inst->dec.size();
    out->DoF = inst->dof();
    out->N = eq.sys.N;
    out->p = inst->p;
    out->iterations = iterations;
    out->converged = converged ? 1 : 0;
    out->e_l2 = err.rel_l2;
    out->e_l1n = err.normalized_l1;
    out->t_assemble = t_assemble;
    out->t_precond = t_precond;
    out->t_solve = t_solve;
    double fr = 0.0;
    for (const auto& r : h->base_reports)
      if (!r.residual_history.empty()) fr = std::max(fr, r.residual_history.back());
    out->final_residual = fr;
    h->inst = std::move(inst);
    h->res.reset();
  });
}

// the phases of run_single one by one (runner.hpp:40-70, 89-101; assembly.hpp:148; schwarz.hpp:39, 93)
int ref_build(void* hv, const rdd_config* c, uint64_t seed, int precond) {
  Ref* h = static_cast<Ref*>(hv);
  return guarded(h, [&] {
    h->cfg = to_run_config(*c);
    h->inst = std::make_unique<rannddm::Instance>(rannddm::build_instance(h->cfg, seed));
    h->eq = std::make_unique<rannddm::EquilibratedSystem>(rannddm::assemble_equilibrated(*h->inst, precond >= 0));
    h->nb.reset();
    h->pre.reset();
    if (precond >= 0) {
      h->nb = std::make_unique<rannddm::NormalBlocks>(rannddm::normal_blocks(h->eq->sys, h->inst->dec.neighbor_sets));
      h->pre = std::make_unique<rannddm::SchwarzPreconditioner>(rannddm::build_preconditioner(
          static_cast<rannddm::SchwarzKind>(precond), *h->nb,
          rannddm::build_index_sets(h->inst->dec, h->inst->column_offsets)));
    }
  });
}

int ref_matvec(void* hv, const double* w, double* y) {
  Ref* h = static_cast<Ref*>(hv);
  return guarded(h, [&] {
    const Eigen::VectorXd r = rannddm::matvec(h->eq->sys, vec_in(w, h->eq->sys.p));
    std::memcpy(y, r.data(), sizeof(double) * r.size());
  });
}
int ref_matvec_transpose(void* hv, const double* rr, double* out) {
  Ref* h = static_cast<Ref*>(hv);
  return guarded(h, [&] {
    const Eigen::VectorXd r = rannddm::matvec_transpose(h->eq->sys, vec_in(rr, h->eq->sys.N));
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}
int ref_precond_apply(void* hv, const double* v, double* z, int transpose) {
  Ref* h = static_cast<Ref*>(hv);
  return guarded(h, [&] {
    if (!h->pre) throw std::invalid_argument("no preconditioner built");
    const Eigen::VectorXd x = vec_in(v, h->pre->size());
    const Eigen::VectorXd r = transpose ? rannddm::apply_transpose(*h->pre, x) : rannddm::apply(*h->pre, x);
    std::memcpy(z, r.data(), sizeof(double) * r.size());
  });
}

// exports: returns the element count (call with out = NULL to size), or -1
int64_t ref_get_i(void* hv, const char* what, int index, int32_t* out, int64_t cap) {
  Ref* h = static_cast<Ref*>(hv);
  std::vector<int> v;
  const std::string w(what);
  const rannddm::Instance* inst = h->inst ? h->inst.get() : (h->res ? h->res->instance.get() : nullptr);
  if (w == "p_j" && inst) for (const auto& r : inst->reduced) v.push_back(r.p);
  else if (w == "p" && inst) v = {inst->p};
  else if (w == "J" && inst) v = {inst->dec.size()};
  else if (w == "local_rank" && h->pre) v = h->pre->local_ranks;
  else if (w == "iterations" && h->res) for (const auto& r : h->res->reports) v.push_back(r.iterations);
  else {
    h->err = "ref_get_i: unknown or unavailable " + w;
    return -1;
  }
  if (out) std::memcpy(out, v.data(), sizeof(int32_t) * std::min<int64_t>(cap, v.size()));
  return static_cast<int64_t>(v.size());
}

int64_t ref_get_d(void* hv, const char* what, int index, double* out, int64_t cap) {
  Ref* h = static_cast<Ref*>(hv);
  std::vector<double> v;
  const std::string w(what);
  const rannddm::Instance* inst = h->inst ? h->inst.get() : (h->res ? h->res->instance.get() : nullptr);
  auto put = [&](const Eigen::MatrixXd& m) { v.assign(m.data(), m.data() + m.size()); };
  if (w == "sigma" && inst) put(inst->reduced[index].singular_values);
  else if (w == "V" && inst) put(inst->reduced[index].V);
  else if (w == "H" && h->eq) put(h->eq->sys.blocks[index]);
  else if (w == "scales" && h->eq) put(h->eq->scales);
  else if (w == "F" && h->eq) put(h->eq->sys.F);
  else if (w == "local_cond" && h->pre) for (const auto& l : h->pre->local_factors) v.push_back(l.cond_estimate);
  else if (w == "hist" && h->res) v = h->res->reports.at(index).residual_history;
  else if (w == "hist" && !h->base_reports.empty()) v = h->base_reports.at(index).residual_history;
  else if (w == "true_hist" && h->res) v = h->res->reports.at(index).true_residual_history;
  else if (w == "W" && h->res) put(h->res->reports.at(index).W);
  else {
    h->err = "ref_get_d: unknown or unavailable " + w;
    return -1;
  }
  if (out) std::memcpy(out, v.data(), sizeof(double) * std::min<int64_t>(cap, v.size()));
  return static_cast<int64_t>(v.size());
}

}  // extern "C"
