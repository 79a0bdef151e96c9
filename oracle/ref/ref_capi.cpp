// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// C entry points over the UNMODIFIED reference (/root/reference/proj/include/rannddm, compiled
// here against the Eigen-subset shim in oracle/eigen_shim/). Built by oracle/ref/Makefile into
// oracle/_ref/libref.so; loaded only by tests/ (oracle/ref.py) and bench.py's CPU legs. It runs
// the reference's own run_single (runner.hpp:202-275) and its phase functions for the
// configurations the reference's RunConfig can express (problems example1/2/3, the reference
// decomposition, absolute or no PCA threshold).
#include <cstdio>
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
};

rannddm::RunConfig to_run_config(const rdd_config& c) {
  if (c.problem < 1 || c.problem > 3)
    throw std::invalid_argument("reference RunConfig: only the reference's problems example1/2/3");
  if (c.decomposition != RDD_DECOMP_REFERENCE)
    throw std::invalid_argument("reference RunConfig: only the reference decomposition");
  if (c.boundary_per_edge != 0) throw std::invalid_argument("reference RunConfig: no extra boundary points");
  if (c.tau_mode == RDD_TAU_RELATIVE) throw std::invalid_argument("reference RunConfig: tau is absolute");
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
