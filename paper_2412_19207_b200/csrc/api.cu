#include <cstdio>
// api.cu — the C ABI (include/rdd.h) and the run_single orchestration (runner.hpp:202-275).
//
// Error mapping mirrors the reference's exception classes: std::invalid_argument -> 1,
// std::runtime_error -> 2, std::domain_error -> 3, CUDA failures -> 4; the message text is the
// reference's where the reference has one. There is no CPU fallback: without a CUDA device
// rdd_create fails and every call reports it.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <future>

#include "ctx.hpp"

struct rdd_ctx {
  rdd::Ctx c;
};

namespace rdd {


void upload_inputs(Ctx& c) {
  c.pts.upload(c.h_pts, c.stream);
  std::vector<double> box(static_cast<size_t>(c.J) * 16, 0.0);
  for (int j = 0; j < c.J; ++j)
    for (int a = 0; a < 4; ++a) {
      box[j * 16 + a] = c.box_lo[j * 4 + a];
      box[j * 16 + 4 + a] = c.box_hi[j * 4 + a];
      box[j * 16 + 8 + a] = c.box_c[j * 4 + a];
      box[j * 16 + 12 + a] = c.box_h[j * 4 + a];
    }
  c.dbox.upload(box, c.stream);
  c.dnbr_ptr.upload(c.nbr_ptr, c.stream);
  c.dnbr_idx.upload(c.nbr_idx, c.stream);
  c.R.upload(c.h_R, c.stream);
  c.bvec.upload(c.h_b, c.stream);
}

static void reset_state(Ctx& c) {
  c.assembled = false;
  c.equilibrated = false;
  c.pkind = RDD_PRECOND_NONE;
  c.nb_j1.clear();
  c.nb_j2.clear();
  c.nb_index.clear();
  c.nb_off.clear();
  c.local_rank.clear();
  c.local_cond.clear();
  c.hist.clear();
  c.true_hist.clear();
  c.iters.clear();
  c.conv.clear();
  c.brk.clear();
  c.approx.clear();
  c.exact.clear();
  c.sum = rdd_summary{};
  c.H = nullptr;
  c.ras_panel = false;
  c.mt_groups = 0;
}

// runner.hpp:40-70
static void build_instance(Ctx& c, const rdd_config& cfg, uint64_t seed) {
  reset_state(c);
  const double h0 = now_s();
  setup_problem(c, cfg, seed);
  const double h1 = now_s();
  upload_inputs(c);
  if (c.verbose) {
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    std::fprintf(stderr, "[host] setup %.3f ms, upload %.3f ms\n", 1e3 * (h1 - h0), 1e3 * (now_s() - h1));
  }
  build_index(c);
  eval_problem(c);
  run_pca(c);
  ensure_col_owner(c);
}

// runner.hpp:40-70 on caller inputs (rdd_set_decomposition / points / bases / problem)
static void build_custom(Ctx& c, const rdd_config& cfg) {
  reset_state(c);
  setup_custom(c, cfg);
  upload_inputs(c);
  build_index(c);
  upload_custom_problem(c);
  run_pca(c);
  ensure_col_owner(c);
}

// runner.hpp:89-101 + assembly.hpp:41-108
static void assemble(Ctx& c, bool equilibrate) {
  if (c.h_p.empty()) throw std::invalid_argument("assemble: build_instance first");
  project_blocks(c);
  // F (assembly.hpp:97-106) was evaluated with the problem closures
  c.F.ensure(static_cast<size_t>(c.N) * c.C);
  RDD_CUDA(cudaMemcpyAsync(c.F.p, c.Fpt.p, sizeof(double) * c.N * c.C, cudaMemcpyDeviceToDevice, c.stream));
  column_norms_scale(c, equilibrate);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  c.assembled = true;
  c.equilibrated = equilibrate;
}

// resident = true reruns the pipeline on the inputs already in HBM (points, boxes, bases)
static void run_single(Ctx& c, const rdd_config& cfg, uint64_t seed, bool resident = false) {
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  double t0 = now_s();
  if (resident) {
    if (c.J == 0 || c.seed != seed) throw std::invalid_argument("rerun: no resident instance for this seed");
    reset_state(c);
    c.cfg = cfg;
    build_index(c);
    if (c.prob.id == 0) upload_custom_problem(c);
    else eval_problem(c);
    run_pca(c);
    ensure_col_owner(c);
  } else {
    build_instance(c, cfg, seed);
  }
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  const double t_pca = now_s() - t0;
  if (c.verbose) std::fprintf(stderr, "[phase] instance+pca %.3f s (J=%d p=%d N=%d) upload-wait %.3f s\n", t_pca, c.J, c.p, c.N, upload_wait_s());
  assemble(c, cfg.precond >= 0);
  const double t_asm = now_s() - t0;
  if (c.verbose) std::fprintf(stderr, "[phase] assemble done %.3f s\n", t_asm);
  double t_pre = 0.0;
  if (cfg.solver == RDD_SOLVER_QR) {  // runner.hpp:217-222: no preconditioner, no Krylov
  } else if (cfg.precond >= 0) {
    t0 = now_s();
    // the Schwarz index sets are host work independent of the normal blocks: a host thread builds
    // them while the device forms the blocks
    auto idx = std::async(std::launch::async, [&c] { return prepare_schwarz_index(c); });
    build_normal_blocks(c);
    SchwarzIndex x = idx.get();
    build_schwarz(c, cfg.precond, &x);
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    t_pre = now_s() - t0;
    if (c.verbose) std::fprintf(stderr, "[phase] precond %.3f s (fallback %d) upload-wait %.3f s\n", t_pre, c.n_fallback, upload_wait_s());
  } else if (cfg.op_form == RDD_OPERATOR_NORMAL) {
    build_normal_blocks(c);
  }
  t0 = now_s();
  if (cfg.solver == RDD_SOLVER_QR) qr_solve_dev(c);
  else solve_all(c, cfg.solver, cfg.rel_tol, cfg.max_iter, cfg.gmres_restart);
  const double t_sol = now_s() - t0;
  if (c.verbose) std::fprintf(stderr, "[phase] solve %.3f s (%d its) upload-wait %.3f s\n", t_sol, c.iters.empty() ? 0 : c.iters[0], upload_wait_s());
  t0 = now_s();
  if (c.prob.id != 0) evaluate(c, cfg.test);  // caller problems evaluate at caller points (evaluate_at)
  const double t_ev = now_s() - t0;
  rdd_summary& s = c.sum;
  s.seed = seed;
  s.J = c.J;
  s.p = c.p;
  s.DoF = c.p * c.C;
  s.N = c.N;
  int it = 0, cv = 1, bk = 0;
  double fr = 0.0;
  for (int k = 0; k < c.C; ++k) {
    it = std::max(it, c.iters[k]);
    cv = cv && c.conv[k];
    bk = bk || c.brk[k];
    if (!c.hist[k].empty()) fr = std::max(fr, c.hist[k].back());
  }
  s.iterations = it;
  s.converged = cv;
  s.breakdown = bk;
  s.final_residual = fr;
  s.t_pca = t_pca;
  s.t_assemble = t_asm;
  s.t_precond = t_pre;
  s.t_solve = t_sol;
  s.t_evaluate = t_ev;
}

}  // namespace rdd

using rdd::Ctx;

template <class F>
static int guarded(rdd_ctx* h, F&& f) {
  if (!h) return RDD_INVALID_ARGUMENT;
  struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(rdd::alloc_stream()) { rdd::alloc_stream() = s; }
    ~StreamScope() { rdd::alloc_stream() = prev; }
  } scope(h->c.stream);
  try {
    RDD_CUDA(cudaSetDevice(h->c.device));
    f(h->c);
    return RDD_OK;
  } catch (const rdd::CudaError& e) {
    h->c.err = e.what();
    return RDD_CUDA_ERROR;
  } catch (const std::invalid_argument& e) {
    h->c.err = e.what();
    return RDD_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    h->c.err = e.what();
    return RDD_DOMAIN_ERROR;
  } catch (const std::exception& e) {
    h->c.err = e.what();
    return RDD_RUNTIME_ERROR;
  }
}

static void need_assembled(const Ctx& c) {
  if (!c.assembled) throw std::invalid_argument("system not assembled");
}

extern "C" {

const char* rdd_version(void) { return "rdd 0.1 (sm_100a, FP64)"; }

int rdd_abi_sizes(int32_t* config_size, int32_t* summary_size) {
  if (config_size) *config_size = static_cast<int32_t>(sizeof(rdd_config));
  if (summary_size) *summary_size = static_cast<int32_t>(sizeof(rdd_summary));
  return RDD_OK;
}

int rdd_create(rdd_ctx** out, int device) {
  if (!out) return RDD_INVALID_ARGUMENT;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device || device < 0) return RDD_CUDA_ERROR;
  auto* h = new rdd_ctx();
  h->c.device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&h->c.stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaGetDeviceProperties(&h->c.prop, device) != cudaSuccess) {
    delete h;
    return RDD_CUDA_ERROR;
  }
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;  // keep freed blocks cached in the pool
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  *out = h;
  return RDD_OK;
}

void rdd_destroy(rdd_ctx* h) {
  if (!h) return;
  cudaSetDevice(h->c.device);
  cudaStreamSynchronize(h->c.stream);
  cudaStream_t s = h->c.stream;
  for (auto& e : h->c.ev)
    if (e) cudaEventDestroy(e);
  {
    const cudaStream_t prev = rdd::alloc_stream();
    rdd::alloc_stream() = s;
    delete h;
    rdd::alloc_stream() = prev;
  }
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
}
int rdd_set_verbose(rdd_ctx* h, int on) {
  if (!h) return RDD_INVALID_ARGUMENT;
  h->c.verbose = on != 0;
  return RDD_OK;
}

int rdd_set_param(rdd_ctx* h, const char* name, double value) {
  if (!h || !name) return RDD_INVALID_ARGUMENT;
  const std::string n(name);
  if (n == "full_rank_cond" && value >= 0.0) {
    h->c.full_rank_cond = value;
    return RDD_OK;
  }
  if (n == "pca_refine" && value >= 0.0 && value <= 4.0) {
    h->c.pca_refine = static_cast<int>(value);
    return RDD_OK;
  }
  if (n == "inv_max" && value >= 0.0 && value <= 1024.0) {
    h->c.inv_max = static_cast<int>(value);
    return RDD_OK;
  }
  if (n == "pca_stop" && value >= 0.0 && value < 1.0) {
    h->c.pca_stop = value;
    return RDD_OK;
  }
  h->c.err = "rdd_set_param: unknown parameter or bad value: " + n;
  return RDD_INVALID_ARGUMENT;
}

const char* rdd_last_error(const rdd_ctx* h) { return h ? h->c.err.c_str() : "null context"; }

int rdd_build_instance(rdd_ctx* h, const rdd_config* cfg, uint64_t seed) {
  return guarded(h, [&](Ctx& c) {
    if (!cfg) throw std::invalid_argument("null config");
    rdd::build_instance(c, *cfg, seed);
  });
}
int rdd_assemble(rdd_ctx* h, int equilibrate) {
  return guarded(h, [&](Ctx& c) { rdd::assemble(c, equilibrate != 0); });
}
int rdd_build_preconditioner(rdd_ctx* h, int kind) {
  return guarded(h, [&](Ctx& c) {
    need_assembled(c);
    if (kind >= 0) {
      auto idx = std::async(std::launch::async, [&c] { return rdd::prepare_schwarz_index(c); });
      rdd::build_normal_blocks(c);
      rdd::SchwarzIndex x = idx.get();
      rdd::build_schwarz(c, kind, &x);
    } else {
      rdd::build_normal_blocks(c);
      c.pkind = RDD_PRECOND_NONE;
    }
  });
}
int rdd_solve(rdd_ctx* h, int solver, double rel_tol, int max_iter, int gmres_restart) {
  return guarded(h, [&](Ctx& c) {
    need_assembled(c);
    if (solver == RDD_SOLVER_QR) rdd::qr_solve_dev(c);
    else rdd::solve_all(c, solver, rel_tol, max_iter, gmres_restart);
  });
}
int rdd_evaluate(rdd_ctx* h, const int* test_res) {
  return guarded(h, [&](Ctx& c) {
    if (!c.W.p) throw std::invalid_argument("evaluate: solve first");
    rdd::evaluate(c, test_res);
  });
}
int rdd_run_single(rdd_ctx* h, const rdd_config* cfg, uint64_t seed, rdd_summary* out) {
  const int st = guarded(h, [&](Ctx& c) {
    if (!cfg) throw std::invalid_argument("null config");
    rdd::run_single(c, *cfg, seed);
  });
  if (st == RDD_OK && out) *out = h->c.sum;
  return st;
}
int rdd_rerun_resident(rdd_ctx* h, rdd_summary* out) {
  const int st = guarded(h, [&](Ctx& c) {
    const rdd_config cfg = c.cfg;
    rdd::run_single(c, cfg, c.seed, true);
  });
  if (st == RDD_OK && out) *out = h->c.sum;
  return st;
}
int64_t rdd_launch_count(void) { return rdd::launch_counter(); }
int rdd_io_bytes(int64_t* h2d, int64_t* d2h) {
  if (h2d) *h2d = rdd::h2d_counter();
  if (d2h) *d2h = rdd::d2h_counter();
  return RDD_OK;
}
int rdd_event_record(rdd_ctx* h, int slot) {
  if (!h || slot < 0 || slot >= 8) return RDD_INVALID_ARGUMENT;
  Ctx& c = h->c;
  cudaSetDevice(c.device);
  if (!c.ev[slot] && cudaEventCreate(&c.ev[slot]) != cudaSuccess) return RDD_CUDA_ERROR;
  return cudaEventRecord(c.ev[slot], c.stream) == cudaSuccess ? RDD_OK : RDD_CUDA_ERROR;
}
int rdd_event_elapsed(rdd_ctx* h, int a, int b, double* ms) {
  if (!h || a < 0 || a >= 8 || b < 0 || b >= 8 || !ms) return RDD_INVALID_ARGUMENT;
  Ctx& c = h->c;
  if (!c.ev[a] || !c.ev[b]) return RDD_INVALID_ARGUMENT;
  if (cudaEventSynchronize(c.ev[b]) != cudaSuccess) return RDD_CUDA_ERROR;
  float f = 0.f;
  if (cudaEventElapsedTime(&f, c.ev[a], c.ev[b]) != cudaSuccess) return RDD_CUDA_ERROR;
  *ms = f;
  return RDD_OK;
}
int rdd_get_summary(rdd_ctx* h, rdd_summary* out) {
  if (!h || !out) return RDD_INVALID_ARGUMENT;
  *out = h->c.sum;
  return RDD_OK;
}

// ---- operators on host vectors
int rdd_matvec(rdd_ctx* h, const double* w, int64_t nw, double* y, int64_t ny) {
  return guarded(h, [&](Ctx& c) {
    need_assembled(c);
    if (nw != c.p) throw std::invalid_argument("matvec: coefficient vector has wrong length");  // assembly.hpp:111
    if (ny != c.N) throw std::invalid_argument("matvec: output vector has wrong length");
    rdd::DBuf<double> dw, dy;
    dw.upload(w, c.p, c.stream);
    dy.ensure(c.N);
    rdd::matvec_dev(c, dw.p, dy.p);
    dy.download(y, c.N, c.stream);
    RDD_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int rdd_matvec_transpose(rdd_ctx* h, const double* r, int64_t nr, double* out, int64_t nout) {
  return guarded(h, [&](Ctx& c) {
    need_assembled(c);
    if (nr != c.N) throw std::invalid_argument("matvec_transpose: residual vector has wrong length");  // :124
    if (nout != c.p) throw std::invalid_argument("matvec_transpose: output vector has wrong length");
    rdd::DBuf<double> dr, dout;
    dr.upload(r, c.N, c.stream);
    dout.ensure(c.p);
    rdd::matvec_t_dev(c, dr.p, dout.p);
    dout.download(out, c.p, c.stream);
    RDD_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int rdd_normal_apply(rdd_ctx* h, const double* w, int64_t nw, double* out, int64_t nout) {
  return guarded(h, [&](Ctx& c) {
    need_assembled(c);
    if (nw != c.p || nout != c.p) throw std::invalid_argument("matvec: coefficient vector has wrong length");
    rdd::DBuf<double> dw, dout;
    dw.upload(w, c.p, c.stream);
    dout.ensure(c.p);
    rdd::normal_operator(c, dw.p, dout.p);
    dout.download(out, c.p, c.stream);
    RDD_CUDA(cudaStreamSynchronize(c.stream));
  });
}
int rdd_precond_apply(rdd_ctx* h, const double* v, int64_t nv, double* z, int64_t nz, int transpose) {
  return guarded(h, [&](Ctx& c) {
    if (c.pkind < 0) throw std::invalid_argument("no preconditioner built");
    if (nv != c.p || nz != c.p)
      throw std::invalid_argument("preconditioner apply: wrong vector length");  // schwarz.hpp:154/190
    rdd::DBuf<double> dv, dz;
    dv.upload(v, c.p, c.stream);
    dz.ensure(c.p);
    rdd::precond_apply_dev(c, dv.p, dz.p, transpose != 0);
    dz.download(z, c.p, c.stream);
    RDD_CUDA(cudaStreamSynchronize(c.stream));
  });
}


// ---- caller inputs (the reference's objects instead of a RunConfig)
int rdd_set_decomposition(rdd_ctx* h, int dim, const int32_t* counts, const double* domain_lo, const double* domain_hi,
                          const double* box_lo, const double* box_hi, const double* center, const double* half,
                          const int32_t* nbr_ptr, const int32_t* nbr_idx) {
  return guarded(h, [&](Ctx& c) {
    if (dim < 1 || dim > rdd::kMaxDim) throw std::invalid_argument("decomposition dimension must be 1..4");
    if (!counts || !domain_lo || !domain_hi || !box_lo || !box_hi || !center || !half || !nbr_ptr || !nbr_idx)
      throw std::invalid_argument("decomposition: null array");
    rdd::CustomInputs& u = c.custom;
    u.d = dim;
    u.counts.assign(counts, counts + dim);
    long long J = 1;
    for (int k : u.counts) {
      if (k < 1) throw std::invalid_argument("per-axis subdomain counts must be >= 1");
      J *= k;
    }
    if (J > (1 << 24)) throw std::invalid_argument("decomposition: too many subdomains");
    u.dom_lo.assign(domain_lo, domain_lo + dim);
    u.dom_hi.assign(domain_hi, domain_hi + dim);
    const size_t n = static_cast<size_t>(J) * dim;
    u.lo.assign(box_lo, box_lo + n);
    u.hi.assign(box_hi, box_hi + n);
    u.ctr.assign(center, center + n);
    u.half.assign(half, half + n);
    u.nbr_ptr.assign(nbr_ptr, nbr_ptr + J + 1);
    if (u.nbr_ptr[0] != 0) throw std::invalid_argument("decomposition: neighbour CSR must start at 0");
    u.nbr_idx.assign(nbr_idx, nbr_idx + u.nbr_ptr[J]);
    for (int v : u.nbr_idx)
      if (v < 0 || v >= J) throw std::invalid_argument("decomposition: neighbour index out of range");
    u.has_dec = true;
  });
}
int rdd_set_points(rdd_ctx* h, int64_t N, const double* pts) {
  return guarded(h, [&](Ctx& c) {
    rdd::CustomInputs& u = c.custom;
    if (!u.has_dec) throw std::invalid_argument("points: set the decomposition first");
    if (N < 1 || !pts) throw std::invalid_argument("points: empty point set");
    u.pts.assign(pts, pts + static_cast<size_t>(N) * u.d);
    u.has_pts = true;
  });
}
int rdd_set_bases(rdd_ctx* h, int J, int m, const double* R, const double* b, int activation) {
  return guarded(h, [&](Ctx& c) {
    rdd::CustomInputs& u = c.custom;
    if (!u.has_dec) throw std::invalid_argument("bases: set the decomposition first");
    if (m < 1) throw std::invalid_argument("hidden width m must be >= 1");
    if (activation != 0 && activation != 1) throw std::invalid_argument("activation must be tanh (0) or sin (1)");
    if (!R || !b || J < 1) throw std::invalid_argument("bases: null array");
    u.m = m;
    u.act = activation;
    u.R.assign(R, R + static_cast<size_t>(J) * m * u.d);
    u.b.assign(b, b + static_cast<size_t>(J) * m);
    u.has_bases = true;
  });
}
int rdd_set_problem(rdd_ctx* h, int C, const double* op_coef, const double* L_jets, const double* F) {
  return guarded(h, [&](Ctx& c) {
    rdd::CustomInputs& u = c.custom;
    if (!u.has_pts) throw std::invalid_argument("problem: set the points first");
    if (C < 1 || C > 3) throw std::invalid_argument("problem: 1..3 solution components");
    if (!op_coef || !L_jets || !F) throw std::invalid_argument("problem: null array");
    const size_t N = u.pts.size() / u.d, jl = rdd::jet_len(u.d);
    u.C = C;
    u.coef.assign(op_coef, op_coef + jl);
    u.Ljet.assign(L_jets, L_jets + N * jl);
    u.F.assign(F, F + N * C);
    u.has_problem = true;
  });
}
int rdd_build_custom(rdd_ctx* h, const rdd_config* cfg) {
  return guarded(h, [&](Ctx& c) {
    if (!cfg) throw std::invalid_argument("null config");
    rdd::build_custom(c, *cfg);
  });
}
int rdd_evaluate_at(rdd_ctx* h, int64_t M, const double* pts, const double* W, const double* L_vals,
                    const double* G_vals, double* u_out) {
  return guarded(h, [&](Ctx& c) {
    if (M > 0 && (!pts || !L_vals || !u_out)) throw std::invalid_argument("evaluate_solution: null array");
    rdd::evaluate_at(c, M, pts, W, L_vals, G_vals, u_out);
  });
}

// ---- exports
int64_t rdd_get_i(rdd_ctx* h, const char* what, int index, int32_t* out, int64_t cap) {
  if (!h || !what) return -1;
  Ctx& c = h->c;
  std::vector<int> v;
  try {
    const std::string w(what);
    if (w == "J") v = {c.J};
    else if (w == "N") v = {c.N};
    else if (w == "p") v = {c.p};
    else if (w == "dim") v = {c.d};
    else if (w == "C") v = {c.C};
    else if (w == "maxcov") v = {c.maxcov};
    else if (w == "n_fallback") v = {c.n_fallback};
    else if (w == "qr_rank") v = {c.qr_rank};
    else if (w == "inv_mode") v = {c.inv_mode ? 1 : 0};
    else if (w == "env_first") {  // first stored tile of every block row of subdomain `index`'s factor
      v.assign(c.env_first.begin() + c.env_off.at(index), c.env_first.begin() + c.env_off.at(index + 1));
    }
    else if (w == "p_j") v = c.h_p;
    else if (w == "col_off") v = c.h_col_off;
    else if (w == "rows") {
      const int n = c.h_row_ptr.at(index + 1) - c.h_row_ptr.at(index);
      v.resize(n);
      if (n) RDD_CUDA(cudaMemcpy(v.data(), c.row_idx.p + c.h_row_ptr[index], sizeof(int) * n, cudaMemcpyDeviceToHost));
    } else if (w == "nbr") v.assign(c.nbr_idx.begin() + c.nbr_ptr.at(index), c.nbr_idx.begin() + c.nbr_ptr.at(index + 1));
    else if (w == "nb_pairs") {
      for (size_t k = 0; k < c.nb_j1.size(); ++k) {
        v.push_back(c.nb_j1[k]);
        v.push_back(c.nb_j2[k]);
      }
    } else if (w == "local_rank") v = c.local_rank;
    else if (w == "local_n") v = c.local_n;
    else if (w == "row_ptr") v = c.h_row_ptr;
    else if (w == "set") v.assign(c.set_idx.begin() + c.set_ptr.at(index), c.set_idx.begin() + c.set_ptr.at(index + 1));
    else if (w == "owner") v = c.h_owner;
    else if (w == "mult") v = c.h_mult;
    else if (w == "iterations") v = c.iters;
    else if (w == "converged") v = c.conv;
    else {
      c.err = "unknown export " + w;
      return -1;
    }
  } catch (const std::exception& e) {
    c.err = e.what();
    return -1;
  }
  const int64_t n = static_cast<int64_t>(v.size());
  if (out) std::copy(v.begin(), v.begin() + std::min(n, cap), out);
  return n;
}

int64_t rdd_get_d(rdd_ctx* h, const char* what, int index, double* out, int64_t cap) {
  if (!h || !what) return -1;
  Ctx& c = h->c;
  std::vector<double> v;
  auto dl = [&](const double* src, size_t n) {
    v.resize(n);
    if (n) RDD_CUDA(cudaMemcpy(v.data(), src, sizeof(double) * n, cudaMemcpyDeviceToHost));
  };
  try {
    const std::string w(what);
    const int rows = (index >= 0 && index + 1 < static_cast<int>(c.h_row_ptr.size()))
                         ? c.h_row_ptr[index + 1] - c.h_row_ptr[index] : 0;
    if (w == "points") {
      for (int i = 0; i < c.N; ++i)
        for (int a = 0; a < c.d; ++a) v.push_back(c.h_pts[static_cast<size_t>(a) * c.N + i]);
    } else if (w == "box_lo" || w == "box_hi") {
      const auto& src = w == "box_lo" ? c.box_lo : c.box_hi;
      for (int j = 0; j < c.J; ++j)
        for (int a = 0; a < c.d; ++a) v.push_back(src[j * 4 + a]);
    } else if (w == "R") {  // m x d column-major (the oracle's layout)
      v.resize(static_cast<size_t>(c.m) * c.d);
      for (int k = 0; k < c.m; ++k)
        for (int a = 0; a < c.d; ++a) v[k + a * c.m] = c.h_R[(static_cast<size_t>(index) * c.m + k) * c.d + a];
    } else if (w == "b") {
      v.assign(c.h_b.begin() + static_cast<size_t>(index) * c.m, c.h_b.begin() + static_cast<size_t>(index + 1) * c.m);
    } else if (w == "S") {
      dl(c.S.p + c.S_off.at(index), static_cast<size_t>(rows) * c.m);
    } else if (w == "sigma") {
      if (c.identity_V) throw std::invalid_argument("no PCA");
      dl(c.sigma.p + static_cast<size_t>(index) * c.m, std::min(rows, c.m));
    } else if (w == "V") {
      if (c.identity_V) throw std::invalid_argument("no PCA");
      dl(c.Vred.p + static_cast<size_t>(index) * c.m * c.m, static_cast<size_t>(c.m) * c.h_p.at(index));
    } else if (w == "H") {
      need_assembled(c);
      dl(c.H + c.H_off.at(index), static_cast<size_t>(rows) * c.h_p.at(index));
    } else if (w == "F") {
      dl(c.F.p ? c.F.p : c.Fpt.p, static_cast<size_t>(c.N) * c.C);
    } else if (w == "scales") {
      dl(c.scales.p, c.p);
    } else if (w == "nb") {
      const size_t k = static_cast<size_t>(index);
      dl(c.NB.p + c.nb_off.at(k), static_cast<size_t>(c.nb_off.at(k + 1) - c.nb_off[k]));
    } else if (w == "nb_dense") {
      v.assign(static_cast<size_t>(c.p) * c.p, 0.0);
      std::vector<double> blk;
      for (size_t k = 0; k < c.nb_j1.size(); ++k) {
        const int j1 = c.nb_j1[k], j2 = c.nb_j2[k], p1 = c.h_p[j1], p2 = c.h_p[j2];
        blk.resize(static_cast<size_t>(p1) * p2);
        RDD_CUDA(cudaMemcpy(blk.data(), c.NB.p + c.nb_off[k], sizeof(double) * blk.size(), cudaMemcpyDeviceToHost));
        for (int cc = 0; cc < p2; ++cc)
          for (int r = 0; r < p1; ++r) {
            const size_t a = c.h_col_off[j1] + r, b = c.h_col_off[j2] + cc;
            v[a + b * c.p] = blk[r + static_cast<size_t>(cc) * p1];
            if (j1 != j2) v[b + a * c.p] = blk[r + static_cast<size_t>(cc) * p1];
          }
      }
    } else if (w == "H_dense") {
      need_assembled(c);
      v.assign(static_cast<size_t>(c.N) * c.p, 0.0);
      std::vector<double> blk;
      std::vector<int> ridx;
      for (int j = 0; j < c.J; ++j) {
        const int nr = c.h_row_ptr[j + 1] - c.h_row_ptr[j], pj = c.h_p[j];
        blk.resize(static_cast<size_t>(nr) * pj);
        ridx.resize(nr);
        if (nr == 0) continue;
        RDD_CUDA(cudaMemcpy(blk.data(), c.H + c.H_off[j], sizeof(double) * blk.size(), cudaMemcpyDeviceToHost));
        RDD_CUDA(cudaMemcpy(ridx.data(), c.row_idx.p + c.h_row_ptr[j], sizeof(int) * nr, cudaMemcpyDeviceToHost));
        for (int cc = 0; cc < pj; ++cc)
          for (int r = 0; r < nr; ++r)
            v[ridx[r] + static_cast<size_t>(c.h_col_off[j] + cc) * c.N] = blk[r + static_cast<size_t>(cc) * nr];
      }
    } else if (w == "local_cond") {
      {
        const cudaStream_t prev = rdd::alloc_stream();
        rdd::alloc_stream() = c.stream;
        rdd::refresh_local_cond(c);
        rdd::alloc_stream() = prev;
      }
      v = c.local_cond;
    } else if (w == "W") {
      dl(c.W.p + static_cast<size_t>(index) * c.p, c.p);
    } else if (w == "hist") {
      v = c.hist.at(index);
    } else if (w == "true_hist") {
      v = c.true_hist.at(index);
    } else if (w == "approx") {
      v = c.approx;
    } else if (w == "exact") {
      v = c.exact;
    } else {
      c.err = "unknown export " + w;
      return -1;
    }
  } catch (const std::exception& e) {
    c.err = e.what();
    return -1;
  }
  const int64_t n = static_cast<int64_t>(v.size());
  if (out) std::copy(v.begin(), v.begin() + std::min(n, cap), out);
  return n;
}

// ---- instrumentation
int rdd_kernel_stats(rdd_ctx* h, const char* family, double* ms_total, int64_t* launches) {
  if (!h || !family) return RDD_INVALID_ARGUMENT;
  auto it = h->c.stats.find(family);
  if (ms_total) *ms_total = it == h->c.stats.end() ? 0.0 : it->second.ms;
  if (launches) *launches = it == h->c.stats.end() ? 0 : it->second.launches;
  return RDD_OK;
}
int rdd_reset_stats(rdd_ctx* h) {
  if (!h) return RDD_INVALID_ARGUMENT;
  h->c.stats.clear();
  return RDD_OK;
}
int rdd_set_timing(rdd_ctx* h, int on) {
  if (!h) return RDD_INVALID_ARGUMENT;
  h->c.timing = on != 0;
  return RDD_OK;
}

int rdd_bench_operator(rdd_ctx* h, int op_form, int reps, double* ms_per_call, double* bytes_per_call) {
  return guarded(h, [&](Ctx& c) {
    need_assembled(c);
    if (op_form == RDD_OPERATOR_NORMAL && !c.NB.p) rdd::build_normal_blocks(c);
    if (op_form != RDD_OPERATOR_TWO_PASS && op_form != RDD_OPERATOR_NORMAL)
      throw std::invalid_argument("unknown normal-operator form");
    rdd::DBuf<double> w, out;
    w.ensure(c.p);
    out.ensure(c.p);
    RDD_CUDA(cudaMemsetAsync(w.p, 0, sizeof(double) * c.p, c.stream));
    c.ytmp.ensure(c.N);
    const int saved = c.cfg.op_form;
    c.cfg.op_form = op_form;
    for (int i = 0; i < 3; ++i) rdd::normal_operator(c, w.p, out.p);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, c.stream);
    for (int i = 0; i < reps; ++i) rdd::normal_operator(c, w.p, out.p);
    cudaEventRecord(e1, c.stream);
    RDD_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    c.cfg.op_form = saved;
    *ms_per_call = ms / reps;
    if (op_form == RDD_OPERATOR_NORMAL)
      *bytes_per_call = 8.0 * static_cast<double>(c.nb_off.back()) + 8.0 * 2 * c.p;
    else  // two passes over H + vectors + row maps
      *bytes_per_call = 2.0 * (8.0 * static_cast<double>(c.H_off[c.J]) + 8.0 * (c.p + c.N) + 4.0 * c.sum_rows);
  });
}

int rdd_bench_precond(rdd_ctx* h, int transpose, int reps, double* ms_per_call, double* bytes_per_call) {
  return guarded(h, [&](Ctx& c) {
    if (c.pkind < 0) throw std::invalid_argument("no preconditioner built");
    rdd::DBuf<double> v, z;
    v.ensure(c.p);
    z.ensure(c.p);
    RDD_CUDA(cudaMemsetAsync(v.p, 0, sizeof(double) * c.p, c.stream));
    for (int i = 0; i < 3; ++i) rdd::precond_apply_dev(c, v.p, z.p, transpose != 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, c.stream);
    for (int i = 0; i < reps; ++i) rdd::precond_apply_dev(c, v.p, z.p, transpose != 0);
    cudaEventRecord(e1, c.stream);
    RDD_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_per_call = ms / reps;
    // algorithmic bytes: per subdomain the local operator (lower triangle incl. diagonal, read
    // twice by the forward and backward solves; once as an explicit inverse; the dense n_i x n_i
    // pseudo-inverse once on eigen-fallback blocks), the gathered v[S_i] and the written z_i
    // with their 4-byte indices, then the reduction (z read through the gather map, out written)
    double b = 0.0;
    const int J = static_cast<int>(c.set_ptr.size()) - 1;
    if (c.ras_panel) {  // RAS owner-row panels: p_i x n_i per subdomain, read once
      b = 8.0 * static_cast<double>(c.ras_off[J]) + 12.0 * static_cast<double>(c.set_idx.size()) +
          8.0 * static_cast<double>(c.set_idx.size()) + 4.0 * static_cast<double>(c.p) + 8.0 * c.p;
      *bytes_per_call = b;
      return;
    }
    for (int i = 0; i < J; ++i) {
      const double n = c.set_ptr[i + 1] - c.set_ptr[i];
      const bool dense = std::binary_search(c.fallback.begin(), c.fallback.end(), i);
      const double tri = n * (n + 1) / 2.0;
      b += 8.0 * (dense ? n * n : (c.inv_mode ? tri : 0.0));
      b += 8.0 * 2.0 * n + 4.0 * n;
    }
    // factor mode: the entries inside the envelopes of the lower triangles (structural zeros left of
    // a row's first nonzero block are not stored), read by the forward and the backward solve; the
    // few eigen-fallback blocks are counted dense above and not subtracted here
    if (!c.inv_mode) b += 2.0 * 8.0 * c.env_entries;
    b += 8.0 * static_cast<double>(c.set_idx.size()) + 4.0 * static_cast<double>(c.set_idx.size()) + 8.0 * c.p;
    *bytes_per_call = b;
  });
}

int rdd_bench_gemm(rdd_ctx* h, int mode, int M, int N, int K, int batch, int reps, double* ms_out) {
  return guarded(h, [&](Ctx& c) {
    // mode + 10: the 80 x 80 CTA tile; mode + 20: the 64 x 80 tile (NN and TN)
    const int tile = mode >= 20 ? 6480 : (mode >= 10 ? 80 : 64);
    const int tile_m = tile == 6480 ? 64 : tile, tile_n = tile == 6480 ? 80 : tile;
    mode %= 10;
    if (M < 1 || N < 1 || K < 1 || batch < 1 || reps < 1 || mode < 0 || mode > 2 || (tile != 64 && mode == 2))
      throw std::invalid_argument("bench_gemm: bad shape");
    const size_t sa = static_cast<size_t>(M) * K, sb = static_cast<size_t>(K) * N, sc = static_cast<size_t>(M) * N;
    rdd::DBuf<double> A, B, Cm;
    A.ensure(sa * batch);
    B.ensure(sb * batch);
    Cm.ensure(sc * batch);
    RDD_CUDA(cudaMemsetAsync(A.p, 0, sizeof(double) * sa * batch, c.stream));
    RDD_CUDA(cudaMemsetAsync(B.p, 0, sizeof(double) * sb * batch, c.stream));
    std::vector<rdd::GemmTask> tasks;
    for (int b = 0; b < batch; ++b)
      for (int tm = 0; tm < (M + tile_m - 1) / tile_m; ++tm)
        for (int tn = 0; tn < (N + tile_n - 1) / tile_n; ++tn) {
          rdd::GemmTask t{};
          t.A = A.p + sa * b;
          t.B = B.p + sb * b;
          t.Cm = Cm.p + sc * b;
          t.M = M;
          t.N = N;
          t.K = K;
          t.lda = mode == 1 ? K : M;
          t.ldb = mode == 2 ? N : K;
          t.ldc = M;
          t.tm = tm;
          t.tn = tn;
          t.beta = 0.0;
          t.alpha = 1.0;
          tasks.push_back(t);
        }
    auto run = [&] {
      if (mode == 0) rdd::gemm_nn(c, tasks, tile);
      else if (mode == 1) rdd::gemm_tn(c, tasks, tile);
      else rdd::gemm_nt(c, tasks);
    };
    run();
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, c.stream);
    for (int r = 0; r < reps; ++r) run();
    cudaEventRecord(e1, c.stream);
    RDD_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_out = ms / reps;
  });
}

// ---- dense diagnostics (krylov.hpp:403-440, runner.hpp:344-400)
static int diag_cap(int cap) { return cap <= 0 ? 4000 : cap; }  // krylov.hpp:404 kDenseSpectrumCap

int rdd_spectra(rdd_ctx* h, int cap, double* normal_re, double* normal_im, double* precond_re, double* precond_im,
                double* cond_normal, double* cond_precond) {
  return guarded(h, [&](Ctx& c) {
    need_assembled(c);
    const bool want_pre = precond_re || precond_im || cond_precond;
    if (want_pre && c.pkind < 0) throw std::invalid_argument("no preconditioner built");
    std::vector<double> nre, nim, pre, pim;
    double cn = 0.0, cp = 0.0;
    rdd::spectra(c, diag_cap(cap), nre, nim, want_pre ? &pre : nullptr, want_pre ? &pim : nullptr,
                 cond_normal ? &cn : nullptr, cond_precond ? &cp : nullptr);
    if (normal_re) std::copy(nre.begin(), nre.end(), normal_re);
    if (normal_im) std::copy(nim.begin(), nim.end(), normal_im);
    if (precond_re) std::copy(pre.begin(), pre.end(), precond_re);
    if (precond_im) std::copy(pim.begin(), pim.end(), precond_im);
    if (cond_normal) *cond_normal = cn;
    if (cond_precond) *cond_precond = cp;
  });
}

// host matrix -> device (transposed when wide, so the reductions see rows >= cols)
static double* upload_dense(Ctx& c, int64_t rows, int64_t cols, const double* A, bool allow_transpose, int& m, int& n) {
  if (rows < 0 || cols < 0 || (rows * cols > 0 && !A)) throw std::invalid_argument("dense diagnostics: bad matrix");
  m = static_cast<int>(rows);
  n = static_cast<int>(cols);
  const size_t nn = static_cast<size_t>(rows) * cols;
  double* d = c.ws("dg_in", nn);
  if (allow_transpose && rows < cols) {
    std::vector<double> t(nn);
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t i = 0; i < rows; ++i) t[j + i * cols] = A[i + j * rows];
    RDD_CUDA(cudaMemcpyAsync(d, t.data(), sizeof(double) * nn, cudaMemcpyHostToDevice, c.stream));
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    std::swap(m, n);
  } else if (nn) {
    RDD_CUDA(cudaMemcpyAsync(d, A, sizeof(double) * nn, cudaMemcpyHostToDevice, c.stream));
  }
  rdd::h2d_counter() += static_cast<int64_t>(nn * sizeof(double));
  return d;
}

int rdd_dense_spectrum(rdd_ctx* h, int64_t rows, int64_t cols, const double* A, int cap, double* wr, double* wi) {
  return guarded(h, [&](Ctx& c) {
    if (rows != cols) throw std::invalid_argument("spectrum: matrix must be square");  // krylov.hpp:414
    rdd::check_dense_cap(rows, diag_cap(cap));
    int m = 0, n = 0;
    double* d = upload_dense(c, rows, cols, A, false, m, n);
    std::vector<double> re, im;
    rdd::dense_eigenvalues_dev(c, d, n, re, im);
    if (wr) std::copy(re.begin(), re.end(), wr);
    if (wi) std::copy(im.begin(), im.end(), wi);
  });
}

int rdd_dense_singular_values(rdd_ctx* h, int64_t rows, int64_t cols, const double* A, int cap, double* s) {
  return guarded(h, [&](Ctx& c) {
    rdd::check_dense_cap(std::min(rows, cols), diag_cap(cap));  // krylov.hpp:424
    int m = 0, n = 0;
    double* d = upload_dense(c, rows, cols, A, true, m, n);
    std::vector<double> sv;
    rdd::singular_values_dev(c, d, m, n, sv);
    if (s) std::copy(sv.begin(), sv.end(), s);
  });
}

int rdd_dense_condition_number(rdd_ctx* h, int64_t rows, int64_t cols, const double* A, int cap, double* cond) {
  return guarded(h, [&](Ctx& c) {
    rdd::check_dense_cap(std::min(rows, cols), diag_cap(cap));
    int m = 0, n = 0;
    double* d = upload_dense(c, rows, cols, A, true, m, n);
    std::vector<double> sv;
    rdd::singular_values_dev(c, d, m, n, sv);
    const double k = rdd::condition_from(sv);
    if (cond) *cond = k;
  });
}

int rdd_bench_jacobi(rdd_ctx* h, int n, int batch, int sweeps, double* ms) {
  return guarded(h, [&](Ctx& c) {
    if (n < 2 || batch < 1 || sweeps < 1) throw std::invalid_argument("bench_jacobi: n >= 2, batch >= 1, sweeps >= 1");
    *ms = rdd::bench_syevj(c, n, batch, sweeps);
  });
}

}  // extern "C"
