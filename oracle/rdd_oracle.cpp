// rdd_oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// CPU oracle for the B200 solve pipeline: a plain C++ restatement of the reference
// rannddm pipeline (runner.hpp:202-275 run_single and everything it calls), used by
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/--impl reference legs as the
// checker. The product (paper_2412_19207_b200/librdd.so) never links or calls this file.
//
// Eigen is not installed here, so the reference cannot be compiled as-is.
// Dense decompositions that the reference takes from Eigen are taken from LAPACK in scipy's
// bundled OpenBLAS, loaded with dlopen at orc_create():
//   Eigen::JacobiSVD            (reduction.hpp:91)  -> dgeqp3 preconditioner + dgesvj on R (Eigen's QR-preconditioned form)
//   SelfAdjointEigenSolver      (schwarz.hpp:131)   -> dsyevd (ascending, as Eigen)
//   ColPivHouseholderQR         (krylov.hpp:100)    -> dgeqp3 + dormqr + back substitution
//   EigenSolver / BDCSVD        (krylov.hpp:416/425)-> dgeev / dgesvd (diagnostics only)
// Everything else (geometry, jets, windows, assembly, normal blocks, Schwarz, CG, GMRES,
// evaluation, errors) is restated with the reference's operation order.
#include <dlfcn.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "../include/rdd.h"
#include "oracle_core.hpp"

namespace orc {

// ---------------------------------------------------------------- LAPACK (scipy-openblas)
struct Lapack {
  using gesvj_t = void (*)(const char*, const char*, const char*, const int*, const int*, double*, const int*,
                           double*, const int*, double*, const int*, double*, const int*, int*, size_t, size_t,
                           size_t);
  using syevd_t = void (*)(const char*, const char*, const int*, double*, const int*, double*, double*,
                           const int*, int*, const int*, int*, size_t, size_t);
  using geqp3_t = void (*)(const int*, const int*, double*, const int*, int*, double*, double*, const int*, int*);
  using ormqr_t = void (*)(const char*, const char*, const int*, const int*, const int*, const double*, const int*,
                           const double*, double*, const int*, double*, const int*, int*, size_t, size_t);
  using gesvd_t = void (*)(const char*, const char*, const int*, const int*, double*, const int*, double*, double*,
                           const int*, double*, const int*, double*, const int*, int*, size_t, size_t);
  using geev_t = void (*)(const char*, const char*, const int*, double*, const int*, double*, double*, double*,
                          const int*, double*, const int*, double*, const int*, int*, size_t, size_t);
  using threads_t = void (*)(int);
  void* h = nullptr;
  gesvj_t gesvj = nullptr;
  syevd_t syevd = nullptr;
  geqp3_t geqp3 = nullptr;
  ormqr_t ormqr = nullptr;
  gesvd_t gesvd = nullptr;
  geev_t geev = nullptr;
  threads_t set_threads = nullptr;
};

static Lapack g_lapack;

static void load_lapack(const char* path) {
  if (g_lapack.h) return;
  if (!path || !*path) throw std::runtime_error("oracle: LAPACK library path not given");
  g_lapack.h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!g_lapack.h) throw std::runtime_error(std::string("oracle: dlopen failed: ") + dlerror());
  auto sym = [](const char* n) {
    void* p = dlsym(g_lapack.h, n);
    if (!p) throw std::runtime_error(std::string("oracle: missing LAPACK symbol ") + n);
    return p;
  };
  g_lapack.gesvj = reinterpret_cast<Lapack::gesvj_t>(sym("scipy_dgesvj_"));
  g_lapack.syevd = reinterpret_cast<Lapack::syevd_t>(sym("scipy_dsyevd_"));
  g_lapack.geqp3 = reinterpret_cast<Lapack::geqp3_t>(sym("scipy_dgeqp3_"));
  g_lapack.ormqr = reinterpret_cast<Lapack::ormqr_t>(sym("scipy_dormqr_"));
  g_lapack.gesvd = reinterpret_cast<Lapack::gesvd_t>(sym("scipy_dgesvd_"));
  g_lapack.geev = reinterpret_cast<Lapack::geev_t>(sym("scipy_dgeev_"));
  g_lapack.set_threads = reinterpret_cast<Lapack::threads_t>(dlsym(g_lapack.h, "scipy_openblas_set_num_threads"));
  // Eigen's decompositions are single-threaded inside the reference's serial loops.
  if (g_lapack.set_threads) g_lapack.set_threads(1);
}

// ---------------------------------------------------------------- dense column-major matrix
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rr, int cc) : r(rr), c(cc), a(static_cast<size_t>(rr) * cc, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(j) * r + i]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(j) * r + i]; }
  double* col(int j) { return a.data() + static_cast<size_t>(j) * r; }
  const double* col(int j) const { return a.data() + static_cast<size_t>(j) * r; }
};
using Vec = std::vector<double>;

static double dot(const Vec& x, const Vec& y) {
  double s = 0.0;
  for (size_t i = 0; i < x.size(); ++i) s += x[i] * y[i];
  return s;
}
static double norm(const Vec& x) { return std::sqrt(dot(x, x)); }

// ---------------------------------------------------------------- decomposition (geometry.hpp:84-185)
struct Decomposition {
  Box domain;
  std::vector<int> counts;
  std::vector<Box> sub;
  std::vector<Point> centers, half;
  std::vector<std::vector<int>> nbr;
  int size() const { return static_cast<int>(sub.size()); }
  int dim() const { return domain.dim; }
};

static bool interiors_intersect(const Box& a, const Box& b) {  // geometry.hpp:99-105
  for (int ax = 0; ax < a.dim; ++ax)
    if (!(std::max(a.lo[ax], b.lo[ax]) < std::min(a.hi[ax], b.hi[ax]))) return false;
  return true;
}

static void finish_decomposition(Decomposition& dec, const std::vector<std::vector<double>>& axis_centers,
                                 const std::vector<double>& axis_half) {
  const int d = dec.dim();
  int total = 1;
  for (int c : dec.counts) total *= c;
  std::vector<int> idx(d, 0);
  for (int flat = 0; flat < total; ++flat) {  // axis 0 slowest (geometry.hpp:146-167)
    Box s;
    s.dim = d;
    Point c{}, h{};
    for (int a = 0; a < d; ++a) {
      c[a] = axis_centers[a][idx[a]];
      h[a] = axis_half[a];
      s.lo[a] = c[a] - h[a];
      s.hi[a] = c[a] + h[a];
    }
    dec.sub.push_back(s);
    dec.centers.push_back(c);
    dec.half.push_back(h);
    for (int a = d - 1; a >= 0; --a) {
      if (++idx[a] < dec.counts[a]) break;
      idx[a] = 0;
    }
  }
  dec.nbr.assign(total, {});
  for (int i = 0; i < total; ++i)
    for (int j = 0; j < total; ++j)
      if (interiors_intersect(dec.sub[i], dec.sub[j])) dec.nbr[i].push_back(j);
}

// geometry.hpp:109-177
static Decomposition build_decomposition(const Box& domain, const std::vector<int>& counts, double delta) {
  if (static_cast<int>(counts.size()) != domain.dim)
    throw std::invalid_argument("per-axis counts must match the domain dimension");
  if (!(delta > 1.0)) throw std::invalid_argument("overlap ratio delta must exceed 1");
  for (int c : counts)
    if (c < 1) throw std::invalid_argument("per-axis subdomain counts must be >= 1");
  const int d = domain.dim;
  Decomposition dec;
  dec.domain = domain;
  dec.counts = counts;
  std::vector<std::vector<double>> ac(d);
  std::vector<double> ah(d);
  for (int a = 0; a < d; ++a) {
    const int l = counts[a];
    const double lo = domain.lo[a], len = domain.width(a);
    if (l == 1) {
      ac[a] = {lo + 0.5 * len};
      ah[a] = 0.5 * len;
    } else {
      ah[a] = (delta / 2.0) / static_cast<double>(l - 1) * len;
      for (int j = 0; j < l; ++j) ac[a].push_back(lo + static_cast<double>(j) / static_cast<double>(l - 1) * len);
    }
  }
  finish_decomposition(dec, ac, ah);
  return dec;
}

// BASELINE layout: cell-centred boxes, each extended by `ext` x its width per side.
static Decomposition build_cell_decomposition(const Box& domain, const std::vector<int>& counts, double ext) {
  if (static_cast<int>(counts.size()) != domain.dim)
    throw std::invalid_argument("per-axis counts must match the domain dimension");
  if (!(ext > 0.0)) throw std::invalid_argument("cell decomposition extension must be positive");
  for (int c : counts)
    if (c < 1) throw std::invalid_argument("per-axis subdomain counts must be >= 1");
  const int d = domain.dim;
  Decomposition dec;
  dec.domain = domain;
  dec.counts = counts;
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
  finish_decomposition(dec, ac, ah);
  return dec;
}

// geometry.hpp:200-232 (cell-centred, last axis fastest) + optional edge points (2-D, §8d C1)
static std::vector<Point> uniform_grid(const Box& domain, const std::vector<int>& res, int boundary_per_edge = 0) {
  if (static_cast<int>(res.size()) != domain.dim)
    throw std::invalid_argument("per-axis resolutions must match the domain dimension");
  for (int r : res)
    if (r < 1) throw std::invalid_argument("grid resolutions must be >= 1");
  const int d = domain.dim;
  long long total = 1;
  for (int r : res) total *= r;
  std::vector<Point> pts;
  pts.reserve(static_cast<size_t>(total));
  std::vector<int> idx(d, 0);
  for (long long flat = 0; flat < total; ++flat) {
    Point p{};
    for (int a = 0; a < d; ++a) {
      const double step = domain.width(a) / static_cast<double>(res[a]);
      p[a] = domain.lo[a] + (static_cast<double>(idx[a]) + 0.5) * step;
    }
    pts.push_back(p);
    for (int a = d - 1; a >= 0; --a) {
      if (++idx[a] < res[a]) break;
      idx[a] = 0;
    }
  }
  if (boundary_per_edge > 0) {
    if (d != 2) throw std::invalid_argument("boundary points are defined for 2-D domains only");
    const int nb = boundary_per_edge;
    // edges in order: y=lo, y=hi (x varies), x=lo, x=hi (y varies); cell-centred along the edge
    for (int e = 0; e < 4; ++e) {
      const int axis = e < 2 ? 0 : 1;        // varying axis
      const int fixed = 1 - axis;
      const double fv = (e % 2 == 0) ? domain.lo[fixed] : domain.hi[fixed];
      const double step = domain.width(axis) / static_cast<double>(nb);
      for (int k = 0; k < nb; ++k) {
        Point p{};
        p[axis] = domain.lo[axis] + (static_cast<double>(k) + 0.5) * step;
        p[fixed] = fv;
        pts.push_back(p);
      }
    }
  }
  return pts;
}

// ---------------------------------------------------------------- basis (basis.hpp:24-105)
struct Basis {
  int m = 0, dim = 0, act = 0;
  Mat R;  // m x d
  Vec b;  // m
};
static Basis make_random_basis(uint64_t seed, int m, int dim, int act) {
  if (m < 1) throw std::invalid_argument("hidden width m must be >= 1");
  Basis B;
  B.m = m;
  B.dim = dim;
  B.act = act;
  B.R = Mat(m, dim);
  B.b.assign(m, 0.0);
  SplitMix64 rng(seed);
  for (int k = 0; k < m; ++k)
    for (int a = 0; a < dim; ++a) B.R(k, a) = rng.next_symmetric();
  for (int k = 0; k < m; ++k) B.b[k] = rng.next_symmetric();
  return B;
}
static inline Triple activation_triple(int act, double s) { return act == 0 ? triple_tanh(s) : triple_sin(s); }

// basis.hpp:74-93: jets of all m features; row k = [v, g, packed H]
static void phi_jets(const Basis& B, const Box& box, const Point& x, std::vector<Jet2>& out) {
  const int d = B.dim;
  const Point xh = normalize_to_box(box, x);
  const Point sc = normalize_scales(box);
  out.resize(B.m);
  for (int k = 0; k < B.m; ++k) {
    double z = B.b[k];
    for (int a = 0; a < d; ++a) z += B.R(k, a) * xh[a];
    const Triple t = activation_triple(B.act, z);
    Jet2& o = out[k];
    o = Jet2();
    o.dim = d;
    o.v = t.f;
    std::array<double, kMaxDim> gz{};
    for (int a = 0; a < d; ++a) gz[a] = B.R(k, a) * sc[a];
    for (int a = 0; a < d; ++a) o.g[a] = t.df * gz[a];
    for (int i = 0; i < d; ++i)
      for (int j = i; j < d; ++j) o.h[hess_index(i, j, d)] = t.d2f * gz[i] * gz[j];
  }
}
static void phi_values(const Basis& B, const Box& box, const Point& x, Vec& out) {  // basis.hpp:96-105
  const int d = B.dim;
  const Point xh = normalize_to_box(box, x);
  out.resize(B.m);
  for (int k = 0; k < B.m; ++k) {
    double z = B.b[k];
    for (int a = 0; a < d; ++a) z += B.R(k, a) * xh[a];
    out[k] = B.act == 0 ? std::tanh(z) : std::sin(z);
  }
}

// ---------------------------------------------------------------- windows (basis.hpp:121-176)
static Jet2 raw_window_jet(const Decomposition& dec, int j, const Point& x) {
  const int d = dec.dim();
  if (!contains(dec.sub[j], x)) return Jet2::constant(d, 0.0);
  Jet2 prod = Jet2::constant(d, 1.0);
  for (int a = 0; a < d; ++a) {
    if (dec.counts[a] == 1) continue;
    const double mu = dec.centers[j][a], sigma = dec.half[j][a];
    const Jet2 s = Jet2::variable(d, a, (x[a] - mu) / sigma, 1.0 / sigma);
    const double pi = 3.14159265358979323846;
    const Jet2 base = Jet2::constant(d, 1.0) + compose(triple_cos(pi * s.v), pi * s);
    prod = prod * (base * base);
  }
  return prod;
}
static double raw_window_value(const Decomposition& dec, int j, const Point& x) {
  const int d = dec.dim();
  if (!contains(dec.sub[j], x)) return 0.0;
  double prod = 1.0;
  for (int a = 0; a < d; ++a) {
    if (dec.counts[a] == 1) continue;
    const double s = (x[a] - dec.centers[j][a]) / dec.half[j][a];
    const double base = 1.0 + std::cos(3.14159265358979323846 * s);
    prod *= base * base;
  }
  return prod;
}
static Jet2 window_jet(const Decomposition& dec, int j, const Point& x) {
  const int d = dec.dim();
  if (!contains(dec.sub[j], x)) return Jet2::constant(d, 0.0);
  const Jet2 wj = raw_window_jet(dec, j, x);
  Jet2 total = Jet2::constant(d, 0.0);
  for (int k : dec.nbr[j]) total = total + raw_window_jet(dec, k, x);
  if (total.v <= 0.0) throw std::domain_error("window normalization vanished; point outside the domain?");
  return wj * compose(triple_recip(total.v), total);
}
static double window_value(const Decomposition& dec, int j, const Point& x) {
  const double wj = raw_window_value(dec, j, x);
  if (wj == 0.0) return 0.0;
  double total = 0.0;
  for (int k : dec.nbr[j]) total += raw_window_value(dec, k, x);
  return wj / total;
}

// ---------------------------------------------------------------- operators (operators.hpp:13-41)
enum OpKind { OP_MINUS_LAPLACIAN, OP_REACTION_DIFFUSION, OP_ADVECTION_DIFFUSION, OP_HEAT, OP_ADVECTION };
struct Op {
  OpKind kind = OP_MINUS_LAPLACIAN;
  double param = 0.0;
  double apply(const Jet2& u) const {
    switch (kind) {
      case OP_MINUS_LAPLACIAN: {
        double tr = 0.0;
        for (int a = 0; a < u.dim; ++a) tr += u.hess(a, a);
        return -tr;
      }
      case OP_REACTION_DIFFUSION: {
        double tr = 0.0;
        for (int a = 0; a < u.dim; ++a) tr += u.hess(a, a);
        return -tr + u.v;
      }
      case OP_ADVECTION_DIFFUSION:
        return u.g[1] + u.g[0] - param * u.hess(0, 0);
      case OP_HEAT: {  // u_t - kappa * sum_{space} u_aa, time = last axis
        double lap = 0.0;
        for (int a = 0; a + 1 < u.dim; ++a) lap += u.hess(a, a);
        return u.g[u.dim - 1] - param * lap;
      }
      case OP_ADVECTION:  // u_t + c u_x, axes (x, t)
        return u.g[1] + param * u.g[0];
    }
    return 0.0;
  }
};

// ---------------------------------------------------------------- problems (problems.hpp:28-173, §8d)
struct Problem {
  std::string name;
  Box domain;
  int C = 1;
  Op op;
  std::function<double(int, const Point&)> rhs;      // component, x
  std::function<Jet2(const Point&)> L;
  std::function<Jet2(int, const Point&)> G;
  std::function<double(int, const Point&)> exact;    // empty when no closed form
  bool has_exact = false;
};

static Box make_box(int d, std::initializer_list<double> lo, std::initializer_list<double> hi) {
  Box b;
  b.dim = d;
  int i = 0;
  for (double v : lo) b.lo[i++] = v;
  i = 0;
  for (double v : hi) b.hi[i++] = v;
  return b;
}

// L = prod_a tanh(x_a) tanh(1 - x_a) in the example3 loop form (problems.hpp:145-151)
static Jet2 ramp_L(int d, const Point& x) {
  Jet2 v = Jet2::constant(d, 1.0);
  for (int a = 0; a < d; ++a) v = v * tanh_of_linear(d, a, x[a], 1.0) * tanh_of_linear(d, a, x[a], -1.0, 1.0);
  return v;
}
// exp(-100 q^2) with q = alpha*x_axis + beta as a jet
static Jet2 gauss_of_linear(int d, int axis, double x, double alpha, double beta) {
  const Jet2 q = Jet2::variable(d, axis, alpha * x + beta, alpha);
  const Jet2 s = -100.0 * (q * q);
  return compose(triple_exp(s.v), s);
}

static Problem make_problem(int id, int n, int dim) {
  Problem P;
  switch (id) {
    case RDD_PROBLEM_EXAMPLE1: {  // problems.hpp:43-85
      if (n < 1 || n > 8) throw std::invalid_argument("example1: n must be in [1,8]");
      P.name = "example1";
      P.domain = make_box(2, {0.0, 0.0}, {1.0, 1.0});
      P.op = {OP_MINUS_LAPLACIAN, 0.0};
      std::vector<double> om;
      for (int i = 1; i <= n; ++i) om.push_back(std::pow(2.0, i));
      const double inv_n = 1.0 / static_cast<double>(n);
      P.exact = [om, inv_n](int, const Point& x) {
        double s = 0.0;
        for (double w : om) s += std::sin(w * kPi * x[0]) * std::sin(w * kPi * x[1]);
        return inv_n * s;
      };
      P.has_exact = true;
      P.rhs = [om, inv_n](int, const Point& x) {
        double s = 0.0;
        for (double w : om) {
          const double wp = w * kPi;
          s += 2.0 * wp * wp * std::sin(wp * x[0]) * std::sin(wp * x[1]);
        }
        return inv_n * s;
      };
      const double rho = std::pow(0.5, n);
      P.L = [rho](const Point& x) {
        return tanh_of_linear(2, 0, x[0], 1.0 / rho) * tanh_of_linear(2, 0, x[0], -1.0 / rho, 1.0 / rho) *
               tanh_of_linear(2, 1, x[1], 1.0 / rho) * tanh_of_linear(2, 1, x[1], -1.0 / rho, 1.0 / rho);
      };
      P.G = [](int, const Point&) { return Jet2::constant(2, 0.0); };
      break;
    }
    case RDD_PROBLEM_EXAMPLE2: {  // problems.hpp:91-104
      P.name = "example2";
      P.domain = make_box(2, {-1.0, 0.0}, {1.0, 1.0});
      P.op = {OP_ADVECTION_DIFFUSION, 0.1 / kPi};
      P.rhs = [](int, const Point&) { return 0.0; };
      P.L = [](const Point& x) {
        return tanh_of_linear(2, 0, x[0], 1.0, 1.0) * tanh_of_linear(2, 0, x[0], -1.0, 1.0) *
               tanh_of_linear(2, 1, x[1], 1.0);
      };
      P.G = [](int, const Point& x) { return -1.0 * sin_of_linear(2, 0, x[0], kPi); };
      P.has_exact = false;
      break;
    }
    case RDD_PROBLEM_EXAMPLE3: {  // problems.hpp:110-166
      P.name = "example3";
      P.domain = make_box(3, {0.0, 0.0, 0.0}, {1.0, 1.0, 1.0});
      P.C = 3;
      P.op = {OP_REACTION_DIFFUSION, 0.0};
      const double w = 2.0 * kPi;
      auto exact_jet = [w](int cos_axis, const Point& x) {
        Jet2 v = Jet2::constant(3, 1.0);
        for (int a = 0; a < 3; ++a)
          v = v * ((a == cos_axis) ? cos_of_linear(3, a, x[a], w) : sin_of_linear(3, a, x[a], w));
        return v;
      };
      P.exact = [w](int c, const Point& x) {
        double v = 1.0;
        for (int a = 0; a < 3; ++a) v *= (a == c) ? std::cos(w * x[a]) : std::sin(w * x[a]);
        return v;
      };
      P.has_exact = true;
      const Op op = P.op;
      P.rhs = [exact_jet, op](int c, const Point& x) { return op.apply(exact_jet(c, x)); };
      P.L = [](const Point& x) { return ramp_L(3, x); };
      P.G = [w](int c, const Point& x) {
        Jet2 v = Jet2::constant(3, 1.0);
        for (int a = 0; a < 3; ++a) {
          if (a == c) continue;
          v = v * sin_of_linear(3, a, x[a], w);
        }
        return v;
      };
      break;
    }
    case RDD_PROBLEM_POISSON: {  // C1 (d=2) / C5 (d=3)
      const int d = dim == 0 ? 2 : dim;
      if (d < 1 || d > 3) throw std::invalid_argument("poisson: dimension must be 1..3");
      P.name = "poisson";
      P.domain.dim = d;
      for (int a = 0; a < d; ++a) {
        P.domain.lo[a] = 0.0;
        P.domain.hi[a] = 1.0;
      }
      P.op = {OP_MINUS_LAPLACIAN, 0.0};
      P.exact = [d](int, const Point& x) {
        double s = 1.0;
        for (int a = 0; a < d; ++a) s *= std::sin(kPi * x[a]);
        return s;
      };
      P.has_exact = true;
      P.rhs = [d](int, const Point& x) {
        double s = 1.0;
        for (int a = 0; a < d; ++a) s *= std::sin(kPi * x[a]);
        return (static_cast<double>(d) * kPi * kPi) * s;
      };
      P.L = [d](const Point& x) { return ramp_L(d, x); };
      P.G = [d](int, const Point&) { return Jet2::constant(d, 0.0); };
      break;
    }
    case RDD_PROBLEM_MULTISCALE: {  // C2
      P.name = "multiscale";
      P.domain = make_box(2, {0.0, 0.0}, {1.0, 1.0});
      P.op = {OP_MINUS_LAPLACIAN, 0.0};
      P.exact = [](int, const Point& x) {
        return std::sin(2.0 * kPi * x[0]) * std::sin(2.0 * kPi * x[1]) +
               0.1 * (std::sin(50.0 * kPi * x[0]) * std::sin(50.0 * kPi * x[1]));
      };
      P.has_exact = true;
      P.rhs = [](int, const Point& x) {
        return (8.0 * kPi * kPi) * (std::sin(2.0 * kPi * x[0]) * std::sin(2.0 * kPi * x[1])) +
               (500.0 * kPi * kPi) * (std::sin(50.0 * kPi * x[0]) * std::sin(50.0 * kPi * x[1]));
      };
      P.L = [](const Point& x) { return ramp_L(2, x); };
      P.G = [](int, const Point&) { return Jet2::constant(2, 0.0); };
      break;
    }
    case RDD_PROBLEM_HEAT: {  // C3: u_t = 0.1 Δu on [0,1]^2 x [0,1]
      P.name = "heat";
      P.domain = make_box(3, {0.0, 0.0, 0.0}, {1.0, 1.0, 1.0});
      P.op = {OP_HEAT, 0.1};
      P.exact = [](int, const Point& x) {
        return std::exp(-0.2 * kPi * kPi * x[2]) * (std::sin(kPi * x[0]) * std::sin(kPi * x[1]));
      };
      P.has_exact = true;
      P.rhs = [](int, const Point&) { return 0.0; };
      P.L = [](const Point& x) {
        return tanh_of_linear(3, 0, x[0], 1.0) * tanh_of_linear(3, 0, x[0], -1.0, 1.0) *
               tanh_of_linear(3, 1, x[1], 1.0) * tanh_of_linear(3, 1, x[1], -1.0, 1.0) *
               tanh_of_linear(3, 2, x[2], 1.0);
      };
      P.G = [](int, const Point& x) { return sin_of_linear(3, 0, x[0], kPi) * sin_of_linear(3, 1, x[1], kPi); };
      break;
    }
    case RDD_PROBLEM_ADVECTION: {  // C4: u_t + 2 u_x = 0 on [0,2] x [0,1]
      P.name = "advection";
      P.domain = make_box(2, {0.0, 0.0}, {2.0, 1.0});
      P.op = {OP_ADVECTION, 2.0};
      P.exact = [](int, const Point& x) {
        const double q = x[0] - 2.0 * x[1] - 0.5;
        return std::exp(-100.0 * (q * q));
      };
      P.has_exact = true;
      P.rhs = [](int, const Point&) { return 0.0; };
      P.L = [](const Point& x) { return tanh_of_linear(2, 0, x[0], 1.0) * tanh_of_linear(2, 1, x[1], 1.0); };
      P.G = [](int, const Point& x) {
        // u0(x) + g(t) - u0(0), u0(x) = exp(-100 (x-0.5)^2), g(t) = exp(-100 (2t+0.5)^2)
        const Jet2 u0 = gauss_of_linear(2, 0, x[0], 1.0, -0.5);
        const Jet2 g = gauss_of_linear(2, 1, x[1], 2.0, 0.5);
        return (u0 + g) - Jet2::constant(2, std::exp(-25.0));
      };
      break;
    }
    default:
      throw std::invalid_argument("unknown problem id " + std::to_string(id));
  }
  return P;
}

// problems.hpp:219-264 Crank-Nicolson reference for example2 (bilinear lookup at 203-216)
struct RefGrid {
  int nx = 0, nt = 0;
  Vec values;
  double at(double x, double t) const {
    const double h = 2.0 / static_cast<double>(nx - 1);
    const double dt = 1.0 / static_cast<double>(nt - 1);
    double fx = (x + 1.0) / h, ft = t / dt;
    int ix = static_cast<int>(std::floor(fx)), it = static_cast<int>(std::floor(ft));
    ix = std::min(std::max(ix, 0), nx - 2);
    it = std::min(std::max(it, 0), nt - 2);
    const double ax = fx - ix, at_ = ft - it;
    const double v00 = values[it * nx + ix], v01 = values[it * nx + ix + 1];
    const double v10 = values[(it + 1) * nx + ix], v11 = values[(it + 1) * nx + ix + 1];
    return (1.0 - at_) * ((1.0 - ax) * v00 + ax * v01) + at_ * ((1.0 - ax) * v10 + ax * v11);
  }
};
static RefGrid reference_example2(int res) {
  if (res < 501) throw std::invalid_argument("reference_example2: resolution must be >= 501");
  const int nx = res, nt = res;
  const double h = 2.0 / static_cast<double>(nx - 1), dt = 1.0 / static_cast<double>(nt - 1);
  const double kappa = 0.1 / kPi, a = kappa * dt / (2.0 * h * h), c = dt / (4.0 * h);
  RefGrid ref;
  ref.nx = nx;
  ref.nt = nt;
  ref.values.assign(static_cast<size_t>(nx) * nt, 0.0);
  for (int i = 0; i < nx; ++i) ref.values[i] = -std::sin(kPi * (-1.0 + i * h));
  ref.values[0] = 0.0;
  ref.values[nx - 1] = 0.0;
  const int ni = nx - 2;
  const double lo = -(a + c), di = 1.0 + 2.0 * a, up = -(a - c);
  Vec cp(ni), rhs(ni), dp(ni);
  cp[0] = up / di;
  for (int i = 1; i < ni; ++i) cp[i] = up / (di - lo * cp[i - 1]);
  for (int step = 1; step < nt; ++step) {
    const double* prev = &ref.values[static_cast<size_t>(step - 1) * nx];
    double* next = &ref.values[static_cast<size_t>(step) * nx];
    for (int i = 0; i < ni; ++i) rhs[i] = (a + c) * prev[i] + (1.0 - 2.0 * a) * prev[i + 1] + (a - c) * prev[i + 2];
    dp[0] = rhs[0] / di;
    for (int i = 1; i < ni; ++i) dp[i] = (rhs[i] - lo * dp[i - 1]) / (di - lo * cp[i - 1]);
    next[ni] = dp[ni - 1];
    for (int i = ni - 2; i >= 0; --i) next[i + 1] = dp[i] - cp[i] * next[i + 2];
    next[0] = 0.0;
    next[nx - 1] = 0.0;
  }
  return ref;
}

// fixture-generation switches (orc_set_option): concurrent per-subdomain PCAs, and whether the
// unreduced sample matrices are kept (needed by the psi-reduction tests, ~15 GB on C5)
static int g_parallel_pca = 0;
static int g_keep_samples = 1;

// ---------------------------------------------------------------- PCA (reduction.hpp:18-155)
struct Reduced {
  Mat V;       // m x p
  Mat Vfull;   // m x min(rows, m): every right singular vector (fixture generation reads it)
  int p = 0;
  Vec sigma;   // min(rows, m), non-increasing
  bool identity = false;
};

// Thin SVD: singular values (non-increasing) and right singular vectors (m x min(rows,m)).
// Tall inputs follow Eigen's JacobiSVD (its default ColPivHouseholderQRPreconditioner): a
// column-pivoted Householder QR S·P = Q·R first, then the Jacobi SVD of the square upper
// triangular R, whose right vectors are carried back through the column permutation
// (V = P·V_R). The Jacobi SVD of R is LAPACK's one-sided dgesvj (same accuracy class as Eigen's
// two-sided sweeps: both relatively accurate on R).
static void svd_thin(const Mat& S, Vec& sv, Mat& V) {
  const int M = S.r, N = S.c;
  if (M > N) {
    Mat A = S;
    int lda = M, info = 0;
    std::vector<int> jpvt(N, 0);
    Vec tau(N);
    double wq = 0.0;
    int lq = -1;
    g_lapack.geqp3(&M, &N, A.a.data(), &lda, jpvt.data(), tau.data(), &wq, &lq, &info);
    lq = std::max(1, static_cast<int>(wq));
    Vec work_q(lq);
    g_lapack.geqp3(&M, &N, A.a.data(), &lda, jpvt.data(), tau.data(), work_q.data(), &lq, &info);
    if (info < 0) throw std::runtime_error("dgeqp3: bad argument");
    Mat R(N, N);
    for (int c = 0; c < N; ++c)
      for (int r = 0; r <= c; ++r) R(r, c) = A(r, c);
    sv.assign(N, 0.0);
    Mat VR(N, N);
    int lwork = std::max(6, 2 * N), mv = 0, ldv = N, ldr = N;
    Vec work(lwork);
    g_lapack.gesvj("U", "N", "V", &N, &N, R.a.data(), &ldr, sv.data(), &mv, VR.a.data(), &ldv, work.data(), &lwork,
                   &info, 1, 1, 1);
    if (info < 0) throw std::runtime_error("dgesvj: bad argument");
    const double scale = work[0];
    if (scale != 1.0)
      for (double& s : sv) s *= scale;
    V = Mat(N, N);
    for (int c = 0; c < N; ++c)
      for (int r = 0; r < N; ++r) V(jpvt[r] - 1, c) = VR(r, c);
  } else if (M == N) {
    Mat A = S;
    sv.assign(N, 0.0);
    V = Mat(N, N);
    int lwork = std::max(6, M + N), info = 0, mv = 0, ldv = N, lda = M;
    Vec work(lwork);
    g_lapack.gesvj("G", "N", "V", &M, &N, A.a.data(), &lda, sv.data(), &mv, V.a.data(), &ldv, work.data(), &lwork,
                   &info, 1, 1, 1);
    if (info < 0) throw std::runtime_error("dgesvj: bad argument");
    const double scale = work[0];
    if (scale != 1.0)
      for (double& s : sv) s *= scale;
  } else {
    // wide: SVD of S^T (N x M, tall); its left vectors are S's right vectors
    Mat A(N, M);
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) A(j, i) = S(i, j);
    sv.assign(M, 0.0);
    Mat dummy(1, 1);
    int lwork = std::max(6, M + N), info = 0, mv = 0, ldv = 1, lda = N, n2 = M, m2 = N;
    Vec work(lwork);
    g_lapack.gesvj("G", "U", "N", &m2, &n2, A.a.data(), &lda, sv.data(), &mv, dummy.a.data(), &ldv, work.data(),
                   &lwork, &info, 1, 1, 1);
    if (info < 0) throw std::runtime_error("dgesvj: bad argument");
    const double scale = work[0];
    if (scale != 1.0)
      for (double& s : sv) s *= scale;
    V = A;  // N x M
  }
  // sort non-increasing (Eigen's order), carrying the vectors
  const int k = static_cast<int>(sv.size());
  std::vector<int> ord(k);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return sv[a] > sv[b]; });
  Vec sv2(k);
  Mat V2(V.r, k);
  for (int i = 0; i < k; ++i) {
    sv2[i] = sv[ord[i]];
    std::copy(V.col(ord[i]), V.col(ord[i]) + V.r, V2.col(i));
  }
  sv = sv2;
  V = V2;
}

// reduction.hpp:89-109 (absolute tau; relative mode scales tau by sigma_max)
static Reduced truncate(const Mat& S, double tau, bool relative) {
  if (tau < 0.0) throw std::invalid_argument("truncation threshold tau must be >= 0");
  Reduced out;
  Mat Vfull;
  svd_thin(S, out.sigma, Vfull);
  const double thr = relative ? tau * (out.sigma.empty() ? 0.0 : out.sigma[0]) : tau;
  int keep = 0;
  for (double s : out.sigma)
    if (s > thr) ++keep;
  if (keep == 0) keep = 1;
  out.p = keep;
  out.V = Mat(Vfull.r, keep);
  for (int c = 0; c < keep; ++c) std::copy(Vfull.col(c), Vfull.col(c) + Vfull.r, out.V.col(c));
  out.Vfull = std::move(Vfull);
  for (int c = 0; c < keep; ++c) {
    for (int r = 0; r < out.V.r; ++r) {
      if (out.V(r, c) != 0.0) {
        if (out.V(r, c) < 0.0)
          for (int q = 0; q < out.V.r; ++q) out.V(q, c) = -out.V(q, c);
        break;
      }
    }
  }
  return out;
}

static Reduced identity_reduction(int m) {  // reduction.hpp:112-118
  Reduced out;
  out.V = Mat(m, m);
  for (int i = 0; i < m; ++i) out.V(i, i) = 1.0;
  out.p = m;
  out.identity = true;
  return out;
}

// ---------------------------------------------------------------- the instance + pipeline
struct SchwarzLocal {
  Mat basis;  // n x rank
  Vec inv_eigs;
  int rank = 0;
  double cond = 0.0;
};

struct Report {
  Vec W;
  int iterations = 0;
  Vec hist, true_hist;
  bool converged = false, breakdown = false;
  double final_res = 0.0;
};

struct Oracle {
  std::string err;
  rdd_config cfg{};
  uint64_t seed = 0;
  Problem prob;
  Decomposition dec;
  std::vector<Point> pts;
  std::vector<Basis> bases;
  std::vector<Mat> samples;  // PCA sample matrices (kept for parity export)
  std::vector<Reduced> red;
  std::vector<int> col_off;
  int p = 0;
  // assembled system (assembly.hpp:23-31)
  int N = 0;
  std::vector<Mat> H;
  std::vector<std::vector<int>> rows;
  Mat F;
  Vec scales;
  // normal blocks (assembly.hpp:137-146)
  std::map<std::pair<int, int>, Mat> nb;
  // Schwarz (schwarz.hpp:32-91)
  int pkind = -1;
  std::vector<std::vector<int>> sets;
  std::vector<int> owner, mult;
  std::vector<SchwarzLocal> loc;
  // solve
  std::vector<Report> reports;
  Mat W;  // p x C (unscaled)
  // evaluation
  Mat approx, exact;
  std::vector<Point> test_pts;
  rdd_summary sum{};
  std::unique_ptr<RefGrid> refgrid;
};

static double elapsed(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// L(x) * window_j(x) (the lw jet of basis.hpp:211 / reduction.hpp:134)
static Jet2 lw_jet(const Oracle& o, int j, const Point& x) { return o.prob.L(x) * window_jet(o.dec, j, x); }

// reduction.hpp:30-48
static Mat build_sample_matrix(const Oracle& o, int j, const std::vector<int>& idx) {
  const Basis& B = o.bases[j];
  Mat S(static_cast<int>(idx.size()), B.m);
  Vec phi;
  for (size_t r = 0; r < idx.size(); ++r) {
    const Point& x = o.pts[idx[r]];
    const double w = window_value(o.dec, j, x);
    phi_values(B, o.dec.sub[j], x, phi);
    for (int k = 0; k < B.m; ++k) S(static_cast<int>(r), k) = w * phi[k];
  }
  return S;
}
// reduction.hpp:53-76
static Mat build_operator_sample_matrix(const Oracle& o, int j, const std::vector<int>& idx) {
  const Basis& B = o.bases[j];
  const int nrows = static_cast<int>(idx.size());
  Mat S(nrows, B.m);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < nrows; ++r) {
    std::vector<Jet2> jets;
    const Point& x = o.pts[idx[r]];
    const Jet2 lw = lw_jet(o, j, x);
    phi_jets(B, o.dec.sub[j], x, jets);
    for (int k = 0; k < B.m; ++k) S(r, k) = o.prob.op.apply(lw * jets[k]);
  }
  return S;
}

static std::vector<int> rows_of(const Oracle& o, int j) {  // assembly.hpp:58-64
  std::vector<int> r;
  for (int i = 0; i < static_cast<int>(o.pts.size()); ++i)
    if (contains(o.dec.sub[j], o.pts[i])) r.push_back(i);
  return r;
}

// runner.hpp:40-70 build_instance
static void build_instance(Oracle& o, const rdd_config& cfg, uint64_t seed) {
  o = Oracle{};
  o.cfg = cfg;
  o.seed = seed;
  o.prob = make_problem(cfg.problem, cfg.n, cfg.dim);
  const int d = o.prob.domain.dim;
  std::vector<int> counts(cfg.counts, cfg.counts + d), colloc(cfg.colloc, cfg.colloc + d);
  if (cfg.decomposition == RDD_DECOMP_REFERENCE)
    o.dec = build_decomposition(o.prob.domain, counts, cfg.delta);
  else
    o.dec = build_cell_decomposition(o.prob.domain, counts, cfg.delta);
  o.pts = uniform_grid(o.prob.domain, colloc, cfg.boundary_per_edge);
  const int J = o.dec.size();
  if (g_parallel_pca && cfg.tau_mode != RDD_TAU_OFF) {
    // fixture generation only (tests/golden/make_fullsize.py): the per-subdomain PCAs are
    // independent, so they run concurrently; each one is the same serial computation as below
    // (the reference's loop, runner.hpp:52-65, is serial)
    for (int j = 0; j < J; ++j) o.bases.push_back(make_random_basis(subdomain_seed(seed, j), cfg.m, d, cfg.activation));
    o.red.assign(J, Reduced{});
    if (g_keep_samples) o.samples.assign(J, Mat{});
    std::string err;
#pragma omp parallel for schedule(dynamic, 1)
    for (int j = 0; j < J; ++j) {
      try {
        const std::vector<int> idx = rows_of(o, j);
        if (idx.empty()) throw std::runtime_error("subdomain " + std::to_string(j) + " contains no collocation points");
        Mat S = cfg.pca_matrix == RDD_PCA_OP_APPLIED ? build_operator_sample_matrix(o, j, idx)
                                                     : build_sample_matrix(o, j, idx);
        o.red[j] = truncate(S, cfg.tau, cfg.tau_mode == RDD_TAU_RELATIVE);
        if (g_keep_samples) o.samples[j] = std::move(S);
      } catch (const std::exception& e) {
#pragma omp critical
        err = e.what();
      }
    }
    if (!err.empty()) throw std::runtime_error(err);
  } else {
    for (int j = 0; j < J; ++j) {
      o.bases.push_back(make_random_basis(subdomain_seed(seed, j), cfg.m, d, cfg.activation));
      if (cfg.tau_mode != RDD_TAU_OFF) {
        const std::vector<int> idx = rows_of(o, j);
        if (idx.empty()) throw std::runtime_error("subdomain " + std::to_string(j) + " contains no collocation points");
        Mat S = cfg.pca_matrix == RDD_PCA_OP_APPLIED ? build_operator_sample_matrix(o, j, idx)
                                                     : build_sample_matrix(o, j, idx);
        o.red.push_back(truncate(S, cfg.tau, cfg.tau_mode == RDD_TAU_RELATIVE));
        if (g_keep_samples) o.samples.push_back(std::move(S));
      } else {
        o.red.push_back(identity_reduction(cfg.m));
      }
    }
  }
  o.col_off.assign(J + 1, 0);
  for (int j = 0; j < J; ++j) o.col_off[j + 1] = o.col_off[j] + o.red[j].p;
  o.p = o.col_off[J];
}

// assembly.hpp:41-108 assemble
static void assemble(Oracle& o) {
  const int J = o.dec.size(), d = o.dec.dim(), C = o.prob.C;
  o.N = static_cast<int>(o.pts.size());
  o.H.assign(J, Mat());
  o.rows.assign(J, {});
  for (int j = 0; j < J; ++j) {
    o.rows[j] = rows_of(o, j);
    o.H[j] = Mat(static_cast<int>(o.rows[j].size()), o.red[j].p);
  }
  long long bad_point = -1, bad_sub = -1;
  for (int j = 0; j < J; ++j) {
    const Reduced& R = o.red[j];
    const int nrows = static_cast<int>(o.rows[j].size());
#pragma omp parallel for schedule(static)
    for (int r = 0; r < nrows; ++r) {
      const Point& x = o.pts[o.rows[j][r]];
      std::vector<Jet2> phi;
      phi_jets(o.bases[j], o.dec.sub[j], x, phi);
      // out = V^T * phi (reduction.hpp:133); identity V reproduces phi exactly
      std::vector<Jet2> red(R.p);
      if (R.identity) {
        red = phi;
      } else {
        const int nh = d * (d + 1) / 2;
        for (int k = 0; k < R.p; ++k) {
          Jet2 s = Jet2::constant(d, 0.0);
          for (int l = 0; l < o.bases[j].m; ++l) {
            const double v = R.V(l, k);
            s.v += v * phi[l].v;
            for (int a = 0; a < d; ++a) s.g[a] += v * phi[l].g[a];
            for (int q = 0; q < nh; ++q) s.h[q] += v * phi[l].h[q];
          }
          red[k] = s;
        }
      }
      const Jet2 lw = lw_jet(o, j, x);
      for (int k = 0; k < R.p; ++k) {
        const double v = o.prob.op.apply(lw * red[k]);
        if (!std::isfinite(v)) {
#pragma omp critical
          {
            bad_point = o.rows[j][r];
            bad_sub = j;
          }
        }
        o.H[j](r, k) = v;
      }
    }
    if (bad_point >= 0)
      throw std::runtime_error("non-finite matrix entry at collocation point " + std::to_string(bad_point) +
                               ", subdomain " + std::to_string(bad_sub));
  }
  o.F = Mat(o.N, C);
  for (int i = 0; i < o.N; ++i)
    for (int c = 0; c < C; ++c) {
      const double v = o.prob.rhs(c, o.pts[i]) - o.prob.op.apply(o.prob.G(c, o.pts[i]));
      if (!std::isfinite(v))
        throw std::runtime_error("non-finite right-hand side at collocation point " + std::to_string(i));
      o.F(i, c) = v;
    }
}

// runner.hpp:89-101 assemble_equilibrated (column_norms / scale_columns, assembly.hpp:186-204)
static void equilibrate(Oracle& o, bool on) {
  o.scales.assign(o.p, 1.0);
  if (!on) return;
  const int J = o.dec.size();
  for (int j = 0; j < J; ++j)
    for (int c = 0; c < o.H[j].c; ++c) {
      double s = 0.0;
      const double* col = o.H[j].col(c);
      for (int r = 0; r < o.H[j].r; ++r) s += col[r] * col[r];
      o.scales[o.col_off[j] + c] = std::sqrt(s);
    }
  for (double& s : o.scales)
    if (s == 0.0) s = 1.0;
  for (int j = 0; j < J; ++j)
    for (int c = 0; c < o.H[j].c; ++c) {
      const double s = o.scales[o.col_off[j] + c];
      if (s > 0.0)
        for (int r = 0; r < o.H[j].r; ++r) o.H[j](r, c) /= s;
    }
}

// assembly.hpp:110-133
static Vec matvec(const Oracle& o, const Vec& w) {
  if (static_cast<int>(w.size()) != o.p) throw std::invalid_argument("matvec: coefficient vector has wrong length");
  Vec y(o.N, 0.0);
  for (size_t j = 0; j < o.H.size(); ++j) {
    const Mat& Hj = o.H[j];
    Vec local(Hj.r, 0.0);
    for (int k = 0; k < Hj.c; ++k) {
      const double wk = w[o.col_off[j] + k];
      const double* col = Hj.col(k);
      for (int r = 0; r < Hj.r; ++r) local[r] += col[r] * wk;
    }
    for (int r = 0; r < Hj.r; ++r) y[o.rows[j][r]] += local[r];
  }
  return y;
}
static Vec matvec_transpose(const Oracle& o, const Vec& rr) {
  if (static_cast<int>(rr.size()) != o.N)
    throw std::invalid_argument("matvec_transpose: residual vector has wrong length");
  Vec y(o.p, 0.0);
  for (size_t j = 0; j < o.H.size(); ++j) {
    const Mat& Hj = o.H[j];
    for (int k = 0; k < Hj.c; ++k) {
      double s = 0.0;
      const double* col = Hj.col(k);
      for (int r = 0; r < Hj.r; ++r) s += col[r] * rr[o.rows[j][r]];
      y[o.col_off[j] + k] = s;
    }
  }
  return y;
}

// assembly.hpp:148-183 normal_blocks
static void normal_blocks(Oracle& o) {
  o.nb.clear();
  const int J = o.dec.size();
  for (int j1 = 0; j1 < J; ++j1)
    for (int j2 : o.dec.nbr[j1]) {
      if (j2 < j1) continue;
      const auto& r1 = o.rows[j1];
      const auto& r2 = o.rows[j2];
      std::vector<int> i1, i2;
      size_t a = 0, b = 0;
      while (a < r1.size() && b < r2.size()) {
        if (r1[a] == r2[b]) {
          i1.push_back(static_cast<int>(a++));
          i2.push_back(static_cast<int>(b++));
        } else if (r1[a] < r2[b]) {
          ++a;
        } else {
          ++b;
        }
      }
      if (i1.empty()) continue;
      const Mat& H1 = o.H[j1];
      const Mat& H2 = o.H[j2];
      Mat B(H1.c, H2.c);
      for (int c2 = 0; c2 < H2.c; ++c2)
        for (int c1 = 0; c1 < H1.c; ++c1) {
          double s = 0.0;
          for (size_t k = 0; k < i1.size(); ++k) s += H1(i1[k], c1) * H2(i2[k], c2);
          B(c1, c2) = s;
        }
      o.nb[{j1, j2}] = std::move(B);
    }
}

static void syevd(Mat& A, Vec& w) {  // ascending eigenvalues, vectors in A
  const int n = A.r;
  w.assign(n, 0.0);
  if (n == 0) return;
  int lwork = -1, liwork = -1, info = 0, lda = n;
  double wq = 0;
  int iq = 0;
  g_lapack.syevd("V", "U", &n, A.a.data(), &lda, w.data(), &wq, &lwork, &iq, &liwork, &info, 1, 1);
  lwork = static_cast<int>(wq) + 1;
  liwork = iq + 1;
  Vec work(lwork);
  std::vector<int> iwork(liwork);
  g_lapack.syevd("V", "U", &n, A.a.data(), &lda, w.data(), work.data(), &lwork, iwork.data(), &liwork, &info, 1, 1);
  if (info != 0) throw std::runtime_error("dsyevd failed");
}

// schwarz.hpp:39-61 build_index_sets + :93-148 build_preconditioner
static void build_preconditioner(Oracle& o, int kind) {
  const int J = o.dec.size();
  o.pkind = kind;
  o.owner.assign(o.p, 0);
  for (int j = 0; j < J; ++j)
    for (int c = o.col_off[j]; c < o.col_off[j + 1]; ++c) o.owner[c] = j;
  o.sets.assign(J, {});
  for (int i = 0; i < J; ++i)
    for (int j : o.dec.nbr[i])
      for (int c = o.col_off[j]; c < o.col_off[j + 1]; ++c) o.sets[i].push_back(c);
  o.mult.assign(o.p, 0);
  for (const auto& s : o.sets)
    for (int c : s) ++o.mult[c];
  o.loc.assign(J, SchwarzLocal{});
  for (int i = 0; i < J; ++i) {
    const auto& S = o.sets[i];
    if (S.empty()) throw std::runtime_error("empty index set for subdomain " + std::to_string(i));
    const int n = static_cast<int>(S.size());
    std::vector<std::pair<int, int>> parts;
    for (size_t k = 0; k < S.size();) {
      const int j = o.owner[S[k]];
      parts.emplace_back(j, static_cast<int>(k));
      k += static_cast<size_t>(o.col_off[j + 1] - o.col_off[j]);
    }
    Mat A(n, n);
    for (const auto& [j1, off1] : parts)
      for (const auto& [j2, off2] : parts) {
        auto it = o.nb.find({std::min(j1, j2), std::max(j1, j2)});
        if (it == o.nb.end()) continue;
        const Mat& B = it->second;
        if (j1 <= j2) {
          for (int c = 0; c < B.c; ++c)
            for (int r = 0; r < B.r; ++r) A(off1 + r, off2 + c) = B(r, c);
        } else {
          for (int c = 0; c < B.c; ++c)
            for (int r = 0; r < B.r; ++r) A(off1 + c, off2 + r) = B(r, c);
        }
      }
    Vec ev;
    syevd(A, ev);
    const double cutoff = 1e-12 * std::max(0.0, ev[n - 1]);  // kLocalRankCutoff (schwarz.hpp:82)
    int first = n;
    for (int k = 0; k < n; ++k)
      if (ev[k] > cutoff) {
        first = k;
        break;
      }
    SchwarzLocal& L = o.loc[i];
    L.rank = n - first;
    L.basis = Mat(n, L.rank);
    for (int c = 0; c < L.rank; ++c) std::copy(A.col(first + c), A.col(first + c) + n, L.basis.col(c));
    L.inv_eigs.assign(L.rank, 0.0);
    for (int c = 0; c < L.rank; ++c) L.inv_eigs[c] = 1.0 / ev[first + c];
    L.cond = L.rank > 0 ? ev[n - 1] / ev[first] : 0.0;
  }
}

static Vec local_solve(const SchwarzLocal& L, const Vec& rhs) {  // schwarz.hpp:76-79
  const int n = static_cast<int>(rhs.size());
  Vec out(n, 0.0);
  if (L.rank == 0) return out;
  Vec t(L.rank, 0.0);
  for (int c = 0; c < L.rank; ++c) {
    double s = 0.0;
    const double* col = L.basis.col(c);
    for (int r = 0; r < n; ++r) s += col[r] * rhs[r];
    t[c] = L.inv_eigs[c] * s;
  }
  for (int c = 0; c < L.rank; ++c) {
    const double* col = L.basis.col(c);
    for (int r = 0; r < n; ++r) out[r] += col[r] * t[c];
  }
  return out;
}

// schwarz.hpp:153-185 apply / :189-215 apply_transpose
static Vec precond_apply(const Oracle& o, const Vec& v, bool transpose) {
  if (static_cast<int>(v.size()) != o.p) throw std::invalid_argument("preconditioner apply: wrong vector length");
  const int J = static_cast<int>(o.sets.size());
  std::vector<Vec> local(J);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < J; ++i) {
    const auto& S = o.sets[i];
    Vec rhs(S.size());
    for (size_t k = 0; k < S.size(); ++k) {
      double val = v[S[k]];
      if (transpose) {
        if (o.pkind == RDD_PRECOND_SAS) val /= o.mult[S[k]];
        else if (o.pkind == RDD_PRECOND_RAS) val = (o.owner[S[k]] == i) ? val : 0.0;
      }
      rhs[k] = val;
    }
    local[i] = local_solve(o.loc[i], rhs);
  }
  Vec out(o.p, 0.0);
  for (int i = 0; i < J; ++i) {
    const auto& S = o.sets[i];
    const Vec& z = local[i];
    if (transpose || o.pkind == RDD_PRECOND_AS) {
      for (size_t k = 0; k < S.size(); ++k) out[S[k]] += z[k];
    } else if (o.pkind == RDD_PRECOND_SAS) {
      for (size_t k = 0; k < S.size(); ++k) out[S[k]] += z[k] / o.mult[S[k]];
    } else {
      for (size_t k = 0; k < S.size(); ++k)
        if (o.owner[S[k]] == i) out[S[k]] += z[k];
    }
  }
  return out;
}

// ---------------------------------------------------------------- Krylov (krylov.hpp:29-401)
struct LinMap {
  std::function<Vec(const Vec&)> apply, apply_t;
  bool identity = false;
  Vec operator()(const Vec& v) const { return apply(v); }
  Vec t(const Vec& v) const { return apply_t ? apply_t(v) : apply(v); }
};
static int effective_max_iter(int max_iter, int p) {
  if (max_iter < 0) throw std::invalid_argument("max_iter must be >= 1");
  return max_iter == 0 ? 10 * p : max_iter;
}
static void axpy(double a, const Vec& x, Vec& y) {
  for (size_t i = 0; i < y.size(); ++i) y[i] += a * x[i];
}

static Report cg(const LinMap& A, const LinMap& M, const Vec& b, double tol, int max_iter_cfg) {  // :106-156
  Report rep;
  const int n = static_cast<int>(b.size());
  const int max_iter = effective_max_iter(max_iter_cfg, n);
  const double bnorm = norm(b);
  Vec x(n, 0.0), r = b, z = M(r);
  const double z0 = norm(z);
  if (z0 == 0.0) {
    rep.W = x;
    rep.converged = true;
    rep.hist = {0.0};
    rep.true_hist = {0.0};
    return rep;
  }
  Vec p = z;
  double rz = dot(r, z);
  rep.hist.push_back(1.0);
  rep.true_hist.push_back(bnorm > 0.0 ? 1.0 : 0.0);
  for (int it = 0; it < max_iter; ++it) {
    const Vec Ap = A(p);
    const double pAp = dot(p, Ap);
    if (pAp <= 0.0 || rz == 0.0) {
      rep.breakdown = true;
      break;
    }
    const double alpha = rz / pAp;
    axpy(alpha, p, x);
    axpy(-alpha, Ap, r);
    z = M(r);
    const double rel = norm(z) / z0;
    rep.hist.push_back(rel);
    rep.true_hist.push_back(bnorm > 0.0 ? norm(r) / bnorm : norm(r));
    ++rep.iterations;
    if (rel <= tol) {
      rep.converged = true;
      break;
    }
    const double rzn = dot(r, z);
    const double beta = rzn / rz;
    rz = rzn;
    for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  rep.W = x;
  rep.final_res = rep.hist.back();
  return rep;
}

static Report cgs(const LinMap& A, const LinMap& M, const Vec& b, double tol, int max_iter_cfg) {  // :159-213
  Report rep;
  const int n = static_cast<int>(b.size());
  const int max_iter = effective_max_iter(max_iter_cfg, n);
  const double bnorm = norm(b);
  auto Cm = [&](const Vec& v) { return M(A(v)); };
  Vec x(n, 0.0);
  const Vec g = M(b);
  const double gnorm = norm(g);
  if (gnorm == 0.0) {
    rep.W = x;
    rep.converged = true;
    rep.hist = {0.0};
    rep.true_hist = {0.0};
    return rep;
  }
  Vec r = g;
  const Vec rstar = g;
  Vec p = r, u = r;
  double rho = dot(rstar, r);
  rep.hist.push_back(1.0);
  rep.true_hist.push_back(bnorm > 0.0 ? 1.0 : 0.0);
  for (int it = 0; it < max_iter; ++it) {
    const Vec Cp = Cm(p);
    const double sigma = dot(rstar, Cp);
    if (sigma == 0.0 || rho == 0.0) {
      rep.breakdown = true;
      break;
    }
    const double alpha = rho / sigma;
    Vec q(n), uq(n);
    for (int i = 0; i < n; ++i) q[i] = u[i] - alpha * Cp[i];
    for (int i = 0; i < n; ++i) uq[i] = u[i] + q[i];
    axpy(alpha, uq, x);
    const Vec Cuq = Cm(uq);
    axpy(-alpha, Cuq, r);
    const double rel = norm(r) / gnorm;
    rep.hist.push_back(rel);
    if (M.identity) {
      rep.true_hist.push_back(rel);
    } else {
      Vec res = A(x);
      for (int i = 0; i < n; ++i) res[i] = b[i] - res[i];
      rep.true_hist.push_back(bnorm > 0.0 ? norm(res) / bnorm : 0.0);
    }
    ++rep.iterations;
    if (rel <= tol) {
      rep.converged = true;
      break;
    }
    const double rhon = dot(rstar, r);
    const double beta = rhon / rho;
    rho = rhon;
    for (int i = 0; i < n; ++i) u[i] = r[i] + beta * q[i];
    for (int i = 0; i < n; ++i) p[i] = u[i] + beta * (q[i] + beta * p[i]);
  }
  rep.W = x;
  rep.final_res = rep.hist.back();
  return rep;
}

static Report bicg(const LinMap& A, const LinMap& M, const Vec& b, double tol, int max_iter_cfg) {  // :217-270
  Report rep;
  const int n = static_cast<int>(b.size());
  const int max_iter = effective_max_iter(max_iter_cfg, n);
  const double bnorm = norm(b);
  auto Cm = [&](const Vec& v) { return M(A(v)); };
  auto Ct = [&](const Vec& v) { return A.t(M.t(v)); };
  Vec x(n, 0.0);
  const Vec g = M(b);
  const double gnorm = norm(g);
  if (gnorm == 0.0) {
    rep.W = x;
    rep.converged = true;
    rep.hist = {0.0};
    rep.true_hist = {0.0};
    return rep;
  }
  Vec r = g, rstar = g, p = r, pstar = rstar;
  double rho = dot(rstar, r);
  rep.hist.push_back(1.0);
  rep.true_hist.push_back(bnorm > 0.0 ? 1.0 : 0.0);
  for (int it = 0; it < max_iter; ++it) {
    const Vec Cp = Cm(p);
    const double sigma = dot(pstar, Cp);
    if (sigma == 0.0 || rho == 0.0) {
      rep.breakdown = true;
      break;
    }
    const double alpha = rho / sigma;
    axpy(alpha, p, x);
    axpy(-alpha, Cp, r);
    const Vec Ctp = Ct(pstar);
    axpy(-alpha, Ctp, rstar);
    const double rel = norm(r) / gnorm;
    rep.hist.push_back(rel);
    if (M.identity) {
      rep.true_hist.push_back(rel);
    } else {
      Vec res = A(x);
      for (int i = 0; i < n; ++i) res[i] = b[i] - res[i];
      rep.true_hist.push_back(bnorm > 0.0 ? norm(res) / bnorm : 0.0);
    }
    ++rep.iterations;
    if (rel <= tol) {
      rep.converged = true;
      break;
    }
    const double rhon = dot(rstar, r);
    const double beta = rhon / rho;
    rho = rhon;
    for (int i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
    for (int i = 0; i < n; ++i) pstar[i] = rstar[i] + beta * pstar[i];
  }
  rep.W = x;
  rep.final_res = rep.hist.back();
  return rep;
}

// upper-triangular solve of Hm[0:k,0:k] y = g[0:k] (Eigen triangularView<Upper>().solve)
static Vec upper_solve(const Mat& Hm, const Vec& g, int k) {
  Vec y(k);
  for (int i = k - 1; i >= 0; --i) {
    double s = g[i];
    for (int j = i + 1; j < k; ++j) s -= Hm(i, j) * y[j];
    y[i] = s / Hm(i, i);
  }
  return y;
}

static Report gmres(const LinMap& A, const LinMap& M, const Vec& b, double tol, int max_iter_cfg, int restart,
                    bool true_residual) {  // krylov.hpp:275-389
  Report rep;
  const int n = static_cast<int>(b.size());
  const int max_iter = effective_max_iter(max_iter_cfg, n);
  const double bnorm = norm(b);
  const Vec g0 = M(b);
  const double gnorm0 = norm(g0);
  if (gnorm0 == 0.0) {
    rep.W.assign(n, 0.0);
    rep.converged = true;
    rep.hist = {0.0};
    rep.true_hist = {0.0};
    return rep;
  }
  const int cycle_len = restart > 0 ? restart : std::min(max_iter, n);
  if (restart == 0 && cycle_len > 4096)
    throw std::runtime_error("full GMRES basis of " + std::to_string(cycle_len) +
                             " vectors exceeds the cap; configure gmres_restart");
  Vec x(n, 0.0);
  rep.hist.push_back(1.0);
  rep.true_hist.push_back(bnorm > 0.0 ? 1.0 : 0.0);
  int iters_left = max_iter;
  while (iters_left > 0 && !rep.converged && !rep.breakdown) {
    Vec res = A(x);
    for (int i = 0; i < n; ++i) res[i] = b[i] - res[i];
    const Vec r0 = M.identity ? res : M(res);
    const double beta = norm(r0);
    if (beta / gnorm0 <= tol) {
      rep.converged = true;
      break;
    }
    const int len = std::min(cycle_len, iters_left);
    std::vector<Vec> V;
    V.reserve(len + 1);
    Vec v0 = r0;
    for (double& e : v0) e /= beta;
    V.push_back(v0);
    Mat Hm(len + 1, len);
    Vec cs(len, 0.0), sn(len, 0.0), gv(len + 1, 0.0);
    gv[0] = beta;
    int k = 0;
    for (; k < len;) {
      Vec w = M.identity ? A(V[k]) : M(A(V[k]));
      for (int i = 0; i <= k; ++i) {
        Hm(i, k) = dot(w, V[i]);
        axpy(-Hm(i, k), V[i], w);
      }
      for (int i = 0; i <= k; ++i) {
        const double corr = dot(w, V[i]);
        Hm(i, k) += corr;
        axpy(-corr, V[i], w);
      }
      const double hnext = norm(w);
      Hm(k + 1, k) = hnext;
      if (hnext > 0.0) {
        for (double& e : w) e /= hnext;
        V.push_back(w);
      }
      for (int i = 0; i < k; ++i) {
        const double t = cs[i] * Hm(i, k) + sn[i] * Hm(i + 1, k);
        Hm(i + 1, k) = -sn[i] * Hm(i, k) + cs[i] * Hm(i + 1, k);
        Hm(i, k) = t;
      }
      const double denom = std::hypot(Hm(k, k), Hm(k + 1, k));
      if (denom == 0.0) {
        rep.breakdown = true;
        break;
      }
      cs[k] = Hm(k, k) / denom;
      sn[k] = Hm(k + 1, k) / denom;
      Hm(k, k) = denom;
      Hm(k + 1, k) = 0.0;
      gv[k + 1] = -sn[k] * gv[k];
      gv[k] *= cs[k];
      const double rel = std::abs(gv[k + 1]) / gnorm0;
      rep.hist.push_back(rel);
      ++rep.iterations;
      --iters_left;
      ++k;
      if (M.identity) {
        rep.true_hist.push_back(rel);
      } else if (true_residual) {
        const Vec y = upper_solve(Hm, gv, k);
        Vec xk = x;
        for (int i = 0; i < k; ++i) axpy(y[i], V[i], xk);
        Vec rr = A(xk);
        for (int i = 0; i < n; ++i) rr[i] = b[i] - rr[i];
        rep.true_hist.push_back(bnorm > 0.0 ? norm(rr) / bnorm : 0.0);
      } else {
        rep.true_hist.push_back(-1.0);
      }
      if (rel <= tol || hnext == 0.0) {
        rep.converged = true;
        break;
      }
      if (iters_left == 0) break;
    }
    if (k > 0) {
      const Vec y = upper_solve(Hm, gv, k);
      for (int i = 0; i < k; ++i) axpy(y[i], V[i], x);
    }
    if (restart == 0 && !rep.converged && !rep.breakdown && iters_left > 0 && k == cycle_len) break;
  }
  rep.W = x;
  rep.final_res = rep.hist.back();
  return rep;
}

// Column-pivoted QR least squares (krylov.hpp:97-101, runner.hpp:217-222), Eigen rank rule.
static Mat qr_solve(const Mat& Hd, const Mat& Fm) {
  const int M = Hd.r, N = Hd.c, C = Fm.c;
  Mat A = Hd;
  std::vector<int> jpvt(N, 0);
  Vec tauv(std::min(M, N));
  int lwork = -1, info = 0, lda = M;
  double wq = 0;
  g_lapack.geqp3(&M, &N, A.a.data(), &lda, jpvt.data(), tauv.data(), &wq, &lwork, &info);
  lwork = static_cast<int>(wq) + 1;
  Vec work(lwork);
  g_lapack.geqp3(&M, &N, A.a.data(), &lda, jpvt.data(), tauv.data(), work.data(), &lwork, &info);
  if (info != 0) throw std::runtime_error("dgeqp3 failed");
  const int kd = std::min(M, N);
  Mat B = Fm;
  int k = kd, ldb = M;
  lwork = -1;
  g_lapack.ormqr("L", "T", &M, &C, &k, A.a.data(), &lda, tauv.data(), B.a.data(), &ldb, &wq, &lwork, &info, 1, 1);
  lwork = static_cast<int>(wq) + 1;
  work.assign(lwork, 0.0);
  g_lapack.ormqr("L", "T", &M, &C, &k, A.a.data(), &lda, tauv.data(), B.a.data(), &ldb, work.data(), &lwork, &info,
                 1, 1);
  double maxpiv = 0.0;
  for (int i = 0; i < kd; ++i) maxpiv = std::max(maxpiv, std::abs(A(i, i)));
  const double thr = maxpiv * (2.220446049250313e-16 * kd);
  int rank = 0;
  for (int i = 0; i < kd; ++i)
    if (std::abs(A(i, i)) > thr) ++rank;
  Mat X(N, C);
  for (int c = 0; c < C; ++c) {
    Vec z(rank);
    for (int i = rank - 1; i >= 0; --i) {
      double s = B(i, c);
      for (int j = i + 1; j < rank; ++j) s -= A(i, j) * z[j];
      z[i] = s / A(i, i);
    }
    for (int i = 0; i < rank; ++i) X(jpvt[i] - 1, c) = z[i];
  }
  return X;
}

static Mat densify(const Oracle& o) {  // assembly.hpp:206-215
  Mat Hd(o.N, o.p);
  for (size_t j = 0; j < o.H.size(); ++j)
    for (int r = 0; r < o.H[j].r; ++r)
      for (int c = 0; c < o.H[j].c; ++c) Hd(o.rows[j][r], o.col_off[j] + c) = o.H[j](r, c);
  return Hd;
}
static Mat densify_nb(const Oracle& o) {  // assembly.hpp:217-228
  Mat A(o.p, o.p);
  for (const auto& [key, B] : o.nb) {
    const auto [j1, j2] = key;
    for (int c = 0; c < B.c; ++c)
      for (int r = 0; r < B.r; ++r) {
        A(o.col_off[j1] + r, o.col_off[j2] + c) = B(r, c);
        if (j1 != j2) A(o.col_off[j2] + c, o.col_off[j1] + r) = B(r, c);
      }
  }
  return A;
}

static LinMap make_A(const Oracle& o) {
  LinMap A;
  A.apply = [&o](const Vec& w) { return matvec_transpose(o, matvec(o, w)); };
  return A;
}
static LinMap make_M(const Oracle& o) {
  LinMap M;
  if (o.pkind < 0) {
    M.apply = [](const Vec& v) { return v; };
    M.identity = true;
  } else {
    M.apply = [&o](const Vec& v) { return precond_apply(o, v, false); };
    M.apply_t = [&o](const Vec& v) { return precond_apply(o, v, true); };
  }
  return M;
}

// runner.hpp:239-251
static void solve(Oracle& o, int solver, double tol, int max_iter, int restart, bool true_residual) {
  const int C = o.prob.C;
  o.W = Mat(o.p, C);
  o.reports.clear();
  if (solver == RDD_SOLVER_QR) {
    const Mat X = qr_solve(densify(o), o.F);
    o.W = X;
  } else {
    const LinMap A = make_A(o), M = make_M(o);
    for (int c = 0; c < C; ++c) {
      Vec Fc(o.F.col(c), o.F.col(c) + o.N);
      const Vec b = matvec_transpose(o, Fc);
      Report rep;
      switch (solver) {
        case RDD_SOLVER_CG: rep = cg(A, M, b, tol, max_iter); break;
        case RDD_SOLVER_CGS: rep = cgs(A, M, b, tol, max_iter); break;
        case RDD_SOLVER_BICG: rep = bicg(A, M, b, tol, max_iter); break;
        case RDD_SOLVER_GMRES: rep = gmres(A, M, b, tol, max_iter, restart, true_residual); break;
        default: throw std::invalid_argument("unknown solver");
      }
      std::copy(rep.W.begin(), rep.W.end(), o.W.col(c));
      o.reports.push_back(std::move(rep));
    }
  }
  for (int c = 0; c < C; ++c)
    for (int i = 0; i < o.p; ++i) o.W(i, c) /= o.scales[i];
}

// runner.hpp:105-127 evaluate_solution; :130-144 exact_values; problems.hpp:275-302 errors
static void evaluate(Oracle& o, const std::vector<int>& test_res) {
  const int C = o.prob.C, J = o.dec.size();
  o.test_pts = uniform_grid(o.prob.domain, test_res, 0);
  const int M = static_cast<int>(o.test_pts.size());
  o.approx = Mat(M, C);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < M; ++i) {
    const Point& x = o.test_pts[i];
    const double Lv = o.prob.L(x).v;
    Vec phi, local;
    for (int j = 0; j < J; ++j) {
      if (!contains(o.dec.sub[j], x)) continue;  // covering_subdomains (geometry.hpp:180-185)
      const Reduced& R = o.red[j];
      phi_values(o.bases[j], o.dec.sub[j], x, phi);
      const double w = window_value(o.dec, j, x);
      local.assign(R.p, 0.0);
      for (int k = 0; k < R.p; ++k) {
        double s = 0.0;
        for (int l = 0; l < o.bases[j].m; ++l) s += R.V(l, k) * phi[l];
        local[k] = s * (Lv * w);
      }
      const int off = o.col_off[j];
      for (int c = 0; c < C; ++c) {
        double s = 0.0;
        for (int k = 0; k < R.p; ++k) s += o.W(off + k, c) * local[k];
        o.approx(i, c) += s;
      }
    }
    for (int c = 0; c < C; ++c) o.approx(i, c) += o.prob.G(c, x).v;
  }
  o.exact = Mat(M, C);
  if (o.prob.has_exact) {
    for (int i = 0; i < M; ++i)
      for (int c = 0; c < C; ++c) o.exact(i, c) = o.prob.exact(c, o.test_pts[i]);
  } else {
    const int res = o.cfg.ref_resolution > 0 ? o.cfg.ref_resolution : 2001;  // config.hpp:28
    if (!o.refgrid || o.refgrid->nx != res) o.refgrid = std::make_unique<RefGrid>(reference_example2(res));
    for (int i = 0; i < M; ++i) o.exact(i, 0) = o.refgrid->at(o.test_pts[i][0], o.test_pts[i][1]);
  }
  double dn = 0.0, num = 0.0, mean = 0.0, l1 = 0.0;
  for (size_t i = 0; i < o.exact.a.size(); ++i) {
    const double e = o.exact.a[i], dv = o.approx.a[i] - e;
    dn += e * e;
    num += dv * dv;
    mean += e;
    l1 += std::abs(dv);
  }
  if (dn == 0.0) throw std::domain_error("rel_l2: exact solution has zero norm");
  mean /= static_cast<double>(o.exact.a.size());
  double var = 0.0;
  for (double e : o.exact.a) var += (e - mean) * (e - mean);
  var /= static_cast<double>(o.exact.a.size());
  const double gamma = std::sqrt(var);
  if (gamma == 0.0) throw std::domain_error("normalized_l1: exact solution set has zero standard deviation");
  o.sum.e_l2 = std::sqrt(num) / std::sqrt(dn);
  o.sum.e_l1n = l1 / (static_cast<double>(M) * gamma);
}

static void run_single(Oracle& o, const rdd_config& cfg, uint64_t seed) {  // runner.hpp:202-275
  auto t0 = std::chrono::steady_clock::now();
  build_instance(o, cfg, seed);
  o.sum.t_pca = elapsed(t0);
  assemble(o);
  equilibrate(o, cfg.precond >= 0);
  o.sum.t_assemble = elapsed(t0);
  o.sum.t_precond = 0.0;
  if (cfg.solver != RDD_SOLVER_QR && cfg.precond >= 0) {
    t0 = std::chrono::steady_clock::now();
    normal_blocks(o);
    build_preconditioner(o, cfg.precond);
    o.sum.t_precond = elapsed(t0);
  }
  t0 = std::chrono::steady_clock::now();
  solve(o, cfg.solver, cfg.rel_tol, cfg.max_iter, cfg.gmres_restart, cfg.true_residual != 0);
  o.sum.t_solve = elapsed(t0);
  t0 = std::chrono::steady_clock::now();
  std::vector<int> test(cfg.test, cfg.test + o.dec.dim());
  evaluate(o, test);
  o.sum.t_evaluate = elapsed(t0);
  o.sum.seed = seed;
  o.sum.J = o.dec.size();
  o.sum.p = o.p;
  o.sum.DoF = o.p * o.prob.C;
  o.sum.N = o.N;
  int it = 0;
  bool conv = true, brk = false;
  double fr = 0.0;
  for (const auto& r : o.reports) {
    it = std::max(it, r.iterations);
    conv = conv && r.converged;
    brk = brk || r.breakdown;
    fr = std::max(fr, r.final_res);
  }
  o.sum.iterations = it;
  o.sum.converged = conv ? 1 : 0;
  o.sum.breakdown = brk ? 1 : 0;
  o.sum.final_residual = fr;
}

}  // namespace orc

// ================================================================ C ABI (prefix orc_)
using orc::Oracle;

template <class F>
static int guarded(Oracle* o, F&& f) {
  try {
    f();
    return RDD_OK;
  } catch (const std::invalid_argument& e) {
    o->err = e.what();
    return RDD_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    o->err = e.what();
    return RDD_DOMAIN_ERROR;
  } catch (const std::exception& e) {
    o->err = e.what();
    return RDD_RUNTIME_ERROR;
  }
}

extern "C" {

void* orc_create(const char* lapack_path, int threads) {
  try {
    orc::load_lapack(lapack_path);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return nullptr;
  }
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  return new Oracle();
}
void orc_destroy(void* h) { delete static_cast<Oracle*>(h); }
const char* orc_last_error(void* h) { return static_cast<Oracle*>(h)->err.c_str(); }
int orc_set_option(const char* name, int value) {
  const std::string n = name ? name : "";
  if (n == "parallel_pca") orc::g_parallel_pca = value;
  else if (n == "keep_samples") orc::g_keep_samples = value;
  else return 1;
  return 0;
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

int orc_build_instance(void* h, const rdd_config* cfg, uint64_t seed) {
  Oracle* o = static_cast<Oracle*>(h);
  return guarded(o, [&] { orc::build_instance(*o, *cfg, seed); });
}
int orc_assemble(void* h, int equilibrate) {
  Oracle* o = static_cast<Oracle*>(h);
  return guarded(o, [&] {
    orc::assemble(*o);
    orc::equilibrate(*o, equilibrate != 0);
  });
}
int orc_build_preconditioner(void* h, int kind) {
  Oracle* o = static_cast<Oracle*>(h);
  return guarded(o, [&] {
    orc::normal_blocks(*o);
    if (kind >= 0) orc::build_preconditioner(*o, kind);
    else o->pkind = -1;
  });
}
int orc_normal_blocks(void* h) {
  Oracle* o = static_cast<Oracle*>(h);
  return guarded(o, [&] { orc::normal_blocks(*o); });
}
int orc_solve(void* h, int solver, double tol, int max_iter, int restart, int true_residual) {
  Oracle* o = static_cast<Oracle*>(h);
  return guarded(o, [&] { orc::solve(*o, solver, tol, max_iter, restart, true_residual != 0); });
}
int orc_evaluate(void* h, const int* test_res) {
  Oracle* o = static_cast<Oracle*>(h);
  return guarded(o, [&] { orc::evaluate(*o, std::vector<int>(test_res, test_res + o->dec.dim())); });
}
int orc_run_single(void* h, const rdd_config* cfg, uint64_t seed, rdd_summary* out) {
  Oracle* o = static_cast<Oracle*>(h);
  const int st = guarded(o, [&] { orc::run_single(*o, *cfg, seed); });
  if (st == RDD_OK && out) *out = o->sum;
  return st;
}
int orc_get_summary(void* h, rdd_summary* out) {
  *out = static_cast<Oracle*>(h)->sum;
  return RDD_OK;
}

int orc_matvec(void* h, const double* w, double* y) {
  Oracle* o = static_cast<Oracle*>(h);
  return guarded(o, [&] {
    const orc::Vec r = orc::matvec(*o, orc::Vec(w, w + o->p));
    std::copy(r.begin(), r.end(), y);
  });
}
int orc_matvec_transpose(void* h, const double* rr, double* out) {
  Oracle* o = static_cast<Oracle*>(h);
  return guarded(o, [&] {
    const orc::Vec r = orc::matvec_transpose(*o, orc::Vec(rr, rr + o->N));
    std::copy(r.begin(), r.end(), out);
  });
}
int orc_precond_apply(void* h, const double* v, double* z, int transpose) {
  Oracle* o = static_cast<Oracle*>(h);
  return guarded(o, [&] {
    const orc::Vec r = orc::precond_apply(*o, orc::Vec(v, v + o->p), transpose != 0);
    std::copy(r.begin(), r.end(), z);
  });
}
// Dense symmetric spectrum of H^T H (ascending) and, if with_precond, eigenvalues of M^-1 H^T H
// (real parts, ascending): the runner.hpp:344-362 spectrum_cmd diagnostics.
int orc_spectra(void* h, double* normal, double* precond_re, double* cond_normal, double* cond_precond) {
  Oracle* o = static_cast<Oracle*>(h);
  return guarded(o, [&] {
    const orc::Mat A = orc::densify_nb(*o);
    const int n = A.r;
    orc::Mat Ac = A;
    orc::Vec ev;
    orc::syevd(Ac, ev);
    if (normal) std::copy(ev.begin(), ev.end(), normal);
    auto cond_of = [&](orc::Mat Mx) {
      const int mm = Mx.r, nn = Mx.c, k = std::min(mm, nn);
      orc::Vec s(k);
      double dummy = 0;
      int ld1 = 1, lwork = -1, info = 0, lda = mm;
      double wq = 0;
      orc::g_lapack.gesvd("N", "N", &mm, &nn, Mx.a.data(), &lda, s.data(), &dummy, &ld1, &dummy, &ld1, &wq, &lwork,
                          &info, 1, 1);
      lwork = static_cast<int>(wq) + 1;
      orc::Vec work(lwork);
      orc::g_lapack.gesvd("N", "N", &mm, &nn, Mx.a.data(), &lda, s.data(), &dummy, &ld1, &dummy, &ld1, work.data(),
                          &lwork, &info, 1, 1);
      double smin = 0.0;
      for (int i = k - 1; i >= 0; --i)
        if (s[i] > 0.0) {
          smin = s[i];
          break;
        }
      return smin > 0.0 ? s[0] / smin : 0.0;
    };
    if (cond_normal) *cond_normal = cond_of(A);
    if (o->pkind >= 0 && (precond_re || cond_precond)) {
      orc::Mat MA(n, n);
      for (int c = 0; c < n; ++c) {
        const orc::Vec col(A.col(c), A.col(c) + n);
        const orc::Vec z = orc::precond_apply(*o, col, false);
        std::copy(z.begin(), z.end(), MA.col(c));
      }
      if (cond_precond) *cond_precond = cond_of(MA);
      if (precond_re) {
        orc::Mat B = MA;
        orc::Vec wr(n), wi(n);
        double dummy = 0;
        int ld1 = 1, lwork = -1, info = 0, lda = n;
        double wq = 0;
        orc::g_lapack.geev("N", "N", &n, B.a.data(), &lda, wr.data(), wi.data(), &dummy, &ld1, &dummy, &ld1, &wq,
                           &lwork, &info, 1, 1);
        lwork = static_cast<int>(wq) + 1;
        orc::Vec work(lwork);
        orc::g_lapack.geev("N", "N", &n, B.a.data(), &lda, wr.data(), wi.data(), &dummy, &ld1, &dummy, &ld1,
                           work.data(), &lwork, &info, 1, 1);
        std::sort(wr.begin(), wr.end());
        std::copy(wr.begin(), wr.end(), precond_re);
      }
    }
  });
}

// ---- exports
int64_t orc_get_i(void* h, const char* what, int index, int32_t* out, int64_t cap) {
  Oracle* o = static_cast<Oracle*>(h);
  std::vector<int> v;
  const std::string w(what);
  if (w == "J") v = {o->dec.size()};
  else if (w == "N") v = {static_cast<int>(o->pts.size())};
  else if (w == "p") v = {o->p};
  else if (w == "dim") v = {o->dec.dim()};
  else if (w == "C") v = {o->prob.C};
  else if (w == "p_j") for (const auto& r : o->red) v.push_back(r.p);
  else if (w == "col_off") v = o->col_off;
  else if (w == "rows") v = index < static_cast<int>(o->rows.size()) && !o->rows.empty() ? o->rows[index] : orc::rows_of(*o, index);
  else if (w == "nbr") v = o->dec.nbr[index];
  else if (w == "nb_pairs") for (const auto& kv : o->nb) { v.push_back(kv.first.first); v.push_back(kv.first.second); }
  else if (w == "local_rank") for (const auto& L : o->loc) v.push_back(L.rank);
  else if (w == "set") v = o->sets[index];
  else if (w == "owner") v = o->owner;
  else if (w == "mult") v = o->mult;
  else if (w == "iterations") for (const auto& r : o->reports) v.push_back(r.iterations);
  else if (w == "converged") for (const auto& r : o->reports) v.push_back(r.converged ? 1 : 0);
  else { o->err = "unknown export " + w; return -1; }
  const int64_t n = static_cast<int64_t>(v.size());
  if (out) std::copy(v.begin(), v.begin() + std::min(n, cap), out);
  return n;
}

int64_t orc_get_d(void* h, const char* what, int index, double* out, int64_t cap) {
  Oracle* o = static_cast<Oracle*>(h);
  std::vector<double> v;
  const std::string w(what);
  if (w == "points") for (const auto& p : o->pts) for (int a = 0; a < o->dec.dim(); ++a) v.push_back(p[a]);
  else if (w == "box_lo") for (const auto& b : o->dec.sub) for (int a = 0; a < o->dec.dim(); ++a) v.push_back(b.lo[a]);
  else if (w == "box_hi") for (const auto& b : o->dec.sub) for (int a = 0; a < o->dec.dim(); ++a) v.push_back(b.hi[a]);
  else if (w == "R") v = o->bases[index].R.a;  // m x d column-major
  else if (w == "b") v = o->bases[index].b;
  else if (w == "S") v = o->samples[index].a;
  else if (w == "sigma") v = o->red[index].sigma;
  else if (w == "V") v = o->red[index].V.a;
  else if (w == "V_full") v = o->red[index].Vfull.a;
  else if (w == "H") v = o->H[index].a;
  else if (w == "F") v = o->F.a;
  else if (w == "scales") v = o->scales;
  else if (w == "nb") {
    int k = 0;
    for (const auto& kv : o->nb) { if (k++ == index) { v = kv.second.a; break; } }
  } else if (w == "nb_dense") v = orc::densify_nb(*o).a;
  else if (w == "H_dense") v = orc::densify(*o).a;
  else if (w == "local_cond") for (const auto& L : o->loc) v.push_back(L.cond);
  else if (w == "W") v.assign(o->W.col(index), o->W.col(index) + o->W.r);
  else if (w == "hist") v = o->reports[index].hist;
  else if (w == "true_hist") v = o->reports[index].true_hist;
  else if (w == "approx") v = o->approx.a;
  else if (w == "exact") v = o->exact.a;
  else { o->err = "unknown export " + w; return -1; }
  const int64_t n = static_cast<int64_t>(v.size());
  if (out) std::copy(v.begin(), v.begin() + std::min(n, cap), out);
  return n;
}

}  // extern "C"
