// host_setup.cpp — host half of build_instance (runner.hpp:40-70): problem descriptor,
// decomposition (geometry.hpp:109-177 or the BASELINE cell layout), collocation grid
// (geometry.hpp:200-232) and random bases (basis.hpp:33-48, random.hpp:9-37).
//
// These are O(J^2 + N) host computations whose outputs must be bit-identical to the
// reference's (they fix the point->subdomain indexing and the frozen weights), so they are
// computed here with the reference's operation order (compiled with -ffp-contract=off) and
// uploaded; everything downstream runs on the device.
#include <cmath>
#include <stdexcept>
#include <string>

#include "ctx.hpp"

namespace rdd {

namespace {

struct Mix {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double sym() { return 2.0 * (static_cast<double>(next() >> 11) * 0x1.0p-53) - 1.0; }
};

uint64_t subdomain_seed(uint64_t base, int j) {
  Mix m{base ^ (0xD1B54A32D192ED03ULL * static_cast<uint64_t>(j + 1))};
  return m.next();
}

constexpr double kPi = 3.14159265358979323846;

void set_coef_laplacian(ProblemDesc& P, double sign_h, double c_v) {
  for (auto& x : P.coef) x = 0.0;
  P.coef[0] = c_v;
  for (int a = 0; a < P.d; ++a) P.coef[1 + P.d + hess_index(a, a, P.d)] = sign_h;
}

ProblemDesc make_desc(const rdd_config& cfg) {
  ProblemDesc P;
  P.id = cfg.problem;
  P.n = cfg.n;
  switch (cfg.problem) {
    case RDD_PROBLEM_EXAMPLE1:
      if (cfg.n < 1 || cfg.n > 8) throw std::invalid_argument("example1: n must be in [1,8]");
      P.d = 2;
      set_coef_laplacian(P, -1.0, 0.0);  // operators.hpp:19-25
      break;
    case RDD_PROBLEM_EXAMPLE2:
      P.d = 2;
      P.lo[0] = -1.0;
      for (auto& x : P.coef) x = 0.0;  // operators.hpp:37-41: u_t + u_x - kappa u_xx
      P.coef[1] = 1.0;
      P.coef[2] = 1.0;
      P.coef[3] = -(0.1 / kPi);
      P.has_exact = false;
      break;
    case RDD_PROBLEM_EXAMPLE3:
      P.d = 3;
      P.C = 3;
      set_coef_laplacian(P, -1.0, 1.0);  // operators.hpp:28-34
      break;
    case RDD_PROBLEM_POISSON:
      P.d = cfg.dim == 0 ? 2 : cfg.dim;
      if (P.d < 1 || P.d > 3) throw std::invalid_argument("poisson: dimension must be 1..3");
      set_coef_laplacian(P, -1.0, 0.0);
      break;
    case RDD_PROBLEM_MULTISCALE:
      P.d = 2;
      set_coef_laplacian(P, -1.0, 0.0);
      break;
    case RDD_PROBLEM_HEAT:  // u_t - 0.1 (u_xx + u_yy)
      P.d = 3;
      for (auto& x : P.coef) x = 0.0;
      P.coef[3] = 1.0;
      P.coef[1 + 3 + hess_index(0, 0, 3)] = -0.1;
      P.coef[1 + 3 + hess_index(1, 1, 3)] = -0.1;
      break;
    case RDD_PROBLEM_ADVECTION:  // u_t + 2 u_x on [0,2] x [0,1]
      P.d = 2;
      P.hi[0] = 2.0;
      for (auto& x : P.coef) x = 0.0;
      P.coef[1] = 2.0;
      P.coef[2] = 1.0;
      break;
    default:
      throw std::invalid_argument("unknown problem id " + std::to_string(cfg.problem));
  }
  return P;
}

bool interiors_intersect(const Ctx& c, int i, int j) {  // geometry.hpp:99-105
  for (int a = 0; a < c.d; ++a) {
    const double lo = std::max(c.box_lo[i * 4 + a], c.box_lo[j * 4 + a]);
    const double hi = std::min(c.box_hi[i * 4 + a], c.box_hi[j * 4 + a]);
    if (!(lo < hi)) return false;
  }
  return true;
}

}  // namespace

// problems.hpp:219-264 reference_example2: space-time Crank-Nicolson field of example2 on a
// res x res grid (level-major), Thomas elimination with the constant coefficients factored once.
// Host-side like the reference (it is the error yardstick, not part of the solve), same operation
// order so the device's bilinear lookups see the identical field.
void reference_example2_grid(int res, std::vector<double>& v) {
  if (res < 501) throw std::invalid_argument("reference_example2: resolution must be >= 501");
  const int nx = res, nt = res, ni = nx - 2;
  const double h = 2.0 / static_cast<double>(nx - 1), dt = 1.0 / static_cast<double>(nt - 1);
  const double kappa = 0.1 / kPi;
  const double a = kappa * dt / (2.0 * h * h), c = dt / (4.0 * h);
  v.assign(static_cast<size_t>(nx) * nt, 0.0);
  for (int i = 0; i < nx; ++i) v[i] = -std::sin(kPi * (-1.0 + i * h));
  v[0] = 0.0;
  v[nx - 1] = 0.0;
  const double lo = -(a + c), di = 1.0 + 2.0 * a, up = -(a - c);
  std::vector<double> cp(ni), rhs(ni), dp(ni);
  cp[0] = up / di;
  for (int i = 1; i < ni; ++i) cp[i] = up / (di - lo * cp[i - 1]);
  for (int step = 1; step < nt; ++step) {
    const double* prev = v.data() + static_cast<size_t>(step - 1) * nx;
    double* next = v.data() + static_cast<size_t>(step) * nx;
    for (int i = 0; i < ni; ++i) rhs[i] = (a + c) * prev[i] + (1.0 - 2.0 * a) * prev[i + 1] + (a - c) * prev[i + 2];
    dp[0] = rhs[0] / di;
    for (int i = 1; i < ni; ++i) dp[i] = (rhs[i] - lo * dp[i - 1]) / (di - lo * cp[i - 1]);
    next[ni] = dp[ni - 1];
    for (int i = ni - 2; i >= 0; --i) next[i + 1] = dp[i] - cp[i] * next[i + 2];
    next[0] = 0.0;
    next[nx - 1] = 0.0;
  }
}

void setup_problem(Ctx& c, const rdd_config& cfg, uint64_t seed) {
  c.cfg = cfg;
  c.seed = seed;
  c.prob = make_desc(cfg);
  const int d = c.d = c.prob.d;
  c.C = c.prob.C;
  c.jl = jet_len(d);
  c.m = cfg.m;
  if (cfg.m < 1) throw std::invalid_argument("hidden width m must be >= 1");
  if (cfg.dim != 0 && cfg.dim != d)  // runner.hpp:45
    throw std::invalid_argument("decomposition counts have dimension " + std::to_string(cfg.dim) +
                                " but the problem has dimension " + std::to_string(d));
  if (cfg.tau_mode != RDD_TAU_OFF && !(cfg.tau >= 0.0))  // reduction.hpp:90
    throw std::invalid_argument("truncation threshold tau must be >= 0");
  if (cfg.max_iter < 0) throw std::invalid_argument("max_iter must be >= 1");  // krylov.hpp:79
  if (cfg.op_form != RDD_OPERATOR_TWO_PASS && cfg.op_form != RDD_OPERATOR_NORMAL)
    throw std::invalid_argument("unknown normal-operator form");
  c.counts.assign(cfg.counts, cfg.counts + d);
  for (int k : c.counts)
    if (k < 1) throw std::invalid_argument("per-axis subdomain counts must be >= 1");

  // ---- per-axis centres / half widths
  std::vector<std::vector<double>> ac(d);
  std::vector<double> ah(d);
  for (int a = 0; a < d; ++a) {
    const int l = c.counts[a];
    const double lo = c.prob.lo[a], len = c.prob.hi[a] - c.prob.lo[a];
    if (l == 1) {
      ac[a] = {lo + 0.5 * len};
      ah[a] = 0.5 * len;
    } else if (cfg.decomposition == RDD_DECOMP_REFERENCE) {  // geometry.hpp:125-137
      if (!(cfg.delta > 1.0)) throw std::invalid_argument("overlap ratio delta must exceed 1");
      ah[a] = (cfg.delta / 2.0) / static_cast<double>(l - 1) * len;
      for (int j = 0; j < l; ++j) ac[a].push_back(lo + static_cast<double>(j) / static_cast<double>(l - 1) * len);
    } else {  // cell-centred, extended by delta x width per side
      if (!(cfg.delta > 0.0)) throw std::invalid_argument("cell decomposition extension must be positive");
      ah[a] = (0.5 + cfg.delta) / static_cast<double>(l) * len;
      for (int j = 0; j < l; ++j) ac[a].push_back(lo + (static_cast<double>(j) + 0.5) / static_cast<double>(l) * len);
    }
  }
  int total = 1;
  for (int k : c.counts) total *= k;
  c.J = total;
  c.box_lo.assign(total * 4, 0.0);
  c.box_hi.assign(total * 4, 0.0);
  c.box_c.assign(total * 4, 0.0);
  c.box_h.assign(total * 4, 0.0);
  c.axis_lo.assign(d, {});
  c.axis_hi.assign(d, {});
  for (int a = 0; a < d; ++a)
    for (size_t k = 0; k < ac[a].size(); ++k) {
      c.axis_lo[a].push_back(ac[a][k] - ah[a]);
      c.axis_hi[a].push_back(ac[a][k] + ah[a]);
    }
  std::vector<int> idx(d, 0);
  for (int flat = 0; flat < total; ++flat) {  // axis 0 slowest (geometry.hpp:146-167)
    for (int a = 0; a < d; ++a) {
      const double cc = ac[a][idx[a]], hh = ah[a];
      c.box_c[flat * 4 + a] = cc;
      c.box_h[flat * 4 + a] = hh;
      c.box_lo[flat * 4 + a] = cc - hh;
      c.box_hi[flat * 4 + a] = cc + hh;
    }
    for (int a = d - 1; a >= 0; --a) {
      if (++idx[a] < c.counts[a]) break;
      idx[a] = 0;
    }
  }
  // neighbour sets (geometry.hpp:169-174): per-axis interval overlap in the tensor product
  c.nbr_ptr.assign(total + 1, 0);
  c.nbr_idx.clear();
  for (int i = 0; i < total; ++i) {
    for (int j = 0; j < total; ++j)
      if (interiors_intersect(c, i, j)) c.nbr_idx.push_back(j);
    c.nbr_ptr[i + 1] = static_cast<int>(c.nbr_idx.size());
  }

  // ---- collocation points (geometry.hpp:200-232) + optional edge points
  std::vector<int> res(cfg.colloc, cfg.colloc + d);
  for (int r : res)
    if (r < 1) throw std::invalid_argument("grid resolutions must be >= 1");
  long long n = 1;
  for (int r : res) n *= r;
  const int nb = cfg.boundary_per_edge;
  if (nb > 0 && d != 2) throw std::invalid_argument("boundary points are defined for 2-D domains only");
  const long long Ntot = n + (nb > 0 ? 4LL * nb : 0);
  if (Ntot > 2000000000LL) throw std::invalid_argument("too many collocation points");
  c.N = static_cast<int>(Ntot);
  c.h_pts.resize(static_cast<size_t>(d) * c.N);  // every entry is written below
  std::vector<double> step(d);
  std::vector<long long> stride(d, 1);
  for (int a = 0; a < d; ++a) step[a] = (c.prob.hi[a] - c.prob.lo[a]) / static_cast<double>(res[a]);
  for (int a = d - 2; a >= 0; --a) stride[a] = stride[a + 1] * res[a + 1];
  // last axis fastest; index of axis a = (flat / stride_a) mod res_a — the same coordinate formula
  // as the reference's incremental counters, evaluated per point so the host threads split the grid
  double* hp = c.h_pts.data();
  const long long NN = c.N;
#pragma omp parallel for schedule(static)
  for (long long flat = 0; flat < n; ++flat)
    for (int a = 0; a < d; ++a) {
      const long long g = (flat / stride[a]) % res[a];
      hp[a * NN + flat] = c.prob.lo[a] + (static_cast<double>(g) + 0.5) * step[a];
    }
  if (nb > 0) {
    long long q = n;
    for (int e = 0; e < 4; ++e) {
      const int axis = e < 2 ? 0 : 1, fixed = 1 - axis;
      const double fv = (e % 2 == 0) ? c.prob.lo[fixed] : c.prob.hi[fixed];
      const double st = (c.prob.hi[axis] - c.prob.lo[axis]) / static_cast<double>(nb);
      for (int k = 0; k < nb; ++k, ++q) {
        c.h_pts[static_cast<size_t>(axis) * c.N + q] = c.prob.lo[axis] + (static_cast<double>(k) + 0.5) * st;
        c.h_pts[static_cast<size_t>(fixed) * c.N + q] = fv;
      }
    }
  }

  // ---- random bases: R (m x d, drawn k-major then axis) then b (basis.hpp:43-46)
  c.h_R.assign(static_cast<size_t>(total) * c.m * d, 0.0);
  c.h_b.assign(static_cast<size_t>(total) * c.m, 0.0);
#pragma omp parallel for schedule(static)
  for (int j = 0; j < total; ++j) {
    Mix rng{subdomain_seed(seed, j)};
    for (int k = 0; k < c.m; ++k)
      for (int a = 0; a < d; ++a) c.h_R[(static_cast<size_t>(j) * c.m + k) * d + a] = rng.sym();
    for (int k = 0; k < c.m; ++k) c.h_b[static_cast<size_t>(j) * c.m + k] = rng.sym();
  }
}


// The instance from caller inputs (rdd_set_*): the reference's CartesianDecomposition (boxes,
// centres, half widths, neighbour sets as build_decomposition made them, geometry.hpp:109-177),
// its PointSet and RandomBasis objects, and a ProblemSpec evaluated at the points by the caller.
// The decomposition must be a tensor product (box j's interval on axis a depends only on j's
// axis-a index, axis 0 slowest), as every CartesianDecomposition is.
void setup_custom(Ctx& c, const rdd_config& cfg) {
  CustomInputs& u = c.custom;
  if (!u.has_dec || !u.has_pts || !u.has_bases || !u.has_problem)
    throw std::invalid_argument("custom instance: set the decomposition, points, bases and problem first");
  const int d = u.d;
  int total = 1;
  for (int k : u.counts) total *= k;
  if (static_cast<int>(u.R.size()) != total * u.m * d) throw std::invalid_argument("custom bases: one per subdomain");
  const long long N = static_cast<long long>(u.pts.size()) / d;
  if (static_cast<long long>(u.Ljet.size()) != N * jet_len(d))
    throw std::invalid_argument("custom problem: L jets must be given at every collocation point");
  c.cfg = cfg;
  c.seed = cfg.seed;
  c.prob = ProblemDesc{};
  c.prob.id = 0;
  c.prob.d = d;
  c.prob.C = u.C;
  c.prob.has_exact = false;
  for (int a = 0; a < d; ++a) {
    c.prob.lo[a] = u.dom_lo[a];
    c.prob.hi[a] = u.dom_hi[a];
  }
  for (int k = 0; k < jet_len(d); ++k) c.prob.coef[k] = u.coef[k];
  c.d = d;
  c.C = u.C;
  c.jl = jet_len(d);
  c.m = u.m;
  c.cfg.m = u.m;
  c.cfg.activation = u.act;
  c.cfg.dim = d;
  for (int a = 0; a < d; ++a) c.cfg.counts[a] = u.counts[a];
  if (cfg.tau_mode != RDD_TAU_OFF && !(cfg.tau >= 0.0))  // reduction.hpp:90
    throw std::invalid_argument("truncation threshold tau must be >= 0");
  if (cfg.max_iter < 0) throw std::invalid_argument("max_iter must be >= 1");  // krylov.hpp:79
  c.counts = u.counts;
  c.J = total;
  c.box_lo.assign(total * 4, 0.0);
  c.box_hi.assign(total * 4, 0.0);
  c.box_c.assign(total * 4, 0.0);
  c.box_h.assign(total * 4, 0.0);
  c.axis_lo.assign(d, std::vector<double>());
  c.axis_hi.assign(d, std::vector<double>());
  for (int a = 0; a < d; ++a) {
    c.axis_lo[a].assign(u.counts[a], 0.0);
    c.axis_hi[a].assign(u.counts[a], 0.0);
  }
  std::vector<int> idx(d, 0);
  std::vector<std::vector<char>> seen(d);
  for (int a = 0; a < d; ++a) seen[a].assign(u.counts[a], 0);
  for (int j = 0; j < total; ++j) {
    for (int a = 0; a < d; ++a) {
      const size_t q = static_cast<size_t>(j) * d + a;
      c.box_lo[j * 4 + a] = u.lo[q];
      c.box_hi[j * 4 + a] = u.hi[q];
      c.box_c[j * 4 + a] = u.ctr[q];
      c.box_h[j * 4 + a] = u.half[q];
      if (!seen[a][idx[a]]) {
        c.axis_lo[a][idx[a]] = u.lo[q];
        c.axis_hi[a][idx[a]] = u.hi[q];
        seen[a][idx[a]] = 1;
      } else if (c.axis_lo[a][idx[a]] != u.lo[q] || c.axis_hi[a][idx[a]] != u.hi[q]) {
        throw std::invalid_argument("custom decomposition: boxes are not a tensor product (axis 0 slowest)");
      }
    }
    for (int a = d - 1; a >= 0; --a) {
      if (++idx[a] < u.counts[a]) break;
      idx[a] = 0;
    }
  }
  c.nbr_ptr = u.nbr_ptr;
  c.nbr_idx = u.nbr_idx;
  if (static_cast<int>(c.nbr_ptr.size()) != total + 1)
    throw std::invalid_argument("custom decomposition: one neighbour set per subdomain");
  if (N > 2000000000LL) throw std::invalid_argument("too many collocation points");
  c.N = static_cast<int>(N);
  c.h_pts.resize(static_cast<size_t>(d) * c.N);
  for (long long i = 0; i < N; ++i)
    for (int a = 0; a < d; ++a) c.h_pts[static_cast<size_t>(a) * N + i] = u.pts[static_cast<size_t>(i) * d + a];
  c.h_R.assign(u.R.begin(), u.R.end());
  c.h_b.assign(u.b.begin(), u.b.end());
}

}  // namespace rdd
