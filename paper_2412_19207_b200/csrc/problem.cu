// problem.cu — device closed forms of the problem closures (problems.hpp:28-173 and the
// BASELINE configs of SURVEY §8d): per collocation point the jet of the constraint L(x)
// (basis.hpp:185-190) and the right-hand side F_c = f_c(x) - A[G_c](x) (assembly.hpp:97-106).
//
// Every L and G here is a product (or, for C4's G, a sum) of univariate factors, so the jets
// are formed from per-axis (f, f', f'') triples; the operator acts on a jet as the coefficient
// vector c·jet (operators.hpp:13-41 are all constant-coefficient).
#include "ctx.hpp"

namespace rdd {

namespace {

constexpr double kPi = 3.14159265358979323846;

struct T3 {
  double f, d1, d2;
};
__device__ __forceinline__ T3 t_one() { return {1.0, 0.0, 0.0}; }
__device__ __forceinline__ T3 t_tanh(double x, double al, double be) {  // tanh(al x + be)
  const double t = tanh(al * x + be);
  const double s2 = 1.0 - t * t;
  return {t, al * s2, al * al * (-2.0 * t * s2)};
}
__device__ __forceinline__ T3 t_sin(double x, double al, double be) {
  double s, c;
  sincos(al * x + be, &s, &c);
  return {s, al * c, -al * al * s};
}
__device__ __forceinline__ T3 t_cos(double x, double al, double be) {
  double s, c;
  sincos(al * x + be, &s, &c);
  return {c, -al * s, -al * al * c};
}
__device__ __forceinline__ T3 t_gauss(double x, double al, double be) {  // exp(-100 (al x + be)^2)
  const double q = al * x + be;
  const double e = exp(-100.0 * (q * q));
  const double dq = -200.0 * q * al;
  return {e, e * dq, e * (dq * dq - 200.0 * al * al)};
}
__device__ __forceinline__ T3 t_mul(T3 a, T3 b) {
  return {a.f * b.f, a.d1 * b.f + a.f * b.d1, a.d2 * b.f + 2.0 * a.d1 * b.d1 + a.f * b.d2};
}

// jet of prod_a F_a(x_a)
__device__ Jet product_jet(const T3* F, int d) {
  Jet o;
  double v = 1.0;
  for (int a = 0; a < d; ++a) v *= F[a].f;
  o.c[0] = v;
  for (int a = 0; a < d; ++a) {
    double g = F[a].d1;
    for (int b = 0; b < d; ++b)
      if (b != a) g *= F[b].f;
    o.c[1 + a] = g;
  }
  for (int a = 0; a < d; ++a)
    for (int b = a; b < d; ++b) {
      double h = (a == b) ? F[a].d2 : F[a].d1 * F[b].d1;
      for (int e = 0; e < d; ++e)
        if (e != a && e != b) h *= F[e].f;
      o.c[1 + d + hess_index(a, b, d)] = h;
    }
  return o;
}

__device__ __forceinline__ double apply_op(const double* coef, const Jet& u, int jl) {
  double s = 0.0;
  for (int k = 0; k < jl; ++k)
    if (coef[k] != 0.0) s += coef[k] * u.c[k];
  return s;
}

struct DevProblem {
  int id, d, C, n;
  double coef[kMaxJet];
};

__device__ Jet L_jet(const DevProblem& P, const double* x) {
  T3 F[kMaxDim];
  const int d = P.d;
  switch (P.id) {
    case RDD_PROBLEM_EXAMPLE1: {  // problems.hpp:78-82, rho = 2^-n
      const double inv = ldexp(1.0, P.n);  // 1/rho
      for (int a = 0; a < 2; ++a) F[a] = t_mul(t_tanh(x[a], inv, 0.0), t_tanh(x[a], -inv, inv));
      break;
    }
    case RDD_PROBLEM_EXAMPLE2:  // problems.hpp:98-101
      F[0] = t_mul(t_tanh(x[0], 1.0, 1.0), t_tanh(x[0], -1.0, 1.0));
      F[1] = t_tanh(x[1], 1.0, 0.0);
      break;
    case RDD_PROBLEM_HEAT:  // tanh x tanh(1-x) tanh y tanh(1-y) tanh t
      F[0] = t_mul(t_tanh(x[0], 1.0, 0.0), t_tanh(x[0], -1.0, 1.0));
      F[1] = t_mul(t_tanh(x[1], 1.0, 0.0), t_tanh(x[1], -1.0, 1.0));
      F[2] = t_tanh(x[2], 1.0, 0.0);
      break;
    case RDD_PROBLEM_ADVECTION:  // tanh x tanh t
      F[0] = t_tanh(x[0], 1.0, 0.0);
      F[1] = t_tanh(x[1], 1.0, 0.0);
      break;
    default:  // example3 / poisson / multiscale: prod_a tanh(x_a) tanh(1 - x_a) (problems.hpp:145-151)
      for (int a = 0; a < d; ++a) F[a] = t_mul(t_tanh(x[a], 1.0, 0.0), t_tanh(x[a], -1.0, 1.0));
      break;
  }
  return product_jet(F, d);
}

// F_c(x) = f_c(x) - A[G_c](x)
__device__ double rhs_value(const DevProblem& P, const double* x, int comp) {
  const int d = P.d, jl = jet_len(d);
  switch (P.id) {
    case RDD_PROBLEM_EXAMPLE1: {  // problems.hpp:69-76, G = 0
      double s = 0.0;
      for (int i = 1; i <= P.n; ++i) {
        const double wp = ldexp(1.0, i) * kPi;
        s += 2.0 * wp * wp * sin(wp * x[0]) * sin(wp * x[1]);
      }
      return (1.0 / static_cast<double>(P.n)) * s;
    }
    case RDD_PROBLEM_EXAMPLE2: {  // f = 0, G = -sin(pi x)
      T3 F[2] = {t_sin(x[0], kPi, 0.0), t_one()};
      F[0].f = -F[0].f;
      F[0].d1 = -F[0].d1;
      F[0].d2 = -F[0].d2;
      return -apply_op(P.coef, product_jet(F, 2), jl);
    }
    case RDD_PROBLEM_EXAMPLE3: {  // f_c = A[u_c], G_c = prod_{a != c} sin(2 pi x_a)
      const double w = 2.0 * kPi;
      T3 E[3], G[3];
      for (int a = 0; a < 3; ++a) {
        E[a] = (a == comp) ? t_cos(x[a], w, 0.0) : t_sin(x[a], w, 0.0);
        G[a] = (a == comp) ? t_one() : t_sin(x[a], w, 0.0);
      }
      return apply_op(P.coef, product_jet(E, 3), jl) - apply_op(P.coef, product_jet(G, 3), jl);
    }
    case RDD_PROBLEM_POISSON: {
      double s = 1.0;
      for (int a = 0; a < d; ++a) s *= sin(kPi * x[a]);
      return (static_cast<double>(d) * kPi * kPi) * s;
    }
    case RDD_PROBLEM_MULTISCALE:
      return (8.0 * kPi * kPi) * (sin(2.0 * kPi * x[0]) * sin(2.0 * kPi * x[1])) +
             (500.0 * kPi * kPi) * (sin(50.0 * kPi * x[0]) * sin(50.0 * kPi * x[1]));
    case RDD_PROBLEM_HEAT: {  // f = 0, G = sin(pi x) sin(pi y)
      T3 F[3] = {t_sin(x[0], kPi, 0.0), t_sin(x[1], kPi, 0.0), t_one()};
      return -apply_op(P.coef, product_jet(F, 3), jl);
    }
    case RDD_PROBLEM_ADVECTION: {  // f = 0, G = u0(x) + g(t) - u0(0)
      const T3 u0 = t_gauss(x[0], 1.0, -0.5), g = t_gauss(x[1], 2.0, 0.5);
      Jet G;
      jet_zero(G, 2);
      G.c[0] = (u0.f + g.f) - exp(-25.0);
      G.c[1] = u0.d1;
      G.c[2] = g.d1;
      G.c[3] = u0.d2;
      G.c[5] = g.d2;
      return -apply_op(P.coef, G, jl);
    }
  }
  return 0.0;
}

__global__ void k_eval_problem(DevProblem P, const double* __restrict__ pts, int N, double* __restrict__ Ljet,
                               double* __restrict__ F, int* __restrict__ bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double x[kMaxDim] = {0, 0, 0, 0};
  for (int a = 0; a < P.d; ++a) x[a] = pts[static_cast<size_t>(a) * N + i];
  const int jl = jet_len(P.d);
  const Jet L = L_jet(P, x);
  for (int k = 0; k < jl; ++k) Ljet[static_cast<size_t>(i) * jl + k] = L.c[k];
  for (int c = 0; c < P.C; ++c) {
    const double v = rhs_value(P, x, c);
    if (!isfinite(v)) atomicMin(bad, i);
    F[static_cast<size_t>(c) * N + i] = v;
  }
}

}  // namespace

// Device-side evaluation of L jets and F (assembly.hpp:97-106 for F).
void eval_problem(Ctx& c) {
  ScopedKernelTimer tk(c, "problem");
  DevProblem P{};
  P.id = c.prob.id;
  P.d = c.d;
  P.C = c.C;
  P.n = c.prob.n;
  for (int k = 0; k < kMaxJet; ++k) P.coef[k] = c.prob.coef[k];
  c.Ljet.ensure(static_cast<size_t>(c.N) * c.jl);
  c.Fpt.ensure(static_cast<size_t>(c.N) * c.C);
  DBuf<int> bad;
  bad.ensure(1);
  const int big = INT32_MAX;
  bad.upload(&big, 1, c.stream);
  k_eval_problem<<<ceil_div(c.N, 256), 256, 0, c.stream>>>(P, c.pts.p, c.N, c.Ljet.p, c.Fpt.p, bad.p);
  RDD_LAUNCH_CHECK();
  int h_bad = 0;
  bad.download(&h_bad, 1, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  if (h_bad != INT32_MAX)
    throw std::runtime_error("non-finite right-hand side at collocation point " + std::to_string(h_bad));
}

// Caller-evaluated problem (CustomInputs): L jets and F = f − A[G] at the collocation points,
// in place of eval_problem; same layouts (Ljet point-major, F column-major per component).
void upload_custom_problem(Ctx& c) {
  const CustomInputs& u = c.custom;
  for (size_t q = 0; q < u.F.size(); ++q)
    if (!std::isfinite(u.F[q]))
      throw std::runtime_error("non-finite right-hand side at collocation point " + std::to_string(q % c.N));
  if (static_cast<long long>(u.F.size()) != static_cast<long long>(c.N) * c.C)
    throw std::invalid_argument("custom problem: F must have N x C entries");
  c.Ljet.upload(u.Ljet.data(), u.Ljet.size(), c.stream);
  c.Fpt.upload(u.F.data(), u.F.size(), c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace rdd

// ---------------------------------------------------------------- K14: evaluation (runner.hpp:105-144)
namespace rdd {
namespace {

__device__ double exact_value(const DevProblem& P, const double* x, int comp) {
  switch (P.id) {
    case RDD_PROBLEM_EXAMPLE1: {
      double s = 0.0;
      for (int i = 1; i <= P.n; ++i) {
        const double w = ldexp(1.0, i);
        s += sin(w * kPi * x[0]) * sin(w * kPi * x[1]);
      }
      return (1.0 / static_cast<double>(P.n)) * s;
    }
    case RDD_PROBLEM_EXAMPLE3: {
      const double w = 2.0 * kPi;
      double v = 1.0;
      for (int a = 0; a < 3; ++a) v *= (a == comp) ? cos(w * x[a]) : sin(w * x[a]);
      return v;
    }
    case RDD_PROBLEM_POISSON: {
      double s = 1.0;
      for (int a = 0; a < P.d; ++a) s *= sin(kPi * x[a]);
      return s;
    }
    case RDD_PROBLEM_MULTISCALE:
      return sin(2.0 * kPi * x[0]) * sin(2.0 * kPi * x[1]) + 0.1 * (sin(50.0 * kPi * x[0]) * sin(50.0 * kPi * x[1]));
    case RDD_PROBLEM_HEAT:
      return exp(-0.2 * kPi * kPi * x[2]) * (sin(kPi * x[0]) * sin(kPi * x[1]));
    case RDD_PROBLEM_ADVECTION: {
      const double q = x[0] - 2.0 * x[1] - 0.5;
      return exp(-100.0 * (q * q));
    }
  }
  return 0.0;
}

__device__ double G_value(const DevProblem& P, const double* x, int comp) {
  switch (P.id) {
    case RDD_PROBLEM_EXAMPLE2: return -sin(kPi * x[0]);
    case RDD_PROBLEM_EXAMPLE3: {
      double v = 1.0;
      for (int a = 0; a < 3; ++a)
        if (a != comp) v *= sin(2.0 * kPi * x[a]);
      return v;
    }
    case RDD_PROBLEM_HEAT: return sin(kPi * x[0]) * sin(kPi * x[1]);
    case RDD_PROBLEM_ADVECTION: {
      const double q0 = x[0] - 0.5, q1 = 2.0 * x[1] + 0.5;
      return (exp(-100.0 * (q0 * q0)) + exp(-100.0 * (q1 * q1))) - exp(-25.0);
    }
  }
  return 0.0;
}

struct EvalArgs {
  DevProblem P;
  int J, m, act, M;
  int res[kMaxDim];
  double lo[kMaxDim], step[kMaxDim];
  const double* box;      // J x 16
  const int* counts1;
  const int* nbr_ptr;
  const int* nbr_idx;
  const double* R;
  const double* b;
  const double* U;        // J x m x C effective output weights u_j = V_j W_j
  double* approx;         // M x C
  double* exact;
  const double* ref;      // example2: reference field (refn x refn), else null
  int refn;
  const double* ax_lo;    // per-axis box intervals: the covering boxes of a test point
  const double* ax_hi;
  int ax_counts[kMaxDim], ax_stride[kMaxDim], ax_off[kMaxDim];
  const double* xin;      // caller points (M x d, point after point), or null: the test grid
  const double* Lin;      // caller L values (M) with xin
  const double* Gin;      // caller G values (M x C) with xin, or null (G = 0)
};

// problems.hpp:203-216 ReferenceGrid::at: bilinear lookup in the space-time field
__device__ double ref_at(const double* v, int n, double x, double t) {
  const double h = 2.0 / static_cast<double>(n - 1);
  const double dt = 1.0 / static_cast<double>(n - 1);
  const double fx = (x + 1.0) / h, ft = t / dt;
  int ix = static_cast<int>(floor(fx)), it = static_cast<int>(floor(ft));
  ix = min(max(ix, 0), n - 2);
  it = min(max(it, 0), n - 2);
  const double ax = fx - ix, at_ = ft - it;
  const double v00 = v[static_cast<size_t>(it) * n + ix], v01 = v[static_cast<size_t>(it) * n + ix + 1];
  const double v10 = v[static_cast<size_t>(it + 1) * n + ix], v11 = v[static_cast<size_t>(it + 1) * n + ix + 1];
  // unfused products and sums (the reference's host arithmetic): bit-identical field values
  const double bx = 1.0 - ax, bt = 1.0 - at_;
  const double r0 = __dadd_rn(__dmul_rn(bx, v00), __dmul_rn(ax, v01));
  const double r1 = __dadd_rn(__dmul_rn(bx, v10), __dmul_rn(ax, v11));
  return __dadd_rn(__dmul_rn(bt, r0), __dmul_rn(at_, r1));
}

__device__ __forceinline__ double raw_wv(const EvalArgs& A, int k, const double* x) {
  const double* bx = A.box + 16 * static_cast<size_t>(k);
  for (int a = 0; a < A.P.d; ++a)
    if (x[a] < bx[a] || x[a] > bx[4 + a]) return 0.0;
  double prod = 1.0;
  for (int a = 0; a < A.P.d; ++a) {
    if (A.counts1[a]) continue;
    const double s = (x[a] - bx[8 + a]) / bx[12 + a];
    const double base = 1.0 + cos(kPi * s);
    prod *= base * base;
  }
  return prod;
}

__global__ void k_evaluate(EvalArgs A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.M) return;
  const int d = A.P.d;
  double x[kMaxDim] = {0, 0, 0, 0};
  if (A.xin) {
    for (int a = 0; a < d; ++a) x[a] = A.xin[static_cast<size_t>(i) * d + a];
  } else {
    int rem = i;
    for (int a = d - 1; a >= 0; --a) {  // last axis fastest (geometry.hpp:216-230)
      const int k = rem % A.res[a];
      rem /= A.res[a];
      // unfused, as uniform_grid computes it on the host: bit-identical test points
      x[a] = __dadd_rn(A.lo[a], __dmul_rn(static_cast<double>(k) + 0.5, A.step[a]));
    }
  }
  const double Lv = A.xin ? A.Lin[i] : L_jet(A.P, x).c[0];
  double acc[3] = {0.0, 0.0, 0.0};
  // covering boxes (geometry.hpp:180-185): per-axis closed-interval candidates, enumerated as the
  // lexicographic product (axis 0 slowest) = ascending j, the reference's accumulation order
  int cand[kMaxDim][8], nc[kMaxDim];
  bool any = true, full = false;  // full: more than 8 candidates on an axis -> scan every box
  for (int a = 0; a < d && any; ++a) {
    nc[a] = 0;
    for (int k = 0; k < A.ax_counts[a]; ++k) {
      const double lo = A.ax_lo[A.ax_off[a] + k], hi = A.ax_hi[A.ax_off[a] + k];
      if (!(x[a] < lo || x[a] > hi)) {
        if (nc[a] < 8) cand[a][nc[a]++] = k;
        else full = true;
      }
    }
    any = nc[a] > 0;
  }
  int itc[kMaxDim] = {0, 0, 0, 0};
  int jf = 0;
  for (bool more = full || any; more;) {
    int j = 0;
    if (full) {
      j = jf++;
      more = jf < A.J;
    } else {
      for (int a = 0; a < d; ++a) j += cand[a][itc[a]] * A.ax_stride[a];
      int a = d - 1;
      for (; a >= 0; --a) {
        if (++itc[a] < nc[a]) break;
        itc[a] = 0;
      }
      more = a >= 0;
    }
    const double wj = raw_wv(A, j, x);
    if (wj == 0.0) continue;  // covering_subdomains + zero window (basis.hpp:169-176)
    double tot = 0.0;
    for (int q = A.nbr_ptr[j]; q < A.nbr_ptr[j + 1]; ++q) tot += raw_wv(A, A.nbr_idx[q], x);
    const double w = wj / tot;
    const double* bx = A.box + 16 * static_cast<size_t>(j);
    double xh[kMaxDim];
    for (int a = 0; a < d; ++a) xh[a] = 2.0 * (x[a] - 0.5 * (bx[a] + bx[4 + a])) / (bx[4 + a] - bx[a]);
    double s[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < A.m; ++k) {
      double z = A.b[static_cast<size_t>(j) * A.m + k];
      for (int a = 0; a < d; ++a) z += A.R[(static_cast<size_t>(j) * A.m + k) * d + a] * xh[a];
      const double ph = A.act == 0 ? tanh(z) : sin(z);
      for (int cc = 0; cc < A.P.C; ++cc) s[cc] += A.U[(static_cast<size_t>(cc) * A.J + j) * A.m + k] * ph;
    }
    for (int cc = 0; cc < A.P.C; ++cc) acc[cc] += s[cc] * (Lv * w);
  }
  for (int cc = 0; cc < A.P.C; ++cc) {
    if (A.xin) {
      A.approx[static_cast<size_t>(cc) * A.M + i] = acc[cc] + (A.Gin ? A.Gin[static_cast<size_t>(cc) * A.M + i] : 0.0);
      continue;
    }
    A.approx[static_cast<size_t>(cc) * A.M + i] = acc[cc] + G_value(A.P, x, cc);
    A.exact[static_cast<size_t>(cc) * A.M + i] = A.ref ? ref_at(A.ref, A.refn, x[0], x[1]) : exact_value(A.P, x, cc);
  }
}

// u_j = V_j W_j (m x p_j times p_j), per component; identity V copies W
__global__ void k_effective_weights(const double* __restrict__ Vred, const double* __restrict__ W,
                                    const int* __restrict__ col_off, int J, int m, int p, int identity,
                                    double* __restrict__ U, int C) {
  const int j = blockIdx.x;
  const int c0 = col_off[j], pj = col_off[j + 1] - c0;
  for (int cc = 0; cc < C; ++cc)
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
      double s = 0.0;
      if (identity) {
        s = k < pj ? W[static_cast<size_t>(cc) * p + c0 + k] : 0.0;
      } else {
        for (int q = 0; q < pj; ++q)
          s += Vred[(static_cast<size_t>(j) * m + q) * m + k] * W[static_cast<size_t>(cc) * p + c0 + q];
      }
      U[(static_cast<size_t>(cc) * J + j) * m + k] = s;
    }
}

}  // namespace

static void eval_common(Ctx& c, EvalArgs& A, DBuf<int>& counts1) {
  A.P.id = c.prob.id;
  A.P.d = c.d;
  A.P.C = c.C;
  A.P.n = c.prob.n;
  for (int k = 0; k < kMaxJet; ++k) A.P.coef[k] = c.prob.coef[k];
  A.J = c.J;
  A.m = c.m;
  A.act = c.cfg.activation;
  std::vector<int> h_c1(kMaxDim, 1);
  for (int a = 0; a < c.d; ++a) h_c1[a] = c.counts[a] == 1 ? 1 : 0;
  counts1.upload(h_c1, c.stream);
  A.box = c.dbox.p;
  A.counts1 = counts1.p;
  A.ax_lo = c.ax_lo.p;
  A.ax_hi = c.ax_hi.p;
  for (int a = 0; a < kMaxDim; ++a) {
    A.ax_counts[a] = c.ax_counts[a];
    A.ax_stride[a] = c.ax_stride[a];
    A.ax_off[a] = c.ax_off[a];
  }
  A.nbr_ptr = c.dnbr_ptr.p;
  A.nbr_idx = c.dnbr_idx.p;
  A.R = c.R.p;
  A.b = c.bvec.p;
}

void evaluate_at(Ctx& c, long long M, const double* pts, const double* W, const double* Lv, const double* Gv,
                 double* out) {
  ScopedKernelTimer tk(c, "evaluate");
  if (c.J == 0 || c.h_p.empty()) throw std::invalid_argument("evaluate_solution: build an instance first");
  if (M < 0 || M > 2000000000LL) throw std::invalid_argument("evaluate_solution: bad point count");
  if (M == 0) return;
  if (!W && c.W.n < static_cast<size_t>(c.p) * c.C) throw std::invalid_argument("evaluate_solution: no solution yet");
  EvalArgs A{};
  DBuf<int> counts1;
  eval_common(c, A, counts1);
  A.M = static_cast<int>(M);
  DBuf<double> dx, dl, dg, dw, U, ap;
  dx.upload(pts, static_cast<size_t>(M) * c.d, c.stream);
  dl.upload(Lv, static_cast<size_t>(M), c.stream);
  if (Gv) dg.upload(Gv, static_cast<size_t>(M) * c.C, c.stream);
  if (W) dw.upload(W, static_cast<size_t>(c.p) * c.C, c.stream);
  A.xin = dx.p;
  A.Lin = dl.p;
  A.Gin = Gv ? dg.p : nullptr;
  U.ensure(static_cast<size_t>(c.C) * c.J * c.m);
  k_effective_weights<<<c.J, 128, 0, c.stream>>>(c.Vred.p, W ? dw.p : c.W.p, c.dcol_off.p, c.J, c.m, c.p,
                                                 c.identity_V ? 1 : 0, U.p, c.C);
  RDD_LAUNCH_CHECK();
  A.U = U.p;
  ap.ensure(static_cast<size_t>(M) * c.C);
  A.approx = ap.p;
  k_evaluate<<<ceil_div(M, 128), 128, 0, c.stream>>>(A);
  RDD_LAUNCH_CHECK();
  ap.download(out, static_cast<size_t>(M) * c.C, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
}

void evaluate(Ctx& c, const int* test_res) {
  ScopedKernelTimer tk(c, "evaluate");
  if (c.prob.id == 0)
    throw std::invalid_argument("caller-supplied problem: evaluate at caller points (rdd_evaluate_at)");
  EvalArgs A{};
  if (!c.prob.has_exact) {  // example2: errors against the Crank-Nicolson field (runner.hpp:286-289)
    const int res = c.cfg.ref_resolution > 0 ? c.cfg.ref_resolution : 2001;
    if (c.ref2_res != res) {
      std::vector<double> v;
      reference_example2_grid(res, v);
      c.ref2.upload(v, c.stream);
      RDD_CUDA(cudaStreamSynchronize(c.stream));  // v is pageable and scoped
      c.ref2_res = res;
    }
    A.ref = c.ref2.p;
    A.refn = res;
  }
  DBuf<int> counts1;
  eval_common(c, A, counts1);
  long long M = 1;
  for (int a = 0; a < c.d; ++a) {
    if (test_res[a] < 1) throw std::invalid_argument("grid resolutions must be >= 1");
    A.res[a] = test_res[a];
    A.lo[a] = c.prob.lo[a];
    A.step[a] = (c.prob.hi[a] - c.prob.lo[a]) / static_cast<double>(test_res[a]);
    M *= test_res[a];
  }
  A.M = static_cast<int>(M);
  DBuf<double> U, ap, ex;
  U.ensure(static_cast<size_t>(c.C) * c.J * c.m);
  k_effective_weights<<<c.J, 128, 0, c.stream>>>(c.Vred.p, c.W.p, c.dcol_off.p, c.J, c.m, c.p, c.identity_V ? 1 : 0,
                                                 U.p, c.C);
  RDD_LAUNCH_CHECK();
  A.U = U.p;
  ap.ensure(static_cast<size_t>(M) * c.C);
  ex.ensure(static_cast<size_t>(M) * c.C);
  A.approx = ap.p;
  A.exact = ex.p;
  k_evaluate<<<ceil_div(M, 128), 128, 0, c.stream>>>(A);
  RDD_LAUNCH_CHECK();
  c.approx.resize(static_cast<size_t>(M) * c.C);
  c.exact.resize(static_cast<size_t>(M) * c.C);
  ap.download(c.approx.data(), c.approx.size(), c.stream);
  ex.download(c.exact.data(), c.exact.size(), c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  // problems.hpp:275-302 (stacked components; normalized_l1 divides by the point count)
  double dn = 0.0, num = 0.0, mean = 0.0, l1 = 0.0;
  for (size_t q = 0; q < c.exact.size(); ++q) {
    const double e = c.exact[q], dv = c.approx[q] - e;
    dn += e * e;
    num += dv * dv;
    mean += e;
    l1 += std::fabs(dv);
  }
  if (dn == 0.0) throw std::domain_error("rel_l2: exact solution has zero norm");
  mean /= static_cast<double>(c.exact.size());
  double var = 0.0;
  for (double e : c.exact) var += (e - mean) * (e - mean);
  var /= static_cast<double>(c.exact.size());
  const double gamma = std::sqrt(var);
  if (gamma == 0.0) throw std::domain_error("normalized_l1: exact solution set has zero standard deviation");
  c.sum.e_l2 = std::sqrt(num) / std::sqrt(dn);
  c.sum.e_l1n = l1 / (static_cast<double>(M) * gamma);
}

}  // namespace rdd
