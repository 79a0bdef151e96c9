// assemble.cu — K2: collocation-block assembly on the FP64 FMA pipe.
//
// Computes, for every subdomain j, row r (point x = pts[rows_j[r]]) and neuron k, either
//   op_applied: S_j[r,k] = A[L·ω_j·φ_k](x)   (reduction.hpp:53-76; = assembly.hpp:74-90 with V = I)
//   psi:        S_j[r,k] = ω_j(x)·φ_k(x)      (reduction.hpp:30-48)
// Per (point, subdomain) the kernel forms the jet LW = L·ω_j once (basis.hpp:121-167 window
// jets, Leibniz products as jet.hpp:107-124); per (subdomain, neuron) it precomputes
// g = R_k ⊙ (2/w), q1 = Σ c_a g_a, q2 = Σ_{a<=b} c_ab g_a g_b, h_a = Σ_b c̃_ab g_b. Since the
// operator is linear in the jet,
//   A[LW·φ_k] = t·A[LW] + t'·(LW·q1 + Σ_a ∂_aLW·h_a) + t''·LW·q2,   t = act(z), z = b_k + R_k·x̂,
// i.e. (2d+6) FMAs + one activation per entry. Output blocks are column-major
// (rows_j x m); a thread owns a row and streams across neurons, so each neuron's column is
// written by a warp as 32 consecutive doubles (coalesced).
#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int kRowsPerBlock = 128;
constexpr double kPiW = 3.14159265358979323846;  // basis.hpp:134

struct AsmArgs {
  int d, m, act, kind, J;
  const double* pts;
  int N;
  const int* row_ptr;
  const int* row_idx;
  const double* box;     // J x 16: lo[4], hi[4], wc[4], wh[4]
  const int* counts1;    // per axis: 1 if counts[a]==1 (window skips the axis)
  const int* nbr_ptr;
  const int* nbr_idx;
  const double* R;       // J x m x d
  const double* b;       // J x m
  const double* Ljet;    // N x jl
  double coef[kMaxJet];
  const int* tile_ptr;   // J+1 prefix of row tiles
  double* out;
  const long long* out_off;  // J+1 element offsets
  int* bad;              // [point, subdomain] of a non-finite entry
};

__device__ __forceinline__ bool in_box(const double* box, const double* x, int d) {
  for (int a = 0; a < d; ++a)
    if (x[a] < box[a] || x[a] > box[4 + a]) return false;
  return true;
}

// basis.hpp:121-138 raw_window_jet
__device__ Jet raw_window_jet(const AsmArgs& A, int k, const double* x) {
  const int d = A.d;
  Jet prod;
  jet_zero(prod, d);
  const double* bx = A.box + 16 * static_cast<size_t>(k);
  if (!in_box(bx, x, d)) return prod;
  prod.c[0] = 1.0;
  for (int a = 0; a < d; ++a) {
    if (A.counts1[a]) continue;
    const double mu = bx[8 + a], sigma = bx[12 + a];
    Jet s;
    jet_zero(s, d);
    s.c[0] = (x[a] - mu) / sigma;
    s.c[1 + a] = 1.0 / sigma;
    Jet ps = s;  // pi * s
    for (int q = 0; q < jet_len(d); ++q) ps.c[q] = s.c[q] * kPiW;
    const double arg = kPiW * s.c[0];
    double sn, cs;
    sincos(arg, &sn, &cs);
    Jet base = jet_compose(cs, -sn, -cs, ps, d);
    base.c[0] = 1.0 + base.c[0];
    prod = jet_mul(prod, jet_mul(base, base, d), d);
  }
  return prod;
}

__device__ double raw_window_value(const AsmArgs& A, int k, const double* x) {  // basis.hpp:140-154
  const double* bx = A.box + 16 * static_cast<size_t>(k);
  if (!in_box(bx, x, A.d)) return 0.0;
  double prod = 1.0;
  for (int a = 0; a < A.d; ++a) {
    if (A.counts1[a]) continue;
    const double s = (x[a] - bx[8 + a]) / bx[12 + a];
    const double base = 1.0 + cos(kPiW * s);
    prod *= base * base;
  }
  return prod;
}

__global__ void __launch_bounds__(kRowsPerBlock) k_assemble(AsmArgs A) {
  extern __shared__ double sm[];
  const int tile = blockIdx.x;
  // find the subdomain owning this tile
  int lo = 0, hi = A.J;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (A.tile_ptr[mid] <= tile) lo = mid;
    else hi = mid;
  }
  const int j = lo;
  const int d = A.d, m = A.m, jl = jet_len(d);
  const int rows = A.row_ptr[j + 1] - A.row_ptr[j];
  const int r = (tile - A.tile_ptr[j]) * kRowsPerBlock + threadIdx.x;
  const double* bx = A.box + 16 * static_cast<size_t>(j);

  // per-neuron parameters: [b, R(d), h(d), q1, q2]
  const int np = 3 + 2 * d;
  double w_[kMaxDim];
  for (int a = 0; a < d; ++a) w_[a] = 2.0 / (bx[4 + a] - bx[a]);  // normalize_scales (geometry.hpp:71-75)
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    double* P = sm + static_cast<size_t>(k) * np;
    const double* Rk = A.R + (static_cast<size_t>(j) * m + k) * d;
    P[0] = A.b[static_cast<size_t>(j) * m + k];
    double g[kMaxDim];
    for (int a = 0; a < d; ++a) {
      P[1 + a] = Rk[a];
      g[a] = Rk[a] * w_[a];
    }
    double q1 = 0.0, q2 = 0.0;
    for (int a = 0; a < d; ++a) {
      q1 += A.coef[1 + a] * g[a];
      double h = 0.0;
      for (int bb = 0; bb < d; ++bb) {
        const double cab = A.coef[1 + d + hess_index(min(a, bb), max(a, bb), d)];
        h += (a == bb ? 2.0 * cab : cab) * g[bb];
        if (bb >= a) q2 += cab * g[a] * g[bb];
      }
      P[1 + d + a] = h;
    }
    P[1 + 2 * d] = q1;
    P[2 + 2 * d] = q2;
  }
  __syncthreads();
  if (r >= rows) return;

  const int gi = A.row_idx[A.row_ptr[j] + r];
  double x[kMaxDim] = {0, 0, 0, 0}, xh[kMaxDim];
  for (int a = 0; a < d; ++a) x[a] = A.pts[static_cast<size_t>(a) * A.N + gi];
  for (int a = 0; a < d; ++a) {
    const double cen = 0.5 * (bx[a] + bx[4 + a]);
    const double wid = bx[4 + a] - bx[a];
    xh[a] = 2.0 * (x[a] - cen) / wid;  // normalize_to_box (geometry.hpp:61-68)
  }
  double* out = A.out + A.out_off[j] + r;

  if (A.kind == RDD_PCA_PSI) {
    const double wj = raw_window_value(A, j, x);
    double w = 0.0;
    if (wj != 0.0) {
      double tot = 0.0;
      for (int q = A.nbr_ptr[j]; q < A.nbr_ptr[j + 1]; ++q) tot += raw_window_value(A, A.nbr_idx[q], x);
      w = wj / tot;
    }
    for (int k = 0; k < m; ++k) {
      const double* P = sm + static_cast<size_t>(k) * np;
      double z = P[0];
      for (int a = 0; a < d; ++a) z += P[1 + a] * xh[a];
      const double t = A.act == 0 ? tanh(z) : sin(z);
      out[static_cast<size_t>(k) * rows] = w * t;
    }
    return;
  }

  // LW = L(x) * window_jet(j, x)  (basis.hpp:158-167, 211)
  const Jet wj = raw_window_jet(A, j, x);
  Jet tot;
  jet_zero(tot, d);
  for (int q = A.nbr_ptr[j]; q < A.nbr_ptr[j + 1]; ++q) {
    const Jet rk = raw_window_jet(A, A.nbr_idx[q], x);
    for (int e = 0; e < jl; ++e) tot.c[e] += rk.c[e];
  }
  if (!(tot.c[0] > 0.0)) atomicExch(A.bad + 2, 1);  // domain_error (basis.hpp:165)
  const double rcp = 1.0 / tot.c[0];
  const Jet win = jet_mul(wj, jet_compose(rcp, -rcp * rcp, 2.0 * rcp * rcp * rcp, tot, d), d);
  Jet L;
  for (int e = 0; e < jl; ++e) L.c[e] = A.Ljet[static_cast<size_t>(gi) * jl + e];
  const Jet LW = jet_mul(L, win, d);
  double alpha = 0.0;
  for (int e = 0; e < jl; ++e) alpha += A.coef[e] * LW.c[e];
  const double lwv = LW.c[0];
  double lwg[kMaxDim];
  for (int a = 0; a < d; ++a) lwg[a] = LW.c[1 + a];

  bool bad = false;
  for (int k = 0; k < m; ++k) {
    const double* P = sm + static_cast<size_t>(k) * np;
    double z = P[0];
    for (int a = 0; a < d; ++a) z += P[1 + a] * xh[a];
    double t, t1, t2;
    if (A.act == 0) {
      t = tanh(z);
      t1 = 1.0 - t * t;
      t2 = -2.0 * t * t1;
    } else {
      double sn, cs;
      sincos(z, &sn, &cs);
      t = sn;
      t1 = cs;
      t2 = -sn;
    }
    double beta = lwv * P[1 + 2 * d];
    for (int a = 0; a < d; ++a) beta += lwg[a] * P[1 + d + a];
    const double v = alpha * t + beta * t1 + (lwv * P[2 + 2 * d]) * t2;
    bad |= !isfinite(v);
    out[static_cast<size_t>(k) * rows] = v;
  }
  if (bad) {
    atomicExch(A.bad, gi);
    atomicExch(A.bad + 1, j);
  }
}

}  // namespace

// Fills `out` (per-block column-major, offsets `off`) with the unreduced sample/collocation blocks.
void assemble_samples(Ctx& c, int kind, double* out, const std::vector<long long>& off) {
  ScopedKernelTimer tk(c, kind == RDD_PCA_PSI ? "assemble_psi" : "assemble");
  AsmArgs A{};
  A.d = c.d;
  A.m = c.m;
  A.act = c.cfg.activation;
  A.kind = kind;
  A.J = c.J;
  A.pts = c.pts.p;
  A.N = c.N;
  A.row_ptr = c.row_ptr.p;
  A.row_idx = c.row_idx.p;
  A.box = c.dbox.p;
  DBuf<int> counts1, tile_ptr, bad;
  std::vector<int> h_c1(kMaxDim, 1);
  for (int a = 0; a < c.d; ++a) h_c1[a] = c.counts[a] == 1 ? 1 : 0;
  counts1.upload(h_c1, c.stream);
  A.counts1 = counts1.p;
  A.nbr_ptr = c.dnbr_ptr.p;
  A.nbr_idx = c.dnbr_idx.p;
  A.R = c.R.p;
  A.b = c.bvec.p;
  A.Ljet = c.Ljet.p;
  for (int k = 0; k < kMaxJet; ++k) A.coef[k] = c.prob.coef[k];
  std::vector<int> tp(c.J + 1, 0);
  for (int j = 0; j < c.J; ++j) tp[j + 1] = tp[j] + ceil_div(c.h_row_ptr[j + 1] - c.h_row_ptr[j], kRowsPerBlock);
  tile_ptr.upload(tp, c.stream);
  A.tile_ptr = tile_ptr.p;
  A.out = out;
  DBuf<long long> doff;
  doff.upload(off, c.stream);
  A.out_off = doff.p;
  const int hbad[3] = {-1, -1, 0};
  bad.upload(hbad, 3, c.stream);
  A.bad = bad.p;
  const size_t smem = static_cast<size_t>(c.m) * (3 + 2 * c.d) * sizeof(double);
  if (smem > 32 * 1024) RDD_CUDA(cudaFuncSetAttribute(k_assemble, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (tp[c.J] > 0) {
    k_assemble<<<tp[c.J], kRowsPerBlock, smem, c.stream>>>(A);
    RDD_LAUNCH_CHECK();
  }
  int hb[3];
  bad.download(hb, 3, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  if (hb[2]) throw std::domain_error("window normalization vanished; point outside the domain?");
  if (hb[0] >= 0)
    throw std::runtime_error("non-finite matrix entry at collocation point " + std::to_string(hb[0]) +
                             ", subdomain " + std::to_string(hb[1]));
}

}  // namespace rdd
