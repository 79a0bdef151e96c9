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
#include <type_traits>

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

// basis.hpp:121-138 raw_window_jet (D compile-time: the jet loops unroll, jets stay in registers)
template <int D>
__device__ __forceinline__ Jet raw_window_jet(const AsmArgs& A, int k, const double* x) {
  constexpr int d = D;
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

// per-row constants of the op_applied entries, held in registers across the neuron loop
template <int D>
struct RowCoef {
  double xh[D];   // local coordinates in [-1, 1]^d
  double lwg[D];  // ∇(L·ω_j)
  double lwv;     // L·ω_j
  double alpha;   // A[L·ω_j] (operator applied to the jet)
};

// the neuron loop of one row: z = b + R·x̂, entry = α·t(z) + β·t'(z) + (LW·q2)·t''(z) with
// β = LW·q1 + ∇LW·h (per-neuron q1, h, q2 in shared memory), stored down the block's column-major
// layout; returns whether any entry was non-finite
template <int D, int ACT>
__device__ __forceinline__ bool row_entries(const double* __restrict__ sm, int m, const RowCoef<D> rc,
                                            double* __restrict__ out, int rows) {
  constexpr int np = 3 + 2 * D;
  // pin the row constants in registers (otherwise they are re-read from the prologue's stack
  // frame on every neuron)
  double xh[D], lwg[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    xh[a] = rc.xh[a];
    lwg[a] = rc.lwg[a];
    asm volatile("" : "+d"(xh[a]), "+d"(lwg[a]));
  }
  double lwv = rc.lwv, alpha = rc.alpha;
  asm volatile("" : "+d"(lwv), "+d"(alpha));
  bool bad = false;
  for (int k = 0; k < m; ++k, out += rows) {
    const double* P = sm + k * np;
    double z = P[0];
#pragma unroll
    for (int a = 0; a < D; ++a) z += P[1 + a] * xh[a];
    double t, t1, t2;
    if constexpr (ACT == 0) {
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
    double beta = lwv * P[1 + 2 * D];
#pragma unroll
    for (int a = 0; a < D; ++a) beta += lwg[a] * P[1 + D + a];
    const double v = alpha * t + beta * t1 + (lwv * P[2 + 2 * D]) * t2;
    bad |= !isfinite(v);
    *out = v;
  }
  return bad;
}

// the subdomain owning row tile `tile` (tile_ptr: J+1 prefix of row tiles)
__device__ __forceinline__ int tile_block(const int* __restrict__ tile_ptr, int J, int tile) {
  int lo = 0, hi = J;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tile_ptr[mid] <= tile) lo = mid;
    else hi = mid;
  }
  return lo;
}

// per-neuron parameters [b, R(d), h(d), q1, q2] of neuron k of subdomain j
template <int D>
__device__ __forceinline__ void neuron_params(const AsmArgs& A, int j, int k, double* P) {
  const double* bx = A.box + 16 * static_cast<size_t>(j);
  const double* Rk = A.R + (static_cast<size_t>(j) * A.m + k) * D;
  P[0] = A.b[static_cast<size_t>(j) * A.m + k];
  double g[D];
  for (int a = 0; a < D; ++a) {
    P[1 + a] = Rk[a];
    g[a] = Rk[a] * (2.0 / (bx[4 + a] - bx[a]));  // normalize_scales (geometry.hpp:71-75)
  }
  double q1 = 0.0, q2 = 0.0;
  for (int a = 0; a < D; ++a) {
    q1 += A.coef[1 + a] * g[a];
    double h = 0.0;
    for (int bb = 0; bb < D; ++bb) {
      const double cab = A.coef[1 + D + hess_index(min(a, bb), max(a, bb), D)];
      h += (a == bb ? 2.0 * cab : cab) * g[bb];
      if (bb >= a) q2 += cab * g[a] * g[bb];
    }
    P[1 + D + a] = h;
  }
  P[1 + 2 * D] = q1;
  P[2 + 2 * D] = q2;
}

// the point of row r of block j and its local coordinates (normalize_to_box, geometry.hpp:61-68)
template <int D>
__device__ __forceinline__ int row_point(const AsmArgs& A, int j, int r, double* x, double* xh) {
  const double* bx = A.box + 16 * static_cast<size_t>(j);
  const int gi = A.row_idx[A.row_ptr[j] + r];
  for (int a = 0; a < kMaxDim; ++a) x[a] = 0.0;
  for (int a = 0; a < D; ++a) x[a] = A.pts[static_cast<size_t>(a) * A.N + gi];
  for (int a = 0; a < D; ++a) {
    const double cen = 0.5 * (bx[a] + bx[4 + a]);
    const double wid = bx[4 + a] - bx[a];
    xh[a] = 2.0 * (x[a] - cen) / wid;
  }
  return gi;
}

// psi sample blocks (reduction.hpp:30-48): S_j[r,k] = ω_j(x)·φ_k(x), one kernel
template <int D>
__global__ void __launch_bounds__(kRowsPerBlock) k_assemble_psi(AsmArgs A) {
  extern __shared__ double sm[];
  const int tile = blockIdx.x;
  const int j = tile_block(A.tile_ptr, A.J, tile);
  const int m = A.m, np = 3 + 2 * D;
  const int rows = A.row_ptr[j + 1] - A.row_ptr[j];
  const int r = (tile - A.tile_ptr[j]) * kRowsPerBlock + threadIdx.x;
  for (int k = threadIdx.x; k < m; k += blockDim.x) neuron_params<D>(A, j, k, sm + static_cast<size_t>(k) * np);
  __syncthreads();
  if (r >= rows) return;
  double x[kMaxDim], xh[D];
  row_point<D>(A, j, r, x, xh);
  double* out = A.out + A.out_off[j] + r;
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
    for (int a = 0; a < D; ++a) z += P[1 + a] * xh[a];
    const double t = A.act == 0 ? tanh(z) : sin(z);
    out[static_cast<size_t>(k) * rows] = w * t;
  }
}

// op_applied, stage 1a: per-neuron parameters of every subdomain (J x m x np) to global memory
template <int D>
__global__ void k_neuron_params(AsmArgs A, double* __restrict__ Pg) {
  const int j = blockIdx.x;
  constexpr int np = 3 + 2 * D;
  for (int k = threadIdx.x; k < A.m; k += blockDim.x)
    neuron_params<D>(A, j, k, Pg + (static_cast<size_t>(j) * A.m + k) * np);
}

// op_applied, stage 1b: per (block, row) the row constants RowCoef (x̂, LW, ∇LW, A[LW]) with
// LW = L(x)·window_jet(j, x) (basis.hpp:158-167, 211), stored field-major (rc[f·nent + entry])
template <int D>
__global__ void __launch_bounds__(kRowsPerBlock) k_row_coefs(AsmArgs A, double* __restrict__ rcg, long long nent) {
  const int tile = blockIdx.x;
  const int j = tile_block(A.tile_ptr, A.J, tile);
  const int jl = jet_len(D);
  const int rows = A.row_ptr[j + 1] - A.row_ptr[j];
  const int r = (tile - A.tile_ptr[j]) * kRowsPerBlock + threadIdx.x;
  if (r >= rows) return;
  double x[kMaxDim], xh[D];
  const int gi = row_point<D>(A, j, r, x, xh);
  const Jet wj = raw_window_jet<D>(A, j, x);
  Jet tot;
  jet_zero(tot, D);
  for (int q = A.nbr_ptr[j]; q < A.nbr_ptr[j + 1]; ++q) {
    const Jet rk = raw_window_jet<D>(A, A.nbr_idx[q], x);
    for (int e = 0; e < jl; ++e) tot.c[e] += rk.c[e];
  }
  if (!(tot.c[0] > 0.0)) atomicExch(A.bad + 2, 1);  // domain_error (basis.hpp:165)
  const double rcp = 1.0 / tot.c[0];
  const Jet win = jet_mul(wj, jet_compose(rcp, -rcp * rcp, 2.0 * rcp * rcp * rcp, tot, D), D);
  Jet L;
  for (int e = 0; e < jl; ++e) L.c[e] = A.Ljet[static_cast<size_t>(gi) * jl + e];
  const Jet LW = jet_mul(L, win, D);
  double alpha = 0.0;
  for (int e = 0; e < jl; ++e) alpha += A.coef[e] * LW.c[e];
  const long long e0 = A.row_ptr[j] + r;
  for (int a = 0; a < D; ++a) {
    rcg[a * nent + e0] = xh[a];
    rcg[(D + a) * nent + e0] = LW.c[1 + a];
  }
  rcg[2 * D * nent + e0] = LW.c[0];
  rcg[(2 * D + 1) * nent + e0] = alpha;
}

// op_applied, stage 2: the entries. No calls and no divisions in this kernel, so the row
// constants live in registers across the neuron loop (a fused prologue with the window jets'
// division / sincos subroutine calls put them on the stack, re-read every neuron).
template <int D, int ACT>
__global__ void __launch_bounds__(kRowsPerBlock) k_assemble_op(AsmArgs A, const double* __restrict__ Pg,
                                                               const double* __restrict__ rcg, long long nent) {
  extern __shared__ double sm[];
  constexpr int np = 3 + 2 * D;
  const int tile = blockIdx.x;
  const int j = tile_block(A.tile_ptr, A.J, tile);
  const int m = A.m;
  const int rows = A.row_ptr[j + 1] - A.row_ptr[j];
  const int r = (tile - A.tile_ptr[j]) * kRowsPerBlock + threadIdx.x;
  const double* Pj = Pg + static_cast<size_t>(j) * m * np;
  for (int q = threadIdx.x; q < m * np; q += blockDim.x) sm[q] = Pj[q];
  __syncthreads();
  if (r >= rows) return;
  const long long e0 = A.row_ptr[j] + r;
  RowCoef<D> rc;
  for (int a = 0; a < D; ++a) {
    rc.xh[a] = rcg[a * nent + e0];
    rc.lwg[a] = rcg[(D + a) * nent + e0];
  }
  rc.lwv = rcg[2 * D * nent + e0];
  rc.alpha = rcg[(2 * D + 1) * nent + e0];
  if (row_entries<D, ACT>(sm, m, rc, A.out + A.out_off[j] + r, rows)) {
    atomicExch(A.bad, A.row_idx[e0]);
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
  if (c.d < 1 || c.d > 4) throw std::invalid_argument("assemble: dimension must be 1..4");
  const long long nent = c.h_row_ptr[c.J];
  auto run = [&](auto dim) {
    constexpr int D = decltype(dim)::value;
    auto launch = [&](auto kernel, auto... extra) {
      if (smem > 32 * 1024) RDD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      kernel<<<tp[c.J], kRowsPerBlock, smem, c.stream>>>(A, extra...);
      RDD_LAUNCH_CHECK();
    };
    if (kind == RDD_PCA_PSI) {
      launch(k_assemble_psi<D>);
      return;
    }
    double* Pg = c.ws("asm_neuron", static_cast<size_t>(c.J) * c.m * (3 + 2 * D));
    double* rcg = c.ws("asm_rowc", static_cast<size_t>(nent) * (2 * D + 2));
    k_neuron_params<D><<<c.J, 128, 0, c.stream>>>(A, Pg);
    RDD_LAUNCH_CHECK();
    k_row_coefs<D><<<tp[c.J], kRowsPerBlock, 0, c.stream>>>(A, rcg, nent);
    RDD_LAUNCH_CHECK();
    if (A.act == 0) launch(k_assemble_op<D, 0>, static_cast<const double*>(Pg), static_cast<const double*>(rcg), nent);
    else launch(k_assemble_op<D, 1>, static_cast<const double*>(Pg), static_cast<const double*>(rcg), nent);
  };
  if (tp[c.J] > 0) {
    switch (c.d) {
      case 1: run(std::integral_constant<int, 1>{}); break;
      case 2: run(std::integral_constant<int, 2>{}); break;
      case 3: run(std::integral_constant<int, 3>{}); break;
      default: run(std::integral_constant<int, 4>{}); break;
    }
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
