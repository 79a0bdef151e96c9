// pca.cu — K3-K5: per-subdomain PCA truncation (reduction.hpp:89-109) on the device.
//
// The reference takes a thin JacobiSVD of each sample block S_j (rows_j x m) and keeps the
// right singular vectors with σ > τ. A Gram matrix alone cannot reproduce that: SᵀS squares
// the condition number, so eigenvalues near a relative threshold of 1e-6 (λ ~ 1e-12 λmax) carry
// O(1e-4) relative error and the kept subspace O(1e-4) error (SURVEY §7.3 hard part 1).
// Main path (DESIGN §4 K4a/K4):
//   1. G = SᵀS (DMMA); pivoted Cholesky of G to its numerical rank r, Jacobi on the graded
//      r x r LᵀL, V_r = L·U;
//   2. one subspace-iteration step from S itself, Y = Sᵀ(S·V_r) (two DMMA GEMMs), orthonormalised
//      by a thin Householder QR (k_house_complete) -> Q;
//   3. Jacobi with the relative criterion (Demmel–Veselić) on the graded r x r (S·Q)ᵀ(S·Q)
//      -> W, σ relatively accurate, V = Q·W.
// Fallback (thresholds below ~1e-7·σmax): the two-stage path — Jacobi on G -> V0, then
// T = S·V0, Jacobi on TᵀT with the relative threshold -> W, V = V0·W.
// Then: sort σ non-increasing, keep σ > τ (strict; τ relative to σ_max in RDD_TAU_RELATIVE
// mode), floor p_j >= 1, canonical signs (first nonzero entry of each kept column >= 0), and
// H_j = S_j·V_j (DMMA) — by linearity equal to assembling the reduced jets (reduction.hpp:122-139).
#include <algorithm>

#include "ctx.hpp"

namespace rdd {

// C_j = A_j·B_j for a batch of row-major-tiled NN products whose widths N_j are all <= 128 take the
// 64 x 128-tile kernel (the tall A_j = S_j streamed once per row tile), otherwise 64 x 64 tiles
struct NNItem {
  const double* A;
  const double* B;
  double* C;
  int M, N, K, lda, ldb, ldc;
};
// CTA tile edge (64 or 80) for a batch of M_i x N_i outputs of TN products: 80 when it cuts the
// padded tile area by more than 12%, its own per-flop deficit (m = 400 is 5 tiles of 80 but 7 of
// 64, 448² vs 400²: Gram and Sᵀ·Z 25 -> 28 TF/s; the NN products lose with it, tools/gemm_bench.py)
int pick_tile(const std::vector<std::pair<int, int>>& mn, bool upper = false) {
  double a64 = 0.0, a80 = 0.0;
  for (const auto& e : mn) {
    const double m64 = ceil_div(e.first, 64), n64 = ceil_div(e.second, 64);
    const double m80 = ceil_div(e.first, 80), n80 = ceil_div(e.second, 80);
    a64 += (upper ? m64 * (m64 + 1) / 2 : m64 * n64) * 64.0 * 64.0;
    a80 += (upper ? m80 * (m80 + 1) / 2 : m80 * n80) * 80.0 * 80.0;
  }
  return a80 < 0.88 * a64 ? 80 : 64;
}
static void nn_batch(Ctx& c, const std::vector<NNItem>& items) {
  int nmax = 0;
  double w64 = 0.0, w80 = 0.0;  // padded widths, weighted by the rows
  for (const NNItem& it : items) {
    nmax = std::max(nmax, it.N);
    w64 += static_cast<double>(it.M) * ceil_div(it.N, 64) * 64;
    w80 += static_cast<double>(it.M) * ceil_div(it.N, 80) * 80;
  }
  const bool wide = nmax > 64 && nmax <= 128;  // N <= 64 fits one 64-wide tile already
  // 64 x 80 tiles when the 80-wide columns pad at least 7% less (r = 386: 400 vs 448 columns;
  // per flop that tile is ~5% slower: S·Q of C5 25.3 -> 26.9 TF/s)
  const bool t80 = !wide && w80 < 0.93 * w64;
  const int tw = wide ? 128 : (t80 ? 80 : 64);
  std::vector<GemmTask> t;
  for (const NNItem& it : items)
    for (int tm = 0; tm < ceil_div(it.M, 64); ++tm)
      for (int tn = 0; tn < ceil_div(it.N, tw); ++tn)
        t.push_back({it.A, it.B, it.C, nullptr, nullptr, it.M, it.N, it.K, it.lda, it.ldb, it.ldc, tm, tn, 0.0});
  if (wide) gemm_nn_wide(c, t);
  else gemm_nn(c, t, t80 ? 6480 : 64);
}


namespace {

// per subdomain: sort eigenvalues descending, threshold, reorder + sign-canonicalise V
// cnt/lam_off (optional): subdomain j has cnt[j] eigenpairs, eigenvalues at lam + lam_off[j] and
// V columns 0..cnt[j]-1 (ld m); the remaining min(rows, m) - cnt[j] singular values are reported as 0
__global__ void k_select(const double* __restrict__ lam, const double* __restrict__ Vin, double* __restrict__ Vout,
                         double* __restrict__ sig, int* __restrict__ p_out, const int* __restrict__ row_ptr, int m,
                         int tau_mode, double tau, const int* __restrict__ cnt, const long long* __restrict__ lam_off) {
  extern __shared__ double sm[];
  double* s = sm;                              // m sigma
  int* perm = reinterpret_cast<int*>(s + m);   // m
  __shared__ int keep;
  const int j = blockIdx.x;
  const int mc = cnt ? cnt[j] : m;
  const double* L = lam + (lam_off ? lam_off[j] : static_cast<long long>(j) * m);
  for (int i = threadIdx.x; i < mc; i += blockDim.x) s[i] = sqrt(fmax(L[i], 0.0));
  __syncthreads();
  for (int i = threadIdx.x; i < mc; i += blockDim.x) {  // stable descending rank
    int rk = 0;
    for (int k = 0; k < mc; ++k) rk += (s[k] > s[i]) || (s[k] == s[i] && k < i);
    perm[rk] = i;
  }
  __syncthreads();
  const int rows = row_ptr[j + 1] - row_ptr[j];
  const int nsv = min(rows, m);  // thin SVD: min(rows, m) singular values
  if (threadIdx.x == 0) {
    const double smax = s[perm[0]];
    const double thr = tau_mode == RDD_TAU_RELATIVE ? tau * smax : tau;
    int k = 0;
    for (int i = 0; i < min(nsv, mc); ++i)
      if (s[perm[i]] > thr) ++k;
    keep = max(k, 1);
    p_out[j] = keep;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x)
    sig[static_cast<size_t>(j) * m + i] = (i < nsv && i < mc) ? s[perm[i]] : 0.0;
  // reorder columns; sign so that the first nonzero entry is >= 0 (reduction.hpp:100-107)
  const double* Vi = Vin + static_cast<size_t>(j) * m * m;
  double* Vo = Vout + static_cast<size_t>(j) * m * m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int c = warp; c < keep; c += nw) {
    const double* src = Vi + static_cast<size_t>(perm[c]) * m;
    int first = m;
    for (int r0 = 0; r0 < m && first == m; r0 += 32) {
      const int r = r0 + lane;
      const unsigned ball = __ballot_sync(0xffffffffu, r < m && src[r] != 0.0);
      if (ball) first = r0 + __ffs(ball) - 1;
    }
    const double sg = (first < m && src[first] < 0.0) ? -1.0 : 1.0;
    for (int r = lane; r < m; r += 32) Vo[static_cast<size_t>(c) * m + r] = sg * src[r];
  }
}

// Stage-1 reduction: pivoted Cholesky of the Gram (upper triangle valid), G ≈ L Lᵀ with L n x r
// in original row order (column-major, ld n). Pivot = largest remaining Schur diagonal (smallest
// index on ties); stops when it is not positive or below stop·(first pivot), so r is the
// numerical rank of G. L's columns are graded, which is what makes the Jacobi on LᵀL short.
constexpr int kPcholThreads = 512;
__global__ void __launch_bounds__(kPcholThreads) k_pchol(const double* __restrict__ G, double* __restrict__ L, int n,
                                                          double stop, int* __restrict__ r_out,
                                                          double* __restrict__ trace_out) {
  extern __shared__ double psm[];
  double* d = psm;                                             // n: remaining diagonal
  double* li = d + n;                                          // n: L[i, :k]
  unsigned char* done = reinterpret_cast<unsigned char*>(li + n);  // n: pivoted flags
  __shared__ double rv[kPcholThreads / 32];
  __shared__ int ri[kPcholThreads / 32];
  __shared__ int piv_s;
  __shared__ double dpiv_s;
  const int j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* Gj = G + static_cast<size_t>(j) * n * n;
  double* Lj = L + static_cast<size_t>(j) * n * n;
  for (int i = tid; i < n; i += blockDim.x) {
    d[i] = Gj[i + static_cast<size_t>(i) * n];
    done[i] = 0;
  }
  __syncthreads();
  double dmax0 = 0.0;
  int r = 0;
  for (int k = 0; k < n; ++k) {
    double bv = -1.0;
    int bi = n;
    for (int i = tid; i < n; i += blockDim.x)
      if (!done[i] && d[i] > bv) {
        bv = d[i];
        bi = i;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      rv[warp] = bv;
      ri[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      double v = rv[0];
      int ix = ri[0];
      for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
        if (rv[w] > v || (rv[w] == v && ri[w] < ix)) {
          v = rv[w];
          ix = ri[w];
        }
      piv_s = ix;
      dpiv_s = v;
    }
    __syncthreads();
    const int i = piv_s;
    const double dp = dpiv_s;
    if (k == 0) dmax0 = dp;
    if (!(dp > 0.0) || dp <= stop * dmax0) break;
    for (int t = tid; t < k; t += blockDim.x) li[t] = Lj[i + static_cast<size_t>(t) * n];
    __syncthreads();
    const double sd = sqrt(dp);
    for (int row = tid; row < n; row += blockDim.x) {
      double x = 0.0;
      if (row == i) {
        x = sd;
      } else if (!done[row]) {
        double s = 0.0;
        for (int t = 0; t < k; ++t) s += Lj[row + static_cast<size_t>(t) * n] * li[t];
        const double g = row <= i ? Gj[row + static_cast<size_t>(i) * n] : Gj[i + static_cast<size_t>(row) * n];
        x = (g - s) / sd;
        d[row] -= x * x;
      }
      Lj[row + static_cast<size_t>(k) * n] = x;
    }
    if (tid == 0) done[i] = 1;
    r = k + 1;
    __syncthreads();
  }
  if (r == 0) {  // G = 0: one zero column (the completion below then yields the identity)
    for (int row = tid; row < n; row += blockDim.x) Lj[row] = 0.0;
    r = 1;
  }
  if (tid == 0) {
    r_out[j] = r;
    double tr = 0.0;
    for (int i = 0; i < n; ++i) tr += Gj[i + static_cast<size_t>(i) * n];
    trace_out[j] = tr;
  }
}

// V0 = [orth(Vr), complement]: columns of Vr (n x r, eigenvectors of LLᵀ up to scale) sorted by
// descending eigenvalue and normalised, Householder QR in that order, and the full n x n
// Q = H_0 ⋯ H_{r-1} accumulated backwards. Q is orthogonal to rounding whatever the accuracy
// of the small directions of Vr; its first r columns span them in order.
constexpr int kHouseThreads = 512;
__global__ void __launch_bounds__(kHouseThreads) k_house_complete(const double* __restrict__ Vr,
                                                                  const double* __restrict__ lam,
                                                                  const long long* __restrict__ lam_off,
                                                                  const int* __restrict__ rr, int n,
                                                                  double* __restrict__ A, double* __restrict__ Q,
                                                                  int thin) {
  extern __shared__ double hsm[];
  double* v = hsm;              // n: current Householder vector
  double* beta = v + n;         // r
  int* perm = reinterpret_cast<int*>(beta + n);  // r
  __shared__ double red[kHouseThreads / 32];
  const int j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int r = rr[j];
  const size_t off = static_cast<size_t>(j) * n * n;
  const double* Vj = Vr + off;
  double* Aj = A + off;
  double* Qj = Q + off;
  const double* lj = lam + lam_off[j];
  for (int c = tid; c < r; c += blockDim.x) {  // stable descending rank of the eigenvalues
    int rk = 0;
    for (int q = 0; q < r; ++q) rk += (lj[q] > lj[c]) || (lj[q] == lj[c] && q < c);
    perm[rk] = c;
  }
  __syncthreads();
  for (int c = warp; c < r; c += nw) {  // A[:, c] = Vr[:, perm[c]] / ||.||
    const double* src = Vj + static_cast<size_t>(perm[c]) * n;
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += src[i] * src[i];
    s = warp_sum(s);
    const double sc = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
    for (int i = lane; i < n; i += 32) Aj[i + static_cast<size_t>(c) * n] = src[i] * sc;
  }
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    double* x = Aj + static_cast<size_t>(k) * n;
    double s = 0.0;
    for (int i = k + tid; i < n; i += blockDim.x) s += x[i] * x[i];
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    double nrm2 = 0.0;
    for (int w = 0; w < nw; ++w) nrm2 += red[w];
    const double alpha = sqrt(nrm2), x0 = x[k];
    const double sg = x0 >= 0.0 ? -alpha : alpha;   // H x = sg e_k
    const double b = alpha > 0.0 ? 1.0 / (sg * (sg - x0)) : 0.0;
    for (int i = k + tid; i < n; i += blockDim.x) v[i] = (i == k) ? x0 - sg : x[i];
    if (tid == 0) beta[k] = b;
    __syncthreads();
    if (tid == 0) x[k] = x0 - sg;  // keep v_k in A[k:, k] for the accumulation
    for (int c = k + 1 + warp; c < r; c += nw) {
      double* y = Aj + static_cast<size_t>(c) * n;
      double w = 0.0;
      for (int i = k + lane; i < n; i += 32) w += v[i] * y[i];
      w = warp_sum(w) * b;
      for (int i = k + lane; i < n; i += 32) y[i] -= w * v[i];
    }
    __syncthreads();
  }
  const int nq = thin ? r : n;  // thin: Q[:, :r] = H_0 ⋯ H_{r-1} [I_r; 0]
  for (size_t e = tid; e < static_cast<size_t>(n) * nq; e += blockDim.x) Qj[e] = (e % (n + 1) == 0) ? 1.0 : 0.0;
  __syncthreads();
  for (int k = r - 1; k >= 0; --k) {
    const double* x = Aj + static_cast<size_t>(k) * n;
    for (int i = k + tid; i < n; i += blockDim.x) v[i] = x[i];
    __syncthreads();
    const double b = beta[k];
    if (b != 0.0)
      for (int c = k + warp; c < nq; c += nw) {
        double* y = Qj + static_cast<size_t>(c) * n;
        double w = 0.0;
        for (int i = k + lane; i < n; i += 32) w += v[i] * y[i];
        w = warp_sum(w) * b;
        for (int i = k + lane; i < n; i += 32) y[i] -= w * v[i];
      }
    __syncthreads();
  }
}

// Thin Householder QR in blocked (compact-WY) form, the same reflectors as k_house_complete's:
// panels of kHP columns are factored in shared memory (column-by-column, H_k = I − β_k v_k v_kᵀ,
// H x = sg e_k), T of the panel (H_p ⋯ H_{p+w−1} = I − V T Vᵀ) is formed from VᵀV, and every
// column right of the panel takes one update y ← y − V Tᵀ (Vᵀ y), a warp per column with the
// panel in shared memory — each trailing column is read once per panel instead of once per
// reflector. Q = H_0 ⋯ H_{r−1} [I_r; 0] is accumulated panel by panel in reverse (y ← y − V T (Vᵀ y)
// on columns >= p). One CTA per subdomain; m <= kHouseMaxM.
constexpr int kHP = 32;
constexpr int kHouseMaxM = 512;
constexpr int kHBThreads = 512;
constexpr int kHBWarps = kHBThreads / 32;
__host__ __device__ constexpr int house_ldp(int n) { return n + ((20 - (n & 15)) & 15); }


__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
// A 32 x 8 matrix held as four DMMA accumulator fragments (tile mt: m = 8 mt + lane/4, n = 2 (lane%4) + e)
// -> its B fragment of k-step kk: the value at (k = 4 kk + lane%4, n = lane/4)
__device__ __forceinline__ double c_to_b(const double (&acc)[4][2], int kk, int lane) {
  const int mt = kk >> 1;
  const int src = ((4 * (kk & 1) + (lane & 3)) << 2) | (lane >> 3);
  const double v0 = __shfl_sync(0xffffffffu, acc[mt][0], src);
  const double v1 = __shfl_sync(0xffffffffu, acc[mt][1], src);
  return ((lane >> 2) & 1) ? v1 : v0;
}

// Eight trailing columns at once on the FP64 tensor cores (one warp): Y <- Y - V M (Vᵀ Y) with
// V = the panel in shared memory (R x w, zero above its diagonal, column stride ldp ≡ 4 mod 16 so
// the fragment reads are conflict-free), M = T (transposed when tr), Y = global columns
// c0 .. min(c0 + 8, cend) - 1 (rows 0..R-1 of the pointer, column stride ldy). W = VᵀY accumulates
// over the rows in four 8 x 8 fragments, Z = M W and the update Y -= V Z are DMMA products too:
// every panel element is read once per eight columns instead of once per column.
__device__ __forceinline__ void wy_update8(const double* __restrict__ P, int ldp, int R, int w, const double* Tm,
                                           bool tr, double* Y, int ldy, int c0, int cend, int lane) {
  double wa[4][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) wa[mt][0] = wa[mt][1] = 0.0;
  {
    const int col = c0 + (lane >> 2);
    const double* yc = Y + static_cast<long long>(col) * ldy;
    for (int r = 0; r < R; r += 4) {
      const int row = r + (lane & 3);
      const bool rv = row < R;
      const double bfr = (rv && col < cend) ? yc[row] : 0.0;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int i = 8 * mt + (lane >> 2);
        const double afr = (rv && i < w) ? P[i * ldp + row] : 0.0;
        dmma884(wa[mt], afr, bfr);
      }
    }
  }
  double za[4][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) za[mt][0] = za[mt][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const double bfr = c_to_b(wa, kk, lane);
    const int kc = 4 * kk + (lane & 3);
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int i = 8 * mt + (lane >> 2);
      double afr = 0.0;
      if (i < w && kc < w) afr = tr ? Tm[kc * kHP + i] : Tm[i * kHP + kc];
      dmma884(za[mt], afr, bfr);
    }
  }
  double bz[8];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) bz[kk] = c_to_b(za, kk, lane);
  const int cc = c0 + 2 * (lane & 3);
  for (int r0 = 0; r0 < R; r0 += 8) {
    const int row = r0 + (lane >> 2);
    double* y0 = Y + row + static_cast<long long>(cc) * ldy;
    const bool v0 = row < R && cc < cend, v1 = row < R && cc + 1 < cend;
    double acc[2];
    acc[0] = v0 ? y0[0] : 0.0;
    acc[1] = v1 ? y0[ldy] : 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int i = 4 * kk + (lane & 3);
      const double afr = (row < R && i < w) ? -P[i * ldp + row] : 0.0;
      dmma884(acc, afr, bz[kk]);
    }
    if (v0) y0[0] = acc[0];
    if (v1) y0[ldy] = acc[1];
  }
}

__global__ void __launch_bounds__(kHBThreads, 2) k_house_blocked(const double* __restrict__ Vr,
                                                               const double* __restrict__ lam,
                                                               const long long* __restrict__ lam_off,
                                                               const int* __restrict__ rr, int n,
                                                               double* __restrict__ A, double* __restrict__ Q,
                                                               double* __restrict__ Tw) {
  extern __shared__ double hsm[];
  const int ldp = house_ldp(n);               // panel column stride ≡ 4 mod 16 (conflict-free DMMA fragments)
  double* P = hsm;                            // panel: kHP columns, ld ldp
  double* Tm = P + static_cast<size_t>(kHP) * ldp;  // kHP x kHP (row i, column j at i*kHP + j)
  double* beta = Tm + kHP * kHP;              // kHP
  double* red = beta + kHP;                   // kHBWarps
  // the column order (n ints) is only needed before the first panel: it borrows T's storage;
  // VᵀV of a panel is kept in T's lower triangle until T is complete. 112 KB at n = 400: two
  // CTAs per SM
  int* perm = reinterpret_cast<int*>(Tm);
  const int j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = rr[j];
  const size_t off = static_cast<size_t>(j) * n * n;
  const double* Vj = Vr + off;
  double* Aj = A + off;
  double* Qj = Q + off;
  double* Tj = Tw + static_cast<size_t>(j) * ((n + kHP - 1) / kHP) * kHP * kHP;
  const double* lj = lam + lam_off[j];
  for (int c = tid; c < r; c += blockDim.x) {  // stable descending rank of the eigenvalues
    int rk = 0;
    for (int q = 0; q < r; ++q) rk += (lj[q] > lj[c]) || (lj[q] == lj[c] && q < c);
    perm[rk] = c;
  }
  __syncthreads();
  for (int c = warp; c < r; c += kHBWarps) {  // A[:, c] = Vr[:, perm[c]] / ||.||
    const double* src = Vj + static_cast<size_t>(perm[c]) * n;
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s += src[i] * src[i];
    s = warp_sum(s);
    const double sc = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
    for (int i = lane; i < n; i += 32) Aj[i + static_cast<size_t>(c) * n] = src[i] * sc;
  }
  __syncthreads();
  // ---- factorisation, panel by panel
  for (int p = 0, pi = 0; p < r; p += kHP, ++pi) {
    const int w = min(kHP, r - p), R = n - p;
    for (int c = 0; c < w; ++c)
      for (int i = tid; i < R; i += blockDim.x) P[c * ldp + i] = Aj[(p + i) + static_cast<size_t>(p + c) * n];
    __syncthreads();
    for (int c = 0; c < w; ++c) {  // the panel's reflectors (column norms over the whole CTA)
      double* x = P + c * ldp;
      double s2 = 0.0;
      for (int i = c + tid; i < R; i += blockDim.x) s2 += x[i] * x[i];
      s2 = warp_sum(s2);
      __syncthreads();
      if (lane == 0) red[warp] = s2;
      __syncthreads();
      double nrm2 = 0.0;
      for (int q = 0; q < kHBWarps; ++q) nrm2 += red[q];
      const double alpha = sqrt(nrm2), x0 = x[c];
      const double sg = x0 >= 0.0 ? -alpha : alpha;  // H x = sg e_c
      const double b = alpha > 0.0 ? 1.0 / (sg * (sg - x0)) : 0.0;
      __syncthreads();
      if (tid == 0) {
        x[c] = x0 - sg;  // v_c (the rest of v is x below the diagonal)
        beta[c] = b;
      }
      __syncthreads();
      for (int cc = c + 1 + warp; cc < w; cc += kHBWarps) {  // the panel's own later columns
        double* y = P + cc * ldp;
        double t = 0.0;
        for (int i = c + lane; i < R; i += 32) t += x[i] * y[i];
        t = warp_sum(t) * b;
        for (int i = c + lane; i < R; i += 32) y[i] -= t * x[i];
      }
      __syncthreads();
    }
    for (int c = 0; c < w; ++c)  // store v (and R above it) back; keep V with zeros above the diagonal
      for (int i = tid; i < R; i += blockDim.x) {
        Aj[(p + i) + static_cast<size_t>(p + c) * n] = P[c * ldp + i];
        if (i < c) P[c * ldp + i] = 0.0;
      }
    __syncthreads();
    // T: T_cc = β_c; T[0:c, c] = -β_c T[0:c, 0:c] (V[:, 0:c]ᵀ v_c)
    for (int e = warp; e < w * w; e += kHBWarps) {
      const int a = e / w, bcol = e % w;
      if (a >= bcol) continue;
      double t = 0.0;
      for (int i = bcol + lane; i < R; i += 32) t += P[a * ldp + i] * P[bcol * ldp + i];
      t = warp_sum(t);
      if (lane == 0) Tm[bcol * kHP + a] = t;  // (VᵀV)[a, bcol], a < bcol, parked below the diagonal
    }
    __syncthreads();
    if (warp == 0) {
      for (int c = 0; c < w; ++c) {
        double t = 0.0;
        if (lane < c)
          for (int k = lane; k < c; ++k) t += Tm[lane * kHP + k] * Tm[c * kHP + k];
        __syncwarp();
        if (lane < c) Tm[lane * kHP + c] = -beta[c] * t;
        if (lane == c) Tm[c * kHP + c] = beta[c];
        __syncwarp();
      }
    }
    __syncthreads();
    for (int e = tid; e < kHP * kHP; e += blockDim.x)
      if (e / kHP > e % kHP) Tm[e] = 0.0;  // T is upper triangular
    __syncthreads();
    for (int e = tid; e < kHP * kHP; e += blockDim.x) Tj[pi * kHP * kHP + e] = Tm[e];
    // trailing columns: y <- (I - V T Vᵀ)ᵀ y = y - V Tᵀ (Vᵀ y)
    for (int c0 = p + w + 8 * warp; c0 < r; c0 += 8 * kHBWarps)
      wy_update8(P, ldp, R, w, Tm, true, Aj + p, n, c0, r, lane);
    __syncthreads();
  }
  // ---- Q = H_0 ⋯ H_{r-1} [I_r; 0], panels in reverse
  for (size_t e = tid; e < static_cast<size_t>(n) * r; e += blockDim.x) Qj[e] = (e % (n + 1) == 0) ? 1.0 : 0.0;
  __syncthreads();
  const int np = (r + kHP - 1) / kHP;
  for (int pi = np - 1; pi >= 0; --pi) {
    const int p = pi * kHP, w = min(kHP, r - p), R = n - p;
    for (int c = 0; c < w; ++c)
      for (int i = tid; i < R; i += blockDim.x) P[c * ldp + i] = i < c ? 0.0 : Aj[(p + i) + static_cast<size_t>(p + c) * n];
    for (int e = tid; e < kHP * kHP; e += blockDim.x) Tm[e] = Tj[pi * kHP * kHP + e];
    __syncthreads();
    for (int c0 = p + 8 * warp; c0 < r; c0 += 8 * kHBWarps)
      wy_update8(P, ldp, R, w, Tm, false, Qj + p, n, c0, r, lane);
    __syncthreads();
  }
}

size_t house_blocked_smem(int n) {
  return (static_cast<size_t>(kHP) * house_ldp(n) + kHP * kHP + kHP + kHBWarps) * sizeof(double);
}

// V0[:, :r_j] = Vs[:, :r_j] (m x r_j leading columns, column-major ld m)
__global__ void k_copy_lead(const double* __restrict__ Vs, double* __restrict__ V0, const int* __restrict__ r, int m) {
  const size_t off = static_cast<size_t>(blockIdx.x) * m * m;
  const long long cnt = static_cast<long long>(r[blockIdx.x]) * m;
  for (long long e = threadIdx.x; e < cnt; e += blockDim.x) V0[off + e] = Vs[off + e];
}

std::vector<GemmTask> gram_tasks(Ctx& c, const double* X, double* G, const std::vector<long long>& offX, int tile) {
  std::vector<GemmTask> t;
  const int m = c.m, nt = ceil_div(m, tile);
  for (int j = 0; j < c.J; ++j) {
    const int rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
    for (int tm = 0; tm < nt; ++tm)
      for (int tn = tm; tn < nt; ++tn)  // upper tiles only (Jacobi reads the upper triangle)
        t.push_back({X + offX[j], X + offX[j], G + static_cast<size_t>(j) * m * m, nullptr, nullptr, m, m, rows,
                     std::max(rows, 1), std::max(rows, 1), m, tm, tn, 0.0});
  }
  return t;
}

}  // namespace

void run_pca(Ctx& c) {
  ScopedKernelTimer tk(c, "pca_total");
  const int J = c.J, m = c.m;
  c.S_off.assign(J + 1, 0);
  for (int j = 0; j <= J; ++j) c.S_off[j] = static_cast<long long>(c.h_row_ptr[j]) * m;
  c.S.ensure(std::max<long long>(1, c.S_off[J]));
  const bool reduce = c.cfg.tau_mode != RDD_TAU_OFF;
  for (int j = 0; j < J; ++j)
    if (reduce && c.h_row_ptr[j + 1] == c.h_row_ptr[j])
      throw std::runtime_error("subdomain " + std::to_string(j) + " contains no collocation points");
  // sample matrices: op_applied / psi for the PCA; with tau off the op_applied blocks are H itself
  assemble_samples(c, reduce ? c.cfg.pca_matrix : RDD_PCA_OP_APPLIED, c.S.p, c.S_off);

  c.h_p.assign(J, m);
  c.identity_V = !reduce;
  if (reduce) {
    const size_t mm = static_cast<size_t>(m) * m;
    struct WS {
      double* p;
    };
    WS G{c.ws("pca.G", J * mm)}, V0{c.ws("pca.V0", J * mm)}, lam{c.ws("pca.lam", static_cast<size_t>(J) * m)};
    WS T{nullptr}, W{nullptr}, Vfull{nullptr};
    std::vector<int> ns(J, m);
    std::vector<long long> offm(J);
    for (int j = 0; j < J; ++j) offm[j] = static_cast<long long>(j) * mm;
    // stage 1 only needs a backward-stable basis (absolute criterion); stage 2 works on the graded
    // Gram with the relative criterion. Directions 4 decades (in λ = σ²) below the threshold are
    // not rotated against each other, and convergence is judged on those within 2 decades.
    const double tau2 = c.cfg.tau * c.cfg.tau;
    const bool rel = c.cfg.tau_mode == RDD_TAU_RELATIVE;
    EigOpts s1, s2;
    s1.absolute = 1;
    s1.tol = 1e-14;
    s1.floor_rel = 1e-13;
    s1.conv_rel = 1e-12;
    s1.conv_angle = 1e-8;  // stage 2 refines: stage 1 only has to make the columns of S·V0 graded
    s2.absolute = 0;
    s2.tol = 1e-14;
    s2.floor_rel = rel ? 1e-4 * tau2 : 0.0;
    s2.floor_abs = rel ? 0.0 : 1e-4 * tau2;
    s2.conv_rel = rel ? 1e-2 * tau2 : 0.0;
    s2.conv_abs = rel ? 0.0 : 1e-2 * tau2;
    // rotations by angles below 1e-12 move the kept subspace and σ by less than the parity
    // tolerance; without this the sweep loop keeps chasing re-coupling through the unrotated
    // sub-floor directions (measured: 16 sweeps → 7 at identical projectors and σ)
    s2.conv_angle = 1e-12;
    // stage 1: Gram, pivoted Cholesky G ≈ L Lᵀ (r = numerical rank), Jacobi on the graded LᵀL
    // (r x r: one CTA, few sweeps), Vr = L U, V0 = Householder completion of Vr to an n x n basis
    {
      ScopedKernelTimer tg(c, "gram");
      const int tgr = pick_tile({{m, m}}, true);
      gemm_tn(c, gram_tasks(c, c.S.p, G.p, c.S_off, tgr), tgr);
    }
    WS Lw{c.ws("pca.L", J * mm)}, Vr{c.ws("pca.Vr", J * mm)}, Hw{c.ws("pca.H", J * mm)};
    DBuf<int> dr;
    DBuf<double> dtrace;
    dr.ensure(J);
    dtrace.ensure(J);
    {
      const size_t sm = static_cast<size_t>(m) * (2 * sizeof(double) + 1) + 16;
      if (sm > 32 * 1024)
        RDD_CUDA(cudaFuncSetAttribute(k_pchol, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
      k_pchol<<<J, kPcholThreads, sm, c.stream>>>(G.p, Lw.p, m, c.pca_stop, dr.p, dtrace.p);
      RDD_LAUNCH_CHECK();
    }
    std::vector<int> rj(J);
    std::vector<double> htrace(J);
    dr.download(rj.data(), J, c.stream);
    dtrace.download(htrace.data(), J, c.stream);
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    // path choice: the refined-subspace path resolves every direction above ~1e-7·σmax (σmax² <=
    // trace G); thresholds below that with r < m take the full two-stage path (stage 2 on all m
    // columns). Wide blocks (cluster-sized r) skip the stage-1 Jacobi and refine twice instead.
    bool fast = true;
    int rmax = 0;
    for (int j = 0; j < J; ++j) {
      rmax = std::max(rmax, rj[j]);
      const bool ok = rel ? c.cfg.tau >= 1e-7 : c.cfg.tau >= 1e-7 * std::sqrt(std::max(htrace[j], 0.0));
      if (!(rj[j] == m || ok)) fast = false;
    }
    const bool skip_s1 = fast && rmax > 223;
    std::vector<std::pair<int, int>> rr_pairs, mr_pairs;  // (r_j, r_j) and (m, r_j): tile-size choices
    for (int j = 0; j < J; ++j) {
      rr_pairs.push_back({rj[j], rj[j]});
      mr_pairs.push_back({m, rj[j]});
    }
    const int nref = c.pca_refine > 0 ? c.pca_refine : (skip_s1 ? 2 : 1);
    {
      std::vector<GemmTask> t;
      const int tl = pick_tile(rr_pairs, true);
      for (int j = 0; j < J; ++j) {
        const int nt = ceil_div(rj[j], tl);
        for (int tm = 0; tm < nt; ++tm)
          for (int tn = tm; tn < nt; ++tn)
            t.push_back({Lw.p + offm[j], Lw.p + offm[j], G.p + offm[j], nullptr, nullptr, rj[j], rj[j], m, m, m,
                         rj[j], tm, tn, 0.0});
      }
      gemm_tn(c, t, tl);  // M = LᵀL (upper tiles) over the Gram buffer
    }
    std::vector<long long> offr(J);
    for (int j = 0, e = 0; j < J; e += rj[j], ++j) offr[j] = e;
    if (!skip_s1) {
      batched_syevj(c, G.p, V0.p, lam.p, rj, offm, s1);  // U (r x r, ld r) in V0's buffer
      std::vector<GemmTask> t;
      for (int j = 0; j < J; ++j)
        for (int tm = 0; tm < ceil_div(m, 64); ++tm)
          for (int tn = 0; tn < ceil_div(rj[j], 64); ++tn)
            t.push_back({Lw.p + offm[j], V0.p + offm[j], Vr.p + offm[j], nullptr, nullptr, m, rj[j], rj[j], m, rj[j],
                         m, tm, tn, 0.0});
      gemm_nn(c, t);  // Vr = L U
    }
    // column order for the QR of the refinement: stage-1 eigenvalues, or the pivot order of L
    std::vector<double> horder(static_cast<size_t>(offr[J - 1] + rj[J - 1]));
    for (int j = 0; j < J; ++j)
      for (int q = 0; q < rj[j]; ++q) horder[offr[j] + q] = -static_cast<double>(q);
    double* dorder = c.ws("pca.order", std::max<size_t>(1, horder.size()));
    RDD_CUDA(cudaMemcpyAsync(dorder, horder.data(), sizeof(double) * horder.size(), cudaMemcpyHostToDevice, c.stream));
    DBuf<long long> doffr_sel;
    doffr_sel.upload(offr, c.stream);
    T.p = c.ws("pca.T", std::max<long long>(1, c.S_off[J]));
    W.p = c.ws("pca.W", J * mm);
    Vfull.p = c.ws("pca.Vfull", J * mm);
    if (fast) {
      // one subspace-iteration step from S itself: Y = Sᵀ(S·Vr). Directions with σ_i ≫ the Gram's
      // rounding floor come out accurate to ~ε·σmax/σ_i (the Gram-based Vr only to ε·σmax²/σ_i²),
      // so span(Y) holds the kept subspace to ~1e-10 and the graded Jacobi on (S·Q)ᵀ(S·Q) within it
      // (relative criterion) gives σ and V to the parity tolerance — no m-wide second stage
      for (int it = 0; it < nref; ++it) {
        const double* Vin = it == 0 ? (skip_s1 ? Lw.p : Vr.p) : V0.p;
        {
          ScopedKernelTimer tr(c, "pca_refine");
          std::vector<NNItem> items;
          for (int j = 0; j < J; ++j) {
            const int rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
            items.push_back({c.S.p + c.S_off[j], Vin + offm[j], T.p + c.S_off[j], rows, rj[j], m, std::max(rows, 1), m,
                             std::max(rows, 1)});
          }
          nn_batch(c, items);  // Z = S·V
        }
        {
          ScopedKernelTimer tr(c, "pca_refine");
          std::vector<GemmTask> t;
          const int ty = pick_tile(mr_pairs);
          for (int j = 0; j < J; ++j) {
            const int rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
            for (int tm = 0; tm < ceil_div(m, ty); ++tm)
              for (int tn = 0; tn < ceil_div(rj[j], ty); ++tn)
                t.push_back({c.S.p + c.S_off[j], T.p + c.S_off[j], Hw.p + offm[j], nullptr, nullptr, m, rj[j], rows,
                             std::max(rows, 1), std::max(rows, 1), m, tm, tn, 0.0});
          }
          gemm_tn(c, t, ty);  // Y = Sᵀ·Z
        }
        const size_t sm = static_cast<size_t>(m) * (2 * sizeof(double) + sizeof(int)) + 16;
        if (sm > 32 * 1024)
          RDD_CUDA(cudaFuncSetAttribute(k_house_complete, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sm)));
        const double* ord = (it == 0 && !skip_s1) ? lam.p : dorder;
        ScopedKernelTimer th(c, "pca_house");
        if (m <= kHouseMaxM && rmax >= 192) {  // wide blocks (C3, C5): blocked compact-WY form, same reflectors
          const size_t hsm = house_blocked_smem(m);
          ensure_smem_attr(reinterpret_cast<const void*>(k_house_blocked), hsm);
          double* Tw = c.ws("pca.houseT", static_cast<size_t>(J) * ceil_div(m, kHP) * kHP * kHP);
          k_house_blocked<<<J, kHBThreads, hsm, c.stream>>>(Hw.p, ord, doffr_sel.p, dr.p, m,
                                                            Lw.p == Vin ? Vr.p : Lw.p, V0.p, Tw);
        } else {
          k_house_complete<<<J, kHouseThreads, sm, c.stream>>>(Hw.p, ord, doffr_sel.p, dr.p, m,
                                                               Lw.p == Vin ? Vr.p : Lw.p, V0.p, 1);
        }
        RDD_LAUNCH_CHECK();  // V0[:, :r] = orthonormal basis of span(Y)
      }
      {
        ScopedKernelTimer ts(c, "pca_stage2_gemm");
        std::vector<NNItem> items;
        for (int j = 0; j < J; ++j) {
          const int rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
          items.push_back({c.S.p + c.S_off[j], V0.p + offm[j], T.p + c.S_off[j], rows, rj[j], m, std::max(rows, 1), m,
                           std::max(rows, 1)});
        }
        nn_batch(c, items);  // T_a = S·Q
      }
      {
        ScopedKernelTimer ts(c, "pca_stage2_gemm");
        std::vector<GemmTask> t;
        const int tg = pick_tile(rr_pairs, true);
        for (int j = 0; j < J; ++j) {
          const int rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
          const int nt = ceil_div(rj[j], tg);
          for (int tm = 0; tm < nt; ++tm)
            for (int tn = tm; tn < nt; ++tn)
              t.push_back({T.p + c.S_off[j], T.p + c.S_off[j], G.p + offm[j], nullptr, nullptr, rj[j], rj[j], rows,
                           std::max(rows, 1), std::max(rows, 1), rj[j], tm, tn, 0.0});
        }
        gemm_tn(c, t, tg);  // G_a = T_aᵀ T_a
      }
      batched_syevj(c, G.p, W.p, lam.p, rj, offm, s2);
      {
        std::vector<GemmTask> t;
        const int tv = 64;
        for (int j = 0; j < J; ++j)
          for (int tm = 0; tm < ceil_div(m, tv); ++tm)
            for (int tn = 0; tn < ceil_div(rj[j], tv); ++tn)
              t.push_back({V0.p + offm[j], W.p + offm[j], Vfull.p + offm[j], nullptr, nullptr, m, rj[j], rj[j], m,
                           rj[j], m, tm, tn, 0.0});
        gemm_nn(c, t, tv);  // V = Q W
      }
    } else {
      {
        DBuf<long long> doffr;
        doffr.upload(offr, c.stream);
        const size_t sm = static_cast<size_t>(m) * (2 * sizeof(double) + sizeof(int)) + 16;
        if (sm > 32 * 1024)
          RDD_CUDA(cudaFuncSetAttribute(k_house_complete, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sm)));
        k_house_complete<<<J, kHouseThreads, sm, c.stream>>>(Vr.p, lam.p, doffr.p, dr.p, m, Hw.p, V0.p, 0);
        RDD_LAUNCH_CHECK();
        RDD_CUDA(cudaStreamSynchronize(c.stream));
      }
      // stage 2a: the graded Jacobi on the leading r columns only (T_a = S·V0[:, :r], one CTA per
      // subdomain), V0[:, :r] <- V0[:, :r]·W_a. The full stage 2 below then mostly decouples them
      // from the complement (measured: 7.1 -> ~5 sweeps of the 300-wide Jacobi)
      {
        std::vector<GemmTask> t;
        for (int j = 0; j < J; ++j) {
          const int rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
          for (int tm = 0; tm < ceil_div(rows, 64); ++tm)
            for (int tn = 0; tn < ceil_div(rj[j], 64); ++tn)
              t.push_back({c.S.p + c.S_off[j], V0.p + offm[j], T.p + c.S_off[j], nullptr, nullptr, rows, rj[j], m,
                           std::max(rows, 1), m, std::max(rows, 1), tm, tn, 0.0});
        }
        gemm_nn(c, t);  // T_a
      }
      {
        ScopedKernelTimer ts(c, "pca_stage2_gemm");
        std::vector<GemmTask> t;
        const int tg = pick_tile(rr_pairs, true);
        for (int j = 0; j < J; ++j) {
          const int rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
          const int nt = ceil_div(rj[j], tg);
          for (int tm = 0; tm < nt; ++tm)
            for (int tn = tm; tn < nt; ++tn)
              t.push_back({T.p + c.S_off[j], T.p + c.S_off[j], G.p + offm[j], nullptr, nullptr, rj[j], rj[j], rows,
                           std::max(rows, 1), std::max(rows, 1), rj[j], tm, tn, 0.0});
        }
        gemm_tn(c, t, tg);  // G_a = T_aᵀ T_a
      }
      batched_syevj(c, G.p, W.p, lam.p, rj, offm, s2);
      {
        std::vector<GemmTask> t;
        for (int j = 0; j < J; ++j)
          for (int tm = 0; tm < ceil_div(m, 64); ++tm)
            for (int tn = 0; tn < ceil_div(rj[j], 64); ++tn)
              t.push_back({V0.p + offm[j], W.p + offm[j], Vfull.p + offm[j], nullptr, nullptr, m, rj[j], rj[j], m, rj[j],
                           m, tm, tn, 0.0});
        gemm_nn(c, t);  // V0[:, :r] W_a
        k_copy_lead<<<J, 256, 0, c.stream>>>(Vfull.p, V0.p, dr.p, m);
        RDD_LAUNCH_CHECK();
      }
      // stage 2: T = S V0, G1 = TᵀT, Jacobi on the graded G1
      {
        std::vector<GemmTask> t;
        for (int j = 0; j < J; ++j) {
          const int rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
          for (int tm = 0; tm < ceil_div(rows, 64); ++tm)
            for (int tn = 0; tn < ceil_div(m, 64); ++tn)
              t.push_back({c.S.p + c.S_off[j], V0.p + offm[j], T.p + c.S_off[j], nullptr, nullptr, rows, m, m,
                           std::max(rows, 1), m, std::max(rows, 1), tm, tn, 0.0});
        }
        gemm_nn(c, t);
      }
      gemm_tn(c, gram_tasks(c, T.p, G.p, c.S_off, 64));
      batched_syevj(c, G.p, W.p, lam.p, ns, offm, s2);
      // V = V0 W
      {
        std::vector<GemmTask> t;
        for (int j = 0; j < J; ++j)
          for (int tm = 0; tm < ceil_div(m, 64); ++tm)
            for (int tn = 0; tn < ceil_div(m, 64); ++tn)
              t.push_back({V0.p + offm[j], W.p + offm[j], Vfull.p + offm[j], nullptr, nullptr, m, m, m, m, m, m, tm, tn,
                           0.0});
        gemm_nn(c, t);
      }
    }
    c.Vred.ensure(J * mm);
    c.sigma.ensure(static_cast<size_t>(J) * m);
    c.dp_j.ensure(J);
    const size_t smem = static_cast<size_t>(m) * (sizeof(double) + sizeof(int));
    k_select<<<J, 256, smem, c.stream>>>(lam.p, Vfull.p, c.Vred.p, c.sigma.p, c.dp_j.p, c.row_ptr.p, m,
                                         c.cfg.tau_mode, c.cfg.tau, fast ? dr.p : nullptr,
                                         fast ? doffr_sel.p : nullptr);
    RDD_LAUNCH_CHECK();
    c.dp_j.download(c.h_p.data(), J, c.stream);
    RDD_CUDA(cudaStreamSynchronize(c.stream));
    // the psi route truncates on ω·φ but the system blocks are always operator-applied
    if (c.cfg.pca_matrix == RDD_PCA_PSI) assemble_samples(c, RDD_PCA_OP_APPLIED, c.S.p, c.S_off);
  }
  c.h_col_off.assign(J + 1, 0);
  for (int j = 0; j < J; ++j) c.h_col_off[j + 1] = c.h_col_off[j] + c.h_p[j];
  c.p = c.h_col_off[J];
  c.H_off.assign(J + 1, 0);
  for (int j = 0; j < J; ++j)
    c.H_off[j + 1] = c.H_off[j] + static_cast<long long>(c.h_row_ptr[j + 1] - c.h_row_ptr[j]) * c.h_p[j];
  c.dcol_off.upload(c.h_col_off, c.stream);
  c.dH_off.upload(c.H_off, c.stream);
}

// H_j = S_j V_j (reduction.hpp:133 by linearity) or H = S when V = I.
void project_blocks(Ctx& c) {
  ScopedKernelTimer tk(c, "project");
  if (c.identity_V) {
    c.H = c.S.p;
    return;
  }
  const int J = c.J, m = c.m;
  c.Hbuf.ensure(std::max<long long>(1, c.H_off[J]));
  std::vector<NNItem> items;
  for (int j = 0; j < J; ++j) {
    const int rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
    items.push_back({c.S.p + c.S_off[j], c.Vred.p + static_cast<size_t>(j) * m * m, c.Hbuf.p + c.H_off[j], rows,
                     c.h_p[j], m, std::max(rows, 1), m, std::max(rows, 1)});
  }
  nn_batch(c, items);  // H_j = S_j·V_j
  c.H = c.Hbuf.p;
}

}  // namespace rdd
