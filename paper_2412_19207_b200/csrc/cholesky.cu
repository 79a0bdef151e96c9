// cholesky.cu — K8: batched blocked Cholesky and explicit SPD inverse for the Schwarz local
// matrices A_i = (HᵀH)[S_i, S_i] (schwarz.hpp:112-130).
//
// The reference pseudo-inverts A_i through a full eigendecomposition (schwarz.hpp:131-146,
// ~9n³ flops). When every eigenvalue is above the reference's cutoff (1e-12·λmax) that
// pseudo-inverse *is* A_i⁻¹, which costs n³ flops via Cholesky: A = LLᵀ (right-looking, 64-wide
// panels: diagonal POTRF and panel TRSM in shared memory, trailing SYRK/GEMM on DMMA), then
// M = L⁻¹ (diagonal TRTRI in shared memory + DMMA block-row updates), then A⁻¹ = MᵀM (DMMA).
// Matrices of different sizes are processed together; each step launches only the work of the
// matrices still active. A failed pivot flags the matrix for the eigen fallback (schwarz.cu).
#include <algorithm>

#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int NB = 64;
constexpr int kPairSmem = 2 * NB * (NB + 1) * sizeof(double);

struct Mat {
  long long off;  // element offset of the matrix
  int n;          // order (= leading dimension)
};

// A[k-block, k-block] <- chol (lower); pads beyond n act as identity
__global__ void k_potrf_diag(double* __restrict__ A, const Mat* __restrict__ mats, const int* __restrict__ act, int k,
                             int* __restrict__ fail) {
  __shared__ double s[NB][NB + 1];
  const Mat M = mats[act[blockIdx.x]];
  const int k0 = k * NB, bs = min(NB, M.n - k0);
  double* a = A + M.off + k0 + static_cast<long long>(k0) * M.n;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e % NB, c = e / NB;
    s[r][c] = (r < bs && c < bs) ? a[r + static_cast<long long>(c) * M.n] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int c = 0; c < NB; ++c) {
    __shared__ double d;
    if (threadIdx.x == 0) {
      const double v = s[c][c];
      if (!(v > 0.0)) fail[act[blockIdx.x]] = 1;
      d = sqrt(fmax(v, 1e-300));
      s[c][c] = d;
    }
    __syncthreads();
    for (int r = c + 1 + threadIdx.x; r < NB; r += blockDim.x) s[r][c] /= d;
    __syncthreads();
    for (int e = threadIdx.x; e < (NB - c - 1) * (NB - c - 1); e += blockDim.x) {
      const int r = c + 1 + e % (NB - c - 1), q = c + 1 + e / (NB - c - 1);
      if (q <= r) s[r][q] -= s[r][c] * s[q][c];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e % NB, c = e / NB;
    if (r < bs && c < bs) a[r + static_cast<long long>(c) * M.n] = r >= c ? s[r][c] : 0.0;
  }
}

// panel: X = A[i-block, k-block] L_kk^{-T} for the task's row block i > k
__global__ void k_trsm_panel(double* __restrict__ A, const Mat* __restrict__ mats, const int2* __restrict__ tasks,
                             int k) {
  extern __shared__ double dsm[];
  double(*L)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm);
  double(*X)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + NB * (NB + 1));
  const int2 t = tasks[blockIdx.x];
  const Mat M = mats[t.x];
  const int k0 = k * NB, bs = min(NB, M.n - k0);
  const int i0 = t.y * NB, rs = min(NB, M.n - i0);
  const double* l = A + M.off + k0 + static_cast<long long>(k0) * M.n;
  double* a = A + M.off + i0 + static_cast<long long>(k0) * M.n;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e % NB, c = e / NB;
    L[r][c] = (r < bs && c < bs) ? l[r + static_cast<long long>(c) * M.n] : (r == c ? 1.0 : 0.0);
    X[r][c] = (r < rs && c < bs) ? a[r + static_cast<long long>(c) * M.n] : 0.0;
  }
  __syncthreads();
  const int r = threadIdx.x;  // one row per thread, forward substitution over columns
  if (r < rs) {
    for (int c = 0; c < bs; ++c) {
      double v = X[r][c];
      for (int q = 0; q < c; ++q) v -= X[r][q] * L[c][q];
      X[r][c] = v / L[c][c];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int rr = e % NB, c = e / NB;
    if (rr < rs && c < bs) a[rr + static_cast<long long>(c) * M.n] = X[rr][c];
  }
}

// M_kk = L_kk^{-1} (lower) for every diagonal block; task = (matrix, k)
__global__ void k_trtri_diag(const double* __restrict__ A, double* __restrict__ Minv, const Mat* __restrict__ mats,
                             const int2* __restrict__ tasks) {
  extern __shared__ double dsm[];
  double(*L)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm);
  double(*X)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dsm + NB * (NB + 1));
  const int2 t = tasks[blockIdx.x];
  const Mat M = mats[t.x];
  const int k0 = t.y * NB, bs = min(NB, M.n - k0);
  const double* l = A + M.off + k0 + static_cast<long long>(k0) * M.n;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e % NB, c = e / NB;
    L[r][c] = (r < bs && c < bs) ? l[r + static_cast<long long>(c) * M.n] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  const int c = threadIdx.x;  // column c of L^{-1}: forward substitution down the rows
  if (c < NB) {
    for (int r = 0; r < NB; ++r) {
      double v = (r == c) ? 1.0 : 0.0;
      for (int q = c; q < r; ++q) v -= L[r][q] * X[q][c];
      X[r][c] = r < c ? 0.0 : v / L[r][r];
    }
  }
  __syncthreads();
  double* m = Minv + M.off + k0 + static_cast<long long>(k0) * M.n;
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int r = e % NB, cc = e / NB;
    if (r < bs && cc < bs) m[r + static_cast<long long>(cc) * M.n] = X[r][cc];
  }
}

__global__ void k_frob(const double* __restrict__ A, const Mat* __restrict__ mats, double* __restrict__ out) {
  const Mat M = mats[blockIdx.x];
  double s = 0.0;
  for (long long e = threadIdx.x; e < static_cast<long long>(M.n) * M.n; e += blockDim.x) {
    const double v = A[M.off + e];
    s += v * v;
  }
  __shared__ double sh[32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    s = warp_sum(s);
    if (threadIdx.x == 0) out[blockIdx.x] = sqrt(s);
  }
}

// λmax of symmetric PSD matrices by power iteration (one CTA per matrix, x in shared memory)
__global__ void k_power(const double* __restrict__ A, const Mat* __restrict__ mats, int iters,
                        double* __restrict__ out) {
  extern __shared__ double x[];
  __shared__ double sh[32];
  __shared__ double nrm;
  const Mat M = mats[blockIdx.x];
  const double* a = A + M.off;
  double* y = x + M.n;
  for (int i = threadIdx.x; i < M.n; i += blockDim.x) x[i] = 1.0 + 0.25 * sin(0.7 * i + 0.3);
  __syncthreads();
  double lam = 0.0;
  for (int it = 0; it <= iters; ++it) {
    double part = 0.0;
    for (int r = threadIdx.x; r < M.n; r += blockDim.x) {
      double s = 0.0;
      for (int c = 0; c < M.n; ++c) s += a[r + static_cast<long long>(c) * M.n] * x[c];
      y[r] = s;
      part += s * s;
    }
    part = warp_sum(part);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0, xx = 0.0;
      for (int w = 0; w < (blockDim.x >> 5); ++w) t += sh[w];
      for (int i = 0; i < M.n; ++i) xx += x[i] * x[i];
      nrm = sqrt(t);
      lam = nrm / sqrt(xx);
      sh[0] = lam;
    }
    __syncthreads();
    lam = sh[0];
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int i = threadIdx.x; i < M.n; i += blockDim.x) x[i] = y[i] * inv;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = lam;
}

// copy the lower triangle onto the upper one
__global__ void k_mirror_lower(double* __restrict__ P, const Mat* __restrict__ mats) {
  const Mat M = mats[blockIdx.x];
  double* a = P + M.off;
  for (long long e = threadIdx.x; e < static_cast<long long>(M.n) * M.n; e += blockDim.x) {
    const int r = static_cast<int>(e % M.n), cc = static_cast<int>(e / M.n);
    if (r < cc) a[e] = a[cc + static_cast<long long>(r) * M.n];
  }
}

}  // namespace

std::vector<double> batched_power(Ctx& c, const double* A, const std::vector<int>& n,
                                  const std::vector<long long>& off, int iters) {
  ScopedKernelTimer tk(c, "power");
  const int B = static_cast<int>(n.size());
  std::vector<double> out(B, 0.0);
  if (B == 0) return out;
  std::vector<Mat> mats(B);
  int nmax = 0;
  for (int i = 0; i < B; ++i) {
    mats[i] = {off[i], n[i]};
    nmax = std::max(nmax, n[i]);
  }
  DBuf<Mat> dm;
  DBuf<double> d;
  dm.upload(mats, c.stream);
  d.ensure(B);
  const size_t smem = 2 * sizeof(double) * nmax;
  if (smem > 48 * 1024)
    RDD_CUDA(cudaFuncSetAttribute(k_power, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  k_power<<<B, 256, smem, c.stream>>>(A, dm.p, iters, d.p);
  RDD_LAUNCH_CHECK();
  d.download(out.data(), B, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  return out;
}

// In: A (batch at off[i], order n[i], symmetric, full storage) — destroyed (holds L).
// Out: P = A^{-1} (full, same layout); fail[i] = 1 when a pivot was not positive;
// frob_A[i], frob_P[i] Frobenius norms (cond(A) <= ||A||_F ||A^{-1}||_F).
void batched_spd_inverse(Ctx& c, double* A, double* P, const std::vector<int>& n, const std::vector<long long>& off,
                         std::vector<int>& fail, std::vector<double>& frob_A, std::vector<double>& frob_P,
                         const std::vector<long long>* offP_in) {
  const std::vector<long long>& offP = offP_in ? *offP_in : off;
  ScopedKernelTimer tk(c, "spd_inverse");
  const int B = static_cast<int>(n.size());
  fail.assign(B, 0);
  frob_A.assign(B, 0.0);
  frob_P.assign(B, 0.0);
  if (B == 0) return;
  std::vector<Mat> mats(B);
  int nmax = 0;
  for (int i = 0; i < B; ++i) {
    mats[i] = {off[i], n[i]};
    nmax = std::max(nmax, n[i]);
  }
  RDD_CUDA(cudaFuncSetAttribute(k_trsm_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmem));
  RDD_CUDA(cudaFuncSetAttribute(k_trtri_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmem));
  DBuf<Mat> dm;
  DBuf<int> dfail, dact;
  DBuf<int2> dt;
  DBuf<double> dfa, dfp;
  struct WS {
    double* p;
  } Mi{nullptr}, tmp{nullptr};
  dm.upload(mats, c.stream);
  dfail.zero(B, c.stream);
  dfa.ensure(B);
  dfp.ensure(B);
  k_frob<<<B, 256, 0, c.stream>>>(A, dm.p, dfa.p);
  RDD_LAUNCH_CHECK();
  const int nbmax = ceil_div(nmax, NB);
  // ---- factor
  for (int k = 0; k < nbmax; ++k) {
    std::vector<int> act;
    std::vector<int2> pan;
    std::vector<GemmTask> upd;
    for (int i = 0; i < B; ++i) {
      const int nb = ceil_div(n[i], NB);
      if (k >= nb) continue;
      act.push_back(i);
      const int k0 = k * NB, bk = std::min(NB, n[i] - k0);
      for (int ib = k + 1; ib < nb; ++ib) {
        pan.push_back(make_int2(i, ib));
        const int bi = std::min(NB, n[i] - ib * NB);
        for (int jb = k + 1; jb <= ib; ++jb) {
          const int bj = std::min(NB, n[i] - jb * NB);
          double* base = A + off[i];
          GemmTask t{};
          t.A = base + ib * NB + static_cast<long long>(k0) * n[i];
          t.B = base + jb * NB + static_cast<long long>(k0) * n[i];
          t.Cm = base + ib * NB + static_cast<long long>(jb * NB) * n[i];
          t.M = bi;
          t.N = bj;
          t.K = bk;
          t.lda = t.ldb = t.ldc = n[i];
          t.beta = 1.0;
          t.alpha = -1.0;
          upd.push_back(t);
        }
      }
    }
    dact.upload(act, c.stream);
    k_potrf_diag<<<static_cast<int>(act.size()), 256, 0, c.stream>>>(A, dm.p, dact.p, k, dfail.p);
    RDD_LAUNCH_CHECK();
    if (!pan.empty()) {
      dt.upload(pan, c.stream);
      k_trsm_panel<<<static_cast<int>(pan.size()), NB, kPairSmem, c.stream>>>(A, dm.p, dt.p, k);
      RDD_LAUNCH_CHECK();
    }
    gemm_nt(c, upd);  // synchronizes (task-buffer lifetime), so dact/dt can be reused
  }
  // ---- M = L^{-1}
  {
    const size_t msz = static_cast<size_t>(off[B - 1] + static_cast<long long>(n[B - 1]) * n[B - 1]);
    Mi.p = c.ws("chol.Minv", msz);
    RDD_CUDA(cudaMemsetAsync(Mi.p, 0, msz * sizeof(double), c.stream));
  }
  {
    std::vector<int2> diag;
    for (int i = 0; i < B; ++i)
      for (int k = 0; k < ceil_div(n[i], NB); ++k) diag.push_back(make_int2(i, k));
    dt.upload(diag, c.stream);
    k_trtri_diag<<<static_cast<int>(diag.size()), NB, kPairSmem, c.stream>>>(A, Mi.p, dm.p, dt.p);
    RDD_LAUNCH_CHECK();
  }
  long long tmp_sz = 0;
  std::vector<long long> toff(B);
  for (int i = 0; i < B; ++i) {
    toff[i] = tmp_sz;
    tmp_sz += static_cast<long long>(NB) * n[i];
  }
  tmp.p = c.ws("chol.tmp", std::max<long long>(1, tmp_sz));
  for (int ib = 1; ib < nbmax; ++ib) {
    std::vector<GemmTask> g1, g2;
    for (int i = 0; i < B; ++i) {
      if (ib >= ceil_div(n[i], NB)) continue;
      const int bi = std::min(NB, n[i] - ib * NB), w = ib * NB;
      double* L = A + off[i];
      double* Mm = Mi.p + off[i];
      for (int tn = 0; tn < ib; ++tn) {
        GemmTask t{};  // tmp[:, tn] = L[ib, tn*64:w] M[tn*64:w, tn]  (M is lower triangular)
        const int k0 = tn * NB;
        t.A = L + ib * NB + static_cast<long long>(k0) * n[i];
        t.B = Mm + k0 + static_cast<long long>(k0) * n[i];
        t.Cm = tmp.p + toff[i] + static_cast<long long>(k0) * NB;
        t.M = bi;
        t.N = NB;
        t.K = w - k0;
        t.lda = n[i];
        t.ldb = n[i];
        t.ldc = NB;
        t.tn = 0;
        t.alpha = 1.0;
        g1.push_back(t);
        GemmTask u{};  // M[ib, 0:w] = -M_ii tmp
        u.A = Mm + ib * NB + static_cast<long long>(ib * NB) * n[i];
        u.B = tmp.p + toff[i];
        u.Cm = Mm + ib * NB;
        u.M = bi;
        u.N = w;
        u.K = bi;
        u.lda = n[i];
        u.ldb = NB;
        u.ldc = n[i];
        u.tn = tn;
        u.alpha = -1.0;
        g2.push_back(u);
      }
    }
    gemm_nn(c, g1);
    gemm_nn(c, g2);
  }
  // ---- P = Mᵀ M, lower tiles only (M(k, i) = 0 for k < i), then mirrored
  std::vector<GemmTask> g;
  for (int i = 0; i < B; ++i)
    for (int tm = 0; tm < ceil_div(n[i], 64); ++tm)
      for (int tn = 0; tn <= tm; ++tn) {
        GemmTask t{};
        const int k0 = tm * 64;  // rows of M below the tile's first output row
        t.A = Mi.p + off[i] + k0;
        t.B = Mi.p + off[i] + k0;
        t.Cm = P + offP[i];
        t.M = t.N = n[i];
        t.K = n[i] - k0;
        t.lda = t.ldb = t.ldc = n[i];
        t.tm = tm;
        t.tn = tn;
        t.alpha = 1.0;
        g.push_back(t);
      }
  gemm_tn(c, g);
  {
    std::vector<Mat> pm(B);
    for (int i = 0; i < B; ++i) pm[i] = {offP[i], n[i]};
    DBuf<Mat> dpm;
    dpm.upload(pm, c.stream);
    k_mirror_lower<<<B, 256, 0, c.stream>>>(P, dpm.p);
    RDD_LAUNCH_CHECK();
    dm.upload(pm, c.stream);  // Frobenius norms of the outputs
  }
  k_frob<<<B, 256, 0, c.stream>>>(P, dm.p, dfp.p);
  RDD_LAUNCH_CHECK();
  dfail.download(fail.data(), B, c.stream);
  dfa.download(frob_A.data(), B, c.stream);
  dfp.download(frob_P.data(), B, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace rdd
