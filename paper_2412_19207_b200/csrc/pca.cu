// pca.cu — K3-K5: per-subdomain PCA truncation (reduction.hpp:89-109) on the device.
//
// The reference takes a thin JacobiSVD of each sample block S_j (rows_j x m) and keeps the
// right singular vectors with σ > τ. A Gram matrix alone cannot reproduce that: SᵀS squares
// the condition number, so eigenvalues near a relative threshold of 1e-6 (λ ~ 1e-12 λmax) carry
// O(1e-4) relative error and the kept subspace O(1e-4) error (SURVEY §7.3 hard part 1). The
// device path therefore runs two Jacobi stages:
//   1. G = SᵀS (DMMA), Jacobi -> V0 (backward stable, absolute accuracy only);
//   2. T = S·V0 (DMMA), G1 = TᵀT (DMMA) — a graded, nearly diagonal matrix whose entries are
//      accurate relative to sqrt(g_ii g_jj) — Jacobi with the relative threshold -> W, whose
//      eigenvalues are relatively accurate (Demmel–Veselić); V = V0·W, σ_i = sqrt(λ_i(G1)).
// Then: sort σ non-increasing, keep σ > τ (strict; τ relative to σ_max in RDD_TAU_RELATIVE
// mode), floor p_j >= 1, canonical signs (first nonzero entry of each kept column >= 0), and
// H_j = S_j·V_j (DMMA) — by linearity equal to assembling the reduced jets (reduction.hpp:122-139).
#include <algorithm>

#include "ctx.hpp"

namespace rdd {

namespace {

// per subdomain: sort eigenvalues descending, threshold, reorder + sign-canonicalise V
__global__ void k_select(const double* __restrict__ lam, const double* __restrict__ Vin, double* __restrict__ Vout,
                         double* __restrict__ sig, int* __restrict__ p_out, const int* __restrict__ row_ptr, int m,
                         int tau_mode, double tau) {
  extern __shared__ double sm[];
  double* s = sm;                              // m sigma
  int* perm = reinterpret_cast<int*>(s + m);   // m
  __shared__ int keep;
  const int j = blockIdx.x;
  const double* L = lam + static_cast<size_t>(j) * m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) s[i] = sqrt(fmax(L[i], 0.0));
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {  // stable descending rank
    int rk = 0;
    for (int k = 0; k < m; ++k) rk += (s[k] > s[i]) || (s[k] == s[i] && k < i);
    perm[rk] = i;
  }
  __syncthreads();
  const int rows = row_ptr[j + 1] - row_ptr[j];
  const int nsv = min(rows, m);  // thin SVD: min(rows, m) singular values
  if (threadIdx.x == 0) {
    const double smax = s[perm[0]];
    const double thr = tau_mode == RDD_TAU_RELATIVE ? tau * smax : tau;
    int k = 0;
    for (int i = 0; i < nsv; ++i)
      if (s[perm[i]] > thr) ++k;
    keep = max(k, 1);
    p_out[j] = keep;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) sig[static_cast<size_t>(j) * m + i] = i < nsv ? s[perm[i]] : 0.0;
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

std::vector<GemmTask> gram_tasks(Ctx& c, const double* X, double* G, const std::vector<long long>& offX) {
  std::vector<GemmTask> t;
  const int m = c.m, nt = ceil_div(m, 64);
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
    // stage 1: Gram + Jacobi
    gemm_tn(c, gram_tasks(c, c.S.p, G.p, c.S_off));
    batched_syevj(c, G.p, V0.p, lam.p, ns, offm, s1);
    // stage 2: T = S V0, G1 = TᵀT, Jacobi on the graded G1
    T.p = c.ws("pca.T", std::max<long long>(1, c.S_off[J]));
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
    gemm_tn(c, gram_tasks(c, T.p, G.p, c.S_off));
    W.p = c.ws("pca.W", J * mm);
    batched_syevj(c, G.p, W.p, lam.p, ns, offm, s2);
    // V = V0 W
    Vfull.p = c.ws("pca.Vfull", J * mm);
    {
      std::vector<GemmTask> t;
      for (int j = 0; j < J; ++j)
        for (int tm = 0; tm < ceil_div(m, 64); ++tm)
          for (int tn = 0; tn < ceil_div(m, 64); ++tn)
            t.push_back({V0.p + offm[j], W.p + offm[j], Vfull.p + offm[j], nullptr, nullptr, m, m, m, m, m, m, tm, tn,
                         0.0});
      gemm_nn(c, t);
    }
    c.Vred.ensure(J * mm);
    c.sigma.ensure(static_cast<size_t>(J) * m);
    c.dp_j.ensure(J);
    const size_t smem = static_cast<size_t>(m) * (sizeof(double) + sizeof(int));
    k_select<<<J, 256, smem, c.stream>>>(lam.p, Vfull.p, c.Vred.p, c.sigma.p, c.dp_j.p, c.row_ptr.p, m,
                                         c.cfg.tau_mode, c.cfg.tau);
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
  std::vector<GemmTask> t;
  for (int j = 0; j < J; ++j) {
    const int rows = c.h_row_ptr[j + 1] - c.h_row_ptr[j];
    for (int tm = 0; tm < ceil_div(rows, 64); ++tm)
      for (int tn = 0; tn < ceil_div(c.h_p[j], 64); ++tn)
        t.push_back({c.S.p + c.S_off[j], c.Vred.p + static_cast<size_t>(j) * m * m, c.Hbuf.p + c.H_off[j], nullptr,
                     nullptr, rows, c.h_p[j], m, std::max(rows, 1), m, std::max(rows, 1), tm, tn, 0.0});
  }
  gemm_nn(c, t);
  c.H = c.Hbuf.p;
}

}  // namespace rdd
