// matvec.cu — K6 column equilibration and K9/K10 block-sparse H·w, Hᵀ·r.
//
// H·w (assembly.hpp:110-121) scatter-adds each block's rows into y; here each global row is
// owned by one thread that gathers the ≤2^d covering blocks' rows (owner-computes, no atomics;
// the per-row sum visits blocks in ascending j like the reference). Hᵀ·r (assembly.hpp:123-133)
// is one warp per column: a contiguous column of a column-major block against r gathered through
// rows_j. Both are HBM-bound streams over H (8·nnz bytes each).
#include "ctx.hpp"

namespace rdd {

namespace {

// one warp per column: 2-norm, zero -> 1 (runner.hpp:96-99), then H col /= s (assembly.hpp:197-204)
__global__ void k_colnorm_scale(double* __restrict__ H, const long long* __restrict__ H_off,
                                const int* __restrict__ row_ptr, const int* __restrict__ col_off,
                                const int* __restrict__ col_owner, int p, double* __restrict__ scales, int apply) {
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (col >= p) return;
  const int j = col_owner[col];
  const int k = col - col_off[j];
  const int rows = row_ptr[j + 1] - row_ptr[j];
  double* h = H + H_off[j] + static_cast<long long>(k) * rows;
  double s = 0.0;
  for (int r = lane; r < rows; r += 32) s += h[r] * h[r];
  s = sqrt(warp_sum(s));
  if (s == 0.0) s = 1.0;
  if (!apply) s = 1.0;
  if (lane == 0) scales[col] = s;
  if (apply && s != 1.0)
    for (int r = lane; r < rows; r += 32) h[r] = h[r] / s;
}

__global__ void k_matvec(const double* __restrict__ H, const long long* __restrict__ H_off,
                         const int* __restrict__ row_ptr, const int* __restrict__ col_off,
                         const int* __restrict__ cov_n, const int* __restrict__ cov_j, const int* __restrict__ cov_r,
                         int maxcov, int N, const double* __restrict__ w, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double acc = 0.0;
  const int nc = cov_n[i];
  for (int s = 0; s < nc; ++s) {
    const int j = cov_j[static_cast<size_t>(i) * maxcov + s];
    const int r = cov_r[static_cast<size_t>(i) * maxcov + s];
    const int rows = row_ptr[j + 1] - row_ptr[j];
    const int c0 = col_off[j], pj = col_off[j + 1] - c0;
    const double* h = H + H_off[j] + r;
    double t = 0.0;
    for (int k = 0; k < pj; ++k) t += h[static_cast<long long>(k) * rows] * w[c0 + k];
    acc += t;
  }
  y[i] = acc;
}

__global__ void k_matvec_t(const double* __restrict__ H, const long long* __restrict__ H_off,
                           const int* __restrict__ row_ptr, const int* __restrict__ row_idx,
                           const int* __restrict__ col_off, const int* __restrict__ col_owner, int p,
                           const double* __restrict__ r, double* __restrict__ out) {
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (col >= p) return;
  const int j = col_owner[col];
  const int k = col - col_off[j];
  const int r0 = row_ptr[j], rows = row_ptr[j + 1] - r0;
  const double* h = H + H_off[j] + static_cast<long long>(k) * rows;
  double s = 0.0;
  for (int q = lane; q < rows; q += 32) s += h[q] * r[row_idx[r0 + q]];
  s = warp_sum(s);
  if (lane == 0) out[col] = s;
}

}  // namespace

void ensure_col_owner(Ctx& c) {
  std::vector<int> own(c.p);
  for (int j = 0; j < c.J; ++j)
    for (int k = c.h_col_off[j]; k < c.h_col_off[j + 1]; ++k) own[k] = j;
  c.h_owner = own;
  c.downer.upload(own, c.stream);
}

void column_norms_scale(Ctx& c, bool equilibrate) {
  ScopedKernelTimer tk(c, "equilibrate");
  c.scales.ensure(std::max(1, c.p));
  const int threads = 256;
  k_colnorm_scale<<<ceil_div(static_cast<long long>(c.p) * 32, threads), threads, 0, c.stream>>>(
      c.H, c.dH_off.p, c.row_ptr.p, c.dcol_off.p, c.downer.p, c.p, c.scales.p, equilibrate ? 1 : 0);
  RDD_LAUNCH_CHECK();
}

void matvec_dev(Ctx& c, const double* w, double* y) {
  ScopedKernelTimer tk(c, "matvec");
  k_matvec<<<ceil_div(c.N, 256), 256, 0, c.stream>>>(c.H, c.dH_off.p, c.row_ptr.p, c.dcol_off.p, c.cov_n.p, c.cov_j.p,
                                                     c.cov_r.p, c.maxcov, c.N, w, y);
  RDD_LAUNCH_CHECK();
}

void matvec_t_dev(Ctx& c, const double* r, double* out) {
  ScopedKernelTimer tk(c, "matvec_t");
  k_matvec_t<<<ceil_div(static_cast<long long>(c.p) * 32, 256), 256, 0, c.stream>>>(
      c.H, c.dH_off.p, c.row_ptr.p, c.row_idx.p, c.dcol_off.p, c.downer.p, c.p, r, out);
  RDD_LAUNCH_CHECK();
}

}  // namespace rdd
