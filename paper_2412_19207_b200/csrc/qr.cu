// qr.cu — §8(f) row 3: the dense column-pivoted QR least-squares solve of the reference's
// qr_direct path (krylov.hpp:97-101 `qr_least_squares`, runner.hpp:217-222: densify H, then
// ColPivHouseholderQR::solve) on the device.
//
// Householder QR with column pivoting in the LAPACK dlaqp2 form: per column i the pivot is the
// first trailing column of largest downdated norm, the reflector is generated as dlarfg does, the
// trailing columns are updated one CTA per column (dot with v, then the rank-1 correction), and
// the partial norms are downdated — recomputed from the column when cancellation makes the
// downdate unreliable (the LAPACK rule). QᵀF follows the same per-column kernel; the rank follows
// Eigen's rule (|R_ii| > ε·min(M,N)·max|R_ii|) and the basic solution is scattered back through
// the pivots. HBM-bound: Σ_i (M-i)(N-i) elements streamed twice and written once.
#include <algorithm>
#include <cfloat>

#include "ctx.hpp"

namespace rdd {

namespace {

constexpr int kQT = 512;

__device__ __forceinline__ double block_sum_q(double v, double* sh) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) sh[0] = t;
  }
  __syncthreads();
  return sh[0];
}

// scatter the blocks into the dense N x p matrix (assembly.hpp:206-215), zero-initialised
__global__ void k_densify(const double* __restrict__ H, const long long* __restrict__ H_off,
                          const int* __restrict__ row_ptr, const int* __restrict__ row_idx,
                          const int* __restrict__ col_off, int N, double* __restrict__ D) {
  const int j = blockIdx.y;
  const int r0 = row_ptr[j], rows = row_ptr[j + 1] - r0;
  const int c0 = col_off[j], pj = col_off[j + 1] - c0;
  for (int k = blockIdx.x; k < pj; k += gridDim.x) {
    const double* src = H + H_off[j] + static_cast<long long>(k) * rows;
    double* dst = D + static_cast<long long>(c0 + k) * N;
    for (int q = threadIdx.x; q < rows; q += blockDim.x) dst[row_idx[r0 + q]] = src[q];
  }
}

// column norms (initial vn1 = vn2)
__global__ void k_colnorms(const double* __restrict__ A, int M, int N, double* __restrict__ vn1,
                           double* __restrict__ vn2) {
  __shared__ double sh[32];
  const int j = blockIdx.x;
  const double* a = A + static_cast<long long>(j) * M;
  double s = 0.0;
  for (int r = threadIdx.x; r < M; r += blockDim.x) s += a[r] * a[r];
  s = block_sum_q(s, sh);
  if (threadIdx.x == 0) vn1[j] = vn2[j] = sqrt(s);
}

// step i, part 1 (one CTA): pivot = first argmax of vn1[i:N]; swap columns i and pivot; generate
// the reflector of A[i:M, i] (dlarfg): A[i,i] = beta, A[i+1:, i] = v (v_i = 1 implicit), tau[i]
__global__ void __launch_bounds__(kQT) k_qr_pivot(double* __restrict__ A, int M, int N, int i, double* __restrict__ vn1,
                                                  double* __restrict__ vn2, int* __restrict__ jpvt,
                                                  double* __restrict__ tau) {
  __shared__ double sh[32];
  __shared__ int shi[32];
  __shared__ int pvt;
  double bv = -1.0;
  int bi = N;
  for (int j = i + threadIdx.x; j < N; j += blockDim.x)
    if (vn1[j] > bv) {
      bv = vn1[j];
      bi = j;
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
  if ((threadIdx.x & 31) == 0) {
    sh[threadIdx.x >> 5] = bv;
    shi[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = sh[0];
    int ix = shi[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (sh[w] > v || (sh[w] == v && shi[w] < ix)) {
        v = sh[w];
        ix = shi[w];
      }
    pvt = ix < N ? ix : i;
  }
  __syncthreads();
  const int p = pvt;
  double* ai = A + static_cast<long long>(i) * M;
  if (p != i) {
    double* ap = A + static_cast<long long>(p) * M;
    for (int r = threadIdx.x; r < M; r += blockDim.x) {
      const double t = ai[r];
      ai[r] = ap[r];
      ap[r] = t;
    }
    if (threadIdx.x == 0) {
      const int t = jpvt[i];
      jpvt[i] = jpvt[p];
      jpvt[p] = t;
      vn1[p] = vn1[i];
      vn2[p] = vn2[i];
    }
  }
  __syncthreads();
  double s = 0.0;
  for (int r = i + 1 + threadIdx.x; r < M; r += blockDim.x) s += ai[r] * ai[r];
  const double xnorm = sqrt(block_sum_q(s, sh));
  const double alpha = ai[i];
  double t = 0.0, scale = 1.0, beta = alpha;
  if (xnorm > 0.0) {
    beta = -copysign(hypot(alpha, xnorm), alpha);
    t = (beta - alpha) / beta;
    scale = 1.0 / (alpha - beta);
  }
  __syncthreads();
  if (xnorm > 0.0)
    for (int r = i + 1 + threadIdx.x; r < M; r += blockDim.x) ai[r] *= scale;
  if (threadIdx.x == 0) {
    ai[i] = beta;
    tau[i] = t;
  }
}

// step i, part 2: columns j in (i, ncols) of X (A itself, or F with norms == nullptr):
// X[i:, j] -= tau v (vᵀ X[i:, j]); for A, downdate vn1/vn2 (dlaqp2)
__global__ void __launch_bounds__(kQT) k_qr_apply(const double* __restrict__ A, int M, int i, const double* __restrict__ tau,
                                                  double* __restrict__ X, int ldx, int j0, int ncols,
                                                  double* __restrict__ vn1, double* __restrict__ vn2) {
  __shared__ double sh[32];
  const int j = j0 + blockIdx.x;
  if (j >= ncols) return;
  const double t = tau[i];
  const double* v = A + static_cast<long long>(i) * M;  // v_i = 1 implicit
  double* x = X + static_cast<long long>(j) * ldx;
  if (t != 0.0) {
    double s = threadIdx.x == 0 ? x[i] : 0.0;
    for (int r = i + 1 + threadIdx.x; r < M; r += blockDim.x) s += v[r] * x[r];
    const double w = t * block_sum_q(s, sh);
    if (threadIdx.x == 0) x[i] -= w;
    for (int r = i + 1 + threadIdx.x; r < M; r += blockDim.x) x[r] -= w * v[r];
  }
  if (!vn1) return;
  __syncthreads();
  const double n1 = vn1[j];
  if (n1 == 0.0) return;
  double temp = fabs(x[i]) / n1;
  temp = fmax(0.0, (1.0 + temp) * (1.0 - temp));
  const double r2 = n1 / vn2[j];
  const double temp2 = temp * r2 * r2;
  if (temp2 <= sqrt(0.5 * DBL_EPSILON)) {  // recompute: LAPACK tol3z = sqrt(dlamch(E)), E = eps/2
    double s = 0.0;
    for (int r = i + 1 + threadIdx.x; r < M; r += blockDim.x) s += x[r] * x[r];
    s = block_sum_q(s, sh);
    if (threadIdx.x == 0) vn1[j] = vn2[j] = sqrt(s);
  } else if (threadIdx.x == 0) {
    vn1[j] = n1 * sqrt(temp);
  }
}

// rank (Eigen's threshold) and back substitution of the basic solution, one CTA per component
__global__ void __launch_bounds__(kQT) k_qr_backsolve(const double* __restrict__ A, int M, int N,
                                                      const double* __restrict__ B, const int* __restrict__ jpvt,
                                                      double* __restrict__ W, int* __restrict__ rank_out) {
  extern __shared__ double z[];
  __shared__ double sh[32];
  __shared__ int rk;
  const int comp = blockIdx.x;
  const int kd = min(M, N);
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int q = 0; q < kd; ++q) mx = fmax(mx, fabs(A[q + static_cast<long long>(q) * M]));
    const double thr = mx * (DBL_EPSILON * kd);
    int r = 0;
    for (int q = 0; q < kd; ++q) r += fabs(A[q + static_cast<long long>(q) * M]) > thr;
    rk = r;
    if (comp == 0) *rank_out = r;
  }
  __syncthreads();
  const int rank = rk;
  const double* b = B + static_cast<long long>(comp) * M;
  for (int q = rank - 1; q >= 0; --q) {
    double s = 0.0;
    for (int c = q + 1 + threadIdx.x; c < rank; c += blockDim.x) s += A[q + static_cast<long long>(c) * M] * z[c];
    s = block_sum_q(s, sh);
    if (threadIdx.x == 0) z[q] = (b[q] - s) / A[q + static_cast<long long>(q) * M];
    __syncthreads();
  }
  double* w = W + static_cast<long long>(comp) * N;
  for (int q = threadIdx.x; q < N; q += blockDim.x) w[q] = 0.0;
  __syncthreads();
  for (int q = threadIdx.x; q < rank; q += blockDim.x) w[jpvt[q]] = z[q];
}

__global__ void k_iota(int* x, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = i;
}
__global__ void k_unscale(double* __restrict__ W, const double* __restrict__ s, int n, int C) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(n) * C;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    W[e] /= s[e % n];
}

}  // namespace

// W (p x C) = argmin ‖H W - F‖ by column-pivoted QR, then W ./= scales (runner.hpp:247-250)
void qr_solve_dev(Ctx& c) {
  ScopedKernelTimer tk(c, "qr");
  const int M = c.N, N = c.p, C = c.C;
  const size_t dense = static_cast<size_t>(M) * N;
  if (dense * sizeof(double) > device_available(c) / 2)
    throw std::runtime_error("qr_direct: dense H (" + std::to_string(dense * 8 / (1 << 20)) + " MiB) does not fit");
  double* D = c.ws("qr.H", dense);
  RDD_CUDA(cudaMemsetAsync(D, 0, dense * sizeof(double), c.stream));
  k_densify<<<dim3(32, c.J), 256, 0, c.stream>>>(c.H, c.dH_off.p, c.row_ptr.p, c.row_idx.p, c.dcol_off.p, M, D);
  RDD_LAUNCH_CHECK();
  double* B = c.ws("qr.F", static_cast<size_t>(M) * C);
  RDD_CUDA(cudaMemcpyAsync(B, c.F.p, sizeof(double) * M * C, cudaMemcpyDeviceToDevice, c.stream));
  DBuf<double> vn1, vn2, tau;
  DBuf<int> jpvt, rank;
  vn1.ensure(N);
  vn2.ensure(N);
  tau.ensure(std::max(1, std::min(M, N)));
  jpvt.ensure(N);
  rank.ensure(1);
  k_iota<<<ceil_div(N, 256), 256, 0, c.stream>>>(jpvt.p, N);
  RDD_LAUNCH_CHECK();
  k_colnorms<<<N, 256, 0, c.stream>>>(D, M, N, vn1.p, vn2.p);
  RDD_LAUNCH_CHECK();
  const int kd = std::min(M, N);
  for (int i = 0; i < kd; ++i) {
    k_qr_pivot<<<1, kQT, 0, c.stream>>>(D, M, N, i, vn1.p, vn2.p, jpvt.p, tau.p);
    RDD_LAUNCH_CHECK();
    if (i + 1 < N) {
      k_qr_apply<<<N - i - 1, kQT, 0, c.stream>>>(D, M, i, tau.p, D, M, i + 1, N, vn1.p, vn2.p);
      RDD_LAUNCH_CHECK();
    }
    k_qr_apply<<<C, kQT, 0, c.stream>>>(D, M, i, tau.p, B, M, 0, C, nullptr, nullptr);  // Qᵀ F
    RDD_LAUNCH_CHECK();
  }
  c.W.ensure(static_cast<size_t>(N) * C);
  const size_t sm = static_cast<size_t>(std::max(1, kd)) * sizeof(double);
  if (sm > 32 * 1024)
    RDD_CUDA(cudaFuncSetAttribute(k_qr_backsolve, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
  k_qr_backsolve<<<C, kQT, sm, c.stream>>>(D, M, N, B, jpvt.p, c.W.p, rank.p);
  RDD_LAUNCH_CHECK();
  k_unscale<<<256, 256, 0, c.stream>>>(c.W.p, c.scales.p, N, C);
  RDD_LAUNCH_CHECK();
  rank.download(&c.qr_rank, 1, c.stream);
  RDD_CUDA(cudaStreamSynchronize(c.stream));
  c.hist.assign(C, {});
  c.true_hist.assign(C, {});
  c.iters.assign(C, 0);
  c.conv.assign(C, 1);
  c.brk.assign(C, 0);
}

}  // namespace rdd
